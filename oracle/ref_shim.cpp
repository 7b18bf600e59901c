// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// sources (lipstream::Segmenter, VadTracker, compute_mel, render_pattern,
// expected_segment_durations, the A/V alignment of align.cpp), compiled
// from /root/reference by
// oracle/Makefile into oracle/_ref/libref_lipstream.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the C restatement
// (lsg_oracle.c) and to generate tests/golden/, and by bench.py's
// --impl reference / cpu_baseline legs as the reference CPU path.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "lipstream/align.hpp"
#include "lipstream/kalman.hpp"
#include "lipstream/visual_mocks.hpp"
#include "lipstream/mel.hpp"
#include "lipstream/rng.hpp"
#include "lipstream/segmenter.hpp"
#include "lipstream/stage.hpp"
#include "lipstream/synth.hpp"
#include "lipstream/vad.hpp"

using namespace lipstream;

extern "C" {

struct ref_cut {
  int64_t begin, end;
  double confidence;
  int32_t cause;
  int32_t pad;
  int64_t sample_off, sample_len;
};

typedef void (*ref_scorer_fn)(void* user, int64_t pause_start, int64_t silence_run_ms,
                              int64_t segment_span_ms, int* cut, double* confidence,
                              double* cost_ms);

static int classify(const std::exception_ptr& e) {
  try {
    std::rethrow_exception(e);
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::logic_error&) {
    return 2;
  } catch (...) {
    return 3;
  }
}

static SpeechPattern make_pattern(int64_t lead, int nb, const int64_t* sp, const int64_t* pa,
                                  double hz, double amp) {
  SpeechPattern p;
  p.lead_silence_ms = lead;
  p.bursts.clear();
  for (int i = 0; i < nb; ++i) p.bursts.push_back({sp[i], pa[i]});
  p.tone_hz = hz;
  p.amplitude = amp;
  return p;
}

int ref_render_pattern(int64_t lead, int nb, const int64_t* sp, const int64_t* pa, double hz,
                       double amp, int64_t total_ms, int rate, int16_t* out, int64_t cap,
                       int64_t* n) {
  try {
    AudioBuffer a = render_pattern(make_pattern(lead, nb, sp, pa, hz, amp), total_ms, rate);
    *n = int64_t(a.samples.size());
    if (*n <= cap) std::memcpy(out, a.samples.data(), a.samples.size() * 2);
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

int ref_pattern_ends_in_speech(int64_t lead, int nb, const int64_t* sp, const int64_t* pa,
                               int64_t total_ms) {
  return pattern_ends_in_speech(make_pattern(lead, nb, sp, pa, 220.0, 0.3), total_ms) ? 1 : 0;
}

int ref_expected_durations(int64_t lead, int nb, const int64_t* sp, const int64_t* pa,
                           int64_t total_ms, int64_t min_sil, int64_t min_seg, int64_t max_seg,
                           int64_t* out, int64_t cap, int64_t* n) {
  try {
    auto d = expected_segment_durations(make_pattern(lead, nb, sp, pa, 220.0, 0.3), total_ms,
                                        min_sil, min_seg, max_seg);
    *n = int64_t(d.size());
    for (int64_t i = 0; i < *n && i < cap; ++i) out[i] = d[size_t(i)];
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

struct CScorer : BoundaryScorer {
  ref_scorer_fn fn;
  void* user;
  BoundaryDecision score(const BoundaryContext& c) override {
    int cut = 1;
    double conf = 1.0, cost = 0.0;
    fn(user, c.pause_start, c.silence_run_ms, c.segment_span_ms, &cut, &conf, &cost);
    return {cut != 0, conf, cost};
  }
};

// Whole-stream segmentation, optionally in random chunks of 37..4037 samples
// drawn exactly like segmenter_tests.cpp:24-58 (splitmix64 chunk_seed).
int ref_segment(const int16_t* pcm, int64_t n, int64_t start_ms, int mode, int peak_mode,
                double half_life, double thr, int64_t frame_ms, int64_t min_sil, int64_t min_seg,
                int64_t max_seg, int rate, uint64_t chunk_seed, ref_scorer_fn scorer,
                void* scorer_user, ref_cut* out, int64_t cap, int64_t* n_out,
                double* metrics /* 7: frames speech pause forced eos calls cost */) {
  try {
    SegmenterConfig cfg;
    cfg.mode = mode == 0 ? SegmenterMode::Baseline : SegmenterMode::Semantic;
    cfg.vad.peak_mode = PeakMode(peak_mode);
    cfg.vad.peak_half_life_ms = half_life;
    cfg.vad.speech_threshold_db = thr;
    cfg.vad.frame_ms = frame_ms;
    cfg.min_silence_ms = min_sil;
    cfg.min_segment_ms = min_seg;
    cfg.max_segment_ms = max_seg;
    cfg.sample_rate = rate;
    CScorer cs;
    cs.fn = scorer;
    cs.user = scorer_user;
    Segmenter seg(cfg, scorer ? &cs : nullptr);
    std::vector<RawSegment> got;
    auto add = [&](std::vector<RawSegment>&& v) {
      for (auto& s : v) got.push_back(std::move(s));
    };
    if (chunk_seed == 0) {
      AudioBuffer a;
      a.sample_rate = rate;
      a.start = start_ms;
      a.samples.assign(pcm, pcm + n);
      add(seg.push(a));
    } else {
      uint64_t state = chunk_seed;
      int64_t off = 0;
      while (off < n) {
        int64_t len = 37 + int64_t(splitmix64(state) % 4001);
        if (len > n - off) len = n - off;
        AudioBuffer c;
        c.sample_rate = rate;
        c.start = start_ms + off * 1000 / rate;
        c.samples.assign(pcm + off, pcm + off + len);
        add(seg.push(c));
        off += len;
      }
    }
    add(seg.finish());
    *n_out = int64_t(got.size());
    int64_t soff = 0;
    for (size_t i = 0; i < got.size(); ++i) {
      if (int64_t(i) < cap) {
        out[i].begin = got[i].begin;
        out[i].end = got[i].end;
        out[i].confidence = got[i].confidence;
        out[i].cause = int32_t(got[i].cause);
        out[i].pad = 0;
        out[i].sample_off = soff;
        out[i].sample_len = int64_t(got[i].audio.samples.size());
      }
      soff += int64_t(got[i].audio.samples.size());
    }
    if (metrics) {
      const auto& m = seg.metrics();
      metrics[0] = double(m.frames);
      metrics[1] = double(m.speech_frames);
      metrics[2] = double(m.cuts_pause);
      metrics[3] = double(m.cuts_forced);
      metrics[4] = double(m.cuts_eos);
      metrics[5] = double(m.scorer_calls);
      metrics[6] = m.scorer_cost_ms;
    }
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

// Per-frame VAD decisions of a whole stream (VadTracker::update per frame).
int ref_vad_frames(const int16_t* pcm, int64_t n, int peak_mode, double half_life, double thr,
                   int64_t frame_ms, int rate, uint8_t* speech, double* rms_db) {
  try {
    VadConfig v;
    v.peak_mode = PeakMode(peak_mode);
    v.peak_half_life_ms = half_life;
    v.speech_threshold_db = thr;
    v.frame_ms = frame_ms;
    VadTracker t(v);
    int64_t fs = int64_t(rate) * frame_ms / 1000;
    for (int64_t f = 0; (f + 1) * fs <= n; ++f) {
      auto r = t.update(pcm + f * fs, size_t(fs));
      speech[f] = r.speech ? 1 : 0;
      if (rms_db) rms_db[f] = r.rms_db;
    }
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

int64_t ref_mel_frame_count(int64_t n) { return mel_frame_count(n); }

int64_t ref_compute_mel(const int16_t* pcm, int64_t n, int rate, int fft, int hop, int n_mels,
                        double fmin, double fmax, float* out, int64_t cap) {
  try {
    MelConfig cfg;
    cfg.sample_rate = rate;
    cfg.fft_size = fft;
    cfg.hop = hop;
    cfg.n_mels = n_mels;
    cfg.fmin = fmin;
    cfg.fmax = fmax;
    AudioBuffer a;
    a.sample_rate = rate;
    a.samples.assign(pcm, pcm + n);
    MelSpectrogram m = compute_mel(a, cfg);
    if (int64_t(m.data.size()) <= cap)
      std::memcpy(out, m.data.data(), m.data.size() * sizeof(float));
    return m.n_frames;
  } catch (...) {
    return -1;
  }
}

int ref_fft(double* interleaved, int64_t n) {
  try {
    std::vector<std::complex<double>> b(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) b[size_t(i)] = {interleaved[2 * i], interleaved[2 * i + 1]};
    fft_radix2(b);
    for (int64_t i = 0; i < n; ++i) {
      interleaved[2 * i] = b[size_t(i)].real();
      interleaved[2 * i + 1] = b[size_t(i)].imag();
    }
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

int ref_write_mel(const char* path, const float* data, int64_t frames, int n_mels) {
  try {
    MelSpectrogram m;
    m.n_frames = frames;
    m.n_mels = n_mels;
    m.data.assign(data, data + frames * n_mels);
    write_mel(path, m);
    return 0;
  } catch (...) {
    return 3;
  }
}

uint64_t ref_splitmix64(uint64_t* state) { return splitmix64(*state); }
double ref_u64_to_unit(uint64_t v) { return u64_to_unit(v); }

// energy_envelope_ms (align.cpp:10-32); returns the length, writes when cap allows
int64_t ref_energy_envelope(const int16_t* pcm, int64_t n, int rate, double* out, int64_t cap) {
  AudioBuffer a;
  a.samples.assign(pcm, pcm + n);
  a.sample_rate = rate;
  std::vector<double> e = energy_envelope_ms(a);
  if ((int64_t)e.size() <= cap) std::memcpy(out, e.data(), e.size() * sizeof(double));
  return (int64_t)e.size();
}

// motion_envelope_ms (align.cpp:34-50) from frame (ts, mouth_motion) pairs
int ref_motion_envelope(const int64_t* ts, const double* motion, int64_t nf, int64_t t0, int64_t span, double* out) {
  try {
    std::vector<FrameRecord> fr((size_t)nf);
    for (int64_t i = 0; i < nf; ++i) {
      fr[(size_t)i].ts = ts[i];
      fr[(size_t)i].mouth_motion = motion[i];
    }
    std::vector<double> e = motion_envelope_ms(fr, t0, span);
    std::memcpy(out, e.data(), e.size() * sizeof(double));
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// mock_face_detect (visual_mocks.cpp:10-22): out = {cx, cy, w, h}
void ref_mock_face_detect(int64_t frame_index, uint64_t seed, double* out) {
  FaceBox b = mock_face_detect(frame_index, seed);
  out[0] = b.cx;
  out[1] = b.cy;
  out[2] = b.w;
  out[3] = b.h;
}

// The per-segment detect + smooth loop of orchestrator.cpp:115-129 /
// runner.cpp:134-141 over n frames: box = the frame's face (has_face[i]) or
// mock_face_detect(frame_index[i], seed); KalmanBoxFilter::update with
// dt = (ts - prev) / 1000 after the first.  out[4 i ..] = smoothed box,
// vel[2 i ..] = (vx, vy).  Returns -1 on a filter exception.
int ref_track_faces(const int64_t* ts, const int64_t* frame_index, const int* has_face, const double* faces,
                    int64_t n, uint64_t seed, double pn, double mn, double iv, double* out, double* vel) {
  try {
    KalmanConfig cfg;
    cfg.process_noise = pn;
    cfg.measurement_noise = mn;
    cfg.initial_variance = iv;
    KalmanBoxFilter smoother(cfg);
    int64_t prev = 0;
    for (int64_t i = 0; i < n; ++i) {
      FaceBox box;
      if (has_face[i]) box = FaceBox{faces[4 * i], faces[4 * i + 1], faces[4 * i + 2], faces[4 * i + 3]};
      else box = mock_face_detect(frame_index[i], seed);
      const double dt = smoother.initialized() ? double(ts[i] - prev) / 1000.0 : 0.0;
      const auto est = smoother.update(box, dt);
      out[4 * i] = est.box.cx;
      out[4 * i + 1] = est.box.cy;
      out[4 * i + 2] = est.box.w;
      out[4 * i + 3] = est.box.h;
      vel[2 * i] = est.vx;
      vel[2 * i + 1] = est.vy;
      prev = ts[i];
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// align_envelopes (align.cpp:52-116)
int ref_align_envelopes(const double* e, int64_t ne, const double* m, int64_t nm, int64_t max_lag, int64_t* offset,
                        double* corr, int* low) {
  try {
    AlignResult r = align_envelopes(std::vector<double>(e, e + ne), std::vector<double>(m, m + nm), max_lag);
    *offset = r.offset_ms;
    *corr = r.peak_corr;
    *low = r.low_confidence ? 1 : 0;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// Wire codecs of the path's stage messages (stage.cpp:176-301): encode into
// out (cap bytes, *n = size); decode back to fields.  -1 = the reference threw
// (wire: truncated / expected tag / trailing bytes), -2 = out too small.
static int copy_out(const WireBytes& b, uint8_t* out, int64_t cap, int64_t* n) {
  *n = (int64_t)b->size();
  if (*n > cap) return -2;
  std::memcpy(out, b->data(), b->size());
  return 0;
}
static Uuid to_uuid(const uint8_t* u) {
  Uuid x;
  std::memcpy(x.bytes.data(), u, 16);
  return x;
}

int ref_encode_segment(const uint8_t* uuid, int64_t birth, int64_t begin, int64_t end, double conf, int32_t rate,
                       const int16_t* s, int64_t ns, uint8_t* out, int64_t cap, int64_t* n) {
  SegmentMsg m;
  m.uuid = to_uuid(uuid);
  m.birth = birth;
  m.begin = begin;
  m.end = end;
  m.confidence = conf;
  m.audio.sample_rate = rate;
  m.audio.samples.assign(s, s + ns);
  return copy_out(encode_segment(m), out, cap, n);
}

int ref_decode_segment(const uint8_t* in, int64_t nin, int64_t* f3, double* conf, int32_t* rate, int16_t* s,
                       int64_t cap, int64_t* ns) {
  try {
    SegmentMsg m = decode_segment(std::vector<uint8_t>(in, in + nin));
    f3[0] = m.birth;
    f3[1] = m.begin;
    f3[2] = m.end;
    *conf = m.confidence;
    *rate = m.audio.sample_rate;
    *ns = (int64_t)m.audio.samples.size();
    if (*ns > cap) return -2;
    std::copy(m.audio.samples.begin(), m.audio.samples.end(), s);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// f9 = birth, begin, end, source_duration_ms, offset_ms, n_frames, first_frame_ts, last_frame_ts, mel_frames
int ref_encode_aligned_pair(const uint8_t* uuid, const int64_t* f9, int32_t low, uint8_t* out, int64_t cap,
                            int64_t* n) {
  AlignedPairMsg m;
  m.uuid = to_uuid(uuid);
  m.birth = f9[0];
  m.begin = f9[1];
  m.end = f9[2];
  m.source_duration_ms = f9[3];
  m.offset_ms = f9[4];
  m.low_confidence = low != 0;
  m.n_frames = f9[5];
  m.first_frame_ts = f9[6];
  m.last_frame_ts = f9[7];
  m.mel_frames = f9[8];
  return copy_out(encode_aligned_pair(m), out, cap, n);
}

int ref_decode_aligned_pair(const uint8_t* in, int64_t nin, uint8_t* uuid, int64_t* f9, int32_t* low) {
  try {
    AlignedPairMsg m = decode_aligned_pair(std::vector<uint8_t>(in, in + nin));
    std::memcpy(uuid, m.uuid.bytes.data(), 16);
    const int64_t v[9] = {m.birth, m.begin, m.end, m.source_duration_ms, m.offset_ms,
                          m.n_frames, m.first_frame_ts, m.last_frame_ts, m.mel_frames};
    std::copy(v, v + 9, f9);
    *low = m.low_confidence ? 1 : 0;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// f6 = birth, begin, end, source_duration_ms, frames_rendered, offset_ms
int ref_encode_final(const uint8_t* uuid, const int64_t* f6, uint8_t* out, int64_t cap, int64_t* n) {
  FinalMsg m;
  m.uuid = to_uuid(uuid);
  m.birth = f6[0];
  m.begin = f6[1];
  m.end = f6[2];
  m.source_duration_ms = f6[3];
  m.frames_rendered = f6[4];
  m.offset_ms = f6[5];
  return copy_out(encode_final(m), out, cap, n);
}

int ref_wire_tag(const uint8_t* in, int64_t nin, uint32_t* tag) {
  try {
    *tag = wire_tag(std::vector<uint8_t>(in, in + nin));
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
