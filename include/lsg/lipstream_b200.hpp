// lipstream_b200.hpp -- C++ drop-ins for the reference's hot-path operators,
// implemented over the C ABI in lsg.h (header-only; link liblsg.so).
//
// Same class/function names, argument meaning and exception types as the
// reference (paths relative to /root/reference/proj/core/include/lipstream/):
//   Segmenter, SegmenterConfig, RawSegment, BoundaryScorer  (segmenter.hpp:11-111)
//   VadConfig, PeakMode                                      (vad.hpp:13-24)
//   MelConfig, MelSpectrogram, compute_mel, mel_frame_count  (mel.hpp:12-39)
//   AudioBuffer                                              (audio.hpp:12-20)
//   LipsyncRender + the generator-backed lip-sync stage      (visual_mocks.hpp:33-43)
// so a reference call site switches by changing the namespace
// (lipstream:: -> lipstream_b200::).  All compute runs on the GPU; the host
// keeps only the per-stream sample bookkeeping a RawSegment::audio needs and,
// when a BoundaryScorer is attached, the integer state machine (the scorer is
// a host callback by contract, segmenter.cpp:84-90).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <map>
#include <memory>
#include <tuple>
#include <stdexcept>
#include <string>
#include <vector>

#include "lsg.h"

namespace lipstream_b200 {

using Timestamp = std::int64_t;
using DurationMs = std::int64_t;

inline void check(lsg_status s) {
  if (s == LSG_OK) return;
  const std::string m = lsg_last_error();
  if (s == LSG_EINVAL) throw std::invalid_argument(m);
  if (s == LSG_ELOGIC) throw std::logic_error(m);
  throw std::runtime_error(m);
}

struct AudioBuffer {
  std::vector<std::int16_t> samples;
  int sample_rate = 16000;
  Timestamp start = 0;
  DurationMs duration_ms() const {  // audio.cpp:8-12
    return static_cast<DurationMs>(std::llround(1000.0 * double(samples.size()) / sample_rate));
  }
  Timestamp end() const { return start + duration_ms(); }
  bool empty() const { return samples.empty(); }
};

// One GPU (device + stream).  A process-wide default context per device.
class Context {
 public:
  explicit Context(int device = 0) { check(lsg_ctx_create(device, &h_)); }
  ~Context() { lsg_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  lsg_ctx handle() const { return h_; }
  static Context& default_context() {
    static Context c(0);
    return c;
  }

 private:
  lsg_ctx h_ = nullptr;
};

// ----------------------------------------------------------------- VAD / seg
enum class PeakMode { Decay, MaxHold, Absolute };

struct VadConfig {
  PeakMode peak_mode = PeakMode::Decay;
  double peak_half_life_ms = 10000.0;
  double speech_threshold_db = -40.0;
  DurationMs frame_ms = 20;
};

enum class CutCause { Pause, Forced, Eos };

struct RawSegment {
  Timestamp begin = 0;
  Timestamp end = 0;
  AudioBuffer audio;
  double confidence = 1.0;
  CutCause cause = CutCause::Eos;
  DurationMs duration_ms() const { return end - begin; }
};

struct BoundaryContext {
  Timestamp pause_start = 0;
  DurationMs silence_run_ms = 0;
  DurationMs segment_span_ms = 0;
};

struct BoundaryDecision {
  bool cut = true;
  double confidence = 1.0;
  double cost_ms = 0.0;
};

class BoundaryScorer {
 public:
  virtual ~BoundaryScorer() = default;
  virtual BoundaryDecision score(const BoundaryContext& ctx) = 0;
};

enum class SegmenterMode { Baseline, Semantic };

struct SegmenterConfig {
  SegmenterMode mode = SegmenterMode::Semantic;
  VadConfig vad;
  DurationMs min_silence_ms = 500;
  DurationMs min_segment_ms = 1500;
  DurationMs max_segment_ms = 10000;
  int sample_rate = 16000;
};

struct SegmenterMetrics {
  std::int64_t frames = 0;
  std::int64_t speech_frames = 0;
  std::int64_t cuts_pause = 0;
  std::int64_t cuts_forced = 0;
  std::int64_t cuts_eos = 0;
  std::int64_t scorer_calls = 0;
  double scorer_cost_ms = 0.0;
};

// Drop-in for lipstream::Segmenter (segmenter.hpp:76-111).
class Segmenter {
 public:
  explicit Segmenter(SegmenterConfig cfg, BoundaryScorer* scorer = nullptr,
                     Context& ctx = Context::default_context(), std::int64_t max_push_samples = 1 << 22)
      : cfg_(cfg), scorer_(scorer) {
    lsg_seg_cfg c{};
    c.mode = cfg.mode == SegmenterMode::Baseline ? 0 : 1;
    c.peak_mode = static_cast<int32_t>(cfg.vad.peak_mode);
    c.peak_half_life_ms = cfg.vad.peak_half_life_ms;
    c.speech_threshold_db = cfg.vad.speech_threshold_db;
    c.frame_ms = cfg.vad.frame_ms;
    c.min_silence_ms = cfg.min_silence_ms;
    c.min_segment_ms = cfg.min_segment_ms;
    c.max_segment_ms = cfg.max_segment_ms;
    c.sample_rate = cfg.sample_rate;
    c.flags_only = scorer ? 1 : 0;
    check(lsg_seg_create(ctx.handle(), &c, 1, max_push_samples, &h_));
    fs_ = std::int64_t(cfg.sample_rate) * cfg.vad.frame_ms / 1000;
  }
  ~Segmenter() { lsg_seg_destroy(h_); }
  Segmenter(const Segmenter&) = delete;
  Segmenter& operator=(const Segmenter&) = delete;

  std::vector<RawSegment> push(const AudioBuffer& chunk) {
    return push(chunk.samples.data(), static_cast<std::int64_t>(chunk.samples.size()), chunk.sample_rate,
                chunk.start);
  }
  // The same push over a borrowed host buffer (no AudioBuffer copy): what
  // the reference-typed adapter (integration/lipstream_gpu.cpp) calls.
  std::vector<RawSegment> push(const std::int16_t* samples, std::int64_t n, int sample_rate, Timestamp start) {
    const int32_t sid = 0;
    const int16_t* ptr = samples;
    const int64_t st = start;
    check(lsg_seg_push(h_, 1, &sid, &ptr, &n, &st, sample_rate, 0));
    std::vector<RawSegment> out;
    if (n == 0) return out;
    if (!started_) {
      started_ = true;
      base_ = seg_start_ = start;
    }
    pending_.insert(pending_.end(), samples, samples + n);
    if (!scorer_) return materialise();
    std::vector<uint8_t> flags = take_flags();
    for (uint8_t f : flags) process_frame(f != 0, out);
    return out;
  }

  std::vector<RawSegment> finish() {
    const int32_t sid = 0;
    check(lsg_seg_finish(h_, 1, &sid));
    if (!scorer_) return materialise();
    std::vector<RawSegment> out;  // segmenter.cpp:120-145 on the host state
    const std::int64_t stage = emitted_ + std::int64_t(pending_.size()) - consumed_ * fs_;
    const DurationMs tail_ms = stage * 1000 / cfg_.sample_rate;
    if (!speech_seen_ || pending_.empty()) {
      pending_.clear();
      return out;
    }
    RawSegment seg;
    seg.begin = seg_start_;
    seg.end = base_ + consumed_ * cfg_.vad.frame_ms + tail_ms;
    seg.audio.sample_rate = cfg_.sample_rate;
    seg.audio.start = seg_start_;
    seg.audio.samples = std::move(pending_);
    pending_.clear();
    out.push_back(std::move(seg));
    host_.cuts_eos += 1;
    return out;
  }

  const SegmenterMetrics& metrics() const {
    lsg_seg_metrics m{};
    check(lsg_seg_get_metrics(h_, 0, &m));
    metrics_.frames = m.frames;
    metrics_.speech_frames = m.speech_frames;
    if (scorer_) {
      metrics_.cuts_pause = host_.cuts_pause;
      metrics_.cuts_forced = host_.cuts_forced;
      metrics_.cuts_eos = host_.cuts_eos;
      metrics_.scorer_calls = host_.scorer_calls;
      metrics_.scorer_cost_ms = host_.scorer_cost_ms;
    } else {
      metrics_.cuts_pause = m.cuts_pause;
      metrics_.cuts_forced = m.cuts_forced;
      metrics_.cuts_eos = m.cuts_eos;
    }
    return metrics_;
  }

 private:
  std::vector<RawSegment> materialise() {
    int64_t n = 0;
    check(lsg_seg_take_cuts(h_, 0, nullptr, 0, &n));
    std::vector<lsg_cut> cuts(static_cast<size_t>(n));
    check(lsg_seg_take_cuts(h_, 0, cuts.data(), n, &n));
    std::vector<RawSegment> out;
    for (const lsg_cut& c : cuts) {
      RawSegment s;
      s.begin = c.begin;
      s.end = c.end;
      s.confidence = c.confidence;
      s.cause = static_cast<CutCause>(c.cause);
      s.audio.sample_rate = cfg_.sample_rate;
      s.audio.start = c.begin;
      s.audio.samples.assign(pending_.begin(), pending_.begin() + c.sample_len);
      pending_.erase(pending_.begin(), pending_.begin() + c.sample_len);
      out.push_back(std::move(s));
    }
    return out;
  }

  std::vector<uint8_t> take_flags() {
    int64_t n = 0;
    check(lsg_seg_take_flags(h_, 0, nullptr, 0, &n));
    std::vector<uint8_t> f(static_cast<size_t>(n));
    check(lsg_seg_take_flags(h_, 0, f.data(), n, &n));
    return f;
  }

  void emit_cut(Timestamp cut_ms, double conf, CutCause cause, std::vector<RawSegment>& out) {
    const auto split = static_cast<std::size_t>((cut_ms - seg_start_) * cfg_.sample_rate / 1000);
    RawSegment seg;
    seg.begin = seg_start_;
    seg.end = cut_ms;
    seg.confidence = conf;
    seg.cause = cause;
    seg.audio.sample_rate = cfg_.sample_rate;
    seg.audio.start = seg_start_;
    seg.audio.samples.assign(pending_.begin(), pending_.begin() + std::ptrdiff_t(split));
    pending_.erase(pending_.begin(), pending_.begin() + std::ptrdiff_t(split));
    emitted_ += std::int64_t(split);
    out.push_back(std::move(seg));
    seg_start_ = cut_ms;
    speech_seen_ = false;
  }

  // process_frame (segmenter.cpp:51-99) over a GPU VAD decision.
  void process_frame(bool speech, std::vector<RawSegment>& out) {
    const Timestamp f0 = base_ + consumed_ * cfg_.vad.frame_ms;
    const Timestamp f1 = f0 + cfg_.vad.frame_ms;
    if (speech) {
      if (speech_seen_ && silence_run_ >= cfg_.min_silence_ms && candidate_open_ && candidate_cut_) {
        emit_cut(pause_start_ + silence_run_ / 2, candidate_confidence_, CutCause::Pause, out);
        host_.cuts_pause += 1;
      }
      silence_run_ = 0;
      candidate_open_ = false;
      candidate_cut_ = false;
      speech_seen_ = true;
    } else {
      if (silence_run_ == 0) pause_start_ = f0;
      silence_run_ += cfg_.vad.frame_ms;
      if (!candidate_open_ && silence_run_ >= cfg_.min_silence_ms && speech_seen_) {
        candidate_open_ = true;
        candidate_cut_ = true;
        candidate_confidence_ = 1.0;
        if (cfg_.mode == SegmenterMode::Semantic) {
          if (pause_start_ - seg_start_ < cfg_.min_segment_ms) {
            candidate_cut_ = false;
          } else if (scorer_) {
            BoundaryDecision d = scorer_->score({pause_start_, silence_run_, pause_start_ - seg_start_});
            host_.scorer_calls += 1;
            host_.scorer_cost_ms += d.cost_ms;
            candidate_cut_ = d.cut;
            candidate_confidence_ = d.confidence;
          }
        }
      }
    }
    if (cfg_.mode == SegmenterMode::Semantic && speech_seen_ && f1 - seg_start_ >= cfg_.max_segment_ms) {
      emit_cut(f1, 1.0, CutCause::Forced, out);
      host_.cuts_forced += 1;
    }
    consumed_ += 1;
  }

  SegmenterConfig cfg_;
  BoundaryScorer* scorer_;
  lsg_seg h_ = nullptr;
  std::int64_t fs_ = 320;
  std::vector<std::int16_t> pending_;
  mutable SegmenterMetrics metrics_;
  SegmenterMetrics host_;
  bool started_ = false;
  Timestamp base_ = 0, seg_start_ = 0, pause_start_ = 0;
  std::int64_t consumed_ = 0, emitted_ = 0;
  DurationMs silence_run_ = 0;
  bool speech_seen_ = false, candidate_open_ = false, candidate_cut_ = false;
  double candidate_confidence_ = 1.0;
};

// ---------------------------------------------------------------------- mel
struct MelConfig {
  int sample_rate = 16000;
  int fft_size = 1024;
  int hop = 256;
  int n_mels = 80;
  double fmin = 0.0;
  double fmax = 8000.0;
};

struct MelSpectrogram {
  std::int64_t n_frames = 0;
  int n_mels = 0;
  std::vector<float> data;
  float at(std::int64_t frame, int mel) const { return data[static_cast<std::size_t>(frame) * n_mels + mel]; }
};

inline lsg_mel_cfg to_c(const MelConfig& c) {
  lsg_mel_cfg m{};
  m.sample_rate = c.sample_rate;
  m.fft_size = c.fft_size;
  m.hop = c.hop;
  m.n_mels = c.n_mels;
  m.fmin = c.fmin;
  m.fmax = c.fmax;
  return m;
}

inline std::int64_t mel_frame_count(std::int64_t n_samples, const MelConfig& cfg = {}) {
  lsg_mel_cfg c = to_c(cfg);
  int64_t f = 0;
  check(lsg_mel_frames(n_samples, &c, &f));
  return f;
}

// compute_mel (mel.hpp:39) with the tables built once: a reusable handle.
class MelExtractor {
 public:
  explicit MelExtractor(const MelConfig& cfg = {}, std::int64_t max_frames = 1 << 16,
                        Context& ctx = Context::default_context())
      : cfg_(cfg) {
    lsg_mel_cfg c = to_c(cfg);
    check(lsg_mel_create(ctx.handle(), &c, max_frames, &h_));
    max_frames_ = max_frames;
  }
  ~MelExtractor() { lsg_mel_destroy(h_); }
  MelExtractor(const MelExtractor&) = delete;
  MelExtractor& operator=(const MelExtractor&) = delete;
  MelSpectrogram operator()(const AudioBuffer& audio) const { return (*this)(audio.samples.data(), audio.samples.size()); }
  MelSpectrogram operator()(const std::int16_t* samples, std::size_t n) const {
    MelSpectrogram m;
    m.n_mels = cfg_.n_mels;
    m.n_frames = mel_frame_count(std::int64_t(n), cfg_);
    m.data.resize(static_cast<std::size_t>(m.n_frames) * cfg_.n_mels);
    int64_t f = 0;
    if (m.n_frames) check(lsg_mel_compute(h_, samples, int64_t(n), m.data.data(), &f));
    return m;
  }
  std::int64_t max_frames() const { return max_frames_; }

 private:
  MelConfig cfg_;
  lsg_mel h_ = nullptr;
  std::int64_t max_frames_ = 0;
};

// Drop-in for compute_mel (mel.hpp:39): pure and re-entrant like the
// reference; each host thread keeps one extractor per config (tables built
// once, device buffers grown to the longest buffer seen), so the hot path
// does not allocate.
inline MelSpectrogram compute_mel(const std::int16_t* samples, std::size_t n, const MelConfig& cfg = {}) {
  const std::int64_t f = mel_frame_count(std::int64_t(n), cfg);
  using Key = std::tuple<int, int, int, int, double, double>;
  thread_local std::map<Key, std::unique_ptr<MelExtractor>> cache;
  auto& ext = cache[Key{cfg.sample_rate, cfg.fft_size, cfg.hop, cfg.n_mels, cfg.fmin, cfg.fmax}];
  if (!ext || ext->max_frames() < f) ext = std::make_unique<MelExtractor>(cfg, std::max<std::int64_t>(f, 1 << 12));
  return (*ext)(samples, n);
}
inline MelSpectrogram compute_mel(const AudioBuffer& audio, const MelConfig& cfg = {}) {
  return compute_mel(audio.samples.data(), audio.samples.size(), cfg);
}

// Drop-in for fft_radix2 (mel.hpp:42): the GPU transform, bit-identical to
// the reference (lsg_fft_radix2); std::invalid_argument on a bad size.
inline void fft_radix2(std::vector<std::complex<double>>& buf, Context& ctx = Context::default_context()) {
  check(lsg_fft_radix2(ctx.handle(), reinterpret_cast<double*>(buf.data()), std::int64_t(buf.size()), 1));
}

// ------------------------------------------------------------------ lipsync
struct LipsyncRender {
  std::int64_t frames = 0;
  std::int64_t cost_us = 0;  // measured device time of the render, microseconds
};

// The lip-sync stage with the generator behind it: validates the pair the
// way mock_lipsync does (visual_mocks.cpp:40-51), then renders.
inline void validate_lipsync(DurationMs audio_span_ms, DurationMs frame_span_ms, std::int64_t n_frames) {
  check(lsg_lipsync_validate(audio_span_ms, frame_span_ms, n_frames));
}

enum class Precision {
  BF16 = LSG_PREC_BF16,
  FP16 = LSG_PREC_FP16,
  FP8_TAIL = LSG_PREC_FP8_TAIL,    // 8-bit: need a CalibrationBatch
  INT8_TAIL = LSG_PREC_INT8_TAIL,  //
};

// Device-resident inputs of a calibration forward (the 8-bit precisions'
// per-tensor activation ranges come from an fp16 forward over them; pick
// frames from the distribution the stage will render).  Same layouts as
// LipsyncStage::render / lsg_gen_forward.
struct CalibrationBatch {
  const float* mel_rows = nullptr;
  const std::int32_t* chunk_row = nullptr;
  const std::uint8_t* target = nullptr;
  const std::uint8_t* refs = nullptr;
  const std::int32_t* ref_index = nullptr;
  std::int32_t frames = 0;
};

// The lip-sync stage with mock_lipsync's contract (visual_mocks.hpp:32-43):
// validate the pair exactly as mock_lipsync does, render every frame through
// the Wav2Lip generator on the GPU, return LipsyncRender{frames, cost_us}
// with cost_us the measured render time instead of the profile's charge.
// render() takes the segment's device-resident inputs (mel rows, each frame's
// 16-row chunk start, face crops, reference crop -- e.g. resolved from a
// DeviceRegistry); render_placeholder() renders n frames of a fixed
// synthetic input for callers that, like the reference's StageFn, hold only
// spans and a frame count.  Weights: a host fp32 blob (lsg_gen_param_count
// floats, BN folded).
class LipsyncStage {
 public:
  LipsyncStage(const std::vector<float>& weights, int max_batch = 128, Precision prec = Precision::FP16,
               Context& ctx = Context::default_context(), const CalibrationBatch* calib = nullptr)
      : ctx_(ctx), max_batch_(max_batch) {
    if (prec != Precision::FP8_TAIL && prec != Precision::INT8_TAIL) {
      check(lsg_gen_create(ctx.handle(), weights.data(), std::int64_t(weights.size()), int32_t(prec), max_batch, &g_));
      return;
    }
    if (!calib || calib->frames <= 0) throw std::invalid_argument("LipsyncStage: 8-bit precisions need a calibration batch");
    // ranges from an fp16 forward over the calibration frames (lsg_gen_calibrate)
    lsg_gen c = nullptr;
    check(lsg_gen_create(ctx.handle(), weights.data(), std::int64_t(weights.size()), LSG_PREC_FP16, calib->frames, &c));
    std::int32_t n = 0;
    lsg_status st = lsg_gen_calibrate(c, calib->mel_rows, calib->chunk_row, calib->target, calib->refs,
                                      calib->ref_index, calib->frames, nullptr, 0, &n);
    std::vector<float> absmax(std::size_t(n > 0 ? n : 0));
    if (st == LSG_OK)
      st = lsg_gen_calibrate(c, calib->mel_rows, calib->chunk_row, calib->target, calib->refs, calib->ref_index,
                             calib->frames, absmax.data(), n, &n);
    if (st != LSG_OK) {  // the error text before the destroy can touch it
      const std::string m = lsg_last_error();
      lsg_gen_destroy(c);
      if (st == LSG_EINVAL) throw std::invalid_argument(m);
      throw std::runtime_error(m);
    }
    lsg_gen_destroy(c);
    check(lsg_gen_create_q(ctx.handle(), weights.data(), std::int64_t(weights.size()), int32_t(prec), absmax.data(),
                           n, max_batch, &g_));
  }
  ~LipsyncStage() {
    for (void* p : bufs_) lsg_dev_free(ctx_.handle(), p);
    lsg_gen_destroy(g_);
  }
  LipsyncStage(const LipsyncStage&) = delete;
  LipsyncStage& operator=(const LipsyncStage&) = delete;

  // All pointers [dev]; out [n][96][96][3] u8.  ref_index may be null (one
  // reference crop for the segment).
  LipsyncRender render(DurationMs audio_span_ms, DurationMs frame_span_ms, std::int64_t n_frames,
                       const float* mel_rows, const std::int32_t* chunk_row, const std::uint8_t* faces,
                       const std::uint8_t* ref, std::uint8_t* out) {
    validate_lipsync(audio_span_ms, frame_span_ms, n_frames);
    const auto t0 = std::chrono::steady_clock::now();
    const std::int32_t* ridx = zeros();
    for (std::int64_t b0 = 0; b0 < n_frames; b0 += max_batch_) {
      const int B = int(std::min<std::int64_t>(max_batch_, n_frames - b0));
      check(lsg_gen_forward(g_, mel_rows, chunk_row + b0, faces + b0 * kCrop, ref, ridx, out + b0 * kCrop,
                            LSG_OUT_U8_NHWC, B));
    }
    check(lsg_ctx_sync(ctx_.handle()));
    const auto us = std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0);
    return LipsyncRender{n_frames, std::int64_t(us.count())};
  }

  LipsyncRender render_placeholder(DurationMs audio_span_ms, DurationMs frame_span_ms, std::int64_t n_frames) {
    validate_lipsync(audio_span_ms, frame_span_ms, n_frames);
    if (!ph_mel_) make_placeholder();
    LipsyncRender r{0, 0};
    for (std::int64_t b0 = 0; b0 < n_frames; b0 += max_batch_) {
      const std::int64_t B = std::min<std::int64_t>(max_batch_, n_frames - b0);
      LipsyncRender p = render(audio_span_ms, frame_span_ms, std::max<std::int64_t>(B, 2), ph_mel_, ph_chunk_,
                               ph_faces_, ph_faces_, ph_out_);
      r.frames += B;
      r.cost_us += p.cost_us;
    }
    return r;
  }

 private:
  static constexpr std::int64_t kCrop = 96 * 96 * 3;
  void* dev(std::size_t bytes) {
    void* p = nullptr;
    check(lsg_dev_alloc(ctx_.handle(), bytes, &p));
    bufs_.push_back(p);
    return p;
  }
  const std::int32_t* zeros() {
    if (!zeros_) {
      std::vector<std::int32_t> z(std::size_t(max_batch_), 0);
      zeros_ = static_cast<std::int32_t*>(dev(z.size() * 4));
      check(lsg_copy(ctx_.handle(), zeros_, z.data(), z.size() * 4));
      check(lsg_ctx_sync(ctx_.handle()));
    }
    return zeros_;
  }
  void make_placeholder() {
    // 16 rows of log-mel silence (ln 1e-10), every frame on chunk 0, a
    // mid-grey crop with a darker lower half
    std::vector<float> mel(16 * 80, float(std::log(1e-10)));
    std::vector<std::int32_t> chunk(std::size_t(max_batch_), 0);
    std::vector<std::uint8_t> face(std::size_t(max_batch_) * kCrop);
    for (std::size_t i = 0; i < face.size(); ++i) face[i] = ((i / (96 * 3)) % 96) < 48 ? 150 : 90;
    ph_mel_ = static_cast<float*>(dev(mel.size() * 4));
    ph_chunk_ = static_cast<std::int32_t*>(dev(chunk.size() * 4));
    ph_faces_ = static_cast<std::uint8_t*>(dev(face.size()));
    ph_out_ = static_cast<std::uint8_t*>(dev(face.size()));
    check(lsg_copy(ctx_.handle(), ph_mel_, mel.data(), mel.size() * 4));
    check(lsg_copy(ctx_.handle(), ph_chunk_, chunk.data(), chunk.size() * 4));
    check(lsg_copy(ctx_.handle(), ph_faces_, face.data(), face.size()));
    check(lsg_ctx_sync(ctx_.handle()));
  }
  Context& ctx_;
  int max_batch_;
  lsg_gen g_ = nullptr;
  std::vector<void*> bufs_;
  std::int32_t* zeros_ = nullptr;
  float* ph_mel_ = nullptr;
  std::int32_t* ph_chunk_ = nullptr;
  std::uint8_t* ph_faces_ = nullptr;
  std::uint8_t* ph_out_ = nullptr;
};

// ---------------------------------------------- zero-copy stage hand-off
// device buffers keyed by (segment uuid, kind); stages pass
// 48-byte references instead of the payload bytes the reference's codecs copy
// (stage.cpp:176-301).  Errors: duplicate key / stale reference ->
// std::logic_error, arena exhausted -> std::runtime_error.
using DevRef = lsg_devref;

class DeviceRegistry {
 public:
  DeviceRegistry(std::int64_t arena_bytes, Context& ctx = Context::default_context()) {
    check(lsg_reg_create(ctx.handle(), arena_bytes, &h_));
  }
  ~DeviceRegistry() { lsg_reg_destroy(h_); }
  DeviceRegistry(const DeviceRegistry&) = delete;
  DeviceRegistry& operator=(const DeviceRegistry&) = delete;
  DevRef put(const std::uint8_t* uuid16, int kind, const void* src, std::int64_t bytes) {
    DevRef r{};
    check(lsg_reg_put(h_, uuid16, kind, src, bytes, &r));
    return r;
  }
  DevRef put_view(const std::uint8_t* uuid16, int kind, const void* dev_ptr, std::int64_t bytes) {
    DevRef r{};
    check(lsg_reg_put_view(h_, uuid16, kind, dev_ptr, bytes, &r));
    return r;
  }
  DevRef alloc(const std::uint8_t* uuid16, int kind, std::int64_t bytes, void** dev_ptr) {
    DevRef r{};
    check(lsg_reg_alloc(h_, uuid16, kind, bytes, dev_ptr, &r));
    return r;
  }
  void* resolve(const DevRef& r, std::int64_t* bytes = nullptr) const {
    void* p = nullptr;
    check(lsg_reg_resolve(h_, &r, &p, bytes));
    return p;
  }
  void retain(const DevRef& r) { check(lsg_reg_retain(h_, &r)); }
  void release(const DevRef& r) { check(lsg_reg_release(h_, &r)); }

 private:
  lsg_reg h_ = nullptr;
};

// AlignedPairMsg (stage.hpp:81-93) with its mel rows / face crops as device
// references; wire layout = encode_aligned_pair's (stage.cpp:243-257) under
// tag 0x105, then u32 count + 48-byte references.
inline constexpr std::uint32_t kTagAlignedPairRef = 0x105;

struct AlignedPairRefMsg {
  std::uint8_t uuid[16] = {};
  Timestamp birth = 0, begin = 0, end = 0;
  DurationMs source_duration_ms = 0, offset_ms = 0;
  bool low_confidence = false;
  std::int64_t n_frames = 0;
  Timestamp first_frame_ts = 0, last_frame_ts = 0;
  std::int64_t mel_frames = 0;
  std::vector<DevRef> refs;
};

inline std::vector<std::uint8_t> encode_aligned_pair_ref(const AlignedPairRefMsg& m) {
  std::vector<std::uint8_t> b;
  auto u32 = [&](std::uint32_t v) {
    for (int i = 0; i < 4; ++i) b.push_back(std::uint8_t(v >> (8 * i)));
  };
  auto i64 = [&](std::int64_t v) {
    for (int i = 0; i < 8; ++i) b.push_back(std::uint8_t(std::uint64_t(v) >> (8 * i)));
  };
  u32(kTagAlignedPairRef);
  b.insert(b.end(), m.uuid, m.uuid + 16);
  i64(m.birth), i64(m.begin), i64(m.end), i64(m.source_duration_ms), i64(m.offset_ms);
  b.push_back(m.low_confidence ? 1 : 0);
  i64(m.n_frames), i64(m.first_frame_ts), i64(m.last_frame_ts), i64(m.mel_frames);
  u32(std::uint32_t(m.refs.size()));
  for (const DevRef& r : m.refs) {
    std::uint8_t w[LSG_DEVREF_WIRE_BYTES];
    check(lsg_devref_encode(&r, w));
    b.insert(b.end(), w, w + LSG_DEVREF_WIRE_BYTES);
  }
  return b;
}

inline AlignedPairRefMsg decode_aligned_pair_ref(const std::vector<std::uint8_t>& b) {
  std::size_t pos = 0;
  auto need = [&](std::size_t n) {
    if (pos + n > b.size()) throw std::runtime_error("wire: truncated");
  };
  auto u32 = [&] {
    need(4);
    std::uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= std::uint32_t(b[pos + i]) << (8 * i);
    pos += 4;
    return v;
  };
  auto i64 = [&] {
    need(8);
    std::uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= std::uint64_t(b[pos + i]) << (8 * i);
    pos += 8;
    return std::int64_t(v);
  };
  const std::uint32_t tag = u32();
  if (tag != kTagAlignedPairRef)
    throw std::runtime_error("wire: expected tag " + std::to_string(kTagAlignedPairRef) + ", got " +
                             std::to_string(tag));
  AlignedPairRefMsg m;
  need(16);
  std::copy(b.begin() + std::ptrdiff_t(pos), b.begin() + std::ptrdiff_t(pos + 16), m.uuid);
  pos += 16;
  m.birth = i64(), m.begin = i64(), m.end = i64(), m.source_duration_ms = i64(), m.offset_ms = i64();
  need(1);
  m.low_confidence = b[pos++] != 0;
  m.n_frames = i64(), m.first_frame_ts = i64(), m.last_frame_ts = i64(), m.mel_frames = i64();
  const std::uint32_t n = u32();
  for (std::uint32_t i = 0; i < n; ++i) {
    need(LSG_DEVREF_WIRE_BYTES);
    DevRef r{};
    check(lsg_devref_decode(b.data() + pos, &r));
    pos += LSG_DEVREF_WIRE_BYTES;
    m.refs.push_back(r);
  }
  if (pos != b.size()) throw std::runtime_error("wire: trailing bytes");
  return m;
}

}  // namespace lipstream_b200
