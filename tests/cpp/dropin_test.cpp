// dropin_test.cpp -- the reference's own known-answer cases, run against the
// C++ drop-ins (include/lsg/lipstream_b200.hpp) on the GPU.  Mirrors
// proj/tests/segmenter_tests.cpp and media_tests.cpp of the reference.
// Built by tests/cpp/Makefile; run by tests/test_cpp_dropin.py (GPU).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "lsg/lipstream_b200.hpp"

using namespace lipstream_b200;

static int g_fail = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    if (!(c)) {                                                         \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++g_fail;                                                         \
    }                                                                   \
  } while (0)
template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

struct Burst {
  int64_t speech, pause;
};

static AudioBuffer pattern(int64_t lead, std::vector<Burst> b, int64_t total, double hz = 220.0, double amp = 0.3) {
  std::vector<int64_t> sp, pa;
  for (auto& x : b) {
    sp.push_back(x.speech);
    pa.push_back(x.pause);
  }
  AudioBuffer a;
  a.samples.resize(size_t(total * 16));
  int64_t n = 0;
  check(lsg_synth_pattern(lead, int32_t(b.size()), sp.data(), pa.data(), hz, amp, total, 16000, a.samples.data(),
                          int64_t(a.samples.size()), &n));
  a.samples.resize(size_t(n));
  return a;
}

static std::vector<RawSegment> segment_all(const AudioBuffer& a, SegmenterConfig cfg, size_t chunk = 0,
                                           BoundaryScorer* scorer = nullptr) {
  Segmenter seg(cfg, scorer);
  std::vector<RawSegment> out;
  if (chunk == 0) {
    out = seg.push(a);
  } else {
    for (size_t off = 0; off < a.samples.size(); off += chunk) {
      AudioBuffer c;
      c.start = a.start + int64_t(off) * 1000 / a.sample_rate;
      size_t e = std::min(a.samples.size(), off + chunk);
      c.samples.assign(a.samples.begin() + off, a.samples.begin() + e);
      auto part = seg.push(c);
      out.insert(out.end(), part.begin(), part.end());
    }
  }
  auto tail = seg.finish();
  out.insert(out.end(), tail.begin(), tail.end());
  return out;
}

static std::vector<int64_t> ends(const std::vector<RawSegment>& s) {
  std::vector<int64_t> e;
  for (auto& x : s) e.push_back(x.end);
  return e;
}

int main(int argc, char** argv) {
  const std::string golden_dir = argc > 1 ? argv[1] : "tests/golden";
  SegmenterConfig cfg;
  // segmenter_tests.cpp:140-151: chunk invariance, stock begins
  AudioBuffer stock = pattern(600, {{1400, 600}}, 8000);
  auto whole = segment_all(stock, cfg);
  CHECK(whole.size() == 4);
  if (whole.size() == 4) {
    CHECK(whole[0].begin == 0 && whole[1].begin == 2300 && whole[2].begin == 4300 && whole[3].begin == 6300);
  }
  for (size_t ch : {37u, 1000u, 4037u}) CHECK(ends(segment_all(stock, cfg, ch)) == ends(whole));
  size_t total = 0;
  for (auto& s : whole) {
    CHECK(s.audio.start == s.begin);
    CHECK(int64_t(s.audio.samples.size()) == s.duration_ms() * 16);
    total += s.audio.samples.size();
  }
  CHECK(total == stock.samples.size());
  // :153-163 pauses under the floor never cut
  auto shortp = segment_all(pattern(0, {{1000, 400}}, 6000), cfg);
  CHECK(shortp.size() == 1 && shortp[0].end == 6000 && shortp[0].cause == CutCause::Eos);
  // :165-182 continuous speech splits at the cap, only in semantic mode
  AudioBuffer cont = pattern(0, {{20000, 600}}, 12000);
  auto sem = segment_all(cont, cfg);
  CHECK(sem.size() == 2 && sem[0].end == 10000 && sem[0].cause == CutCause::Forced && sem[1].end == 12000);
  SegmenterConfig base = cfg;
  base.mode = SegmenterMode::Baseline;
  auto bl = segment_all(cont, base);
  CHECK(bl.size() == 1 && bl[0].end == 12000);
  // :184-198 baseline vs semantic fixture
  AudioBuffer fx = pattern(600, {{800, 600}}, 5600);
  CHECK((ends(segment_all(fx, base)) == std::vector<int64_t>{1700, 3100, 4500, 5600}));
  CHECK((ends(segment_all(fx, cfg)) == std::vector<int64_t>{3100, 5600}));
  // :200-230 scorer veto
  struct Scripted : BoundaryScorer {
    int calls = 0;
    BoundaryDecision score(const BoundaryContext& c) override {
      ++calls;
      CHECK(c.silence_run_ms >= 500);
      CHECK(c.segment_span_ms >= 1500);
      if (calls == 1) return {false, 0.0, 1.5};
      return {true, 0.7, 1.5};
    }
  } scorer;
  {
    Segmenter seg(cfg, &scorer);
    auto segs = seg.push(pattern(0, {{1600, 600}}, 6000));
    auto tail = seg.finish();
    segs.insert(segs.end(), tail.begin(), tail.end());
    CHECK(segs.size() == 2);
    if (segs.size() == 2) {
      CHECK(segs[0].end == 4100 && segs[0].confidence == 0.7 && segs[0].cause == CutCause::Pause);
      CHECK(segs[1].end == 6000);
    }
    CHECK(scorer.calls == 2);
    CHECK(seg.metrics().scorer_calls == 2);
    CHECK(std::fabs(seg.metrics().scorer_cost_ms - 3.0) < 1e-12);
  }
  // :232-239 silence only
  AudioBuffer silence;
  silence.samples.assign(16000 * 3, 0);
  CHECK(segment_all(silence, cfg).empty());
  // :241-256 stream discipline
  {
    Segmenter seg(cfg);
    AudioBuffer a = pattern(600, {{1400, 600}}, 1000);
    seg.push(a);
    AudioBuffer gap = a;
    gap.start = 5000;
    CHECK(throws<std::invalid_argument>([&] { seg.push(gap); }));
    AudioBuffer wrong = a;
    wrong.sample_rate = 8000;
    CHECK(throws<std::invalid_argument>([&] { seg.push(wrong); }));
    seg.finish();
    CHECK(throws<std::logic_error>([&] { seg.push(a); }));
    CHECK(throws<std::logic_error>([&] { seg.finish(); }));
  }
  // :258-269 broken configs
  {
    SegmenterConfig c = cfg;
    c.min_silence_ms = 0;
    CHECK(throws<std::invalid_argument>([&] { Segmenter s(c); }));
    c = cfg;
    c.max_segment_ms = c.min_segment_ms;
    CHECK(throws<std::invalid_argument>([&] { Segmenter s(c); }));
    c = cfg;
    c.sample_rate = 44100;
    CHECK(throws<std::invalid_argument>([&] { Segmenter s(c); }));
  }
  // media_tests.cpp:83-97 frame counts
  CHECK(mel_frame_count(1023) == 0 && mel_frame_count(1024) == 1 && mel_frame_count(1279) == 1 &&
        mel_frame_count(1280) == 2 && mel_frame_count(160000) == 622);
  // :99-117 440 Hz lands in band 11; :172-179 golden within 1e-4 rel
  AudioBuffer tone = pattern(0, {{1000, 0}}, 1000, 440.0);
  MelSpectrogram mel = compute_mel(tone);
  CHECK(mel.n_frames == 59 && mel.n_mels == 80);
  int arg = 0;
  std::vector<double> band(80, 0.0);
  for (int64_t f = 0; f < mel.n_frames; ++f)
    for (int b = 0; b < 80; ++b) band[size_t(b)] += mel.at(f, b);
  for (int b = 1; b < 80; ++b)
    if (band[size_t(b)] > band[size_t(arg)]) arg = b;
  CHECK(arg == 11);
  std::ifstream g(golden_dir + "/mel_golden.bin", std::ios::binary);
  uint32_t hdr[2] = {0, 0};
  g.read(reinterpret_cast<char*>(hdr), 8);
  std::vector<float> want(size_t(hdr[0]) * hdr[1]);
  g.read(reinterpret_cast<char*>(want.data()), std::streamsize(want.size() * 4));
  CHECK(g.good() && hdr[0] == 59 && hdr[1] == 80);
  size_t bad = 0;
  for (size_t i = 0; i < want.size() && i < mel.data.size(); ++i)
    if (std::fabs(mel.data[i] - want[i]) > 1e-4 * std::max(1.0, std::fabs(double(want[i])))) ++bad;
  CHECK(bad == 0);
  // :119-126 silence -> log floor
  AudioBuffer sil;
  sil.samples.assign(4096, 0);
  for (float v : compute_mel(sil).data) CHECK(v == float(std::log(1e-10)));
  // visual_mocks.cpp:43-46 lip-sync contract
  CHECK(throws<std::invalid_argument>([] { validate_lipsync(2000, 2020, 1); }));
  CHECK(throws<std::invalid_argument>([] { validate_lipsync(2000, 2400, 61); }));
  validate_lipsync(2000, 2020, 61);
  // zero-copy hand-off: mel into registry space, the pair
  // message carries the reference, the consumer resolves the same buffer
  {
    DeviceRegistry reg(1 << 20);
    std::uint8_t u[16];
    for (int i = 0; i < 16; ++i) u[i] = std::uint8_t(i * 7);
    void* mel_dev = nullptr;
    const std::int64_t bytes = mel.n_frames * 80 * 4;
    DevRef rm = reg.alloc(u, LSG_BUF_MEL, bytes, &mel_dev);
    CHECK(mel_dev != nullptr && rm.bytes == bytes && rm.kind == LSG_BUF_MEL);
    AlignedPairRefMsg m;
    std::copy(u, u + 16, m.uuid);
    m.end = 1000, m.n_frames = 25, m.mel_frames = mel.n_frames;
    m.refs.push_back(rm);
    const auto wire_bytes = encode_aligned_pair_ref(m);
    CHECK(wire_bytes.size() == 4 + 16 + 8 * 5 + 1 + 8 * 4 + 4 + LSG_DEVREF_WIRE_BYTES);
    const AlignedPairRefMsg back = decode_aligned_pair_ref(wire_bytes);
    std::int64_t nb = 0;
    CHECK(reg.resolve(back.refs.at(0), &nb) == mel_dev && nb == bytes && back.mel_frames == mel.n_frames);
    CHECK(throws<std::runtime_error>([&] {
      auto t = wire_bytes;
      t.pop_back();
      decode_aligned_pair_ref(t);
    }));
    CHECK(throws<std::logic_error>([&] { reg.put(u, LSG_BUF_MEL, mel.data.data(), 64); }));  // duplicate key
    reg.release(rm);
    CHECK(throws<std::logic_error>([&] { reg.resolve(rm); }));  // stale
    CHECK(throws<std::runtime_error>([&] {
      void* p = nullptr;
      reg.alloc(u, LSG_BUF_MEL, 2 << 20, &p);  // exhausted
    }));
  }
  // the lip-sync stage at 16 and 8 bits (weights: argv[2], a raw f32 blob
  // written by tests/test_cpp_dropin.py): an INT8 stage needs a calibration
  // batch, and calibrated on the frames it renders it lands within the
  // INT8 floor of the fp16 render
  if (argc > 2) {
    std::ifstream wf(argv[2], std::ios::binary | std::ios::ate);
    const std::streamsize nb = wf.tellg();
    std::vector<float> w(std::size_t(nb / 4));
    wf.seekg(0);
    wf.read(reinterpret_cast<char*>(w.data()), nb);
    CHECK(wf.good() && !w.empty());
    constexpr int B = 16, R = B + 16;
    std::vector<float> mel(std::size_t(R) * 80);
    for (std::size_t i = 0; i < mel.size(); ++i) mel[i] = float(-5.0 + 2.5 * std::sin(0.37 * double(i)));
    std::vector<std::int32_t> chunk(B), ridx(B, 0);
    for (int b = 0; b < B; ++b) chunk[b] = b;
    const std::size_t crop = 96 * 96 * 3;
    std::vector<std::uint8_t> faces(B * crop);
    for (std::size_t i = 0; i < faces.size(); ++i)
      faces[i] = std::uint8_t((i % crop) / (96 * 3) * 2 + (i / crop) * 3 + (i % 3) * 40);
    Context& ctx = Context::default_context();
    auto up = [&](const void* src, std::size_t bytes) {
      void* d = nullptr;
      check(lsg_dev_alloc(ctx.handle(), bytes, &d));
      check(lsg_copy(ctx.handle(), d, src, bytes));
      return d;
    };
    auto* d_mel = static_cast<float*>(up(mel.data(), mel.size() * 4));
    auto* d_chunk = static_cast<std::int32_t*>(up(chunk.data(), chunk.size() * 4));
    auto* d_ridx = static_cast<std::int32_t*>(up(ridx.data(), ridx.size() * 4));
    auto* d_faces = static_cast<std::uint8_t*>(up(faces.data(), faces.size()));
    std::uint8_t* d_out[2];
    for (auto& o : d_out) o = static_cast<std::uint8_t*>(up(faces.data(), faces.size()));
    check(lsg_ctx_sync(ctx.handle()));
    CHECK(throws<std::invalid_argument>([&] { LipsyncStage bad(w, B, Precision::INT8_TAIL); }));
    const CalibrationBatch cal{d_mel, d_chunk, d_faces, d_faces, d_ridx, B};
    {
      LipsyncStage f16(w, B, Precision::FP16);
      LipsyncStage i8(w, B, Precision::INT8_TAIL, ctx, &cal);
      CHECK(f16.render(640, 640, B, d_mel, d_chunk, d_faces, d_faces, d_out[0]).frames == B);
      CHECK(i8.render(640, 640, B, d_mel, d_chunk, d_faces, d_faces, d_out[1]).frames == B);
    }
    std::vector<std::uint8_t> o16(faces.size()), o8(faces.size());
    check(lsg_copy(ctx.handle(), o16.data(), d_out[0], o16.size()));
    check(lsg_copy(ctx.handle(), o8.data(), d_out[1], o8.size()));
    check(lsg_ctx_sync(ctx.handle()));
    double se = 0.0;
    for (std::size_t i = 0; i < o16.size(); ++i) se += (double(o16[i]) - o8[i]) * (double(o16[i]) - o8[i]);
    const double psnr = 10.0 * std::log10(255.0 * 255.0 / std::max(se / double(o16.size()), 1e-12));
    std::printf("INT8-tail stage vs fp16 stage: %.2f dB\n", psnr);
    CHECK(psnr >= 30.0);
    for (void* p : {(void*)d_mel, (void*)d_chunk, (void*)d_ridx, (void*)d_faces, (void*)d_out[0], (void*)d_out[1]})
      lsg_dev_free(ctx.handle(), p);
  }
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "all drop-in checks passed", g_fail);
  return g_fail ? 1 : 0;
}
