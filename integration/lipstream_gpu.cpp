// lipstream_gpu.cpp -- the GPU hot path as LINK-LEVEL drop-ins for the
// reference's own symbols: compiled against the reference's unmodified
// headers (lipstream/segmenter.hpp, mel.hpp, visual_mocks.hpp), it defines
//
//   lipstream::Segmenter::Segmenter / push / finish   (segmenter.cpp:9-145)
//   lipstream::compute_mel, mel_frame_count, fft_radix2 (mel.cpp:40-127)
//   lipstream::mock_lipsync                             (visual_mocks.cpp:40-51)
//
// on top of include/lsg/lipstream_b200.hpp (the C ABI of liblsg.so).  Link it
// in place of segmenter.cpp (and with mel.cpp / visual_mocks.cpp compiled
// with those three / one symbols renamed, see integration/Makefile) and the
// reference's callers -- segment_audio (runner.cpp:44-54),
// Orchestrator::finish_pair's compute_mel (orchestrator.cpp:152), the
// lip-sync StageFn (runner.cpp:285-302), run_pipeline_input -- run on the
// GPU without a source change.  These are the to_b200 / from_b200
// conversions INTEGRATION.md describes, as code.
//
// Segmenter: the reference class's data members are fixed by its header, so
// each instance's GPU segmenter lives in a side table keyed by `this`
// (created in the constructor, released by finish(); a constructor at a
// reused address replaces a stale entry).  The members the header's inline
// accessors read are kept current: metrics_ (metrics()) and finished_.
#include <cstdlib>
#include <fstream>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <unordered_map>

#include "lipstream/mel.hpp"
#include "lipstream/segmenter.hpp"
#include "lipstream/visual_mocks.hpp"
#include "lsg/lipstream_b200.hpp"

namespace b2 = lipstream_b200;

namespace lipstream {
namespace {

// ------------------------------------------------------------ conversions
b2::SegmenterConfig to_b200(const SegmenterConfig& c) {
  b2::SegmenterConfig o;
  o.mode = c.mode == SegmenterMode::Baseline ? b2::SegmenterMode::Baseline : b2::SegmenterMode::Semantic;
  o.vad.peak_mode = static_cast<b2::PeakMode>(static_cast<int>(c.vad.peak_mode));
  o.vad.peak_half_life_ms = c.vad.peak_half_life_ms;
  o.vad.speech_threshold_db = c.vad.speech_threshold_db;
  o.vad.frame_ms = c.vad.frame_ms;
  o.min_silence_ms = c.min_silence_ms;
  o.min_segment_ms = c.min_segment_ms;
  o.max_segment_ms = c.max_segment_ms;
  o.sample_rate = c.sample_rate;
  return o;
}

b2::MelConfig to_b200(const MelConfig& c) {
  return b2::MelConfig{c.sample_rate, c.fft_size, c.hop, c.n_mels, c.fmin, c.fmax};
}

RawSegment from_b200(b2::RawSegment&& s) {
  RawSegment o;
  o.begin = s.begin;
  o.end = s.end;
  o.confidence = s.confidence;
  o.cause = static_cast<CutCause>(static_cast<int>(s.cause));
  o.audio.samples = std::move(s.audio.samples);
  o.audio.sample_rate = s.audio.sample_rate;
  o.audio.start = s.audio.start;
  return o;
}

std::vector<RawSegment> from_b200(std::vector<b2::RawSegment>&& v) {
  std::vector<RawSegment> out;
  out.reserve(v.size());
  for (auto& s : v) out.push_back(from_b200(std::move(s)));
  return out;
}

// The reference scorer behind the b200 scorer interface (called once per
// qualifying pause, in order: the host state machine runs in flags mode).
class ScorerBridge final : public b2::BoundaryScorer {
 public:
  explicit ScorerBridge(lipstream::BoundaryScorer* s) : s_(s) {}
  b2::BoundaryDecision score(const b2::BoundaryContext& c) override {
    const lipstream::BoundaryDecision d =
        s_->score(lipstream::BoundaryContext{c.pause_start, c.silence_run_ms, c.segment_span_ms});
    return b2::BoundaryDecision{d.cut, d.confidence, d.cost_ms};
  }

 private:
  lipstream::BoundaryScorer* s_;
};

struct GpuSegmenter {
  std::unique_ptr<ScorerBridge> bridge;
  std::unique_ptr<b2::Segmenter> seg;
};

std::mutex g_mu;
std::unordered_map<const Segmenter*, std::unique_ptr<GpuSegmenter>>& table() {
  static std::unordered_map<const Segmenter*, std::unique_ptr<GpuSegmenter>> t;
  return t;
}

GpuSegmenter& state_of(const Segmenter* s) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = table().find(s);
  if (it == table().end()) throw std::logic_error("segmenter: no GPU state (finished)");
  return *it->second;
}

void copy_metrics(const b2::SegmenterMetrics& m, SegmenterMetrics& o) {
  o.frames = m.frames;
  o.speech_frames = m.speech_frames;
  o.cuts_pause = m.cuts_pause;
  o.cuts_forced = m.cuts_forced;
  o.cuts_eos = m.cuts_eos;
  o.scorer_calls = m.scorer_calls;
  o.scorer_cost_ms = m.scorer_cost_ms;
}

}  // namespace

// ------------------------------------------------------------- Segmenter
// vad_ is the reference's VadTracker: constructing it runs the reference's
// own VAD config checks (vad.cpp:14-19) first, exactly as segmenter.cpp:9-10
// does; the GPU segmenter then applies segmenter.cpp:11-20's checks with the
// same messages.
Segmenter::Segmenter(SegmenterConfig cfg, BoundaryScorer* scorer)
    : cfg_(cfg), scorer_(scorer), vad_(cfg.vad), frame_samples_(0) {
  auto st = std::make_unique<GpuSegmenter>();
  if (scorer) st->bridge = std::make_unique<ScorerBridge>(scorer);
  st->seg = std::make_unique<b2::Segmenter>(to_b200(cfg), st->bridge.get());
  frame_samples_ = static_cast<std::size_t>(std::int64_t(cfg.sample_rate) * cfg.vad.frame_ms / 1000);
  std::lock_guard<std::mutex> lk(g_mu);
  table()[this] = std::move(st);
}

std::vector<RawSegment> Segmenter::push(const AudioBuffer& chunk) {
  if (finished_) throw std::logic_error("segmenter: push after finish");
  GpuSegmenter& g = state_of(this);
  auto out = from_b200(g.seg->push(chunk.samples.data(), std::int64_t(chunk.samples.size()), chunk.sample_rate,
                                   chunk.start));
  copy_metrics(g.seg->metrics(), metrics_);
  return out;
}

std::vector<RawSegment> Segmenter::finish() {
  if (finished_) throw std::logic_error("segmenter: finish twice");
  GpuSegmenter& g = state_of(this);
  auto out = from_b200(g.seg->finish());
  copy_metrics(g.seg->metrics(), metrics_);
  finished_ = true;
  std::lock_guard<std::mutex> lk(g_mu);
  table().erase(this);  // the GPU segmenter's workspaces go back now
  return out;
}

// ------------------------------------------------------------------- mel
std::int64_t mel_frame_count(std::int64_t n_samples, const MelConfig& cfg) {
  return b2::mel_frame_count(n_samples, to_b200(cfg));
}

MelSpectrogram compute_mel(const AudioBuffer& audio, const MelConfig& cfg) {
  // like the reference, the rate comes from cfg (mel.cpp:72-80 reads samples only)
  b2::MelSpectrogram m = b2::compute_mel(audio.samples.data(), audio.samples.size(), to_b200(cfg));
  MelSpectrogram o;
  o.n_frames = m.n_frames;
  o.n_mels = m.n_mels;
  o.data = std::move(m.data);
  return o;
}

void fft_radix2(std::vector<std::complex<double>>& buf) { b2::fft_radix2(buf); }

// --------------------------------------------------------------- lip-sync
// The StageFn (runner.cpp:285-302) passes spans and a frame count only, so
// the stage renders that many frames of its placeholder input through the
// generator; frames = n_frames as the reference reports, cost_us measured.
// Weights: the fp32 blob in $LSG_GEN_WEIGHTS (e.g. the library's calibrated
// synthetic weights written by tests/test_reference_pipeline_gpu.py), else
// deterministic He-normal weights.
namespace {
std::vector<float> stage_weights() {
  int64_t n = 0;
  b2::check(lsg_gen_param_count(&n));
  std::vector<float> w(static_cast<std::size_t>(n));
  if (const char* path = std::getenv("LSG_GEN_WEIGHTS")) {
    std::ifstream f(path, std::ios::binary);
    if (!f.read(reinterpret_cast<char*>(w.data()), std::streamsize(w.size() * 4)))
      throw std::runtime_error(std::string("lipsync: cannot read weights ") + path);
    return w;
  }
  int32_t info[12 * 64];
  int32_t nl = 0;
  b2::check(lsg_gen_layer_info(info, 64, &nl));
  std::mt19937_64 rng(0);
  std::size_t off = 0;
  for (int l = 0; l < nl; ++l) {
    const int* L = info + 12 * l;
    const double fan_in = double(L[1]) * L[3] * L[4] / (L[0] ? double(L[5]) * L[6] : 1.0);
    std::normal_distribution<float> d(0.f, float(std::sqrt(2.0 / fan_in)));
    const std::size_t nw = std::size_t(L[1]) * L[2] * L[3] * L[4];
    for (std::size_t i = 0; i < nw; ++i) w[off++] = d(rng);
    for (int c = 0; c < L[2]; ++c) w[off++] = 0.f;
  }
  return w;
}

b2::LipsyncStage& stage() {
  static b2::LipsyncStage s(stage_weights(), 128, b2::Precision::FP16);
  return s;
}
}  // namespace

LipsyncRender mock_lipsync(const LipsyncProfile& profile, DurationMs audio_span_ms, DurationMs frame_span_ms,
                           std::int64_t n_frames) {
  (void)profile;  // the profile names the cost model this render replaces
  const b2::LipsyncRender r = stage().render_placeholder(audio_span_ms, frame_span_ms, n_frames);
  LipsyncRender o;
  o.frames = r.frames;
  o.cost_us = r.cost_us;
  return o;
}

}  // namespace lipstream
