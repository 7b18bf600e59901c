// pipeline_driver.cpp -- runs the reference's own pipeline entry points and
// prints a canonical dump of everything they return, so the stock CPU build
// and the GPU build (reference sources + integration/lipstream_gpu.cpp) can
// be compared line by line (tests/test_reference_pipeline_gpu.py).
//
//   run_pipeline_input (runner.cpp:239-351) on synthetic_clip of the paper
//   scenario and four random_scenario seeds at 3/8/12/30 s: segment table,
//   segmenter metrics, orchestrator stats, every event (event_to_ndjson);
//   segment_audio's callers' known answers: stock 8 s begins {0, 2300, 4300,
//   6300} (segmenter_tests.cpp:140-151);
//   compute_mel on the 3 s stock clip split 2300 / 700 ms -> 140 / 40 frames
//   (pipeline_tests.cpp:417-418) -- in the GPU build also compared value by
//   value with the reference's CPU compute_mel linked under another name;
//   fft_radix2's media_tests.cpp:128-150 known answer.
#include <cinttypes>
#include <cmath>
#include <complex>
#include <cstdio>
#include <string>
#include <vector>

#include "lipstream/mel.hpp"
#include "lipstream/rng.hpp"
#include "lipstream/runner.hpp"
#include "lipstream/scenario.hpp"
#include "lipstream/segmenter.hpp"
#include "lipstream/synth.hpp"

using namespace lipstream;

#ifdef LSG_GPU_BUILD
namespace lipstream {
// mel.cpp compiled with -Dcompute_mel=ref_cpu_compute_mel (integration/Makefile)
MelSpectrogram ref_cpu_compute_mel(const AudioBuffer& audio, const MelConfig& cfg);
}  // namespace lipstream
#endif

static void dump_run(const char* tag, const Scenario& sc, DurationMs clip_ms) {
  const ClipInput in = synthetic_clip(sc, clip_ms);
  const ClipRunResult r = run_pipeline_input(sc, in, run_seed_for(sc.seed, clip_ms, 0));
  std::printf("run %s clip=%" PRId64 " segments=%zu completed=%" PRId64 " clip_latency=%" PRId64 "\n", tag, clip_ms,
              r.segments.size(), r.completed, r.clip_latency_ms);
  for (const auto& s : r.segments)
    std::printf("  seg %s %" PRId64 " %" PRId64 " dur=%" PRId64 " conf=%.17g forced=%d birth=%" PRId64
                " done=%" PRId64 " lat=%" PRId64 "\n",
                s.uuid.to_string().c_str(), s.begin, s.end, s.duration_ms, s.confidence, int(s.forced), s.birth,
                s.completion_ts, s.latency_ms);
  const SegmenterMetrics& m = r.segmenter;
  std::printf("  segmenter frames=%" PRId64 " speech=%" PRId64 " pause=%" PRId64 " forced=%" PRId64
              " eos=%" PRId64 "\n",
              m.frames, m.speech_frames, m.cuts_pause, m.cuts_forced, m.cuts_eos);
  const OrchestratorStats& o = r.orch;
  std::printf("  orch gathers=%" PRId64 " retries=%" PRId64 " sync_fail=%" PRId64 " drops=%" PRId64
              " detect=%" PRId64 " completions=%" PRId64 " resyncs=%" PRId64 " audio_hwm=%zu frame_hwm=%zu"
              " sum_lat=%" PRId64 " last=%" PRId64 " max_off=%" PRId64 " max_sync=%" PRId64 "\n",
              o.gathers, o.gather_retries, o.sync_failures, o.cap_drops, o.detector_calls, o.completions, o.resyncs,
              o.audio_hwm_bytes, o.frame_hwm_bytes, o.sum_latency_ms, o.last_completion_ts, o.max_abs_offset_ms,
              o.max_sync_overhead_ms);
  std::printf("  mem queue_hwm=%zu buffer_hwm=%zu depth=%.17g\n", r.queue_mem_hwm_bytes, r.buffer_mem_hwm_bytes,
              r.depth_time_avg);
  for (const auto& e : r.events) std::printf("  event %s\n", event_to_ndjson(e).c_str());
}

int main() {
  int fail = 0;
  // ---- run_pipeline_input over the reference's own scenarios
  dump_run("paper", paper_table3_scenario(), 8000);
  for (std::uint64_t seed = 1; seed <= 4; ++seed)
    for (DurationMs clip : {3000, 8000, 12000, 30000}) dump_run(("random" + std::to_string(seed)).c_str(),
                                                                random_scenario(seed), clip);
  // ---- segment_audio's known answer: stock 8 s (segmenter_tests.cpp:140-151)
  {
    SpeechPattern p;  // 600 ms lead, 1400/600 bursts repeating
    Segmenter seg(SegmenterConfig{});
    auto segs = seg.push(render_pattern(p, 8000));
    auto tail = seg.finish();
    segs.insert(segs.end(), tail.begin(), tail.end());
    std::printf("stock8s begins");
    for (const auto& s : segs) std::printf(" %" PRId64, s.begin);
    std::printf("\n");
  }
  // ---- mel frames of the orchestrator's pair (pipeline_tests.cpp:381-421)
  {
    SpeechPattern p;
    const AudioBuffer full = render_pattern(p, 3000);
    for (auto [b, e] : {std::pair<int, int>{0, 2300}, {2300, 3000}}) {
      AudioBuffer a;
      a.start = b;
      a.samples.assign(full.samples.begin() + b * 16, full.samples.begin() + e * 16);
      const MelSpectrogram m = compute_mel(a);
      std::printf("mel [%d,%d) frames=%" PRId64 " mels=%d\n", b, e, m.n_frames, m.n_mels);
#ifdef LSG_GPU_BUILD
      const MelSpectrogram c = ref_cpu_compute_mel(a, MelConfig{});
      double worst = 0;
      for (std::size_t i = 0; i < c.data.size(); ++i)
        worst = std::max(worst, std::fabs(double(m.data[i]) - c.data[i]) / std::max(1.0, std::fabs(double(c.data[i]))));
      const bool ok = c.n_frames == m.n_frames && worst <= 1e-4;
      std::fprintf(stderr, "gpu mel [%d,%d) vs reference cpu: max rel %.3g %s\n", b, e, worst, ok ? "ok" : "FAIL");
      fail += !ok;
#endif
    }
  }
  // ---- fft_radix2 known answer (media_tests.cpp:128-150)
  {
    std::uint64_t state = 555;
    std::vector<std::complex<double>> buf(16);
    for (auto& c : buf) {
      const double re = u64_to_unit(splitmix64(state)) - 0.5;
      const double im = u64_to_unit(splitmix64(state)) - 0.5;
      c = {re, im};
    }
    constexpr double pi = 3.141592653589793238462643383279502884;
    std::vector<std::complex<double>> want;
    for (int k = 0; k < 16; ++k) {
      std::complex<double> sum = 0;
      for (int n = 0; n < 16; ++n) sum += buf[std::size_t(n)] * std::exp(std::complex<double>(0, -2.0 * pi * k * n / 16.0));
      want.push_back(sum);
    }
    fft_radix2(buf);
    double worst = 0;
    for (int k = 0; k < 16; ++k) worst = std::max(worst, std::abs(buf[std::size_t(k)] - want[std::size_t(k)]));
    bool threw = false;
    std::vector<std::complex<double>> bad(12);
    try {
      fft_radix2(bad);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    std::printf("fft16 %s bad12_throws=%d\n", worst < 1e-9 ? "ok" : "FAIL", int(threw));
    fail += !(worst < 1e-9 && threw);
  }
  return fail ? 1 : 0;
}
