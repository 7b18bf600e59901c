// synth.cpp -- synthetic workload generation (include/lsg.h "synthetic input").
//
// render_pattern (synth.cpp:46-65 of the reference) restated for the bench
// and pipeline inputs: a speech pattern is a lead silence followed by a
// cycling list of (speech, pause) bursts, truncated at total_ms; adjacent
// spans of the same kind merge (pattern_pieces, synth.cpp:8-38); bursts are
// a tone lround(peak*sin(2*pi*f*(s-s0)/rate)) whose phase restarts per
// burst, silence is exact zero.  Same libm calls as the reference, so the
// PCM is bit-identical (tests/test_host.py).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "lsg.h"

namespace {
struct Piece {
  bool speech;
  int64_t begin, end;
};
}  // namespace

extern "C" lsg_status lsg_synth_pattern(int64_t lead, int32_t nb, const int64_t* speech_ms,
                                        const int64_t* pause_ms, double tone_hz, double amplitude,
                                        int64_t total_ms, int32_t rate, int16_t* out, int64_t cap,
                                        int64_t* n_out) {
  if (total_ms <= 0 || nb <= 0 || rate <= 0 || lead < 0) return LSG_EINVAL;
  for (int i = 0; i < nb; ++i)
    if (speech_ms[i] <= 0 || pause_ms[i] < 0) return LSG_EINVAL;
  std::vector<Piece> pieces;
  int64_t t = 0;
  auto push = [&](bool sp, int64_t len) {
    if (t >= total_ms || len == 0) return;
    int64_t end = std::min<int64_t>(total_ms, t + len);
    if (!pieces.empty() && pieces.back().speech == sp)
      pieces.back().end = end;
    else
      pieces.push_back({sp, t, end});
    t = end;
  };
  push(false, lead);
  for (int64_t i = 0; t < total_ms; ++i) {
    push(true, speech_ms[i % nb]);
    push(false, pause_ms[i % nb]);
  }
  const int64_t n = total_ms * (int64_t)rate / 1000;  // make_silence (audio.cpp:38-41)
  *n_out = n;
  if (n > cap) return LSG_OK;
  std::memset(out, 0, (size_t)n * sizeof(int16_t));
  const double two_pi = 8.0 * std::atan(1.0);
  const double peak = amplitude * 32767.0;
  for (const auto& p : pieces) {
    if (!p.speech) continue;
    int64_t s0 = p.begin * rate / 1000, s1 = p.end * rate / 1000;
    if (s1 > n) s1 = n;
    for (int64_t s = s0; s < s1; ++s) {
      double ph = two_pi * tone_hz * static_cast<double>(s - s0) / rate;
      out[s] = static_cast<int16_t>(std::lround(peak * std::sin(ph)));
    }
  }
  return LSG_OK;
}
