// segmenter.cu -- energy/silence segmenter on sm_100a (include/lsg.h "segmenter").
//
// Replaces lipstream::VadTracker::update (vad.cpp:26-53) and the Segmenter
// state machine (segmenter.cpp:25-145) for many streams per launch.
//
//   K1 seg_frame_stats  HBM-streaming pass: per 20 ms frame, sum of squares
//                       (int64, exact like the reference's double sum of
//                       integer squares) and max|s|; 16-byte vector loads,
//                       warp-shuffle reductions.  2 B/sample read, 16 B/frame
//                       written (2.5% of the input).
//   K2a seg_peaks       the decaying-peak recurrence (sequential by
//                       definition, one DMUL + compare per frame), one LANE
//                       per stream;
//   K2b seg_decide      per-frame dB decisions, thread per frame,
//                       ballot-packed bit rows;
//   K2c seg_machine     the integer-millisecond state machine, a warp per
//                       stream (bits staged by the warp, run by lane 0),
//                       fast-forwarding over runs of frames that
//                       cannot raise an event and stepping event frames
//                       exactly like process_frame (segmenter.cpp:51-99).
//   K3 seg_carry        keeps each stream's sub-frame tail (stage_,
//                       segmenter.cpp:40-48) on the device.
//   K4 seg_collect_scan + seg_collect_copy: cut offsets, then a warp per
//                       stream compacts cuts/flags/state into mapped pinned
//                       memory, so a collection costs one synchronisation.
//
// Bit-exactness: sqrt, division and the peak multiply are
// IEEE round-to-nearest on both sides (__dsqrt_rn/__ddiv_rn/__dmul_rn, no
// FMA contraction); the decay factor exp2(-frame/half_life) is computed on
// the host by the same libm call as vad.cpp:37.  log10 is the only libm
// function on the device: frames whose fast log10 lands within 1e-9 dB of
// the threshold are re-decided with a double-double log10 (error ~1e-30),
// i.e. with the correctly rounded value, which agrees with glibc's log10 on
// every decision tested (tests/test_segmenter_gpu.py exact-threshold frames).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <utility>
#include <vector>

#include "lsg_common.cuh"
#include "tc.cuh"

namespace lsg {
namespace seg {

struct Params {
  int32_t mode, peak_mode;
  double decay;  // exp2(-frame_ms / half_life), host libm
  double thr;
  // rms/peak outside [x_lo, x_hi] decides without a logarithm: x_lo / x_hi
  // are 10^(thr/20) -/+ 1e-9 relative, so 20 log10(x) is 8.7e-9 dB or more
  // from thr there -- ~10^6 ulps, far beyond log10's error (0 / inf: always
  // take the logarithm, e.g. thr <= -120 where the -120 clamp decides)
  double x_lo, x_hi;
  int64_t frame_ms, min_sil, min_seg, max_seg;
  int32_t rate, fs;
  int32_t flags_only, cut_cap;
  int32_t flag_words;  // per stream, per push
  int32_t pk_stride;   // K2a -> K2b peaks: doubles per stream row (even: 16-byte aligned rows)
};

struct alignas(16) DevState {
  double peak;
  int64_t base, seg_start, pause_start, silence_run, consumed, emitted;
  double cand_conf;
  int32_t speech_seen, cand_open, cand_cut, carry_len;
  int32_t n_cuts, overflow, n_flag_frames, pad;
  int64_t m_frames, m_speech, m_pause, m_forced, m_eos;
};

struct alignas(16) Chunk {
  const int16_t* pcm;  // device
  int64_t n;
  int64_t frame_off;   // into the push-global stats array
  int64_t start_ms;
  int64_t total_after; // samples pushed to the stream including this chunk
  int32_t nframes;
  int32_t stream;
  int32_t carry_len;
  int32_t first;
};

struct alignas(16) FrameStat {
  long long sumsq;
  double fmax;  // max |s| (an integer <= 32768), stored as the double the peak chain compares
};

// ---------------------------------------------------------------- K1 -----
#ifndef LSG_K1_WARPS
#define LSG_K1_WARPS 8
#endif
#ifndef LSG_K1_FPW
#define LSG_K1_FPW 4
#endif
constexpr int K1_WARPS = LSG_K1_WARPS;
constexpr int K1_FPW = LSG_K1_FPW;  // frames per warp per block
constexpr int K1_MAXV = 2;  // int4 per lane per frame held in registers (frames up to 512 samples)

// 8 samples: squares summed pairwise in uint32 (each pair <= 2^31, exact),
// one 64-bit add per pair; max |s| from packed int16 max/min (exact for
// -32768, whose magnitude does not fit int16).
__device__ __forceinline__ void acc8(int4 v, unsigned long long& ss, unsigned& pmax, unsigned& pmin) {
  const int w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int lo = (int)(int16_t)(w[k] & 0xffff);
    const int hi = w[k] >> 16;
    ss += (unsigned)(lo * lo) + (unsigned)(hi * hi);
    pmax = __vmaxs2(pmax, (unsigned)w[k]);
    pmin = __vmins2(pmin, (unsigned)w[k]);
  }
}
__device__ __forceinline__ int absmax_packed(unsigned pmax, unsigned pmin) {
  const int mx = max((int)(int16_t)(pmax & 0xffff), (int)pmax >> 16);
  const int mn = min((int)(int16_t)(pmin & 0xffff), (int)pmin >> 16);
  return max(mx, -mn);
}

__global__ void __launch_bounds__(K1_WARPS * 32)
seg_frame_stats(const Chunk* __restrict__ chunks, const int16_t* __restrict__ carry, int fs,
                FrameStat* __restrict__ out) {
  const Chunk c = chunks[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t f0 = ((int64_t)blockIdx.x * K1_WARPS + warp) * K1_FPW;
  if (f0 >= c.nframes) return;
  const bool vec = c.carry_len == 0 && (fs & 7) == 0 &&
                   ((reinterpret_cast<uintptr_t>(c.pcm) & 15) == 0);
  long long ss[K1_FPW];
  int mx[K1_FPW];
#pragma unroll
  for (int j = 0; j < K1_FPW; ++j) { ss[j] = 0; mx[j] = 0; }
  const int nv = fs >> 3;  // int4 per frame
  if (K1_FPW == 4 && vec && nv == 40 && f0 + 4 <= c.nframes) {
    // the reference default (16 kHz, 20 ms = 320 samples): the warp's 4
    // frames are 160 contiguous int4, exactly 5 per lane, so no lane reduces
    // padding; int4 q = lane + 32k belongs to frame q / 40, one of two
    // frames known at compile time per k.  Then one transposed butterfly
    // reduces the 4 frames together (18 shuffles instead of 60): the kernel
    // was issue-bound (SM 83%, DRAM 57% in ncu).
    const int4* p = reinterpret_cast<const int4*>(c.pcm + f0 * fs);
    int4 b[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) b[k] = __ldg(p + lane + 32 * k);
    unsigned long long s4[4] = {0, 0, 0, 0};
    unsigned px[4], pn[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) { px[j] = 0x80008000u; pn[j] = 0x7fff7fffu; }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      unsigned long long s2 = 0;
      unsigned mxk = 0x80008000u, mnk = 0x7fff7fffu;
      acc8(b[k], s2, mxk, mnk);
      const int jlo = (32 * k) / 40;               // frame of lane 0's int4
      const bool up = lane + 32 * k >= 40 * (jlo + 1);  // this lane's int4 is in frame jlo + 1
      if (!up) {
        s4[jlo] += s2;
        px[jlo] = __vmaxs2(px[jlo], mxk);
        pn[jlo] = __vmins2(pn[jlo], mnk);
      } else if (jlo + 1 < 4) {
        s4[jlo + 1] += s2;
        px[jlo + 1] = __vmaxs2(px[jlo + 1], mxk);
        pn[jlo + 1] = __vmins2(pn[jlo + 1], mnk);
      }
    }
    int m4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) m4[j] = absmax_packed(px[j], pn[j]);
    // xor 16: the lower half keeps frames 0,1, the upper half frames 2,3
    const bool hi16 = lane & 16, hi8 = lane & 8;
    unsigned long long k0 = hi16 ? s4[2] : s4[0], k1 = hi16 ? s4[3] : s4[1];
    int n0 = hi16 ? m4[2] : m4[0], n1 = hi16 ? m4[3] : m4[1];
    {
      const unsigned long long t0 = hi16 ? s4[0] : s4[2], t1 = hi16 ? s4[1] : s4[3];
      const int u0 = hi16 ? m4[0] : m4[2], u1 = hi16 ? m4[1] : m4[3];
      k0 += __shfl_xor_sync(0xffffffffu, t0, 16);
      k1 += __shfl_xor_sync(0xffffffffu, t1, 16);
      n0 = max(n0, __shfl_xor_sync(0xffffffffu, u0, 16));
      n1 = max(n1, __shfl_xor_sync(0xffffffffu, u1, 16));
    }
    // xor 8: bit 3 picks which of the two frames the lane keeps
    unsigned long long v = hi8 ? k1 : k0;
    int w = hi8 ? n1 : n0;
    v += __shfl_xor_sync(0xffffffffu, hi8 ? k0 : k1, 8);
    w = max(w, __shfl_xor_sync(0xffffffffu, hi8 ? n0 : n1, 8));
#pragma unroll
    for (int o = 4; o; o >>= 1) {
      v += __shfl_xor_sync(0xffffffffu, v, o);
      w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
    }
    if ((lane & 7) == 0) {
      FrameStat r;
      r.sumsq = (long long)v;
      r.fmax = (double)w;
      out[c.frame_off + f0 + 2 * (lane >> 4) + ((lane >> 3) & 1)] = r;
    }
    return;
  }
  if (vec && nv <= 32 * K1_MAXV) {
    // every load of the warp's frames in flight before any is consumed (a
    // 320-sample frame is 40 int4: lanes 0-7 take two); zero padding adds
    // nothing to the sum of squares or to |max|
    int4 buf[K1_FPW][K1_MAXV];
#pragma unroll
    for (int j = 0; j < K1_FPW; ++j) {
      const int4* p = reinterpret_cast<const int4*>(c.pcm + (f0 + j) * fs);
      const bool live = f0 + j < c.nframes;
#pragma unroll
      for (int k = 0; k < K1_MAXV; ++k) {
        const int q = lane + 32 * k;
        buf[j][k] = (live && q < nv) ? __ldg(p + q) : make_int4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int j = 0; j < K1_FPW; ++j) {
      unsigned long long s2 = 0;
      unsigned pmax = 0x80008000u, pmin = 0x7fff7fffu;
#pragma unroll
      for (int k = 0; k < K1_MAXV; ++k) acc8(buf[j][k], s2, pmax, pmin);
      ss[j] = (long long)s2;
      mx[j] = absmax_packed(pmax, pmin);
    }
  } else if (vec) {
    // issue every load of the warp's frames before reducing (memory-level parallelism)
#pragma unroll
    for (int j = 0; j < K1_FPW; ++j) {
      const int64_t f = f0 + j;
      if (f >= c.nframes) break;
      const int4* p = reinterpret_cast<const int4*>(c.pcm + f * fs);
      unsigned long long s2 = 0;
      unsigned pmax = 0x80008000u, pmin = 0x7fff7fffu;
      for (int q = lane; q < nv; q += 32) acc8(__ldg(p + q), s2, pmax, pmin);
      ss[j] = (long long)s2;
      mx[j] = absmax_packed(pmax, pmin);
    }
  } else {
    const int16_t* cs = carry + (int64_t)c.stream * fs;
    for (int j = 0; j < K1_FPW; ++j) {
      const int64_t f = f0 + j;
      if (f >= c.nframes) break;
      for (int q = lane; q < fs; q += 32) {
        const int64_t idx = f * fs + q;  // index into carry ++ chunk
        int v = idx < c.carry_len ? cs[idx] : c.pcm[idx - c.carry_len];
        ss[j] += (long long)(v * v);
        mx[j] = max(mx[j], abs(v));
      }
    }
  }
#pragma unroll
  for (int j = 0; j < K1_FPW; ++j) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      ss[j] += __shfl_xor_sync(0xffffffffu, ss[j], o);
      mx[j] = max(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], o));
    }
  }
  if (lane < K1_FPW) {
    const int64_t f = f0 + lane;
    long long s = ss[0];
    int m = mx[0];
#pragma unroll
    for (int j = 1; j < K1_FPW; ++j)
      if (lane == j) { s = ss[j]; m = mx[j]; }
    if (f < c.nframes) {
      FrameStat r;
      r.sumsq = s;
      r.fmax = (double)m;
      out[c.frame_off + f] = r;
    }
  }
}

// ------------------------------------------------------ exact log10 ------
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double e = __dsub_rn(b, __dsub_rn(s, a));
  return {s, e};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = quick_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  double p = __dmul_rn(a.hi, b.hi);
  double e = __fma_rn(a.hi, b.hi, -p);
  e = __fma_rn(a.hi, b.lo, e);
  e = __fma_rn(a.lo, b.hi, e);
  return quick_two_sum(p, e);
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {
  double q1 = __ddiv_rn(a.hi, b.hi);
  dd r = dd_add(a, dd_mul({-q1, 0.0}, b));
  double q2 = __ddiv_rn(r.hi, b.hi);
  r = dd_add(r, dd_mul({-q2, 0.0}, b));
  double q3 = __ddiv_rn(r.hi, b.hi);
  dd q = quick_two_sum(q1, q2);
  return dd_add(q, {q3, 0.0});
}

// log10(x) in double-double, rounded once to double.  x = m 2^e with
// m in [sqrt(1/2), sqrt(2)); ln m = 2 atanh((m-1)/(m+1)) by its series.
__device__ double log10_dd(double x) {
  int e;
  double m = frexp(x, &e);  // m in [0.5, 1)
  if (m < 0.70710678118654752440) {
    m *= 2.0;
    e -= 1;
  }
  dd num = two_sum(m, -1.0);
  dd den = two_sum(m, 1.0);
  dd s = dd_div(num, den);
  dd s2 = dd_mul(s, s);
  dd term = s;
  dd sum = s;
  for (int k = 3; k < 80; k += 2) {
    term = dd_mul(term, s2);
    dd t = dd_div(term, {(double)k, 0.0});
    sum = dd_add(sum, t);
    if (fabs(t.hi) < 1e-40) break;
  }
  const dd ln2 = {6.93147180559945286227e-01, 2.31904681384629955842e-17};
  const dd inv_ln10 = {4.34294481903251816668e-01, 1.09872180683456050377e-17};
  dd lnm = dd_add(sum, sum);
  dd ln = dd_add(dd_mul(ln2, {(double)e, 0.0}), lnm);
  dd r = dd_mul(ln, inv_ln10);
  return __dadd_rn(r.hi, r.lo);
}

// VadTracker::update's decision (vad.cpp:47-52) from exact frame stats.
__device__ __forceinline__ bool vad_decide(long long sumsq, double peak, int n, double thr, double x_lo,
                                           double x_hi) {
  double rms = __dsqrt_rn(__ddiv_rn((double)sumsq, (double)n));
  double db = -120.0;
  if (rms > 0.0 && peak > 0.0) {
    double x = __ddiv_rn(rms, peak);
    if (x < x_lo) return false;  // db = max(20 log10 x, -120) < thr
    if (x > x_hi) return true;
    double d = __dmul_rn(20.0, log10(x));
    if (fabs(d - thr) < 1e-9 * fmax(1.0, fabs(thr))) d = __dmul_rn(20.0, log10_dd(x));
    db = d > -120.0 ? d : -120.0;
  }
  return db > thr;
}

// ---------------------------------------------------------------- K2 -----
struct Machine {
  int64_t base, seg_start, pause_start, silence_run, consumed, emitted;
  double conf;
  int speech_seen, cand_open, cand_cut;
  int64_t n_pause, n_forced;
  int n_cuts, overflow;
};

__device__ __forceinline__ int64_t cdiv(int64_t a, int64_t b) {  // ceil(a/b), b > 0
  // 32-bit division when both fit (the machine's operands are millisecond
  // spans and the frame length): a 64-bit division is a long software
  // sequence on the state machine's critical path
  if (a > -0x7fffffffLL && a < 0x7fffffffLL && b < 0x7fffffffLL) {
    const int ai = (int)a, bi = (int)b;
    return ai >= 0 ? (ai + bi - 1) / bi : -((-ai) / bi);
  }
  return a >= 0 ? (a + b - 1) / b : -((-a) / b);
}

// emit_cut (segmenter.cpp:101-118)
__device__ __forceinline__ void emit(Machine& M, const Params& P, lsg_cut* cuts, int stream,
                                     int64_t cut_ms, double conf, int cause) {
  const int64_t split = (cut_ms - M.seg_start) * P.rate / 1000;
  if (M.n_cuts < P.cut_cap) {
    lsg_cut c;
    c.begin = M.seg_start;
    c.end = cut_ms;
    c.confidence = conf;
    c.cause = cause;
    c.stream = stream;
    c.sample_off = M.emitted;
    c.sample_len = split;
    cuts[M.n_cuts] = c;
    M.n_cuts++;
  } else {
    M.overflow = 1;
  }
  M.emitted += split;
  M.seg_start = cut_ms;
  M.speech_seen = 0;
}

// process_frame (segmenter.cpp:51-99), device state machine (no scorer).
__device__ __forceinline__ void step(Machine& M, const Params& P, lsg_cut* cuts, int stream,
                                     bool speech) {
  const int64_t f0 = M.base + M.consumed * P.frame_ms;
  const int64_t f1 = f0 + P.frame_ms;
  if (speech) {
    if (M.speech_seen && M.silence_run >= P.min_sil && M.cand_open && M.cand_cut) {
      emit(M, P, cuts, stream, M.pause_start + M.silence_run / 2, M.conf, 0);
      M.n_pause++;
    }
    M.silence_run = 0;
    M.cand_open = 0;
    M.cand_cut = 0;
    M.speech_seen = 1;
  } else {
    if (M.silence_run == 0) M.pause_start = f0;
    M.silence_run += P.frame_ms;
    if (!M.cand_open && M.silence_run >= P.min_sil && M.speech_seen) {
      M.cand_open = 1;
      M.cand_cut = 1;
      M.conf = 1.0;
      if (P.mode == 1 && M.pause_start - M.seg_start < P.min_seg) M.cand_cut = 0;
    }
  }
  if (P.mode == 1 && M.speech_seen && f1 - M.seg_start >= P.max_seg) {
    emit(M, P, cuts, stream, f1, 1.0, 1);
    M.n_forced++;
  }
  M.consumed++;
}

__device__ __forceinline__ int get_bit(const uint32_t* bits, int i) { return (bits[i >> 5] >> (i & 31)) & 1; }

// first index >= i in [i, n) whose bit differs from b, or n
__device__ __forceinline__ int run_end(const uint32_t* bits, int i, int n, int b) {
  int wi = i >> 5;
  uint32_t w = (b ? ~bits[wi] : bits[wi]) & (0xffffffffu << (i & 31));
  const int nw = (n + 31) >> 5;
  while (!w) {
    if (++wi >= nw) return n;
    w = b ? ~bits[wi] : bits[wi];
  }
  int p = (wi << 5) + __ffs(w) - 1;
  return p < n ? p : n;
}

// The state machine over n decided frames, skipping event-free runs.
__device__ void run_machine(Machine& M, const Params& P, lsg_cut* cuts, int stream,
                            const uint32_t* bits, int n) {
  int i = 0;
  while (i < n) {
    const int b = get_bit(bits, i);
    const int e = run_end(bits, i, n, b);
    if (b && M.silence_run == 0 && !M.cand_open && !M.cand_cut && M.speech_seen) {
      // steady speech: only the forced split can fire (segmenter.cpp:94-98)
      if (P.mode == 1) {
        int64_t k = cdiv(P.max_seg + M.seg_start - M.base, P.frame_ms) - M.consumed - 1;
        if (k < 0) k = 0;
        if (i + k < e) {
          M.consumed += k;
          i += (int)k;
          step(M, P, cuts, stream, true);
          ++i;
          continue;
        }
      }
      M.consumed += e - i;
      i = e;
      continue;
    }
    if (!b && M.silence_run > 0) {
      // steady silence: candidate opening and forced split are the only events
      int64_t k = INT64_MAX;
      if (!M.cand_open && M.speech_seen) {
        int64_t kc = cdiv(P.min_sil - M.silence_run, P.frame_ms) - 1;
        k = kc < 0 ? 0 : kc;
      }
      if (P.mode == 1 && M.speech_seen) {
        int64_t kf = cdiv(P.max_seg + M.seg_start - M.base, P.frame_ms) - M.consumed - 1;
        if (kf < 0) kf = 0;
        k = kf < k ? kf : k;
      }
      if (k < (int64_t)(e - i)) {
        M.silence_run += k * P.frame_ms;
        M.consumed += k;
        i += (int)k;
        step(M, P, cuts, stream, false);
        ++i;
        continue;
      }
      M.silence_run += (int64_t)(e - i) * P.frame_ms;
      M.consumed += e - i;
      i = e;
      continue;
    }
    step(M, P, cuts, stream, b != 0);
    ++i;
  }
}

// K2 runs as three launches so that only the two inherently sequential
// recurrences are sequential, and those run ONE LANE PER STREAM (a warp
// carries 32 streams' recurrences in one instruction stream):
//   K2a seg_peaks    the decaying peak (vad.cpp:35-45): p = max(RN(p*c), m),
//                    one DMUL + compare per frame and stream; peaks -> HBM;
//   K2b seg_decide   every frame's decision in parallel (thread per frame),
//                    ballot-packed into the stream's bit row;
//   K2c seg_machine  the state machine over the bits (segmenter.cpp:51-99),
//                    warp per stream, fast-forwarding event-free runs.
constexpr int K2_LANES = 32;  // streams per K2a / K2c block: one warp, a lane per stream
// Time-sliced pushes: a push of many frames per stream is processed in
// slices of kSlice frames so that the per-stream sequential work (the peak
// chain and the state machine, latency-bound on a few SMs) of slice s
// overlaps the HBM-bound K1 of slice s + 1 and of each other.
#ifndef LSG_SEG_SLICE
#define LSG_SEG_SLICE 512
#endif
constexpr int kSlice = LSG_SEG_SLICE;  // frames (a multiple of 256)
constexpr int kSlots = 3;    // slices in flight
constexpr int PK_T = 128;     // K2a frames per tile
constexpr int PK_ROW = PK_T * 16 + 16;  // stats row stride in smem (bytes; +16 spreads the banks)
constexpr int PK_PROW = PK_T * 8 + 16;  // peaks row stride in smem (bytes)
constexpr size_t PK_SMEM = 2 * K2_LANES * PK_ROW + 2 * K2_LANES * PK_PROW + 64;

// fmax of frames f..f+7 of a staged stats row, issued back to back
// (volatile: kept ahead of the chain that consumes them)
__device__ __forceinline__ void ld8(const unsigned char* row, int f, double (&m)[8]) {
  const uint32_t a = tc::smem_u32(row) + f * 16 + 8;
#pragma unroll
  for (int k = 0; k < 8; ++k) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(m[k]) : "r"(a + 16 * k));
}

// K2a: each lane's stream is brought in by the TMA engine, tile by tile and
// double-buffered (a 2 KB bulk copy per stream and tile), so the chain --
// one DMUL and a compare per frame -- never waits on memory; each tile's
// peaks leave the same way (one bulk store per stream, double-buffered).
__global__ void __launch_bounds__(K2_LANES)
seg_peaks(const Chunk* __restrict__ chunks, int nc, const FrameStat* __restrict__ stats, DevState* st,
          double* __restrict__ peaks, Params P, int pk_off) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned char* buf = sm;                                // [2][32][PK_ROW] stats tiles
  unsigned char* pbuf = sm + 2 * K2_LANES * PK_ROW;       // [2][32][PK_PROW] peak tiles
  uint64_t* full = reinterpret_cast<uint64_t*>(pbuf + 2 * K2_LANES * PK_PROW);
  const int lane = threadIdx.x;
  const int i = blockIdx.x * K2_LANES + lane;
  const bool live = i < nc;
  Chunk c{};
  if (live) c = chunks[i];
  const int n = live ? c.nframes : 0;
  int tiles = (n + PK_T - 1) / PK_T;
#pragma unroll
  for (int o = 16; o; o >>= 1) tiles = max(tiles, __shfl_xor_sync(0xffffffffu, tiles, o));
  if (lane == 0) {
    tc::mbar_init(&full[0], K2_LANES);
    tc::mbar_init(&full[1], K2_LANES);
    tc::fence_mbar_init();
  }
  __syncwarp();
  const FrameStat* fst = stats + c.frame_off;
  auto issue = [&](int t) {  // tile t of this lane's stream into buffer t & 1
    const int f0 = t * PK_T, nf = max(0, min(PK_T, n - f0));
    tc::mbar_arrive_expect_tx(&full[t & 1], (uint32_t)nf * 16);
    if (nf) tc::bulk_g2s(tc::smem_u32(buf + ((t & 1) * K2_LANES + lane) * PK_ROW), fst + f0, (uint32_t)nf * 16,
                         &full[t & 1]);
  };
  if (tiles > 0) issue(0);
  if (tiles > 1) issue(1);
  double peak = live ? st[c.stream].peak : 0.0;
  const double decay = P.decay;
  for (int t = 0; t < tiles; ++t) {
    tc::mbar_wait(&full[t & 1], (t >> 1) & 1);
    const unsigned char* row = buf + ((t & 1) * K2_LANES + lane) * PK_ROW;
    double* prow = reinterpret_cast<double*>(pbuf + ((t & 1) * K2_LANES + lane) * PK_PROW);
    // the bulk store that read this peak buffer two tiles ago has finished
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    const int nf = max(0, min(PK_T, n - t * PK_T));
    if (P.peak_mode == 0) {
      int f = 0;
      for (; f + 8 <= nf; f += 8) {
        // the 8 frame maxima are loaded before the chain uses any of them (the
        // compiler would otherwise put each load's latency on the chain)
        double m[8];
        ld8(row, f, m);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          peak = __dmul_rn(peak, decay);
          peak = m[k] > peak ? m[k] : peak;
          prow[f + k] = peak;
        }
      }
      for (; f < nf; ++f) {
        peak = __dmul_rn(peak, decay);
        const double m = reinterpret_cast<const FrameStat*>(row)[f].fmax;
        peak = m > peak ? m : peak;
        prow[f] = peak;
      }
    } else if (P.peak_mode == 1) {
      int f = 0;
      for (; f + 8 <= nf; f += 8) {
        double m[8];
        ld8(row, f, m);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          peak = m[k] > peak ? m[k] : peak;
          prow[f + k] = peak;
        }
      }
      for (; f < nf; ++f) {
        const double m = reinterpret_cast<const FrameStat*>(row)[f].fmax;
        peak = m > peak ? m : peak;
        prow[f] = peak;
      }
    } else {
      for (int f = 0; f < nf; ++f) prow[f] = peak;
    }
    // the tile's peaks go out on the TMA engine: one bulk store per stream
    if (nf) {
      tc::fence_proxy_async();  // generic smem writes -> visible to the async proxy
      // stream rows are 16-byte aligned; an odd tail carries one spare double
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                       peaks + (int64_t)c.stream * P.pk_stride + pk_off + t * PK_T),
                   "r"(tc::smem_u32(prow)), "r"(((nf + 1) & ~1) * 8)
                   : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    __syncwarp();
    if (t + 2 < tiles) {
      tc::fence_proxy_async();  // this buffer's generic reads before the TMA overwrites it
      issue(t + 2);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete before the kernel ends
  if (live) st[c.stream].peak = peak;
}

__global__ void __launch_bounds__(256)
seg_decide(const Chunk* __restrict__ chunks, const FrameStat* __restrict__ stats, const double* __restrict__ peaks,
           DevState* st, uint32_t* __restrict__ bits_all, Params P, int pk_off, int bits_off) {
  const Chunk c = chunks[blockIdx.y];
  const int f = blockIdx.x * 256 + threadIdx.x;
  if (blockIdx.x * 256 >= c.nframes) return;  // whole block past the chunk (uniform)
  bool sp = false;
  if (f < c.nframes)
    sp = vad_decide(stats[c.frame_off + f].sumsq, peaks[(int64_t)c.stream * P.pk_stride + pk_off + f], P.fs, P.thr,
                    P.x_lo, P.x_hi);
  const unsigned bal = __ballot_sync(0xffffffffu, sp);
  if ((threadIdx.x & 31) == 0) {
    if (f < c.nframes) bits_all[(int64_t)c.stream * P.flag_words + bits_off + (f >> 5)] = bal;
    if (bal) atomicAdd(reinterpret_cast<unsigned long long*>(&st[c.stream].m_speech), (unsigned long long)__popc(bal));
  }
}

// K2c: one warp per stream -- the lanes stage the stream's bit row in shared
// memory, then lane 0 runs the machine (warp-uniform control flow: no
// divergence between streams; 512 streams are 512 concurrent warps).
constexpr int MC_WARPS = 4;
__global__ void __launch_bounds__(MC_WARPS * 32)
seg_machine(const Chunk* __restrict__ chunks, int nc, DevState* st, lsg_cut* __restrict__ cuts_all,
            const uint32_t* __restrict__ bits_all, Params P, int row_words, int bits_off) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * MC_WARPS + warp;
  if (i >= nc) return;
  uint32_t* sb = reinterpret_cast<uint32_t*>(sm) + warp * row_words;
  const Chunk c = chunks[i];
  const int nw = (c.nframes + 31) >> 5;
  const uint32_t* src = bits_all + (int64_t)c.stream * P.flag_words + bits_off;
  for (int w = lane; w < nw; w += 32) sb[w] = src[w];
  __syncwarp();
  if (lane != 0) return;
  DevState* S = st + c.stream;
  if (c.first) {
    S->base = c.start_ms;
    S->seg_start = c.start_ms;
  }
  if (P.flags_only) {  // the host runs the machine (scorer order): bits are the output
    S->consumed += c.nframes;
    S->n_flag_frames = c.nframes;
    S->m_frames += c.nframes;
    return;
  }
  Machine M;
  M.base = S->base;
  M.seg_start = S->seg_start;
  M.pause_start = S->pause_start;
  M.silence_run = S->silence_run;
  M.consumed = S->consumed;
  M.emitted = S->emitted;
  M.conf = S->cand_conf;
  M.speech_seen = S->speech_seen;
  M.cand_open = S->cand_open;
  M.cand_cut = S->cand_cut;
  M.n_pause = 0;
  M.n_forced = 0;
  M.n_cuts = S->n_cuts;  // cuts not collected yet stay in front (collection is deferred)
  M.overflow = S->overflow;
  run_machine(M, P, cuts_all + (int64_t)c.stream * P.cut_cap, c.stream, sb, c.nframes);
  S->seg_start = M.seg_start;
  S->pause_start = M.pause_start;
  S->silence_run = M.silence_run;
  S->consumed = M.consumed;
  S->emitted = M.emitted;
  S->cand_conf = M.conf;
  S->speech_seen = M.speech_seen;
  S->cand_open = M.cand_open;
  S->cand_cut = M.cand_cut;
  S->n_cuts = M.n_cuts;
  S->overflow = M.overflow;
  S->n_flag_frames = c.nframes;
  S->m_frames += c.nframes;
  S->m_pause += M.n_pause;
  S->m_forced += M.n_forced;
}

// ---------------------------------------------------------------- K3 -----
// New stage_ after the push: the last (carry_len + n) % fs samples.
__global__ void seg_carry(const Chunk* __restrict__ chunks, int16_t* carry, DevState* st, int fs) {
  const Chunk c = chunks[blockIdx.x];
  int16_t* cs = carry + (int64_t)c.stream * fs;
  const int64_t total = c.carry_len + c.n;
  const int r = (int)(total % fs);
  if (c.nframes == 0) {
    for (int64_t i = threadIdx.x; i < c.n; i += blockDim.x) cs[c.carry_len + i] = c.pcm[i];
  } else {
    for (int i = threadIdx.x; i < r; i += blockDim.x) cs[i] = c.pcm[c.n - r + i];
  }
  if (threadIdx.x == 0) st[c.stream].carry_len = r;
}

// ---------------------------------------------------------------- K4 -----
// finish() (segmenter.cpp:120-145): EOS flush of the open segment.
__global__ void seg_finish(const int32_t* __restrict__ streams, const int64_t* __restrict__ totals,
                           int n, DevState* st, lsg_cut* cuts_all, Params P) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int s = streams[i];
  DevState* S = st + s;
  S->n_flag_frames = 0;
  const int64_t tail_ms = (int64_t)S->carry_len * 1000 / P.rate;
  const int64_t pending = totals[i] - S->emitted;
  if (!S->speech_seen || pending == 0) return;
  lsg_cut c;
  c.begin = S->seg_start;
  c.end = S->base + S->consumed * P.frame_ms + tail_ms;
  c.confidence = 1.0;
  c.cause = 2;
  c.stream = s;
  c.sample_off = S->emitted;
  c.sample_len = pending;
  if (S->n_cuts < P.cut_cap) {
    cuts_all[(int64_t)s * P.cut_cap + S->n_cuts] = c;
    S->n_cuts += 1;
  } else {
    S->overflow = 1;
  }
  S->emitted += pending;
  S->m_eos += 1;
}

// Compacts the touched streams' cuts + state (+flags) into mapped host
// memory in two launches: seg_collect_scan (one block) turns the per-stream
// cut counts into offsets; seg_collect_copy then runs a warp per stream over
// the whole GPU, copying its state, its cuts as coalesced 16-byte words
// (lsg_cut is 48 B) and its flags -- many SMs' worth of outstanding writes to
// the mapped buffers instead of one block's.
constexpr int COLLECT_THREADS = 1024;
constexpr int COLLECT_MAX = 4096;  // streams per push / finish
constexpr int COPY_WARPS = 8;
__global__ void __launch_bounds__(COLLECT_THREADS)
seg_collect_scan(const int32_t* __restrict__ streams, int n, const DevState* __restrict__ st,
                 int32_t* __restrict__ d_offsets, int32_t* h_offsets) {
  __shared__ int s_warp[COLLECT_THREADS / 32];
  __shared__ int s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += COLLECT_THREADS) {
    const int i = base + tid;
    const int v = i < n ? st[streams[i]].n_cuts : 0;
    int x = v;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = s_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_warp[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int excl = s_carry + (warp ? s_warp[warp - 1] : 0) + x - v;
    if (i < n) {
      d_offsets[i] = excl;
      h_offsets[i] = excl;
    }
    __syncthreads();
    if (tid == 0) s_carry += s_warp[31];
    __syncthreads();
  }
  if (tid == 0) {
    d_offsets[n] = s_carry;
    h_offsets[n] = s_carry;
  }
}

__global__ void __launch_bounds__(COPY_WARPS * 32)
seg_collect_copy(const int32_t* __restrict__ streams, int n, DevState* st, const lsg_cut* __restrict__ cuts_all,
                 const uint32_t* __restrict__ flags_all, Params P, const int32_t* __restrict__ d_offsets,
                 DevState* h_state, lsg_cut* h_cuts, uint32_t* h_flags, int cut_cap_total) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * COPY_WARPS + (threadIdx.x >> 5);
  if (i >= n) return;
  const int s = streams[i];
  const DevState d = st[s];
  if (lane == 0) h_state[i] = d;
  const int off = d_offsets[i];
  const int k = min(d.n_cuts, max(0, cut_cap_total - off));
  const uint4* src = reinterpret_cast<const uint4*>(cuts_all + (int64_t)s * P.cut_cap);
  uint4* dst = reinterpret_cast<uint4*>(h_cuts + off);
  for (int u = lane; u < k * 3; u += 32) dst[u] = src[u];
  if (P.flags_only) {
    const int nw = (d.n_flag_frames + 31) >> 5;
    for (int j = lane; j < nw; j += 32) h_flags[(int64_t)i * P.flag_words + j] = flags_all[(int64_t)s * P.flag_words + j];
  }
  __syncwarp();
  if (lane == 0) st[s].n_cuts = 0;  // after every lane read d
}

}  // namespace seg
}  // namespace lsg

using namespace lsg;
using namespace lsg::seg;

struct StreamHost {
  bool finished = false;
  int64_t base = 0;
  int64_t consumed = 0;   // frames
  int64_t stage_len = 0;  // samples
  int64_t total = 0;      // samples pushed
  std::vector<lsg_cut> cuts;
  std::vector<uint8_t> flags;
  lsg_seg_metrics metrics{};
};

constexpr int kMaxCollect = seg::COLLECT_MAX;  // streams per push call handled by one collect launch

struct lsg_seg_s {
  Ctx* ctx = nullptr;
  Params P{};
  int32_t n_streams = 0;
  int64_t max_push = 0;
  int64_t max_frames_push = 0;
  std::vector<StreamHost> hs;
  DevBuf<DevState> st;
  DevBuf<int16_t> carry;
  DevBuf<lsg_cut> cuts;
  DevBuf<uint32_t> flags;
  DevBuf<FrameStat> stats;
  DevBuf<double> peaks;  // K2a -> K2b: every frame's decayed peak
  bool attrs_set = false;
  // time-sliced pushes (see launch_sliced): K1 on the context stream, the
  // peak chain on sB, decisions + machine on sC, kSlots slices in flight
  cudaStream_t sB = nullptr, sC = nullptr;
  cudaEvent_t eK1[3] = {}, ePk[3] = {}, eM[3] = {}, eJoin = nullptr;
  DevBuf<Chunk> chunks_sl;
  PinnedBuf<Chunk> chunks_sl_host;
  int max_slices = 0;
  // the pinned chunk / stream tables are copied asynchronously: the next
  // call waits for the last copy before rewriting them (pushes do not
  // synchronise the stream any more)
  cudaEvent_t tab_ev = nullptr;
  bool tab_pending = false;
  // the sliced launch sequence, captured once per (chunks, slices) shape: the
  // tables it reads live at fixed device addresses, so a replay is one
  // cudaGraphLaunch instead of ~9 API calls per slice
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    int kernels = 0;
  };
  std::map<std::pair<int, int>, Graph> graphs;
  cudaStream_t cap = nullptr;  // capture stream
  int prio_hi = 0;             // greatest stream / launch priority of the device
  bool slicing = true;  // lsgdbg_seg_slicing
  void tables_free() {
    if (tab_pending) {
      LSG_CUDA(cudaEventSynchronize(tab_ev));
      tab_pending = false;
    }
  }
  void tables_sent(cudaStream_t st) {
    LSG_CUDA(cudaEventRecord(tab_ev, st));
    tab_pending = true;
  }
  DevBuf<Chunk> chunks_dev;
  DevBuf<int16_t> staging;
  DevBuf<int32_t> streams_dev;
  DevBuf<int32_t> collect_dev;  // streams whose results are still on the device
  DevBuf<int32_t> collect_off;  // their cut offsets (seg_collect_scan)
  DevBuf<int64_t> totals_dev;
  PinnedBuf<Chunk> chunks_host;
  PinnedBuf<int32_t> streams_host;
  PinnedBuf<int32_t> collect_host;
  PinnedBuf<int64_t> totals_host;
  // Deferred collection: a push leaves its cuts, state and metrics on the
  // device (no stream synchronisation); they are gathered into mapped host
  // memory by the next call that needs them (take_cuts / metrics / finish)
  // or when a stream's pending-cut bound could reach its device capacity.
  std::vector<char> dirty;
  std::vector<int32_t> dirty_list;
  std::vector<int64_t> cut_bound;  // upper bound of uncollected cuts per stream
  // mapped (zero-copy) result area
  DevState* h_state = nullptr;
  int32_t* h_off = nullptr;
  lsg_cut* h_cuts = nullptr;
  uint32_t* h_flags = nullptr;
  int64_t h_cut_cap = 0;
  // device time of the last push's K1 (the HBM-streaming pass), for the
  // benchmark's per-kernel roofline (lsgdbg_seg_k1_ms)
  cudaEvent_t k1a = nullptr, k1b = nullptr;
  bool k1_recorded = false;
  double collect_wait_ms = 0.0, collect_host_ms = 0.0;  // last collection: sync wait, host distribution
  ~lsg_seg_s() {
    for (int j = 0; j < 3; ++j) {
      if (eK1[j]) cudaEventDestroy(eK1[j]);
      if (ePk[j]) cudaEventDestroy(ePk[j]);
      if (eM[j]) cudaEventDestroy(eM[j]);
    }
    if (eJoin) cudaEventDestroy(eJoin);
    if (tab_ev) cudaEventDestroy(tab_ev);
    for (auto& g : graphs)
      if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
    if (cap) cudaStreamDestroy(cap);
    if (sB) cudaStreamDestroy(sB);
    if (sC) cudaStreamDestroy(sC);
    if (k1a) cudaEventDestroy(k1a);
    if (k1b) cudaEventDestroy(k1b);
    if (h_state) cudaFreeHost(h_state);
    if (h_off) cudaFreeHost(h_off);
    if (h_cuts) cudaFreeHost(h_cuts);
    if (h_flags) cudaFreeHost(h_flags);
  }
};

static void validate_cfg(const lsg_seg_cfg* c) {
  // member init order: VadTracker(cfg.vad) runs before the Segmenter body
  // checks (segmenter.cpp:9-10, vad.cpp:13-19)
  if (c->peak_half_life_ms <= 0) invalid("vad: non-positive half life");
  if (c->frame_ms <= 0) invalid("vad: non-positive frame");
  if (c->sample_rate <= 0 || c->sample_rate % 1000 != 0)
    invalid("segmenter: rate must be a multiple of 1 kHz");
  if (c->min_silence_ms <= 0) invalid("segmenter: non-positive min silence");
  if (c->mode == 1) {
    if (c->min_segment_ms < 0 || c->max_segment_ms <= 0) invalid("segmenter: bad segment bounds");
    if (c->max_segment_ms <= c->min_segment_ms) invalid("segmenter: max segment under min");
  }
  if (c->mode != 0 && c->mode != 1) invalid("segmenter: unknown mode");
  if (c->peak_mode < 0 || c->peak_mode > 2) invalid("vad: unknown peak mode");
}

// Gathers every dirty stream's cuts + state (+flags) into mapped host
// memory, synchronises once, and distributes the results to the host mirror.
static void collect(lsg_seg h, bool finishing) {
  Ctx* ctx = h->ctx;
  const int n = (int)h->dirty_list.size();
  if (n == 0) return;
  std::memcpy(h->collect_host.p, h->dirty_list.data(), sizeof(int32_t) * n);
  LSG_CUDA(cudaMemcpyAsync(h->collect_dev.p, h->collect_host.p, sizeof(int32_t) * n, cudaMemcpyHostToDevice,
                           ctx->stream));
  seg_collect_scan<<<1, COLLECT_THREADS, 0, ctx->stream>>>(h->collect_dev.p, n, h->st.p, h->collect_off.p, h->h_off);
  LSG_LAUNCHED(ctx);
  seg_collect_copy<<<(unsigned)ceil_div(n, COPY_WARPS), COPY_WARPS * 32, 0, ctx->stream>>>(
      h->collect_dev.p, n, h->st.p, h->cuts.p, h->flags.p, h->P, h->collect_off.p, h->h_state, h->h_cuts, h->h_flags,
      (int)h->h_cut_cap);
  LSG_LAUNCHED(ctx);
  const auto tw0 = std::chrono::steady_clock::now();
  ctx->sync();
  const auto tw1 = std::chrono::steady_clock::now();
  struct Stamp {  // host distribution time of this collection (lsgdbg_seg_collect_ms)
    lsg_seg h;
    std::chrono::steady_clock::time_point t0;
    ~Stamp() { h->collect_host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
  } stamp{h, tw1};
  h->collect_wait_ms = std::chrono::duration<double, std::milli>(tw1 - tw0).count();
  for (int s : h->dirty_list) {
    h->dirty[s] = 0;
    h->cut_bound[s] = 0;
  }
  h->dirty_list.clear();
  for (int i = 0; i < n; ++i) {
    const int s = h->collect_host.p[i];
    StreamHost& S = h->hs[s];
    const DevState& D = h->h_state[i];
    if (D.overflow) fail(LSG_ERUNTIME, "segmenter: cut buffer overflow");
    const int a = h->h_off[i], b = h->h_off[i + 1];
    S.cuts.insert(S.cuts.end(), h->h_cuts + a, h->h_cuts + b);
    S.metrics.frames = D.m_frames;
    S.metrics.speech_frames = D.m_speech;
    S.metrics.cuts_pause = D.m_pause;
    S.metrics.cuts_forced = D.m_forced;
    S.metrics.cuts_eos = D.m_eos;
    if (h->P.flags_only && !finishing) {
      S.flags.resize((size_t)D.n_flag_frames);
      const uint32_t* w = h->h_flags + (int64_t)i * h->P.flag_words;
      for (int f = 0; f < D.n_flag_frames; ++f) S.flags[f] = (w[f >> 5] >> (f & 31)) & 1;
    }
  }
}

// Time-sliced push (see kSlice): slice k of every chunk is frames
// [k*kSlice, (k+1)*kSlice) (the chunk's last slice also holds its sub-frame
// tail, which seg_carry keeps).  Per slice, on three streams:
//   ctx stream: K1 (stats of the slice into slot k % kSlots)     -> eK1
//   sB:         K2a peak chain (in slice order: the peak carries) -> ePk
//   sC:         K2b decisions + K2c machine (in slice order)      -> eM
// A slot is reused only after the machine of the slice that last used it
// (the slot's last reader) has completed.  Bit-identical to one launch: the
// peak and machine state carry through DevState exactly as across pushes.
// cudaLaunchKernelEx with a priority attribute (kept by stream capture)
template <typename... KArgs, typename... Args>
static void launch_hi(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int prio,
                      Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributePriority;
  at[0].val.priority = prio;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  LSG_CUDA(cudaLaunchKernelEx(&cfg, k, args...));
}

static void launch_sliced(lsg_seg h, int nc, int64_t max_frames) {
  Ctx* ctx = h->ctx;
  const Params& P = h->P;
  cudaStream_t sA = ctx->stream;
  const int K = (int)((max_frames + kSlice - 1) / kSlice);
  if (K > h->max_slices) fail(LSG_ERUNTIME, "lsg_seg_push: push longer than the slice tables");
  // all slices' chunk tables in one copy
  for (int k = 0; k < K; ++k) {
    int64_t off = 0;
    for (int i = 0; i < nc; ++i) {
      const Chunk& c = h->chunks_host.p[i];
      Chunk& d = h->chunks_sl_host.p[(size_t)k * nc + i];
      d = c;
      const int last = std::max(0, (c.nframes + kSlice - 1) / kSlice - 1);
      const int64_t s0 = (int64_t)k * kSlice * P.fs;
      d.pcm = c.pcm + s0;
      d.n = k < last ? (int64_t)kSlice * P.fs : (k == last ? c.n - s0 : 0);
      d.nframes = k <= last ? std::min(kSlice, c.nframes - k * kSlice) : 0;
      if (d.nframes < 0) d.nframes = 0;
      d.first = k == 0 ? c.first : 0;
      d.frame_off = (int64_t)(k % kSlots) * nc * kSlice + off;
      off += d.nframes;
    }
  }
  LSG_CUDA(cudaMemcpyAsync(h->chunks_sl.p, h->chunks_sl_host.p, sizeof(Chunk) * (size_t)K * nc,
                           cudaMemcpyHostToDevice, sA));
  h->tables_sent(sA);
  if (!h->k1a) {
    LSG_CUDA(cudaEventCreate(&h->k1a));
    LSG_CUDA(cudaEventCreate(&h->k1b));
  }
  auto& g = h->graphs[std::make_pair(nc, K)];
  if (!g.exec) {
    // capture on a private stream (the context stream may be the legacy
    // stream, which cannot capture): sB / sC fork from it and join back
    if (!h->cap) LSG_CUDA(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
    cudaStream_t cs = h->cap;
    LSG_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    struct EndOnError {  // a failure inside the capture must not leave the stream capturing
      cudaStream_t st;
      bool armed = true;
      ~EndOnError() {
        if (!armed) return;
        cudaGraph_t gr = nullptr;
        cudaStreamEndCapture(st, &gr);
        if (gr) cudaGraphDestroy(gr);
        cudaGetLastError();
      }
    } guard_capture{cs};
    LSG_CUDA(cudaEventRecord(h->eJoin, cs));
    LSG_CUDA(cudaStreamWaitEvent(h->sB, h->eJoin, 0));
    LSG_CUDA(cudaStreamWaitEvent(h->sC, h->eJoin, 0));
    const unsigned g2 = (unsigned)ceil_div(nc, K2_LANES);
    const int row_words = kSlice / 32 + 1;
    int kernels = 0;
    for (int k = 0; k < K; ++k) {
      const int j = k % kSlots;
      const Chunk* tab = h->chunks_sl.p + (size_t)k * nc;
      if (k >= kSlots) LSG_CUDA(cudaStreamWaitEvent(cs, h->eM[j], 0));  // slot free
      dim3 grid((unsigned)ceil_div(kSlice, K1_WARPS * K1_FPW), (unsigned)nc);
      seg_frame_stats<<<grid, K1_WARPS * 32, 0, cs>>>(tab, h->carry.p, P.fs, h->stats.p);
      LSG_CUDA(cudaEventRecord(h->eK1[j], cs));
      LSG_CUDA(cudaStreamWaitEvent(h->sB, h->eK1[j], 0));
      // the K2 kernels carry the highest priority as a launch attribute, so it
      // survives into the graph's nodes (stream priorities do not)
      launch_hi(seg_peaks, dim3(g2), dim3(K2_LANES), PK_SMEM, h->sB, h->prio_hi, tab, nc,
                (const FrameStat*)h->stats.p, h->st.p, h->peaks.p, P, j * kSlice);
      LSG_CUDA(cudaEventRecord(h->ePk[j], h->sB));
      LSG_CUDA(cudaStreamWaitEvent(h->sC, h->ePk[j], 0));
      launch_hi(seg_decide, dim3((unsigned)(kSlice / 256), (unsigned)nc), dim3(256), 0, h->sC, h->prio_hi, tab,
                (const FrameStat*)h->stats.p, (const double*)h->peaks.p, h->st.p, h->flags.p, P, j * kSlice,
                j * kSlice / 32);
      launch_hi(seg_machine, dim3((unsigned)ceil_div(nc, MC_WARPS)), dim3(MC_WARPS * 32),
                (size_t)MC_WARPS * row_words * 4, h->sC, h->prio_hi, tab, nc, h->st.p, h->cuts.p,
                (const uint32_t*)h->flags.p, P, row_words, j * kSlice / 32);
      LSG_CUDA(cudaEventRecord(h->eM[j], h->sC));
      kernels += 4;
    }
    // join: the context stream continues after the last machine
    LSG_CUDA(cudaStreamWaitEvent(cs, h->eM[(K - 1) % kSlots], 0));
    LSG_CUDA(cudaStreamWaitEvent(cs, h->ePk[(K - 1) % kSlots], 0));
    seg_carry<<<nc, 256, 0, cs>>>(h->chunks_dev.p, h->carry.p, h->st.p, P.fs);
    kernels += 1;
    cudaGraph_t graph = nullptr;
    guard_capture.armed = false;
    LSG_CUDA(cudaStreamEndCapture(cs, &graph));
    const cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    LSG_CUDA(e);
    g.kernels = kernels;
  }
  LSG_CUDA(cudaEventRecord(h->k1a, sA));
  LSG_CUDA(cudaGraphLaunch(g.exec, sA));
  LSG_CUDA(cudaEventRecord(h->k1b, sA));  // (sliced: K1 overlapped with K2 -- the whole sequence)
  h->k1_recorded = true;
  ctx->launches.fetch_add(g.kernels, std::memory_order_relaxed);
}

extern "C" {

lsg_status lsg_seg_cfg_default(lsg_seg_cfg* c) {
  return guard(__func__, [&] {
    c->mode = 1;
    c->peak_mode = 0;
    c->peak_half_life_ms = 10000.0;
    c->speech_threshold_db = -40.0;
    c->frame_ms = 20;
    c->min_silence_ms = 500;
    c->min_segment_ms = 1500;
    c->max_segment_ms = 10000;
    c->sample_rate = 16000;
    c->flags_only = 0;
  });
}

lsg_status lsg_seg_create(lsg_ctx ctx, const lsg_seg_cfg* cfg, int32_t n_streams,
                          int64_t max_push_samples, lsg_seg* out) {
  return guard(__func__, [&] {
    *out = nullptr;
    validate_cfg(cfg);
    if (n_streams <= 0 || n_streams > kMaxCollect) invalid("lsg_seg_create: n_streams out of range");
    if (max_push_samples <= 0) invalid("lsg_seg_create: max_push_samples must be positive");
    DeviceGuard g(ctx);
    auto h = new lsg_seg_s();
    try {
      h->ctx = ctx;
      Params& P = h->P;
      P.mode = cfg->mode;
      P.peak_mode = cfg->peak_mode;
      P.decay = std::exp2(-double(cfg->frame_ms) / cfg->peak_half_life_ms);  // vad.cpp:37
      P.thr = cfg->speech_threshold_db;
      if (P.thr > -119.0 && P.thr < 300.0) {
        const double xs = std::pow(10.0, P.thr / 20.0);
        P.x_lo = xs * (1.0 - 1e-9);
        P.x_hi = xs * (1.0 + 1e-9);
      } else {
        P.x_lo = 0.0;
        P.x_hi = INFINITY;
      }
      P.frame_ms = cfg->frame_ms;
      P.min_sil = cfg->min_silence_ms;
      P.min_seg = cfg->min_segment_ms;
      P.max_seg = cfg->max_segment_ms;
      P.rate = cfg->sample_rate;
      const int64_t fs = int64_t(cfg->sample_rate) * cfg->frame_ms / 1000;
      if (fs > (1 << 24)) invalid("segmenter: frame too long");
      P.fs = (int32_t)fs;
      P.flags_only = cfg->flags_only ? 1 : 0;
      h->n_streams = n_streams;
      h->max_push = max_push_samples;
      h->max_frames_push = (max_push_samples + fs) / fs + 1;
      P.cut_cap = (int32_t)std::min<int64_t>(2 * h->max_frames_push + 2, INT32_MAX);  // <= 2 cuts/frame
      P.flag_words = (int32_t)((h->max_frames_push + 31) / 32);
      P.pk_stride = (int32_t)((h->max_frames_push + 2) & ~int64_t(1));
      h->hs.resize(n_streams);
      h->st.alloc(n_streams);
      LSG_CUDA(cudaMemsetAsync(h->st.p, 0, h->st.bytes(), ctx->stream));
      if (cfg->peak_mode == 2) {
        std::vector<DevState> init(n_streams);
        std::memset(init.data(), 0, init.size() * sizeof(DevState));
        for (auto& d : init) d.peak = 32767.0;  // vad.cpp:22-24
        LSG_CUDA(cudaMemcpy(h->st.p, init.data(), h->st.bytes(), cudaMemcpyHostToDevice));
      }
      for (auto& d : h->hs) d = StreamHost{};
      h->carry.alloc((size_t)n_streams * fs);
      h->cuts.alloc((size_t)n_streams * P.cut_cap);
      h->flags.alloc((size_t)n_streams * P.flag_words);
      h->stats.alloc((size_t)n_streams * h->max_frames_push);
      h->peaks.alloc((size_t)n_streams * P.pk_stride);
      h->chunks_dev.alloc(n_streams);
      // each staged chunk starts 64-sample (128 B) aligned: <= one chunk per
      // stream per push, each rounded up to 64 samples
      h->staging.alloc((size_t)n_streams * (size_t)((max_push_samples + 63) & ~int64_t(63)) + 64);
      h->streams_dev.alloc(n_streams);
      h->collect_dev.alloc(n_streams);
      h->collect_off.alloc(n_streams + 1);
      h->totals_dev.alloc(n_streams);
      h->chunks_host.alloc(n_streams);
      h->streams_host.alloc(n_streams);
      h->collect_host.alloc(n_streams);
      h->totals_host.alloc(n_streams);
      h->dirty.assign(n_streams, 0);
      h->cut_bound.assign(n_streams, 0);
      LSG_CUDA(cudaEventCreateWithFlags(&h->tab_ev, cudaEventDisableTiming));
      if (h->max_frames_push >= kSlots * kSlice) {
        h->max_slices = (int)((h->max_frames_push + kSlice - 1) / kSlice);
        h->chunks_sl.alloc((size_t)n_streams * h->max_slices);
        h->chunks_sl_host.alloc((size_t)n_streams * h->max_slices);
        // the sequential K2 work is latency-bound on a few SMs: its CTAs get
        // the highest priority so that they are dispatched as soon as a
        // (short) K1 CTA retires instead of after the whole K1 grid
        int lo = 0, hi = 0;
        LSG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        h->prio_hi = hi;
        LSG_CUDA(cudaStreamCreateWithPriority(&h->sB, cudaStreamNonBlocking, hi));
        LSG_CUDA(cudaStreamCreateWithPriority(&h->sC, cudaStreamNonBlocking, hi));
        for (int j = 0; j < kSlots; ++j) {
          LSG_CUDA(cudaEventCreateWithFlags(&h->eK1[j], cudaEventDisableTiming));
          LSG_CUDA(cudaEventCreateWithFlags(&h->ePk[j], cudaEventDisableTiming));
          LSG_CUDA(cudaEventCreateWithFlags(&h->eM[j], cudaEventDisableTiming));
        }
        LSG_CUDA(cudaEventCreateWithFlags(&h->eJoin, cudaEventDisableTiming));
      }
      h->h_cut_cap = (int64_t)n_streams * P.cut_cap;
      LSG_CUDA(cudaHostAlloc(&h->h_state, sizeof(DevState) * n_streams, cudaHostAllocMapped));
      LSG_CUDA(cudaHostAlloc(&h->h_off, sizeof(int32_t) * (n_streams + 1), cudaHostAllocMapped));
      LSG_CUDA(cudaHostAlloc(&h->h_cuts, sizeof(lsg_cut) * h->h_cut_cap, cudaHostAllocMapped));
      LSG_CUDA(cudaHostAlloc(&h->h_flags, sizeof(uint32_t) * (size_t)n_streams * P.flag_words,
                             cudaHostAllocMapped));
      ctx->sync();
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

lsg_status lsg_seg_reset(lsg_seg h) {
  return guard(__func__, [&] {
    Ctx* ctx = h->ctx;
    DeviceGuard g(ctx);
    std::vector<DevState> init(h->n_streams);
    std::memset(init.data(), 0, init.size() * sizeof(DevState));
    if (h->P.peak_mode == 2)
      for (auto& d : init) d.peak = 32767.0;  // vad.cpp:22-24
    LSG_CUDA(cudaMemcpyAsync(h->st.p, init.data(), h->st.bytes(), cudaMemcpyHostToDevice, ctx->stream));
    ctx->sync();
    for (auto& d : h->hs) d = StreamHost{};
    h->dirty.assign(h->n_streams, 0);
    h->cut_bound.assign(h->n_streams, 0);
    h->dirty_list.clear();
  });
}

// Time slicing of long device-resident pushes on (1, default) or off (0):
// off measures K1 alone (lsgdbg_seg_k1_ms) for the HBM roofline.
lsg_status lsgdbg_seg_slicing(lsg_seg h, int32_t on) {
  return guard(__func__, [&] { h->slicing = on != 0; });
}

// Device time (ms) of the last push's frame-statistics kernel (K1; for a
// time-sliced push, the whole overlapped K1 + K2 sequence).
lsg_status lsgdbg_seg_k1_ms(lsg_seg h, float* ms) {
  return guard(__func__, [&] {
    if (!h || !ms) invalid("lsgdbg_seg_k1_ms: null argument");
    if (!h->k1_recorded) logic("lsgdbg_seg_k1_ms: no push with frames yet");
    DeviceGuard g(h->ctx);
    LSG_CUDA(cudaEventSynchronize(h->k1b));
    LSG_CUDA(cudaEventElapsedTime(ms, h->k1a, h->k1b));
  });
}

// Host-side split of the last collection (ms): waiting in its stream
// synchronisation, distributing the cuts / state to the per-stream mirrors.
lsg_status lsgdbg_seg_collect_ms(lsg_seg h, double* wait_ms, double* host_ms) {
  return guard(__func__, [&] {
    if (!h || !wait_ms || !host_ms) invalid("lsgdbg_seg_collect_ms: null argument");
    *wait_ms = h->collect_wait_ms;
    *host_ms = h->collect_host_ms;
  });
}

lsg_status lsg_seg_destroy(lsg_seg h) {
  return guard(__func__, [&] {
    if (!h) return;
    DeviceGuard g(h->ctx);
    h->ctx->sync();
    delete h;
  });
}

lsg_status lsg_seg_push(lsg_seg h, int32_t n_chunks, const int32_t* streams, const int16_t* const* pcm,
                        const int64_t* n_samples, const int64_t* start_ms, int32_t sample_rate,
                        int32_t pcm_on_device) {
  return guard(__func__, [&] {
    Ctx* ctx = h->ctx;
    const Params& P = h->P;
    if (n_chunks < 0 || n_chunks > h->n_streams) invalid("lsg_seg_push: bad chunk count");
    // pass 1: the reference's discipline checks (segmenter.cpp:26-38), all
    // chunks before any state changes
    std::vector<char> seen(h->n_streams, 0);
    for (int i = 0; i < n_chunks; ++i) {
      const int s = streams[i];
      if (s < 0 || s >= h->n_streams) invalid("lsg_seg_push: stream id out of range");
      if (seen[s]) invalid("lsg_seg_push: stream listed twice in one push");
      seen[s] = 1;
      const StreamHost& S = h->hs[s];
      if (S.finished) logic("segmenter: push after finish");
      if (sample_rate != P.rate) invalid("segmenter: sample rate mismatch");
      if (n_samples[i] < 0 || n_samples[i] > h->max_push) invalid("lsg_seg_push: chunk longer than max_push_samples");
      if (n_samples[i] == 0) continue;
      const int64_t staged_ms = S.consumed * P.frame_ms + S.stage_len * 1000 / P.rate;
      const bool first = S.consumed == 0 && S.stage_len == 0;
      if (!first && std::llabs(start_ms[i] - (S.base + staged_ms)) > 1)
        invalid("segmenter: non-contiguous chunk");
    }
    DeviceGuard g(ctx);
    // uncollected cuts of a stream must fit its device cut buffer: <= 2 per
    // frame (a pause cut and a forced split) + the EOS cut
    for (int i = 0; i < n_chunks; ++i) {
      const int s = streams[i];
      const int64_t fr = (h->hs[s].stage_len + n_samples[i]) / P.fs;
      if (h->cut_bound[s] + 2 * fr + 1 > P.cut_cap) {
        collect(h, false);
        break;
      }
    }
    // time-sliced processing (launch_sliced): long device-resident pushes
    // with no sub-frame carry, outside the scorer (flags) mode
    bool sliced = h->max_slices > 0 && !P.flags_only && h->slicing;
    int64_t longest = 0;
    for (int i = 0; i < n_chunks && sliced; ++i) {
      const StreamHost& S = h->hs[streams[i]];
      if (S.stage_len != 0 || !(pcm_on_device || is_device_ptr(pcm[i])) ||
          (reinterpret_cast<uintptr_t>(pcm[i]) & 15) != 0)
        sliced = false;
      longest = std::max<int64_t>(longest, n_samples[i] / P.fs);
    }
    sliced = sliced && longest >= 2 * kSlice;
    h->tables_free();
    // pass 2: stage + describe chunks
    int nc = 0;
    int64_t frame_total = 0, max_frames = 0, stage_off = 0;
    for (int i = 0; i < n_chunks; ++i) {
      if (n_samples[i] == 0) continue;
      const int s = streams[i];
      StreamHost& S = h->hs[s];
      Chunk& c = h->chunks_host.p[nc];
      const bool first = S.consumed == 0 && S.stage_len == 0;
      const int16_t* src = pcm[i];
      if (!pcm_on_device && !is_device_ptr(src)) {
        int16_t* dst = h->staging.p + stage_off;
        if (stage_off + n_samples[i] > (int64_t)h->staging.n) fail(LSG_ERUNTIME, "lsg_seg_push: staging overflow");
        LSG_CUDA(cudaMemcpyAsync(dst, src, n_samples[i] * 2, cudaMemcpyHostToDevice, ctx->stream));
        src = dst;
        stage_off += (n_samples[i] + 63) & ~int64_t(63);  // keep 128 B alignment
      }
      c.pcm = src;
      c.n = n_samples[i];
      c.frame_off = frame_total;
      c.start_ms = start_ms[i];
      c.stream = s;
      c.carry_len = (int32_t)S.stage_len;
      c.first = first ? 1 : 0;
      const int64_t tot = S.stage_len + n_samples[i];
      c.nframes = (int32_t)(tot / P.fs);
      c.total_after = S.total + n_samples[i];
      frame_total += c.nframes;
      max_frames = std::max<int64_t>(max_frames, c.nframes);
      h->streams_host.p[nc] = s;
      h->cut_bound[s] += 2 * (int64_t)c.nframes;
      if (!h->dirty[s]) {
        h->dirty[s] = 1;
        h->dirty_list.push_back(s);
      }
      // host mirror
      if (first) S.base = start_ms[i];
      S.consumed += c.nframes;
      S.stage_len = tot % P.fs;
      S.total += n_samples[i];
      ++nc;
    }
    for (int i = 0; i < n_chunks; ++i) {
      StreamHost& S = h->hs[streams[i]];
      S.flags.clear();
    }
    if (nc == 0) return;
    LSG_CUDA(cudaMemcpyAsync(h->chunks_dev.p, h->chunks_host.p, sizeof(Chunk) * nc, cudaMemcpyHostToDevice,
                             ctx->stream));
    LSG_CUDA(cudaMemcpyAsync(h->streams_dev.p, h->streams_host.p, sizeof(int32_t) * nc,
                             cudaMemcpyHostToDevice, ctx->stream));
    if (!sliced) h->tables_sent(ctx->stream);
    if (max_frames > 0 && !sliced) {
      dim3 grid((unsigned)ceil_div(max_frames, K1_WARPS * K1_FPW), (unsigned)nc);
      if (!h->k1a) {
        LSG_CUDA(cudaEventCreate(&h->k1a));
        LSG_CUDA(cudaEventCreate(&h->k1b));
      }
      LSG_CUDA(cudaEventRecord(h->k1a, ctx->stream));
      seg_frame_stats<<<grid, K1_WARPS * 32, 0, ctx->stream>>>(h->chunks_dev.p, h->carry.p, P.fs,
                                                               h->stats.p);
      LSG_LAUNCHED(ctx);
      LSG_CUDA(cudaEventRecord(h->k1b, ctx->stream));
      h->k1_recorded = true;
    }
    if (!h->attrs_set) {  // per handle: kernel attributes are per device
      LSG_CUDA(cudaFuncSetAttribute(seg_peaks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PK_SMEM));
      LSG_CUDA(cudaFuncSetAttribute(seg_machine, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      h->attrs_set = true;
    }
    if (sliced) {
      launch_sliced(h, nc, max_frames);
      if (P.flags_only) collect(h, false);
      return;
    }
    const unsigned g2 = (unsigned)ceil_div(nc, K2_LANES);
    seg_peaks<<<g2, K2_LANES, PK_SMEM, ctx->stream>>>(h->chunks_dev.p, nc, h->stats.p, h->st.p, h->peaks.p, P, 0);
    LSG_LAUNCHED(ctx);
    if (max_frames > 0) {
      seg_decide<<<dim3((unsigned)ceil_div(max_frames, 256), (unsigned)nc), 256, 0, ctx->stream>>>(
          h->chunks_dev.p, h->stats.p, h->peaks.p, h->st.p, h->flags.p, P, 0, 0);
      LSG_LAUNCHED(ctx);
    }
    const int row_words = (int)((max_frames + 31) / 32) | 1;
    if ((size_t)MC_WARPS * row_words * 4 > 200 * 1024) fail(LSG_ERUNTIME, "lsg_seg_push: push too long for K2c");
    seg_machine<<<(unsigned)ceil_div(nc, MC_WARPS), MC_WARPS * 32, (size_t)MC_WARPS * row_words * 4, ctx->stream>>>(
        h->chunks_dev.p, nc, h->st.p, h->cuts.p, h->flags.p, P, row_words, 0);
    LSG_LAUNCHED(ctx);
    seg_carry<<<nc, 256, 0, ctx->stream>>>(h->chunks_dev.p, h->carry.p, h->st.p, P.fs);
    LSG_LAUNCHED(ctx);
    // per-push flags feed the host state machine (scorer order): collect now;
    // otherwise the results stay on the device until they are asked for
    if (P.flags_only) collect(h, false);
  });
}

lsg_status lsg_seg_finish(lsg_seg h, int32_t n, const int32_t* streams) {
  return guard(__func__, [&] {
    Ctx* ctx = h->ctx;
    if (n < 0 || n > h->n_streams) invalid("lsg_seg_finish: bad stream count");
    std::vector<char> seen(h->n_streams, 0);
    for (int i = 0; i < n; ++i) {
      const int s = streams[i];
      if (s < 0 || s >= h->n_streams) invalid("lsg_seg_finish: stream id out of range");
      if (seen[s]) invalid("lsg_seg_finish: stream listed twice");
      seen[s] = 1;
      if (h->hs[s].finished) logic("segmenter: finish twice");
    }
    if (n == 0) return;
    DeviceGuard g(ctx);
    h->tables_free();
    for (int i = 0; i < n; ++i) {
      const int s = streams[i];
      h->streams_host.p[i] = s;
      h->totals_host.p[i] = h->hs[s].total;
      h->hs[s].finished = true;
      h->hs[s].stage_len = 0;
      if (!h->dirty[s]) {
        h->dirty[s] = 1;
        h->dirty_list.push_back(s);
      }
    }
    LSG_CUDA(cudaMemcpyAsync(h->streams_dev.p, h->streams_host.p, sizeof(int32_t) * n, cudaMemcpyHostToDevice,
                             ctx->stream));
    LSG_CUDA(cudaMemcpyAsync(h->totals_dev.p, h->totals_host.p, sizeof(int64_t) * n, cudaMemcpyHostToDevice,
                             ctx->stream));
    seg_finish<<<(unsigned)ceil_div(n, 128), 128, 0, ctx->stream>>>(h->streams_dev.p, h->totals_dev.p, n,
                                                                    h->st.p, h->cuts.p, h->P);
    LSG_LAUNCHED(ctx);
    collect(h, true);  // one synchronisation for every stream's remaining cuts
  });
}

lsg_status lsg_seg_take_cuts(lsg_seg h, int32_t stream, lsg_cut* out, int64_t cap, int64_t* n_out) {
  return guard(__func__, [&] {
    if (stream < 0 || stream >= h->n_streams) invalid("lsg_seg_take_cuts: stream id out of range");
    if (h->dirty[stream]) {
      DeviceGuard g(h->ctx);
      collect(h, false);
    }
    auto& v = h->hs[stream].cuts;
    *n_out = (int64_t)v.size();
    if ((int64_t)v.size() > cap) return;
    if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(lsg_cut));
    v.clear();
  });
}

lsg_status lsg_seg_take_all_cuts(lsg_seg h, lsg_cut* out, int64_t cap, int64_t* n_out) {
  return guard(__func__, [&] {
    if (!h->dirty_list.empty()) {
      DeviceGuard g(h->ctx);
      collect(h, false);
    }
    int64_t tot = 0;
    for (auto& s : h->hs) tot += (int64_t)s.cuts.size();
    *n_out = tot;
    if (tot > cap) return;
    int64_t k = 0;
    for (auto& s : h->hs) {
      if (!s.cuts.empty()) std::memcpy(out + k, s.cuts.data(), s.cuts.size() * sizeof(lsg_cut));
      k += (int64_t)s.cuts.size();
      s.cuts.clear();
    }
  });
}

lsg_status lsg_seg_get_metrics(lsg_seg h, int32_t stream, lsg_seg_metrics* out) {
  return guard(__func__, [&] {
    if (stream < 0 || stream >= h->n_streams) invalid("lsg_seg_get_metrics: stream id out of range");
    if (h->dirty[stream]) {
      DeviceGuard g(h->ctx);
      collect(h, false);
    }
    *out = h->hs[stream].metrics;
  });
}

lsg_status lsg_seg_take_flags(lsg_seg h, int32_t stream, uint8_t* speech, int64_t cap, int64_t* n_out) {
  return guard(__func__, [&] {
    if (stream < 0 || stream >= h->n_streams) invalid("lsg_seg_take_flags: stream id out of range");
    if (!h->P.flags_only) logic("lsg_seg_take_flags: handle was not created with flags_only");
    auto& v = h->hs[stream].flags;
    *n_out = (int64_t)v.size();
    if ((int64_t)v.size() > cap) return;
    if (!v.empty()) std::memcpy(speech, v.data(), v.size());
    v.clear();
  });
}

}  // extern "C"
