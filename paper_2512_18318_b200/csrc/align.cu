// align.cu -- A/V alignment on sm_100a (include/lsg.h "alignment";
// SURVEY.md §8 row f2).
//
// Replaces align.cpp: energy_envelope_ms (align.cpp:10-32),
// motion_envelope_ms (:34-50) and align_envelopes (:52-116), batched over
// many segments / pairs per call.  Every floating-point sum keeps the
// reference's sequential order and uses round-to-nearest intrinsics (no
// FMA contraction, like the reference's x86-64 build), so the envelopes,
// offsets and correlations are bit-identical to the reference's:
//   energy   one warp per 32 hops of a segment (coalesced staging), one lane
//            per 10 ms hop (its 160-sample sum is sequential);
//   motion   one thread per millisecond, binary search over frame times;
//   NCC      one CTA per pair, one thread per lag: each lag's mean /
//            variance / dot sums run sequentially over t in its own thread
//            (threads of neighbouring lags read neighbouring motion samples,
//            so the loads coalesce); the energy statistics once per CTA; the
//            argmax with the reference's tie rule sequentially over lags.
// The work is tiny next to the generator (101 lags x D ms per segment), so
// the kernels are latency-bound; they exist so alignment stays on the
// device with the audio and the frame records.
#include <algorithm>
#include <cmath>
#include <vector>

#include "lsg_common.cuh"

namespace lsg {
namespace align {

constexpr int kMaxLag = 511;  // 2 * max_lag + 1 threads per CTA

// hop h of the batch -> (segment, hop within segment) by binary search over hop0
__device__ __forceinline__ int find_seg(const int64_t* __restrict__ first, int n, int64_t x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(first + mid) <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// tab: [n] pcm_off | [n] n_samples | [n] out_off | [n] total_ms | [n+1] chunk0
// One warp per 32 consecutive hops of one segment: the warp stages the
// chunk's PCM into shared memory with coalesced loads (16-byte vectors when
// aligned), then each lane sums its own hop in the reference's order.
constexpr int EW = 4;  // warps per CTA (41 KB staged: 5 CTAs = 20 warps per SM)
__global__ void __launch_bounds__(EW * 32) energy_kernel(const int16_t* __restrict__ pcm, const int64_t* __restrict__ tab,
                                                         int n, int64_t total_chunks, int hop_samples,
                                                         double* __restrict__ out) {
  // staged as 32 rows (one per hop) of hop_samples + 2 int16: an odd number
  // of 4-byte words per row, so the lanes' per-hop reads are conflict-free
  extern __shared__ __align__(16) int16_t stage[];  // [EW][32][hop_samples + 2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ch = (int64_t)blockIdx.x * EW + warp;
  if (ch >= total_chunks) return;
  const int64_t* chunk0 = tab + 4 * n;
  const int s = find_seg(chunk0, n, ch);
  const int64_t pcm_off = __ldg(tab + s), ns = __ldg(tab + n + s), out_off = __ldg(tab + 2 * n + s);
  const int64_t total = __ldg(tab + 3 * n + s);
  const int64_t hop_first = (ch - __ldg(chunk0 + s)) * 32;
  const int64_t s_begin = hop_first * hop_samples;
  const int64_t s_end = min(ns, s_begin + 32 * (int64_t)hop_samples);
  const int row = hop_samples + 2;
  int16_t* buf = stage + warp * 32 * row;
  const int16_t* x = pcm + pcm_off;
  const int64_t cnt = s_end - s_begin;
  if ((((uintptr_t)(x + s_begin)) & 15) == 0 && (hop_samples & 7) == 0) {
    const int4* src = reinterpret_cast<const int4*>(x + s_begin);
    const int nv = (int)(cnt >> 3), per_row = hop_samples >> 3;
    // 16 loads per lane in flight before any store (a load-store loop
    // serialised one DRAM round trip per 512 B of the warp's 10 KB)
    for (int q0 = 0; q0 < nv; q0 += 32 * 16) {
      int4 v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int q = q0 + lane + 32 * u;
        if (q < nv) v[u] = __ldg(src + q);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int q = q0 + lane + 32 * u;
        if (q < nv) {
          const int r = q / per_row, c = (q - r * per_row) * 8;
          uint32_t* d = reinterpret_cast<uint32_t*>(buf + r * row + c);  // 4-byte aligned (row is even)
          d[0] = (uint32_t)v[u].x;
          d[1] = (uint32_t)v[u].y;
          d[2] = (uint32_t)v[u].z;
          d[3] = (uint32_t)v[u].w;
        }
      }
    }
    for (int64_t i = (int64_t)nv * 8 + lane; i < cnt; i += 32) buf[(i / hop_samples) * row + i % hop_samples] = __ldg(x + s_begin + i);
  } else {
    for (int64_t i = lane; i < cnt; i += 32) buf[(i / hop_samples) * row + i % hop_samples] = __ldg(x + s_begin + i);
  }
  __syncwarp();
  const int64_t t = (hop_first + lane) * 10;
  if (t >= total) return;
  const int64_t s0 = t / 10 * hop_samples;
  const int64_t s1 = min(ns, s0 + hop_samples);
  double sumsq = 0.0;
  for (int64_t i = s0; i < s1; ++i) {
    const double v = __dmul_rn((double)buf[lane * row + (i - s0)], 0x1p-15);  // == s / 32768.0 exactly
    sumsq = __dadd_rn(sumsq, __dmul_rn(v, v));
  }
  const double rms = s1 > s0 ? __dsqrt_rn(__ddiv_rn(sumsq, (double)(s1 - s0))) : 0.0;
  const int64_t e = min(t + 10, total);
  for (int64_t k = t; k < e; ++k) out[out_off + k] = rms;
}

// tab: [n] frame_off | [n] n_frames | [n] t0 | [n] span | [n] out_off | [n+1] ms0
__global__ void motion_kernel(const int64_t* __restrict__ ts, const double* __restrict__ motion,
                              const int64_t* __restrict__ tab, int n, int64_t total_ms, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total_ms) return;
  const int64_t* ms0 = tab + 5 * n;
  const int s = find_seg(ms0, n, i);
  const int64_t f0 = __ldg(tab + s), nf = __ldg(tab + n + s), t0 = __ldg(tab + 2 * n + s);
  const int64_t t = i - __ldg(ms0 + s);
  // last frame with ts <= t0 + t (frames sorted by ts; the reference's
  // while-loop consumes them in order, so the held value is the last such)
  int64_t lo = 0, hi = nf;  // first index with ts > t0 + t
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(ts + f0 + mid) <= t0 + t) lo = mid + 1;
    else hi = mid;
  }
  out[__ldg(tab + 4 * n + s) + t] = lo > 0 ? __ldg(motion + f0 + lo - 1) : 0.0;
}

// tab: [n] e_off | [n] e_len | [n] m_off | [n] m_len
__global__ void __launch_bounds__(1024) ncc_kernel(const double* __restrict__ e_base, const double* __restrict__ m_base,
                                                   const int64_t* __restrict__ tab, int n, int max_lag,
                                                   lsg_align_result* __restrict__ out) {
  __shared__ double s_corr[2 * kMaxLag + 1];
  __shared__ int s_ok[2 * kMaxLag + 1];
  __shared__ double s_emean, s_esigma;
  __shared__ int s_state;  // 0 ok, 1 low confidence
  const int p = blockIdx.x;
  const double* e = e_base + __ldg(tab + p);
  const double* m = m_base + __ldg(tab + 2 * n + p);
  const int64_t d = min(__ldg(tab + n + p), __ldg(tab + 3 * n + p));
  const int64_t lo = max_lag, hi = d - max_lag;
  const int nl = 2 * max_lag + 1;
  if (threadIdx.x == 0) {
    s_state = 0;
    if (hi - lo < 2) {
      s_state = 1;
    } else {
      const double nn = (double)(hi - lo);
      double em = 0.0;
      for (int64_t t = lo; t < hi; ++t) em = __dadd_rn(em, __ldg(e + t));
      em = __ddiv_rn(em, nn);
      double ev = 0.0;
      for (int64_t t = lo; t < hi; ++t) {
        const double v = __dsub_rn(__ldg(e + t), em);
        ev = __dadd_rn(ev, __dmul_rn(v, v));
      }
      s_emean = em;
      s_esigma = __dsqrt_rn(ev);
      if (s_esigma < 1e-12) s_state = 1;
    }
  }
  __syncthreads();
  if (s_state) {
    if (threadIdx.x == 0) out[p] = lsg_align_result{0, 0.0, 1, 0};
    return;
  }
  const double nn = (double)(hi - lo), em = s_emean, es = s_esigma;
  for (int j = threadIdx.x; j < nl; j += blockDim.x) {
    const int lag = j - max_lag;
    double mm = 0.0;
    for (int64_t t = lo; t < hi; ++t) mm = __dadd_rn(mm, __ldg(m + t + lag));
    mm = __ddiv_rn(mm, nn);
    double mv = 0.0, dot = 0.0;
    for (int64_t t = lo; t < hi; ++t) {
      const double me = __dsub_rn(__ldg(m + t + lag), mm);
      mv = __dadd_rn(mv, __dmul_rn(me, me));
      dot = __dadd_rn(dot, __dmul_rn(__dsub_rn(__ldg(e + t), em), me));
    }
    const double ms = __dsqrt_rn(mv);
    s_ok[j] = ms >= 1e-12;
    s_corr[j] = s_ok[j] ? __ddiv_rn(dot, __dmul_rn(es, ms)) : 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // the reference's scan order and tie rule (align.cpp:97-107)
    bool any = false;
    double best = 0.0;
    int best_lag = 0;
    for (int j = 0; j < nl; ++j) {
      if (!s_ok[j]) continue;
      const int lag = j - max_lag;
      const double corr = s_corr[j];
      bool better = !any || corr > best;
      if (any && corr == best) better = abs(lag) < abs(best_lag) || (abs(lag) == abs(best_lag) && lag < best_lag);
      if (better) {
        any = true;
        best = corr;
        best_lag = lag;
      }
    }
    out[p] = any ? lsg_align_result{best_lag, best, 0, 0} : lsg_align_result{0, 0.0, 1, 0};
  }
}

}  // namespace align
}  // namespace lsg

using namespace lsg;
using namespace lsg::align;

namespace {

using Scratch = ScratchLease;

}  // namespace

extern "C" {

lsg_status lsg_align_energy(lsg_ctx ctx, int32_t n, const int16_t* pcm_base, const int64_t* pcm_off,
                            const int64_t* n_samples, int32_t sample_rate, double* out_base, const int64_t* out_off,
                            int64_t* out_len) {
  return guard(__func__, [&] {
    if (n < 0) invalid("lsg_align_energy: negative count");
    if (sample_rate <= 0) invalid("AudioBuffer: bad sample rate");
    const int hop = (int)((int64_t)sample_rate * 10 / 1000);
    if (hop <= 0) invalid("align: rate too low");  // align.cpp:18
    // the energy kernel stages EW warps x 32 hops of PCM in shared memory
    if ((size_t)EW * 32 * (hop + 2) * sizeof(int16_t) > (size_t)ctx->smem_optin)
      invalid("lsg_align_energy: sample rate too high for the shared-memory staging (max hop " +
              std::to_string(ctx->smem_optin / (EW * 32 * 2) - 2) + " samples)");
    std::vector<int64_t> tab(5 * (size_t)n + 1);
    int64_t chunks = 0;
    for (int i = 0; i < n; ++i) {
      if (n_samples[i] < 0) invalid("lsg_align_energy: negative length");
      const int64_t total = std::llround(1000.0 * (double)n_samples[i] / sample_rate);  // audio.cpp:8-12
      out_len[i] = total;
      tab[i] = pcm_off[i];
      tab[n + i] = n_samples[i];
      tab[2 * n + i] = out_off[i];
      tab[3 * n + i] = total;
      tab[4 * n + i] = chunks;
      chunks += ((total + 9) / 10 + 31) / 32;
    }
    tab[5 * (size_t)n] = chunks;
    if (chunks == 0) return;
    DeviceGuard g(ctx);
    Scratch sc(ctx, tab.size() * 8);
    LSG_CUDA(cudaMemcpyAsync(sc.p, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    const size_t smem = (size_t)EW * 32 * (hop + 2) * sizeof(int16_t);
    if (smem > 48 * 1024)
      LSG_CUDA(cudaFuncSetAttribute(energy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    energy_kernel<<<(unsigned)ceil_div(chunks, EW), EW * 32, smem, ctx->stream>>>(
        pcm_base, static_cast<int64_t*>(sc.p), n, chunks, hop, out_base);
    LSG_LAUNCHED(ctx);
    ctx->sync();  // the table is host-staged per call
  });
}

lsg_status lsg_align_motion(lsg_ctx ctx, int32_t n, const int64_t* ts_base, const double* motion_base,
                            const int64_t* frame_off, const int64_t* n_frames, const int64_t* t0, const int64_t* span,
                            double* out_base, const int64_t* out_off) {
  return guard(__func__, [&] {
    if (n < 0) invalid("lsg_align_motion: negative count");
    std::vector<int64_t> tab(6 * (size_t)n + 1);
    int64_t ms = 0;
    for (int i = 0; i < n; ++i) {
      if (span[i] < 0) invalid("align: negative span");  // align.cpp:36
      if (n_frames[i] < 0) invalid("lsg_align_motion: negative frame count");
      tab[i] = frame_off[i];
      tab[n + i] = n_frames[i];
      tab[2 * n + i] = t0[i];
      tab[3 * n + i] = span[i];
      tab[4 * n + i] = out_off[i];
      tab[5 * n + i] = ms;
      ms += span[i];
    }
    tab[6 * (size_t)n] = ms;
    if (ms == 0) return;
    DeviceGuard g(ctx);
    Scratch sc(ctx, tab.size() * 8);
    LSG_CUDA(cudaMemcpyAsync(sc.p, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    motion_kernel<<<(unsigned)ceil_div(ms, 256), 256, 0, ctx->stream>>>(ts_base, motion_base,
                                                                        static_cast<int64_t*>(sc.p), n, ms, out_base);
    LSG_LAUNCHED(ctx);
    ctx->sync();
  });
}

lsg_status lsg_align_batch(lsg_ctx ctx, int32_t n, const double* energy_base, const int64_t* e_off,
                           const int64_t* e_len, const double* motion_base, const int64_t* m_off, const int64_t* m_len,
                           int64_t max_lag, lsg_align_result* out) {
  return guard(__func__, [&] {
    if (max_lag < 0) invalid("align: negative lag bound");  // align.cpp:55
    if (max_lag > kMaxLag) invalid("lsg_align_batch: max_lag above 511");
    if (n < 0) invalid("lsg_align_batch: negative count");
    if (n == 0) return;
    std::vector<int64_t> tab(4 * (size_t)n);
    for (int i = 0; i < n; ++i) {
      tab[i] = e_off[i];
      tab[n + i] = e_len[i];
      tab[2 * n + i] = m_off[i];
      tab[3 * n + i] = m_len[i];
    }
    DeviceGuard g(ctx);
    Scratch sc(ctx, tab.size() * 8 + (size_t)n * sizeof(lsg_align_result));
    int64_t* dtab = static_cast<int64_t*>(sc.p);
    lsg_align_result* dres = reinterpret_cast<lsg_align_result*>(dtab + tab.size());
    LSG_CUDA(cudaMemcpyAsync(dtab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    const int threads = (int)std::min<int64_t>(1024, ((2 * max_lag + 1 + 31) / 32) * 32);
    ncc_kernel<<<(unsigned)n, threads, 0, ctx->stream>>>(energy_base, motion_base, dtab, n, (int)max_lag, dres);
    LSG_LAUNCHED(ctx);
    LSG_CUDA(cudaMemcpyAsync(out, dres, (size_t)n * sizeof(lsg_align_result), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  });
}

}  // extern "C"
