// conv_kernel.cuh -- persistent implicit-GEMM convolution on tcgen05 + TMA.
//
// One launch = one conv layer (all of its phases).  Grid = one CTA per SM;
// each CTA walks output tiles t = blockIdx.x, +gridDim.x, ... (128 output
// pixels x BN channels).  Warp roles:
//   warp 0     TMA producer (one elected thread): per K stage, im2col TMA
//              loads of the A tile straight from the NHWC activation
//              (cp.async.bulk.tensor.4d ... .im2col: the tensor-map bounding
//              box encodes the conv padding and stride, the per-load offsets
//              the filter tap, out-of-bounds pixels are zero-filled), plus a
//              bulk async copy of the packed weight tile B.
//   warp 1     MMA issuer (one thread): tcgen05.mma kind::f16 (M=128, N=BN,
//              K=16) into one of two TMEM accumulators.
//   warps 2-9  epilogue, two warps per TMEM lane quadrant (each half of the
//              BN columns): tcgen05.ld -> folded-BN bias -> residual -> ReLU ->
//              16-bit store into a channel slice of the destination, or the
//              fused 1x1 32->3 + sigmoid of the output block.  The second TMEM
//              accumulator lets tile i's epilogue overlap tile i+1's mainloop.
//
// A smem layouts by channel chunk CC (the largest of 64/32/16/8 dividing
// Cin): CC=64 -> 128B swizzle, 32 -> 64B, 16 -> 32B, 8 -> no swizzle (two
// 8-channel loads per K=16 step, LBO = 2 KB).  Every A stage is 128 x 64
// 16-bit elements (16 KB); B stays 128B-swizzled 64-wide K blocks.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include <cstdint>

#include "tc.cuh"

namespace lsg {
namespace gen {

// Phase timestamps (globaltimer, ns) per layer and CTA, only in builds with
// -DLSG_TRACE (tools/layer_trace.py): where a layer's time goes.
#ifdef LSG_TRACE
constexpr int TRACE_EV = 16, TRACE_CTAS = 160, TRACE_LAYERS = 64;
__device__ unsigned long long g_lsg_trace[TRACE_LAYERS * TRACE_CTAS * TRACE_EV];
#define LSG_TR(slot, i)                                                                                 \
  do {                                                                                                  \
    unsigned long long t_;                                                                              \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                              \
    if ((slot) >= 0 && blockIdx.x < TRACE_CTAS)                                                         \
      g_lsg_trace[((size_t)(slot) * TRACE_CTAS + blockIdx.x) * TRACE_EV + (i)] = t_;                    \
  } while (0)
// conv_halo's role accounting: clock64 cycles spent in each wait, summed per
// CTA (tools/halo_waits.py): LSG_HW(acc, i, stmt) times stmt into acc[i],
// LSG_HW_FLUSH adds acc[i0, i1) into the layer's per-CTA slots.
#define LSG_HW(acc, i, ...)                        \
  do {                                             \
    const long long t0_ = clock64();               \
    __VA_ARGS__;                                   \
    (acc)[i] += clock64() - t0_;                   \
  } while (0)
#define LSG_HW_FLUSH(slot, acc, i0, i1)                                                                    \
  do {                                                                                                  \
    if ((slot) >= 0 && blockIdx.x < TRACE_CTAS)                                                         \
      for (int i_ = (i0); i_ < (i1); ++i_)                                                              \
        atomicAdd(&g_lsg_trace[((size_t)(slot) * TRACE_CTAS + blockIdx.x) * TRACE_EV + i_],             \
                  (unsigned long long)(acc)[i_]);                                                       \
  } while (0)
#else
#define LSG_TR(slot, i) \
  do {                  \
  } while (0)
#define LSG_HW(acc, i, ...) \
  do {                      \
    __VA_ARGS__;            \
  } while (0)
#define LSG_HW_FLUSH(slot, acc, i0, i1) \
  do {                                  \
  } while (0)
#endif

constexpr int BM = 128;  // UMMA M (TMEM lanes)
constexpr int BK = 64;   // 16-bit elements per K stage
constexpr int MAX_TAPS = 49;
constexpr int MAX_PHASES = 9;
constexpr int NUM_EPI_WARPS = 8;
constexpr int NUM_THREADS = 64 + 32 * NUM_EPI_WARPS;  // TMA warp, MMA warp, epilogue warps
constexpr int OOB_OFFSET = 200;  // im2col offset that always lands outside the input (zero fill)

enum OutMode { OUT_16 = 0, OUT_F32_NCHW = 1, OUT_U8_NHWC = 2, OUT_F32_LOGITS = 3 };

struct Phase {
  const uint16_t* w;  // packed [ntiles][kblocks][BN][64], 128 B swizzled rows
  int ntaps, K;
  int nloads;         // TMA loads of this phase (ntaps * C / CC, +1 pad load for CC = 8)
  int kblocks;        // ceil(nloads / (64 / CC))
  int nsteps;         // MMA K=16 steps, ceil(K / 16)
  int oy, ox;         // output offset of this phase
  int GH, GW;         // GEMM pixel grid of this phase (per image)
  int M, mtiles;      // B * GH * GW, ceil(M / 128)
  int tile0;          // first global tile of this phase
  unsigned char offh[MAX_TAPS + 1], offw[MAX_TAPS + 1];  // im2col offsets per tap (+ pad tap)
};

struct alignas(64) ConvParams {
  CUtensorMap tmap;  // im2col map of the input view; first member (64 B aligned in param space)
  int cc;            // channel chunk per TMA load
  int lower_h, lower_w;
  int H, W, C;
  uint16_t* out;
  int OH, OW, out_pitch, out_coff;
  const uint16_t* res;
  int res_pitch, res_coff;
  const float* bias;
  const float* oscale;  // 8-bit: per output channel s_in * s_w[co] (dequantizes the accumulator), else null
  float res_scale;      // 8-bit: scale of the residual tensor, else 1
  float out_inv;        // 8-bit: 1 / scale of the output tensor, else 1
  int sy, sx, osy, osx;
  int relu, out_mode;
  const float* w1;  // fused output 1x1: [3][32]
  const float* b1;  // [3]
  void* final_out;
  int nphases, ntiles_n, total_tiles;
  int interleave;  // all phases have equal mtiles: t = (mt * nphases + z) * ntiles_n + nt
  // split-K (grid-starved low-resolution layers): work unit u = t * ksplit + ks
  // runs kblocks [ks*KB/ksplit, (ks+1)*KB/ksplit) of tile t and stores its fp32
  // partial into slot ws[u] (layout [BN/4][BM] float4).  The ksplit CTAs of a
  // tile are ONE thread-block cluster (launched with clusterDim.x = ksplit), so
  // the hardware co-schedules them and they meet at a cluster barrier -- never
  // a spin on CTAs that might not be resident (a concurrent kernel on another
  // stream can hold the other SMs); then each reduces 1/ksplit of the tile.
  int ksplit, total_units;
  float* ws;
  int trace_slot;  // layer index (LSG_TRACE builds)
  int pbn;         // tile width the weights are packed for (a multiple of BN: a
                   // BN-wide tile is a contiguous, swizzle-aligned slice of it)
  CUtensorMap wmap;  // the layer's packed weights as 2-D [rows][64] (no swizzle:
                     // the bytes are pre-swizzled), for CTA-pair TMA loads
  int wrow0[MAX_PHASES];  // first weight row of each phase in wmap
  Phase ph[MAX_PHASES];
};

// Element formats.  Activations and weights are always moved as 16-bit
// "units": a bf16/fp16 value, or a PAIR of 8-bit values (fp8 e4m3, or u8
// activations / s8 weights).  One MMA step is 32 bytes of a row in every
// format (kind::f16 K=16, kind::f8f6f4 and kind::i8 K=32), so tensor maps,
// shared-memory layouts, descriptors and K loops are identical across
// formats; only the MMA kind, the weight packing and the epilogue's
// (de)quantisation differ.  The 8-bit formats (Q8) carry per-output-channel
// weight scales and per-tensor activation scales; INT8 accumulates in s32.
enum Prec { PR_BF16 = 0, PR_FP16 = 1, PR_FP8 = 2, PR_I8 = 3 };

template <int PR>
struct Num {
  static constexpr bool Q8 = PR == PR_FP8 || PR == PR_I8;  // 8-bit storage, scaled
  static constexpr bool I8 = PR == PR_I8;
  static constexpr uint32_t kFmt = PR == PR_BF16 ? 1u : 0u;  // bf16 = 1; fp16 = 0; e4m3 = 0
  static constexpr int CPU = Q8 ? 2 : 1;                     // channels per 16-bit unit
  static constexpr int U4 = Q8 ? 1 : 2;                      // uint4 words per 16 channels
  __host__ __device__ static constexpr uint32_t idesc(int M, int N) {
    return I8 ? tc::idesc_i8(M, N) : tc::idesc_f16kind(M, N, kFmt);
  }
  // one TMEM accumulator word as a float (s32 for INT8, f32 otherwise)
  __device__ __forceinline__ static float acc(uint32_t u) {
    if constexpr (I8) return (float)(int32_t)u;
    else return __uint_as_float(u);
  }
  __device__ __forceinline__ static uint32_t pack(float a, float b) {  // 16-bit formats
    if constexpr (PR == PR_FP16) {
      __half2 v = __floats2half2_rn(a, b);
      return *reinterpret_cast<uint32_t*>(&v);
    } else {
      __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
      return *reinterpret_cast<uint32_t*>(&v);
    }
  }
  __device__ __forceinline__ static float2 unpack(uint32_t u) {
    if constexpr (PR == PR_FP16) {
      return __half22float2(*reinterpret_cast<__half2*>(&u));
    } else {
      return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u));
    }
  }
  // 16 channels <-> their U4 uint4 words
  __device__ __forceinline__ static void to_float16(const uint4* w, float (&x)[16]) {
    if constexpr (I8) {
      // byte b -> the float 2^23 + b (PRMT into 0x4B0000bb) - 2^23: full-rate
      // ALU/FMA work instead of the quarter-rate I2F conversion
      const uint32_t r[4] = {w[0].x, w[0].y, w[0].z, w[0].w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          x[4 * k + b] = __uint_as_float(__byte_perm(r[k], 0x4B000000u, 0x7540u + b)) - 8388608.f;
    } else if constexpr (Q8) {
      const uint32_t r[4] = {w[0].x, w[0].y, w[0].z, w[0].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const __half2_raw hr = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(r[k] >> (16 * h)), __NV_E4M3);
          const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&hr));
          x[4 * k + 2 * h] = f.x;
          x[4 * k + 2 * h + 1] = f.y;
        }
      }
    } else {
      const uint32_t r[8] = {w[0].x, w[0].y, w[0].z, w[0].w, w[1].x, w[1].y, w[1].z, w[1].w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float2 f = unpack(r[k]);
        x[2 * k] = f.x;
        x[2 * k + 1] = f.y;
      }
    }
  }
  __device__ __forceinline__ static void from_float16(const float (&f)[16], uint4* w) {
    if constexpr (I8) {
      // u8: saturate to [0, 255], round to nearest even by adding 2^23 (the
      // code lands in the low mantissa byte), pack the four low bytes with
      // PRMTs -- no quarter-rate F2I
      uint32_t r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t q[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) q[b] = __float_as_uint(fminf(fmaxf(f[4 * k + b], 0.f), 255.f) + 8388608.f);
        r[k] = __byte_perm(__byte_perm(q[0], q[1], 0x0040u), __byte_perm(q[2], q[3], 0x0040u), 0x5410u);
      }
      w[0] = make_uint4(r[0], r[1], r[2], r[3]);
    } else if constexpr (Q8) {
      uint32_t r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2(f[4 * k], f[4 * k + 1]), __NV_SATFINITE, __NV_E4M3);
        const uint32_t hi =
            __nv_cvt_float2_to_fp8x2(make_float2(f[4 * k + 2], f[4 * k + 3]), __NV_SATFINITE, __NV_E4M3);
        r[k] = lo | (hi << 16);
      }
      w[0] = make_uint4(r[0], r[1], r[2], r[3]);
    } else {
      w[0] = make_uint4(pack(f[0], f[1]), pack(f[2], f[3]), pack(f[4], f[5]), pack(f[6], f[7]));
      w[1] = make_uint4(pack(f[8], f[9]), pack(f[10], f[11]), pack(f[12], f[13]), pack(f[14], f[15]));
    }
  }
  __device__ __forceinline__ static void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if constexpr (I8) tc::mma_i8(d, a, b, idesc, acc);
    else if constexpr (Q8) tc::mma_f8(d, a, b, idesc, acc);
    else tc::mma_f16(d, a, b, idesc, acc);
  }
  __device__ __forceinline__ static void mma_nc(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if constexpr (I8) tc::mma_i8_nc(d, a, b, idesc, acc);
    else if constexpr (Q8) tc::mma_f8_nc(d, a, b, idesc, acc);
    else tc::mma_f16_nc(d, a, b, idesc, acc);
  }
  // cta_group::2 (the CTA-pair kernels)
  __device__ __forceinline__ static void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if constexpr (I8) tc::mma2_i8(d, a, b, idesc, acc);
    else if constexpr (Q8) tc::mma2_f8(d, a, b, idesc, acc);
    else tc::mma2_f16(d, a, b, idesc, acc);
  }
};

// The per-channel math of every epilogue, 16 channels at a time:
// y = acc * oscale + bias (+ residual * res_scale), ReLU, * out_inv (fp8).
// INT8 works in output-code units: the plan folds 1 / (output scale) into
// oscale, bias and res_scale, and the u8 conversion's saturation at 0 is the
// ReLU (8.75 instructions per value instead of 12: these epilogues bound
// the int8 halo layers).
// FACC: v holds f32 bits whatever the format (split-K's reduced partials).
template <int PR, bool FACC = false>
__device__ __forceinline__ void epi16(const uint32_t (&v)[16], const float* bias, const float* oscale,
                                      const uint4* res, float res_scale, bool relu, float out_inv, uint4* out) {
  using NF = Num<PR>;
  float f[16];
  const float4* bp = reinterpret_cast<const float4*>(bias);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float4 b4 = __ldg(bp + j);
    f[4 * j + 0] = b4.x;
    f[4 * j + 1] = b4.y;
    f[4 * j + 2] = b4.z;
    f[4 * j + 3] = b4.w;
  }
  if constexpr (NF::Q8) {
    const float4* sp = reinterpret_cast<const float4*>(oscale);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 s4 = __ldg(sp + j);
      f[4 * j + 0] = fmaf(FACC ? __uint_as_float(v[4 * j + 0]) : NF::acc(v[4 * j + 0]), s4.x, f[4 * j + 0]);
      f[4 * j + 1] = fmaf(FACC ? __uint_as_float(v[4 * j + 1]) : NF::acc(v[4 * j + 1]), s4.y, f[4 * j + 1]);
      f[4 * j + 2] = fmaf(FACC ? __uint_as_float(v[4 * j + 2]) : NF::acc(v[4 * j + 2]), s4.z, f[4 * j + 2]);
      f[4 * j + 3] = fmaf(FACC ? __uint_as_float(v[4 * j + 3]) : NF::acc(v[4 * j + 3]), s4.w, f[4 * j + 3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) f[j] += __uint_as_float(v[j]);
  }
  if (res) {
    float x[16];
    NF::to_float16(res, x);
#pragma unroll
    for (int j = 0; j < 16; ++j) f[j] = NF::Q8 ? fmaf(x[j], res_scale, f[j]) : f[j] + x[j];
  }
  if (!NF::I8 && relu) {
#pragma unroll
    for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], 0.f);
  }
  if constexpr (NF::Q8 && !NF::I8) {
#pragma unroll
    for (int j = 0; j < 16; ++j) f[j] *= out_inv;
  }
  NF::from_float16(f, out);
}

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
  static constexpr int TMEM_COLS =
      2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 256;
};

struct TileId {
  int z, nt, mt;
};

__device__ __forceinline__ TileId decode_tile(const ConvParams& p, int t) {
  // Tiles that read the same input rows are adjacent in t, so the ~148 CTAs
  // in flight share them through L2: n tiles of one m tile, and (when the
  // phases are congruent, i.e. a stride-2 ConvT) the 4 output phases of one
  // input region.  Otherwise phase-major, n tile fastest within a phase.
  if (p.interleave) {
    // the phase rotates with the m tile: a grid stride that is a multiple of
    // nphases (148 = 37 x 4) would otherwise pin each CTA to one phase, and
    // ConvT phases carry 1/2/2/4 taps
    const int q = t / p.ntiles_n, nt = t - q * p.ntiles_n;
    const int mt = q / p.nphases;
    int z = q - mt * p.nphases + mt;
    z -= (z / p.nphases) * p.nphases;
    return {z, nt, mt};
  }
  int z = 0;
#pragma unroll 1
  while (z + 1 < p.nphases && t >= p.ph[z + 1].tile0) ++z;
  const int r = t - p.ph[z].tile0;
  const int mt = r / p.ntiles_n;
  return {z, r - mt * p.ntiles_n, mt};
}

// Weight tile (nt, kb) of a BN-wide launch over weights packed PBN wide:
// [PBN tiles][kblocks][PBN rows][64], rows 128 B swizzled in 8-row atoms.
template <int BN>
__device__ __forceinline__ const uint16_t* wtile(const ConvParams& p, const Phase& P, int nt, int kb) {
  const int sub = p.pbn / BN;
  const int ntp = nt / sub, q = nt - ntp * sub;
  return P.w + (((size_t)ntp * P.kblocks + kb) * p.pbn + (size_t)q * BN) * BK;
}

__device__ __forceinline__ void tma_im2col_4d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c, int w,
                                              int h, int n, uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(tc::smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w),
      "h"(off_h)
      : "memory");
}

// A descriptor of a stage: constant fields per channel chunk CC, start address
// advanced per K=16 step by a compile-time offset (16-byte units).
template <int CC>
__device__ __forceinline__ uint64_t a_desc_base(uint32_t sa) {
  constexpr uint64_t lbo = CC == 8 ? 2048 : 16;
  constexpr uint64_t sbo = CC == 64 ? 1024 : (CC == 32 ? 512 : (CC == 16 ? 256 : 128));
  constexpr uint64_t layout = CC == 64 ? 2 : (CC == 32 ? 4 : (CC == 16 ? 6 : 0));
  return (uint64_t)((sa >> 4) & 0x3FFF) | ((lbo >> 4) << 16) | ((sbo >> 4) << 32) | (1ull << 46) | (layout << 61);
}
template <int CC>
__device__ __forceinline__ constexpr uint32_t a_koff(int k) {
  return CC == 64 ? k * 2 : (CC == 32 ? (k >> 1) * 512 + (k & 1) * 2 : k * 256);
}

// One epilogue thread's share of an output row: HC accumulator columns ->
// epi16 -> 16-bit-unit store (orow/rrow point at the row's first channel).
// The whole residual slice is requested before the accumulator wait
// (HC <= 64), so its latency hides under the mainloop.
template <int HC, int PR>
__device__ __forceinline__ void epilogue_row(uint32_t tbase, uint16_t* orow, const uint16_t* rrow, const float* bias,
                                             const float* oscale, float res_scale, float out_inv, bool relu,
                                             bool valid, uint64_t* tfull_bar, uint32_t parity) {
  using NF = Num<PR>;
  constexpr int W16 = NF::U4;                 // uint4 per 16 channels
  constexpr int NR = HC <= 64 ? HC / 16 * W16 : 2 * W16;
  uint4 rv[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) rv[i] = rrow ? __ldg(reinterpret_cast<const uint4*>(rrow) + i) : make_uint4(0, 0, 0, 0);
  // tcgen05.wait::ld orders memory, so per-chunk loads cannot be hoisted past
  // it: pull this row's bias / scale / residual lines into L1 under the mainloop
#pragma unroll
  for (int c = 0; c < HC; c += 32) {
    tc::prefetch_l1(bias + c);
    if constexpr (NF::Q8) tc::prefetch_l1(oscale + c);
  }
  if constexpr (HC > 64) {
    if (rrow) {
#pragma unroll
      for (int c = 128; c < HC / NF::CPU * 2; c += 128) tc::prefetch_l1(reinterpret_cast<const uint8_t*>(rrow) + c);
    }
  }
  tc::mbar_wait(tfull_bar, parity);
  tc::tc_fence_after();
#pragma unroll
  for (int c0 = 0; c0 < HC; c0 += 16) {
    uint32_t v[16];
    tc::tmem_ld16(tbase + c0, v);
    uint4 rcur[W16];
    if constexpr (HC <= 64) {
#pragma unroll
      for (int w = 0; w < W16; ++w) rcur[w] = rv[c0 / 16 * W16 + w];
    } else {  // rolling two-chunk prefetch
#pragma unroll
      for (int w = 0; w < W16; ++w) rcur[w] = rv[w];
      if (rrow && c0 + 16 < HC) {
#pragma unroll
        for (int w = 0; w < W16; ++w)
          rv[w] = __ldg(reinterpret_cast<const uint4*>(rrow) + (c0 + 16) / 16 * W16 + w);
      }
    }
    tc::tmem_ld_wait();
    if (valid) {
      uint4 o[W16];
      epi16<PR>(v, bias + c0, oscale + (NF::Q8 ? c0 : 0), rrow ? rcur : nullptr, res_scale, relu, out_inv, o);
#pragma unroll
      for (int w = 0; w < W16; ++w) reinterpret_cast<uint4*>(orow)[c0 / 16 * W16 + w] = o[w];
    }
  }
}

// Output pixel of GEMM row m of phase P (m < P.M).
__device__ __forceinline__ size_t out_pixel(const ConvParams& p, const Phase& P, int m) {
  const int HW = P.GH * P.GW;
  const int n = m / HW;
  const int rem = m - n * HW;
  const int gy = rem / P.GW, gx = rem - gy * P.GW;
  return ((size_t)n * p.OH + gy * p.osy + P.oy) * p.OW + gx * p.osx + P.ox;
}

// Split-K epilogue (all 256 epilogue threads take part).  Each split stores
// its TMEM partial into its own slot ws[u] ([BN/4][BM] float4: coalesced) and
// frees the accumulator; the ksplit CTAs of a tile (one cluster, one unit per
// CTA) meet at the cluster barrier; then CTA ks sums
// its 1/ksplit share of the tile's (row, 16-channel) items over the slots in
// slot order -- deterministic -- and runs the ordinary epilogue math on them.
template <int BN, int HC, int PR>
__device__ __forceinline__ void splitk_tile(const ConvParams& p, int u, int t, const TileId& id, int r, int cbeg,
                                            uint32_t tbase, uint64_t* tfull_bar, uint64_t* tempty_bar,
                                            uint32_t parity) {
  using NF = Num<PR>;
  constexpr int W16 = NF::U4;
  constexpr int SLOT = BN / 4 * BM;  // float4 per slot
  const int S = p.ksplit, ks = u - t * S;
  float4* ws = reinterpret_cast<float4*>(p.ws);
  {
    float4* mine = ws + (size_t)u * SLOT + (size_t)(cbeg / 4) * BM + r;
    tc::mbar_wait(tfull_bar, parity);
    tc::tc_fence_after();
    if (threadIdx.x == 64) LSG_TR(p.trace_slot, 6);
#pragma unroll
    for (int c0 = 0; c0 < HC; c0 += 16) {
      uint32_t v[16];
      tc::tmem_ld16(tbase + c0, v);
      tc::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 4; ++j)
        __stcg(mine + (size_t)(c0 / 4 + j) * BM,
               make_float4(NF::acc(v[4 * j]), NF::acc(v[4 * j + 1]), NF::acc(v[4 * j + 2]), NF::acc(v[4 * j + 3])));
    }
    tc::tc_fence_before();
    tc::mbar_arrive(tempty_bar);
  }
  // every thread of the cluster arrives once (the producer / MMA warps after
  // their loops, see conv_tc): release the slot stores, acquire the siblings'
  __threadfence();
  if (threadIdx.x == 64) LSG_TR(p.trace_slot, 7);
  tc::cluster_arrive_wait();
  if (threadIdx.x == 64) LSG_TR(p.trace_slot, 8);
  const Phase& P = p.ph[id.z];
  const int n0 = id.nt * BN;
  constexpr int NI = BM * (BN / 16);
  const int i0 = ks * NI / S, i1 = (ks + 1) * NI / S;
  const float4* slots = ws + (size_t)t * S * SLOT;
#pragma unroll 1
  for (int i = i0 + (int)threadIdx.x - 64; i < i1; i += 32 * NUM_EPI_WARPS) {
    const int chunk = i / BM, row = i - chunk * BM;
    const int m = id.mt * BM + row;
    if (m >= P.M) continue;
    float f[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) f[j] = 0.f;
    // four slots' loads in flight at a time; summed in slot order
#pragma unroll 1
    for (int s2 = 0; s2 < S; s2 += 4) {
      float4 x[4][4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4* q = slots + (size_t)(s2 + k) * SLOT + (size_t)(chunk * 4) * BM + row;
#pragma unroll
        for (int j = 0; j < 4; ++j) x[k][j] = s2 + k < S ? __ldcg(q + (size_t)j * BM) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (s2 + k < S) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            f[4 * j] += x[k][j].x;
            f[4 * j + 1] += x[k][j].y;
            f[4 * j + 2] += x[k][j].z;
            f[4 * j + 3] += x[k][j].w;
          }
        }
      }
    }
    uint32_t v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(f[j]);
    const size_t pix = out_pixel(p, P, m);
    const int ch = n0 + chunk * 16;
    uint4 res[W16], o[W16];
    if (p.res) {
      const uint4* rp = reinterpret_cast<const uint4*>(p.res + pix * p.res_pitch + p.res_coff + ch / NF::CPU);
#pragma unroll
      for (int w = 0; w < W16; ++w) res[w] = __ldg(rp + w);
    }
    epi16<PR, true>(v, p.bias + ch, p.oscale + (NF::Q8 ? ch : 0), p.res ? res : nullptr, p.res_scale, p.relu != 0,
              p.out_inv, o);
    uint4* op = reinterpret_cast<uint4*>(p.out + pix * p.out_pitch + p.out_coff + ch / NF::CPU);
#pragma unroll
    for (int w = 0; w < W16; ++w) op[w] = o[w];
  }
  if (threadIdx.x == 64) LSG_TR(p.trace_slot, 9);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\t"
      "elect.sync rx|px, 0xffffffff;\n\t"
      "@px mov.s32 %0, 1;\n\t}"
      : "+r"(pred));
  return pred != 0;
}

template <int BN, int CC, bool FUSED_OUT, int PR>
__global__ void __launch_bounds__(NUM_THREADS, 1) conv_tc(const __grid_constant__ ConvParams p) {
  using CF = Cfg<BN>;
  using NF = Num<PR>;
  constexpr int S = CF::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * CF::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * CF::B_BYTES);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) LSG_TR(p.trace_slot, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 32 * NUM_EPI_WARPS);
    }
    tc::fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap)) : "memory");
  }
  if (warp == 1) tc::tmem_alloc<CF::TMEM_COLS>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr int LPS = BK / CC;  // TMA loads per stage
  tc::griddep_launch();
  if (threadIdx.x == 0) LSG_TR(p.trace_slot, 1);

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (whole warp;
    // lane j issues load j of a stage, lane 0 the weights + expect_tx)
    const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB);
    constexpr uint32_t LOAD_BYTES = BM * CC * 2;
    const int cpt = p.C / CC;  // loads per tap
    // The weights do not depend on the previous layer: the first unit's first
    // S weight stages are issued (and the rest of its weight range prefetched
    // into L2) before waiting for the previous layer's activations.
    int pre = 0;
    if (blockIdx.x < p.total_units) {
      const int u = blockIdx.x, t = u / p.ksplit, ks = u - t * p.ksplit;
      const TileId id = decode_tile(p, t);
      const Phase& P = p.ph[id.z];
      const int KB = P.kblocks, NL = P.nloads;
      const int kb0 = ks * KB / p.ksplit, kb1 = (ks + 1) * KB / p.ksplit;
      pre = min(S, kb1 - kb0);
      for (int kb = kb0 + pre + lane; kb < kb1; kb += 32) tc::prefetch_l2(wtile<BN>(p, P, id.nt, kb), CF::B_BYTES);
      if (lane == 0) {
        for (int i = 0; i < pre; ++i) {
          const int kb = kb0 + i;
          const int nl = min(LPS, NL - kb * LPS);
          tc::mbar_arrive_expect_tx(&full[i], CF::B_BYTES + nl * LOAD_BYTES);
          tc::bulk_g2s(sB0 + i * CF::B_BYTES, wtile<BN>(p, P, id.nt, kb), CF::B_BYTES, &full[i]);
        }
      }
      __syncwarp();
    }
    tc::griddep_wait();  // previous layer's activations complete
    if (lane == 0) LSG_TR(p.trace_slot, 2);
    int s = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < p.total_units; u += gridDim.x) {
      const int t = u / p.ksplit, ks = u - t * p.ksplit;
      const TileId id = decode_tile(p, t);
      const Phase& P = p.ph[id.z];
      const int KB = P.kblocks, NL = P.nloads;
      const int kb0 = ks * KB / p.ksplit, kb1 = (ks + 1) * KB / p.ksplit;
      const int m0 = id.mt * BM;
      const int HW = P.GH * P.GW;
      const int n = m0 / HW, rem = m0 - n * HW;
      const int gy = rem / P.GW, gx = rem - gy * P.GW;
      const int w0 = gx * p.sx + p.lower_w, h0 = gy * p.sy + p.lower_h;
      for (int kb = kb0; kb < kb1; ++kb) {
        const int l = kb * LPS + lane;
        const int nl = min(LPS, NL - kb * LPS);
        if (pre > 0) {  // weights already in flight (fresh stage: no empty wait)
          --pre;
        } else {
          tc::mbar_wait(&empty[s], ph ^ 1);
          if (lane == 0) {
            tc::mbar_arrive_expect_tx(&full[s], CF::B_BYTES + nl * LOAD_BYTES);
            tc::bulk_g2s(sB0 + s * CF::B_BYTES, wtile<BN>(p, P, id.nt, kb), CF::B_BYTES, &full[s]);
          }
        }
        if (lane < nl) {
          const int tap = l / cpt, ch = (l - tap * cpt) * CC;
          tma_im2col_4d(sA0 + s * CF::A_BYTES + lane * LOAD_BYTES, &p.tmap, &full[s], ch, w0, h0, n,
                        P.offw[tap], P.offh[tap]);
        }
        __syncwarp();
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    if (lane == 0) LSG_TR(p.trace_slot, 3);
    if (p.ksplit > 1) tc::cluster_arrive_wait();  // splitk_tile's meeting
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (whole warp
    // runs the loop, one elected lane issues: descriptors stay uniform)
    constexpr uint32_t idesc = NF::idesc(BM, BN);
    const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB);
    int s = 0;
    uint32_t ph = 0, tl = 0;
    for (int u = blockIdx.x; u < p.total_units; u += gridDim.x, ++tl) {
      const int t = u / p.ksplit, ks = u - t * p.ksplit;
      const TileId id = decode_tile(p, t);
      const int KB = p.ph[id.z].kblocks, NS = p.ph[id.z].nsteps;
      const int kb0 = ks * KB / p.ksplit, kb1 = (ks + 1) * KB / p.ksplit;
      const uint32_t a = tl & 1, use = tl >> 1;
      tc::mbar_wait(&tempty[a], (use & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t d = tmem + a * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        tc::mbar_wait(&full[s], ph);
        tc::tc_fence_after();
        if (kb == kb0 && lane == 0) LSG_TR(p.trace_slot, 4);
        const uint64_t da = a_desc_base<CC>(sA0 + s * CF::A_BYTES);
        const uint64_t db = tc::sdesc_sw128(sB0 + s * CF::B_BYTES);
        if (elect_one()) {
          if (kb * 4 + 4 <= NS) {
#pragma unroll
            for (int k = 0; k < 4; ++k) NF::mma(d, da + a_koff<CC>(k), db + 2 * k, idesc, (kb != kb0) | (k != 0));
          } else {
            const int ns = NS - kb * 4;
            for (int k = 0; k < ns; ++k) NF::mma(d, da + a_koff<CC>(k), db + 2 * k, idesc, (kb != kb0) | (k != 0));
          }
          tc::mma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) tc::mma_commit(&tfull[a]);
      __syncwarp();
    }
    if (lane == 0) LSG_TR(p.trace_slot, 5);
    if (p.ksplit > 1) tc::cluster_arrive_wait();  // splitk_tile's meeting
  } else {
    // ------------------------------------------------ epilogue (warps 2-9)
    tc::griddep_wait();  // the output / residual buffers are free / complete
    const int q = warp & 3;               // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;     // which half of the BN columns
    constexpr bool SPLIT = !FUSED_OUT && BN >= 32;
    constexpr int HC = SPLIT ? BN / 2 : BN;
    const int cbeg = SPLIT ? half * HC : 0;
    const bool active = SPLIT || half == 0;
    const int r = q * 32 + lane;
    uint32_t tl = 0;
    for (int u = blockIdx.x; u < p.total_units; u += gridDim.x, ++tl) {
      const int t = u / p.ksplit;
      const TileId id = decode_tile(p, t);
      const Phase& P = p.ph[id.z];
      const uint32_t a = tl & 1, use = tl >> 1;
      const int m = id.mt * BM + r;
      const int n0 = id.nt * BN;
      const bool valid = m < P.M;
      int n = 0, oy = 0, ox = 0;
      if (valid) {
        const int HW = P.GH * P.GW;
        n = m / HW;
        const int rem = m - n * HW;
        const int gy = rem / P.GW, gx = rem - gy * P.GW;
        oy = gy * p.osy + P.oy;
        ox = gx * p.osx + P.ox;
      }
      const size_t pix = ((size_t)n * p.OH + oy) * p.OW + ox;
      if constexpr (!FUSED_OUT) {
        // channel offsets in 16-bit units (fp8: two channels per unit)
        uint16_t* orow = p.out + pix * p.out_pitch + p.out_coff + (n0 + cbeg) / NF::CPU;
        const uint16_t* rrow =
            (p.res && valid && active) ? p.res + pix * p.res_pitch + p.res_coff + (n0 + cbeg) / NF::CPU : nullptr;
        if (!active) {
          tc::mbar_wait(&tfull[a], use & 1);
          tc::tc_fence_after();
          tc::tc_fence_before();
          tc::mbar_arrive(&tempty[a]);
          continue;
        }
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + a * BN + cbeg;
        if constexpr (SPLIT) {
          if (p.ksplit > 1) {
            splitk_tile<BN, HC, PR>(p, u, t, id, r, cbeg, tbase, &tfull[a], &tempty[a], use & 1);
            continue;
          }
        }
        epilogue_row<HC, PR>(tbase, orow, rrow, p.bias + n0 + cbeg, p.oscale + (NF::Q8 ? n0 + cbeg : 0), p.res_scale,
                             p.out_inv, p.relu != 0, valid, &tfull[a], use & 1);
      } else {
        // out0 (BN = 32 channels, ReLU) fused with out1 (1x1 32->3) + sigmoid;
        // the second warp of each quadrant only keeps the barrier count
        tc::mbar_wait(&tfull[a], use & 1);
        tc::tc_fence_after();
        if (half == 0) {
          const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + a * BN;
          float o[3] = {__ldg(p.b1 + 0), __ldg(p.b1 + 1), __ldg(p.b1 + 2)};
#pragma unroll
          for (int c0 = 0; c0 < BN; c0 += 16) {
            uint32_t v[16];
            tc::tmem_ld16(tbase + c0, v);
            tc::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float acc = NF::Q8 ? NF::acc(v[j]) * __ldg(p.oscale + c0 + j) : __uint_as_float(v[j]);
              const float x = fmaxf(acc + __ldg(p.bias + c0 + j), 0.f);
#pragma unroll
              for (int o3 = 0; o3 < 3; ++o3) o[o3] = fmaf(__ldg(p.w1 + o3 * 32 + c0 + j), x, o[o3]);
            }
          }
          if (valid) {
            const int HWo = p.OH * p.OW;
            const size_t pp = (size_t)oy * p.OW + ox;
            if (p.out_mode == OUT_F32_LOGITS) {
              float* out = reinterpret_cast<float*>(p.final_out);
#pragma unroll
              for (int o3 = 0; o3 < 3; ++o3) out[((size_t)n * 3 + o3) * HWo + pp] = o[o3];
            } else if (p.out_mode == OUT_F32_NCHW) {
              float* out = reinterpret_cast<float*>(p.final_out);
#pragma unroll
              for (int o3 = 0; o3 < 3; ++o3) out[((size_t)n * 3 + o3) * HWo + pp] = 1.f / (1.f + __expf(-o[o3]));
            } else {
              uint8_t* out = reinterpret_cast<uint8_t*>(p.final_out) + ((size_t)n * HWo + pp) * 3;
#pragma unroll
              for (int o3 = 0; o3 < 3; ++o3) {
                const float s = 1.f / (1.f + __expf(-o[o3]));
                out[o3] = (uint8_t)__float2int_rn(fminf(fmaxf(s * 255.f, 0.f), 255.f));
              }
            }
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&tempty[a]);
    }
    if (threadIdx.x == 64) LSG_TR(p.trace_slot, 10);
  }
  __syncthreads();
  if (threadIdx.x == 0) LSG_TR(p.trace_slot, 11);
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<CF::TMEM_COLS>(tmem);
  }
}

}  // namespace gen
}  // namespace lsg
