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

#include <cstdint>

#include "tc.cuh"

namespace lsg {
namespace gen {

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
  int sy, sx, osy, osx;
  int relu, out_mode;
  const float* w1;  // fused output 1x1: [3][32]
  const float* b1;  // [3]
  void* final_out;
  int nphases, ntiles_n, total_tiles;
  int interleave;  // all phases have equal mtiles: t = (mt * nphases + z) * ntiles_n + nt
  Phase ph[MAX_PHASES];
};

// 16-bit number format: HALF = fp16 (kind::f16 format 0), else bf16 (format 1)
template <bool HALF>
struct Num {
  static constexpr uint32_t kFmt = HALF ? 0u : 1u;
  __device__ __forceinline__ static uint32_t pack(float a, float b) {
    if constexpr (HALF) {
      __half2 v = __floats2half2_rn(a, b);
      return *reinterpret_cast<uint32_t*>(&v);
    } else {
      __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
      return *reinterpret_cast<uint32_t*>(&v);
    }
  }
  __device__ __forceinline__ static float2 unpack(uint32_t u) {
    if constexpr (HALF) {
      return __half22float2(*reinterpret_cast<__half2*>(&u));
    } else {
      return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u));
    }
  }
};

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
// + bias (+ residual) (ReLU) -> 16-bit store.  The whole residual slice is
// requested before the accumulator wait (HC <= 64: 32 registers), so its
// latency hides under the mainloop instead of once per 16-column chunk.
template <int HC, bool HALF>
__device__ __forceinline__ void epilogue_row(uint32_t tbase, uint16_t* orow, const uint16_t* rrow, const float* bias,
                                             bool relu, bool valid, uint64_t* tfull_bar, uint32_t parity) {
  using NF = Num<HALF>;
  constexpr int NR = HC <= 64 ? HC / 8 : 2;
  uint4 rv[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) rv[i] = rrow ? __ldg(reinterpret_cast<const uint4*>(rrow) + i) : make_uint4(0, 0, 0, 0);
  tc::mbar_wait(tfull_bar, parity);
  tc::tc_fence_after();
#pragma unroll
  for (int c0 = 0; c0 < HC; c0 += 16) {
    uint32_t v[16];
    tc::tmem_ld16(tbase + c0, v);
    uint4 ra, rb;
    if constexpr (HC <= 64) {
      ra = rv[c0 / 8];
      rb = rv[c0 / 8 + 1];
    } else {
      ra = rv[0];
      rb = rv[1];
      if (rrow && c0 + 16 < HC) {
        rv[0] = __ldg(reinterpret_cast<const uint4*>(rrow + c0 + 16));
        rv[1] = __ldg(reinterpret_cast<const uint4*>(rrow + c0 + 16) + 1);
      }
    }
    tc::tmem_ld_wait();
    if (valid) {
      float f[16];
      const float4* bp = reinterpret_cast<const float4*>(bias + c0);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 b4 = __ldg(bp + j);
        f[4 * j + 0] = __uint_as_float(v[4 * j + 0]) + b4.x;
        f[4 * j + 1] = __uint_as_float(v[4 * j + 1]) + b4.y;
        f[4 * j + 2] = __uint_as_float(v[4 * j + 2]) + b4.z;
        f[4 * j + 3] = __uint_as_float(v[4 * j + 3]) + b4.w;
      }
      if (rrow) {
        const uint32_t rr[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 x = NF::unpack(rr[j]);
          f[2 * j] += x.x;
          f[2 * j + 1] += x.y;
        }
      }
      if (relu) {
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], 0.f);
      }
      uint4 o0, o1;
      o0.x = NF::pack(f[0], f[1]);
      o0.y = NF::pack(f[2], f[3]);
      o0.z = NF::pack(f[4], f[5]);
      o0.w = NF::pack(f[6], f[7]);
      o1.x = NF::pack(f[8], f[9]);
      o1.y = NF::pack(f[10], f[11]);
      o1.z = NF::pack(f[12], f[13]);
      o1.w = NF::pack(f[14], f[15]);
      *reinterpret_cast<uint4*>(orow + c0) = o0;
      *reinterpret_cast<uint4*>(orow + c0 + 8) = o1;
    }
  }
}

// As epilogue_row, with the residual slice already in registers (loaded a
// tile ahead by the caller, so its latency hides under the previous tile's
// epilogue when the epilogue, not the MMA, is the bottleneck).  HC <= 64.
template <int HC, bool HALF>
__device__ __forceinline__ void epilogue_row_pre(uint32_t tbase, uint16_t* orow, const uint4 (&rv)[HC / 8],
                                                 bool has_res, const float* bias, bool relu, bool valid,
                                                 uint64_t* tfull_bar, uint32_t parity) {
  using NF = Num<HALF>;
  static_assert(HC % 16 == 0 && HC <= 64, "epilogue_row_pre: HC");
  tc::mbar_wait(tfull_bar, parity);
  tc::tc_fence_after();
#pragma unroll
  for (int c0 = 0; c0 < HC; c0 += 16) {
    uint32_t v[16];
    tc::tmem_ld16(tbase + c0, v);
    float bf[16];
    const float4* bp = reinterpret_cast<const float4*>(bias + c0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 b4 = __ldg(bp + j);
      bf[4 * j + 0] = b4.x;
      bf[4 * j + 1] = b4.y;
      bf[4 * j + 2] = b4.z;
      bf[4 * j + 3] = b4.w;
    }
    tc::tmem_ld_wait();
    if (valid) {
      float f[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v[j]) + bf[j];
      if (has_res) {
        const uint4 ra = rv[c0 / 8], rb = rv[c0 / 8 + 1];
        const uint32_t rr[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 x = NF::unpack(rr[j]);
          f[2 * j] += x.x;
          f[2 * j + 1] += x.y;
        }
      }
      if (relu) {
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], 0.f);
      }
      uint4 o0, o1;
      o0.x = NF::pack(f[0], f[1]);
      o0.y = NF::pack(f[2], f[3]);
      o0.z = NF::pack(f[4], f[5]);
      o0.w = NF::pack(f[6], f[7]);
      o1.x = NF::pack(f[8], f[9]);
      o1.y = NF::pack(f[10], f[11]);
      o1.z = NF::pack(f[12], f[13]);
      o1.w = NF::pack(f[14], f[15]);
      *reinterpret_cast<uint4*>(orow + c0) = o0;
      *reinterpret_cast<uint4*>(orow + c0 + 8) = o1;
    }
  }
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

template <int BN, int CC, bool FUSED_OUT, bool HALF>
__global__ void __launch_bounds__(NUM_THREADS, 1) conv_tc(const __grid_constant__ ConvParams p) {
  using CF = Cfg<BN>;
  using NF = Num<HALF>;
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

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (whole warp;
    // lane j issues load j of a stage, lane 0 the weights + expect_tx)
    tc::griddep_wait();  // previous layer's activations complete
    const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB);
    constexpr uint32_t LOAD_BYTES = BM * CC * 2;
    const int cpt = p.C / CC;  // loads per tap
    int s = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
      const TileId id = decode_tile(p, t);
      const Phase& P = p.ph[id.z];
      const int KB = P.kblocks, NL = P.nloads;
      const int m0 = id.mt * BM;
      const int HW = P.GH * P.GW;
      const int n = m0 / HW, rem = m0 - n * HW;
      const int gy = rem / P.GW, gx = rem - gy * P.GW;
      const int w0 = gx * p.sx + p.lower_w, h0 = gy * p.sy + p.lower_h;
      const uint16_t* wbase = P.w + (size_t)id.nt * KB * BN * BK;
      for (int kb = 0; kb < KB; ++kb) {
        tc::mbar_wait(&empty[s], ph ^ 1);
        const int l = kb * LPS + lane;
        const int nl = min(LPS, NL - kb * LPS);
        if (lane == 0) {
          tc::mbar_arrive_expect_tx(&full[s], CF::B_BYTES + nl * LOAD_BYTES);
          tc::bulk_g2s(sB0 + s * CF::B_BYTES, wbase + (size_t)kb * BN * BK, CF::B_BYTES, &full[s]);
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
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (whole warp
    // runs the loop, one elected lane issues: descriptors stay uniform)
    constexpr uint32_t idesc = tc::idesc_f16kind(BM, BN, NF::kFmt);
    const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB);
    int s = 0;
    uint32_t ph = 0, tl = 0;
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++tl) {
      const TileId id = decode_tile(p, t);
      const int KB = p.ph[id.z].kblocks, NS = p.ph[id.z].nsteps;
      const uint32_t a = tl & 1, use = tl >> 1;
      tc::mbar_wait(&tempty[a], (use & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t d = tmem + a * BN;
      for (int kb = 0; kb < KB; ++kb) {
        tc::mbar_wait(&full[s], ph);
        tc::tc_fence_after();
        const uint64_t da = a_desc_base<CC>(sA0 + s * CF::A_BYTES);
        const uint64_t db = tc::sdesc_sw128(sB0 + s * CF::B_BYTES);
        if (elect_one()) {
          if (kb * 4 + 4 <= NS) {
#pragma unroll
            for (int k = 0; k < 4; ++k) tc::mma_f16(d, da + a_koff<CC>(k), db + 2 * k, idesc, (kb | k) != 0);
          } else {
            const int ns = NS - kb * 4;
            for (int k = 0; k < ns; ++k) tc::mma_f16(d, da + a_koff<CC>(k), db + 2 * k, idesc, (kb | k) != 0);
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
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++tl) {
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
        uint16_t* orow = p.out + pix * p.out_pitch + p.out_coff + n0 + cbeg;
        const uint16_t* rrow =
            (p.res && valid && active) ? p.res + pix * p.res_pitch + p.res_coff + n0 + cbeg : nullptr;
        if (!active) {
          tc::mbar_wait(&tfull[a], use & 1);
          tc::tc_fence_after();
          tc::tc_fence_before();
          tc::mbar_arrive(&tempty[a]);
          continue;
        }
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + a * BN + cbeg;
        epilogue_row<HC, HALF>(tbase, orow, rrow, p.bias + n0 + cbeg, p.relu != 0, valid, &tfull[a], use & 1);
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
              const float x = fmaxf(__uint_as_float(v[j]) + __ldg(p.bias + c0 + j), 0.f);
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
  }
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<CF::TMEM_COLS>(tmem);
  }
}

}  // namespace gen
}  // namespace lsg
