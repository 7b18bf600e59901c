// conv_pair.cuh -- the im2col conv (conv_kernel.cuh) on CTA pairs:
// tcgen05.mma.cta_group::2, M = 256 rows over two SMs of a TPC.
//
// Why: an SS-mode MMA is bounded by shared-memory bandwidth (DESIGN.md §3.1:
// M=128, N=256, K=16 reads 4 KB of A + 8 KB of B per instruction, and the
// TMA fills of both compete for the same 128 B/clk).  On a pair each CTA
// stages its own 128 A rows and only HALF of the weight tile (N/2 rows); the
// one MMA reads A from both CTAs and B halves from both -- per-SM operand
// traffic per FLOP drops by a third for N = 256, and the weight bytes each SM
// pulls through L2 halve.
//
// Roles: warp 0 of each CTA is a TMA producer for its own A rows and its own
// half of the weight tile; both CTAs' loads complete on the EVEN CTA's
// `full` barrier (cta_group::2 TMA forms), whose expect_tx covers the pair's
// bytes.  Warp 1 of the even CTA issues the MMAs; completion is committed to
// both CTAs' barriers at once (multicast commit).  Warps 2-9 of each CTA run
// the epilogue of its own 128 rows from its own TMEM and release the
// accumulator on the even CTA's `tempty` barrier (one arrive per warp).
#pragma once

#include "conv_kernel.cuh"

namespace lsg {
namespace gen {

template <int BN>
struct Cfg2 {
  static constexpr int BH = BN / 2;  // weight rows per CTA
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BH * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = Cfg<BN>::TMEM_COLS;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 256;
  static_assert(BH % 8 == 0, "weight half-tile must be whole 8-row swizzle atoms");
};

template <int PR>
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  Num<PR>::mma2(d, a, b, idesc, acc);
}

// Pair TMA loads: data to this CTA's shared memory, completion to the
// barrier at cluster address `mbar` (the even CTA's).
__device__ __forceinline__ void tma_im2col_4d_pair(uint32_t dst, const CUtensorMap* map, uint32_t mbar, int c,
                                                   int w, int h, int n, uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w), "h"(off_h)
      : "memory");
}
__device__ __forceinline__ void tma_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t mbar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(tc::smem_u32(p)), "r"(rank));
  return r;
}
// first weight row (in wmap) of this CTA's half of tile (nt, kb)
template <int BN>
__device__ __forceinline__ int wrow_pair(const ConvParams& p, const Phase& P, int z, int nt, int kb, uint32_t rank) {
  const int sub = p.pbn / BN;
  const int ntp = nt / sub, q = nt - ntp * sub;
  return p.wrow0[z] + (ntp * P.kblocks + kb) * p.pbn + q * BN + (int)rank * (BN / 2);
}

// Tiles are PAIRS of m-tiles (host: Phase::mtiles = ceil(m-tiles / 2)); CTA
// rank r of a cluster takes m-tile 2 * id.mt + r.
template <int BN, int CC, int PR>
__global__ void __launch_bounds__(NUM_THREADS, 1) conv_tc2(const __grid_constant__ ConvParams p) {
  using CF = Cfg2<BN>;
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
  const uint32_t rank = tc::cluster_ctarank();
  const int pair = (int)(blockIdx.x >> 1), npairs = (int)(gridDim.x >> 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);   // even CTA: its producer's arrive (+ both CTAs' bytes)
      tc::mbar_init(&empty[s], 1);  // the multicast MMA commit
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 2 * NUM_EPI_WARPS);  // even CTA: every epilogue warp of the pair
    }
    tc::fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.wmap)) : "memory");
  }
  if (warp == 1) tc::tmem_alloc2<CF::TMEM_COLS>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();  // both CTAs' barriers exist before any cross-CTA signal
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr int LPS = BK / CC;
  tc::griddep_launch();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer: own A rows, own B half
    const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB);
    constexpr uint32_t LOAD_BYTES = BM * CC * 2;
    const int cpt = p.C / CC;
    int pre = 0;
    if (pair < p.total_tiles) {  // first tile's weights before the PDL wait
      const TileId id = decode_tile(p, pair);
      const Phase& P = p.ph[id.z];
      const int KB = P.kblocks, NL = P.nloads;
      pre = min(S, KB);
      if (lane == 0) {
        for (int i = 0; i < pre; ++i) {
          const int nl = min(LPS, NL - i * LPS);
          if (rank == 0) tc::mbar_arrive_expect_tx(&full[i], 2 * (CF::B_BYTES + nl * LOAD_BYTES));
          tma_2d_pair(sB0 + i * CF::B_BYTES, &p.wmap, cluster_addr(&full[i], 0), 0,
                      wrow_pair<BN>(p, P, id.z, id.nt, i, rank));
        }
      }
      __syncwarp();
    }
    tc::griddep_wait();
    int s = 0;
    uint32_t ph = 0;
    for (int t = pair; t < p.total_tiles; t += npairs) {
      const TileId id = decode_tile(p, t);
      const Phase& P = p.ph[id.z];
      const int KB = P.kblocks, NL = P.nloads;
      const int m0 = (2 * id.mt + (int)rank) * BM;
      const int HW = P.GH * P.GW;
      const int n = m0 / HW, rem = m0 - n * HW;
      const int gy = rem / P.GW, gx = rem - gy * P.GW;
      const int w0 = gx * p.sx + p.lower_w, h0 = gy * p.sy + p.lower_h;
      for (int kb = 0; kb < KB; ++kb) {
        const int l = kb * LPS + lane;
        const int nl = min(LPS, NL - kb * LPS);
        const uint32_t fb = cluster_addr(&full[s], 0);
        if (pre > 0) {
          --pre;
        } else {
          tc::mbar_wait(&empty[s], ph ^ 1);
          if (lane == 0) {
            if (rank == 0) tc::mbar_arrive_expect_tx(&full[s], 2 * (CF::B_BYTES + nl * LOAD_BYTES));
            tma_2d_pair(sB0 + s * CF::B_BYTES, &p.wmap, fb, 0, wrow_pair<BN>(p, P, id.z, id.nt, kb, rank));
          }
        }
        if (lane < nl) {
          const int tap = l / cpt, ch = (l - tap * cpt) * CC;
          tma_im2col_4d_pair(sA0 + s * CF::A_BYTES + lane * LOAD_BYTES, &p.tmap, fb, ch, w0, h0, n,
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
    if (rank == 0) {
      // ---------------------------------------------- MMA issuer (even CTA)
      constexpr uint32_t idesc = NF::idesc(2 * BM, BN);
      const uint32_t sA0 = tc::smem_u32(sA), sB0 = tc::smem_u32(sB);
      int s = 0;
      uint32_t ph = 0, tl = 0;
      for (int t = pair; t < p.total_tiles; t += npairs, ++tl) {
        const TileId id = decode_tile(p, t);
        const int KB = p.ph[id.z].kblocks, NS = p.ph[id.z].nsteps;
        const uint32_t a = tl & 1, use = tl >> 1;
        tc::mbar_wait_cluster(&tempty[a], (use & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + a * BN;
        for (int kb = 0; kb < KB; ++kb) {
          tc::mbar_wait(&full[s], ph);
          tc::tc_fence_after();
          const uint64_t da = a_desc_base<CC>(sA0 + s * CF::A_BYTES);
          const uint64_t db = tc::sdesc_sw128(sB0 + s * CF::B_BYTES);
          if (elect_one()) {
            const int ns = min(4, NS - kb * 4);
            for (int k = 0; k < ns; ++k) mma2<PR>(d, da + a_koff<CC>(k), db + 2 * k, idesc, (kb | k) != 0);
            tc::mma_commit2(&empty[s]);
          }
          __syncwarp();
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
        if (elect_one()) tc::mma_commit2(&tfull[a]);
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------ epilogue: own 128 rows, own TMEM
    tc::griddep_wait();
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int HC = BN / 2;
    const int cbeg = half * HC;
    const int r = q * 32 + lane;
    uint32_t tl = 0;
    for (int t = pair; t < p.total_tiles; t += npairs, ++tl) {
      const TileId id = decode_tile(p, t);
      const Phase& P = p.ph[id.z];
      const uint32_t a = tl & 1, use = tl >> 1;
      const int m = (2 * id.mt + (int)rank) * BM + r;
      const int n0 = id.nt * BN;
      const bool valid = m < P.M;
      const size_t pix = valid ? out_pixel(p, P, m) : 0;
      uint16_t* orow = p.out + pix * p.out_pitch + p.out_coff + (n0 + cbeg) / NF::CPU;
      const uint16_t* rrow =
          (p.res && valid) ? p.res + pix * p.res_pitch + p.res_coff + (n0 + cbeg) / NF::CPU : nullptr;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + a * BN + cbeg;
      epilogue_row<HC, PR>(tbase, orow, rrow, p.bias + n0 + cbeg, p.oscale + (NF::Q8 ? n0 + cbeg : 0), p.res_scale,
                           p.out_inv, p.relu != 0, valid, &tfull[a], use & 1);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_remote(&tempty[a], 0);  // the even CTA's barrier (itself for rank 0)
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();  // the peer's TMEM / smem / barriers stay live until both CTAs are done
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc2<CF::TMEM_COLS>(tmem);
  }
}

}  // namespace gen
}  // namespace lsg
