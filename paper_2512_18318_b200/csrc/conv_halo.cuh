// conv_halo.cuh -- patch-reuse convolution: one input patch in shared memory
// feeds every filter tap of a 128-position output tile.
//
// The im2col kernel (conv_kernel.cuh) re-reads each input pixel once per
// filter tap and is bound by L2->SM operand traffic on the narrow (N <= 64),
// high-resolution layers.  Here a tile is a 16-row x 8-column block of grid
// positions of one image.  Per channel block the TMA (tile mode, zero fill
// outside the image) loads the input patch around it ONCE as up to eight
// "planes" of [ph][pw][8] elements (16 B per pixel); every tap is then a
// UMMA operand view into the patch: a no-swizzle K-major descriptor whose
// start address is shifted by the tap's patch offset, core matrices = 8
// consecutive patch pixels x 16 B, SBO = one patch row, LBO = one plane, two
// planes per K=16 step.  The layer supplies a tap list (patch offset, output
// phase, first-tap-of-phase), which covers
//   * 3x3 stride-1 convs: 1 phase, 9 taps, planes = 8-channel granules;
//   * stride-2 3x3 ConvTranspose (fd5.0/fd6.0 shapes): the grid is the INPUT
//     grid, 4 output phases (oy, ox) with 1/2/2/4 taps, each phase its own
//     TMEM accumulator, all fed by the same patch;
//   * the 7x7 stem on 8-channel faces (fe0): planes are the patch shifted by
//     kx = 0..7 columns, so one K block = 8 horizontal taps x 8 channels and
//     the tap list is the 7 rows.
// Weights are resident in shared memory for the whole persistent CTA when
// they fit, otherwise they stream per (channel block, tap) through a ring.
// Epilogue as conv_tc (bias, residual, ReLU, channel-slice store, fused
// 1x1 + sigmoid output), per phase.
#pragma once

#include "conv_kernel.cuh"

namespace lsg {
namespace gen {

constexpr int HTH = 16, HTW = 8;  // tile: 16 rows x 8 columns = 128 grid positions
constexpr int MAX_HTAPS = 12;

// Routing modes and their compile-time tap tables (patch offset in pixels,
// output phase).  The host builds the same lists from the layer geometry and
// checks them against these (generator.cu), so packing and issue agree.
enum HaloMode {
  HALO_NONE = 0, HALO_CONV3 = 1, HALO_CONVT2 = 2, HALO_STEM7 = 3, HALO_STEM4X = 4, HALO_CONV3S2 = 5, HALO_CONV3X2 = 6
};

template <int MODE>
struct HaloTaps;
template <>
struct HaloTaps<HALO_CONV3> {  // 3x3 "same": patch (16+2) x (8+2), taps (ky, kx)
  static constexpr int NPH = 1, NT = 9, PW = HTW + 2, PH = HTH + 2;
  __host__ __device__ static constexpr int aoff(int t) { return (t / 3) * PW + t % 3; }
  __host__ __device__ static constexpr int phase(int) { return 0; }
};
template <>
struct HaloTaps<HALO_CONVT2> {  // stride-2 ConvT: patch (16+1) x (8+1) of the input, 4 phases (oy, ox)
  static constexpr int NPH = 4, NT = 9, PW = HTW + 1, PH = HTH + 1;
  // (dy, dx) per tap: phase 0 (0,0) | 1 (0,1) (0,0) | 2 (1,0) (0,0) | 3 (1,1) (1,0) (0,1) (0,0)
  __host__ __device__ static constexpr int aoff(int t) {
    return t == 1 || t == 7 ? 1 : (t == 3 || t == 6 ? PW : (t == 5 ? PW + 1 : 0));
  }
  __host__ __device__ static constexpr int phase(int t) { return t == 0 ? 0 : (t < 3 ? 1 : (t < 5 ? 2 : 3)); }
};
template <>
struct HaloTaps<HALO_STEM7> {  // 7x7 on 8 channels: planes = x shifts, taps = kernel rows
  static constexpr int NPH = 1, NT = 7, PW = HTW, PH = HTH + 6;
  __host__ __device__ static constexpr int aoff(int t) { return t * PW; }
  __host__ __device__ static constexpr int phase(int) { return 0; }
};
// The stem on "macro-pixels": a GEMM row is 4 horizontally adjacent output
// pixels (N = 4 x 16 channels per MMA instead of 16 -- the SS-mode MMA cost
// is set by the A read, so 4 pixels per row cost 48 instead of 4 x 36
// cycles).  Plane g (g = 0..9) holds input column 4j + g - 3 for macro
// column j (a W-strided TMA box), so a K step still reads 2 planes; the
// 4 pixel offsets are the epilogue's "phases" (element-strided stores).
// Stride-2 3x3 (fe1.0, fe2.0): the input under a tile is loaded as its 4
// parity sub-grids (TMA boxes with element stride 2 in H and W), so every
// tap is a fixed offset into one (16+1) x (8+1) parity patch instead of an
// im2col row per output pixel.  Output o, tap k reads input 2o + k - 1: k = 1
// the even grid at o, k = 0 / 2 the odd grid at o - 1 / o; with the patch
// origin at o0 - 1 the local offset is (k != 0).  A stage holds 8 planes =
// [parity ey*2+ex][2 channel granules]; a K step reads both granules of one
// parity (LBO = 1 plane), a tap adds its parity base.
template <>
struct HaloTaps<HALO_CONV3S2> {
  static constexpr int NPH = 1, NT = 9, PW = HTW + 1, PH = HTH + 1;
  static constexpr int PL16 = ((PW * PH * 16 + 127) / 128 * 128) / 16;  // plane, 16-byte units
  __host__ __device__ static constexpr int aoff(int t) {
    return ((t / 3 == 1 ? 0 : 2) + (t % 3 == 1 ? 0 : 1)) * 2 * PL16 + (t / 3 != 0) * PW + (t % 3 != 0);
  }
  __host__ __device__ static constexpr int phase(int) { return 0; }
};
// The output conv (out0, 80 -> 32 channels, fused with out1) on macro-pixels
// of 2 horizontally adjacent outputs: N = 2 x 32 per MMA and half the tiles
// (its N = 32 MMAs cost ~45 cycles each plus a per-tile overhead, DESIGN
// §3.1).  Output 2j + z, column tap kx reads input 2j + d - 1 with d = z + kx
// in 0..3: the patch is stored as x-parity planes (W-strided TMA boxes,
// element stride 2), plane parity d & 1 at macro column j + (d >> 1).  A stage
// holds [parity][4 channel granules]; taps t = (ky, d), 12 of them.
template <>
struct HaloTaps<HALO_CONV3X2> {
  static constexpr int NPH = 2, NT = 12, PW = HTW + 1, PH = HTH + 2;
  static constexpr int PL16 = ((PW * PH * 16 + 127) / 128 * 128) / 16;  // plane, 16-byte units
  __host__ __device__ static constexpr int aoff(int t) {
    return ((t % 4) & 1) * 4 * PL16 + (t / 4) * PW + ((t % 4) >> 1);
  }
  __host__ __device__ static constexpr int phase(int) { return 0; }
};
template <>
struct HaloTaps<HALO_STEM4X> {
  static constexpr int NPH = 4, NT = 7, PW = HTW, PH = HTH + 6;
  __host__ __device__ static constexpr int aoff(int t) { return t * PW; }
  __host__ __device__ static constexpr int phase(int) { return 0; }
};

struct alignas(64) HaloParams {
  CUtensorMap tmap;      // tiled map of the input view (C, W, H, N), box (8, pw, ph, 1)
  CUtensorMap tmap_out;  // output view, box (min(BN,64), 8, 16, 1) output positions (x2 stride for ConvT)
  CUtensorMap tmap_res;  // residual view, box (min(BN,64), 8, 16, 1)
  CUtensorMap wmap;      // packed weights as 2-D [rows][64 units], box (64, MN/2): CTA-pair loads
  CUtensorMap tmap_out2; // second copy of the output (out2): fe0 also writes a dense 16-channel tensor
                         // for fe1.0 (its concat-buffer slice is 16 of 80 channels)
  int H, W, C, B;    // input view
  int GH, GW;        // grid (output positions for convs, input positions for ConvT)
  int oy0, ox0;      // patch origin relative to the tile origin (-pad for convs)
  int pw, ph;        // patch width / height in pixels
  int plane;         // bytes per plane in smem (pw*ph*16, 128-aligned)
  int ngran;         // planes per tile over all channel blocks (C/8, or 8 shifted copies)
  int ncb;           // channel blocks of <= 8 planes
  int shift_planes;  // planes are x-shifted copies of channels 0..7 (fe0)
  int xmul;          // input columns per grid column (4 for the macro-pixel stem)
  int out2;          // also store every output box through tmap_out2
  int trace_slot;    // layer index (LSG_TRACE builds: wait accounting)
  int ntaps;
  int aoff[MAX_HTAPS];   // tap start offset in the patch, 16-byte units (= pixels)
  int tphase[MAX_HTAPS]; // output phase the tap accumulates into
  int tfirst;            // bit t: tap t is the first tap of its phase
  int osy, osx;          // output stride of the grid (2 for ConvT phases)
  int poy[4], pox[4];    // per-phase output offset
  int tiles_x, tiles_y, tiles_per_img, total_tiles;
  int ntn;  // N tiles of BN output channels (streamed weights only); see halo_tile()
  const uint16_t* w;  // packed [cb][tap][BN][64] (128 B swizzled rows)
  int wblocks;        // ncb * ntaps
  // epilogue (as ConvParams)
  uint16_t* out;
  int OH, OW;
  int out_pitch, out_coff;
  const uint16_t* res;
  int res_pitch, res_coff;
  const float* bias;
  const float* oscale;  // 8-bit: per output channel s_in * s_w[co], else null
  float res_scale;      // 8-bit: residual tensor scale, else 1
  float out_inv;        // 8-bit: 1 / output tensor scale, else 1
  int relu, out_mode;
  const float* w1;
  const float* b1;
  void* final_out;
};

// Shared memory plan (bytes): patch ring | weights (resident or ring) |
// output staging (TMA-store source) | residual tiles (TMA-load target) |
// barriers.  Staging / residual tiles are [128 positions][IB bytes] boxes in
// the tensor map's swizzle (IB = 128 -> 128B, 64 -> 64B, 32 -> 32B) so the
// epilogue's per-position 16-byte accesses are bank-conflict free.
// PAIR: CTA-pair variant (cta_group::2): each CTA holds half of every weight
// block (MN / 2 rows), so the same smem carries twice the weight ring.
template <int BN, int MODE, bool FUSED, bool B_RES, int ES = 2, bool PAIR = false>
struct HaloCfg {
  static constexpr int NPH = HaloTaps<MODE>::NPH;
  static constexpr bool HAS_RES = MODE == HALO_CONV3 && !FUSED;  // every routed 3x3 block is residual
  static constexpr int PLANE_MAX = 2944;  // 18 x 10 x 16 B rounded to 128; also 22 x 8 and 17 x 9
  static constexpr int HSTAGE = 8 * PLANE_MAX;
  static constexpr bool MACRO = MODE == HALO_STEM4X || MODE == HALO_CONV3X2;
  static constexpr int MN = MACRO ? NPH * BN : BN;  // MMA N: every phase at once for macro-pixels
  static constexpr int BROWS = PAIR ? MN / 2 : MN;  // weight rows of a block held by one CTA
  // one (cb, tap) weight block (this CTA's rows); the macro-pixel output conv
  // keeps one block per tap: 64 channels SW128 + (16-bit) 16 channels SW32
  static constexpr int BBLK = MODE == HALO_CONV3X2 ? MN * BK * 2 + (ES == 2 ? MN * 32 : 0) : BROWS * BK * 2;
  static constexpr int WG = 3;              // streamed weights: taps per ring slot (one wait + commit each)
  static constexpr int GBLK = WG * BBLK;
  static constexpr int W_RES_BYTES = MODE == HALO_STEM4X ? 112 * 1024 : (MODE == HALO_CONV3X2 ? 120 * 1024 : 72 * 1024);
  static constexpr int IB = BN * ES < 128 ? BN * ES : 128;  // bytes per position per box
  static constexpr int NCH = BN * ES > 128 ? BN * ES / 128 : 1;  // boxes across the channels
  static constexpr int BOX = 128 * IB;                 // one [128][IB] box
  static constexpr int STG_BYTES = FUSED ? 0 : NPH * NCH * BOX;
  static constexpr int NSTG = FUSED ? 0 : (B_RES ? 2 : 1);
  static constexpr int RES_BYTES = HAS_RES ? NCH * BOX : 0;
  static constexpr int NRES = HAS_RES ? (B_RES ? 2 : 1) : 0;
  static constexpr int EPI_BYTES = NSTG * STG_BYTES + NRES * RES_BYTES;
  // patch stages: 3 where the weight ring still gets >= 2 groups; the ConvT's
  // 4-phase staging leaves room for only 3 weight groups (~0.9 us of MMAs,
  // less than the L2 round trip), so it trades a patch stage for a 4th group
  static constexpr int HS =
      MODE == HALO_CONVT2 ? 2 : ((B_RES || 3 * HSTAGE + EPI_BYTES + 2 * GBLK <= 220 * 1024) ? 3 : 2);
  static constexpr int FIXED = HS * HSTAGE + EPI_BYTES;
  static constexpr int BS_FIT = (220 * 1024 - FIXED) / GBLK;
  static constexpr int BS = B_RES ? 1 : (BS_FIT > 4 ? 4 : BS_FIT);
  static constexpr int B_BYTES = B_RES ? W_RES_BYTES : BS * GBLK;
  static constexpr int OFF_B = HS * HSTAGE;
  static constexpr int OFF_STG = OFF_B + B_BYTES;
  static constexpr int OFF_RES = OFF_STG + NSTG * STG_BYTES;
  static constexpr int OFF_BAR = OFF_RES + NRES * RES_BYTES;
  static constexpr int SMEM = 1024 + OFF_BAR + 512;
  static constexpr int ACC_COLS = NPH * BN;                // one accumulator: every phase
  static constexpr int NACC = 2 * ACC_COLS <= 512 ? 2 : 1;  // double-buffered when TMEM allows
  static constexpr int TMEM_COLS = NACC * ACC_COLS <= 32    ? 32
                                   : NACC * ACC_COLS <= 64  ? 64
                                   : NACC * ACC_COLS <= 128 ? 128
                                   : NACC * ACC_COLS <= 256 ? 256
                                                            : 512;
  static_assert(NACC * ACC_COLS <= 512, "accumulators exceed TMEM");
  static_assert(B_RES || BS >= 2, "weight ring too small");
  static_assert(SMEM <= 227 * 1024, "shared memory plan exceeds 227 KB");
};

// byte offset of 16-byte chunk j of box row r under the box's swizzle
template <int IB>
__device__ __forceinline__ uint32_t swz(int r, int j) {
  const uint32_t off = (uint32_t)(r * IB + j * 16);
  constexpr uint32_t mask = IB == 128 ? 7u : (IB == 64 ? 3u : (IB == 32 ? 1u : 0u));  // 16 B rows: no swizzle
  return off ^ (((off >> 7) & mask) << 4);
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int c, int x, int y, int n) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c), "r"(x), "r"(y), "r"(n)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void tma_tile_4d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c, int x, int y,
                                            int n) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(tc::smem_u32(bar)), "r"(c), "r"(x), "r"(y), "r"(n)
      : "memory");
}

// CTA-pair forms: data to this CTA's smem, completion on the even CTA's
// barrier (cluster address)
__device__ __forceinline__ void tma_tile_4d_pair(uint32_t dst, const CUtensorMap* map, uint32_t mbar, int c, int x,
                                                 int y, int n) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(c), "r"(x), "r"(y), "r"(n)
      : "memory");
}
__device__ __forceinline__ void tma_2d_pair_h(uint32_t dst, const CUtensorMap* map, uint32_t mbar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(tc::smem_u32(p)));
  return r;
}

// Tile t -> (spatial tile ts, N tile nt): pairs of adjacent t are two adjacent
// spatial tiles of the SAME N tile (a CTA pair shares its weights), and
// consecutive pairs walk the N tiles of one spatial pair (its patches stay in
// L2).  With one N tile this is the identity.  Needs an even spatial count.
__device__ __forceinline__ void halo_tile(const HaloParams& p, int t, int& ts, int& nt) {
  const int g = t >> 1, sp = g / p.ntn;
  nt = g - sp * p.ntn;
  ts = 2 * sp + (t & 1);
}

__device__ __forceinline__ uint64_t halo_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // layout 0: no swizzle
}

// PAIR: launched in clusters of two; CTA r of a cluster owns tile
// blockIdx.x + k * gridDim.x as usual (the pair = two adjacent tiles, the tile
// count is even), the even CTA issues M = 256 MMAs over both CTAs' patches
// and weight halves, both CTAs' TMA loads complete on the even CTA's
// barriers, commits are multicast, and every epilogue warp of the pair
// releases the accumulator on the even CTA's tempty barrier.
template <int BN, int MODE, bool FUSED_OUT, int PR, bool B_RES, bool PAIR = false>
__global__ void __launch_bounds__(NUM_THREADS, 1) conv_halo(const __grid_constant__ HaloParams p) {
  static_assert(MODE != HALO_CONV3S2 || (B_RES && !PAIR && !FUSED_OUT), "stride-2 halo: resident weights only");
  using NF = Num<PR>;
  using CF = HaloCfg<BN, MODE, FUSED_OUT, B_RES, NF::Q8 ? 1 : 2, PAIR>;
  using TT = HaloTaps<MODE>;
  constexpr int NPH = TT::NPH;
  constexpr int HS = CF::HS, BS = CF::BS, NACC = CF::NACC;
  static_assert(!FUSED_OUT || NPH == 1 || MODE == HALO_CONV3X2, "fused output conv: one phase, or 2-pixel macro columns");
  // epilogue warps 2-9 = two groups of four (one per TMEM lane quadrant).
  // SPLIT: both groups take every tile, half the channels each.  Otherwise
  // (BN = 16, or the fused 1x1 output) the groups alternate tiles, group g
  // owning accumulator g.
  // Resident-weight variants have double-buffered staging/residual tiles, so
  // the groups can own alternate tiles (one accumulator, staging buffer and
  // residual slot each; 128-thread barriers) and two tiles' epilogues run
  // concurrently -- the epilogue, not the MMA, bounds these narrow layers in
  // fp8.  Streamed-weight variants (single staging buffer) split channels.
  constexpr bool SPLIT = !FUSED_OUT && BN >= 32 && !B_RES;
  constexpr bool EPI_ALT = !SPLIT && NACC == 2;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* sH = smem;
  uint8_t* sB = smem + CF::OFF_B;
  uint64_t* hfull = reinterpret_cast<uint64_t*>(smem + CF::OFF_BAR);
  uint64_t* hempty = hfull + HS;
  uint64_t* bfull = hempty + HS;
  uint64_t* bempty = bfull + BS;
  uint64_t* tfull = bempty + BS;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;
  uint64_t* rempty = rfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty + 2);
  constexpr int EPI_THREADS = EPI_ALT ? 32 * NUM_EPI_WARPS / 2 : 32 * NUM_EPI_WARPS;  // per tile
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? tc::cluster_ctarank() : 0u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < HS; ++s) {
      tc::mbar_init(&hfull[s], 1);
      tc::mbar_init(&hempty[s], 1);
    }
    for (int s = 0; s < BS; ++s) {
      tc::mbar_init(&bfull[s], 1);
      tc::mbar_init(&bempty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], PAIR ? 2 * (EPI_THREADS / 32) : EPI_THREADS);  // pair: one arrive per warp
      tc::mbar_init(&rfull[a], 1);
      tc::mbar_init(&rempty[a], EPI_THREADS);
    }
    tc::fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap)) : "memory");
    if constexpr (!FUSED_OUT)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap_out)) : "memory");
    if constexpr (CF::HAS_RES)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap_res)) : "memory");
    if constexpr (PAIR) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.wmap)) : "memory");
  }
  if (warp == 1) {
    if constexpr (PAIR) tc::tmem_alloc2<CF::TMEM_COLS>(tmem_slot);
    else tc::tmem_alloc<CF::TMEM_COLS>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) tc::cluster_sync();  // both CTAs' barriers exist before cross-CTA signals
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t box_bytes = (uint32_t)(p.pw * p.ph * 16);
  tc::griddep_launch();
  // LSG_TRACE: cycles per role -- 0 producer hempty, 1 MMA bfull (streamed weights),
  // 2 producer total, 3 MMA tempty, 4 MMA hfull, 5 MMA total, 6 epilogue
  // staging drain + group barrier, 7 epilogue rfull, 8 epilogue tfull,
  // 9 epilogue math + staging, 10 epilogue total (summed over the two groups)
  long long hw[11] = {};
  (void)hw;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
#ifdef LSG_TRACE
    const long long tr0 = clock64();
#endif
    const uint32_t sH0 = tc::smem_u32(sH), sB0 = tc::smem_u32(sB);
    if constexpr (B_RES) {
      if (lane == 0) {  // every weight block of this layer, once per CTA
        const uint32_t bytes = (uint32_t)(p.wblocks * CF::BBLK);
        if constexpr (PAIR) {  // this CTA's half of each block, completing on the even CTA's barrier
          if (rank == 0) tc::mbar_arrive_expect_tx(&bfull[0], 2 * bytes);
          const uint32_t fb = leader_addr(&bfull[0]);
          for (int b = 0; b < p.wblocks; ++b)
            tma_2d_pair_h(sB0 + b * CF::BBLK, &p.wmap, fb, 0, b * CF::MN + (int)rank * CF::BROWS);
        } else {
          tc::mbar_arrive_expect_tx(&bfull[0], bytes);
          for (uint32_t off = 0; off < bytes; off += 32768) {
            const uint32_t chunk = bytes - off < 32768 ? bytes - off : 32768;
            tc::bulk_g2s(sB0 + off, reinterpret_cast<const uint8_t*>(p.w) + off, chunk, &bfull[0]);
          }
        }
      }
      __syncwarp();
    }
    tc::griddep_wait();  // weights are constant; activations come from the previous layer
    // plane g of channel block cb: channels (cb*8 + g)*8 at x0, or channels 0..7 at x0 + g
    const int cstep = p.shift_planes ? 0 : 8, xstep = p.shift_planes ? 1 : 0;
    int hs = 0, bs = 0;
    uint32_t hph = 0, bph = 0;
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
      int ts, nt;
      halo_tile(p, t, ts, nt);
      const int n = ts / p.tiles_per_img, r = ts - n * p.tiles_per_img;
      const int ty = r / p.tiles_x, tx = r - ty * p.tiles_x;
      const int y0 = ty * HTH + p.oy0, x0 = tx * HTW * p.xmul + p.ox0;

      for (int cb = 0; cb < p.ncb; ++cb) {
        const int g0 = cb * 8, ng = min(8, p.ngran - g0);
        LSG_HW(hw, 0, tc::mbar_wait(&hempty[hs], hph ^ 1));
        if (lane == 0 && rank == 0)
          tc::mbar_arrive_expect_tx(&hfull[hs], (PAIR ? 2 : 1) *
                                                    (MODE == HALO_CONV3S2   ? 8
                                                     : MODE == HALO_CONV3X2 ? 2 * min(4, p.ngran - cb * 4)
                                                                            : ng) *
                                                    box_bytes);
        __syncwarp();
        if constexpr (MODE == HALO_CONV3X2) {
          const int gs = lane & 3, g = cb * 4 + gs;  // plane lane = parity (lane >> 2) x granule slot
          if (lane < 8 && g < p.ngran)
            tma_tile_4d(sH0 + hs * CF::HSTAGE + lane * p.plane, &p.tmap, &hfull[hs], g * 8,
                        2 * (tx * HTW) - 1 + (lane >> 2), ty * HTH - 1, n);
        } else if constexpr (MODE == HALO_CONV3S2) {
          if (lane < 8) {  // plane lane = parity (lane >> 1) x granule (lane & 1) of this channel block
            const int pp = lane >> 1;
            tma_tile_4d(sH0 + hs * CF::HSTAGE + lane * p.plane, &p.tmap, &hfull[hs], (cb * 2 + (lane & 1)) * 8,
                        2 * (tx * HTW - 1) + (pp & 1), 2 * (ty * HTH - 1) + (pp >> 1), n);
          }
        } else if (lane < ng) {
          if constexpr (PAIR)
            tma_tile_4d_pair(sH0 + hs * CF::HSTAGE + lane * p.plane, &p.tmap, leader_addr(&hfull[hs]),
                             (g0 + lane) * cstep, x0 + (g0 + lane) * xstep, y0, n);
          else
            tma_tile_4d(sH0 + hs * CF::HSTAGE + lane * p.plane, &p.tmap, &hfull[hs], (g0 + lane) * cstep,
                        x0 + (g0 + lane) * xstep, y0, n);
        }
        if (++hs == HS) {
          hs = 0;
          hph ^= 1;
        }
        if constexpr (!B_RES) {  // taps [g*WG, g*WG+WG) of this channel block per ring slot
          const uint16_t* wb = p.w + ((size_t)nt * p.ncb + cb) * p.ntaps * CF::MN * BK;
          for (int t0 = 0; t0 < p.ntaps; t0 += CF::WG) {
            const uint32_t bytes = (uint32_t)(min(CF::WG, p.ntaps - t0) * CF::BBLK);
            tc::mbar_wait(&bempty[bs], bph ^ 1);
            if (lane == 0) {
              if constexpr (PAIR) {
                if (rank == 0) tc::mbar_arrive_expect_tx(&bfull[bs], 2 * bytes);
                const uint32_t fb = leader_addr(&bfull[bs]);
                for (int i = 0; i < min(CF::WG, p.ntaps - t0); ++i)
                  tma_2d_pair_h(sB0 + bs * CF::GBLK + i * CF::BBLK, &p.wmap, fb, 0,
                                ((nt * p.ncb + cb) * p.ntaps + t0 + i) * CF::MN + (int)rank * CF::BROWS);
              } else {
                tc::mbar_arrive_expect_tx(&bfull[bs], bytes);
                tc::bulk_g2s(sB0 + bs * CF::GBLK, wb + (size_t)t0 * CF::MN * BK, bytes, &bfull[bs]);
              }
            }
            __syncwarp();
            if (++bs == BS) {
              bs = 0;
              bph ^= 1;
            }
          }
        }
      }
    }
#ifdef LSG_TRACE
    hw[2] = clock64() - tr0;
    if (lane == 0) {
      LSG_HW_FLUSH(p.trace_slot, hw, 0, 1);
      LSG_HW_FLUSH(p.trace_slot, hw, 2, 3);
    }
#endif
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // One elected lane issues everything.  Descriptors are linear in the
    // start address (14-bit field; smem < 256 KB never carries), so every
    // tap / K step is a compile-time add to a per-patch base, and the
    // clobber-free wrappers let parameters stay in registers: the issue loop
    // is a handful of uniform adds per 4 MMAs (profiles/r01: with divisions,
    // parameter reloads and per-tap warp reconvergence it cost more than the
    // MMAs themselves).
    constexpr uint32_t idesc = NF::idesc(PAIR ? 2 * BM : BM, CF::MN);
    constexpr int NT = TT::NT;
    constexpr uint64_t PLANE2 = (uint64_t)((2 * ((TT::PW * TT::PH * 16 + 127) / 128 * 128)) >> 4);
    constexpr uint64_t BBLK16 = CF::BBLK >> 4;
    constexpr uint64_t HST16 = CF::HSTAGE >> 4;
    if ((!PAIR || rank == 0) && elect_one()) {
#ifdef LSG_TRACE
      const long long tr0 = clock64();
#endif
      const uint32_t sH0 = tc::smem_u32(sH), sB0 = tc::smem_u32(sB);
      if constexpr (B_RES) tc::mbar_wait_nc(&bfull[0], 0);
      const uint64_t a_desc0 = halo_desc(sH0, (uint32_t)(PLANE2 << 3), (uint32_t)(TT::PW * 16));
      const uint64_t b_desc0 = tc::sdesc_sw128(sB0);
      const int ncb = p.ncb, ngran = p.ngran, total = p.total_tiles;
      int hs = 0, bs = 0;
      uint32_t hph = 0, bph = 0, tl = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++tl) {
        const uint32_t a = NACC == 2 ? (tl & 1) : 0, use = NACC == 2 ? (tl >> 1) : tl;
        if constexpr (PAIR) LSG_HW(hw, 3, tc::mbar_wait_cluster(&tempty[a], (use & 1) ^ 1));  // both CTAs' epilogues
        else LSG_HW(hw, 3, tc::mbar_wait_fast(&tempty[a], (use & 1) ^ 1));
        tc::tc_fence_after_nc();  // TMEM reuse after the epilogue's reads
        const uint32_t d = tmem + a * CF::ACC_COLS;
        for (int cb = 0; cb < ncb; ++cb) {
          const int ksteps = MODE == HALO_CONV3S2   ? 1
                             : MODE == HALO_CONV3X2 ? min(4, ngran - cb * 4) >> 1
                                                    : min(8, ngran - cb * 8) >> 1;
          LSG_HW(hw, 4, tc::mbar_wait_fast(&hfull[hs], hph));  // TMA data: the mbarrier alone orders it
          const uint64_t ah = a_desc0 + (uint64_t)hs * HST16;
          const uint64_t bcb = b_desc0 + (uint64_t)(cb * NT) * BBLK16;
#pragma unroll
          for (int tap = 0; tap < NT; ++tap) {
            uint64_t db;
            if constexpr (MODE == HALO_CONV3X2) {  // one block per tap; K step cb*2+ks (B below)
              db = b_desc0 + (uint64_t)tap * BBLK16;
            } else if constexpr (MODE == HALO_CONV3S2) {  // one block per tap; channel block cb = K offset 32 * cb bytes
              db = b_desc0 + (uint64_t)tap * BBLK16 + (uint64_t)(2 * cb);
            } else if constexpr (B_RES) {
              db = bcb + (uint64_t)tap * BBLK16;
            } else {
              if (tap % CF::WG == 0) LSG_HW(hw, 1, tc::mbar_wait_fast(&bfull[bs], bph));
              db = b_desc0 + (uint64_t)bs * (CF::GBLK >> 4) + (uint64_t)(tap % CF::WG) * BBLK16;
            }
            const uint64_t at = ah + (uint64_t)TT::aoff(tap);
            const uint32_t dd = d + (uint32_t)(MODE == HALO_STEM4X ? 0 : TT::phase(tap) * BN);
            bool first = true;  // first tap of its phase (compile time)
#pragma unroll
            for (int u = 0; u < tap; ++u) first = first && TT::phase(u) != TT::phase(tap);
            const uint32_t acc0 = (first && cb == 0) ? 0u : 1u;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              if constexpr (MODE == HALO_CONV3X2) {
                if (ks < ksteps) {
                  const int kg = cb * 2 + ks;  // global K step: 0-3 in the SW128 part, 4 in the SW32 part
                  uint64_t bk;
                  if (kg < 4) {
                    bk = db + (uint64_t)(2 * kg);
                  } else {
                    const uint32_t a32 = sB0 + (uint32_t)(tap * CF::BBLK + CF::MN * BK * 2);
                    bk = (uint64_t)((a32 >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
                         (1ull << 46) | (6ull << 61);  // K-major, 32-byte swizzle, 8-row groups 256 B apart
                  }
                  NF::mma_nc(dd, at + ks * PLANE2, bk, idesc, (ks || cb || tap) ? 1u : 0u);
                }
              } else if (ks < ksteps) {
                if constexpr (PAIR) {
                  NF::mma2(dd, at + ks * PLANE2, db + 2 * ks, idesc, ks ? 1u : acc0);
                } else {
                  NF::mma_nc(dd, at + ks * PLANE2, db + 2 * ks, idesc, ks ? 1u : acc0);
                }
              }
            if constexpr (!B_RES) {
              if (tap % CF::WG == CF::WG - 1 || tap == NT - 1) {
                if constexpr (PAIR) tc::mma_commit2(&bempty[bs]);
                else tc::mma_commit_nc(&bempty[bs]);
                if (++bs == BS) {
                  bs = 0;
                  bph ^= 1;
                }
              }
            }
          }
          if constexpr (PAIR) tc::mma_commit2(&hempty[hs]);
          else tc::mma_commit_nc(&hempty[hs]);
          if (++hs == HS) {
            hs = 0;
            hph ^= 1;
          }
        }
        if constexpr (PAIR) tc::mma_commit2(&tfull[a]);
        else tc::mma_commit_nc(&tfull[a]);
      }
#ifdef LSG_TRACE
      hw[5] = clock64() - tr0;
      LSG_HW_FLUSH(p.trace_slot, hw, 3, 6);
      LSG_HW_FLUSH(p.trace_slot, hw, 1, 2);
#endif
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ epilogue (warps 2-9)
    tc::griddep_wait();
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int HC = SPLIT ? BN / 2 : BN;
    const int cbeg = SPLIT ? half * HC : 0;
    const int r = q * 32 + lane;  // tile position: row r / 8, column r % 8
    constexpr int step = EPI_ALT ? 2 : 1;
    uint32_t tl = EPI_ALT ? (uint32_t)half : 0u;
    // grid position of tile t for this thread
    auto gpos = [&](int t, int& n, int& gy, int& gx) {
      n = t / p.tiles_per_img;
      const int rr = t - n * p.tiles_per_img;
      const int ty = rr / p.tiles_x, tx = rr - ty * p.tiles_x;
      gy = ty * HTH + (r >> 3);
      gx = tx * HTW + (r & 7);
    };
    if constexpr (!FUSED_OUT) {
      // Staged epilogue: TMEM -> +bias (+residual from the TMA-loaded tile)
      // -> ReLU -> 16-bit -> swizzled staging box -> one TMA tensor store per
      // (phase, 64-channel chunk).  Coalescing is the TMA's job; the 16-byte
      // row accesses of the threads stay bank-conflict free.
      constexpr int IB = CF::IB;
      const int grp = EPI_ALT ? half : 0;
      const bool leader = (warp == 2 + 4 * grp) && lane == 0;  // issues the group's stores
      int sb = 0;
      // Residual boxes: the group's leader loads them (not the producer, whose
      // patch prefetch would otherwise stall behind the epilogue on the ring),
      // the next tile's as soon as every thread of the group holds this
      // tile's in registers -- its latency hides under this tile's math.  One
      // slot per group (NRES == step): tile tl's slot is tl % NRES.
      static_assert(!CF::HAS_RES || (CF::NRES == step && NPH == 1), "residual ring: one slot per epilogue group");
      auto issue_res = [&](int tt, int slot) {
        int ts2, nt2;
        halo_tile(p, tt, ts2, nt2);
        const int n2 = ts2 / p.tiles_per_img, r2 = ts2 - n2 * p.tiles_per_img;
        const int ty2 = r2 / p.tiles_x, tx2 = r2 - ty2 * p.tiles_x;
        tc::mbar_arrive_expect_tx(&rfull[slot], CF::RES_BYTES);
        const uint32_t dst = tc::smem_u32(smem + CF::OFF_RES + slot * CF::RES_BYTES);
#pragma unroll
        for (int cc = 0; cc < CF::NCH; ++cc)
          tma_tile_4d(dst + cc * CF::BOX, &p.tmap_res, &rfull[slot], nt2 * (BN / NF::CPU) + cc * 64, tx2 * HTW,
                      ty2 * HTH, n2);
      };
      if constexpr (CF::HAS_RES) {
        const int t0 = blockIdx.x + (int)tl * gridDim.x;
        if (leader && t0 < p.total_tiles) issue_res(t0, (int)(tl % (uint32_t)step));
      }
#ifdef LSG_TRACE
      const long long tr0 = clock64();
#endif
      for (int t = blockIdx.x + (int)tl * gridDim.x; t < p.total_tiles; t += step * gridDim.x, tl += step) {
        const uint32_t a = NACC == 2 ? (tl & 1) : 0, use = NACC == 2 ? (tl >> 1) : tl;
        // residual ring slot of this tile
        const int rs = CF::NRES ? (int)(tl % (uint32_t)(CF::NRES ? CF::NRES : 1)) : 0;
        const uint32_t rph = CF::NRES ? (tl / (uint32_t)(CF::NRES ? CF::NRES : 1)) & 1u : 0u;
        int ts, nt;
        halo_tile(p, t, ts, nt);
        const int n = ts / p.tiles_per_img, rr = ts - n * p.tiles_per_img;
        const int ty = rr / p.tiles_x, tx = rr - ty * p.tiles_x;
        uint8_t* stg = smem + CF::OFF_STG + (EPI_ALT ? grp : sb) * CF::STG_BYTES;
        // the store that last read this staging buffer must have drained
        LSG_HW(hw, 6, if (leader) bulk_wait_read<EPI_ALT ? 0 : CF::NSTG - 1>(); named_bar(1 + grp, EPI_THREADS));
        constexpr int W16 = NF::U4, ES = NF::Q8 ? 1 : 2;
        uint4 rvall[CF::HAS_RES ? HC / 16 : 1][W16];
        if constexpr (CF::HAS_RES) {
          const uint8_t* res = smem + CF::OFF_RES + rs * CF::RES_BYTES;
          LSG_HW(hw, 7, tc::mbar_wait(&rfull[rs], rph));
#pragma unroll
          for (int c0 = 0; c0 < HC; c0 += 16) {
            const int byte0 = (cbeg + c0) * ES;
            const int cc = byte0 >> 7, j0 = (byte0 & 127) >> 4;
#pragma unroll
            for (int w = 0; w < W16; ++w)
              rvall[c0 / 16][w] = *reinterpret_cast<const uint4*>(res + cc * CF::BOX + swz<IB>(r, j0 + w));
          }
          tc::mbar_arrive(&rempty[rs]);
          if (leader && t + step * (int)gridDim.x < p.total_tiles) {
            tc::mbar_wait(&rempty[rs], rph);  // the whole group holds this box
            issue_res(t + step * (int)gridDim.x, rs);
          }
        }
        LSG_HW(hw, 8, tc::mbar_wait(&tfull[a], use & 1));
        tc::tc_fence_after();
#ifdef LSG_TRACE
        const long long tm0 = clock64();
#endif
        // EARLY: this thread's whole share of the accumulator (<= 64 columns)
        // goes to registers in one TMEM round trip and the accumulator is
        // released before the math, so the next-but-one tile's MMAs overlap
        // this epilogue instead of waiting for it (2 accumulators)
        constexpr bool EARLY = NPH * HC <= 64;
        uint32_t vall[EARLY ? NPH * HC / 16 : 1][16];
        if constexpr (EARLY) {
#pragma unroll
          for (int z = 0; z < NPH; ++z)
#pragma unroll
            for (int c0 = 0; c0 < HC; c0 += 16)
              tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + a * CF::ACC_COLS + z * BN + cbeg + c0,
                            vall[(z * HC + c0) / 16]);
          tc::tmem_ld_wait();
          tc::tc_fence_before();
          if constexpr (PAIR) {
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_remote(&tempty[a], 0);
          } else {
            tc::mbar_arrive(&tempty[a]);
          }
        }
#pragma unroll
        for (int z = 0; z < NPH; ++z) {
          const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + a * CF::ACC_COLS + z * BN + cbeg;
#pragma unroll
          for (int c0 = 0; c0 < HC; c0 += 16) {
            uint32_t v[16];
            if constexpr (EARLY) {
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = vall[(z * HC + c0) / 16][j];
            } else {
              tc::tmem_ld16(tbase + c0, v);
            }
            // 16 channels = W16 16-byte chunks of the position's box row
            const int byte0 = (cbeg + c0) * ES;
            const int cc = byte0 >> 7, j0 = (byte0 & 127) >> 4;
            if constexpr (!EARLY) tc::tmem_ld_wait();
            uint4 o[W16];
            epi16<PR>(v, p.bias + nt * BN + cbeg + c0, p.oscale + (NF::Q8 ? nt * BN + cbeg + c0 : 0),
                      CF::HAS_RES ? rvall[c0 / 16] : nullptr, p.res_scale, p.relu != 0, p.out_inv, o);
#pragma unroll
            for (int w = 0; w < W16; ++w)
              *reinterpret_cast<uint4*>(stg + (z * CF::NCH + cc) * CF::BOX + swz<IB>(r, j0 + w)) = o[w];
          }
        }
        if constexpr (!EARLY) {
          tc::tc_fence_before();
          if constexpr (PAIR) {
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_remote(&tempty[a], 0);
          } else {
            tc::mbar_arrive(&tempty[a]);
          }
        }
#ifdef LSG_TRACE
        hw[9] += clock64() - tm0;
#endif
        tc::fence_proxy_async();  // staging writes -> visible to the TMA (async proxy)
        named_bar(1 + grp, EPI_THREADS);
        if (leader) {
          const uint32_t src = tc::smem_u32(stg);
#pragma unroll
          for (int z = 0; z < NPH; ++z)
#pragma unroll
            for (int cc = 0; cc < CF::NCH; ++cc)
              tma_store_4d(&p.tmap_out, src + (z * CF::NCH + cc) * CF::BOX, nt * (BN / NF::CPU) + cc * 64,
                           tx * HTW * p.osx + p.pox[z], ty * HTH * p.osy + p.poy[z], n);
          if (p.out2) {
#pragma unroll
            for (int z = 0; z < NPH; ++z)
#pragma unroll
              for (int cc = 0; cc < CF::NCH; ++cc)
                tma_store_4d(&p.tmap_out2, src + (z * CF::NCH + cc) * CF::BOX, cc * 64, tx * HTW * p.osx + p.pox[z],
                             ty * HTH * p.osy + p.poy[z], n);
          }
          bulk_commit();
        }
        if (++sb == CF::NSTG) sb = 0;
      }
      if (leader) bulk_wait_all();
#ifdef LSG_TRACE
      hw[10] = clock64() - tr0;
      if ((warp & 3) == 2 && lane == 0) LSG_HW_FLUSH(p.trace_slot, hw, 6, 11);
#endif
    } else {
      for (int t = blockIdx.x + (int)tl * gridDim.x; t < p.total_tiles; t += step * gridDim.x, tl += step) {
        const uint32_t a = tl & 1, use = tl >> 1;
        int n, gy, gx;
        gpos(t, n, gy, gx);
        const bool gvalid = gy < p.GH && gx < p.GW;
        tc::mbar_wait(&tfull[a], use & 1);
        tc::tc_fence_after();
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + a * CF::ACC_COLS;
        float oz[NPH][3];
#pragma unroll
        for (int z = 0; z < NPH; ++z) {  // macro-pixels: phase z = output column 2 gx + z
          float* o = oz[z];
          o[0] = __ldg(p.b1 + 0);
          o[1] = __ldg(p.b1 + 1);
          o[2] = __ldg(p.b1 + 2);
#pragma unroll
          for (int c0 = 0; c0 < BN; c0 += 16) {
            uint32_t v[16];
            tc::tmem_ld16(tbase + z * BN + c0, v);
            tc::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float acc = NF::Q8 ? NF::acc(v[j]) * __ldg(p.oscale + c0 + j) : __uint_as_float(v[j]);
              const float xx = fmaxf(acc + __ldg(p.bias + c0 + j), 0.f);
#pragma unroll
              for (int o3 = 0; o3 < 3; ++o3) o[o3] = fmaf(__ldg(p.w1 + o3 * 32 + c0 + j), xx, o[o3]);
            }
          }
        }
        tc::tc_fence_before();
        if constexpr (PAIR) {  // accumulator drained: stores below overlap the next tile's MMAs
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_remote(&tempty[a], 0);
        } else {
          tc::mbar_arrive(&tempty[a]);
        }
#pragma unroll
        for (int z = 0; z < NPH; ++z) {
        const float* o = oz[z];
        if (gvalid) {
          const int HWo = p.OH * p.OW;
          const size_t pp = (size_t)gy * p.OW + gx * p.osx + p.pox[z];
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
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) tc::cluster_sync();  // the peer's TMEM / smem / barriers stay live until both are done
  if (warp == 1) {
    tc::tc_fence_after();
    if constexpr (PAIR) tc::tmem_dealloc2<CF::TMEM_COLS>(tmem);
    else tc::tmem_dealloc<CF::TMEM_COLS>(tmem);
  }
}

}  // namespace gen
}  // namespace lsg
