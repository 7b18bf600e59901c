// generator.cu -- Wav2Lip generator forward on sm_100a tensor cores
// (include/lsg.h "generator").
//
// The reference renders with a cost model only (mock_lipsync,
// visual_mocks.cpp:40-51; profiles wav2lip_fp32 / wav2lip_trt_fp16 at
// visual_mocks.cpp:24-26); this is the network those profiles stand for,
// restated from the public Wav2Lip topology: audio
// encoder on the [80 x 16] mel window, face encoder on [target(masked) ||
// reference], decoder of transposed convs with skip concatenation, 1x1 +
// sigmoid output.  BatchNorm is folded into the weights on the host.
//
// Every layer is one launch of conv_tc, an implicit-GEMM convolution:
//   M = output pixels (batch folded in), N = Cout, K = taps x Cin (NHWC, K
//   ordered tap-major so a 64-wide K block is one tap when Cin >= 64).
//   * producer warps 0-3 gather the im2col rows of A straight from the NHWC
//     activation with 16-byte cp.async (zero-fill for padding/halo) into a
//     128-byte-swizzled K-major tile;
//   * the packed weight tile B is one bulk async copy (TMA engine) per stage;
//   * warp 8 issues tcgen05.mma (M=128, N=BN, K=16) into a TMEM accumulator;
//   * warps 4-7 drain TMEM with tcgen05.ld and run the fused epilogue:
//     folded-BN bias, residual add, ReLU, bf16 store into a channel slice of
//     the destination (skip concatenation is free: encoder features are
//     written straight into the decoder's concat buffers), or, for the last
//     layer, the 1x1 32->3 conv + sigmoid of the output block.
//   * stride-2 transposed convs run as 4 phase GEMMs (1/2/2/4 taps) in one
//     launch (grid.z = phase), so no zero-insertion work is done.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "conv_halo.cuh"
#include "conv_kernel.cuh"
#include "conv_pair.cuh"
#include "gen_internal.h"
#include "lsg_common.cuh"
#include "tc.cuh"

namespace lsg {
namespace gen {

enum { CONV = 0, CONVT = 1 };

struct LayerSpec {
  const char* name;
  int kind, cin, cout, kh, kw, sh, sw, ph, pw, oph, opw, res;
};

// Layer order = weight blob order.  conv weights are
// [cout][cin][kh][kw], convT weights [cin][cout][kh][kw], each followed by
// bias[cout]; BN already folded.
static const LayerSpec kLayers[] = {
    // face encoder (7 blocks)
    {"fe0", CONV, 6, 16, 7, 7, 1, 1, 3, 3, 0, 0, 0},
    {"fe1.0", CONV, 16, 32, 3, 3, 2, 2, 1, 1, 0, 0, 0},
    {"fe1.1", CONV, 32, 32, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fe1.2", CONV, 32, 32, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fe2.0", CONV, 32, 64, 3, 3, 2, 2, 1, 1, 0, 0, 0},
    {"fe2.1", CONV, 64, 64, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fe2.2", CONV, 64, 64, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fe2.3", CONV, 64, 64, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fe3.0", CONV, 64, 128, 3, 3, 2, 2, 1, 1, 0, 0, 0},
    {"fe3.1", CONV, 128, 128, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fe3.2", CONV, 128, 128, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fe4.0", CONV, 128, 256, 3, 3, 2, 2, 1, 1, 0, 0, 0},
    {"fe4.1", CONV, 256, 256, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fe4.2", CONV, 256, 256, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fe5.0", CONV, 256, 512, 3, 3, 2, 2, 1, 1, 0, 0, 0},
    {"fe5.1", CONV, 512, 512, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fe6.0", CONV, 512, 512, 3, 3, 1, 1, 0, 0, 0, 0, 0},
    {"fe6.1", CONV, 512, 512, 1, 1, 1, 1, 0, 0, 0, 0, 0},
    // audio encoder
    {"ae0", CONV, 1, 32, 3, 3, 1, 1, 1, 1, 0, 0, 0},
    {"ae1", CONV, 32, 32, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"ae2", CONV, 32, 32, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"ae3", CONV, 32, 64, 3, 3, 3, 1, 1, 1, 0, 0, 0},
    {"ae4", CONV, 64, 64, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"ae5", CONV, 64, 64, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"ae6", CONV, 64, 128, 3, 3, 3, 3, 1, 1, 0, 0, 0},
    {"ae7", CONV, 128, 128, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"ae8", CONV, 128, 128, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"ae9", CONV, 128, 256, 3, 3, 3, 2, 1, 1, 0, 0, 0},
    {"ae10", CONV, 256, 256, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"ae11", CONV, 256, 512, 3, 3, 1, 1, 0, 0, 0, 0, 0},
    {"ae12", CONV, 512, 512, 1, 1, 1, 1, 0, 0, 0, 0, 0},
    // decoder
    {"fd0", CONV, 512, 512, 1, 1, 1, 1, 0, 0, 0, 0, 0},
    {"fd1.0", CONVT, 1024, 512, 3, 3, 1, 1, 0, 0, 0, 0, 0},
    {"fd1.1", CONV, 512, 512, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fd2.0", CONVT, 1024, 512, 3, 3, 2, 2, 1, 1, 1, 1, 0},
    {"fd2.1", CONV, 512, 512, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fd2.2", CONV, 512, 512, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fd3.0", CONVT, 768, 384, 3, 3, 2, 2, 1, 1, 1, 1, 0},
    {"fd3.1", CONV, 384, 384, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fd3.2", CONV, 384, 384, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fd4.0", CONVT, 512, 256, 3, 3, 2, 2, 1, 1, 1, 1, 0},
    {"fd4.1", CONV, 256, 256, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fd4.2", CONV, 256, 256, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fd5.0", CONVT, 320, 128, 3, 3, 2, 2, 1, 1, 1, 1, 0},
    {"fd5.1", CONV, 128, 128, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fd5.2", CONV, 128, 128, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fd6.0", CONVT, 160, 64, 3, 3, 2, 2, 1, 1, 1, 1, 0},
    {"fd6.1", CONV, 64, 64, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    {"fd6.2", CONV, 64, 64, 3, 3, 1, 1, 1, 1, 0, 0, 1},
    // output block: conv 80->32 (+BN, ReLU), conv 1x1 32->3 (bias), sigmoid
    {"out0", CONV, 80, 32, 3, 3, 1, 1, 1, 1, 0, 0, 0},
    {"out1", CONV, 32, 3, 1, 1, 1, 1, 0, 0, 0, 0, 0},
};
constexpr int kNumLayers = sizeof(kLayers) / sizeof(kLayers[0]);
constexpr int kAe0 = 18;  // plan index of ae0 (checked against the layer table at create)
static_assert(kNumLayers == 51, "Wav2Lip has 51 conv layers");

// ------------------------------------------------------------ input prep
// Both inputs are 16 bytes per pixel: 8 channels of bf16/fp16, or 16 fp8
// channels (values * inv_scale) -- the same tensor-map geometry either way.
template <int PR>
__device__ __forceinline__ uint4 pack_px(const float (&c)[6], float inv_scale) {
  using NF = Num<PR>;
  if constexpr (NF::Q8) {
    float f[16] = {};
#pragma unroll
    for (int j = 0; j < 6; ++j) f[j] = c[j] * inv_scale;
    uint4 o;
    NF::from_float16(f, &o);
    return o;
  } else {
    return make_uint4(NF::pack(c[0], c[1]), NF::pack(c[2], c[3]), NF::pack(c[4], c[5]), 0u);
  }
}

// faces: [B][96][96][3] u8 target (rows >= 48 masked), refs [R][96][96][3]
// -> [B][96][96][16 B] = (target/255 masked, ref/255, 0...)
template <int PR>
__global__ void prep_faces(const uint8_t* __restrict__ target, const int64_t* __restrict__ target_idx,
                           const uint8_t* __restrict__ refs, const int32_t* __restrict__ ref_index,
                           uint16_t* __restrict__ out, int B, float inv_scale) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // pixel
  const int64_t total = (int64_t)B * 96 * 96;
  if (i >= total) return;
  const int b = (int)(i / (96 * 96));
  const int pix = (int)(i - (int64_t)b * 96 * 96);
  const int y = pix / 96;
  const int64_t tf = target_idx ? __ldg(target_idx + b) : b;
  const uint8_t* t = target + (tf * 96 * 96 + pix) * 3;
  const uint8_t* r = refs + ((int64_t)__ldg(ref_index + b) * 96 * 96 + pix) * 3;
  const float k = 1.f / 255.f;
  const bool mask = y >= 48;
  const float c[6] = {mask ? 0.f : t[0] * k, mask ? 0.f : t[1] * k, mask ? 0.f : t[2] * k,
                      r[0] * k, r[1] * k, r[2] * k};
  reinterpret_cast<uint4*>(out)[i] = pack_px<PR>(c, inv_scale);
}

// mel rows [rows][80] f32, chunk_row [B] -> [B][80][16][16 B], chunk[h][w] = rows[r0 + w][h]
template <int PR>
__global__ void prep_mel(const float* __restrict__ rows, const int32_t* __restrict__ chunk_row,
                         uint16_t* __restrict__ out, int B, float inv_scale) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (b, h, w)
  const int64_t total = (int64_t)B * 80 * 16;
  if (i >= total) return;
  const int b = (int)(i / (80 * 16));
  const int hw = (int)(i - (int64_t)b * 80 * 16);
  const int h = hw / 16, w = hw - h * 16;
  const float c[6] = {__ldg(rows + ((int64_t)__ldg(chunk_row + b) + w) * 80 + h), 0.f, 0.f, 0.f, 0.f, 0.f};
  reinterpret_cast<uint4*>(out)[i] = pack_px<PR>(c, inv_scale);
}

// ae0 (1 -> 32 channels, 3x3, 80x16 mel chunk) on CUDA cores: on the tensor
// cores its K is 9 taps x 8 padded channels with ONE real one, so the MMAs and
// im2col loads are ~8x padding (71 us at B = 512 for 0.7 MFLOP/frame).  Same
// arithmetic as the tensor-core path: the quantized input (channel 0 of
// x_mel), the quantized weights (w [32][9] as the packed MMA operand holds
// them), fp32 accumulation, y = acc (* oscale, fp8) + bias, ReLU (* out_inv).
template <int PR>
__global__ void audio_stem(const uint16_t* __restrict__ x, const float* __restrict__ w, const float* __restrict__ bias,
                           const float* __restrict__ oscale, float out_inv, uint16_t* __restrict__ out,
                           int out_pitch, int out_coff, int B) {
  using NF = Num<PR>;
  __shared__ float sw[32 * 9], sb[32], so[32];
  for (int i = threadIdx.x; i < 32 * 9; i += blockDim.x) sw[i] = w[i];
  if (threadIdx.x < 32) {
    sb[threadIdx.x] = bias[threadIdx.x];
    so[threadIdx.x] = NF::Q8 ? oscale[threadIdx.x] : 1.f;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (b, h, w) of the 80 x 16 grid
  if (i >= (int64_t)B * 1280) return;
  const int b = (int)(i / 1280), hw = (int)(i - (int64_t)b * 1280), h = hw >> 4, wc = hw & 15;
  float xv[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int hh = h + t / 3 - 1, ww = wc + t % 3 - 1;
    float v = 0.f;
    if (hh >= 0 && hh < 80 && ww >= 0 && ww < 16) {
      const uint32_t u = __ldg(x + (((int64_t)b * 80 + hh) * 16 + ww) * 8);  // unit 0 of the 16-byte pixel
      if constexpr (NF::Q8) {
        const __half_raw hr = __nv_cvt_fp8_to_halfraw((__nv_fp8_storage_t)(u & 0xffu), __NV_E4M3);
        v = __half2float(*reinterpret_cast<const __half*>(&hr));
      } else {
        v = NF::unpack(u).x;
      }
    }
    xv[t] = v;
  }
  uint16_t* o = out + i * out_pitch + out_coff;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    float f[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int co = half * 16 + j;
      float acc = 0.f;
#pragma unroll
      for (int t = 0; t < 9; ++t) acc = fmaf(xv[t], sw[co * 9 + t], acc);
      float y = fmaxf(acc * so[co] + sb[co], 0.f);
      if constexpr (NF::Q8) y *= out_inv;
      f[j] = y;
    }
    NF::from_float16(f, reinterpret_cast<uint4*>(o) + half * NF::U4);
  }
}

// max |x| over a 16-bit (bf16/fp16) channel-slice view (calibration)
template <int PR>
__global__ void absmax_view(const uint16_t* __restrict__ src, int pitch, int coff, int C, int64_t pixels,
                            unsigned* __restrict__ out) {
  using NF = Num<PR>;
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pixels * C; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t px = i / C;
    const int c = (int)(i - px * C);
    const uint32_t u = __ldg(src + px * pitch + coff + c);
    m = fmaxf(m, fabsf(NF::unpack(u).x));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));  // non-negative floats order as uints
}

}  // namespace gen
}  // namespace lsg

using namespace lsg;
using namespace lsg::gen;

namespace {

struct View {
  uint16_t* p = nullptr;
  int H = 0, W = 0, pitch = 0, coff = 0, C = 0;
};

struct LayerRun {
  int layer;
  int bn;
  int nphases;
  int ntiles;
  bool fused;
  ConvParams p;
  View in_view;
  int GH[MAX_PHASES], GW[MAX_PHASES];  // per phase, per image
  bool halo = false;                   // routed to conv_halo
  bool halo_bres = false;              // weights resident in shared memory
  int halo_mode = 0;                   // HaloMode of a conv_halo layer
  bool pair_ok = false;                // conv_tc layer with a weight map for CTA-pair launches
  bool hp_pair_ok = false;             // halo layer with a weight map (HaloParams::wmap) for CTA pairs
  HaloParams hp;
};

// A/B switches for tuning runs (env LSG_GEN_KNOBS, read once): bit 0 keeps
// the packed tile width, bit 1 disables split-K, bit 5 (32) CTA pairs, bit 6 (64) the macro-pixel stem,
// bit 9 (512) the concurrent audio-encoder branch, bit 10 (1024) halo CTA pairs, bit 11 (2048)
// the 128-channel ConvT (fd5.0) on the halo kernel, bit 13 (8192) ae0 on the tensor cores,
// bit 14 (16384) the stride-2 3x3 convs on the im2col kernel, bit 15 (32768) fe1.0 reading the concat slice,
// bit 16 (65536) out0 on one pixel per GEMM row.
static int gen_knobs() {
  static const int k = [] {
    const char* e = std::getenv("LSG_GEN_KNOBS");
    return e ? std::atoi(e) : 0;
  }();
  return k;
}

// Layers routed to the patch-reuse kernel (conv_halo.cuh); everything else
// goes to the im2col kernel.
HaloMode halo_mode(const LayerSpec& L) {
  // (fd4.1/4.2, 256 channels, as two 128-channel N tiles on CTA pairs measured
  // 1.3% slower end to end than the im2col pair kernel: kept there)
  if (std::string(L.name) == "out0" && L.cout == 32 && L.cin == 80 && !(gen_knobs() & 65536))
    return HALO_CONV3X2;  // the fused output conv on 2-pixel macro columns
  if (L.kind == CONV && L.kh == 3 && L.kw == 3 && L.sh == 1 && L.sw == 1 && L.ph == 1 && L.pw == 1 && L.cout <= 128 &&
      L.cin % 16 == 0)
    return HALO_CONV3;  // 3x3 "same": fe1.x, fe2.x, ae1-5, fd5.x, fd6.x, out0
  if (L.kind == CONV && L.kh == 3 && L.kw == 3 && L.sh == 2 && L.sw == 2 && L.ph == 1 && L.pw == 1 && L.cin % 16 == 0 &&
      L.cin <= 64 && L.cout <= 64 && !(gen_knobs() & 16384))
    return HALO_CONV3S2;  // fe1.0, fe2.0: stride-2 3x3 on parity sub-grids
  if (L.kind != CONV && L.kh == 3 && L.kw == 3 && L.sh == 2 && L.sw == 2 && L.ph == 1 && L.pw == 1 && L.oph == 1 &&
      L.opw == 1 && L.cin % 16 == 0 && (L.cout <= 64 || (L.cout == 128 && !(gen_knobs() & 2048))))
    return HALO_CONVT2;  // fd6.0, fd5.0 (as two 64-channel N tiles): 4 output phases share one accumulator set
  if (L.kind == CONV && L.kh == 7 && L.kw == 7 && L.sh == 1 && L.sw == 1 && L.ph == 3 && L.pw == 3 && L.cin <= 8 &&
      L.cout <= 16)  // fe0 on the 8-channel face tensor: macro-pixels (LSG_GEN_KNOBS bit 64: one pixel per row)
    return (gen_knobs() & 64) ? HALO_STEM7 : HALO_STEM4X;
  return HALO_NONE;
}

// Geometry + tap list of a halo-routed layer (see HaloParams).
struct HaloGeo {
  HaloMode mode = HALO_NONE;
  int oy0 = 0, ox0 = 0, pw = 0, ph = 0, nph = 1, ntaps = 0, tfirst = 0;
  int aoff[MAX_HTAPS] = {}, tphase[MAX_HTAPS] = {}, ky[MAX_HTAPS] = {}, kx[MAX_HTAPS] = {};
  int poy[4] = {}, pox[4] = {};
  int64_t off = -1;  // packed weights
};

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled tiled_fn() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    LSG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) fail(LSG_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiled>(f);
  }
  return fn;
}

// tiled map of an NHWC channel-slice view, box = 8 channels x pw x ph x 1 image
// (ex > 1: every ex-th column, pw of them -- the macro-pixel stem's planes)
void encode_patch(CUtensorMap* map, const View& v, int n, int pw, int ph, int ex = 1, int ey = 1) {
  const cuuint64_t dims[4] = {(cuuint64_t)v.C, (cuuint64_t)v.W, (cuuint64_t)v.H, (cuuint64_t)n};
  const cuuint64_t strides[3] = {(cuuint64_t)v.pitch * 2, (cuuint64_t)v.W * v.pitch * 2,
                                 (cuuint64_t)v.H * v.W * v.pitch * 2};
  const cuuint32_t box[4] = {8, (cuuint32_t)(pw * ex), (cuuint32_t)(ph * ey), 1};
  const cuuint32_t estr[4] = {1, (cuuint32_t)ex, (cuuint32_t)ey, 1};
  CUresult r = tiled_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, v.p + v.coff, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(LSG_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

// tiled map of an NHWC channel-slice view for the staged epilogue: box =
// (bc channels, bx, by, 1) with element strides (1, ex, ey, 1); the swizzle
// matches the box row width (bc * 2 bytes = 128 / 64 / 32).
void encode_box(CUtensorMap* map, const View& v, int n, int bc, int bx, int by, int ex, int ey) {
  const cuuint64_t dims[4] = {(cuuint64_t)v.C, (cuuint64_t)v.W, (cuuint64_t)v.H, (cuuint64_t)n};
  const cuuint64_t strides[3] = {(cuuint64_t)v.pitch * 2, (cuuint64_t)v.W * v.pitch * 2,
                                 (cuuint64_t)v.H * v.W * v.pitch * 2};
  const cuuint32_t box[4] = {(cuuint32_t)bc, (cuuint32_t)bx, (cuuint32_t)by, 1};
  const cuuint32_t estr[4] = {1, (cuuint32_t)ex, (cuuint32_t)ey, 1};
  const CUtensorMapSwizzle sw = bc == 64   ? CU_TENSOR_MAP_SWIZZLE_128B
                                : bc == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : bc == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                           : CU_TENSOR_MAP_SWIZZLE_NONE;
  if (bc != 64 && bc != 32 && bc != 16 && bc != 8) fail(LSG_ERUNTIME, "encode_box: channel box must be 8..64 units");
  CUresult r = tiled_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, v.p + v.coff, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(LSG_ECUDA, "cuTensorMapEncodeTiled (box) failed (" + std::to_string((int)r) + ")");
}

// cuTensorMapEncodeIm2col through the runtime's driver entry point (no
// link-time dependency on libcuda).
using EncodeIm2col = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2col im2col_fn() {
  static EncodeIm2col fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    LSG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) fail(LSG_ECUDA, "cuTensorMapEncodeIm2col unavailable");
    fn = reinterpret_cast<EncodeIm2col>(f);
  }
  return fn;
}

// im2col tensor map of an NHWC channel-slice view: dims (C, W, H, N), strides
// in bytes, bounding box corners (W, H order), 128 pixels x cc channels per load.
void encode_im2col(CUtensorMap* map, const View& v, int n, int cc, int lw, int lh, int uw, int uh, int sx, int sy) {
  const cuuint64_t dims[4] = {(cuuint64_t)v.C, (cuuint64_t)v.W, (cuuint64_t)v.H, (cuuint64_t)n};
  const cuuint64_t strides[3] = {(cuuint64_t)v.pitch * 2, (cuuint64_t)v.W * v.pitch * 2,
                                 (cuuint64_t)v.H * v.W * v.pitch * 2};
  const int lower[2] = {lw, lh}, upper[2] = {uw, uh};
  const cuuint32_t estr[4] = {1, (cuuint32_t)sx, (cuuint32_t)sy, 1};
  const CUtensorMapSwizzle sw = cc == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                         : (cc == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                     : (cc == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE));
  CUresult r = im2col_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, v.p + v.coff, dims, strides, lower, upper,
                           (cuuint32_t)cc, (cuuint32_t)BM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(LSG_ECUDA, "cuTensorMapEncodeIm2col failed (" + std::to_string((int)r) + ")");
}

int pick_bn(int cout) {
  if (cout <= 256) return cout;
  if (cout == 384) return 192;
  return 256;
}

uint16_t f2bf(float f) {  // round to nearest even
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffff) > 0x7f800000) return 0x7fc0;
  u += 0x7fff + ((u >> 16) & 1);
  return (uint16_t)(u >> 16);
}

uint16_t f2h(float f) {  // round to nearest even (host)
  __half h = __float2half_rn(f);
  uint16_t u;
  std::memcpy(&u, &h, 2);
  return u;
}

}  // namespace

struct lsg_gen_s {
  Ctx* ctx = nullptr;
  int max_batch = 0;
  int sm_count = 148;
  int prec = PR_BF16;  // Prec (conv_kernel.cuh): LSG_PREC_BF16 / FP16 / FP8, or PR_I8 (an INT8 tail's engine)
  int cpu = 1;         // channels per 16-bit storage unit (2 for the 8-bit formats)
  float inv_face = 1.f, inv_mel = 1.f;  // fp8 input quantisation (1 / scale)
  DevBuf<uint16_t> wpack;
  DevBuf<float> bias;
  DevBuf<float> oscale;  // 8-bit: per layer, per output channel s_in * s_w[co]
  std::vector<int> plan_in_id, plan_out_id;  // tensor ids (kTensors) of each layer's input / output
  std::vector<float> ascale;                 // 8-bit: scale per tensor id (1 otherwise)
  DevBuf<float> w1b1;
  DevBuf<uint16_t> act;  // all activation buffers
  DevBuf<float> splitk_ws;   // split-K partial slots (conv_kernel.cuh ConvParams::ws)
  int splitk_tiles = 0;      // tiles the workspace holds
  // the audio encoder runs on a side stream, concurrently with the face
  // encoder (disjoint buffers: x_mel/A0/A1 vs x_face/S0/S1/cat), joined
  // before the decoder; its split-K layers use their own workspace
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  DevBuf<float> splitk_ws2;
  DevBuf<float> ae0w;  // ae0 weights [32][9] as quantized for the MMA (audio_stem)
  ~lsg_gen_s() {
    for (auto& g : fwd_graphs) {
      if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
      if (g.second.graph) cudaGraphDestroy(g.second.graph);
    }
    if (cap) cudaStreamDestroy(cap);
    delete head;
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
  }
  View x_face, x_mel, cat[7], S0, S1, A0, A1;
  View X16;  // dense copy of fe0's output (fe1.0's input; cat[6] keeps the concat copy)
  std::vector<LayerRun> plan;
  // The forward at B = max_batch as a CUDA graph (one cudaGraphLaunch instead
  // of ~55 launches; the round-1 tools/graph_test.py measured -40 us), one per
  // (output mode, gathered targets); the three kernels that take caller
  // pointers -- input prep and the fused output conv -- are re-pointed per
  // call (cudaGraphExecKernelNodeSetParams).
  struct FwdGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t n_face = nullptr, n_mel = nullptr, n_out = nullptr;
    int kernels = 0;
  };
  std::map<std::tuple<int, int, int>, FwdGraph> fwd_graphs;
  cudaStream_t cap = nullptr;  // capture stream (the caller's may be the legacy stream, which cannot capture)
  // LSG_PREC_FP8_TAIL / _INT8_TAIL: this 8-bit engine runs plan layers
  // [tail0, end), which start decoder block tail_blk; the 16-bit engine
  // `head` runs [0, tail0) and the tensors the tail reads from it (the
  // block's input cat[tail_blk - 1] whole, the encoder slices of
  // cat[tail_blk..6]) are requantised into this engine's buffers in between
  lsg_gen_s* head = nullptr;
  int tail0 = 0, tail_blk = 0;
};

static int64_t layer_params(const LayerSpec& L) { return (int64_t)L.cin * L.cout * L.kh * L.kw + L.cout; }

// Every layer kernel is launched with programmatic stream serialization so its
// prologue overlaps the previous layer's tail (tc.cuh griddep_*).
template <typename P>
static void launch_pdl(void (*kernel)(P), int grid, int block, int smem, cudaStream_t st, const P& p) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  LSG_CUDA(cudaLaunchKernelEx(&cfg, kernel, p));
}

// Persistent launch: one CTA per SM walks the tiles round-robin in the
// L2-friendly order of decode_tile().
// Split-K factor of a conv_tc layer: grid-starved layers (fewer than half an
// SM wave of tiles: the low-resolution encoder / decoder blocks) split their K
// loop so about one wave of CTAs runs, each split keeping >= 2 kblocks.
static int splitk_factor(const ConvParams& p, int nphases, int tiles, int bn, bool fused, int sms, int ws_tiles) {
  if (fused || bn < 32 || tiles * 2 > sms || tiles > ws_tiles || (gen_knobs() & 2)) return 1;
  int kbmin = 1 << 30, kbmax = 0;
  for (int z = 0; z < nphases; ++z) {
    kbmin = std::min(kbmin, p.ph[z].kblocks);
    kbmax = std::max(kbmax, p.ph[z].kblocks);
  }
  // a split costs ~5 us (partial store, meeting, reduce): only mainloops of
  // >= ~6 us (4 MMAs per kblock at the SS-mode rate, ~1.9 GHz) are split
  const double mma_cyc = std::max(bn / 2.0, (128.0 + bn) / 4.0);
  const double main_us = kbmax * 4 * mma_cyc / 1900.0;
  const int kn = gen_knobs();
  if (main_us < ((kn & 4) ? 3.0 : (kn & 16) ? 10.0 : 6.0)) return 1;
  // <= 8: the splits of a tile form one (portable-size) cluster
  const int s = std::min({sms / tiles, (kn & 8) ? kbmin / 2 : kbmin / 4, 8});
  return s >= 2 ? s : 1;
}

// Tiles of a conv_tc layer at batch B and tile width bn.
static int conv_tiles(const LayerRun& r, int B, int bn) {
  int tiles = 0;
  for (int z = 0; z < r.nphases; ++z) tiles += (int)ceil_div((int64_t)B * r.GH[z] * r.GW[z], BM) * (r.ntiles * r.bn / bn);
  return tiles;
}

// Launch tile width: the packed width, halved (to slices of the packed tiles)
// while the layer fills less than half an SM wave and stays within one --
// grid-starved low-resolution layers get more CTAs, each streaming fewer bytes.
static int conv_launch_bn(const LayerRun& r, int B, int sms, int ws_tiles) {
  int bn = r.bn;
  if (r.fused || (gen_knobs() & 1)) return bn;
  // a long mainloop is better split along K at full width (narrow tiles
  // re-stream the A tile once per extra column tile)
  if (splitk_factor(r.p, r.nphases, conv_tiles(r, B, bn), bn, false, sms, ws_tiles) > 1) return bn;
  while (bn > 64 && r.bn % (bn / 2) == 0 && (bn / 2) % 64 == 0 && conv_tiles(r, B, bn) * 2 <= sms &&
         conv_tiles(r, B, bn / 2) <= sms)
    bn /= 2;
  return bn;
}

template <int BN, int CC, bool F, int PR>
static void launch_conv(const LayerRun& r, int B, int sms, cudaStream_t st, float* ws, int ws_tiles) {
  ConvParams p = r.p;
  const int ntiles = r.ntiles * r.bn / BN;
  int tiles = 0;
  for (int z = 0; z < r.nphases; ++z) {
    Phase& P = p.ph[z];
    P.M = B * r.GH[z] * r.GW[z];
    P.mtiles = (int)ceil_div(P.M, BM);
    P.tile0 = tiles;
    tiles += P.mtiles * ntiles;
  }
  p.pbn = r.bn;
  p.nphases = r.nphases;
  p.ntiles_n = ntiles;
  p.total_tiles = tiles;
  p.interleave = 1;
  for (int z = 1; z < r.nphases; ++z) p.interleave &= p.ph[z].mtiles == p.ph[0].mtiles;
  p.ksplit = splitk_factor(p, r.nphases, tiles, BN, F, sms, ws ? ws_tiles : 0);
  p.total_units = tiles * p.ksplit;
  p.ws = ws;
  if (p.ksplit == 1) {
    launch_pdl(conv_tc<BN, CC, F, PR>, std::min(p.total_units, sms), NUM_THREADS, Cfg<BN>::SMEM, st, p);
    return;
  }
  // split-K: the ksplit CTAs of a tile are one cluster (co-scheduled by the
  // hardware, so their meeting in splitk_tile cannot wait on a CTA that is
  // not resident); grid = tiles * ksplit <= SMs
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)p.total_units);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = (size_t)Cfg<BN>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)p.ksplit;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  LSG_CUDA(cudaLaunchKernelEx(&cfg, conv_tc<BN, CC, F, PR>, p));
}

// CTA-pair launch (conv_pair.cuh): tiles are pairs of m-tiles, one cluster of
// two CTAs per pair, grid = an even number of SMs.
template <int BN, int CC, int PR>
static void launch_pair(const LayerRun& r, int B, int sms, cudaStream_t st) {
  ConvParams p = r.p;
  const int ntiles = r.ntiles * r.bn / BN;
  int tiles = 0;
  for (int z = 0; z < r.nphases; ++z) {
    Phase& P = p.ph[z];
    P.M = B * r.GH[z] * r.GW[z];
    P.mtiles = (int)ceil_div(ceil_div(P.M, BM), 2);
    P.tile0 = tiles;
    tiles += P.mtiles * ntiles;
  }
  p.pbn = r.bn;
  p.nphases = r.nphases;
  p.ntiles_n = ntiles;
  p.total_tiles = tiles;
  p.interleave = 1;
  for (int z = 1; z < r.nphases; ++z) p.interleave &= p.ph[z].mtiles == p.ph[0].mtiles;
  p.ksplit = 1;
  p.total_units = tiles;
  p.ws = nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)std::min(2 * tiles, sms & ~1));
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = (size_t)Cfg2<BN>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  LSG_CUDA(cudaLaunchKernelEx(&cfg, conv_tc2<BN, CC, PR>, p));
}

// (tile width, channel chunk) combinations of the pair kernel
#define LSG_PAIR_VARIANTS(X) \
  X(128, 64)                 \
  X(192, 64)                 \
  X(256, 64)                 \
  X(128, 32)                 \
  X(192, 32)                 \
  X(256, 32)

// (tile width BN, channel chunk CC in 16-bit units, fused output)
// combinations the Wav2Lip layers use; every combination is compiled for
// bf16, fp16 and fp8 (fp8 halves the units per channel, hence CC 8/16/32 with
// the wider tiles).
#define LSG_CONV_VARIANTS(X) \
  X(16, 8, false)            \
  X(32, 8, false)            \
  X(32, 16, false)           \
  X(32, 32, false)           \
  X(64, 32, false)           \
  X(64, 64, false)           \
  X(128, 64, false)          \
  X(192, 64, false)          \
  X(256, 64, false)          \
  X(32, 16, true)            \
  X(64, 16, false)           \
  X(128, 32, false)          \
  X(192, 32, false)          \
  X(256, 32, false)          \
  X(32, 8, true)

// halo kernel variants: (tile width, mode, fused output, weights resident)
#define LSG_HALO_VARIANTS(X)             \
  X(16, HALO_STEM7, false, true)         \
  X(16, HALO_STEM4X, false, true)        \
  X(32, HALO_CONV3S2, false, true)        \
  X(64, HALO_CONV3S2, false, true)        \
  X(32, HALO_CONV3, false, true)         \
  X(64, HALO_CONV3, false, true)         \
  X(128, HALO_CONV3, false, false)       \
  X(64, HALO_CONVT2, false, false)       \
  X(32, HALO_CONV3, true, true)          \
  X(32, HALO_CONV3X2, true, true)

// halo variants that also run as CTA pairs (cta_group::2; HaloCfg PAIR).
// Measured per layer (B = 512): the streamed-weight 3x3 at N = 128 (fd5.1/5.2,
// 288 KB of weights per 128-position tile) gains 18% from halving each SM's
// weight stream; resident-weight layers (fe1/fe2/ae/fd6.1-2, N <= 64) and the
// streamed ConvT fd6.0 lose 15-35% (and fd5.0's N-tiled ConvT, despite twice
// the weight stream, about as much as fd5.1/5.2 gain), the fused output layer
// is neutral.
#define LSG_HALO_PAIR_VARIANTS(X) X(128, HALO_CONV3, false, false)

// The host-built tap list of a halo layer must be the kernel's compile-time
// table (conv_halo.cuh HaloTaps): packing order == issue order.
template <int MODE>
bool taps_match(const HaloGeo& g) {
  using TT = HaloTaps<MODE>;
  if (g.ntaps != TT::NT || g.nph != TT::NPH || g.pw != TT::PW || g.ph != TT::PH) return false;
  for (int t = 0; t < TT::NT; ++t)
    if (g.aoff[t] != TT::aoff(t) || g.tphase[t] != TT::phase(t)) return false;
  return true;
}

template <int PR>
static void set_smem_attrs_t() {
#define LSG_SET_ATTR(BN, CC, F)                                                                                   \
  LSG_CUDA(cudaFuncSetAttribute(conv_tc<BN, CC, F, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
  LSG_CONV_VARIANTS(LSG_SET_ATTR)
#undef LSG_SET_ATTR
#define LSG_SET_HALO_ATTR(BN, MD, F, R)                                                                           \
  LSG_CUDA(cudaFuncSetAttribute(conv_halo<BN, MD, F, PR, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                HaloCfg<BN, MD, F, R, Num<PR>::Q8 ? 1 : 2>::SMEM));
  LSG_HALO_VARIANTS(LSG_SET_HALO_ATTR)
#undef LSG_SET_HALO_ATTR
#define LSG_SET_HALO_PAIR_ATTR(BN, MD, F, R)                                                                      \
  LSG_CUDA(cudaFuncSetAttribute(conv_halo<BN, MD, F, PR, R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                HaloCfg<BN, MD, F, R, Num<PR>::Q8 ? 1 : 2, true>::SMEM));
  LSG_HALO_PAIR_VARIANTS(LSG_SET_HALO_PAIR_ATTR)
#undef LSG_SET_HALO_PAIR_ATTR
#define LSG_SET_PAIR_ATTR(BN, CC) \
  LSG_CUDA(cudaFuncSetAttribute(conv_tc2<BN, CC, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2<BN>::SMEM));
  LSG_PAIR_VARIANTS(LSG_SET_PAIR_ATTR)
#undef LSG_SET_PAIR_ATTR
}
static void set_smem_attrs(int prec) {
  if (prec == PR_I8) set_smem_attrs_t<PR_I8>();
  else if (prec == PR_FP8) set_smem_attrs_t<PR_FP8>();
  else if (prec == PR_FP16) set_smem_attrs_t<PR_FP16>();
  else set_smem_attrs_t<PR_BF16>();
}

template <int BN, int MD, bool F, int PR, bool R>
static void launch_halo(const LayerRun& r, int B, int sms, cudaStream_t st) {
  HaloParams hp = r.hp;
  hp.B = B;
  hp.total_tiles = B * hp.tiles_per_img * hp.ntn;
  const int grid = std::min(hp.total_tiles, sms);
  launch_pdl(conv_halo<BN, MD, F, PR, R>, grid, NUM_THREADS, HaloCfg<BN, MD, F, R, Num<PR>::Q8 ? 1 : 2>::SMEM, st,
             hp);
}

// CTA-pair halo launch: clusters of two adjacent tiles (the tile count is even)
template <int BN, int MD, bool F, int PR, bool R>
static void launch_halo_pair(const LayerRun& r, int B, int sms, cudaStream_t st) {
  HaloParams hp = r.hp;
  hp.B = B;
  hp.total_tiles = B * hp.tiles_per_img * hp.ntn;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)std::min(hp.total_tiles, sms & ~1));
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = (size_t)HaloCfg<BN, MD, F, R, Num<PR>::Q8 ? 1 : 2, true>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  LSG_CUDA(cudaLaunchKernelEx(&cfg, conv_halo<BN, MD, F, PR, R, true>, hp));
}

// Kernel route of a plan layer at batch B: decided here ONCE, used by the
// launch and reported by lsgdbg_gen_routes (tests assert which kernel paths
// a benchmarked batch size exercises).
enum Route : int { RT_HALO = 1, RT_HALO_PAIR = 2, RT_CONV = 3, RT_CONV_SPLITK = 4, RT_CONV_NARROW = 5,
                   RT_PAIR = 6, RT_STEM = 7 };
struct RouteInfo {
  int route, bn, ksplit;
};
static bool has_halo_pair_variant(const LayerRun& r) {
#define LSG_HAS_HP(BN, MD, F, R) \
  if (r.bn == BN && r.halo_mode == MD && r.fused == F && r.halo_bres == R) return true;
  LSG_HALO_PAIR_VARIANTS(LSG_HAS_HP)
#undef LSG_HAS_HP
  return false;
}
static bool has_pair_variant(const LayerRun& r) {
#define LSG_HAS_P(BN, CC) \
  if (r.bn == BN && r.p.cc == CC) return true;
  LSG_PAIR_VARIANTS(LSG_HAS_P)
#undef LSG_HAS_P
  return false;
}
static RouteInfo route_of(const LayerRun& r, int B, int sms, int ws_tiles) {
  if (r.halo) {
    const bool pair = !(gen_knobs() & 1024) && r.hp_pair_ok && (B * r.hp.tiles_per_img) % 2 == 0 &&
                      B * r.hp.tiles_per_img >= sms && has_halo_pair_variant(r);
    return {pair ? RT_HALO_PAIR : RT_HALO, r.bn, 1};
  }
  const int lbn = conv_launch_bn(r, B, sms, ws_tiles);
  const int ks = splitk_factor(r.p, r.nphases, conv_tiles(r, B, lbn), lbn, r.fused, sms, ws_tiles);
  // wide layers with at least a full wave of tiles: CTA pairs
  if (r.pair_ok && lbn == r.bn && !(gen_knobs() & 32) && conv_tiles(r, B, r.bn) >= sms && ks == 1 &&
      has_pair_variant(r))
    return {RT_PAIR, r.bn, 1};
  return {ks > 1 ? RT_CONV_SPLITK : (lbn < r.bn ? RT_CONV_NARROW : RT_CONV), lbn, ks};
}

template <int PR>
static void dispatch_t(const LayerRun& r, int B, int sms, cudaStream_t st, float* ws, int ws_tiles) {
  const RouteInfo ri = route_of(r, B, sms, ws ? ws_tiles : 0);
  if (ri.route == RT_HALO_PAIR) {
#define LSG_HALO_PAIR_DISPATCH(BN, MD, F, R)                                                  \
  if (r.bn == BN && r.halo_mode == MD && r.fused == F && r.halo_bres == R)                    \
    return launch_halo_pair<BN, MD, F, PR, R>(r, B, sms, st);
    LSG_HALO_PAIR_VARIANTS(LSG_HALO_PAIR_DISPATCH)
#undef LSG_HALO_PAIR_DISPATCH
  }
  if (ri.route == RT_HALO || ri.route == RT_HALO_PAIR) {
#define LSG_HALO_DISPATCH(BN, MD, F, R)                                                       \
  if (r.bn == BN && r.halo_mode == MD && r.fused == F && r.halo_bres == R)                    \
    return launch_halo<BN, MD, F, PR, R>(r, B, sms, st);
    LSG_HALO_VARIANTS(LSG_HALO_DISPATCH)
#undef LSG_HALO_DISPATCH
    fail(LSG_ERUNTIME, "generator: no halo kernel for tile width " + std::to_string(r.bn) + " / mode " +
                           std::to_string(r.halo_mode) + (r.halo_bres ? " / resident weights" : " / streamed weights"));
  }
  if (ri.route == RT_PAIR) {
#define LSG_PAIR_DISPATCH(BN, CC) \
  if (r.bn == BN && r.p.cc == CC) return launch_pair<BN, CC, PR>(r, B, sms, st);
    LSG_PAIR_VARIANTS(LSG_PAIR_DISPATCH)
#undef LSG_PAIR_DISPATCH
  }
  const int lbn = ri.bn;
#define LSG_DISPATCH(BN, CC, F) \
  if (lbn == BN && r.p.cc == CC && r.fused == F) return launch_conv<BN, CC, F, PR>(r, B, sms, st, ws, ws_tiles);
  LSG_CONV_VARIANTS(LSG_DISPATCH)
#undef LSG_DISPATCH
  fail(LSG_ERUNTIME, "generator: no conv kernel for tile width " + std::to_string(r.bn) + " / channel chunk " +
                         std::to_string(r.p.cc));
}

static void dispatch(const lsg_gen_s* h, const LayerRun& r, int B, cudaStream_t st, int wset = 0) {
  float* ws = wset ? h->splitk_ws2.p : h->splitk_ws.p;
  const int wt = h->splitk_tiles;
  if (h->prec == PR_I8) dispatch_t<PR_I8>(r, B, h->sm_count, st, ws, wt);
  else if (h->prec == PR_FP8) dispatch_t<PR_FP8>(r, B, h->sm_count, st, ws, wt);
  else if (h->prec == PR_FP16) dispatch_t<PR_FP16>(r, B, h->sm_count, st, ws, wt);
  else dispatch_t<PR_BF16>(r, B, h->sm_count, st, ws, wt);
}

// Activation tensors for fp8 scales: 0 face input, 1 mel input, 2..8 the
// concat buffers cat0..cat6 (both producers share the scale), 9 + l the
// output of layer l when it is not a concat slice.
constexpr int kTensors = 9 + kNumLayers;

extern "C" {

lsg_status lsg_lipsync_validate(int64_t audio_span_ms, int64_t frame_span_ms, int64_t n_frames) {
  return guard(__func__, [&] {  // visual_mocks.cpp:43-46
    if (n_frames < 2) invalid("lipsync: need at least 2 frames");
    if (std::llabs(audio_span_ms - frame_span_ms) > 150) invalid("lipsync: audio and frame spans diverge");
  });
}

lsg_status lsg_gen_param_count(int64_t* n) {
  return guard(__func__, [&] {
    int64_t t = 0;
    for (const auto& L : kLayers) t += layer_params(L);
    *n = t;
  });
}

lsg_status lsg_gen_layer_info(int32_t* info, int32_t cap, int32_t* n_layers) {
  return guard(__func__, [&] {
    *n_layers = kNumLayers;
    for (int i = 0; i < kNumLayers && i < cap; ++i) {
      const auto& L = kLayers[i];
      const int32_t v[12] = {L.kind, L.cin, L.cout, L.kh, L.kw, L.sh, L.sw, L.ph, L.pw, L.oph, L.opw, L.res};
      std::memcpy(info + 12 * i, v, sizeof(v));
    }
  });
}

lsg_status lsg_gen_create_q(lsg_ctx ctx, const float* weights, int64_t n_floats, int32_t precision,
                            const float* act_absmax, int32_t n_act, int32_t max_batch, lsg_gen* out) {
  return guard(__func__, [&] {
    *out = nullptr;
    int64_t want = 0;
    lsg_gen_param_count(&want);
    if (n_floats != want) invalid("lsg_gen_create: weight blob has " + std::to_string(n_floats) + " floats, expected " +
                                  std::to_string(want));
    if (precision != LSG_PREC_BF16 && precision != LSG_PREC_FP16 && precision != LSG_PREC_FP8 &&
        precision != LSG_PREC_FP8_TAIL && precision != LSG_PREC_INT8_TAIL)
      invalid("lsg_gen_create: unsupported precision");
    const bool tail = precision == LSG_PREC_FP8_TAIL || precision == LSG_PREC_INT8_TAIL;
    if ((precision == LSG_PREC_FP8 || tail) && (!act_absmax || n_act != kTensors))
      invalid("lsg_gen_create: 8-bit precisions need the calibrated activation ranges (lsg_gen_calibrate)");
    if (max_batch <= 0 || max_batch > 4096) invalid("lsg_gen_create: max_batch out of range");
    DeviceGuard g(ctx);
    auto h = new lsg_gen_s();
    try {
      h->ctx = ctx;
      h->max_batch = max_batch;
      h->prec = precision == LSG_PREC_INT8_TAIL                                 ? PR_I8
                : (precision == LSG_PREC_FP8 || precision == LSG_PREC_FP8_TAIL) ? PR_FP8
                : (precision == LSG_PREC_FP16 ? PR_FP16 : PR_BF16);
      const bool f8 = h->prec == PR_FP8 || h->prec == PR_I8;  // 8-bit storage (e4m3, or u8 / s8)
      const bool i8 = h->prec == PR_I8;
      const int cpu = h->cpu = f8 ? 2 : 1;
      h->sm_count = ctx->sm_count;
      const int B = max_batch;
      // 8-bit activation scales: calibrated |x| max with 10% headroom onto e4m3's
      // 448; u8 spans [0, max] exactly (saturating; tools/int8_sweep.py: headroom
      // costs u8 0.4 dB and buys nothing)
      std::vector<float> ascale(kTensors, 1.f);
      if (f8)
        for (int i = 0; i < kTensors; ++i)
          ascale[i] = i8 ? std::max(act_absmax[i], 1e-6f) / 255.f : std::max(act_absmax[i], 1e-6f) * 1.1f / 448.f;
      h->inv_face = 1.f / ascale[0];
      h->inv_mel = 1.f / ascale[1];
      h->ascale = ascale;
      // ---------------- activation buffers (NHWC, 16-bit units: bf16/fp16, or fp8 pairs)
      struct Req { View* v; int H, W, C; };
      const int cat_hw[7] = {1, 3, 6, 12, 24, 48, 96};
      const int cat_c[7] = {1024, 1024, 768, 512, 320, 160, 80};
      std::vector<Req> reqs;
      reqs.push_back({&h->x_face, 96, 96, 8});  // 16 bytes per pixel in every format
      reqs.push_back({&h->x_mel, 80, 16, 8});
      for (int l = 0; l < 7; ++l) reqs.push_back({&h->cat[l], cat_hw[l], cat_hw[l], cat_c[l] / cpu});
      reqs.push_back({&h->X16, 96, 96, 16 / cpu});
      reqs.push_back({&h->S0, 96, 96, 64 / cpu});
      reqs.push_back({&h->S1, 96, 96, 64 / cpu});
      reqs.push_back({&h->A0, 80, 16, 32 / cpu});
      reqs.push_back({&h->A1, 80, 16, 32 / cpu});
      size_t tot = 0;
      for (auto& r : reqs) tot += ((size_t)B * r.H * r.W * r.C + 127) & ~size_t(127);
      h->act.alloc(tot);
      LSG_CUDA(cudaMemset(h->act.p, 0, h->act.bytes()));
      // split-K workspace: one 128 x 256 fp32 slot per work unit (units <= SMs,
      // tiles <= SMs / 2)
      h->splitk_tiles = h->sm_count / 2;
      h->splitk_ws.alloc((size_t)h->sm_count * BM * 256);
      h->splitk_ws2.alloc((size_t)h->sm_count * BM * 256);
      LSG_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
      LSG_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
      LSG_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
      size_t off = 0;
      for (auto& r : reqs) {
        *r.v = View{h->act.p + off, r.H, r.W, r.C, 0, r.C};
        off += ((size_t)B * r.H * r.W * r.C + 127) & ~size_t(127);
      }
      // K-block element j of row r (a row = 128 bytes = 64 units): 16-bit
      // value, or fp8 byte (value / s_w[row's channel]); 16-byte chunks
      // 128B-swizzled as the UMMA K-major SW128 layout expects
      const int KE = 64 * cpu;  // elements per K block
      auto store = [&](uint16_t* blk, int r, int j, float v, float sw) {
        if (f8) {  // s8: round(v / s_w) half-even, as torch.round(w / s) in the tests' models
          uint8_t* b8 = reinterpret_cast<uint8_t*>(blk);
          b8[r * 128 + (((j >> 4) ^ (r & 7)) << 4) + (j & 15)] =
              i8 ? (uint8_t)(int8_t)std::nearbyint(std::min(127.f, std::max(-127.f, v / sw)))
                 : (uint8_t)__nv_cvt_float_to_fp8(v * (1.f / sw), __NV_SATFINITE, __NV_E4M3);
        } else {
          blk[r * BK + (((j >> 3) ^ (r & 7)) << 3) + (j & 7)] = h->prec == PR_FP16 ? f2h(v) : f2bf(v);
        }
      };
      std::vector<std::vector<float>> wscale(kNumLayers);  // 8-bit: per output channel max|w| / 448 (e4m3), / 127 (s8)
      // ---------------- weights: pack per layer / phase / N tile / K block
      std::vector<uint16_t> pack;
      std::vector<float> bias;
      std::vector<float> w1b1(3 * 32 + 3);
      std::vector<int64_t> pack_off(kNumLayers * MAX_PHASES, 0);
      std::vector<int64_t> bias_off(kNumLayers, 0);
      std::vector<HaloGeo> hgeo(kNumLayers);  // conv_halo routing, taps and packing
      struct PhaseGeo { int ntaps; signed char dy[MAX_TAPS], dx[MAX_TAPS]; int ky[MAX_TAPS], kx[MAX_TAPS]; int oy, ox; };
      std::vector<std::vector<PhaseGeo>> geo(kNumLayers);
      const float* wp = weights;
      for (int li = 0; li < kNumLayers; ++li) {
        const LayerSpec& L = kLayers[li];
        const float* w = wp;
        const float* b = wp + (int64_t)L.cin * L.cout * L.kh * L.kw;
        wp = b + L.cout;
        if (li == kNumLayers - 1) {  // out1: fused into out0's epilogue
          for (int o = 0; o < 3; ++o)
            for (int c = 0; c < 32; ++c) w1b1[o * 32 + c] = w[o * 32 + c];
          for (int o = 0; o < 3; ++o) w1b1[96 + o] = b[o];
          continue;
        }
        bias_off[li] = (int64_t)bias.size();
        bias.insert(bias.end(), b, b + L.cout);
        auto wat = [&](int co, int ci, int ky, int kx) {  // conv [co][ci][ky][kx], convT [ci][co][ky][kx]
          return L.kind == CONV ? w[(((int64_t)co * L.cin + ci) * L.kh + ky) * L.kw + kx]
                                : w[(((int64_t)ci * L.cout + co) * L.kh + ky) * L.kw + kx];
        };
        std::vector<float>& sw = wscale[li];
        sw.assign(L.cout, 1.f);
        if (f8)
          for (int co = 0; co < L.cout; ++co) {
            float m = 0.f;
            for (int ci = 0; ci < L.cin; ++ci)
              for (int ky = 0; ky < L.kh; ++ky)
                for (int kx = 0; kx < L.kw; ++kx) m = std::max(m, std::fabs(wat(co, ci, ky, kx)));
            sw[co] = m > 0.f ? m / (i8 ? 127.f : 448.f) : 1.f;
          }
        if (std::string(L.name) == "ae0") {  // audio_stem's copy of the quantized operand
          if (li != kAe0 || L.cin != 1 || L.cout != 32 || L.kh != 3 || L.kw != 3 || L.sh != 1 || L.ph != 1)
            fail(LSG_ERUNTIME, "generator: ae0 shape / position");
          std::vector<float> q(32 * 9);
          for (int co = 0; co < 32; ++co)
            for (int t = 0; t < 9; ++t) {
              const float v = wat(co, 0, t / 3, t % 3);
              if (i8) {
                q[co * 9 + t] = (float)std::nearbyint(std::min(127.f, std::max(-127.f, v / sw[co])));
              } else if (f8) {
                const __nv_fp8_storage_t e = __nv_cvt_float_to_fp8(v / sw[co], __NV_SATFINITE, __NV_E4M3);
                const __half_raw hr = __nv_cvt_fp8_to_halfraw(e, __NV_E4M3);
                q[co * 9 + t] = __half2float(__half(hr));
              } else if (h->prec == PR_FP16) {
                const uint16_t bits = f2h(v);
                __half_raw hr;
                hr.x = bits;
                q[co * 9 + t] = __half2float(__half(hr));
              } else {
                const uint32_t u = (uint32_t)f2bf(v) << 16;
                float f;
                std::memcpy(&f, &u, 4);
                q[co * 9 + t] = f;
              }
            }
          h->ae0w.alloc(q.size());
          LSG_CUDA(cudaMemcpy(h->ae0w.p, q.data(), q.size() * 4, cudaMemcpyHostToDevice));
        }
        // phases
        std::vector<PhaseGeo>& G = geo[li];
        if (L.kind == CONV) {
          PhaseGeo pg{};
          pg.ntaps = 0;
          for (int ky = 0; ky < L.kh; ++ky)
            for (int kx = 0; kx < L.kw; ++kx) {
              pg.dy[pg.ntaps] = (signed char)(ky - L.ph);
              pg.dx[pg.ntaps] = (signed char)(kx - L.pw);
              pg.ky[pg.ntaps] = ky;
              pg.kx[pg.ntaps] = kx;
              ++pg.ntaps;
            }
          pg.oy = pg.ox = 0;
          G.push_back(pg);
        } else if (L.sh == 1 && L.sw == 1 && L.ph == 0 && L.pw == 0) {
          // fd1.0: stride-1 convT of a 1x1 map -- output pixel (a, b) is
          // exactly tap (a, b) of the single input pixel: kh*kw one-tap
          // phases, no zero taps (the plan asserts the 1x1 input)
          for (int a = 0; a < L.kh; ++a)
            for (int bb = 0; bb < L.kw; ++bb) {
              PhaseGeo pg{};
              pg.ntaps = 1;
              pg.dy[0] = pg.dx[0] = 0;
              pg.ky[0] = a;
              pg.kx[0] = bb;
              pg.oy = a;
              pg.ox = bb;
              G.push_back(pg);
            }
        } else {
          // out[o] = sum_{i,k: o = i*s - p + k} in[i] w[k]; phase a of o = g*s + a
          for (int a = 0; a < L.sh; ++a)
            for (int bb = 0; bb < L.sw; ++bb) {
              PhaseGeo pg{};
              pg.ntaps = 0;
              for (int ky = 0; ky < L.kh; ++ky) {
                if (((a + L.ph - ky) % L.sh + L.sh) % L.sh) continue;
                for (int kx = 0; kx < L.kw; ++kx) {
                  if (((bb + L.pw - kx) % L.sw + L.sw) % L.sw) continue;
                  pg.dy[pg.ntaps] = (signed char)((a + L.ph - ky) / L.sh);
                  pg.dx[pg.ntaps] = (signed char)((bb + L.pw - kx) / L.sw);
                  pg.ky[pg.ntaps] = ky;
                  pg.kx[pg.ntaps] = kx;
                  ++pg.ntaps;
                }
              }
              pg.oy = a;
              pg.ox = bb;
              G.push_back(pg);
            }
        }
        if (const HaloMode hm = halo_mode(L); hm != HALO_NONE) {
          HaloGeo& hg = hgeo[li];
          hg.mode = hm;
          auto add_tap = [&](int aoff, int z, int ky, int kx) {
            if (hg.ntaps == MAX_HTAPS) fail(LSG_ERUNTIME, std::string("generator: halo tap list overflow at ") + L.name);
            bool first = true;
            for (int t = 0; t < hg.ntaps; ++t) first &= hg.tphase[t] != z;
            if (first) hg.tfirst |= 1 << hg.ntaps;
            hg.aoff[hg.ntaps] = aoff;
            hg.tphase[hg.ntaps] = z;
            hg.ky[hg.ntaps] = ky;
            hg.kx[hg.ntaps] = kx;
            ++hg.ntaps;
          };
          if (hm == HALO_CONV3) {  // patch = tile + 1-pixel halo, taps = (ky, kx)
            hg.oy0 = hg.ox0 = -1;
            hg.pw = HTW + 2;
            hg.ph = HTH + 2;
            for (int ky = 0; ky < 3; ++ky)
              for (int kx = 0; kx < 3; ++kx) add_tap(ky * hg.pw + kx, 0, ky, kx);
          } else if (hm == HALO_CONVT2) {  // grid = input positions, patch = tile + 1 (bottom/right)
            hg.pw = HTW + 1;
            hg.ph = HTH + 1;
            hg.nph = (int)G.size();
            if (hg.nph != 4) fail(LSG_ERUNTIME, std::string("generator: ConvT phase count at ") + L.name);
            for (int z = 0; z < hg.nph; ++z) {
              hg.poy[z] = G[z].oy;
              hg.pox[z] = G[z].ox;
              for (int t = 0; t < G[z].ntaps; ++t) {
                if (G[z].dy[t] < 0 || G[z].dy[t] > 1 || G[z].dx[t] < 0 || G[z].dx[t] > 1)
                  fail(LSG_ERUNTIME, std::string("generator: ConvT tap outside patch at ") + L.name);
                add_tap(G[z].dy[t] * hg.pw + G[z].dx[t], z, G[z].ky[t], G[z].kx[t]);
              }
            }
          } else if (hm == HALO_CONV3X2) {  // x-parity planes, 12 taps (ky, d = z + kx)
            hg.pw = HTW + 1;
            hg.ph = HTH + 2;
            hg.nph = 2;
            hg.pox[1] = 1;
            const int pl16 = ((hg.pw * hg.ph * 16 + 127) / 128 * 128) / 16;
            for (int ky = 0; ky < 3; ++ky)
              for (int d = 0; d < 4; ++d) add_tap((d & 1) * 4 * pl16 + ky * hg.pw + (d >> 1), 0, ky, d);
          } else if (hm == HALO_CONV3S2) {  // parity sub-grid patch (tile + 1), taps at parity base + (k != 0)
            hg.pw = HTW + 1;
            hg.ph = HTH + 1;
            const int pl16 = ((hg.pw * hg.ph * 16 + 127) / 128 * 128) / 16;
            for (int ky = 0; ky < 3; ++ky)
              for (int kx = 0; kx < 3; ++kx)
                add_tap(((ky == 1 ? 0 : 2) + (kx == 1 ? 0 : 1)) * 2 * pl16 + (ky != 0) * hg.pw + (kx != 0), 0, ky, kx);
          } else {  // stem: planes = x shifts, taps = the 7 kernel rows
            hg.oy0 = hg.ox0 = -3;
            hg.pw = HTW;
            hg.ph = HTH + 6;
            if (hm == HALO_STEM4X) {  // 4-pixel macro columns: pixel offset z is output phase z
              hg.nph = 4;
              for (int z = 0; z < 4; ++z) hg.pox[z] = z;
            }
            for (int ky = 0; ky < 7; ++ky) add_tap(ky * hg.pw, 0, ky, -1);
          }
          const bool ok = hm == HALO_CONV3    ? taps_match<HALO_CONV3>(hg)
                          : hm == HALO_CONVT2 ? taps_match<HALO_CONVT2>(hg)
                          : hm == HALO_STEM4X ? taps_match<HALO_STEM4X>(hg)
                          : hm == HALO_CONV3S2 ? taps_match<HALO_CONV3S2>(hg)
                          : hm == HALO_CONV3X2 ? taps_match<HALO_CONV3X2>(hg)
                                              : taps_match<HALO_STEM7>(hg);
          if (!ok) fail(LSG_ERUNTIME, std::string("generator: halo tap table mismatch at ") + L.name);
          if (hm == HALO_CONV3X2) {
            // per tap: rows (z, co) x K = input channel; 16-bit: a SW128 block of
            // channels 0..63 then a SW32 block of channels 64..79; fp8: one SW128 block
            const int rows = 2 * L.cout;
            const int64_t blk_units = (int64_t)rows * BK + (f8 ? 0 : rows * 16);
            hg.off = (int64_t)pack.size();
            pack.resize(pack.size() + (size_t)hg.ntaps * blk_units, 0);
            for (int tap = 0; tap < hg.ntaps; ++tap) {
              uint16_t* blk = pack.data() + hg.off + tap * blk_units;
              for (int r = 0; r < rows; ++r) {
                const int z = r / L.cout, co = r % L.cout, kx = hg.kx[tap] - z, ky = hg.ky[tap];
                for (int c = 0; c < L.cin; ++c) {
                  const float v = (kx >= 0 && kx < 3) ? wat(co, c, ky, kx) : 0.f;
                  if (f8 || c < 64) {
                    store(blk, r, c, v, sw[co]);
                  } else {  // SW32: 32-byte rows, 16-byte chunk ^= (row >> 2) & 1
                    const int j = c - 64;
                    uint16_t* b32 = blk + rows * BK;
                    b32[r * 16 + (((j >> 3) ^ ((r >> 2) & 1)) << 3) + (j & 7)] = h->prec == PR_FP16 ? f2h(v) : f2bf(v);
                  }
                }
              }
            }
          } else {
          // [cb][tap][cout][KE]: one K block per (channel block of KE channels, tap);
          // macro-pixel stem: rows (pixel offset z, cout), K = (x-shift plane, channel)
          const bool x4 = hm == HALO_STEM4X;
          // N tiles of 64 channels for the wide ConvT (4 phase accumulators x 64 fill TMEM)
          const int hbn = hm == HALO_CONVT2 ? std::min(L.cout, 64) : hm == HALO_CONV3 ? std::min(L.cout, 128) : L.cout,
                    hnt = L.cout / hbn;
          const int ncb = (hm == HALO_STEM7 || hm == HALO_CONV3S2) ? 1 : x4 ? 2 : (L.cin + KE - 1) / KE,
                    bnh = x4 ? 4 * L.cout : hbn;
          hg.off = (int64_t)pack.size();
          pack.resize(pack.size() + (size_t)hnt * ncb * hg.ntaps * bnh * BK, 0);
          uint16_t* dst = pack.data() + hg.off;
          const int gch = 8 * cpu;  // channels per 16-byte granule (stem: one x-shifted plane)
          for (int nt = 0; nt < hnt; ++nt)
          for (int cb = 0; cb < ncb; ++cb)
            for (int tap = 0; tap < hg.ntaps; ++tap) {
              uint16_t* blk = dst + (((size_t)nt * ncb + cb) * hg.ntaps + tap) * bnh * BK;
              for (int r = 0; r < bnh; ++r)
                for (int j = 0; j < KE; ++j) {
                  const int co = x4 ? r % L.cout : nt * hbn + r;
                  int c = cb * KE + j, ky = hg.ky[tap], kx = hg.kx[tap];
                  if (hm == HALO_STEM7) {
                    kx = j / gch;
                    c = j % gch;
                  } else if (x4) {  // plane cb*8 + j/gch reads input column 4*jm + plane - 3
                    kx = cb * 8 + j / gch - r / L.cout;
                    c = j % gch;
                  }
                  const float v = (c < L.cin && kx >= 0 && kx < L.kw) ? wat(co, c, ky, kx) : 0.f;
                  store(blk, r, j, v, sw[co]);
                }
            }
          }
        }
        // input channels padded to whole 16-byte granules (8 units)
        const int cin_pad = (L.cin + 8 * cpu - 1) / (8 * cpu) * (8 * cpu);
        const int bn = (li == kNumLayers - 2) ? 32 : pick_bn(L.cout);
        const int ntiles = L.cout / bn;
        for (size_t z = 0; z < G.size(); ++z) {
          const PhaseGeo& pg = G[z];
          const int K = pg.ntaps * cin_pad;  // elements
          const int kbs = (int)ceil_div(K, KE);
          pack_off[li * MAX_PHASES + z] = (int64_t)pack.size();
          pack.resize(pack.size() + (size_t)ntiles * kbs * bn * BK, 0);
          uint16_t* dst = pack.data() + pack_off[li * MAX_PHASES + z];
          for (int nt = 0; nt < ntiles; ++nt)
            for (int kb = 0; kb < kbs; ++kb) {
              uint16_t* blk = dst + ((size_t)nt * kbs + kb) * bn * BK;
              for (int r = 0; r < bn; ++r) {
                const int co = nt * bn + r;
                for (int j = 0; j < KE; ++j) {
                  const int k = kb * KE + j;
                  float v = 0.f;
                  if (k < K) {
                    const int t = k / cin_pad, ci = k % cin_pad;
                    if (ci < L.cin) v = wat(co, ci, pg.ky[t], pg.kx[t]);
                  }
                  store(blk, r, j, v, sw[co]);
                }
              }
            }
        }
      }
      h->wpack.alloc(pack.size());
      LSG_CUDA(cudaMemcpy(h->wpack.p, pack.data(), pack.size() * 2, cudaMemcpyHostToDevice));
      h->bias.alloc(bias.size());
      LSG_CUDA(cudaMemcpy(h->bias.p, bias.data(), bias.size() * 4, cudaMemcpyHostToDevice));
      h->w1b1.alloc(w1b1.size());
      LSG_CUDA(cudaMemcpy(h->w1b1.p, w1b1.data(), w1b1.size() * 4, cudaMemcpyHostToDevice));

      // ---------------- plan: input/output views per layer
      // channel arguments below are real channels; views count 16-bit units
      auto slice = [cpu](View v, int coff, int C) {
        View s = v;
        s.pitch = v.C;
        s.coff = coff / cpu;
        s.C = C / cpu;
        return s;
      };
      auto resize = [cpu](View v, int H, int W, int C) {
        View s = v;
        s.H = H;
        s.W = W;
        s.C = C / cpu;
        s.pitch = C / cpu;
        s.coff = 0;
        return s;
      };
      // (in, out) views per layer, in layer order
      std::vector<std::pair<View, View>> io(kNumLayers);
      View S0 = h->S0, S1 = h->S1, A0 = h->A0, A1 = h->A1;
      View* cat = h->cat;
      int li = 0;
      // face encoder
      io[li++] = {h->x_face, slice(cat[6], 64, 16)};
      io[li++] = {(gen_knobs() & 32768) ? slice(cat[6], 64, 16) : h->X16, resize(S0, 48, 48, 32)};
      io[li++] = {resize(S0, 48, 48, 32), resize(S1, 48, 48, 32)};
      io[li++] = {resize(S1, 48, 48, 32), slice(cat[5], 128, 32)};
      io[li++] = {slice(cat[5], 128, 32), resize(S0, 24, 24, 64)};
      io[li++] = {resize(S0, 24, 24, 64), resize(S1, 24, 24, 64)};
      io[li++] = {resize(S1, 24, 24, 64), resize(S0, 24, 24, 64)};
      io[li++] = {resize(S0, 24, 24, 64), slice(cat[4], 256, 64)};
      io[li++] = {slice(cat[4], 256, 64), resize(S0, 12, 12, 128)};
      io[li++] = {resize(S0, 12, 12, 128), resize(S1, 12, 12, 128)};
      io[li++] = {resize(S1, 12, 12, 128), slice(cat[3], 384, 128)};
      io[li++] = {slice(cat[3], 384, 128), resize(S0, 6, 6, 256)};
      io[li++] = {resize(S0, 6, 6, 256), resize(S1, 6, 6, 256)};
      io[li++] = {resize(S1, 6, 6, 256), slice(cat[2], 512, 256)};
      io[li++] = {slice(cat[2], 512, 256), resize(S0, 3, 3, 512)};
      io[li++] = {resize(S0, 3, 3, 512), slice(cat[1], 512, 512)};
      io[li++] = {slice(cat[1], 512, 512), resize(S0, 1, 1, 512)};
      io[li++] = {resize(S0, 1, 1, 512), slice(cat[0], 512, 512)};
      // audio encoder
      io[li++] = {h->x_mel, resize(A0, 80, 16, 32)};
      io[li++] = {resize(A0, 80, 16, 32), resize(A1, 80, 16, 32)};
      io[li++] = {resize(A1, 80, 16, 32), resize(A0, 80, 16, 32)};
      io[li++] = {resize(A0, 80, 16, 32), resize(A1, 27, 16, 64)};
      io[li++] = {resize(A1, 27, 16, 64), resize(A0, 27, 16, 64)};
      io[li++] = {resize(A0, 27, 16, 64), resize(A1, 27, 16, 64)};
      io[li++] = {resize(A1, 27, 16, 64), resize(A0, 9, 6, 128)};
      io[li++] = {resize(A0, 9, 6, 128), resize(A1, 9, 6, 128)};
      io[li++] = {resize(A1, 9, 6, 128), resize(A0, 9, 6, 128)};
      io[li++] = {resize(A0, 9, 6, 128), resize(A1, 3, 3, 256)};
      io[li++] = {resize(A1, 3, 3, 256), resize(A0, 3, 3, 256)};
      io[li++] = {resize(A0, 3, 3, 256), resize(A1, 1, 1, 512)};
      io[li++] = {resize(A1, 1, 1, 512), resize(A0, 1, 1, 512)};
      // decoder
      io[li++] = {resize(A0, 1, 1, 512), slice(cat[0], 0, 512)};
      io[li++] = {cat[0], resize(S0, 3, 3, 512)};
      io[li++] = {resize(S0, 3, 3, 512), slice(cat[1], 0, 512)};
      io[li++] = {cat[1], resize(S0, 6, 6, 512)};
      io[li++] = {resize(S0, 6, 6, 512), resize(S1, 6, 6, 512)};
      io[li++] = {resize(S1, 6, 6, 512), slice(cat[2], 0, 512)};
      io[li++] = {cat[2], resize(S0, 12, 12, 384)};
      io[li++] = {resize(S0, 12, 12, 384), resize(S1, 12, 12, 384)};
      io[li++] = {resize(S1, 12, 12, 384), slice(cat[3], 0, 384)};
      io[li++] = {cat[3], resize(S0, 24, 24, 256)};
      io[li++] = {resize(S0, 24, 24, 256), resize(S1, 24, 24, 256)};
      io[li++] = {resize(S1, 24, 24, 256), slice(cat[4], 0, 256)};
      io[li++] = {cat[4], resize(S0, 48, 48, 128)};
      io[li++] = {resize(S0, 48, 48, 128), resize(S1, 48, 48, 128)};
      io[li++] = {resize(S1, 48, 48, 128), slice(cat[5], 0, 128)};
      io[li++] = {cat[5], resize(S0, 96, 96, 64)};
      io[li++] = {resize(S0, 96, 96, 64), resize(S1, 96, 96, 64)};
      io[li++] = {resize(S1, 96, 96, 64), slice(cat[6], 0, 64)};
      io[li++] = {cat[6], View{}};  // out0 (+ out1 fused)
      if (li != kNumLayers - 1) fail(LSG_ERUNTIME, "generator plan does not cover every layer");

      // tensor ids (fp8 scales): fixed for inputs / concat buffers, per layer otherwise
      std::vector<int> in_id(kNumLayers, 0), out_id(kNumLayers, 0);
      {
        auto fixed = [&](const View& v) -> int {
          if (v.p == h->x_face.p) return 0;
          if (v.p == h->x_mel.p) return 1;
          if (v.p == h->X16.p) return 8;  // fe0's output: same values (and fp8 scale) as its cat[6] slice
          for (int k = 0; k < 7; ++k)
            if (v.p == h->cat[k].p) return 2 + k;
          return -1;
        };
        std::vector<std::pair<const uint16_t*, int>> last;  // scratch buffer -> tensor id it holds
        auto holder = [&](const uint16_t* p0) {
          for (auto& e : last)
            if (e.first == p0) return e.second;
          fail(LSG_ERUNTIME, "generator plan: read of an unwritten scratch buffer");
          return -1;
        };
        for (int l = 0; l < kNumLayers - 1; ++l) {
          const View& in = io[l].first;
          const View& ov = io[l].second;
          in_id[l] = fixed(in) >= 0 ? fixed(in) : holder(in.p);
          if (l == kNumLayers - 2) continue;  // fused output layer: no stored tensor
          const int f = fixed(ov);
          out_id[l] = f >= 0 ? f : 9 + l;
          if (f < 0) {
            bool found = false;
            for (auto& e : last)
              if (e.first == ov.p) {
                e.second = out_id[l];
                found = true;
              }
            if (!found) last.push_back({ov.p, out_id[l]});
          }
        }
      }
      h->plan_in_id = in_id;
      h->plan_out_id = out_id;
      std::vector<float> osc;
      std::vector<int64_t> osc_off(kNumLayers, 0);
      if (f8) {
        for (int l = 0; l < kNumLayers - 1; ++l) {
          // int8 epilogues work in output-code units (epi16): 1 / s_out folded
          // into this layer's oscale and bias here, into res_scale below
          const float fold = i8 && l != kNumLayers - 2 ? 1.f / ascale[out_id[l]] : 1.f;
          osc_off[l] = (int64_t)osc.size();
          for (int co = 0; co < kLayers[l].cout; ++co) osc.push_back(ascale[in_id[l]] * wscale[l][co] * fold);
          for (int co = 0; co < kLayers[l].cout; ++co) bias[bias_off[l] + co] *= fold;
        }
        h->oscale.alloc(osc.size());
        LSG_CUDA(cudaMemcpy(h->oscale.p, osc.data(), osc.size() * 4, cudaMemcpyHostToDevice));
        if (i8) LSG_CUDA(cudaMemcpy(h->bias.p, bias.data(), bias.size() * 4, cudaMemcpyHostToDevice));
      }
      for (int l = 0; l < kNumLayers - 1; ++l) {
        const LayerSpec& L = kLayers[l];
        const View in = io[l].first, ov = io[l].second;
        const bool fused = (l == kNumLayers - 2);
        LayerRun r{};
        r.layer = l;
        r.fused = fused;
        r.bn = fused ? 32 : pick_bn(L.cout);
        r.ntiles = L.cout / r.bn;
        r.nphases = (int)geo[l].size();
        ConvParams& p = r.p;
        r.in_view = in;
        p.H = in.H;
        p.W = in.W;
        p.C = (L.cin + 8 * cpu - 1) / (8 * cpu) * 8;  // 16-bit units, whole 16-byte granules
        if (in.C != p.C) fail(LSG_ERUNTIME, std::string("generator plan: channel mismatch at ") + L.name);
        p.cc = p.C % 64 == 0 ? 64 : (p.C % 32 == 0 ? 32 : (p.C % 16 == 0 ? 16 : 8));
        // output geometry
        int OH, OW;
        if (L.kind == CONV) {
          OH = (in.H + 2 * L.ph - L.kh) / L.sh + 1;
          OW = (in.W + 2 * L.pw - L.kw) / L.sw + 1;
        } else {
          OH = (in.H - 1) * L.sh - 2 * L.ph + L.kh + L.oph;
          OW = (in.W - 1) * L.sw - 2 * L.pw + L.kw + L.opw;
        }
        if (!fused && (ov.H != OH || ov.W != OW || ov.C != L.cout / cpu))
          fail(LSG_ERUNTIME, std::string("generator plan: shape mismatch at ") + L.name);
        p.out = ov.p;
        p.OH = OH;
        p.OW = OW;
        p.out_pitch = ov.pitch;
        p.out_coff = ov.coff;
        p.res = L.res ? in.p : nullptr;
        p.res_pitch = in.pitch;
        p.res_coff = in.coff;
        p.bias = h->bias.p + bias_off[l];
        p.oscale = f8 ? h->oscale.p + osc_off[l] : nullptr;
        p.res_scale = f8 ? ascale[in_id[l]] / (i8 && !fused ? ascale[out_id[l]] : 1.f) : 1.f;
        p.out_inv = f8 && !i8 && !fused ? 1.f / ascale[out_id[l]] : 1.f;  // int8: folded (epi16)
        p.relu = 1;
        p.out_mode = OUT_16;
        if (L.kind == CONV) {
          p.sy = L.sh;
          p.sx = L.sw;
          p.osy = p.osx = 1;
        } else {
          p.sy = p.sx = 1;
          p.osy = L.sh;
          p.osx = L.sw;
          if ((int)geo[l].size() == L.kh * L.kw && L.sh == 1) {  // one-tap phases of a 1x1 input
            if (in.H != 1 || in.W != 1) fail(LSG_ERUNTIME, std::string("generator plan: ") + L.name + " needs a 1x1 input");
            p.osy = L.kh;
            p.osx = L.kw;
          }
        }
        if (fused) {
          p.w1 = h->w1b1.p;
          p.b1 = h->w1b1.p + 96;
        }
        if (r.nphases > MAX_PHASES) fail(LSG_ERUNTIME, "generator: too many phases");
        // im2col bounding box: conv -> lower = -pad, upper = pad - (k - 1), traversal
        // stride = conv stride; convT phases walk the input grid (lower = upper = 0)
        int lower_w = 0, lower_h = 0, upper_w = 0, upper_h = 0;
        if (L.kind == CONV) {
          lower_w = -L.pw;
          lower_h = -L.ph;
          upper_w = L.pw - (L.kw - 1);
          upper_h = L.ph - (L.kh - 1);
        }
        p.lower_w = lower_w;
        p.lower_h = lower_h;
        encode_im2col(&p.tmap, in, max_batch, p.cc, lower_w, lower_h, upper_w, upper_h, p.sx, p.sy);
        for (int z = 0; z < r.nphases; ++z) {
          const PhaseGeo& pg = geo[l][z];
          Phase& P = p.ph[z];
          P.w = h->wpack.p + pack_off[l * MAX_PHASES + z];
          P.ntaps = pg.ntaps;
          P.K = pg.ntaps * p.C;
          P.nsteps = (int)ceil_div(P.K, 16);
          P.nloads = pg.ntaps * (p.C / p.cc);
          if (p.cc == 8 && (P.nloads & 1)) P.nloads += 1;  // K=16 steps read loads in pairs: zero pad load
          P.kblocks = (int)ceil_div(P.nloads, BK / p.cc);
          if (P.kblocks != (int)ceil_div(P.K, BK)) fail(LSG_ERUNTIME, std::string("generator: K blocking at ") + L.name);
          P.oy = pg.oy;
          P.ox = pg.ox;
          for (int t = 0; t < pg.ntaps; ++t) {
            const int ow = pg.dx[t] - lower_w, oh = pg.dy[t] - lower_h;
            if (ow < 0 || oh < 0 || ow > 255 || oh > 255) fail(LSG_ERUNTIME, "generator: im2col offset range");
            P.offw[t] = (unsigned char)ow;
            P.offh[t] = (unsigned char)oh;
          }
          P.offw[pg.ntaps] = (unsigned char)OOB_OFFSET;  // pad tap: always outside the input
          P.offh[pg.ntaps] = 0;
          r.GH[z] = L.kind == CONV ? OH : (int)ceil_div(OH - pg.oy, p.osy);
          r.GW[z] = L.kind == CONV ? OW : (int)ceil_div(OW - pg.ox, p.osx);
          P.GH = r.GH[z];
          P.GW = r.GW[z];
          // the tensor map's bounding box must generate exactly the phase grid
          const int gw = (in.W + upper_w - lower_w - 1) / p.sx + 1, gh = (in.H + upper_h - lower_h - 1) / p.sy + 1;
          if (gw != P.GW || gh != P.GH) fail(LSG_ERUNTIME, std::string("generator: im2col grid mismatch at ") + L.name);
        }
        // CTA-pair launches load weight half-tiles through a 2-D map over the
        // layer's packed weights (all phases, rows of 64 units, pre-swizzled)
        if (!fused && r.bn >= 128) {
          int64_t rows = 0;
          for (int z = 0; z < r.nphases; ++z) {
            p.wrow0[z] = (int)((p.ph[z].w - p.ph[0].w) / BK);
            rows = std::max<int64_t>(rows, p.wrow0[z] + (int64_t)r.ntiles * p.ph[z].kblocks * r.bn);
          }
          const cuuint64_t dims[2] = {(cuuint64_t)BK, (cuuint64_t)rows};
          const cuuint64_t strides[1] = {(cuuint64_t)BK * 2};
          const cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)(r.bn / 2)};
          const cuuint32_t estr[2] = {1, 1};
          CUresult cr = tiled_fn()(&p.wmap, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<uint16_t*>(p.ph[0].w), dims,
                                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (cr != CUDA_SUCCESS) fail(LSG_ECUDA, "cuTensorMapEncodeTiled (weights) failed");
          r.pair_ok = true;
        }
        const HaloGeo& hg = hgeo[l];
        if (hg.mode != HALO_NONE && (hg.mode != HALO_CONV3 || in.W >= 16)) {
          HaloParams& hp = r.hp;
          r.halo = true;
          r.halo_mode = hg.mode;
          hp.H = in.H;
          hp.W = in.W;
          hp.C = p.C;
          hp.GH = hg.mode == HALO_CONVT2 ? in.H : OH;
          hp.GW = hg.mode == HALO_CONVT2   ? in.W
                  : hg.mode == HALO_STEM4X ? (int)ceil_div(OW, 4)
                  : hg.mode == HALO_CONV3X2 ? (int)ceil_div(OW, 2)
                                            : OW;
          hp.xmul = hg.mode == HALO_STEM4X ? 4 : 1;
          hp.oy0 = hg.oy0;
          hp.ox0 = hg.ox0;
          hp.pw = hg.pw;
          hp.ph = hg.ph;
          hp.plane = (hp.pw * hp.ph * 16 + 127) / 128 * 128;
          if (hp.plane > HaloCfg<32, HALO_CONV3, false, true>::PLANE_MAX) fail(LSG_ERUNTIME, "generator: halo patch too large");
          hp.shift_planes = hg.mode == HALO_STEM7 || hg.mode == HALO_STEM4X;
          // planes come in pairs per K step; an odd last plane reads channels past the
          // view, which the TMA zero-fills (fp8 out0: 80 channels = 5 planes)
          hp.ngran = hg.mode == HALO_STEM4X ? 10 : hp.shift_planes ? 8 : ((p.C / 8 + 1) & ~1);
          hp.ncb = hg.mode == HALO_CONV3S2   ? hp.ngran / 2         // S2: 2 granules x 4 parities
                   : hg.mode == HALO_CONV3X2 ? (hp.ngran + 3) / 4  // X2: 4 granules x 2 parities
                                             : (hp.ngran + 7) / 8;
          hp.ntaps = hg.ntaps;
          for (int t = 0; t < MAX_HTAPS; ++t) {
            hp.aoff[t] = hg.aoff[t];
            hp.tphase[t] = hg.tphase[t];
          }
          hp.tfirst = hg.tfirst;
          hp.osy = hg.mode == HALO_CONVT2 ? 2 : 1;
          hp.osx = hg.mode == HALO_CONVT2 || hg.mode == HALO_CONV3X2 ? 2 : hg.mode == HALO_STEM4X ? 4 : 1;
          for (int z = 0; z < 4; ++z) {
            hp.poy[z] = hg.poy[z];
            hp.pox[z] = hg.pox[z];
          }
          hp.tiles_x = (int)ceil_div(hp.GW, HTW);
          hp.tiles_y = (int)ceil_div(hp.GH, HTH);
          hp.tiles_per_img = hp.tiles_x * hp.tiles_y;
          if (hg.mode == HALO_CONVT2) r.bn = std::min(L.cout, 64);  // N tiles (packed per tile above)
          if (hg.mode == HALO_CONV3) r.bn = std::min(L.cout, 128);
          hp.ntn = L.cout / r.bn;
          hp.w = h->wpack.p + hg.off;
          hp.wblocks = (hg.mode == HALO_CONV3S2 || hg.mode == HALO_CONV3X2) ? hg.ntaps  // one block per tap
                                                                            : hp.ncb * hg.ntaps;
          if (hg.mode == HALO_CONV3S2 && hp.ncb * 32 > 128) fail(LSG_ERUNTIME, "generator: stride-2 halo needs <= 4 channel blocks");
          if (hg.mode != HALO_STEM4X && hg.mode != HALO_STEM7) {  // CTA pairs: weight half-blocks by TMA
            const cuuint64_t dims[2] = {(cuuint64_t)BK, (cuuint64_t)hp.wblocks * r.bn * hp.ntn};
            const cuuint64_t strides[1] = {(cuuint64_t)BK * 2};
            const cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)(r.bn / 2)};
            const cuuint32_t estr[2] = {1, 1};
            CUresult cr = tiled_fn()(&hp.wmap, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<uint16_t*>(hp.w), dims,
                                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (cr != CUDA_SUCCESS) fail(LSG_ECUDA, "cuTensorMapEncodeTiled (halo weights) failed");
            r.hp_pair_ok = true;
          }
          r.halo_bres = hg.mode == HALO_STEM4X
                            ? (int64_t)hp.wblocks * 4 * r.bn * BK * 2 <= HaloCfg<16, HALO_STEM4X, false, true>::W_RES_BYTES
                            : (int64_t)hp.wblocks * r.bn * BK * 2 <= HaloCfg<32, HALO_CONV3, false, true>::W_RES_BYTES;
          if (r.bn * hp.ntn != L.cout || (hp.ntn > 1 && (r.halo_bres || fused || hp.tiles_per_img % 2)))
            fail(LSG_ERUNTIME, "generator: halo N tiling needs streamed weights and an even tile count");
          hp.OH = OH;
          hp.OW = OW;
          hp.out = p.out;
          hp.out_pitch = p.out_pitch;
          hp.out_coff = p.out_coff;
          hp.res = p.res;
          hp.res_pitch = p.res_pitch;
          hp.res_coff = p.res_coff;
          hp.bias = p.bias;
          hp.oscale = p.oscale;
          hp.res_scale = p.res_scale;
          hp.out_inv = p.out_inv;
          hp.relu = p.relu;
          hp.out_mode = p.out_mode;
          hp.w1 = p.w1;
          hp.b1 = p.b1;
          if (hg.mode == HALO_CONV3S2) encode_patch(&hp.tmap, in, max_batch, hp.pw, hp.ph, 2, 2);
          else if (hg.mode == HALO_CONV3X2) encode_patch(&hp.tmap, in, max_batch, hp.pw, hp.ph, 2, 1);
          else encode_patch(&hp.tmap, in, max_batch, hp.pw, hp.ph, hp.xmul);
          const int bc = std::min(r.bn * 2 / cpu, 128) / 2;  // box channels in 16-bit units (128-byte rows max)
          if (!fused) encode_box(&hp.tmap_out, ov, max_batch, bc, HTW * hp.osx, HTH * hp.osy, hp.osx, hp.osy);
          hp.out2 = l == 0 && !(gen_knobs() & 32768);  // fe0: the dense copy fe1.0 reads
          if (hp.out2) encode_box(&hp.tmap_out2, h->X16, max_batch, bc, HTW * hp.osx, HTH * hp.osy, hp.osx, hp.osy);
          if (hg.mode == HALO_CONV3 && !fused) {
            if (!L.res || in.C != L.cout / cpu) fail(LSG_ERUNTIME, std::string("generator: halo 3x3 block without residual at ") + L.name);
            encode_box(&hp.tmap_res, in, max_batch, bc, HTW, HTH, 1, 1);
          }
        }
        r.p.trace_slot = (int)h->plan.size();
        r.hp.trace_slot = r.p.trace_slot;
        h->plan.push_back(r);
      }
      set_smem_attrs(h->prec);
      if (tail) {
        // fp8 on the decoder's last block + the output conv only (fd6.0 ..
        // out0: 28% of the FLOPs); int8 from fd1.0 (90%); the 16-bit engine
        // before them -- the splits the sensitivity sweeps pick for a >= 30 dB
        // floor on this network (tools/precision_sweep.py, tools/int8_sweep.py,
        // DESIGN.md §4)
        h->tail_blk = precision == LSG_PREC_INT8_TAIL ? 1 : 6;
        const std::string first = "fd" + std::to_string(h->tail_blk) + ".0";
        for (int l = 0; l < kNumLayers; ++l)
          if (first == kLayers[l].name) h->tail0 = l;
        if (h->tail0 == 0 || h->plan[h->tail0].in_view.p != h->cat[h->tail_blk - 1].p)
          fail(LSG_ERUNTIME, "generator: tail split is not at a decoder block reading a concat buffer");
        lsg_gen hd = nullptr;
        if (lsg_gen_create_q(ctx, weights, n_floats, LSG_PREC_FP16, nullptr, 0, max_batch, &hd) != LSG_OK)
          fail(LSG_ERUNTIME, std::string("lsg_gen_create: fp16 head: ") + lsg_last_error());
        h->head = hd;
      }
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

lsg_status lsg_gen_destroy(lsg_gen h) {
  return guard(__func__, [&] {
    if (!h) return;
    DeviceGuard g(h->ctx);
    h->ctx->sync();
    delete h;
  });
}

lsg_status lsg_gen_forward(lsg_gen h, const float* mel_rows, const int32_t* chunk_row, const uint8_t* target,
                           const uint8_t* refs, const int32_t* ref_index, void* out, int32_t out_format, int32_t B) {
  return guard(__func__, [&] {
    DeviceGuard g(h->ctx);
    gen::forward_gather(h, mel_rows, chunk_row, target, nullptr, refs, ref_index, out, out_format, B);
  });
}

}  // extern "C"

// ------------------------------------------------------ input prep launch
static void prep_inputs(lsg_gen h, const float* mel_rows, const int32_t* chunk_row, const uint8_t* target,
                        const int64_t* target_idx, const uint8_t* refs, const int32_t* ref_index, int B,
                        cudaStream_t st) {
  const unsigned gf = (unsigned)ceil_div((int64_t)B * 96 * 96, 256), gm = (unsigned)ceil_div((int64_t)B * 80 * 16, 256);
  if (h->prec == PR_I8) fail(LSG_ERUNTIME, "generator: an INT8 engine has no input stage (it is a tail)");
  if (h->prec == PR_FP8) {
    prep_faces<PR_FP8><<<gf, 256, 0, st>>>(target, target_idx, refs, ref_index, h->x_face.p, B, h->inv_face);
    prep_mel<PR_FP8><<<gm, 256, 0, st>>>(mel_rows, chunk_row, h->x_mel.p, B, h->inv_mel);
  } else if (h->prec == PR_FP16) {
    prep_faces<PR_FP16><<<gf, 256, 0, st>>>(target, target_idx, refs, ref_index, h->x_face.p, B, 1.f);
    prep_mel<PR_FP16><<<gm, 256, 0, st>>>(mel_rows, chunk_row, h->x_mel.p, B, 1.f);
  } else {
    prep_faces<PR_BF16><<<gf, 256, 0, st>>>(target, target_idx, refs, ref_index, h->x_face.p, B, 1.f);
    prep_mel<PR_BF16><<<gm, 256, 0, st>>>(mel_rows, chunk_row, h->x_mel.p, B, 1.f);
  }
}

static void absmax_into(lsg_gen h, const uint16_t* src, int pitch, int coff, int C, int64_t pixels, unsigned* dst,
                        cudaStream_t st) {
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(pixels * C, 256), 4096);
  if (h->prec == PR_FP16) absmax_view<PR_FP16><<<grid, 256, 0, st>>>(src, pitch, coff, C, pixels, dst);
  else absmax_view<PR_BF16><<<grid, 256, 0, st>>>(src, pitch, coff, C, pixels, dst);
}

extern "C" {

// max |activation| of every fp8 scale group (kTensors: face, mel, cat0..6,
// per-layer outputs) over a calibration batch, on a 16-bit engine
lsg_status lsg_gen_calibrate(lsg_gen h, const float* mel_rows, const int32_t* chunk_row, const uint8_t* target,
                             const uint8_t* refs, const int32_t* ref_index, int32_t B, float* absmax, int32_t cap,
                             int32_t* n_tensors) {
  return guard(__func__, [&] {
    *n_tensors = kTensors;
    if (cap < kTensors) return;
    if (h->prec == PR_FP8 || h->prec == PR_I8) invalid("lsg_gen_calibrate: calibrate on a bf16/fp16 engine");
    if (B <= 0 || B > h->max_batch) invalid("lsg_gen_calibrate: batch out of range");
    Ctx* ctx = h->ctx;
    DeviceGuard g(ctx);
    cudaStream_t st = ctx->stream;
    DevBuf<unsigned> acc;
    acc.alloc(kTensors);
    LSG_CUDA(cudaMemsetAsync(acc.p, 0, kTensors * sizeof(unsigned), st));
    prep_inputs(h, mel_rows, chunk_row, target, nullptr, refs, ref_index, B, st);
    absmax_into(h, h->x_face.p, h->x_face.pitch, h->x_face.coff, h->x_face.C, (int64_t)B * 96 * 96, acc.p + 0, st);
    absmax_into(h, h->x_mel.p, h->x_mel.pitch, h->x_mel.coff, h->x_mel.C, (int64_t)B * 80 * 16, acc.p + 1, st);
    for (size_t l = 0; l < h->plan.size(); ++l) {
      LayerRun& r = h->plan[l];
      if (r.fused) {
        r.p.out_mode = r.hp.out_mode = OUT_F32_LOGITS;
        r.p.final_out = r.hp.final_out = nullptr;
        continue;  // its result is not stored as a tensor
      }
      dispatch(h, r, B, st);
      const ConvParams& p = r.p;
      absmax_into(h, p.out, p.out_pitch, p.out_coff, kLayers[l].cout, (int64_t)B * p.OH * p.OW,
                  acc.p + h->plan_out_id[l], st);
    }
    std::vector<unsigned> hv(kTensors);
    LSG_CUDA(cudaMemcpyAsync(hv.data(), acc.p, kTensors * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    LSG_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < kTensors; ++i) {
      float f;
      std::memcpy(&f, &hv[i], 4);
      absmax[i] = f;
    }
  });
}

lsg_status lsg_gen_create(lsg_ctx ctx, const float* weights, int64_t n_floats, int32_t precision, int32_t max_batch,
                          lsg_gen* out) {
  return lsg_gen_create_q(ctx, weights, n_floats, precision, nullptr, 0, max_batch, out);
}

}  // extern "C"

// ---------------------------------------------------------------- debug
// Not part of include/lsg.h: test-only introspection used by
// tests/test_generator.py to check each layer in isolation.
template <int PR>
__global__ void view_to_f32(const uint16_t* src, int pitch, int coff, int C, int64_t pixels, float* dst, float scale) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // unit index
  if (i >= pixels * C) return;
  const int64_t px = i / C;
  const int c = (int)(i - px * C);
  const uint16_t u = src[px * pitch + coff + c];
  if constexpr (PR == PR_I8) {
    dst[2 * i] = (float)(u & 0xffu) * scale;
    dst[2 * i + 1] = (float)(u >> 8) * scale;
  } else if constexpr (PR == PR_FP8) {
    const __half2_raw hr = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)u, __NV_E4M3);
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&hr));
    dst[2 * i] = f.x * scale;
    dst[2 * i + 1] = f.y * scale;
  } else {
    dst[i] = PR == PR_FP16 ? __half2float(__ushort_as_half(u)) : __bfloat162float(__ushort_as_bfloat16(u));
  }
}

// LSG_TRACE builds: copy the phase timestamps out ([64 layers][160 CTAs][16], ns).
extern "C" lsg_status lsgdbg_trace_read(unsigned long long* out, int64_t n) {
  return guard(__func__, [&] {
#ifdef LSG_TRACE
    if (n == 0) {  // clear
      void* a = nullptr;
      LSG_CUDA(cudaGetSymbolAddress(&a, g_lsg_trace));
      LSG_CUDA(cudaMemset(a, 0, sizeof(unsigned long long) * TRACE_LAYERS * TRACE_CTAS * TRACE_EV));
      return;
    }
    const size_t cnt = std::min<size_t>((size_t)n, (size_t)TRACE_LAYERS * TRACE_CTAS * TRACE_EV);
    LSG_CUDA(cudaMemcpyFromSymbol(out, g_lsg_trace, cnt * sizeof(unsigned long long)));
#else
    (void)out;
    (void)n;
    invalid("lsgdbg_trace_read: library built without LSG_TRACE");
#endif
  });
}

// Per plan layer at batch B: {layer index, Route, launch tile width, split-K
// factor} -- the decisions forward() takes (route_of), for the tests.
extern "C" lsg_status lsgdbg_gen_routes(lsg_gen h, int32_t B, int32_t* out, int32_t cap, int32_t* n_out) {
  return guard(__func__, [&] {
    if (!h || !n_out) invalid("lsgdbg_gen_routes: null argument");
    if (B < 1 || B > h->max_batch) invalid("lsgdbg_gen_routes: bad batch");
    const int n = (int)h->plan.size();
    *n_out = n;
    if (!out) return;
    for (int i = 0; i < n && i < cap; ++i) {
      const lsg_gen_s* e = (h->head && i < h->tail0) ? h->head : h;  // fp8 tail: head's layers
      const LayerRun& r = e->plan[i];
      RouteInfo ri = route_of(r, B, e->sm_count, e->splitk_tiles);
      if (r.layer == kAe0 && e->ae0w.p && !(gen_knobs() & 8192)) ri = {RT_STEM, 0, 1};
      out[4 * i] = r.layer;
      out[4 * i + 1] = ri.route;
      out[4 * i + 2] = ri.bn;
      out[4 * i + 3] = ri.ksplit;
    }
  });
}

namespace lsg {
namespace gen {
static void run_plan(lsg_gen h, int l0, int l1, int mode, void* out, int B, cudaStream_t st);
static void requant_tail_inputs(lsg_gen h, int B, cudaStream_t st);
}  // namespace gen
}  // namespace lsg

extern "C" lsg_status lsgdbg_run_until(lsg_gen h, const float* mel_rows, const int32_t* chunk_row,
                                        const uint8_t* target, const uint8_t* refs, const int32_t* ref_index,
                                        int32_t B, int32_t stop_layer, int32_t which, float* out_dev,
                                        int32_t* shape4) {
  return guard(__func__, [&] {
    Ctx* ctx = h->ctx;
    DeviceGuard g(ctx);
    cudaStream_t st = ctx->stream;
    if (stop_layer < 0 || stop_layer >= (int)h->plan.size() - 1) invalid("lsgdbg_run_until: bad layer");
    if (h->head) {  // an 8-bit tail: its own layers only, after the head and the requantisation
      if (stop_layer < h->tail0) invalid("lsgdbg_run_until: a head layer of a tail engine (check the head separately)");
      prep_inputs(h->head, mel_rows, chunk_row, target, nullptr, refs, ref_index, B, st);
      run_plan(h->head, 0, h->tail0, OUT_F32_LOGITS, nullptr, B, st);
      requant_tail_inputs(h, B, st);
      for (int l = h->tail0; l <= stop_layer; ++l) dispatch(h, h->plan[l], B, st);
    } else {
      prep_inputs(h, mel_rows, chunk_row, target, nullptr, refs, ref_index, B, st);
      for (int l = 0; l <= stop_layer; ++l) dispatch(h, h->plan[l], B, st);
    }
    if (!out_dev) return;  // timing a prefix of the layer chain
    const LayerRun& r = h->plan[stop_layer];
    const ConvParams& p = r.p;
    const LayerSpec& L = kLayers[stop_layer];
    const uint16_t* src = which ? p.out : r.in_view.p;
    const int H = which ? p.OH : p.H, W = which ? p.OW : p.W;
    const int pitch = which ? p.out_pitch : r.in_view.pitch, coff = which ? p.out_coff : r.in_view.coff;
    const int C = which ? L.cout / h->cpu : p.C;  // units
    const float scale = h->ascale[which ? h->plan_out_id[stop_layer] : h->plan_in_id[stop_layer]];
    const int64_t pixels = (int64_t)B * H * W;
    const unsigned grid = (unsigned)ceil_div(pixels * C, 256);
    if (h->prec == PR_I8) view_to_f32<PR_I8><<<grid, 256, 0, st>>>(src, pitch, coff, C, pixels, out_dev, scale);
    else if (h->prec == PR_FP8) view_to_f32<PR_FP8><<<grid, 256, 0, st>>>(src, pitch, coff, C, pixels, out_dev, scale);
    else if (h->prec == PR_FP16) view_to_f32<PR_FP16><<<grid, 256, 0, st>>>(src, pitch, coff, C, pixels, out_dev, 1.f);
    else view_to_f32<PR_BF16><<<grid, 256, 0, st>>>(src, pitch, coff, C, pixels, out_dev, 1.f);
    LSG_CUDA(cudaGetLastError());
    shape4[0] = B;
    shape4[1] = H;
    shape4[2] = W;
    shape4[3] = C * h->cpu;
  });
}

namespace lsg {
namespace gen {

int32_t max_batch(lsg_gen h) { return h->max_batch; }
lsg_ctx context(lsg_gen h) { return static_cast<lsg_ctx>(h->ctx); }

// Launches plan layers [l0, l1) on st (the audio encoder, when in range, on
// the side stream, joined before the first decoder layer).
static void run_plan(lsg_gen h, int l0, int l1, int mode, void* out, int B, cudaStream_t st) {
  Ctx* ctx = h->ctx;
  bool any_audio = false;
  for (int l = l0; l < l1; ++l) any_audio |= kLayers[h->plan[l].layer].name[0] == 'a';
  // audio encoder (plan layers whose name starts with "ae") on the side
  // stream, forked after the input prep and joined before the decoder
  const bool fork = any_audio && !(gen_knobs() & 512);
  if (fork) {
    LSG_CUDA(cudaEventRecord(h->ev_fork, st));
    LSG_CUDA(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
  }
  bool joined = !fork;
  for (int l = l0; l < l1; ++l) {
    LayerRun& r = h->plan[l];
    if (r.fused) {
      r.p.out_mode = r.hp.out_mode = mode;
      r.p.final_out = r.hp.final_out = out;
    }
    // (both branches launch full-SM grids: capping either branch's SMs measured
    // slower at B = 128 and 512 -- the concurrency is in the small layers' tails)
    const bool audio = kLayers[r.layer].name[0] == 'a';
    if (audio && r.layer == kAe0 && h->ae0w.p && !(gen_knobs() & 8192)) {  // ae0 on CUDA cores
      cudaStream_t s2 = fork ? h->side : st;
      const unsigned grid = (unsigned)ceil_div((int64_t)B * 1280, 256);
      const ConvParams& p = r.p;
      if (h->prec == PR_I8) fail(LSG_ERUNTIME, "generator: an INT8 engine has no audio stem (it is a tail)");
      if (h->prec == PR_FP8)
        audio_stem<PR_FP8><<<grid, 256, 0, s2>>>(h->x_mel.p, h->ae0w.p, p.bias, p.oscale, p.out_inv, p.out, p.out_pitch,
                                                p.out_coff, B);
      else if (h->prec == PR_FP16)
        audio_stem<PR_FP16><<<grid, 256, 0, s2>>>(h->x_mel.p, h->ae0w.p, p.bias, p.oscale, p.out_inv, p.out,
                                                 p.out_pitch, p.out_coff, B);
      else
        audio_stem<PR_BF16><<<grid, 256, 0, s2>>>(h->x_mel.p, h->ae0w.p, p.bias, p.oscale, p.out_inv, p.out,
                                                 p.out_pitch, p.out_coff, B);
    } else if (fork && audio) {
      dispatch(h, r, B, h->side, 1);
    } else {
      if (!joined && kLayers[r.layer].name[0] == 'f' && kLayers[r.layer].name[1] == 'd') {
        LSG_CUDA(cudaEventRecord(h->ev_join, h->side));
        LSG_CUDA(cudaStreamWaitEvent(st, h->ev_join, 0));
        joined = true;
      }
      dispatch(h, r, B, st);
    }
    LSG_LAUNCHED(ctx);
  }
  if (!joined) {  // (a range without decoder layers)
    LSG_CUDA(cudaEventRecord(h->ev_join, h->side));
    LSG_CUDA(cudaStreamWaitEvent(st, h->ev_join, 0));
  }
}

// fp16 tensor (the head's) -> this 8-bit engine's buffer, x / scale with the
// epilogues' own conversion (e4m3 RN satfinite, or u8 RN saturating): 8
// channels per thread.
template <int PRD>
__global__ void requant8(const uint16_t* __restrict__ src, int spitch, int scoff, uint16_t* __restrict__ dst,
                         int dpitch, int dcoff, int C, int64_t pixels, float inv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int G = C / 8;
  if (i >= pixels * G) return;
  const int64_t px = i / G;
  const int g = (int)(i - px * G);
  const uint4 v = *reinterpret_cast<const uint4*>(src + px * spitch + scoff + 8 * g);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  float f[16] = {};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 x = Num<PR_FP16>::unpack(w[k]);
    f[2 * k] = x.x * inv;
    f[2 * k + 1] = x.y * inv;
  }
  uint4 o;
  Num<PRD>::from_float16(f, &o);
  *reinterpret_cast<uint2*>(dst + px * dpitch + dcoff + 4 * g) = make_uint2(o.x, o.y);
}

// channels [c0, c0 + C) of concat buffer k: head's fp16 copy -> h's 8-bit copy
static void requant_cat(lsg_gen h, int k, int c0, int C, int B, cudaStream_t st) {
  const View& s = h->head->cat[k];
  const View& d = h->cat[k];
  const int64_t pixels = (int64_t)B * s.H * s.W;
  const unsigned grid = (unsigned)ceil_div(pixels * (C / 8), 256);
  const float inv = 1.f / h->ascale[2 + k];
  if (h->prec == PR_I8)
    requant8<PR_I8><<<grid, 256, 0, st>>>(s.p, s.pitch, s.coff + c0, d.p, d.pitch, d.coff + c0 / 2, C, pixels, inv);
  else
    requant8<PR_FP8><<<grid, 256, 0, st>>>(s.p, s.pitch, s.coff + c0, d.p, d.pitch, d.coff + c0 / 2, C, pixels, inv);
  LSG_LAUNCHED(h->ctx);
}

// Everything an 8-bit tail reads from the head: its first block's input
// cat[j0 - 1] whole, and the encoder slices of cat[j0..6] (the decoder
// halves are written by the tail's own epilogues).
constexpr int kCatC[7] = {1024, 1024, 768, 512, 320, 160, 80};  // channels of cat k
constexpr int kCatDec[7] = {512, 512, 512, 384, 256, 128, 64};  // ... of which the decoder writes [0, kCatDec)
static void requant_tail_inputs(lsg_gen h, int B, cudaStream_t st) {
  const int j0 = h->tail_blk;
  requant_cat(h, j0 - 1, 0, kCatC[j0 - 1], B, st);
  for (int k = j0; k < 7; ++k) requant_cat(h, k, kCatDec[k], kCatC[k] - kCatDec[k], B, st);
}

// a whole forward's layers: the plan, or head + requantisation + tail
static void run_all(lsg_gen h, int mode, void* out, int B, cudaStream_t st) {
  const int n = (int)h->plan.size();
  if (!h->head) return run_plan(h, 0, n, mode, out, B, st);
  run_plan(h->head, 0, h->tail0, mode, out, B, st);
  requant_tail_inputs(h, B, st);
  run_plan(h, h->tail0, n, mode, out, B, st);
}

// the node the last operation captured on st created
static cudaGraphNode_t last_captured(cudaStream_t st) {
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  LSG_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd));
  if (cs != cudaStreamCaptureStatusActive || nd != 1) fail(LSG_ERUNTIME, "generator graph: unexpected capture state");
  return deps[0];
}

// re-point a captured kernel node at new arguments (same kernel, grid, smem)
static void set_node_args(cudaGraphExec_t exec, cudaGraphNode_t node, void** args) {
  cudaKernelNodeParams kp{};
  LSG_CUDA(cudaGraphKernelNodeGetParams(node, &kp));
  kp.kernelParams = args;
  kp.extra = nullptr;
  LSG_CUDA(cudaGraphExecKernelNodeSetParams(exec, node, &kp));
}

static void forward_graph(lsg_gen h, const float* mel_rows, const int32_t* chunk_row, const uint8_t* target,
                          const int64_t* target_idx, const uint8_t* refs, const int32_t* ref_index, void* out,
                          int mode, int B, cudaStream_t launch_st) {
  Ctx* ctx = h->ctx;
  if (!h->cap) LSG_CUDA(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
  cudaStream_t st = h->cap;  // recording only: nothing runs on it
  const int n = (int)h->plan.size();
  LayerRun& last = h->plan[n - 1];
  lsg_gen pe = h->head ? h->head : h;  // the engine whose input stage runs
  float inv_face = pe->prec == PR_FP8 ? pe->inv_face : 1.f, inv_mel = pe->prec == PR_FP8 ? pe->inv_mel : 1.f;
  auto& g = h->fwd_graphs[std::make_tuple(B, mode, target_idx ? 1 : 0)];
  if (!g.exec) {
    const int64_t l0 = ctx->launches.load();
    LSG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    struct EndOnError {  // a failure inside the capture must not leave st capturing
      cudaStream_t st;
      bool armed = true;
      ~EndOnError() {
        if (!armed) return;
        cudaGraph_t gr = nullptr;
        cudaStreamEndCapture(st, &gr);
        if (gr) cudaGraphDestroy(gr);
        cudaGetLastError();
      }
    } guard_capture{st};
    const unsigned gf = (unsigned)ceil_div((int64_t)B * 96 * 96, 256), gm = (unsigned)ceil_div((int64_t)B * 80 * 16, 256);
    if (pe->prec == PR_FP8) prep_faces<PR_FP8><<<gf, 256, 0, st>>>(target, target_idx, refs, ref_index, pe->x_face.p, B, inv_face);
    else if (pe->prec == PR_FP16) prep_faces<PR_FP16><<<gf, 256, 0, st>>>(target, target_idx, refs, ref_index, pe->x_face.p, B, 1.f);
    else prep_faces<PR_BF16><<<gf, 256, 0, st>>>(target, target_idx, refs, ref_index, pe->x_face.p, B, 1.f);
    g.n_face = last_captured(st);
    if (pe->prec == PR_FP8) prep_mel<PR_FP8><<<gm, 256, 0, st>>>(mel_rows, chunk_row, pe->x_mel.p, B, inv_mel);
    else if (pe->prec == PR_FP16) prep_mel<PR_FP16><<<gm, 256, 0, st>>>(mel_rows, chunk_row, pe->x_mel.p, B, 1.f);
    else prep_mel<PR_BF16><<<gm, 256, 0, st>>>(mel_rows, chunk_row, pe->x_mel.p, B, 1.f);
    g.n_mel = last_captured(st);
    LSG_LAUNCHED(ctx);
    LSG_LAUNCHED(ctx);
    run_all(h, mode, out, B, st);
    g.n_out = last_captured(st);  // the fused output conv: the plan's last launch
    guard_capture.armed = false;
    LSG_CUDA(cudaStreamEndCapture(st, &g.graph));
    LSG_CUDA(cudaGraphInstantiate(&g.exec, g.graph, 0));
    g.kernels = (int)(ctx->launches.load() - l0);
  } else {
    void* fa[] = {(void*)&target, (void*)&target_idx, (void*)&refs, (void*)&ref_index, (void*)&pe->x_face.p,
                  (void*)&B, (void*)&inv_face};
    set_node_args(g.exec, g.n_face, fa);
    void* ma[] = {(void*)&mel_rows, (void*)&chunk_row, (void*)&pe->x_mel.p, (void*)&B, (void*)&inv_mel};
    set_node_args(g.exec, g.n_mel, ma);
    // the output conv's parameter block as captured (launch_* derive grid
    // fields from B there), with only the caller's pointer replaced
    cudaKernelNodeParams kp{};
    LSG_CUDA(cudaGraphKernelNodeGetParams(g.n_out, &kp));
    if (last.halo) {
      HaloParams hp;
      std::memcpy(&hp, kp.kernelParams[0], sizeof(hp));
      hp.out_mode = mode;
      hp.final_out = out;
      void* oa[] = {(void*)&hp};
      set_node_args(g.exec, g.n_out, oa);
    } else {
      ConvParams cp;
      std::memcpy(&cp, kp.kernelParams[0], sizeof(cp));
      cp.out_mode = mode;
      cp.final_out = out;
      void* oa[] = {(void*)&cp};
      set_node_args(g.exec, g.n_out, oa);
    }
    ctx->launches.fetch_add(g.kernels, std::memory_order_relaxed);
  }
  LSG_CUDA(cudaGraphLaunch(g.exec, launch_st));
}

void forward_gather(lsg_gen h, const float* mel_rows, const int32_t* chunk_row, const uint8_t* target_base,
                    const int64_t* target_idx, const uint8_t* refs, const int32_t* ref_index, void* out,
                    int32_t out_format, int32_t B) {
  if (B <= 0 || B > h->max_batch) invalid("lsg_gen_forward: batch out of range");
  if (out_format < 0 || out_format > 2) invalid("lsg_gen_forward: unknown output format");
  Ctx* ctx = h->ctx;
  cudaStream_t st = ctx->stream;
  const int mode = out_format == LSG_OUT_F32_NCHW ? OUT_F32_NCHW
                                                  : (out_format == LSG_OUT_U8_NHWC ? OUT_U8_NHWC : OUT_F32_LOGITS);
  if (B == h->max_batch && !(gen_knobs() & (1 << 17))) {
    forward_graph(h, mel_rows, chunk_row, target_base, target_idx, refs, ref_index, out, mode, B, st);
    return;
  }
  // (8-bit tails: the fp16 head's input stage)
  prep_inputs(h->head ? h->head : h, mel_rows, chunk_row, target_base, target_idx, refs, ref_index, B, st);
  LSG_LAUNCHED(ctx);
  LSG_LAUNCHED(ctx);
  run_all(h, mode, out, B, st);
}

}  // namespace gen
}  // namespace lsg
