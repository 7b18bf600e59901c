// face.cu -- face-crop preparation on sm_100a (include/lsg.h "face";
// SURVEY.md §8 row f1).
//
// The generator's missing upstream: per segment, the gathered frames'
// detector boxes (the frame's own box, or mock_face_detect,
// visual_mocks.cpp:10-22) go through KalmanBoxFilter::update
// (kalman.cpp:58-144) exactly as orchestrator.cpp:115-129 /
// runner.cpp:134-141 do, then each frame is cropped to the smoothed box and
// resampled to the generator's 96x96 input.
//   track   one thread per segment (the filter is a sequential recurrence
//           over the segment's frames; segments are independent).  Every
//           fp64 operation is a round-to-nearest intrinsic in the reference's
//           order (no FMA contraction, as its x86-64 build), so boxes and
//           velocities are bit-identical to the reference's.
//   crop    one thread per output pixel: bilinear resample of the box into
//           96x96 (source x = cx - w/2 + (u + 0.5) w / 96 - 0.5, clamp to
//           the frame, round half up) -- our semantics: the reference
//           carries no pixels, so the crop is pinned to the C restatement
//           (oracle or_crop96), not to reference output.
#include <algorithm>
#include <cmath>
#include <vector>

#include "lsg_common.cuh"

namespace lsg {
namespace face {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t& s) {  // rng.hpp:14-19
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix_u64(uint64_t h, uint64_t v) {  // rng.hpp:21-25
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  uint64_t s = h;
  return splitmix64(s);
}
// mock_face_detect (visual_mocks.cpp:10-22)
__host__ __device__ __forceinline__ void mock_detect(int64_t frame_index, uint64_t seed, double* z) {
  const char tag[] = "facedetect";
  uint64_t h = seed;
  for (int i = 0; i < 10; ++i) h = mix_u64(h, (uint8_t)tag[i]);
  h = mix_u64(h, (uint64_t)frame_index);
  z[0] = 320.0 + ((double)(splitmix64(h) % 7) - 3.0);
  z[1] = 240.0 + ((double)(splitmix64(h) % 7) - 3.0);
  z[2] = 160.0;
  z[3] = 200.0;
}

#define DM __dmul_rn
#define DA __dadd_rn
#define DS __dsub_rn
#define DD __ddiv_rn

struct Kf {
  double x[6], p[6][6];
};

// kalman.cpp:58-77
__device__ void predict(Kf& f, double dt, double pn) {
  f.x[0] = DA(f.x[0], DM(f.x[4], dt));
  f.x[1] = DA(f.x[1], DM(f.x[5], dt));
  double fp[6][6];
  for (int j = 0; j < 6; ++j) {
    for (int i = 0; i < 6; ++i) fp[i][j] = f.p[i][j];
    fp[0][j] = DA(fp[0][j], DM(dt, f.p[4][j]));
    fp[1][j] = DA(fp[1][j], DM(dt, f.p[5][j]));
  }
  for (int i = 0; i < 6; ++i) {
    for (int j = 0; j < 6; ++j) f.p[i][j] = fp[i][j];
    f.p[i][0] = DA(f.p[i][0], DM(dt, fp[i][4]));
    f.p[i][1] = DA(f.p[i][1], DM(dt, fp[i][5]));
  }
  const double q = DM(pn, dt);
  for (int i = 0; i < 6; ++i) f.p[i][i] = DA(f.p[i][i], q);
}

// kalman.cpp:16-49
__device__ bool chol4(const double a[4][4], double l[4][4]) {
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) l[i][j] = 0.0;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j <= i; ++j) {
      double sum = a[i][j];
      for (int k = 0; k < j; ++k) sum = DS(sum, DM(l[i][k], l[j][k]));
      if (i == j) {
        if (sum <= 0.0 || !isfinite(sum)) return false;
        l[i][i] = __dsqrt_rn(sum);
      } else {
        l[i][j] = DD(sum, l[j][j]);
      }
    }
  return true;
}
__device__ void chol_solve4(const double l[4][4], const double b[4], double x[4]) {
  double y[4];
  for (int i = 0; i < 4; ++i) {
    double sum = b[i];
    for (int k = 0; k < i; ++k) sum = DS(sum, DM(l[i][k], y[k]));
    y[i] = DD(sum, l[i][i]);
  }
  for (int i = 3; i >= 0; --i) {
    double sum = y[i];
    for (int k = i + 1; k < 4; ++k) sum = DS(sum, DM(l[k][i], x[k]));
    x[i] = DD(sum, l[i][i]);
  }
}

// kalman.cpp:79-135: 0 ok, -1 what the reference throws on
__device__ int update(Kf& f, bool& init, const double z[4], double dt, const lsg_kalman_cfg& c) {
  for (int i = 0; i < 4; ++i)
    if (!isfinite(z[i])) return -1;
  if (!init) {
    for (int i = 0; i < 4; ++i) f.x[i] = z[i];
    f.x[4] = f.x[5] = 0.0;
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) f.p[i][j] = i == j ? c.initial_variance : 0.0;
    init = true;
    return 0;
  }
  if (dt < 0 || !isfinite(dt)) return -1;
  predict(f, dt, c.process_noise);
  double s[4][4], l[4][4], k[6][4];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) s[i][j] = DA(f.p[i][j], i == j ? c.measurement_noise : 0.0);
  if (!chol4(s, l)) return -1;
  for (int i = 0; i < 6; ++i) {
    double row[4], sol[4];
    for (int j = 0; j < 4; ++j) row[j] = f.p[i][j];
    chol_solve4(l, row, sol);
    for (int j = 0; j < 4; ++j) k[i][j] = sol[j];
  }
  double y[4];
  for (int i = 0; i < 4; ++i) y[i] = DS(z[i], f.x[i]);
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 4; ++j) f.x[i] = DA(f.x[i], DM(k[i][j], y[j]));
  double ikh[6][6], tmp[6][6];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) ikh[i][j] = DS(i == j ? 1.0 : 0.0, j < 4 ? k[i][j] : 0.0);
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      double acc = 0.0;
      for (int m = 0; m < 6; ++m) acc = DA(acc, DM(ikh[i][m], f.p[m][j]));
      tmp[i][j] = acc;
    }
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      double acc = 0.0;
      for (int m = 0; m < 6; ++m) acc = DA(acc, DM(tmp[i][m], ikh[j][m]));
      for (int m = 0; m < 4; ++m) acc = DA(acc, DM(DM(k[i][m], c.measurement_noise), k[j][m]));
      f.p[i][j] = acc;
    }
  return 0;
}

// tab: [n] seg_off | [n] seg_len
__global__ void track_kernel(const int64_t* __restrict__ tab, int n, const int64_t* __restrict__ ts,
                             const int64_t* __restrict__ frame_index, const int32_t* __restrict__ has_face,
                             const double* __restrict__ faces, uint64_t seed, lsg_kalman_cfg cfg,
                             double* __restrict__ out_box, double* __restrict__ out_vel, int32_t* __restrict__ status) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t off = tab[s], len = tab[n + s];
  Kf f;
  bool init = false;
  int64_t prev = 0;
  int rc = 0;
  for (int64_t i = off; i < off + len && rc == 0; ++i) {
    double z[4];
    if (has_face && has_face[i]) {
      for (int c = 0; c < 4; ++c) z[c] = faces[4 * i + c];
    } else {
      mock_detect(frame_index[i], seed, z);
    }
    const double dt = init ? DD((double)(ts[i] - prev), 1000.0) : 0.0;
    rc = update(f, init, z, dt, cfg);
    if (rc) break;
    for (int c = 0; c < 4; ++c) out_box[4 * i + c] = f.x[c];
    if (out_vel) {
      out_vel[2 * i] = f.x[4];
      out_vel[2 * i + 1] = f.x[5];
    }
    prev = ts[i];
  }
  status[s] = rc;
}

// one thread per (crop, output pixel); 3 channels each
__global__ void crop_kernel(const uint8_t* __restrict__ frames, int H, int W, const int64_t* __restrict__ frame_of,
                            const double* __restrict__ boxes, int n, uint8_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * 96 * 96) return;
  const int64_t k = i / (96 * 96);
  const int uv = (int)(i - k * 96 * 96), v = uv / 96, u = uv - v * 96;
  const double* b = boxes + 4 * k;
  const double x0 = DS(b[0], DM(0.5, b[2])), y0 = DS(b[1], DM(0.5, b[3]));
  const double sx = DD(b[2], 96.0), sy = DD(b[3], 96.0);
  double fx = DS(DA(x0, DM(u + 0.5, sx)), 0.5), fy = DS(DA(y0, DM(v + 0.5, sy)), 0.5);
  fx = fx < 0 ? 0 : (fx > W - 1 ? W - 1 : fx);
  fy = fy < 0 ? 0 : (fy > H - 1 ? H - 1 : fy);
  const int ix = (int)fx < W - 1 ? (int)fx : W - 2, iy = (int)fy < H - 1 ? (int)fy : H - 2;
  const double ax = DS(fx, (double)ix), ay = DS(fy, (double)iy);
  const uint8_t* f = frames + frame_of[k] * (int64_t)H * W * 3;
  const uint8_t* r0 = f + ((int64_t)iy * W + ix) * 3;
  const uint8_t* r1 = r0 + (int64_t)W * 3;
  uint8_t* o = out + i * 3;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double p00 = r0[c], p01 = r0[3 + c], p10 = r1[c], p11 = r1[3 + c];
    const double top = DA(p00, DM(ax, DS(p01, p00)));
    const double bot = DA(p10, DM(ax, DS(p11, p10)));
    const double val = DA(top, DM(ay, DS(bot, top)));
    o[c] = (uint8_t)DA(val, 0.5);
  }
}

#undef DM
#undef DA
#undef DS
#undef DD

}  // namespace face
}  // namespace lsg

using namespace lsg;

extern "C" {

lsg_status lsg_kalman_cfg_default(lsg_kalman_cfg* c) {
  return guard(__func__, [&] {  // kalman.hpp:8-12
    c->process_noise = 1e-2;
    c->measurement_noise = 25.0;
    c->initial_variance = 1e6;
  });
}

lsg_status lsg_face_mock_detect(int64_t frame_index, uint64_t seed, double* box4) {
  return guard(__func__, [&] { face::mock_detect(frame_index, seed, box4); });
}

lsg_status lsg_face_track(lsg_ctx ctx, int32_t n, const int64_t* seg_off, const int64_t* seg_len, const int64_t* ts,
                          const int64_t* frame_index, const int32_t* has_face, const double* faces, uint64_t seed,
                          const lsg_kalman_cfg* cfg, double* out_box, double* out_vel, int32_t* status) {
  return guard(__func__, [&] {
    if (cfg->process_noise <= 0 || cfg->measurement_noise <= 0 || cfg->initial_variance <= 0)
      invalid("kalman: non-positive noise");  // kalman.cpp:52-55
    if (n < 0) invalid("lsg_face_track: negative count");
    if (n == 0) return;
    if (has_face && !faces) invalid("lsg_face_track: has_face without faces");
    std::vector<int64_t> tab(2 * (size_t)n);
    for (int i = 0; i < n; ++i) {
      if (seg_len[i] < 0) invalid("lsg_face_track: negative segment length");
      tab[i] = seg_off[i];
      tab[n + i] = seg_len[i];
    }
    DeviceGuard g(ctx);
    ScratchLease sc(ctx, tab.size() * 8 + (size_t)n * 4);
    int64_t* dtab = static_cast<int64_t*>(sc.p);
    int32_t* dst = reinterpret_cast<int32_t*>(dtab + tab.size());
    LSG_CUDA(cudaMemcpyAsync(dtab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    face::track_kernel<<<(unsigned)ceil_div(n, 64), 64, 0, ctx->stream>>>(dtab, n, ts, frame_index, has_face, faces,
                                                                          seed, *cfg, out_box, out_vel, dst);
    LSG_LAUNCHED(ctx);
    LSG_CUDA(cudaMemcpyAsync(status, dst, (size_t)n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  });
}

lsg_status lsg_face_crop(lsg_ctx ctx, int32_t n, const uint8_t* frames, int32_t H, int32_t W, const int64_t* frame_of,
                         const double* boxes, uint8_t* out) {
  return guard(__func__, [&] {
    if (n < 0) invalid("lsg_face_crop: negative count");
    if (H < 2 || W < 2) invalid("lsg_face_crop: frame smaller than 2x2");
    if (n == 0) return;
    DeviceGuard g(ctx);
    const int64_t total = (int64_t)n * 96 * 96;
    face::crop_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, ctx->stream>>>(frames, H, W, frame_of, boxes, n, out);
    LSG_LAUNCHED(ctx);
  });
}

}  // extern "C"
