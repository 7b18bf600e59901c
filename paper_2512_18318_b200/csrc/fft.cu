// fft_radix2 (mel.cpp:46-70, mel.hpp:42) as a device transform.
//
// The reference's in-place radix-2 decimation-in-time FFT, bit for bit: the
// same bit-reversal permutation, the same stage order and, per stage, the
// reference's twiddle recurrence w_{k+1} = w_k * wlen with
// wlen = (cos(-2 pi / len), sin(-2 pi / len)).  The twiddle tables are that
// recurrence evaluated on the host in IEEE double (exactly the reference's
// operation sequence, libm cos/sin), so every butterfly input is the
// reference's; the butterflies themselves use round-to-nearest intrinsics so
// nvcc cannot contract (ac - bd) into an FMA that x86-64 -O2 does not form.
// One CTA per transform; the transform and its twiddles live in shared memory.
#include <cmath>
#include <complex>
#include <vector>

#include "lsg_common.cuh"

namespace lsg {
namespace fft {

constexpr double kPi = 3.14159265358979323846;  // mel.cpp's kPi
constexpr int kMaxLog2 = 13;                    // 8192 points: 128 KB + 64 KB of twiddles

__global__ void __launch_bounds__(512) radix2_kernel(double2* __restrict__ data, const double2* __restrict__ tw,
                                                     int log2n) {
  extern __shared__ double2 sm[];
  const int n = 1 << log2n;
  double2* x = sm;
  double2* w = sm + n;
  double2* g = data + (size_t)blockIdx.x * n;
  // bit-reversal permutation (the reference's swap loop is exactly i <-> rev(i))
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[__brev(i) >> (32 - log2n)] = g[i];
  __syncthreads();
  // per-stage twiddles packed back to back: stage len uses tw[len/2 - 1 + k]
  for (int len = 2, s = 0; len <= n; len <<= 1, ++s) {
    const int half = len >> 1;
    for (int k = threadIdx.x; k < half; k += blockDim.x) w[k] = tw[half - 1 + k];
    __syncthreads();
    for (int b = threadIdx.x; b < n / 2; b += blockDim.x) {
      const int blk = b / half, k = b - blk * half;
      const int i0 = blk * len + k, i1 = i0 + half;
      const double2 u = x[i0], a = x[i1], t = w[k];
      // v = a * t, std::complex<double> multiply: (ar tr - ai ti, ar ti + ai tr)
      const double vr = __dsub_rn(__dmul_rn(a.x, t.x), __dmul_rn(a.y, t.y));
      const double vi = __dadd_rn(__dmul_rn(a.x, t.y), __dmul_rn(a.y, t.x));
      x[i0] = make_double2(__dadd_rn(u.x, vr), __dadd_rn(u.y, vi));
      x[i1] = make_double2(__dsub_rn(u.x, vr), __dsub_rn(u.y, vi));
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) g[i] = x[i];
}

// Twiddles of every stage, the reference's recurrence on the host.
static std::vector<double2> twiddles(int log2n) {
  const size_t n = size_t(1) << log2n;
  std::vector<double2> t(n - 1);
  for (size_t len = 2; len <= n; len <<= 1) {
    const double ang = -2.0 * kPi / double(len);
    const std::complex<double> wlen(std::cos(ang), std::sin(ang));
    std::complex<double> w(1.0, 0.0);
    for (size_t k = 0; k < len / 2; ++k) {
      t[len / 2 - 1 + k] = make_double2(w.real(), w.imag());
      w *= wlen;
    }
  }
  return t;
}

}  // namespace fft
}  // namespace lsg

using namespace lsg;

extern "C" lsg_status lsg_fft_radix2(lsg_ctx ctx, double* data, int64_t n, int32_t count) {
  return guard(__func__, [&] {
    if (n <= 0 || (n & (n - 1)) != 0) invalid("fft: size must be a power of two");  // mel.cpp:48-49
    if (count < 0) invalid("lsg_fft_radix2: negative count");
    int log2n = 0;
    while ((int64_t(1) << log2n) < n) ++log2n;
    if (log2n > fft::kMaxLog2) invalid("lsg_fft_radix2: size above 8192 points");
    if (count == 0 || n == 1) return;  // a 1-point transform is the identity
    DeviceGuard g(ctx);
    const std::vector<double2> tw = fft::twiddles(log2n);
    const bool dev = is_device_ptr(data);
    // host data goes through the context scratch in batches of <= 32 MiB
    const int64_t per = dev ? count : std::max<int64_t>(1, (int64_t(32) << 20) / (n * (int64_t)sizeof(double2)));
    const size_t bytes = size_t(n) * std::min<int64_t>(per, count) * sizeof(double2);
    ScratchLease sc(ctx, tw.size() * sizeof(double2) + (dev ? 0 : bytes));
    double2* dtw = static_cast<double2*>(sc.p);
    LSG_CUDA(cudaMemcpyAsync(dtw, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
    const size_t smem = size_t(n) * sizeof(double2) * 3 / 2;
    if (smem > 48 * 1024)
      LSG_CUDA(cudaFuncSetAttribute(fft::radix2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int64_t c0 = 0; c0 < count; c0 += per) {
      const int64_t cn = std::min<int64_t>(per, count - c0);
      double2* host = reinterpret_cast<double2*>(data) + c0 * n;
      double2* buf = dev ? host : dtw + tw.size();
      if (!dev) LSG_CUDA(cudaMemcpyAsync(buf, host, size_t(n) * cn * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
      fft::radix2_kernel<<<(unsigned)cn, (unsigned)std::min<int64_t>(512, std::max<int64_t>(32, n / 2)), smem,
                           ctx->stream>>>(buf, dtw, log2n);
      LSG_LAUNCHED(ctx);
      if (!dev)
        LSG_CUDA(cudaMemcpyAsync(host, buf, size_t(n) * cn * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    }
    ctx->sync();  // the twiddle table lives in the context scratch
  });
}
