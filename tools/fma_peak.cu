// fma_peak.cu -- measured FP32 / FP64 CUDA-core FMA throughput (the mel
// kernel's roofline denominators; MEASURED_PEAKS.json carries only HBM and
// bf16 tensor peaks).  8 independent FMA chains per thread, all SMs, CUDA
// events, best of 5.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_peak fma_peak.cu
#include <cstdio>

template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b);
      x1 = fma(x1, a, b);
      x2 = fma(x2, a, b);
      x3 = fma(x3, a, b);
      x4 = fma(x4, a, b);
      x5 = fma(x5, a, b);
      x6 = fma(x6, a, b);
      x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

template <typename T>
double run(const char* name, int sms) {
  const int blocks = sms * 8, threads = 256, iters = 4096;
  T* out;
  cudaMalloc(&out, sizeof(T) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_loop<T><<<blocks, threads>>>(out, 16, (T)0.999, (T)0.001);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  const double tf = flops / (best * 1e-3) / 1e12;
  printf("{\"dtype\": \"%s\", \"tflops\": %.2f, \"ms\": %.3f, \"blocks\": %d, \"threads\": %d}\n", name, tf, best, blocks,
         threads);
  cudaFree(out);
  return tf;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<float>("fp32", sms);
  run<double>("fp64", sms);
  return 0;
}
