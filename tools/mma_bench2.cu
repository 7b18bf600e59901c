// mma_bench2.cu -- cycles per tcgen05.mma.cta_group::2 (M=256 over an SM
// pair, operands resident in both CTAs' shared memory) vs N, to compare with
// the cta_group::1 floor measured by mma_bench.cu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2512_18318_b200/csrc -o mma_bench2 mma_bench2.cu
#include <cstdio>
#include <cstdint>

#include "tc.cuh"

using namespace lsg;

constexpr int SMEM = 100 * 1024;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) bench2(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cta_rank();
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(tc::smem_u32(&slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t a = tc::smem_u32(smem), b = a + 32768;
    const uint64_t da = tc::sdesc_sw128(a), db = tc::sdesc_sw128(b);
    constexpr uint32_t idesc = tc::idesc_f16kind(256, N, 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc)
            : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     tc::smem_u32(&bar)),
                 "h"((uint16_t)1)
                 : "memory");
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x / 2] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

template <int N>
void run() {
  const int pairs = 74;
  long long* d;
  cudaMalloc(&d, sizeof(long long) * pairs);
  cudaFuncSetAttribute(bench2<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const int iters = 4000;
  bench2<N><<<2 * pairs, 128, SMEM>>>(d, 10);
  bench2<N><<<2 * pairs, 128, SMEM>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[74];
  cudaMemcpy(h, d, sizeof(long long) * pairs, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < pairs; ++i) avg += h[i];
  avg /= pairs;
  const double per = avg / (iters * 4.0);
  const double ideal = 256.0 * N / 512.0;  // per SM: 128 rows x N at 2 B/cycle... floor formula, cta_group 2
  printf("cta_group::2 M=256 N=%3d: %7.1f cyc/MMA (floor %5.1f) -> %5.1f%% of pair tensor peak  %s\n", N, per, ideal,
         100.0 * ideal / per, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<32>();
  run<64>();
  run<128>();
  run<256>();
  return 0;
}
