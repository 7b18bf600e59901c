// sync_bench.cu -- issue cost of the pipeline primitives on the MMA thread:
// mbarrier.try_wait on an already-completed phase, tcgen05.commit, and
// tcgen05.mma interleaved with each of them (N=64, operands resident).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2512_18318_b200/csrc -o sync_bench sync_bench.cu
#include <cstdio>
#include <cstdint>

#include "tc.cuh"

using namespace lsg;

template <int MODE>
__global__ void bench(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar[4];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) tc::mbar_init(&bar[i], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<256>(&slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    tc::mbar_arrive(&bar[0]);  // phase 0 of bar[0] complete: waits on parity 0 succeed at once
    const uint32_t a = tc::smem_u32(smem), b = a + 32768;
    const uint64_t da = tc::sdesc_sw128(a), db = tc::sdesc_sw128(b);
    constexpr uint32_t idesc = tc::idesc_f16kind(128, 64, 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if constexpr (MODE == 0) {  // 4 MMAs
#pragma unroll
        for (int k = 0; k < 4; ++k) tc::mma_f16_nc(tmem, da + 2 * k, db + 2 * k, idesc, 1);
      } else if constexpr (MODE == 1) {  // try_wait (complete) only
        tc::mbar_wait_nc(&bar[0], 0);
      } else if constexpr (MODE == 2) {  // commit only
        tc::mma_commit_nc(&bar[1]);
      } else if constexpr (MODE == 3) {  // wait + fence + 4 MMAs + commit (streamed-weight tap)
        tc::mbar_wait_nc(&bar[0], 0);
        tc::tc_fence_after_nc();
#pragma unroll
        for (int k = 0; k < 4; ++k) tc::mma_f16_nc(tmem, da + 2 * k, db + 2 * k, idesc, 1);
        tc::mma_commit_nc(&bar[1]);
      } else if constexpr (MODE == 4) {  // 4 MMAs + commit
#pragma unroll
        for (int k = 0; k < 4; ++k) tc::mma_f16_nc(tmem, da + 2 * k, db + 2 * k, idesc, 1);
        tc::mma_commit_nc(&bar[1]);
      } else if constexpr (MODE == 5) {  // wait + fence + 4 MMAs
        tc::mbar_wait_nc(&bar[0], 0);
        tc::tc_fence_after_nc();
#pragma unroll
        for (int k = 0; k < 4; ++k) tc::mma_f16_nc(tmem, da + 2 * k, db + 2 * k, idesc, 1);
      } else if constexpr (MODE == 6) {  // wait + 4 MMAs (no fence)
        tc::mbar_wait_nc(&bar[0], 0);
#pragma unroll
        for (int k = 0; k < 4; ++k) tc::mma_f16_nc(tmem, da + 2 * k, db + 2 * k, idesc, 1);
      } else if constexpr (MODE == 7) {  // fence + 4 MMAs
        tc::tc_fence_after_nc();
#pragma unroll
        for (int k = 0; k < 4; ++k) tc::mma_f16_nc(tmem, da + 2 * k, db + 2 * k, idesc, 1);
      } else if constexpr (MODE == 8) {  // test_wait (non-blocking probe) + 4 MMAs
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(tc::smem_u32(&bar[0])), "r"(0u));
        if (ok) {
#pragma unroll
          for (int k = 0; k < 4; ++k) tc::mma_f16_nc(tmem, da + 2 * k, db + 2 * k, idesc, 1);
        }
      } else if constexpr (MODE == 9) {  // wait + 4 MMAs + commit (no fence)
        tc::mbar_wait_nc(&bar[0], 0);
#pragma unroll
        for (int k = 0; k < 4; ++k) tc::mma_f16_nc(tmem, da + 2 * k, db + 2 * k, idesc, 1);
        tc::mma_commit_nc(&bar[1]);
      } else {  // 8 MMAs per wait (no fence)
        tc::mbar_wait_nc(&bar[0], 0);
#pragma unroll
        for (int k = 0; k < 8; ++k) tc::mma_f16_nc(tmem, da + 2 * (k & 3), db + 2 * (k & 3), idesc, 1);
      }
    }
    tc::mma_commit_nc(&bar[2]);
    tc::mbar_wait(&bar[2], 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<256>(tmem);
  }
}

template <int MODE>
void run(const char* what) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 148);
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int iters = 4000;
  bench<MODE><<<148, 128, 96 * 1024>>>(d, 10);
  bench<MODE><<<148, 128, 96 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%-44s %8.1f cycles / iteration  %s\n", what, avg / iters, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("4 x mma N=64");
  run<1>("mbarrier try_wait (phase complete)");
  run<2>("tcgen05.commit");
  run<3>("wait + fence + 4 x mma + commit");
  run<4>("4 x mma + commit");
  run<5>("wait + fence + 4 x mma");
  run<6>("wait + 4 x mma (no fence)");
  run<7>("fence + 4 x mma");
  run<8>("test_wait + 4 x mma");
  run<9>("wait + 4 x mma + commit (no fence)");
  run<10>("wait + 8 x mma (no fence)");
  return 0;
}
