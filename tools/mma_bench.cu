// mma_bench.cu -- cycles per tcgen05.mma (kind::f16, cta_group::1, SS) as a
// function of M, N, the A-operand layout and concurrent shared-memory fill
// traffic.  Used to find what bounds the narrow-N conv layers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2512_18318_b200/csrc -o mma_bench mma_bench.cu
// modes: 0 SW128 A fixed | 1 SW128 A cycling over 4 stages | 2 no-swizzle A
//        3 = 1 + bulk-copy fill traffic from L2 into a separate region
//        4 no-swizzle, SBO 160 (halo patch rows), start +16 B (shifted tap)
//        5 no-swizzle, SBO 160, 128-aligned start | 6 no-swizzle, SBO 128, start +16 B
// bench_coll: groups of 4 MMAs sharing one A (halo-patch descriptor) with 4
// different B blocks -- the ConvT phases of one input shift -- without and
// with the A collector (.collector::a::fill / use / lastuse).
#include <cstdio>
#include <cstdint>

#include "tc.cuh"

using namespace lsg;

__device__ __forceinline__ uint64_t desc_noswz(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

constexpr int SMEM = 200 * 1024;

template <int M, int N, int mode>
__global__ void bench(long long* out, int iters, const uint8_t* src, unsigned long long* fill_bytes) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar, fbar[2];
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 128 * 1024; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&fbar[0], 1);
    tc::mbar_init(&fbar[1], 1);
    tc::fence_mbar_init();
    done = 0;
  }
  if (warp == 0) tc::tmem_alloc<256>(&slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t base = tc::smem_u32(smem);
  if (threadIdx.x == 0) {
    const uint32_t b = base + 65536;
    const uint64_t db = tc::sdesc_sw128(b);
    constexpr uint32_t idesc = tc::idesc_f16kind(M, N, 0);
    // descriptor of K step 0 and the per-step increment (16-byte units)
    uint64_t da0;
    uint64_t kstep;
    if constexpr (mode == 2) {
      da0 = desc_noswz(base, 2048, 128);
      kstep = 4096 >> 4;
    } else if constexpr (mode == 4) {
      da0 = desc_noswz(base + 16, 2944, 160);
      kstep = 5888 >> 4;
    } else if constexpr (mode == 5) {
      da0 = desc_noswz(base, 2944, 160);
      kstep = 5888 >> 4;
    } else if constexpr (mode == 6) {
      da0 = desc_noswz(base + 16, 2048, 128);
      kstep = 4096 >> 4;
    } else {
      da0 = tc::sdesc_sw128(base);
      kstep = 2;
    }
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t da = da0 + (mode == 1 || mode == 3 ? (uint64_t)((i & 3) * (16384 >> 4)) : 0ull);
#pragma unroll
      for (int k = 0; k < 4; ++k) tc::mma_f16(tmem, da + k * kstep, db + 2 * k, idesc, 1);
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    done = 1;
  } else if (warp == 1 && mode == 3 && lane == 0) {
    // keep two 32 KB bulk copies in flight into [96K, 160K)
    unsigned long long bytes = 0;
    uint32_t ph[2] = {0, 0};
    int s = 0;
    const uint8_t* g = src + (size_t)blockIdx.x * 65536;
    tc::mbar_arrive_expect_tx(&fbar[0], 32768);
    tc::bulk_g2s(base + 98304, g, 32768, &fbar[0]);
    tc::mbar_arrive_expect_tx(&fbar[1], 32768);
    tc::bulk_g2s(base + 98304 + 32768, g + 32768, 32768, &fbar[1]);
    while (!done) {
      tc::mbar_wait(&fbar[s], ph[s]);
      ph[s] ^= 1;
      bytes += 32768;
      tc::mbar_arrive_expect_tx(&fbar[s], 32768);
      tc::bulk_g2s(base + 98304 + s * 32768, g + s * 32768, 32768, &fbar[s]);
      s ^= 1;
    }
    tc::mbar_wait(&fbar[0], ph[0]);
    tc::mbar_wait(&fbar[1], ph[1]);
    fill_bytes[blockIdx.x] = bytes;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<256>(tmem);
  }
}

__device__ __forceinline__ void mma_coll(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, int c) {
  if (c == 0)
    asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b),
                 "r"(idesc));
  else if (c == 1)
    asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::use [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b),
                 "r"(idesc));
  else
    asm volatile("tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a),
                 "l"(b), "r"(idesc));
}

template <int N, int G, bool COLL>
__global__ void bench_coll(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 128 * 1024; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<256>(&slot);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t base = tc::smem_u32(smem);
  if (threadIdx.x == 0) {
    const uint64_t db0 = tc::sdesc_sw128(base + 65536);
    constexpr uint32_t idesc = tc::idesc_f16kind(128, N, 0);
    const uint64_t da0 = desc_noswz(base + 16, 2944, 160);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t da = da0 + (uint64_t)((i & 3) * (5888 >> 4));
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint64_t db = db0 + (uint64_t)(g * (N * 128 >> 4));  // B block g (N rows x 128 B)
        if constexpr (COLL) mma_coll(tmem + (g & 3) * 64 % 256, da, db, idesc, g == 0 ? 0 : (g == G - 1 ? 2 : 1));
        else tc::mma_f16(tmem + (g & 3) * 64 % 256, da, db, idesc, 1);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<256>(tmem);
  }
}

template <int N, int G, bool COLL>
void run_coll(int blocks) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * blocks);
  cudaFuncSetAttribute(bench_coll<N, G, COLL>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const int iters = 4000;
  bench_coll<N, G, COLL><<<blocks, 128, SMEM>>>(d, 10);
  bench_coll<N, G, COLL><<<blocks, 128, SMEM>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  printf("A shared by %d MMAs, N=%3d, collector %d: %7.1f cyc/MMA (ideal %5.1f)  %s\n", G, N, (int)COLL,
         avg / (iters * (double)G), 128 * N / 256.0, cudaGetErrorString(e));
  cudaFree(d);
}

static uint8_t* g_src;
static unsigned long long* g_fill;

template <int M, int N, int mode>
void run(int blocks) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * blocks);
  cudaMemset(g_fill, 0, sizeof(unsigned long long) * 148);
  cudaFuncSetAttribute(bench<M, N, mode>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const int iters = 4000;
  bench<M, N, mode><<<blocks, 128, SMEM>>>(d, 10, g_src, g_fill);
  bench<M, N, mode><<<blocks, 128, SMEM>>>(d, iters, g_src, g_fill);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  unsigned long long f[148];
  cudaMemcpy(h, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  cudaMemcpy(f, g_fill, sizeof(unsigned long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0, fb = 0;
  for (int i = 0; i < blocks; ++i) {
    avg += h[i];
    fb += f[i];
  }
  avg /= blocks;
  fb /= blocks;
  const double per = avg / (iters * 4.0);
  const double ideal = (M < 128 ? 128 : M) * N / 256.0;
  printf("mode %d M=%3d N=%3d blocks=%3d: %7.1f cyc/MMA (ideal %5.1f) %5.1f%% | fill %.1f B/cyc  %s\n", mode, M, N,
         blocks, per, ideal, 100.0 * ideal / per * (M == 64 ? 0.5 : 1.0), fb / avg, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  cudaMalloc(&g_src, 148 * 65536);
  cudaMemset(g_src, 1, 148 * 65536);
  cudaMalloc(&g_fill, sizeof(unsigned long long) * 148);
#define RUN(MODE)            \
  run<128, 32, MODE>(148);   \
  run<128, 64, MODE>(148);   \
  run<128, 128, MODE>(148);  \
  run<128, 256, MODE>(148);
  RUN(0)
  RUN(1)
  RUN(2)
  RUN(3)
  RUN(4)
  RUN(5)
  RUN(6)
  run_coll<64, 4, false>(148);
  run_coll<64, 4, true>(148);
  run_coll<64, 2, false>(148);
  run_coll<64, 2, true>(148);
  run_coll<128, 4, false>(148);
  run_coll<128, 4, true>(148);
  return 0;
}
