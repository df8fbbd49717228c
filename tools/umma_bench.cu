// Microbenchmark (diagnostic, not product): tcgen05.mma issue/throughput on sm_100a for
// the shapes the output-layer kernel uses.  One CTA per SM, one thread issues `reps`
// back-to-back MMAs (M=128, K=16 bf16, accumulate) on fixed SMEM/TMEM operands and
// waits for completion via tcgen05.commit; cycles per MMA are reported.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_bench umma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N, uint32_t a_mn, uint32_t b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <int N, int TS, int BMN>
__global__ void __launch_bounds__(128, 1) bench(unsigned long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t id = idesc_bf16(128, N, 0, BMN);
    const uint64_t ad = sdesc(smem_u32(smem), 16, 1024);
    const uint64_t bd = BMN ? sdesc(smem_u32(smem) + 32768, 8192, 1024) : sdesc(smem_u32(smem) + 32768, 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (TS) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(tm),
                     "r"(tm + 256 + (r & 7) * 8), "l"(bd + (uint64_t)((r & 3) * 2)), "r"(id), "r"(1u), "r"(0u));
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                     "l"(ad + (uint64_t)((r & 3) * 2)), "l"(bd + (uint64_t)((r & 3) * 2)), "r"(id), "r"(1u));
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
    long long t2 = clock64();
    out[blockIdx.x * 2 + 0] = (unsigned long long)(t1 - t0);
    out[blockIdx.x * 2 + 1] = (unsigned long long)(t2 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int N, int TS, int BMN>
void run(const char* name, int ctas) {
  unsigned long long* d;
  cudaMalloc(&d, 2 * 148 * sizeof(unsigned long long));
  const int reps = 4096;
  cudaFuncSetAttribute(bench<N, TS, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  bench<N, TS, BMN><<<ctas, 128, 100 * 1024>>>(d, reps);
  cudaDeviceSynchronize();
  bench<N, TS, BMN><<<ctas, 128, 100 * 1024>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2 * 148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double issue = 0, total = 0;
  for (int i = 0; i < ctas; ++i) { issue += h[2 * i]; total += h[2 * i + 1]; }
  issue /= ctas; total /= ctas;
  const double macs = 128.0 * N * 16;
  printf("%-28s ctas=%3d  issue %.1f cyc/mma  complete %.1f cyc/mma  -> %.0f MAC/cyc/SM  (%s)\n", name, ctas,
         issue / reps, total / reps, macs * reps / total, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int ctas : {1, 148}) {
    run<64, 0, 0>("SS M128 N64  K-major", ctas);
    run<128, 0, 0>("SS M128 N128 K-major", ctas);
    run<256, 0, 0>("SS M128 N256 K-major", ctas);
    run<64, 1, 0>("TS M128 N64  K-major", ctas);
    run<128, 1, 0>("TS M128 N128 K-major", ctas);
    run<256, 1, 0>("TS M128 N256 K-major", ctas);
    run<256, 1, 1>("TS M128 N256 B MN-major", ctas);
    run<256, 0, 1>("SS M128 N256 B MN-major", ctas);
  }
  return 0;
}
