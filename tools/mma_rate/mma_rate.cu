// Microbenchmark: tcgen05.mma kind::f16 (bf16 -> fp32) issue throughput per SM for
// M = 128 and N = 64 / 128 / 256, both operands from SMEM (SS, K-major SW128), one CTA per
// SM, back-to-back MMAs into one TMEM accumulator.  Prints cycles per MMA and flop/cycle/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu && ./mma_rate
#include <cstdint>
#include <cstdio>
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
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <int N>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (64 + 64) * 1024 / 4; i += 128) ((uint32_t*)smem)[i] = 0;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 64 * 1024;
    const uint32_t id = idesc_bf16(128, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t kk = i & 3;                       // K16 steps inside one 64-k SW128 box
      const uint64_t ad = sdesc(sa + kk * 32, 16, 1024), bd = sdesc(sb + kk * 32, 16, 1024);
      const uint32_t acc = i > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                   "l"(ad), "l"(bd), "r"(id), "r"(acc) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    out[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

template <int N>
void run(int sms) {
  const int iters = 8192;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = 128 * 1024 + 1024;
  cudaFuncSetAttribute(mma_rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate<N><<<sms, 128, smem>>>(iters, d);   // warm-up
  mma_rate<N><<<sms, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256] = {};
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double cyc = (double)mx / iters, flop = 2.0 * 128 * N * 16;
  printf("M128 N%-3d K16 SS: %s  %.1f cycles/MMA  %.0f flop/cycle/SM\n", N, cudaGetErrorString(e), cyc, flop / cyc);
  cudaFree(d);
}


// K1's MMA mix per 64-row chunk: 16 forward M128 N64 K16 (SS) into a 64-column accumulator,
// then 4 dW M128 N256 K16 with A from TMEM (TS) into a 256-column accumulator
__global__ void __launch_bounds__(128, 1) mma_mix(int chunks, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (64 + 64) * 1024 / 4; i += 128) ((uint32_t*)smem)[i] = 0;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 64 * 1024;
    const uint32_t id_f = idesc_bf16(128, 64), id_d = idesc_bf16(128, 256) | (1u << 16);   // dW: B MN-major
    long long t0 = clock64();
    for (int c = 0; c < chunks; ++c) {
      const uint32_t yb = (c & 3) * 64;
      for (int kk = 0; kk < 16; ++kk) {
        const uint64_t ad = sdesc(sa + (kk & 3) * 32 + (kk >> 2) * 16384, 16, 1024);
        const uint64_t bd = sdesc(sb + (kk & 3) * 32 + (kk >> 2) * 8192, 16, 1024);
        const uint32_t acc = kk > 0;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + yb),
                     "l"(ad), "l"(bd), "r"(id_f), "r"(acc) : "memory");
      }
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t bd = sdesc(sb + kk * 2048, 8192, 1024);
        const uint32_t acc = (c > 0 || kk > 0);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(tm + 256),
                     "r"(tm + ((c + 3) & 3) * 64 + kk * 8), "l"(bd), "r"(id_d), "r"(acc), "r"(0u) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    out[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

void run_mix(int sms) {
  const int chunks = 512;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = 128 * 1024 + 1024;
  cudaFuncSetAttribute(mma_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_mix<<<sms, 128, smem>>>(chunks, d);
  mma_mix<<<sms, 128, smem>>>(chunks, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256] = {};
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("K1 chunk mix (16 x N64 SS + 4 x N256 TS): %s  %.0f cycles/chunk (isolated rates: 1280)\n",
         cudaGetErrorString(e), (double)mx / chunks);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64>(sms);
  run<128>(sms);
  run<256>(sms);
  run_mix(sms);
  return 0;
}
