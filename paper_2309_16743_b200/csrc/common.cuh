// Shared device helpers for libmel (sm_100a).  Product code: nothing here is
// shared with the CPU oracle (independent numpy), per DESIGN.md "Boundary".
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <utility>

namespace mel {

// ---- Philox4x32-10 (Salmon et al., SC'11), stream layout of DESIGN.md ---------
// key = (lo32(seed), hi32(seed)), counter = (lo32(n), hi32(n), c2, tag)
enum : uint32_t { TAG_SAMPLE = 1, TAG_EVICT = 2, TAG_DRAIN = 3, TAG_INIT = 4 };

__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

__host__ __device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t hi0 = mulhi32(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// one 64-bit draw per counter value n: r64 = (o1 << 32) | o0
__host__ __device__ __forceinline__ uint64_t philox_r64(uint64_t seed, uint32_t tag, uint64_t n, uint32_t c2) {
  const uint4 o = philox4x32_10(make_uint4((uint32_t)n, (uint32_t)(n >> 32), c2, tag),
                                (uint32_t)seed, (uint32_t)(seed >> 32));
  return ((uint64_t)o.y << 32) | o.x;
}

// floor(r * n / 2^64): no rejection, consumption is one counter per draw
__host__ __device__ __forceinline__ uint32_t bounded(uint64_t r, uint32_t n) {
#ifdef __CUDA_ARCH__
  return (uint32_t)__umul64hi(r, (uint64_t)n);
#else
  return (uint32_t)(((unsigned __int128)r * n) >> 64);
#endif
}

__host__ __device__ __forceinline__ double unit_double(uint64_t r) {
  return (double)(r >> 11) * 0x1.0p-53;
}

// ---- numerics -----------------------------------------------------------------------
__device__ __forceinline__ float normalise_rn(float u, float lo, float span) {
  // RN_f32((u - lo) / span), each op correctly rounded (no fast-math contraction)
  return __fdiv_rn(__fsub_rn(u, lo), span);
}

// One Adam element in the PyTorch form (the step scalars from StepDev):
//   m' = b1 m + (1 - b1) g,  v' = b2 v + (1 - b2) g^2,  p' = p - step m' / (sqrt(v') isc2 + eps)
// with step = lr / (1 - b1^k) and isc2 = 1 / sqrt(1 - b2^k).  The square root and the
// division use the SFU (sqrt.approx, rcp.approx: a few ulp, reading R26); the separate Adam
// kernel and the one fused into K1 call this same function, so they agree bit for bit.  An
// element whose new second moment would not be finite (a non-finite gradient or one whose
// square overflows) keeps p, m, v (include/mel.h surrogate_step).
__device__ __forceinline__ void adam_elem(float& p, float& m, float& v, float g, float scale, float step, float isc2,
                                          float b1, float b2, float eps) {
  const float gr = g * scale;
  const float nv = fmaf(b2, v, (1.f - b2) * gr * gr);
  if (!(nv < __int_as_float(0x7f800000))) return;
  const float nm = fmaf(b1, m, (1.f - b1) * gr);
  float s, r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(nv));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaf(s, isc2, eps)));
  p = fmaf(-step, nm * r, p);
  m = nm;
  v = nv;
}

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t h) {
  return __uint_as_float(((uint32_t)h) << 16);
}

}  // namespace mel

// Programmatic dependent launch: every library kernel starts with pdl_enter() -- wait for
// the preceding kernel in the stream to complete (its writes visible), then let the next
// kernel's CTAs be scheduled on SMs as this grid's last CTAs retire -- and is launched with
// launch_pdl, so a kernel's launch and prologue overlap its predecessor's tail without
// changing stream semantics (griddepcontrol.wait is a no-op without the attribute).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
