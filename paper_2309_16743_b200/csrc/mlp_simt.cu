// SIMT (FFMA) kernels of the surrogate trainer: the head layers (6 -> 256 ->
// 256, 0.03% of the step FLOPs at paper shape), the fp32 parity mode of
// the output layer, deterministic reductions, Adam and Philox
// init.  The tensor-core output layer (bf16 mode) lives in tc_out.cu.
#include "common.cuh"
#include "kernels.h"

namespace mel {

namespace {

constexpr int TM = 64, TN = 64, TK = 32;

// C[M][N] = sum_k A(m,k) B(k,n);  A(m,k) = TA ? A[k*lda+m] : A[m*lda+k];
// B(k,n) = TB ? B[n*ldb+k] : B[k*ldb+n].  gridDim.z = split-K partitions; with
// splits > 1, C points at the partial buffer [z][M][ldc].
// T: the CTA's output tile is T x T (64, or 32 for the head's small GEMMs: 4x the CTAs,
// so they fill the GPU without a split-K pass and its reduction launch)
template <bool TA, bool TB, int T = 64>
__global__ void __launch_bounds__(256)
sgemm_kernel(int M, int N, int K, const float* __restrict__ A, int lda, const float* __restrict__ B, int ldb,
             float* __restrict__ C, int ldc, int epi, const float* __restrict__ bias, float* __restrict__ H, int ldh,
             int k_chunk, EpiExtra ex) {
  pdl_enter();
  constexpr int TM = T, TN = T, RI = T / 16;
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int kb = blockIdx.z * k_chunk;
  const int ke = min(K, kb + k_chunk);
  float acc[RI][RI] = {};
  // tile loads double-buffered through registers: tile k0 + TK is fetched from global memory
  // while tile k0 is multiplied out of SMEM (the head's GEMMs are latency-bound otherwise)
  constexpr int LA = TM * TK / 256, LB = TN * TK / 256;
  float ra[LA], rb[LB];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int u = 0; u < LA; ++u) {
      const int i = threadIdx.x + 256 * u;
      int mm, kk;
      if (TA) { mm = i % TM; kk = i / TM; } else { kk = i % TK; mm = i / TK; }
      const int gm = m0 + mm, gk = k0 + kk;
      ra[u] = (gm < M && gk < ke) ? (TA ? A[(size_t)gk * lda + gm] : A[(size_t)gm * lda + gk]) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < LB; ++u) {
      const int i = threadIdx.x + 256 * u;
      int nn, kk;
      if (TB) { kk = i % TK; nn = i / TK; } else { nn = i % TN; kk = i / TN; }
      const int gn = n0 + nn, gk = k0 + kk;
      rb[u] = (gn < N && gk < ke) ? (TB ? B[(size_t)gn * ldb + gk] : B[(size_t)gk * ldb + gn]) : 0.f;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int u = 0; u < LA; ++u) {
      const int i = threadIdx.x + 256 * u;
      int mm, kk;
      if (TA) { mm = i % TM; kk = i / TM; } else { kk = i % TK; mm = i / TK; }
      As[kk][mm] = ra[u];
    }
#pragma unroll
    for (int u = 0; u < LB; ++u) {
      const int i = threadIdx.x + 256 * u;
      int nn, kk;
      if (TB) { kk = i % TK; nn = i / TK; } else { nn = i % TN; kk = i / TN; }
      Bs[kk][nn] = rb[u];
    }
  };
  if (kb < ke) fetch(kb);
  for (int k0 = kb; k0 < ke; k0 += TK) {
    stash();
    __syncthreads();
    if (k0 + TK < ke) fetch(k0 + TK);
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[RI], b[RI];
#pragma unroll
      for (int i = 0; i < RI; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < RI; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < RI; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* Cz = C + (size_t)blockIdx.z * M * ldc;
#pragma unroll
  for (int i = 0; i < RI; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < RI; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (epi == EPI_BIAS || epi == EPI_BIAS_RELU) v += bias[n];
      if (epi == EPI_RELU_MASK && !(ex.mask[(size_t)m * ex.ldm + n] > 0.f)) v = 0.f;
      Cz[(size_t)m * ldc + n] = v;
      if (epi == EPI_BIAS_RELU) {
        const float h = fmaxf(v, 0.f);
        H[(size_t)m * ldh + n] = h;
        if (ex.Hb) ex.Hb[(size_t)m * ldh + n] = __float2bfloat16_rn(h);
      }
    }
  }
}

__global__ void splitk_reduce_kernel(int M, int N, int splits, const float* __restrict__ part, float* __restrict__ C,
                                     int ldc, const float* __restrict__ mask, int ldm) {
  pdl_enter();
  const size_t total = (size_t)M * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / N), n = (int)(i % N);
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[(size_t)z * M * N + i];   // fixed order
    if (mask && !(mask[(size_t)m * ldm + n] > 0.f)) s = 0.f;             // ReLU'(0) = 0
    C[(size_t)m * ldc + n] = s;
  }
}

// The same reduction, 4 consecutive columns per thread (N, ldc, ldm multiples of 4, 16-byte
// aligned pointers): float4 loads of 8 splits are issued before the 8 adds, which still run
// in split order (bit-identical to splitk_reduce_kernel; that one waited on every load)
__global__ void splitk_reduce4_kernel(int M, int N, int splits, const float4* __restrict__ part, float* __restrict__ C,
                                      int ldc, const float* __restrict__ mask, int ldm) {
  pdl_enter();
  const size_t total4 = (size_t)M * N / 4, stride = total4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total4; i += (size_t)gridDim.x * blockDim.x) {
    const int m = (int)(4 * i / N), n = (int)(4 * i % N);
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    int z = 0;
    for (; z + 8 <= splits; z += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(part + (size_t)(z + u) * stride + i);
#pragma unroll
      for (int u = 0; u < 8; ++u) { s.x += v[u].x; s.y += v[u].y; s.z += v[u].z; s.w += v[u].w; }
    }
    for (; z < splits; ++z) {
      const float4 v = __ldg(part + (size_t)z * stride + i);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    if (mask) {                                                          // ReLU'(0) = 0
      const float4 mk = *reinterpret_cast<const float4*>(mask + (size_t)m * ldm + n);
      if (!(mk.x > 0.f)) s.x = 0.f;
      if (!(mk.y > 0.f)) s.y = 0.f;
      if (!(mk.z > 0.f)) s.z = 0.f;
      if (!(mk.w > 0.f)) s.w = 0.f;
    }
    *reinterpret_cast<float4*>(C + (size_t)m * ldc + n) = s;
  }
}

// Output layer, fp32 parity mode: Y = H W^T + b, raw gradient dS/dY = 2 (Y - T)
// for valid rows/cols (0 elsewhere), SSE partial per block.
__global__ void __launch_bounds__(256)
out_fwd_f32_kernel(OutArgs a) {
  pdl_enter();
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  __shared__ double s_red[256];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int M = a.B, K = a.K;
  const int Nn = (int)a.Npad;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int i = threadIdx.x; i < TM * TK; i += 256) {
      const int kk = i % TK, mm = i / TK, gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? a.H[(size_t)gm * a.ldh + gk] : 0.f;
    }
    for (int i = threadIdx.x; i < TN * TK; i += 256) {
      const int kk = i % TK, nn = i / TK, gn = n0 + nn, gk = k0 + kk;
      Bs[kk][nn] = (gn < Nn && gk < K) ? a.W[(size_t)gn * K + gk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  const uint32_t n_valid = a.st->n_last;
  double sse = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= M) continue;
    const bool row_ok = (uint32_t)m < n_valid;
    const int32_t slot = row_ok ? a.slots[m] : 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= Nn) continue;
      float g = 0.f;
      if (row_ok && (uint32_t)n < a.N) {
        const float y = acc[i][j] + a.b[n];
        const size_t off = (size_t)slot * a.Npad + n;
        const float t = a.storage == 0 ? static_cast<const float*>(a.payload)[off]
                                       : bf16_bits_to_f32(static_cast<const uint16_t*>(a.payload)[off]);
        const float r = y - t;
        sse += (double)r * (double)r;
        g = 2.f * r;
      }
      a.dY[(size_t)m * a.Npad + n] = g;
    }
  }
  s_red[threadIdx.x] = sse;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) s_red[threadIdx.x] += s_red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) a.sse_part[blockIdx.y * gridDim.x + blockIdx.x] = s_red[0];
}

// column sums over the batch (bias gradients): 32 columns x 32 row groups per CTA; each
// thread sums rows g, g+32, ... (4 loads in flight), then a fixed-order tree over the 32
// groups.  Accumulated in fp64 and rounded once, so the result is the fp32 rounding of the
// (near-)exact sum whatever the order -- closest to the fp64 oracle and insensitive to the
// grouping (the free-running bf16 trajectory amplifies fp32 order effects)
// ColSumJob: up to two matrices per launch (the head's bias gradients: one launch for both
// hidden layers); CTAs [0, ceil(cols0 / 32)) take matrix 0, the rest matrix 1
struct ColSumJob {
  const float* X[2];
  int cols[2], ld[2];
  float* out[2];
};

__global__ void __launch_bounds__(1024)
col_sum_kernel(ColSumJob J, int rows) {
  pdl_enter();
  __shared__ double part[32][33];
  const int nb0 = (J.cols[0] + 31) / 32;
  const int w = blockIdx.x < (unsigned)nb0 ? 0 : 1;
  const float* __restrict__ X = J.X[w];
  const int cols = J.cols[w], ld = J.ld[w];
  float* __restrict__ out = J.out[w];
  const int cl = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int c = (blockIdx.x - (w ? nb0 : 0)) * 32 + cl;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (c < cols) {
    int r = grp;
    for (; r + 96 < rows; r += 128) {
      s0 += X[(size_t)r * ld + c];
      s1 += X[(size_t)(r + 32) * ld + c];
      s2 += X[(size_t)(r + 64) * ld + c];
      s3 += X[(size_t)(r + 96) * ld + c];
    }
    for (; r < rows; r += 32) s0 += X[(size_t)r * ld + c];
  }
  part[grp][cl] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  for (int o = 16; o > 0; o >>= 1) {
    if (grp < o) part[grp][cl] += part[grp + o][cl];
    __syncthreads();
  }
  if (grp == 0 && c < cols) out[c] = (float)part[0][cl];
}

// split-K reduction with the GEMM epilogues: out = sum_z part[z] (+ bias, then Z/H
// with ReLU for EPI_BIAS_RELU), fixed order over z
__global__ void splitk_reduce_epi_kernel(int M, int N, int splits, const float* __restrict__ part, float* __restrict__ C,
                                         int ldc, int epi, const float* __restrict__ bias, float* __restrict__ H,
                                         int ldh, EpiExtra ex) {
  pdl_enter();
  const size_t total = (size_t)M * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / N), n = (int)(i % N);
    float v = 0.f;
    for (int z = 0; z < splits; ++z) v += part[(size_t)z * M * N + i];
    if (epi == EPI_BIAS || epi == EPI_BIAS_RELU) v += bias[n];
    if (epi == EPI_RELU_MASK && !(ex.mask[(size_t)m * ex.ldm + n] > 0.f)) v = 0.f;
    C[(size_t)m * ldc + n] = v;
    if (epi == EPI_BIAS_RELU) {
      const float h = fmaxf(v, 0.f);
      H[(size_t)m * ldh + n] = h;
      if (ex.Hb) ex.Hb[(size_t)m * ldh + n] = __float2bfloat16_rn(h);
    }
  }
}

// [SSE, n] of this rank's step from K1's per-CTA SSE partials (256 threads, fixed order)
__device__ __forceinline__ void reduce_local_block(StepDev* sd, const double* parts, int n_parts, const ResDev* st,
                                                   double* s) {
  double v = 0.0;
  for (int i = threadIdx.x; i < n_parts; i += 256) v += parts[i];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  // a batch with non-finite inputs contributes NaN to the global count: every rank skips
  if (threadIdx.x == 0) { sd->red[0] = s[0]; sd->red[1] = st->bad_batch ? nan("") : (double)st->n_last; }
}

__global__ void reduce_local_kernel(StepDev* sd, const double* parts, int n_parts, const ResDev* st) {
  pdl_enter();
  __shared__ double s[256];
  reduce_local_block(sd, parts, n_parts, st, s);
}

__device__ void finalize_scalars(StepDev* sd, double n_field, double lr0, double lr_min, uint64_t halving, double b1,
                                 double b2, Mirror* mirror, ResDev* st, uint32_t slot) {
  const double sse = sd->red[0], n = sd->red[1];
  st->n_last = 0;                       // a batch is consumed by exactly one step
  st->bad_batch = 0;
  mirror->n_last = 0;
  if (isnan(n) || (n > 0.0 && !isfinite(sse))) {
    // some rank's batch held non-finite inputs (n = NaN: nothing was updated, reading of
    // the ABI's "state unchanged"), or the loss itself is not finite: skip the update
    sd->skip = 1; sd->nonfinite = 1;
    mirror->status = 3; mirror->n_total = n; mirror->loss = sse;
    mirror->ring_status[slot] = 3; mirror->ring_loss[slot] = nan("");
    return;
  }
  if (n <= 0.0) {
    sd->skip = 1;
    mirror->status = 1; mirror->n_total = 0.0;
    mirror->ring_status[slot] = 1; mirror->ring_loss[slot] = 0.0;
    return;
  }
  sd->skip = 0;
  const double denom = n_field * n;
  sd->loss = sse / denom;
  sd->nonfinite = !isfinite(sd->loss);
  sd->scale = (float)(1.0 / denom);
  // lr halved every `halving` global samples, floor lr_min (reading Q24)
  const uint64_t S = sd->S;
  const double lr = fmax(lr_min, lr0 * exp2(-(double)(S / halving)));
  const uint64_t k = sd->k + 1;
  sd->lr = (float)lr;
  sd->c1 = (float)(1.0 - pow(b1, (double)k));
  sd->c2 = (float)(1.0 - pow(b2, (double)k));
  sd->k = k;
  sd->S = S + (uint64_t)n;
  mirror->status = 0; mirror->loss = sd->loss; mirror->n_total = n;
  mirror->ring_status[slot] = 0; mirror->ring_loss[slot] = sd->loss;
  mirror->adam_k = k; mirror->samples = sd->S;
}

__global__ void step_finalize_kernel(StepDev* sd, double n_field, double lr0, double lr_min, uint64_t halving,
                                     double b1, double b2, Mirror* mirror, ResDev* st, uint32_t slot) {
  pdl_enter();
  finalize_scalars(sd, n_field, lr0, lr_min, halving, b1, b2, mirror, st, slot);
}

// Step scalars ahead of the output-layer kernel (world == 1, fused Adam): the same
// values step_finalize computes afterwards (scale, lr, bias corrections of step k+1).
// the step's scalars ahead of K1 (the fused Adam needs lr, bias corrections, the gradient scale)
__device__ __forceinline__ void prepare_scalars(StepDev* sd, const ResDev* st, double n_field, double lr0,
                                                double lr_min, uint64_t halving, double b1, double b2, int global_n) {
  const uint32_t bad = *(volatile const uint32_t*)&st->bad_batch;
  const double n = global_n ? sd->n_glob : (bad ? nan("") : (double)st->n_last);
  if (!(n > 0.0)) { sd->skip = 1; return; }            // no samples, or non-finite inputs (NaN)
  sd->skip = 0;
  sd->scale = (float)(1.0 / (n_field * n));
  sd->lr = (float)fmax(lr_min, lr0 * exp2(-(double)(sd->S / halving)));
  const uint64_t k = sd->k + 1;
  sd->c1 = (float)(1.0 - pow(b1, (double)k));
  sd->c2 = (float)(1.0 - pow(b2, (double)k));
}

__global__ void step_prepare_kernel(StepDev* sd, const ResDev* st, double n_field, double lr0, double lr_min,
                                    uint64_t halving, double b1, double b2, int global_n) {
  pdl_enter();
  prepare_scalars(sd, st, n_field, lr0, lr_min, halving, b1, b2, global_n);
}

// Adam (bias-corrected), flat over every tensor; g is the raw dS/dtheta and is
// scaled by 1/(N * n_total) here.  Writes the bf16 shadow of [sh_begin, sh_end).
// Two float4 per array in flight per thread (memory-level parallelism).
__device__ __forceinline__ void adam4(float4& pp, float4& mm, float4& vv, const float4& gg, float scale, float step,
                                      float inv_sqrt_c2, float b1, float b2, float eps) {
  float* P = &pp.x; float* Mv = &mm.x; float* V = &vv.x; const float* G = &gg.x;
#pragma unroll
  for (int c = 0; c < 4; ++c) adam_elem(P[c], Mv[c], V[c], G[c], scale, step, inv_sqrt_c2, b1, b2, eps);
}

__device__ __forceinline__ void store_shadow(__nv_bfloat16* shadow, uint64_t e, uint64_t b0, uint64_t b1,
                                             const float4& p) {
  if (shadow && e >= b0 && e < b1) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(p.x, p.y);
    __nv_bfloat162 hi = __floats2bfloat162_rn(p.z, p.w);
    reinterpret_cast<uint2*>(shadow + (e - b0))[0] =
        make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
}

// UNR float4 of each array in flight per thread; the tail loop handles the rest
template <int UNR>
__global__ void __launch_bounds__(256)
adam_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v, const float* __restrict__ g,
            uint64_t n4, const StepDev* __restrict__ sd, float b1, float b2, float eps,
            __nv_bfloat16* __restrict__ shadow, uint64_t sh_begin, uint64_t sh_end) {
  pdl_enter();
  if (sd->skip) return;
  const float scale = sd->scale, step = sd->lr / sd->c1, isc2 = rsqrtf(sd->c2);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  float4* P4 = reinterpret_cast<float4*>(p);
  float4* M4 = reinterpret_cast<float4*>(m);
  float4* V4 = reinterpret_cast<float4*>(v);
  const float4* G4 = reinterpret_cast<const float4*>(g);
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i + (UNR - 1) * stride < n4; i += UNR * stride) {
    float4 pa[UNR], ma[UNR], va[UNR], ga[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint64_t j = i + u * stride;
      pa[u] = P4[j]; ma[u] = M4[j]; va[u] = V4[j]; ga[u] = __ldcs(G4 + j);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint64_t j = i + u * stride;
      adam4(pa[u], ma[u], va[u], ga[u], scale, step, isc2, b1, b2, eps);
      P4[j] = pa[u]; M4[j] = ma[u]; V4[j] = va[u];
      store_shadow(shadow, 4 * j, sh_begin, sh_end, pa[u]);
    }
  }
  for (; i < n4; i += stride) {
    float4 pa = P4[i], ma = M4[i], va = V4[i];
    const float4 ga = G4[i];
    adam4(pa, ma, va, ga, scale, step, isc2, b1, b2, eps);
    P4[i] = pa; M4[i] = ma; V4[i] = va;
    store_shadow(shadow, 4 * i, sh_begin, sh_end, pa);
  }
}

__global__ void init_kernel(float* dst, uint64_t count, uint32_t tid, uint32_t fan_in, uint64_t seed) {
  pdl_enter();
  const double a = 1.0 / sqrt((double)fan_in);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
    const double u = unit_double(philox_r64(seed, TAG_INIT, i, tid));
    dst[i] = (float)((2.0 * u - 1.0) * a);     // fp64 then RNE to fp32 (reading Q22)
  }
}

__global__ void to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, uint64_t n) {
  pdl_enter();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

__global__ void relu_mask_kernel(float* X, const float* Z, uint64_t n) {
  pdl_enter();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (!(Z[i] > 0.f)) X[i] = 0.f;
}

__global__ void eval_mse_kernel(const float* __restrict__ Y, const float* __restrict__ T, int rows, int cols, int ld,
                                double* part) {
  pdl_enter();
  __shared__ double s[256];
  double acc = 0.0;
  const size_t total = (size_t)rows * cols;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / cols, c = i % cols;
    const double d = (double)Y[r * ld + c] - (double)T[r * cols + c];
    acc += d * d;
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

__global__ void eval_inputs_kernel(const float* X, const uint32_t* t, int n, uint32_t tau, float lo, float span,
                                   float* xn) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  float o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int c = 0; c < 5; ++c) o[c] = normalise_rn(X[b * 5 + c], lo, span);
  o[5] = __fdiv_rn((float)t[b], (float)tau);
  for (int c = 0; c < 8; ++c) xn[b * 8 + c] = o[c];
}

__global__ void normalise_kernel(const float* src, float* dst, uint64_t n, float lo, float span) {
  pdl_enter();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = normalise_rn(src[i], lo, span);
}

inline unsigned grid_for(uint64_t n, unsigned block = 256, unsigned cap = 148 * 16) {
  uint64_t g = (n + block - 1) / block;
  if (g > cap) g = cap;
  if (g == 0) g = 1;
  return (unsigned)g;
}

}  // namespace

void sgemm(bool ta, bool tb, int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
           int ldc, int epi, const float* bias, float* H, int ldh, int splits, cudaStream_t s, EpiExtra ex) {
  if (splits < 1) splits = 1;
  int k_chunk = (K + splits - 1) / splits;
  k_chunk = ((k_chunk + TK - 1) / TK) * TK;
  dim3 grid((N + TN - 1) / TN, (M + TM - 1) / TM, splits);
  if (!ta && !tb) launch_pdl(sgemm_kernel<false, false>, dim3(grid), dim3(256), 0, s, M, N, K, A, lda, B, ldb, C, ldc, epi, bias, H, ldh, k_chunk, ex);
  else if (!ta && tb) launch_pdl(sgemm_kernel<false, true>, dim3(grid), dim3(256), 0, s, M, N, K, A, lda, B, ldb, C, ldc, epi, bias, H, ldh, k_chunk, ex);
  else if (ta && !tb) launch_pdl(sgemm_kernel<true, false>, dim3(grid), dim3(256), 0, s, M, N, K, A, lda, B, ldb, C, ldc, epi, bias, H, ldh, k_chunk, ex);
  else launch_pdl(sgemm_kernel<true, true>, dim3(grid), dim3(256), 0, s, M, N, K, A, lda, B, ldb, C, ldc, epi, bias, H, ldh, k_chunk, ex);
}

void splitk_reduce(int M, int N, int splits, const float* part, float* C, int ldc, const float* relu_mask, int ldm,
                   cudaStream_t s) {
  const bool v4 = N % 4 == 0 && ldc % 4 == 0 && (!relu_mask || ldm % 4 == 0) && ((uintptr_t)part & 15) == 0 &&
                  ((uintptr_t)C & 15) == 0 && ((uintptr_t)relu_mask & 15) == 0;
  if (v4)
    launch_pdl(splitk_reduce4_kernel, dim3(grid_for((uint64_t)M * N / 4)), dim3(256), 0, s, M, N, splits,
               reinterpret_cast<const float4*>(part), C, ldc, relu_mask, ldm);
  else
    launch_pdl(splitk_reduce_kernel, dim3(grid_for((uint64_t)M * N)), dim3(256), 0, s, M, N, splits, part, C, ldc, relu_mask, ldm);
}

int out_fwd_f32(const OutArgs& a, cudaStream_t s) {
  dim3 grid((unsigned)((a.Npad + TN - 1) / TN), (a.B + TM - 1) / TM);
  launch_pdl(out_fwd_f32_kernel, dim3(grid), dim3(256), 0, s, a);
  return (int)(grid.x * grid.y);
}

void col_sum(const float* X, int rows, int cols, int ld, float* out, cudaStream_t s) {
  col_sum2(X, cols, ld, out, nullptr, 0, 0, nullptr, rows, s);
}

void col_sum2(const float* X0, int cols0, int ld0, float* out0, const float* X1, int cols1, int ld1, float* out1,
              int rows, cudaStream_t s) {
  ColSumJob J;
  J.X[0] = X0; J.cols[0] = cols0; J.ld[0] = ld0; J.out[0] = out0;
  J.X[1] = X1; J.cols[1] = X1 ? cols1 : 0; J.ld[1] = ld1; J.out[1] = out1;
  const int nb = (cols0 + 31) / 32 + (J.cols[1] + 31) / 32;
  launch_pdl(col_sum_kernel, dim3(nb), dim3(1024), 0, s, J, rows);
}

// SIMT GEMM that fills the GPU: split-K through `scratch` (>= splits*M*N floats) when
// the output grid is smaller than one wave; returns the number of launches
int sgemm_auto(bool ta, bool tb, int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C, int ldc,
               int epi, const float* bias, float* H, int ldh, float* scratch, size_t scratch_elems, cudaStream_t s,
               EpiExtra ex) {
  const int tiles = ((M + TM - 1) / TM) * ((N + TN - 1) / TN);
  int sk = 1;
  while (tiles * sk < 148 && K / (sk * 2) >= 64 && (size_t)(sk * 2) * M * N <= scratch_elems) sk *= 2;
  if (sk == 1) {
    sgemm(ta, tb, M, N, K, A, lda, B, ldb, C, ldc, epi, bias, H, ldh, 1, s, ex);
    return 1;
  }
  sgemm(ta, tb, M, N, K, A, lda, B, ldb, scratch, N, EPI_STORE, nullptr, nullptr, 0, sk, s);
  launch_pdl(splitk_reduce_epi_kernel, dim3(grid_for((uint64_t)M * N)), dim3(256), 0, s, M, N, sk, scratch, C, ldc, epi, bias, H, ldh, ex);
  return 2;
}

// ---- fused head (paper shape: 6 -> 256 -> 256) --------------------------------
// Forward: every output is accumulated k ascending from 0, then + bias (the generic sgemm's
// order without its split-K).  Backward: phase 1 (head_bwd3) writes per-block partial sums,
// phase 2 (head_fin3) reduces them in a fixed order -- deterministic, no atomics on data.
// Every CTA stages its whole weight / activation block in SMEM with cp.async issued up front
// (one memory latency per CTA instead of one per chunk: these kernels are latency-bound).
constexpr int HF_ROWS = 16;      // forward: batch rows per CTA pair (one CTA per 128-unit half)
constexpr int HF_P = 260;        // forward: W2 row pitch in SMEM (float4 reads conflict-free)
constexpr int HB_ROWS = 32;      // backward row CTAs: batch rows (x 64 hidden units)
constexpr int HB_KQ = 64;        // backward row CTAs: layer-1 units per CTA
constexpr int HSL = 64;          // backward dW2 CTAs: batch rows per slice
constexpr int HJT = 32;          // backward dW2 CTAs: W2 rows per CTA
constexpr size_t HF_SMEM = (size_t)(128 * HF_P + HF_ROWS * 256 + HF_ROWS * 8) * 4;
constexpr size_t HB_SMEM_ROW = (size_t)(256 * HB_KQ + HB_ROWS * 256 + HB_ROWS * 8 + 4 * HB_KQ * 9) * 4 +
                               (size_t)4 * HB_KQ * 8;
constexpr size_t HB_SMEM_W2 = (size_t)(HSL * 256 + HSL * HJT) * 4;
constexpr size_t HB_SMEM = HB_SMEM_ROW > HB_SMEM_W2 ? HB_SMEM_ROW : HB_SMEM_W2;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__global__ void __launch_bounds__(256) head_fwd3_kernel(HeadFwdArgs a) {
  pdl_enter();
  extern __shared__ __align__(16) float hsm[];
  float* ws = hsm;                                   // [128 units][HF_P]: this half of W2
  float* h1s = ws + 128 * HF_P;                      // [HF_ROWS][256]
  float* xs = h1s + HF_ROWS * 256;                   // [HF_ROWS][8]
  const int tid = threadIdx.x;
  // CTA pair (2 rb, 2 rb + 1): row block rb, layer-2 units [128 half, 128 half + 128); both
  // compute layer 1 for the block (6 inputs: cheap), the even one stores it
  const uint32_t b0 = (blockIdx.x >> 1) * HF_ROWS;
  const int half = blockIdx.x & 1;
  const int nu = min(128, a.d2 - 128 * half);        // units of this half (<= 0: none)
  for (int f = tid; f < 128 * (a.d1 / 4); f += 256) {
    const int jj = f / (a.d1 / 4), c4 = f % (a.d1 / 4);
    if (jj < nu) cp_async16(ws + jj * HF_P + 4 * c4, a.W2 + (uint64_t)(128 * half + jj) * a.d1 + 4 * c4);
  }
  // the batch's normalised inputs (reading Q13), gather_inputs' arithmetic
  if (tid < HF_ROWS) {
    const uint32_t b = b0 + tid;
    float out[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (b < a.B) {
      const uint32_t n = a.ra.st->n_last;
      if (b < n) {
        if (half == 0 && a.ra.bad[a.slots[b]]) atomicOr(&a.ra.st->bad_batch, 1u);   // reset by step_finalize
        const SlotMeta m = a.ra.meta[a.slots[b]];
#pragma unroll
        for (int c = 0; c < 5; ++c) out[c] = normalise_rn(m.X[c], a.ra.lo, a.ra.span);
        out[5] = __fdiv_rn((float)m.t, (float)a.tau);
      }
      if (half == 0) {
        float4* dst = reinterpret_cast<float4*>(a.xn + (uint64_t)b * 8);
        dst[0] = make_float4(out[0], out[1], out[2], out[3]);
        dst[1] = make_float4(out[4], out[5], out[6], out[7]);
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) xs[tid * 8 + c] = out[c];
  }
  __syncthreads();
  const int nr = (int)min((uint32_t)HF_ROWS, a.B > b0 ? a.B - b0 : 0u);
  // layer 1: thread j -> unit j
  if (tid < a.d1) {
    float w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = i < a.d0 ? a.W1[tid * a.d0 + i] : 0.f;
    const float bj = a.b1[tid];
#pragma unroll 4
    for (int r = 0; r < HF_ROWS; ++r) {
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < a.d0) acc = fmaf(xs[r * 8 + i], w[i], acc);
      const float z = acc + bj, h = fmaxf(z, 0.f);
      h1s[r * 256 + tid] = h;
      if (r < nr && half == 0) {
        const uint64_t o = (uint64_t)(b0 + r) * a.d1 + tid;
        a.Z1[o] = z;
        a.H1[o] = h;
      }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  // layer 2: thread (rq, jl) -> unit 128 half + jl, rows 8 rq .. 8 rq + 7
  const int jl = tid & 127, rq = tid >> 7;
  const int j2 = 128 * half + jl;
  constexpr int R2 = HF_ROWS / 2;
  float acc[R2];
#pragma unroll
  for (int r = 0; r < R2; ++r) acc[r] = 0.f;
  const float* wrow = ws + jl * HF_P;
  const float* hrow = h1s + R2 * rq * 256;
#pragma unroll 2
  for (int k = 0; k < a.d1; k += 4) {
    const float4 w = *reinterpret_cast<const float4*>(wrow + k);
#pragma unroll
    for (int r = 0; r < R2; ++r) {
      const float4 h = *reinterpret_cast<const float4*>(hrow + r * 256 + k);
      acc[r] = fmaf(h.x, w.x, acc[r]);
      acc[r] = fmaf(h.y, w.y, acc[r]);
      acc[r] = fmaf(h.z, w.z, acc[r]);
      acc[r] = fmaf(h.w, w.w, acc[r]);
    }
  }
  if (jl < nu) {
    const float bj = a.b2[j2];
#pragma unroll
    for (int r = 0; r < R2; ++r) {
      if (R2 * rq + r >= nr) break;
      const uint64_t o = (uint64_t)(b0 + R2 * rq + r) * a.d2 + j2;
      const float z = acc[r] + bj, h = fmaxf(z, 0.f);
      a.Z2[o] = z;
      a.H2[o] = h;
      if (a.Hb) a.Hb[o] = __float2bfloat16_rn(h);
    }
  }
  if (a.sd) {
    // fused step_prepare: the last CTA to arrive sees every CTA's bad-input flag
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(a.counter, 1u) == a.target - 1u) {
        __threadfence();
        prepare_scalars(a.sd, a.ra.st, a.n_field, a.lr0, a.lr_min, a.halving, a.beta1, a.beta2, 0);
      }
    }
  }
}

__global__ void __launch_bounds__(256, 2) head_bwd3_kernel(HeadBwdArgs a) {
  pdl_enter();
  extern __shared__ __align__(16) float hsm[];
  const int tid = threadIdx.x;
  const int n_kq = (a.d1 + HB_KQ - 1) / HB_KQ;
  const int n_rowc = head_bwd3_row_ctas(a.B) * n_kq;
  if ((int)blockIdx.x < n_rowc) {
    // ===== row CTA: dZ1 = (dZ2 W2) . ReLU'(Z1) for HB_ROWS rows x HB_KQ units; partial
    // dW1 / db1 of the row block =====
    float* ws = hsm;                                 // [256 j][HB_KQ]: W2[:, this quarter]
    float* dz = ws + 256 * HB_KQ;                    // [HB_ROWS][256]
    float* xs = dz + HB_ROWS * 256;                  // [HB_ROWS][8]
    float* pw_s = xs + HB_ROWS * 8;                  // [4 row groups][HB_KQ][9]
    double* pdb_s = reinterpret_cast<double*>(pw_s + 4 * HB_KQ * 9);   // [4][HB_KQ]
    const int rb = blockIdx.x / n_kq, kq = blockIdx.x % n_kq;
    const int b0 = rb * HB_ROWS, k0 = kq * HB_KQ;
    const int nr = min(HB_ROWS, a.B - b0), nk = min(HB_KQ, a.d1 - k0);
    for (int f = tid; f < a.d2 * (HB_KQ / 4); f += 256) {
      const int j = f / (HB_KQ / 4), c4 = f % (HB_KQ / 4);
      if (4 * c4 < nk) cp_async16(ws + j * HB_KQ + 4 * c4, a.W2 + (uint64_t)j * a.d1 + k0 + 4 * c4);
    }
    for (int f = tid; f < HB_ROWS * (a.d2 / 4); f += 256) {
      const int r = f / (a.d2 / 4), c4 = f % (a.d2 / 4);
      if (r < nr) cp_async16(dz + r * 256 + 4 * c4, a.dz2 + (uint64_t)(b0 + r) * a.d2 + 4 * c4);
      else *reinterpret_cast<float4*>(dz + r * 256 + 4 * c4) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    {
      const int r = tid / 8, i = tid % 8;
      xs[tid] = r < nr ? a.xn[(uint64_t)(b0 + r) * 8 + i] : 0.f;
    }
    cp_async_wait_all();
    __syncthreads();
    const int kl = tid % HB_KQ, rg = tid / HB_KQ;    // unit k0 + kl, rows 8 rg .. 8 rg + 7
    const int k = k0 + kl;
    float acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r] = 0.f;
    const float* drow = dz + 8 * rg * 256;
#pragma unroll 2
    for (int j = 0; j < a.d2; j += 4) {
      const float w0 = ws[j * HB_KQ + kl], w1 = ws[(j + 1) * HB_KQ + kl];
      const float w2 = ws[(j + 2) * HB_KQ + kl], w3 = ws[(j + 3) * HB_KQ + kl];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const float4 d = *reinterpret_cast<const float4*>(drow + r * 256 + j);
        acc[r] = fmaf(d.x, w0, acc[r]);
        acc[r] = fmaf(d.y, w1, acc[r]);
        acc[r] = fmaf(d.z, w2, acc[r]);
        acc[r] = fmaf(d.w, w3, acc[r]);
      }
    }
    float pw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    double pdb = 0.0;
    if (kl < nk) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int rr = 8 * rg + r;
        if (rr >= nr) break;
        const float d = a.z1[(uint64_t)(b0 + rr) * a.d1 + k] > 0.f ? acc[r] : 0.f;   // ReLU'(0) = 0 (R20)
        pdb += (double)d;
#pragma unroll
        for (int i = 0; i < 8; ++i) pw[i] = fmaf(d, xs[rr * 8 + i], pw[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) pw_s[(rg * HB_KQ + kl) * 9 + i] = pw[i];
    pdb_s[rg * HB_KQ + kl] = pdb;
    __syncthreads();
    if (tid < HB_KQ && tid < nk) {
      // the block's four row groups in order
      float t[8];
      double tb = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) t[i] = 0.f;
      for (int g = 0; g < 4; ++g) {
#pragma unroll
        for (int i = 0; i < 8; ++i) t[i] += pw_s[(g * HB_KQ + tid) * 9 + i];
        tb += pdb_s[g * HB_KQ + tid];
      }
      float4* dst = reinterpret_cast<float4*>(a.p_dw1 + ((uint64_t)rb * a.d1 + k0 + tid) * 8);
      dst[0] = make_float4(t[0], t[1], t[2], t[3]);
      dst[1] = make_float4(t[4], t[5], t[6], t[7]);
      a.p_db1[(uint64_t)rb * a.d1 + k0 + tid] = tb;
    }
    return;
  }
  // ===== dW2 CTA: slice sl (HSL batch rows) x W2 rows [HJT jt, HJT jt + HJT): partial
  // dW2[j][k] = sum_b dZ2[b][j] H1[b][k] (thread k), partial db2 (fp64) =====
  const int w = blockIdx.x - n_rowc;
  const int njt = a.d2 / HJT;
  const int sl = w / njt, jt = w % njt;
  const int bs = sl * HSL, nb = min(HSL, a.B - bs);
  float* hs = hsm;                                     // [HSL][256]
  float* dzs = hs + HSL * 256;                         // [HSL][HJT]
  for (int f = tid; f < HSL * (a.d1 / 4); f += 256) {
    const int r = f / (a.d1 / 4), c4 = f % (a.d1 / 4);
    if (r < nb) cp_async16(hs + r * 256 + 4 * c4, a.h1 + (uint64_t)(bs + r) * a.d1 + 4 * c4);
    else *reinterpret_cast<float4*>(hs + r * 256 + 4 * c4) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int f = tid; f < HSL * (HJT / 4); f += 256) {
    const int r = f / (HJT / 4), c4 = f % (HJT / 4);
    if (r < nb) cp_async16(dzs + r * HJT + 4 * c4, a.dz2 + (uint64_t)(bs + r) * a.d2 + jt * HJT + 4 * c4);
    else *reinterpret_cast<float4*>(dzs + r * HJT + 4 * c4) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  cp_async_wait_all();
  __syncthreads();
  const int k = tid < a.d1 ? tid : 0;
  float acc[HJT];
#pragma unroll
  for (int j = 0; j < HJT; ++j) acc[j] = 0.f;
#pragma unroll 2
  for (int r = 0; r < HSL; ++r) {
    const float h = hs[r * 256 + k];
#pragma unroll
    for (int j = 0; j < HJT; j += 4) {
      const float4 d = *reinterpret_cast<const float4*>(&dzs[r * HJT + j]);
      acc[j] = fmaf(d.x, h, acc[j]);
      acc[j + 1] = fmaf(d.y, h, acc[j + 1]);
      acc[j + 2] = fmaf(d.z, h, acc[j + 2]);
      acc[j + 3] = fmaf(d.w, h, acc[j + 3]);
    }
  }
  if (tid < a.d1) {
#pragma unroll
    for (int j = 0; j < HJT; ++j) a.p_dw2[((uint64_t)sl * a.d2 + jt * HJT + j) * a.d1 + k] = acc[j];
  }
  if (tid < HJT) {
    double t = 0.0;
    for (int r = 0; r < HSL; ++r) t += (double)dzs[r * HJT + tid];
    a.p_db2[(uint64_t)sl * a.d2 + jt * HJT + tid] = t;
  }
}

// phase 2: the fixed-order reductions of the head's partial gradients (one output per
// thread); with sd set (world 1) block 0 then also folds K1's SSE partials into [SSE, n]
// and runs step_finalize's scalars (the step's last small kernels in one launch)
__global__ void __launch_bounds__(256) head_fin3_kernel(HeadBwdArgs a) {
  pdl_enter();
  __shared__ double sred[256];
  const int n_row = head_bwd3_row_ctas(a.B), n_sl = (a.B + HSL - 1) / HSL;
  const int n_w2 = a.d2 * a.d1;
  const int nb_w2 = (n_w2 + 255) / 256;
  if ((int)blockIdx.x < nb_w2) {
    // dW2: one output per thread, the slice partials in slice order (loads all in flight)
    const int o = blockIdx.x * 256 + threadIdx.x;
    if (o < n_w2) {
      float t = 0.f;
      for (int c0 = 0; c0 < n_sl; c0 += 16) {
        float v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = c0 + u < n_sl ? __ldcg(a.p_dw2 + (uint64_t)(c0 + u) * n_w2 + o) : 0.f;
#pragma unroll
        for (int u = 0; u < 16; ++u) t += v[u];
      }
      a.gW2[o] = t;
    }
  } else {
    // dW1 / db1 (row-CTA partials) and db2 (slice partials): one warp per unit k; lane l
    // takes partials l, l + 32, ... in order, then a fixed xor-butterfly across the warp
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = ((int)blockIdx.x - nb_w2) * 8 + warp;
    if (k < a.d1 || k < a.d2) {
      float pw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      double pdb1 = 0.0, pdb2 = 0.0;
      if (k < a.d1) {
        for (int c = lane; c < n_row; c += 32) {
          const float4* src = reinterpret_cast<const float4*>(a.p_dw1 + ((uint64_t)c * a.d1 + k) * 8);
          const float4 x0 = __ldcg(src), x1 = __ldcg(src + 1);
          pw[0] += x0.x; pw[1] += x0.y; pw[2] += x0.z; pw[3] += x0.w;
          pw[4] += x1.x; pw[5] += x1.y; pw[6] += x1.z; pw[7] += x1.w;
          pdb1 += __ldcg(a.p_db1 + (uint64_t)c * a.d1 + k);
        }
      }
      if (k < a.d2)
        for (int c = lane; c < n_sl; c += 32) pdb2 += __ldcg(a.p_db2 + (uint64_t)c * a.d2 + k);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int i = 0; i < 8; ++i) pw[i] += __shfl_xor_sync(0xffffffffu, pw[i], o);
        pdb1 += __shfl_xor_sync(0xffffffffu, pdb1, o);
        pdb2 += __shfl_xor_sync(0xffffffffu, pdb2, o);
      }
      if (lane == 0) {
        if (k < a.d1) {
          for (int i = 0; i < a.d0; ++i) a.gW1[k * a.d0 + i] = pw[i];
          a.gb1[k] = (float)pdb1;
        }
        if (k < a.d2) a.gb2[k] = (float)pdb2;
      }
    }
  }
  if (a.sd && blockIdx.x == 0) {
    reduce_local_block(a.sd, a.sse_parts, a.n_sse_parts, a.st, sred);
    __syncthreads();
    if (threadIdx.x == 0)
      finalize_scalars(a.sd, a.n_field, a.lr0, a.lr_min, a.halving, a.beta1, a.beta2, a.mirror, a.st, a.slot);
  }
}

int head3_init() {
  if (cudaFuncSetAttribute(head_fwd3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HF_SMEM) != cudaSuccess)
    return -1;
  if (cudaFuncSetAttribute(head_bwd3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HB_SMEM) != cudaSuccess)
    return -1;
  return 0;
}

int head_fwd3_ctas(int B) { return 2 * ((B + HF_ROWS - 1) / HF_ROWS); }

void head_fwd3(const HeadFwdArgs& a, cudaStream_t s) {
  launch_pdl(head_fwd3_kernel, dim3(head_fwd3_ctas((int)a.B)), dim3(256), HF_SMEM, s, a);
}

void head_bwd3(const HeadBwdArgs& a, cudaStream_t s) {
  const int n = head_bwd3_row_ctas(a.B) * ((a.d1 + HB_KQ - 1) / HB_KQ) + ((a.B + HSL - 1) / HSL) * (a.d2 / HJT);
  launch_pdl(head_bwd3_kernel, dim3(n), dim3(256), HB_SMEM, s, a);
  const int nb = (a.d2 * a.d1 + 255) / 256 + ((a.d1 > a.d2 ? a.d1 : a.d2) + 7) / 8;
  launch_pdl(head_fin3_kernel, dim3(nb), dim3(256), 0, s, a);
}

size_t head_dw2_part_elems(int B, int d1, int d2) { return (size_t)((B + HSL - 1) / HSL) * d1 * d2; }

void reduce_local(StepDev* sd, const double* parts, int n_parts, const ResDev* st, cudaStream_t s) {
  launch_pdl(reduce_local_kernel, dim3(1), dim3(256), 0, s, sd, parts, n_parts, st);
}

void step_finalize(StepDev* sd, double n_field, double lr0, double lr_min, uint64_t halving, double b1, double b2,
                   Mirror* mirror, ResDev* st, cudaStream_t s, uint32_t slot) {
  launch_pdl(step_finalize_kernel, dim3(1), dim3(1), 0, s, sd, n_field, lr0, lr_min, halving, b1, b2, mirror, st, slot);
}

void step_prepare(StepDev* sd, const ResDev* st, double n_field, double lr0, double lr_min, uint64_t halving, double b1,
                  double b2, cudaStream_t s, bool global_n) {
  launch_pdl(step_prepare_kernel, dim3(1), dim3(1), 0, s, sd, st, n_field, lr0, lr_min, halving, b1, b2, global_n ? 1 : 0);
}

__global__ void stage_count_kernel(StepDev* sd, const ResDev* st) {
  pdl_enter(); sd->n_glob = st->bad_batch ? nan("") : (double)st->n_last; }

void stage_count(StepDev* sd, const ResDev* st, cudaStream_t s) { launch_pdl(stage_count_kernel, dim3(1), dim3(1), 0, s, sd, st); }

void adam_flat(float* p, float* m, float* v, const float* g, uint64_t n, const StepDev* sd, float b1, float b2,
               float eps, __nv_bfloat16* shadow, uint64_t sh_begin, uint64_t sh_end, cudaStream_t s) {
  const uint64_t n4 = n / 4;   // the flat buffer is padded to a multiple of 4
  launch_pdl(adam_kernel<2>, dim3(grid_for(n4, 256, 148 * 16)), dim3(256), 0, s, p, m, v, g, n4, sd, b1, b2, eps, shadow, sh_begin, sh_end);
}

void init_tensor(float* dst, uint64_t count, uint32_t tid, uint32_t fan_in, uint64_t seed, cudaStream_t s) {
  launch_pdl(init_kernel, dim3(grid_for(count)), dim3(256), 0, s, dst, count, tid, fan_in, seed);
}

void to_bf16(const float* src, __nv_bfloat16* dst, uint64_t n, cudaStream_t s) {
  launch_pdl(to_bf16_kernel, dim3(grid_for(n)), dim3(256), 0, s, src, dst, n);
}

void relu_mask_mul(float* X, const float* Z, uint64_t n, cudaStream_t s) {
  launch_pdl(relu_mask_kernel, dim3(grid_for(n)), dim3(256), 0, s, X, Z, n);
}

int eval_mse_partial(const float* Y, const float* T, int rows, int cols, int ld, double* part, cudaStream_t s) {
  const unsigned g = grid_for((uint64_t)rows * cols, 256, 256);
  launch_pdl(eval_mse_kernel, dim3(g), dim3(256), 0, s, Y, T, rows, cols, ld, part);
  return (int)g;
}

void eval_inputs(const float* X, const uint32_t* t, int n, uint32_t tau, float lo, float span, float* xn,
                 cudaStream_t s) {
  launch_pdl(eval_inputs_kernel, dim3((n + 127) / 128), dim3(128), 0, s, X, t, n, tau, lo, span, xn);
}

void normalise_fields(const float* src, float* dst, uint64_t n, float lo, float span, cudaStream_t s) {
  launch_pdl(normalise_kernel, dim3(grid_for(n)), dim3(256), 0, s, src, dst, n, lo, span);
}

}  // namespace mel

namespace mel {

// ---------------------------------------------------------------------------------
// Virtual ranks (mel_create_virtual): the all-reduce of R ranks living on one device as
// a rank-ordered sum written back to every rank ("all-reduced"), fp32 or fp64.
// ---------------------------------------------------------------------------------
template <typename T>
__global__ void vsum_kernel(T* const* bufs, int R, uint64_t n) {
  pdl_enter();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    T acc = bufs[0][i];
    for (int q = 1; q < R; ++q) acc += bufs[q][i];
    for (int q = 0; q < R; ++q) bufs[q][i] = acc;
  }
}

void vsum_f32(float* const* d_bufs, int R, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  launch_pdl(vsum_kernel<float>, dim3(grid_for(n, 256, 148 * 8)), dim3(256), 0, s, d_bufs, R, n);
}
void vsum_f64(double* const* d_bufs, int R, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  launch_pdl(vsum_kernel<double>, dim3(grid_for(n, 256, 148 * 8)), dim3(256), 0, s, d_bufs, R, n);
}

}  // namespace mel
