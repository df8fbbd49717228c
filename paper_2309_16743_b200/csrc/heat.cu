// On-device heat-equation client (include/mel_heat.h).
//
// Basis build: for each component c (X = e_c) and step t = 1..tau-1 the implicit Euler
// system (I - alpha dt L_h) u^t = u^{t-1} + c_h b is solved exactly by DST-I
// diagonalisation (S orthonormal and symmetric, S^2 = I):
//     u^t = S ( (S (u^{t-1} + c_h b) S) ./ D ) S,   D_ij = 1 + alpha dt (lambda_i + lambda_j)
// as four fp64 GEMMs of the m x m interior (m = n - 2) plus two elementwise passes, then
// the full n x n field (Dirichlet edges, averaged corners) is written to the basis.
// Field generation: one pass out[j] = RNE_f32(sum_c X_jc phi_c^{t_j}) (HBM-bound; fields
// of the same t share the basis rows through L2).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <new>

#include "../../include/mel_heat.h"
#include "common.cuh"

struct mel_heat {
  uint32_t n = 0, tau = 0;
  double* phi = nullptr;   // [5][tau][n*n] fp64
  uint64_t bytes = 0;
};

namespace {

constexpr int ST_OK = 0, ST_EINVAL = -1, ST_ECUDA = -4, ST_ENOMEM = -6;
constexpr int DT_M = 64, DT_N = 64, DT_K = 16;

// C[M][N] = A[M][K] B[K][N], row-major fp64, 64x64 tiles, 256 threads x 4x4 outputs
__global__ void __launch_bounds__(256) dgemm_nn(int M, int N, int K, const double* __restrict__ A,
                                                 const double* __restrict__ B, double* __restrict__ C) {
  __shared__ double As[DT_K][DT_M + 1];
  __shared__ double Bs[DT_K][DT_N + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * DT_M, n0 = blockIdx.x * DT_N;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += DT_K) {
    for (int i = threadIdx.x; i < DT_M * DT_K; i += 256) {
      const int kk = i % DT_K, mm = i / DT_K;
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? A[(size_t)gm * K + gk] : 0.0;
    }
    for (int i = threadIdx.x; i < DT_N * DT_K; i += 256) {
      const int nn = i % DT_N, kk = i / DT_N;
      const int gn = n0 + nn, gk = k0 + kk;
      Bs[kk][nn] = (gn < N && gk < K) ? B[(size_t)gk * N + gn] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < DT_K; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int nn = n0 + tx + 16 * j;
      if (nn < N) C[(size_t)m * N + nn] = acc[i][j];
    }
  }
}

__global__ void dst_matrix(int m, int n, double* S) {
  const double scale = sqrt(2.0 / (n - 1));
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < m * m; idx += gridDim.x * blockDim.x) {
    const int i = idx / m, j = idx % m;
    // sin(pi (i+1)(j+1) / (n-1)) with the integer product reduced mod 2(n-1) first
    const long long p = ((long long)(i + 1) * (j + 1)) % (2LL * (n - 1));
    S[idx] = scale * sin(M_PI * (double)p / (double)(n - 1));
  }
}

// v = u + c_h * b(e_comp) on the interior: b collects the Dirichlet neighbours
__global__ void add_boundary(int m, int comp, double ch, const double* __restrict__ u, double* __restrict__ v) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < m * m; idx += gridDim.x * blockDim.x) {
    const int j = idx / m, i = idx % m;      // [y][x] interior indices
    double b = 0.0;
    if (comp == 1 && i == 0) b += 1.0;       // T_x1 at x = 0
    if (comp == 3 && i == m - 1) b += 1.0;   // T_x2 at x = L
    if (comp == 2 && j == 0) b += 1.0;       // T_y1 at y = 0
    if (comp == 4 && j == m - 1) b += 1.0;   // T_y2 at y = L
    v[idx] = u[idx] + ch * b;
  }
}

__global__ void divide_denominator(int m, int n, double alpha_dt, double h, double* __restrict__ a) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < m * m; idx += gridDim.x * blockDim.x) {
    const int j = idx / m, i = idx % m;
    const double si = sin((i + 1) * M_PI / (2.0 * (n - 1))), sj = sin((j + 1) * M_PI / (2.0 * (n - 1)));
    const double lam = (4.0 / (h * h)) * (si * si + sj * sj);
    a[idx] = a[idx] / (1.0 + alpha_dt * lam);
  }
}

// full n x n field of component comp at step t >= 1 from the interior u
__global__ void assemble(int n, int comp, const double* __restrict__ u, double* __restrict__ f) {
  const int m = n - 2;
  const double tx1 = comp == 1, ty1 = comp == 2, tx2 = comp == 3, ty2 = comp == 4;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) {
    const int y = idx / n, x = idx % n;
    double v;
    if (x > 0 && x < n - 1 && y > 0 && y < n - 1) v = u[(size_t)(y - 1) * m + (x - 1)];
    else if ((x == 0 || x == n - 1) && (y == 0 || y == n - 1))
      v = 0.5 * ((x == 0 ? tx1 : tx2) + (y == 0 ? ty1 : ty2));
    else if (x == 0) v = tx1;
    else if (x == n - 1) v = tx2;
    else if (y == 0) v = ty1;
    else v = ty2;
    f[idx] = v;
  }
}

__global__ void fill(double* p, uint64_t count, double v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// out[j][k] = RNE_f32(sum_c X[j][c] * phi[c][t_j][k]); grid.y = field, grid.x strides the
// field in float4 groups
__global__ void __launch_bounds__(256) combine(uint32_t nn, uint32_t tau, const double* __restrict__ phi,
                                               const float* __restrict__ X, const uint32_t* __restrict__ t,
                                               float* __restrict__ out) {
  pdl_enter();
  const uint32_t j = blockIdx.y;
  const uint32_t tj = t[j];
  double x[5];
#pragma unroll
  for (int c = 0; c < 5; ++c) x[c] = (double)X[5 * j + c];
  const uint64_t plane = (uint64_t)tau * nn;
  const double* base = phi + (uint64_t)tj * nn;
  float* o = out + (uint64_t)j * nn;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nn; k += gridDim.x * blockDim.x) {
    double s = x[0] * __ldg(base + k);
#pragma unroll
    for (int c = 1; c < 5; ++c) s = fma(x[c], __ldg(base + c * plane + k), s);
    o[k] = __double2float_rn(s);
  }
}

unsigned grid1(uint64_t count) {
  uint64_t g = (count + 255) / 256;
  return (unsigned)(g < 148 * 16 ? (g ? g : 1) : 148 * 16);
}

}  // namespace

extern "C" {

int mel_heat_create(uint32_t n, uint32_t tau, double alpha, double dt, double length, mel_heat** out) {
  if (!out || n < 3 || tau < 1 || !(alpha > 0) || !(dt > 0) || !(length > 0)) return ST_EINVAL;
  *out = nullptr;
  mel_heat* h = new (std::nothrow) mel_heat;
  if (!h) return ST_ENOMEM;
  h->n = n;
  h->tau = tau;
  const uint64_t nn = (uint64_t)n * n, m = n - 2;
  h->bytes = 5ull * tau * nn * sizeof(double);
  if (cudaMalloc(&h->phi, h->bytes) != cudaSuccess) {
    (void)cudaGetLastError();
    delete h;
    return ST_ENOMEM;
  }
  double *S = nullptr, *u = nullptr, *a = nullptr, *b = nullptr;
  const size_t mm = (size_t)m * m * sizeof(double);
  int st = ST_OK;
  if (cudaMalloc(&S, mm) != cudaSuccess || cudaMalloc(&u, mm) != cudaSuccess || cudaMalloc(&a, mm) != cudaSuccess ||
      cudaMalloc(&b, mm) != cudaSuccess) {
    (void)cudaGetLastError();
    st = ST_ENOMEM;
  }
  if (!st) {
    const double hh = length / (n - 1), ch = alpha * dt / (hh * hh);
    const dim3 gg((unsigned)((m + DT_N - 1) / DT_N), (unsigned)((m + DT_M - 1) / DT_M));
    dst_matrix<<<grid1(m * m), 256>>>((int)m, (int)n, S);
    for (int c = 0; c < 5; ++c) {
      const double t_ic = c == 0 ? 1.0 : 0.0;
      double* phic = h->phi + (uint64_t)c * tau * nn;
      fill<<<grid1(nn), 256>>>(phic, nn, t_ic);                 // t = 0: T_IC at every node
      fill<<<grid1(m * m), 256>>>(u, m * m, t_ic);
      for (uint32_t t = 1; t < tau; ++t) {
        add_boundary<<<grid1(m * m), 256>>>((int)m, c, ch, u, a);
        dgemm_nn<<<gg, 256>>>((int)m, (int)m, (int)m, S, a, b);  // S (u + c b)
        dgemm_nn<<<gg, 256>>>((int)m, (int)m, (int)m, b, S, a);  // ... S
        divide_denominator<<<grid1(m * m), 256>>>((int)m, (int)n, alpha * dt, hh, a);
        dgemm_nn<<<gg, 256>>>((int)m, (int)m, (int)m, S, a, b);
        dgemm_nn<<<gg, 256>>>((int)m, (int)m, (int)m, b, S, u);
        assemble<<<grid1(nn), 256>>>((int)n, c, u, phic + (uint64_t)t * nn);
      }
    }
    if (cudaDeviceSynchronize() != cudaSuccess || cudaGetLastError() != cudaSuccess) st = ST_ECUDA;
  }
  cudaFree(S); cudaFree(u); cudaFree(a); cudaFree(b);
  if (st) {
    cudaFree(h->phi);
    delete h;
    return st;
  }
  *out = h;
  return ST_OK;
}

uint64_t mel_heat_basis_bytes(const mel_heat* h) { return h ? h->bytes : 0; }
uint32_t mel_heat_grid(const mel_heat* h) { return h ? h->n : 0; }
uint32_t mel_heat_tau(const mel_heat* h) { return h ? h->tau : 0; }

int mel_heat_fields(mel_heat* h, const float* X, const uint32_t* t, uint32_t k, float* out, void* stream) {
  if (!h || !X || !t || !out || k == 0 || k > 65535) return ST_EINVAL;
  const uint32_t nn = h->n * h->n;
  const unsigned gx = (unsigned)((nn + 256 * 8 - 1) / (256 * 8));
  if (launch_pdl(combine, dim3(gx, k), dim3(256), 0, (cudaStream_t)stream, nn, h->tau, (const double*)h->phi, X, t,
                 out) != cudaSuccess)
    return ST_ECUDA;
  return ST_OK;
}

void mel_heat_destroy(mel_heat* h) {
  if (!h) return;
  cudaFree(h->phi);
  delete h;
}

}  // extern "C"
