/*
 * mel_heat.h -- C ABI of the on-device heat-equation client: the
 * data generator of the paper's experiments running on the training GPU itself, so that
 * generation and training share one allocation.
 *
 * What the paper fixes (§4.1, Eq. 2): dT/dt = alpha lap(T) on a square,
 * T(.,.,0) = T_IC, Dirichlet T_x1, T_x2 (x = 0, L), T_y1, T_y2 (y = 0, L); finite
 * differences with implicit Euler on an n x n grid (1000 x 1000), 100 steps of dt = 0.01,
 * alpha = 1; X = (T_IC, T_x1, T_y1, T_x2, T_y2) in [100, 500] K; fields leave the client
 * as fp32.  Readings Q16-Q19: unit square, h = L/(n-1), t = 0 emits
 * T_IC everywhere, edges carry their Dirichlet value and corners the mean of the two
 * adjacent ones for t >= 1, the implicit system solved exactly.
 *
 * Method (B200): the scheme is linear in X, so u_X^t = sum_c X_c phi_c^t with phi_c the
 * solution for X = e_c.  mel_heat_create computes the 5 x tau basis fields on the GPU in
 * fp64 (each implicit step exactly, by DST-I diagonalisation of the 5-point Laplacian:
 * u <- S ((S (u + b) S) / (1 + alpha dt (lambda_i + lambda_j))) S, S the orthonormal DST-I
 * matrix, as fp64 GEMMs), and keeps it in HBM (5 tau n^2 doubles: 4 GB at paper shape).
 * A field is then one fused kernel pass: out = RNE_fp32(sum_c X_c phi_c^t).
 *
 * Conventions: int status (0 OK, -1 MEL_EINVAL, -4 MEL_ECUDA, -6 MEL_ENOMEM).  Device
 * pointers are named *_dev and are used in stream order on `stream` (a cudaStream_t, NULL
 * = the legacy default stream); *_host pointers are read during the call.
 */
#ifndef MEL_HEAT_H_
#define MEL_HEAT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef MEL_HEAT_TYPEDEF_
#define MEL_HEAT_TYPEDEF_
typedef struct mel_heat mel_heat;
#endif

/* Builds the basis on the current CUDA device (blocking).  n >= 3, tau >= 1, alpha, dt,
 * length > 0.  MEL_ENOMEM if the basis does not fit. */
int mel_heat_create(uint32_t n, uint32_t tau, double alpha, double dt, double length, mel_heat** out);

/* Bytes of HBM the basis holds; grid size n; time steps tau. */
uint64_t mel_heat_basis_bytes(const mel_heat* h);
uint32_t mel_heat_grid(const mel_heat* h);
uint32_t mel_heat_tau(const mel_heat* h);

/* out_dev[j][0..n*n) = u_{X_j}^{t_j} as fp32 kelvin (RNE of the fp64 combination), for
 * j < k; X_dev is [k][5] fp32 kelvin, t_dev [k] (each < tau).  Layout k = row*n + col,
 * row = y index.  MEL_EINVAL on a null pointer or k = 0. */
int mel_heat_fields(mel_heat* h, const float* X_dev, const uint32_t* t_dev, uint32_t k, float* out_dev,
                    void* stream);

/* Frees the basis. */
void mel_heat_destroy(mel_heat* h);

#ifdef __cplusplus
}
#endif
#endif
