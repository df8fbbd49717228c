// Tensor-core (tcgen05 / TMEM / TMA) output layer of the surrogate, bf16 mode.
// See tc_out.cu and DESIGN.md "Kernels".
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace mel {
namespace tc {

struct TcBuffers {
  __nv_bfloat16* h_bf16 = nullptr;   // [B][K] last hidden activations (bf16)
  __nv_bfloat16* dyT = nullptr;      // [Npad][B] dS/dY transposed (bf16)
  float* ring = nullptr;             // overlapped K1: per-CTA dW hand-off ring [160][2][128][K] fp32
  void* ctl = nullptr;               // overlapped K1: queue / ring counters (tc_out.cu K1Ctl)
  void* entries = nullptr;           // overlapped K1: queue of handed-off tiles [Npad / 128]
  void* maps = nullptr;              // device copy of the TMA descriptors
  void* h_maps = nullptr;            // host copies (CUtensorMap)
  uint64_t Npad = 0;
  uint32_t B = 0, K = 0;
  int dh_splits = 0;
  int fwd_ctas = 0;
};

constexpr int MAX_WORLD = 8;

// In-kernel exchange: owner rank of W_L tile t (128 rows) when K1 runs on G CTAs, tile
// t = b + G*i going to CTA b in its i-th iteration.  Every CTA alternates between tiles it
// owns and tiles it sends, and every wave splits evenly across owners, so both NVLink
// directions stay busy and no CTA carries more Adam work than another.
__host__ __device__ inline uint32_t tile_owner(uint32_t t, uint32_t G, uint32_t R) { return (t % G + t / G) % R; }

struct OutTcArgs {
  uint32_t N, B, K;
  uint64_t Npad;
  const __nv_bfloat16* w_bf16;       // [Npad][K] shadow of W_L
  const float* b;                    // [Npad] b_L
  const __nv_bfloat16* h_bf16;       // [B][K]
  const __nv_bfloat16* payload;      // reservoir slots [C][Npad] bf16 (normalised)
  const int32_t* slots;              // [B]
  const ResDev* st;                  // n_valid = st->n_last
  __nv_bfloat16* dyT;                // out: [Npad][B]
  float* gW;                         // out: raw dS/dW_L [Npad][K]
  float* gb;                         // out: raw dS/db_L [Npad]
  double* sse_part;                  // out: per-CTA SSE partials
  float* dh_part;                    // scratch: split-K partials of dS/dH
  float* dz;                         // out: dS/dZ_{L-1} [B][K]
  const float* z;                    // Z_{L-1} [B][K] (ReLU mask)
  int shadow_idx;                    // which ping-pong W_L shadow K1 and K2 read
  int fused_adam;                    // K1 applies Adam to W_L (world == 1)
  float *adam_p, *adam_m, *adam_v;   // W_L fp32 master / moments (fused)
  __nv_bfloat16* shadow_out;         // updated bf16 shadow (fused), the other buffer
  const StepDev* sd;                 // step scalars (scale, lr, bias corrections, skip)
  uint32_t k1_seq;                   // launch counter (tags the overlapped K1's queue entries)
  float b1, b2, eps;
  // in-kernel exchange (world > 1, bf16; tc_out.cu K1Params): the fused Adam runs on the
  // tiles this rank owns, the other tiles' dW are reduce-added into their owners' acc
  int peer;
  uint32_t rank, world, epoch;
  uint32_t acc_bf16;
  uint32_t* cnt_local;
  uint32_t* cnt_peer[MAX_WORLD];
  __nv_bfloat16* sh_peer[MAX_WORLD];
};

int alloc_buffers(TcBuffers& t, uint64_t Npad, uint32_t B, uint32_t K);
// tensor maps of the in-kernel exchange: this rank's acc and every rank's (peer-mapped) acc
int prepare_peer(TcBuffers& t, uint32_t K, uint64_t rows, int rank, int world, void* const* acc, bool acc_bf16,
                 __nv_bfloat16* const* sh0, __nv_bfloat16* const* sh1);
// dst = src on the rows of the tiles `rank` owns, 0 elsewhere ([Npad][K] fp32)
void owned_rows(const TcBuffers& t, const float* src, float* dst, uint32_t K, int rank, int world, cudaStream_t s);
inline uint32_t k1_grid(const TcBuffers& t) {                // CTAs of a full-range K1 launch
  const uint32_t tiles = (uint32_t)(t.Npad / 128);
  return tiles < (uint32_t)t.fwd_ctas ? tiles : (uint32_t)t.fwd_ctas;
}
void free_buffers(TcBuffers& t);
int prepare(TcBuffers& t, uint64_t Npad, uint32_t B, uint32_t K, const __nv_bfloat16* const* w_bf16,
            const __nv_bfloat16* payload, uint32_t capacity, const float* grad_w, int sm_reserve,
            const float* p_w, const float* m_w, const float* v_w);   // TMA descriptors, kernel attributes
size_t dh_part_elems(uint32_t B, uint32_t K);
int max_sse_parts(uint64_t Npad);
// forward + MSE gradient + dW_L/db_L (per 128-row tile of W_L); returns #SSE partials
int launch_out_fwd_dw(const OutTcArgs& a, const TcBuffers& t, cudaStream_t s, uint32_t tile0 = 0, uint32_t tile1 = 0,
                      uint32_t part_base = 0);
// virtual ranks (mel_create_virtual): ONE cooperative K1 launch over R ranks' tiles, each
// rank's maps + parameters copied into d_desc (R x virt_desc_bytes() device bytes); returns
// the per-rank CTA count (= SSE partials per rank)
int launch_out_fwd_dw_virtual(const OutTcArgs* a, const TcBuffers* const* t, int R, void* d_desc, cudaStream_t s);
int virt_desc_bytes();
// dst = src on the rows of the tiles `rank` owns, untouched elsewhere ([Npad][K] fp32)
void copy_owned_rows(const TcBuffers& t, const float* src, float* dst, uint32_t K, int rank, int world, cudaStream_t s);
// dS/dH = dY W_L (split-K over N) then the ReLU' mask -> dz
void launch_out_dh(const OutTcArgs& a, const TcBuffers& t, cudaStream_t s);
const char* last_error();
int read_k1_profile(unsigned long long* out, int n);

}  // namespace tc
}  // namespace mel
