// Internal launch interface between the ABI layer (mel.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace mel {

constexpr int HIST_BINS = 64;

// Reservoir device state (one per rank), DESIGN.md "Data layout in HBM".
struct ResDev {
  uint64_t q;          // committed puts (put_seq of the next item)
  uint64_t d;          // draws (SAMPLE + DRAIN counters)
  uint64_t evictions;
  uint64_t consumed;   // staging-ring entries consumed by commits
  uint32_t p;          // population
  uint32_t u;          // unseen items
  uint32_t over;       // closed && pending empty
  uint32_t n_last;     // size of the last batch (0 = EAGAIN / empty)
  uint32_t n_plan;     // entries committed by the last commit
  uint32_t head;       // FIFO: ring position of the oldest item
  uint32_t bad_batch;  // the current batch holds an item with non-finite X or field values
  uint32_t pad0;
  uint64_t hist[HIST_BINS];
};

// Host-visible mirror (mapped pinned memory), written at the end of the
// reservoir kernels and of the step; read by the host after a stream sync.
struct Mirror {
  uint64_t consumed, q, d, evictions;
  uint32_t p, u, over, n_last;
  uint64_t adam_k, samples;
  double loss;
  double n_total;
  int32_t status;      // step: 0 ok, 1 skip (no samples), 3 skipped: non-finite inputs or loss
  uint32_t pad;
  // per-call results of the last MEL_RESULT_RING surrogate_step calls (slot = call % ring),
  // read by surrogate_step_result without draining the stream
  double ring_loss[16];
  int32_t ring_status[16];
};
constexpr int MEL_RESULT_RING = 16;

struct StMeta {        // staging-ring metadata (32 B)
  uint32_t sim, t;
  float X[5];
  uint32_t pad;
};
typedef StMeta SlotMeta;

// per-step scalars computed on device (loss finalize -> Adam)
struct StepDev {
  double red[2];       // [sse, n] (all-reduced when world > 1)
  double loss;
  float scale;         // 1 / (N * n_total)
  float lr, c1, c2;    // lr and Adam bias corrections 1 - beta^k
  uint64_t k, S;       // Adam step, global samples consumed
  int32_t skip;        // no samples this step
  int32_t nonfinite;
  double n_glob;       // this rank's batch size, all-reduced ahead of K1 (exchange mode)
};

struct ResArgs {
  ResDev* st;
  Mirror* mirror;
  const StMeta* st_meta;
  const float* st_field;     // staging ring [S][Npad] fp32 kelvin
  uint32_t S;
  SlotMeta* meta;            // [C]
  uint32_t* seen;            // [C]
  uint64_t* put_seq;         // [C]
  uint32_t* bitmap;          // [ceil(C/32)]
  uint32_t* pos;             // [C]
  uint32_t* bad;             // [C] slot holds non-finite X or field values (set at commit)
  void* payload;             // [C][Npad] f32 or bf16
  uint32_t C, theta;
  uint64_t Npad;
  uint32_t N;
  int storage;
  float lo, span;
  uint64_t seed;
  uint32_t rank;
  uint2* plan;               // [S] (entry, slot)
  uint32_t policy;           // 0 Reservoir, 1 FIFO, 2 FIRO (mel_policy)
  const float* const* st_src;  // [S] mapped: the caller's device field of a zero-copy put, else null
  const float** plan_src;      // [S] the source field of plan entry i (null: the staging ring)
};

// reservoir.cu
void launch_commit(const ResArgs& a, uint64_t tail, uint32_t closed, uint32_t max_entries, cudaStream_t s);
void launch_sample(const ResArgs& a, int32_t* slots, uint32_t B, cudaStream_t s);
// Reservoir policy: commit control + sample in one launch, then the commit's data plane
void launch_commit_sample(const ResArgs& a, uint64_t tail, uint32_t closed, uint32_t max_entries, int32_t* slots,
                          uint32_t B, cudaStream_t s);
void launch_gather(const ResArgs& a, const int32_t* slots, uint32_t B, uint32_t tau, float* xn, cudaStream_t s);
void launch_init_res(const ResArgs& a, cudaStream_t s);

// mlp_simt.cu
enum Epi { EPI_STORE = 0, EPI_BIAS_RELU = 1, EPI_BIAS = 2, EPI_RELU_MASK = 3 };
// optional epilogue outputs / inputs: Hb = bf16 copy of H (EPI_BIAS_RELU), mask = Z whose
// ReLU' multiplies the result (EPI_RELU_MASK, ReLU'(0) = 0, reading R20)
struct EpiExtra {
  __nv_bfloat16* Hb = nullptr;
  const float* mask = nullptr;
  int ldm = 0;
};
void sgemm(bool ta, bool tb, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
           float* C, int ldc, int epi, const float* bias, float* H, int ldh, int splits, cudaStream_t s, EpiExtra ex = EpiExtra());
int sgemm_auto(bool ta, bool tb, int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C, int ldc,
               int epi, const float* bias, float* H, int ldh, float* scratch, size_t scratch_elems, cudaStream_t s, EpiExtra ex = EpiExtra());
void splitk_reduce(int M, int N, int splits, const float* part, float* C, int ldc, const float* relu_mask,
                   int ldm, cudaStream_t s);
struct OutArgs {
  const float* H; int ldh;        // [B][K]
  const float* W; const float* b; // W [Npad][K], b [Npad]
  int K;
  const void* payload; int storage; uint64_t Npad; uint32_t N;
  const int32_t* slots; const ResDev* st;   // n_valid = st->n_last
  float* dY;                      // [B][Npad] raw dS/dY = 2 (Y - T) (0 outside valid)
  double* sse_part;               // per-block partial sums
  int B;
};
int out_fwd_f32(const OutArgs& a, cudaStream_t s);   // returns number of partials
void col_sum(const float* X, int rows, int cols, int ld, float* out, cudaStream_t s);
// column sums of two matrices with the same row count in one launch (X1 nullable)
void col_sum2(const float* X0, int cols0, int ld0, float* out0, const float* X1, int cols1, int ld1, float* out1,
              int rows, cudaStream_t s);
void reduce_local(StepDev* sd, const double* parts, int n_parts, const ResDev* st, cudaStream_t s);
void step_finalize(StepDev* sd, double n_field, double lr0, double lr_min, uint64_t halving, double b1, double b2,
                   Mirror* mirror, ResDev* st, cudaStream_t s, uint32_t slot = 0);
void step_prepare(StepDev* sd, const ResDev* st, double n_field, double lr0, double lr_min, uint64_t halving, double b1,
                  double b2, cudaStream_t s, bool global_n = false);   // global_n: use sd->n_glob
void stage_count(StepDev* sd, const ResDev* st, cudaStream_t s);     // sd->n_glob = st->n_last
// virtual ranks: bufs[q][i] <- sum over q of bufs[q][i] (rank order), for every q; d_bufs is a
// device array of R pointers
void vsum_f32(float* const* d_bufs, int R, uint64_t n, cudaStream_t s);
void vsum_f64(double* const* d_bufs, int R, uint64_t n, cudaStream_t s);
void adam_flat(float* p, float* m, float* v, const float* g, uint64_t n, const StepDev* sd,
               float b1, float b2, float eps, __nv_bfloat16* shadow, uint64_t sh_begin, uint64_t sh_end,
               cudaStream_t s);
void init_tensor(float* dst, uint64_t count, uint32_t tid, uint32_t fan_in, uint64_t seed, cudaStream_t s);
void to_bf16(const float* src, __nv_bfloat16* dst, uint64_t n, cudaStream_t s);
void relu_mask_mul(float* X, const float* Z, uint64_t n, cudaStream_t s);
int eval_mse_partial(const float* Y, const float* T, int rows, int cols, int ld, double* part, cudaStream_t s);
void eval_inputs(const float* X, const uint32_t* t, int n, uint32_t tau, float lo, float span, float* xn, cudaStream_t s);
void normalise_fields(const float* src, float* dst, uint64_t n, float lo, float span, cudaStream_t s);

// Fused head of the paper's network (two hidden layers; d0 <= 8 inputs, hidden widths
// <= 256 and multiples of 32).  head3_init: once per process (dynamic SMEM attributes).
int head3_init();
int head_fwd3_ctas(int B);
// forward in one launch: the batch inputs gathered from the slot metadata (gather_inputs'
// arithmetic), Z1/H1, Z2/H2 (+ the bf16 copy of H2); with sd set, the last CTA to finish
// also computes step_prepare's scalars (world 1, fused Adam) once every bad-input flag is in
struct HeadFwdArgs {
  ResArgs ra;
  const int32_t* slots;
  uint32_t B, tau;
  const float *W1, *b1, *W2, *b2;
  int d0, d1, d2;
  float *xn, *Z1, *H1, *Z2, *H2;
  __nv_bfloat16* Hb;                    // nullable
  StepDev* sd;                          // nullable: no fused prepare
  double n_field, lr0, lr_min, beta1, beta2;
  uint64_t halving;
  uint32_t* counter;                    // monotonic CTA-arrival counter (prepare)
  uint32_t target;                      // its value once every CTA of this launch arrived
};
void head_fwd3(const HeadFwdArgs& a, cudaStream_t s);
// backward in two launches, given dZ2 (ReLU' applied).  head_bwd3_kernel: row CTAs compute
// dZ1 = (dZ2 W2) . ReLU'(Z1) for HEAD_R rows and their partial dW1 / db1 sums; dW2 CTAs the
// partial dW2 = dZ2^T H1 (+ db2, fp64) of a 64-row batch slice.  head_fin3_kernel: the
// fixed-order reductions into the gradient (deterministic); with sd set (world 1) it also
// folds K1's SSE partials and runs step_finalize's scalars.
struct HeadBwdArgs {
  const float *dz2, *W2, *z1, *h1, *xn;
  int B, d0, d1, d2;
  float *gW1, *gb1, *gW2, *gb2;
  float* p_dw1;                         // [row CTAs][d1][8]
  double* p_db1;                        // [row CTAs][d1]
  float* p_dw2;                         // [slices][d2][d1]
  double* p_db2;                        // [slices][d2]
  // fused reduce_local + step_finalize (world 1); sd == nullptr: off
  StepDev* sd;
  const double* sse_parts;
  int n_sse_parts;
  ResDev* st;
  Mirror* mirror;
  uint32_t slot;
  double n_field, lr0, lr_min, beta1, beta2;
  uint64_t halving;
};
__host__ __device__ inline int head_bwd3_row_ctas(int B) { return (B + 31) / 32; }   // row blocks (partials)
void head_bwd3(const HeadBwdArgs& a, cudaStream_t s);
size_t head_dw2_part_elems(int B, int d1, int d2);

}  // namespace mel
