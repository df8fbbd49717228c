// libmel C ABI (include/mel.h): context, device arenas, streams, op sequencing
// of the reservoir-fed training step, NCCL gradient all-reduce.  Host logic only;
// every step of the method runs in the kernels of reservoir.cu, mlp_simt.cu and
// tc_out.cu.
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <future>
#include <string>
#include <vector>

#include "../../include/mel.h"
#include "../../include/mel_ingest.h"
#include "../../include/mel_dataset.h"
#include "../../include/mel_heat.h"
#include "kernels.h"
#include "tc_out.h"

using namespace mel;

namespace {

struct TimedPair {
  int k;
  cudaEvent_t a, b;
};

}  // namespace

// Virtual ranks (mel_create_virtual): R contexts on one device and one stream; the
// collectives are device-side rank-ordered sums over the members' buffers and K1 runs as one
// cooperative launch over every member's tiles (tc::launch_out_fwd_dw_virtual).
struct VGroup {
  int R = 0, refs = 0;
  mel_ctx* cs[tc::MAX_WORLD] = {};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  void* d_desc = nullptr;                  // K1Virt[R]
  float** d_tab_g = nullptr;               // [R] every member's flat gradient buffer
  double** d_tab_red = nullptr;            // [R] &d_sd->red[0]
  double** d_tab_nglob = nullptr;          // [R] &d_sd->n_glob
};

struct mel_ctx {
  mel_config cfg{};
  bool virt = false;                        // a member of a virtual-rank group
  VGroup* vg = nullptr;
  int rank = 0, world = 1, dev = 0;
  cudaStream_t stream = nullptr, copy_stream = nullptr;
  bool own_stream = false;
  std::string err;
  int poisoned = 0;

  // model geometry
  int L = 0;                       // number of weight layers
  uint32_t dims[4] = {0, 0, 0, 0}; // [6, hidden..., N]
  uint32_t N = 0, B = 0, C = 0, Klast = 0, hmax = 0;
  uint32_t Bs = 0;                 // batch the sampler draws (cfg.batch); B = rows the kernels run
                                   // (bf16: Bs padded to the 64-row K1 chunk, rows >= n masked)
  uint64_t Npad = 0;
  uint64_t off[2 * 3] = {};        // tensor offsets in the flat buffers
  uint64_t cnt[2 * 3] = {};
  uint64_t n_flat = 0;

  // reservoir
  ResArgs ra{};
  ResDev* d_st = nullptr;
  Mirror* h_mirror = nullptr;
  Mirror* d_mirror = nullptr;
  StMeta* h_stmeta = nullptr;      // pinned ring mirror of staging metadata
  const float** h_stsrc = nullptr; // pinned [S]: a zero-copy device put's field, else null
  uint64_t tail = 0;               // accepted puts
  uint64_t known_consumed = 0;
  bool copy_fence = false;                  // see ensure_ring_space
  uint64_t drawn = 0;                       // items handed out (FIFO / FIRO remove them)
  uint64_t calls = 0;                       // surrogate_step calls (surrogate_step_result)
  cudaEvent_t ev_call[MEL_RESULT_RING] = {};
  bool closed = false;
  bool copy_pending = false;
  cudaEvent_t ev_copy = nullptr, ev_fence = nullptr;
  void* ing_base = nullptr;                 // ingest segment page-locked for DMA (reservoir_ingest)
  uint64_t ing_bytes = 0;
  bool ing_pinned = false;
  static constexpr int ING_EVENTS = 8;      // deferred slot releases: one event per ingest call
  cudaEvent_t ing_ev[ING_EVENTS] = {};
  uint32_t ing_cnt[ING_EVENTS] = {};
  uint32_t ing_head = 0, ing_n = 0;         // FIFO of (event, message count) not yet released
  mel_ingest* ing_handle = nullptr;
  float* d_gen = nullptr;                   // on-device client scratch (reservoir_put_generated)
  float* d_gen_x = nullptr;
  uint32_t* d_gen_t = nullptr;
  float* off_buf[2] = {};                   // offline loader: pinned chunk buffers (surrogate_train_offline)
  uint32_t off_chunk = 0;
  cudaEvent_t off_ev[2] = {};
  int32_t* d_slots = nullptr;
  bool batch_known = false;        // host knows the last batch size
  uint32_t batch_n = 0;

  // parameters (flat fp32: p, m, v, g) and the bf16 shadow(s) of the output layer
  float *d_p = nullptr, *d_m = nullptr, *d_v = nullptr, *d_g = nullptr;
  __nv_bfloat16* d_shadow[2] = {nullptr, nullptr};
  int shadow_cur = 0;

  // activations / scratch
  float* d_xn = nullptr;           // [B][8]
  float* d_z[2] = {nullptr, nullptr};
  float* d_h[2] = {nullptr, nullptr};
  float* d_dz[2] = {nullptr, nullptr};
  float* d_dy = nullptr;           // fp32 mode [B][Npad]
  // fused head (two hidden layers): one forward and one backward launch per step
  bool head_fused = false;
  bool prep_fused = false;         // this step's step_prepare ran inside the head forward
  int last_nparts = 0;             // K1's SSE partials of this step
  uint32_t* d_hcnt = nullptr;      // monotonic CTA-arrival counter of the head forward
  uint32_t hf_n = 0;               // head-forward launches with the fused prepare so far
  float* d_hp_dw1 = nullptr;       // [row CTAs][d1][8] partial dW1
  double* d_hp_db1 = nullptr;      // [row CTAs][d1] partial db1
  float* d_hp_dw2 = nullptr;       // [64-row slices][d2][d1] partial dW2
  double* d_hp_db2 = nullptr;      // [64-row slices][d2] partial db2
  float* d_part = nullptr;         // split-K partials
  size_t part_elems = 0;
  double* d_sse_part = nullptr;
  int max_parts = 0;
  StepDev* d_sd = nullptr;
  tc::TcBuffers tcb{};

  // eval scratch (lazy)
  float* d_eval_x = nullptr; uint32_t* d_eval_t = nullptr; float* d_eval_y = nullptr; float* d_eval_f = nullptr;
  float *d_eval_z[2] = {nullptr, nullptr}, *d_eval_h[2] = {nullptr, nullptr}; float* d_eval_xn = nullptr;

  ncclComm_t comm = nullptr;
  // ZeRO-1 style exchange (world > 1, bf16 mode): reduce-scatter of dW_L on a comm
  // stream overlapped with the rest of the backward, Adam on this rank's W_L row
  // shard, all-gather of the bf16 shadow
  bool zero = false;
  bool fused_adam = false;                  // world == 1, bf16: Adam of W_L inside K1
  uint64_t shard_elems = 0, shard_off = 0;   // W_L elements per rank, this rank's offset in W_L
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_gw = nullptr, ev_head = nullptr, ev_ar = nullptr, ev_adam = nullptr, ev_ag = nullptr;
  bool ag_pending = false;
  // bucketed pipeline: K1 runs over NB tile ranges; bucket j's dW_L reduce-scatter overlaps
  // K1 of bucket j+1, and the next step's K1 bucket j waits only for its shadow all-gather
  static constexpr int NBMAX = 8;
  int nb = 1;
  uint32_t bt0[NBMAX] = {}, bt1[NBMAX] = {};
  cudaEvent_t ev_k1[NBMAX] = {}, ev_agb[NBMAX] = {};
  int sm_reserve = 0;
  // in-kernel exchange (world > 1, bf16, default; MEL_FLAG_NCCL_EXCHANGE turns it off):
  // every rank TMA-reduce-adds the dW tiles it does not own into the owner's acc over
  // NVLink (CUDA IPC mappings), owners run the fused Adam and write the bf16 shadow rows to
  // every rank from inside K1; only the small region + [SSE, n] go through NCCL
  bool peer = false;
  void* d_acc = nullptr;                    // [Npad][Klast] bf16 (fp32 with MEL_FLAG_FP32_EXCHANGE): peers' dW sum
  bool acc_bf16 = false;
  uint32_t* d_cnt = nullptr;                // [Npad / 128] arrival counters (owned tiles)
  void* p_acc[tc::MAX_WORLD] = {};          // every rank's acc / counters / shadows (IPC)
  uint32_t* p_cnt[tc::MAX_WORLD] = {};
  __nv_bfloat16* p_sh[2][tc::MAX_WORLD] = {};
  uint32_t epoch = 0;
  uint32_t k1_launches = 0;                 // tags the overlapped K1's hand-off queue entries

  // timing
  std::vector<TimedPair> pending;
  std::vector<cudaEvent_t> ev_pool;
  double kms[MEL_K_COUNT] = {};
  uint64_t klaunch[MEL_K_COUNT] = {};
  uint64_t launches = 0;
};

namespace {

int fail(mel_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) {
    c->err = buf;
    if (code == MEL_ECUDA || code == MEL_ENCCL) c->poisoned = code;
  }
  return code;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(c, MEL_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                 \
  } while (0)

#define NK(call)                                                                                \
  do {                                                                                          \
    ncclResult_t r_ = (call);                                                                   \
    if (r_ != ncclSuccess) return fail(c, MEL_ENCCL, "%s failed: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

#define GUARD(c)                                 \
  do {                                           \
    if (!(c)) return MEL_EINVAL;                 \
    if ((c)->poisoned) return (c)->poisoned;     \
    cudaSetDevice((c)->dev);                     \
  } while (0)

template <class T>
int dalloc(mel_ctx* c, T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, MEL_ENOMEM, "cudaMalloc(%zu bytes) failed: %s", count * sizeof(T), cudaGetErrorString(e));
  }
  return MEL_OK;
}

#define DALLOC(p, n)                      \
  do {                                    \
    int r_ = dalloc(c, &(p), (size_t)(n)); \
    if (r_) return r_;                    \
  } while (0)

cudaEvent_t take_event(mel_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// RAII-free timing brackets around one launch group of kernel class k
struct Timer {
  mel_ctx* c; int k; cudaEvent_t a = nullptr; cudaStream_t st;
  Timer(mel_ctx* c_, int k_, int nlaunch, cudaStream_t s_ = nullptr) : c(c_), k(k_), st(s_ ? s_ : c_->stream) {
    c->launches += nlaunch;
    c->klaunch[k] += nlaunch;
    if (c->cfg.flags & MEL_FLAG_TIMING) { a = take_event(c); cudaEventRecord(a, st); }
  }
  ~Timer() {
    if (a) {
      cudaEvent_t b = take_event(c);
      cudaEventRecord(b, st);
      c->pending.push_back({k, a, b});
    }
  }
};

void drain_timers(mel_ctx* c) {
  for (auto& t : c->pending) {
    float ms = 0.f;
    cudaEventSynchronize(t.b);
    cudaEventElapsedTime(&ms, t.a, t.b);
    c->kms[t.k] += ms;
    c->ev_pool.push_back(t.a);
    c->ev_pool.push_back(t.b);
  }
  c->pending.clear();
}

int check_launch(mel_ctx* c, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, MEL_ECUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
  return MEL_OK;
}

int sync_stream(mel_ctx* c) {
  CK(cudaStreamSynchronize(c->stream));
  c->known_consumed = c->h_mirror->consumed;
  return MEL_OK;
}

int validate(const mel_config* g, int world, mel_ctx* c) {
  if (g->abi_version != MEL_ABI_VERSION) return fail(c, MEL_EINVAL, "abi_version %u != %u", g->abi_version, MEL_ABI_VERSION);
  if (g->n_field == 0) return fail(c, MEL_EINVAL, "n_field must be > 0");
  if (g->hidden[0] == 0) return fail(c, MEL_EINVAL, "hidden[0] must be > 0");
  if (g->capacity == 0 || g->threshold >= g->capacity) return fail(c, MEL_EINVAL, "require threshold < capacity (P:321)");
  if (g->batch == 0) return fail(c, MEL_EINVAL, "batch must be > 0");
  if (g->steps_per_sim == 0) return fail(c, MEL_EINVAL, "steps_per_sim must be > 0");
  if (!(g->temp_hi > g->temp_lo)) return fail(c, MEL_EINVAL, "temp_hi must exceed temp_lo");
  if (g->precision > MEL_BF16 || g->storage > MEL_STORE_BF16) return fail(c, MEL_EINVAL, "bad precision/storage");
  if (g->staging_entries == 0) return fail(c, MEL_EINVAL, "staging_entries must be >= 1");
  if (g->policy > MEL_FIRO) return fail(c, MEL_EINVAL, "unknown buffer policy %u", g->policy);
  if (!(g->eps > 0.0) || !(g->beta1 >= 0.0 && g->beta1 < 1.0) || !(g->beta2 >= 0.0 && g->beta2 < 1.0))
    return fail(c, MEL_EINVAL, "Adam needs eps > 0 and 0 <= beta < 1");
  if (g->policy == MEL_FIFO && g->batch > g->capacity) return fail(c, MEL_EINVAL, "FIFO needs batch <= capacity");
  if (g->policy == MEL_FIRO && (uint64_t)g->threshold + g->batch > g->capacity)
    return fail(c, MEL_EINVAL, "FIRO needs threshold + batch <= capacity");
  if (g->lr_halving_samples == 0) return fail(c, MEL_EINVAL, "lr_halving_samples must be > 0");
  const uint32_t klast = g->hidden[1] ? g->hidden[1] : g->hidden[0];
  if (g->precision == MEL_BF16) {
    if (klast % 64 != 0 || klast > 256) return fail(c, MEL_EINVAL, "bf16 mode needs the last hidden width in {64,128,192,256}");
    if (g->storage != MEL_STORE_BF16) return fail(c, MEL_EINVAL, "bf16 mode stores targets as bf16 (MEL_STORE_BF16)");
  }
  if (world < 1) return fail(c, MEL_EINVAL, "world must be >= 1");
  return MEL_OK;
}

// A put needs a free staging entry.  The commit kernel publishes its progress in the
// mapped mirror, so instead of draining the stream the host polls it while the queued
// steps run (the host may be many steps ahead); only an idle stream with the ring still
// full is back-pressure (MEL_EAGAIN).  Entries freed this way may still be read by a
// queued commit_copy, so the next host-buffer put fences the copy stream (copy_fence).
int ensure_ring_space(mel_ctx* c) {
  const uint32_t S = c->cfg.staging_entries;
  if (c->tail - c->known_consumed < S) return MEL_OK;
  for (;;) {
    const uint64_t seen = *reinterpret_cast<volatile uint64_t*>(&c->h_mirror->consumed);
    if (seen > c->known_consumed) {
      c->known_consumed = seen;
      c->copy_fence = true;
    }
    if (c->tail - c->known_consumed < S) return MEL_OK;
    const cudaError_t q = cudaStreamQuery(c->stream);
    if (q == cudaSuccess) {
      int r = sync_stream(c);
      if (r) return r;
      return c->tail - c->known_consumed < S ? MEL_OK : MEL_EAGAIN;
    }
    if (q != cudaErrorNotReady) return fail(c, MEL_ECUDA, "stream query: %s", cudaGetErrorString(q));
    struct timespec ts{0, 20000};
    nanosleep(&ts, nullptr);
  }
}

int commit(mel_ctx* c) {
  const uint64_t max_e = c->tail - c->known_consumed;
  if (c->copy_pending) {
    CK(cudaStreamWaitEvent(c->stream, c->ev_copy, 0));
    c->copy_pending = false;
  }
  {
    Timer t(c, MEL_K_COMMIT, max_e ? 2 : 1);
    launch_commit(c->ra, c->tail, c->closed ? 1u : 0u, (uint32_t)max_e, c->stream);
  }
  return check_launch(c, "commit");
}

// Gradient exchange (the locally computed gradients are all-reduced so that
// every replica applies the same mean update).  Plain mode: one grouped all-reduce of
// the flat fp32 gradients + [SSE, n].  ZeRO mode: the W_L gradient is reduce-scattered
// on the comm stream as soon as K1 has written it (overlapping K2 and the head
// backward); the small region (head weights, every bias) and [SSE, n] are
// all-reduced after the head backward.  Same sums, same mean update.
int world_exchange(mel_ctx* c) {
  if (c->world == 1) return MEL_OK;
  if (!c->zero) {
    Timer t(c, MEL_K_ALLREDUCE, 0);
    NK(ncclGroupStart());
    NK(ncclAllReduce(c->d_g, c->d_g, c->n_flat, ncclFloat32, ncclSum, c->comm, c->stream));
    NK(ncclAllReduce(c->d_sd->red, c->d_sd->red, 2, ncclFloat64, ncclSum, c->comm, c->stream));
    NK(ncclGroupEnd());
    return MEL_OK;
  }
  const uint64_t offW = c->off[2 * (c->L - 1)];
  CK(cudaEventRecord(c->ev_head, c->stream));
  {
    Timer t(c, MEL_K_ALLREDUCE, 0, c->comm_stream);
    CK(cudaStreamWaitEvent(c->comm_stream, c->ev_head, 0));
    NK(ncclGroupStart());
    NK(ncclAllReduce(c->d_g, c->d_g, offW, ncclFloat32, ncclSum, c->comm, c->comm_stream));
    NK(ncclAllReduce(c->d_sd->red, c->d_sd->red, 2, ncclFloat64, ncclSum, c->comm, c->comm_stream));
    NK(ncclGroupEnd());
    CK(cudaEventRecord(c->ev_ar, c->comm_stream));
  }
  CK(cudaStreamWaitEvent(c->stream, c->ev_ar, 0));
  return MEL_OK;
}

// bucket j of W_L: rows [128 bt0, 128 bt1); this rank owns the r-th of R equal parts
inline uint64_t bucket_row0(const mel_ctx* c, int j) { return (uint64_t)c->bt0[j] * 128; }
inline uint64_t bucket_rows(const mel_ctx* c, int j) { return (uint64_t)(c->bt1[j] - c->bt0[j]) * 128; }
inline uint64_t part_elems(const mel_ctx* c, int j) { return bucket_rows(c, j) / c->world * c->Klast; }
inline uint64_t part_off(const mel_ctx* c, int j) {   // elements from the start of W_L
  return bucket_row0(c, j) * c->Klast + (uint64_t)c->rank * part_elems(c, j);
}

// all-gather of one bucket of a W_L-shaped buffer from the rank parts (comm stream)
int gather_bucket(mel_ctx* c, void* base, size_t esz, ncclDataType_t ty, int j) {
  char* b = static_cast<char*>(base) + bucket_row0(c, j) * c->Klast * esz;
  NK(ncclAllGather(b + (uint64_t)c->rank * part_elems(c, j) * esz, b, part_elems(c, j), ty, c->comm, c->comm_stream));
  return MEL_OK;
}
int gather_shards(mel_ctx* c, void* base, size_t esz, ncclDataType_t ty) {
  for (int j = 0; j < c->nb; ++j) {
    int r = gather_bucket(c, base, esz, ty, j);
    if (r) return r;
  }
  return MEL_OK;
}

// wait (device-side) for the pending shadow all-gather before anything reads W_L
int wait_shadow(mel_ctx* c) {
  if (c->ag_pending) {
    for (int j = 0; j < c->nb; ++j) CK(cudaStreamWaitEvent(c->stream, c->ev_agb[j], 0));
    c->ag_pending = false;
  }
  return MEL_OK;
}

// full fp32 W_L master (and moments) on every rank, for host reads (collective)
int gather_master(mel_ctx* c, bool moments) {
  if (!c->zero) return MEL_OK;
  const uint64_t offW = c->off[2 * (c->L - 1)];
  if (c->peer && c->virt) {
    // virtual ranks: the rows every other member owns, copied from its buffers
    const uint64_t offW = c->off[2 * (c->L - 1)];
    for (int q = 0; q < c->world; ++q) {
      if (q == c->rank) continue;
      mel_ctx* o = c->vg->cs[q];
      tc::copy_owned_rows(c->tcb, o->d_p + offW, c->d_p + offW, c->Klast, q, c->world, c->stream);
      if (moments) {
        tc::copy_owned_rows(c->tcb, o->d_m + offW, c->d_m + offW, c->Klast, q, c->world, c->stream);
        tc::copy_owned_rows(c->tcb, o->d_v + offW, c->d_v + offW, c->Klast, q, c->world, c->stream);
      }
    }
    return check_launch(c, "virtual gather");
  }
  if (c->peer) {
    // owners are interleaved by tile (tc::tile_owner): every rank contributes its owned
    // rows and zeros elsewhere; an integer sum of the bit patterns is an exact gather.
    // The W_L gradient region is free scratch in this mode.
    float* arrs[3] = {c->d_p + offW, c->d_m + offW, c->d_v + offW};
    float* tmp = c->d_g + offW;
    for (int i = 0; i < (moments ? 3 : 1); ++i) {
      tc::owned_rows(c->tcb, arrs[i], tmp, c->Klast, c->rank, c->world, c->stream);
      NK(ncclAllReduce(tmp, arrs[i], c->Npad * c->Klast, ncclUint32, ncclSum, c->comm, c->stream));
    }
    return MEL_OK;
  }
  CK(cudaEventRecord(c->ev_head, c->stream));
  CK(cudaStreamWaitEvent(c->comm_stream, c->ev_head, 0));
  NK(ncclGroupStart());
  int r = gather_shards(c, c->d_p + offW, 4, ncclFloat32);
  if (!r && moments) r = gather_shards(c, c->d_m + offW, 4, ncclFloat32);
  if (!r && moments) r = gather_shards(c, c->d_v + offW, 4, ncclFloat32);
  NK(ncclGroupEnd());
  if (r) return r;
  CK(cudaEventRecord(c->ev_ar, c->comm_stream));
  CK(cudaStreamWaitEvent(c->stream, c->ev_ar, 0));
  return MEL_OK;
}

// backward of the head layers given dZ of the last hidden layer (d_dz[L-2]); every
// GEMM is split-K through the partial buffer when its grid is below one wave
// world 1 with the fused head: reduce_local and step_finalize run inside the head backward's
// reduction launch (nothing is exchanged between them and the step's scalars)
inline bool fin_fused(const mel_ctx* c) { return c->head_fused && c->world == 1 && !c->virt; }

int head_backward(mel_ctx* c) {
  const int L = c->L;
  Timer t(c, MEL_K_HEAD_BWD, 0);
  uint64_t nl = 0;
  if (c->head_fused) {
    HeadBwdArgs a;
    a.dz2 = c->d_dz[1]; a.W2 = c->d_p + c->off[2]; a.z1 = c->d_z[0]; a.h1 = c->d_h[0]; a.xn = c->d_xn;
    a.B = (int)c->B; a.d0 = (int)c->dims[0]; a.d1 = (int)c->dims[1]; a.d2 = (int)c->dims[2];
    a.gW1 = c->d_g + c->off[0]; a.gb1 = c->d_g + c->off[1]; a.gW2 = c->d_g + c->off[2]; a.gb2 = c->d_g + c->off[3];
    a.p_dw1 = c->d_hp_dw1; a.p_db1 = c->d_hp_db1; a.p_dw2 = c->d_hp_dw2; a.p_db2 = c->d_hp_db2;
    a.sd = nullptr;
    if (fin_fused(c)) {
      // world 1: nothing is exchanged before the step's scalars, so K1's SSE partials and
      // step_finalize fold into the gradient reduction's launch
      a.sd = c->d_sd; a.sse_parts = c->d_sse_part; a.n_sse_parts = c->last_nparts; a.st = c->d_st;
      a.mirror = c->d_mirror; a.slot = (uint32_t)(c->calls % MEL_RESULT_RING);
      a.n_field = (double)c->N; a.lr0 = c->cfg.lr0; a.lr_min = c->cfg.lr_min; a.halving = c->cfg.lr_halving_samples;
      a.beta1 = c->cfg.beta1; a.beta2 = c->cfg.beta2;
    }
    head_bwd3(a, c->stream);
    c->launches += 2;
    c->klaunch[MEL_K_HEAD_BWD] += 2;
    return check_launch(c, "head backward");
  }
  // dZ of every hidden layer first: dZ_{l-1} = (dZ_l W_l) * ReLU'(Z_{l-1}), fused mask (W_l is
  // only updated by the Adam after the exchange)
  for (int l = L - 1; l >= 2; --l) {
    const int dout = c->dims[l], din = c->dims[l - 1];
    const float* W = c->d_p + c->off[2 * (l - 1)];
    EpiExtra ex;
    ex.mask = c->d_z[l - 2];
    ex.ldm = din;
    nl += sgemm_auto(false, false, (int)c->B, din, dout, c->d_dz[l - 1], dout, W, din, c->d_dz[l - 2], din,
                     EPI_RELU_MASK, nullptr, nullptr, 0, c->d_part, c->part_elems, c->stream, ex);
  }
  // weight gradients dW_l = dZ_l^T H_{l-1} (K = B; 32 x 32 tiles fill the GPU without split-K)
  for (int l = L - 1; l >= 1; --l) {
    const int dout = c->dims[l], din = c->dims[l - 1];
    const float* Hin = (l == 1) ? c->d_xn : c->d_h[l - 2];
    const int ldin = (l == 1) ? 8 : din;
    nl += sgemm_auto(true, false, dout, din, (int)c->B, c->d_dz[l - 1], dout, Hin, ldin, c->d_g + c->off[2 * (l - 1)],
                     din, EPI_STORE, nullptr, nullptr, 0, c->d_part, c->part_elems, c->stream);
  }
  // bias gradients of the hidden layers (column sums over the batch, fp64 accumulation): one launch
  for (int l = L - 1; l >= 1; l -= 2) {
    const int l2 = l - 1;
    col_sum2(c->d_dz[l - 1], c->dims[l], c->dims[l], c->d_g + c->off[2 * (l - 1) + 1],
             l2 >= 1 ? c->d_dz[l2 - 1] : nullptr, l2 >= 1 ? c->dims[l2] : 0, l2 >= 1 ? c->dims[l2] : 0,
             l2 >= 1 ? c->d_g + c->off[2 * (l2 - 1) + 1] : nullptr, (int)c->B, c->stream);
    nl += 1;
  }
  c->launches += nl;
  c->klaunch[MEL_K_HEAD_BWD] += nl;
  return check_launch(c, "head backward");
}

int head_forward(mel_ctx* c, const float* xn, float** Z, float** H, int rows, __nv_bfloat16* h_last_bf16 = nullptr) {
  int nl = 0;
  for (int l = 1; l < c->L; ++l) {
    const int din = c->dims[l - 1], dout = c->dims[l];
    const float* Hin = (l == 1) ? xn : H[l - 2];
    const int ldin = (l == 1) ? 8 : din;
    EpiExtra ex;
    if (l == c->L - 1) ex.Hb = h_last_bf16;     // bf16 operand of the tensor-core output layer
    nl += sgemm_auto(false, true, rows, dout, din, Hin, ldin, c->d_p + c->off[2 * (l - 1)], din, Z[l - 1], dout,
                     EPI_BIAS_RELU, c->d_p + c->off[2 * (l - 1) + 1], H[l - 1], dout, c->d_part, c->part_elems,
                     c->stream, ex);
  }
  return nl;
}

int splits_for(uint64_t K) {
  int s = (int)(K / 8192);
  if (s < 1) s = 1;
  if (s > 64) s = 64;
  return s;
}

int train_step_fp32(mel_ctx* c) {
  const int L = c->L;
  const uint32_t B = c->B, K = c->Klast;
  float* Hl = c->d_h[L - 2];
  const float* WL = c->d_p + c->off[2 * (L - 1)];
  const float* bL = c->d_p + c->off[2 * (L - 1) + 1];
  int nparts;
  {
    Timer t(c, MEL_K_OUT_FWD_DW, 3);
    OutArgs oa{Hl, (int)K, WL, bL, (int)K, c->ra.payload, c->ra.storage, c->Npad, c->N, c->d_slots, c->d_st,
               c->d_dy, c->d_sse_part, (int)B};
    nparts = out_fwd_f32(oa, c->stream);
    // dW_L = dY^T H  (M = Npad, N = K, K = B)
    sgemm(true, false, (int)c->Npad, (int)K, (int)B, c->d_dy, (int)c->Npad, Hl, (int)K, c->d_g + c->off[2 * (L - 1)],
          (int)K, EPI_STORE, nullptr, nullptr, 0, 1, c->stream);
    col_sum(c->d_dy, (int)B, (int)c->Npad, (int)c->Npad, c->d_g + c->off[2 * (L - 1) + 1], c->stream);
  }
  if (c->zero) CK(cudaEventRecord(c->ev_gw, c->stream));
  {
    Timer t(c, MEL_K_OUT_DH, 2);
    // dH = dY W  (M = B, N = K, K = Npad), split-K, then ReLU' mask -> dZ_{L-1}
    const int sp = splits_for(c->Npad);
    sgemm(false, false, (int)B, (int)K, (int)c->Npad, c->d_dy, (int)c->Npad, WL, (int)K, c->d_part, (int)K, EPI_STORE,
          nullptr, nullptr, 0, sp, c->stream);
    splitk_reduce((int)B, (int)K, sp, c->d_part, c->d_dz[L - 2], (int)K, c->d_z[L - 2], (int)K, c->stream);
  }
  int r = check_launch(c, "output layer fp32");
  if (r) return r;
  c->last_nparts = nparts;
  if (!fin_fused(c)) reduce_local(c->d_sd, c->d_sse_part, nparts, c->d_st, c->stream);
  return MEL_OK;
}

// the output layer's kernel arguments (no launches)
void bf16_args(mel_ctx* c, tc::OutTcArgs& a) {
  const int L = c->L;
  const uint32_t B = c->B, K = c->Klast;
  a = tc::OutTcArgs{};
  a.N = c->N; a.Npad = c->Npad; a.B = B; a.K = K;
  a.shadow_idx = c->shadow_cur;
  a.w_bf16 = c->d_shadow[c->shadow_cur];
  a.fused_adam = (c->fused_adam || c->peer) ? 1 : 0;
  if (a.fused_adam) {
    const uint64_t offW = c->off[2 * (L - 1)];
    a.adam_p = c->d_p + offW; a.adam_m = c->d_m + offW; a.adam_v = c->d_v + offW;
    a.shadow_out = c->d_shadow[c->shadow_cur ^ 1];
    a.sd = c->d_sd;
    a.k1_seq = c->k1_launches++;
    a.b1 = (float)c->cfg.beta1; a.b2 = (float)c->cfg.beta2; a.eps = (float)c->cfg.eps;
  }
  if (c->peer) {
    a.peer = 1; a.rank = (uint32_t)c->rank; a.world = (uint32_t)c->world; a.epoch = ++c->epoch;
    a.acc_bf16 = c->acc_bf16 ? 1u : 0u;
    a.cnt_local = c->d_cnt;
    for (int q = 0; q < c->world; ++q) { a.cnt_peer[q] = c->p_cnt[q]; a.sh_peer[q] = c->p_sh[c->shadow_cur ^ 1][q]; }
  }
  a.b = c->d_p + c->off[2 * (L - 1) + 1];
  a.h_bf16 = c->tcb.h_bf16;
  a.payload = static_cast<const __nv_bfloat16*>(c->ra.payload);
  a.slots = c->d_slots; a.st = c->d_st;
  a.dyT = c->tcb.dyT;
  a.gW = c->d_g + c->off[2 * (L - 1)];
  a.gb = c->d_g + c->off[2 * (L - 1) + 1];
  a.sse_part = c->d_sse_part;
  a.dh_part = c->d_part;
  a.dz = c->d_dz[L - 2];
  a.z = c->d_z[L - 2];
}

// step scalars ahead of K1 (the fused Adam needs lr, bias corrections, the gradient scale)
void bf16_prepare(mel_ctx* c) {
  Timer t(c, MEL_K_LOSS, 1);
  step_prepare(c->d_sd, c->d_st, (double)c->N, c->cfg.lr0, c->cfg.lr_min, c->cfg.lr_halving_samples,
               c->cfg.beta1, c->cfg.beta2, c->stream, c->peer);
}

// after K1: K2 (dH) and this rank's SSE
int bf16_post_k1(mel_ctx* c, const tc::OutTcArgs& a, int nparts) {
  {
    Timer t(c, MEL_K_OUT_DH, 2);
    tc::launch_out_dh(a, c->tcb, c->stream);
  }
  int r = check_launch(c, "output layer tcgen05");
  if (r) return r;
  c->last_nparts = nparts;
  if (!fin_fused(c)) reduce_local(c->d_sd, c->d_sse_part, nparts, c->d_st, c->stream);
  return MEL_OK;
}

int train_step_bf16(mel_ctx* c) {
  const int L = c->L;
  const uint32_t K = c->Klast;
  tc::OutTcArgs a;
  bf16_args(c, a);
  if (a.fused_adam) {
    if (c->peer) {
      // the Adam inside K1 needs the global batch size (gradient scale, skip) up front
      Timer t(c, MEL_K_ALLREDUCE, 1);
      stage_count(c->d_sd, c->d_st, c->stream);
      NK(ncclAllReduce(&c->d_sd->n_glob, &c->d_sd->n_glob, 1, ncclFloat64, ncclSum, c->comm, c->stream));
    }
    if (!c->prep_fused) bf16_prepare(c);
  }
  int nparts = 0;
  if (!c->zero || c->peer) {
    int r0 = wait_shadow(c);
    if (r0) return r0;
    Timer t(c, MEL_K_OUT_FWD_DW, 1);
    nparts = tc::launch_out_fwd_dw(a, c->tcb, c->stream);
  } else {
    float* gW = c->d_g + c->off[2 * (L - 1)];
    for (int j = 0; j < c->nb; ++j) {
      if (c->ag_pending) CK(cudaStreamWaitEvent(c->stream, c->ev_agb[j], 0));   // this bucket's shadow rows
      {
        Timer t(c, MEL_K_OUT_FWD_DW, 1);
        nparts += tc::launch_out_fwd_dw(a, c->tcb, c->stream, c->bt0[j], c->bt1[j], (uint32_t)nparts);
      }
      CK(cudaEventRecord(c->ev_k1[j], c->stream));
      Timer t(c, MEL_K_ALLREDUCE, 0, c->comm_stream);
      CK(cudaStreamWaitEvent(c->comm_stream, c->ev_k1[j], 0));
      float* gb = gW + bucket_row0(c, j) * K;
      NK(ncclReduceScatter(gb, gb + (uint64_t)c->rank * part_elems(c, j), part_elems(c, j), ncclFloat32, ncclSum,
                           c->comm, c->comm_stream));
    }
    c->ag_pending = false;
  }
  return bf16_post_k1(c, a, nparts);
}

// a step's front: the batch bookkeeping, the gather of the batch inputs, the head forward
int step_front(mel_ctx* c) {
  if (!c->batch_known) {
    // no sample since the last step: this rank contributes nothing
    CK(cudaMemsetAsync(&c->d_st->n_last, 0, 4, c->stream));
    c->batch_n = 0;
  }
  c->prep_fused = false;
  if (c->head_fused) {
    // gather + both hidden layers (+ the step scalars of the fused Adam, world 1) in one launch
    Timer t(c, MEL_K_HEAD_FWD, 1);
    HeadFwdArgs a;
    memset(&a, 0, sizeof a);
    a.ra = c->ra; a.slots = c->d_slots; a.B = c->B; a.tau = c->cfg.steps_per_sim;
    a.W1 = c->d_p + c->off[0]; a.b1 = c->d_p + c->off[1]; a.W2 = c->d_p + c->off[2]; a.b2 = c->d_p + c->off[3];
    a.d0 = (int)c->dims[0]; a.d1 = (int)c->dims[1]; a.d2 = (int)c->dims[2];
    a.xn = c->d_xn; a.Z1 = c->d_z[0]; a.H1 = c->d_h[0]; a.Z2 = c->d_z[1]; a.H2 = c->d_h[1];
    a.Hb = c->cfg.precision == MEL_BF16 ? c->tcb.h_bf16 : nullptr;
    if (c->cfg.precision == MEL_BF16 && c->fused_adam && !c->peer) {
      a.sd = c->d_sd; a.n_field = (double)c->N; a.lr0 = c->cfg.lr0; a.lr_min = c->cfg.lr_min;
      a.halving = c->cfg.lr_halving_samples; a.beta1 = c->cfg.beta1; a.beta2 = c->cfg.beta2;
      a.counter = c->d_hcnt;
      a.target = (c->hf_n + 1) * (uint32_t)head_fwd3_ctas((int)c->B);
      c->hf_n += 1;
      c->prep_fused = true;
    }
    head_fwd3(a, c->stream);
    return check_launch(c, "head forward");
  }
  {
    Timer t(c, MEL_K_GATHER, 1);
    launch_gather(c->ra, c->d_slots, c->B, c->cfg.steps_per_sim, c->d_xn, c->stream);
  }
  {
    Timer t(c, MEL_K_HEAD_FWD, 0);
    const int nl = head_forward(c, c->d_xn, c->d_z, c->d_h, (int)c->B,
                                c->cfg.precision == MEL_BF16 ? c->tcb.h_bf16 : nullptr);
    c->launches += nl;
    c->klaunch[MEL_K_HEAD_FWD] += nl;
  }
  return check_launch(c, "head forward");
}

// a step's end, after the gradient exchange: loss / step scalars, Adam (the part K1 did not
// fuse), the shadow flip, the result record for surrogate_step_result
int step_finish(mel_ctx* c) {
  int r;
  if (!fin_fused(c)) {
    Timer t(c, MEL_K_LOSS, 1);
    step_finalize(c->d_sd, (double)c->N, c->cfg.lr0, c->cfg.lr_min, c->cfg.lr_halving_samples, c->cfg.beta1,
                  c->cfg.beta2, c->d_mirror, c->d_st, c->stream, (uint32_t)(c->calls % MEL_RESULT_RING));
  }
  if (c->fused_adam || c->peer) {
    // W_L was updated inside K1 (new shadow in the other buffer, written to every rank in
    // exchange mode); the small region here
    Timer t(c, MEL_K_ADAM, 1);
    adam_flat(c->d_p, c->d_m, c->d_v, c->d_g, c->off[2 * (c->L - 1)], c->d_sd, (float)c->cfg.beta1,
              (float)c->cfg.beta2, (float)c->cfg.eps, nullptr, 0, 0, c->stream);
    c->shadow_cur ^= 1;
  } else if (c->zero) {
    // small region (head weights, every bias) replicated; W_L on this rank's row shard,
    // refreshing the shard of the bf16 shadow, then all-gather of the shadow
    Timer t(c, MEL_K_ADAM, 1 + c->nb);
    const uint64_t offW = c->off[2 * (c->L - 1)];
    const float b1 = (float)c->cfg.beta1, b2 = (float)c->cfg.beta2, eps = (float)c->cfg.eps;
    adam_flat(c->d_p, c->d_m, c->d_v, c->d_g, offW, c->d_sd, b1, b2, eps, nullptr, 0, 0, c->stream);
    for (int j = 0; j < c->nb; ++j) {
      const uint64_t po = part_off(c, j), so = offW + po, n = part_elems(c, j);
      adam_flat(c->d_p + so, c->d_m + so, c->d_v + so, c->d_g + so, n, c->d_sd, b1, b2, eps,
                c->d_shadow[c->shadow_cur] + po, 0, n, c->stream);
    }
  } else {
    Timer t(c, MEL_K_ADAM, 1);
    __nv_bfloat16* sh = nullptr;
    uint64_t b0 = 0, b1 = 0;
    if (c->cfg.precision == MEL_BF16) {
      // the output-layer kernels of this step have completed (stream order), so
      // the bf16 shadow is refreshed in place from the updated fp32 master
      sh = c->d_shadow[c->shadow_cur];
      b0 = c->off[2 * (c->L - 1)];
      b1 = b0 + c->Npad * c->Klast;
    }
    adam_flat(c->d_p, c->d_m, c->d_v, c->d_g, c->n_flat, c->d_sd, (float)c->cfg.beta1, (float)c->cfg.beta2,
              (float)c->cfg.eps, sh, b0, b1, c->stream);
  }
  if (c->zero && !c->peer) {
    Timer t(c, MEL_K_ALLREDUCE, 0, c->comm_stream);
    CK(cudaEventRecord(c->ev_adam, c->stream));
    CK(cudaStreamWaitEvent(c->comm_stream, c->ev_adam, 0));
    for (int j = 0; j < c->nb; ++j) {
      if ((r = gather_bucket(c, c->d_shadow[c->shadow_cur], 2, ncclBfloat16, j))) return r;
      CK(cudaEventRecord(c->ev_agb[j], c->comm_stream));
    }
    c->ag_pending = true;
  }
  if ((r = check_launch(c, "adam"))) return r;
  CK(cudaEventRecord(c->ev_call[c->calls % MEL_RESULT_RING], c->stream));
  c->calls += 1;
  c->batch_known = false;
  return MEL_OK;
}

}  // namespace

extern "C" {

int mel_config_default(mel_config* g, uint32_t n_field, uint32_t batch) {
  if (!g) return MEL_EINVAL;
  memset(g, 0, sizeof *g);
  g->abi_version = MEL_ABI_VERSION;
  g->n_field = n_field;
  g->hidden[0] = 256; g->hidden[1] = 256;
  g->capacity = 6000; g->threshold = 1000;
  g->batch = batch;
  g->steps_per_sim = 100;
  g->temp_lo = 100.f; g->temp_hi = 500.f;
  g->precision = MEL_FP32; g->storage = MEL_STORE_F32;
  g->lr0 = 1e-3; g->lr_min = 2.5e-4; g->lr_halving_samples = 10000;
  g->beta1 = 0.9; g->beta2 = 0.999; g->eps = 1e-8;
  g->seed = 1;
  g->staging_entries = 16;
  return MEL_OK;
}

int mel_nccl_unique_id(void* out128) {
  if (!out128) return MEL_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return MEL_ENCCL;
  memcpy(out128, &id, sizeof id);
  return MEL_OK;
}

const char* mel_last_error(const mel_ctx* c) { return c ? c->err.c_str() : "null context"; }

// In-kernel exchange setup: this rank's acc + counters, then every rank's acc, counters and
// both shadow buffers mapped through CUDA IPC (handles all-gathered over NCCL).  Needs
// peer access between every pair of GPUs (NVLink / NVSwitch); otherwise the NCCL exchange
// stays.  Collective: every rank decides the same (the all-reduced minimum).
static int setup_peer(mel_ctx* c) {
  int ok = 1;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  // the peers' device ordinals are not known here; require access to every visible device
  for (int d = 0; d < ndev; ++d) {
    if (d == c->dev) continue;
    int can = 0;
    CK(cudaDeviceCanAccessPeer(&can, c->dev, d));
    if (!can) ok = 0;
  }
  const uint64_t rows = c->Npad;
  const uint32_t tiles = (uint32_t)(rows / 128);
  int* d_ok;
  CK(cudaMalloc(&d_ok, sizeof(int)));
  CK(cudaMemcpy(d_ok, &ok, sizeof(int), cudaMemcpyHostToDevice));
  NK(ncclAllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, c->comm, c->stream));
  CK(cudaMemcpyAsync(&ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(d_ok);
  if (!ok) return MEL_OK;
  c->acc_bf16 = !(c->cfg.flags & MEL_FLAG_FP32_EXCHANGE) && c->Klast % 128 == 0;
  const size_t acc_bytes = (c->acc_bf16 ? 2 : 4) * rows * c->Klast;
  CK(cudaMalloc(&c->d_acc, acc_bytes));
  DALLOC(c->d_cnt, tiles);
  CK(cudaMemset(c->d_acc, 0, acc_bytes));
  CK(cudaMemset(c->d_cnt, 0, 4 * tiles));
  // handles: [acc, cnt, shadow0, shadow1] per rank
  const int NH = 4;
  std::vector<cudaIpcMemHandle_t> mine(NH), all((size_t)NH * c->world);
  void* bufs[NH] = {c->d_acc, c->d_cnt, c->d_shadow[0], c->d_shadow[1]};
  for (int i = 0; i < NH; ++i) CK(cudaIpcGetMemHandle(&mine[i], bufs[i]));
  char* d_h;
  const size_t hb = sizeof(cudaIpcMemHandle_t) * NH;
  CK(cudaMalloc(&d_h, hb * c->world));
  CK(cudaMemcpy(d_h + hb * c->rank, mine.data(), hb, cudaMemcpyHostToDevice));
  NK(ncclAllGather(d_h + hb * c->rank, d_h, hb, ncclChar, c->comm, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(all.data(), d_h, hb * c->world, cudaMemcpyDeviceToHost));
  cudaFree(d_h);
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) {
      c->p_acc[q] = c->d_acc; c->p_cnt[q] = c->d_cnt;
      c->p_sh[0][q] = c->d_shadow[0]; c->p_sh[1][q] = c->d_shadow[1];
      continue;
    }
    void* p[NH];
    for (int i = 0; i < NH; ++i)
      CK(cudaIpcOpenMemHandle(&p[i], all[(size_t)q * NH + i], cudaIpcMemLazyEnablePeerAccess));
    c->p_acc[q] = p[0]; c->p_cnt[q] = static_cast<uint32_t*>(p[1]);
    c->p_sh[0][q] = static_cast<__nv_bfloat16*>(p[2]); c->p_sh[1][q] = static_cast<__nv_bfloat16*>(p[3]);
  }
  if (tc::prepare_peer(c->tcb, c->Klast, rows, c->rank, c->world, c->p_acc, c->acc_bf16, c->p_sh[0], c->p_sh[1]))
    return fail(c, MEL_ECUDA, "exchange tensor maps: %s", tc::last_error());
  c->peer = true;
  return MEL_OK;
}

static int create_impl(mel_ctx* c, const mel_config* g, const void* nccl_id, void* stream) {
  int r = validate(g, c->world, c);
  if (r) return r;
  if (!c->virt && (c->world > 1) != (nccl_id != nullptr))
    return fail(c, MEL_EINVAL, "nccl_id must be given iff world > 1");
  c->cfg = *g;
  CK(cudaSetDevice(c->dev));
  if (stream) { c->stream = (cudaStream_t)stream; }
  else { CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)); c->own_stream = true; }
  CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_copy, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_fence, cudaEventDisableTiming));
  for (int i = 0; i < MEL_RESULT_RING; ++i) CK(cudaEventCreateWithFlags(&c->ev_call[i], cudaEventDisableTiming));

  // geometry: dims = [6, hidden..., N]
  c->dims[0] = 6;
  int nd = 1;
  c->dims[nd++] = g->hidden[0];
  if (g->hidden[1]) c->dims[nd++] = g->hidden[1];
  c->dims[nd++] = g->n_field;
  c->L = nd - 1;
  c->N = g->n_field; c->Bs = g->batch; c->C = g->capacity;
  c->B = g->precision == MEL_BF16 ? (g->batch + 63) / 64 * 64 : g->batch;
  // rows of W_L padded to 128 (UMMA M) x world (equal row shards under ZeRO)
  const uint64_t row_quant = 128ull * (uint64_t)c->world;
  c->Npad = ((uint64_t)c->N + row_quant - 1) / row_quant * row_quant;
  c->Klast = c->dims[c->L - 1];
  c->hmax = g->hidden[0] > g->hidden[1] ? g->hidden[0] : g->hidden[1];
  // flat layout: W_1 b_1 ... W_{L-1} b_{L-1} b_L W_L, i.e. everything but W_L forms one
  // small contiguous region [0, off(W_L)) (replicated under ZeRO), tensors 64-B aligned
  uint64_t o = 0;
  for (int l = 0; l < c->L; ++l) {
    const uint64_t rows = (l == c->L - 1) ? c->Npad : c->dims[l + 1];
    c->cnt[2 * l] = rows * c->dims[l];
    c->cnt[2 * l + 1] = rows;
    if (l < c->L - 1) {
      c->off[2 * l] = o; o += (c->cnt[2 * l] + 15) / 16 * 16;
      c->off[2 * l + 1] = o; o += (rows + 15) / 16 * 16;
    } else {
      c->off[2 * l + 1] = o; o += (rows + 15) / 16 * 16;
      c->off[2 * l] = o; o += (c->cnt[2 * l] + 15) / 16 * 16;
    }
  }
  c->n_flat = o;

  // reservoir arenas
  const uint32_t S = g->staging_entries, C = g->capacity;
  ResArgs& a = c->ra;
  DALLOC(c->d_st, 1);
  CK(cudaMemset(c->d_st, 0, sizeof(ResDev)));
  CK(cudaHostAlloc((void**)&c->h_mirror, sizeof(Mirror), cudaHostAllocMapped));
  memset(c->h_mirror, 0, sizeof(Mirror));
  CK(cudaHostGetDevicePointer((void**)&c->d_mirror, c->h_mirror, 0));
  // staging metadata lives in mapped pinned memory: the commit kernel reads the 32-byte
  // entries straight from the host (no per-put copy on the stream)
  CK(cudaHostAlloc((void**)&c->h_stmeta, sizeof(StMeta) * S, cudaHostAllocMapped));
  memset(c->h_stmeta, 0, sizeof(StMeta) * S);
  StMeta* d_stmeta; float* d_stfield;
  CK(cudaHostGetDevicePointer((void**)&d_stmeta, c->h_stmeta, 0));
  DALLOC(d_stfield, (size_t)S * c->Npad);
  CK(cudaMemset(d_stfield, 0, sizeof(float) * (size_t)S * c->Npad));
  DALLOC(a.meta, C);
  DALLOC(a.seen, C);
  DALLOC(a.put_seq, C);
  DALLOC(a.bitmap, (C + 31) / 32);
  CK(cudaMemset(a.bitmap, 0, sizeof(uint32_t) * ((C + 31) / 32)));
  DALLOC(a.pos, C);
  DALLOC(a.bad, C);
  CK(cudaMemset(a.bad, 0, sizeof(uint32_t) * C));
  const size_t esz = g->storage == MEL_STORE_F32 ? 4 : 2;
  {
    void* pl = nullptr;
    cudaError_t e = cudaMalloc(&pl, esz * (size_t)C * c->Npad);
    if (e != cudaSuccess) { cudaGetLastError(); return fail(c, MEL_ENOMEM, "reservoir payload (%zu B): %s", esz * (size_t)C * c->Npad, cudaGetErrorString(e)); }
    CK(cudaMemset(pl, 0, esz * (size_t)C * c->Npad));
    a.payload = pl;
  }
  DALLOC(a.plan, S);
  DALLOC(a.plan_src, S);
  CK(cudaHostAlloc((void**)&c->h_stsrc, sizeof(float*) * S, cudaHostAllocMapped));
  memset(c->h_stsrc, 0, sizeof(float*) * S);
  {
    const float** d_stsrc;
    CK(cudaHostGetDevicePointer((void**)&d_stsrc, c->h_stsrc, 0));
    a.st_src = d_stsrc;
  }
  a.st = c->d_st; a.mirror = c->d_mirror; a.st_meta = d_stmeta; a.st_field = d_stfield; a.S = S;
  a.C = C; a.theta = g->threshold; a.Npad = c->Npad; a.N = c->N; a.storage = (int)g->storage;
  a.lo = g->temp_lo; a.span = g->temp_hi - g->temp_lo; a.seed = g->seed; a.rank = (uint32_t)c->rank;
  a.policy = g->policy;
  launch_init_res(a, c->stream);
  DALLOC(c->d_slots, c->B);

  // parameters
  DALLOC(c->d_p, c->n_flat); DALLOC(c->d_m, c->n_flat); DALLOC(c->d_v, c->n_flat); DALLOC(c->d_g, c->n_flat);
  CK(cudaMemset(c->d_p, 0, 4 * c->n_flat)); CK(cudaMemset(c->d_m, 0, 4 * c->n_flat));
  CK(cudaMemset(c->d_v, 0, 4 * c->n_flat)); CK(cudaMemset(c->d_g, 0, 4 * c->n_flat));
  for (int l = 0; l < c->L; ++l) {
    const uint64_t rows = c->dims[l + 1];     // real rows (padding rows stay zero)
    init_tensor(c->d_p + c->off[2 * l], rows * c->dims[l], 2 * l, c->dims[l], g->seed, c->stream);
    init_tensor(c->d_p + c->off[2 * l + 1], rows, 2 * l + 1, c->dims[l], g->seed, c->stream);
  }
  // activations
  DALLOC(c->d_xn, (size_t)c->B * 8);
  CK(cudaMemset(c->d_xn, 0, sizeof(float) * c->B * 8));
  for (int l = 0; l < c->L - 1; ++l) {
    DALLOC(c->d_z[l], (size_t)c->B * c->dims[l + 1]);
    DALLOC(c->d_h[l], (size_t)c->B * c->dims[l + 1]);
    DALLOC(c->d_dz[l], (size_t)c->B * c->dims[l + 1]);
  }
  DALLOC(c->d_sd, 1);
  CK(cudaMemset(c->d_sd, 0, sizeof(StepDev)));
  {
    const char* hf = getenv("MEL_HEAD_FUSED");
    c->head_fused = (!hf || atoi(hf) != 0) && c->L == 3 && c->dims[0] <= 8 && c->dims[1] % 32 == 0 &&
                    c->dims[2] % 32 == 0 && c->dims[1] <= 256 && c->dims[2] <= 256;
    if (c->head_fused && head3_init() != 0) return fail(c, MEL_ECUDA, "fused head: SMEM attribute rejected");
    if (c->head_fused) {
      const int nrow = head_bwd3_row_ctas((int)c->B);
      DALLOC(c->d_hcnt, 1);
      CK(cudaMemset(c->d_hcnt, 0, 4));
      DALLOC(c->d_hp_dw1, (size_t)nrow * c->dims[1] * 8);
      DALLOC(c->d_hp_db1, (size_t)nrow * c->dims[1]);
      DALLOC(c->d_hp_dw2, head_dw2_part_elems((int)c->B, (int)c->dims[1], (int)c->dims[2]));
      DALLOC(c->d_hp_db2, head_dw2_part_elems((int)c->B, 1, (int)c->dims[2]));
    }
  }
  if (g->precision == MEL_FP32) {
    DALLOC(c->d_dy, (size_t)c->B * c->Npad);
    const int sp = splits_for(c->Npad);
    c->part_elems = (size_t)sp * c->B * c->Klast;
    if (c->part_elems < (size_t)16 * c->hmax * c->hmax) c->part_elems = (size_t)16 * c->hmax * c->hmax;
    DALLOC(c->d_part, c->part_elems);
    c->max_parts = (int)(((c->Npad + 63) / 64) * ((c->B + 63) / 64));
    DALLOC(c->d_sse_part, c->max_parts);
  } else {
    DALLOC(c->d_shadow[0], (size_t)c->Npad * c->Klast);
    DALLOC(c->d_shadow[1], (size_t)c->Npad * c->Klast);
    r = tc::alloc_buffers(c->tcb, c->Npad, c->B, c->Klast);
    if (r) return fail(c, MEL_ENOMEM, "tensor-core scratch allocation failed");
    c->part_elems = tc::dh_part_elems(c->B, c->Klast);
    if (c->part_elems < (size_t)16 * c->hmax * c->hmax) c->part_elems = (size_t)16 * c->hmax * c->hmax;
    DALLOC(c->d_part, c->part_elems);
    c->max_parts = tc::max_sse_parts(c->Npad);
    DALLOC(c->d_sse_part, c->max_parts);
    to_bf16(c->d_p + c->off[2 * (c->L - 1)], c->d_shadow[0], c->Npad * c->Klast, c->stream);
    const __nv_bfloat16* shadows[2] = {c->d_shadow[0], c->d_shadow[1]};
    c->zero = (c->world > 1) && !(g->flags & MEL_FLAG_NO_ZERO);
    // tuning knobs for the overlapped exchange (environment, diagnostics only)
    const char* e_res = getenv("MEL_SM_RESERVE");
    const char* e_nb = getenv("MEL_BUCKETS");
    c->sm_reserve = c->zero ? (e_res ? atoi(e_res) : 0) : 0;
    if (c->zero) {
      const uint32_t tiles = (uint32_t)(c->Npad / 128);
      c->nb = tiles >= 64 ? (e_nb ? atoi(e_nb) : 1) : 1;
      if (c->nb < 1) c->nb = 1;
      if (c->nb > mel_ctx::NBMAX) c->nb = mel_ctx::NBMAX;
      // bucket boundaries on whole groups of `world` tiles, so every bucket's rows split into
      // `world` equal parts (tiles is a multiple of world: Npad is padded to 128 x world)
      const uint32_t groups = tiles / (uint32_t)c->world;
      if ((uint32_t)c->nb > groups) c->nb = (int)groups;
      for (int j = 0; j < c->nb; ++j) {
        c->bt0[j] = (uint32_t)((uint64_t)groups * j / c->nb) * (uint32_t)c->world;
        c->bt1[j] = (uint32_t)((uint64_t)groups * (j + 1) / c->nb) * (uint32_t)c->world;
      }
    }
    r = tc::prepare(c->tcb, c->Npad, c->B, c->Klast, shadows,
                    static_cast<const __nv_bfloat16*>(c->ra.payload), c->C, c->d_g + c->off[2 * (c->L - 1)],
                    c->sm_reserve, c->d_p + c->off[2 * (c->L - 1)], c->d_m + c->off[2 * (c->L - 1)],
                    c->d_v + c->off[2 * (c->L - 1)]);
    if (r) return fail(c, MEL_ECUDA, "tensor-core kernel setup failed: %s", tc::last_error());
  }
  r = check_launch(c, "create");
  if (r) return r;
  CK(cudaStreamSynchronize(c->stream));

  // the Adam of W_L runs inside K1 at every batch size (end of round 2,
  // step ms at B = 10 / 64 / 128 / 192 / 256: separate kernel 1.80 / 1.79 / 1.84 / 1.93 / 2.06,
  // fused 1.57 / 1.59 / 1.65 / 1.73 / 1.77 -- the fused path saves the 2 GB gradient round
  // trip; early in round 2 it lost below 4 chunks per tile and the policy was B >= 256)
  uint32_t fused_min_b = 1;
  if (const char* e = getenv("MEL_FUSED_MIN_B")) fused_min_b = (uint32_t)atoi(e);   // diagnostics (A/B of the policy)
  c->fused_adam = (c->world == 1) && (g->precision == MEL_BF16) && !(g->flags & MEL_FLAG_UNFUSED_ADAM) &&
                  c->B >= fused_min_b;
  if (c->world > 1) {
    if (!c->virt) {
      ncclUniqueId id;
      memcpy(&id, nccl_id, sizeof id);
      ncclConfig_t ncfg = NCCL_CONFIG_INITIALIZER;
      if (c->zero && c->sm_reserve > 0) ncfg.maxCTAs = c->sm_reserve;   // NCCL on the SMs the kernels leave free
      NK(ncclCommInitRankConfig(&c->comm, c->world, id, c->rank, &ncfg));
    }
    c->shard_elems = c->Npad / c->world * c->Klast;
    c->shard_off = (uint64_t)c->rank * c->shard_elems;
    CK(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    cudaEvent_t* evs[] = {&c->ev_gw, &c->ev_head, &c->ev_ar, &c->ev_adam, &c->ev_ag};
    for (cudaEvent_t* e : evs) CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    for (int j = 0; j < c->nb; ++j) {
      CK(cudaEventCreateWithFlags(&c->ev_k1[j], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_agb[j], cudaEventDisableTiming));
    }
    if (!c->virt && c->zero && !(g->flags & MEL_FLAG_NCCL_EXCHANGE) && c->world <= tc::MAX_WORLD) {
      r = setup_peer(c);
      if (r) return r;
    }
  }
  return MEL_OK;
}

int mel_create(const mel_config* g, int rank, int world, const void* nccl_id, int cuda_device, void* stream,
               mel_ctx** out) {
  if (!g || !out) return MEL_EINVAL;
  *out = nullptr;
  mel_ctx* c = new mel_ctx();
  c->rank = rank; c->world = world; c->dev = cuda_device;
  int r = create_impl(c, g, nccl_id, stream);
  if (r) {
    static thread_local std::string last;
    last = c->err;
    fprintf(stderr, "mel_create: %s\n", c->err.c_str());
    mel_destroy(c);
    return r;
  }
  *out = c;
  return MEL_OK;
}

void mel_destroy(mel_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->dev);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  for (auto& e : c->ing_ev)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (c->off_buf[i]) cudaFreeHost(c->off_buf[i]);
    if (c->off_ev[i]) cudaEventDestroy(c->off_ev[i]);
  }
  if (c->ing_pinned) cudaHostUnregister(c->ing_base);
  if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
  if (c->peer && !c->virt) {
    for (int q = 0; q < c->world; ++q) {
      if (q == c->rank) continue;
      void* h[] = {c->p_acc[q], c->p_cnt[q], c->p_sh[0][q], c->p_sh[1][q]};
      for (void* p : h)
        if (p) cudaIpcCloseMemHandle(p);
    }
  }
  if (c->comm) ncclCommDestroy(c->comm);
  cudaEvent_t evs[] = {c->ev_gw, c->ev_head, c->ev_ar, c->ev_adam, c->ev_ag};
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  for (int j = 0; j < mel_ctx::NBMAX; ++j) {
    if (c->ev_k1[j]) cudaEventDestroy(c->ev_k1[j]);
    if (c->ev_agb[j]) cudaEventDestroy(c->ev_agb[j]);
  }
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  drain_timers(c);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  void* ptrs[] = {c->d_st, (void*)c->ra.st_field, c->ra.meta, c->ra.seen, c->ra.put_seq,
                  c->ra.bitmap, c->ra.pos, c->ra.bad, c->ra.payload, c->ra.plan, c->d_slots, c->d_p, c->d_m, c->d_v, c->d_g,
                  c->d_shadow[0], c->d_shadow[1], c->d_xn, c->d_z[0], c->d_z[1], c->d_h[0], c->d_h[1], c->d_dz[0],
                  c->d_dz[1], c->d_dy, c->d_part, c->d_sse_part, c->d_sd, c->d_eval_x, c->d_eval_t, c->d_eval_y,
                  c->d_eval_f, c->d_eval_z[0], c->d_eval_z[1], c->d_eval_h[0], c->d_eval_h[1], c->d_eval_xn,
                  c->d_acc, c->d_cnt, c->d_gen, c->d_gen_x, c->d_gen_t};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  tc::free_buffers(c->tcb);
  if (c->h_mirror) cudaFreeHost(c->h_mirror);
  if (c->h_stmeta) cudaFreeHost(c->h_stmeta);
  if (c->h_stsrc) cudaFreeHost(c->h_stsrc);
  if (c->ra.plan_src) cudaFree(c->ra.plan_src);
  if (c->ev_copy) cudaEventDestroy(c->ev_copy);
  if (c->ev_fence) cudaEventDestroy(c->ev_fence);
  for (int i = 0; i < MEL_RESULT_RING; ++i)
    if (c->ev_call[i]) cudaEventDestroy(c->ev_call[i]);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->vg) {
    VGroup* vg = c->vg;
    vg->cs[c->rank] = nullptr;
    if (--vg->refs == 0) {
      void* ptrs[] = {vg->d_desc, vg->d_tab_g, vg->d_tab_red, vg->d_tab_nglob};
      for (void* p : ptrs)
        if (p) cudaFree(p);
      if (vg->own_stream && vg->stream) cudaStreamDestroy(vg->stream);
      delete vg;
    }
  }
  delete c;
}

// Virtual ranks (test mode): `world` contexts on ONE device sharing one stream, each a full
// rank (its own reservoir, batch and replica); their collectives run as device-side
// rank-ordered sums and the bf16 in-kernel exchange as one cooperative K1 launch over every
// rank's tiles, ~#SMs / world CTAs per rank.  out[world] receives the contexts in rank order.
int mel_create_virtual(const mel_config* g, int world, int cuda_device, void* stream, mel_ctx** out) {
  if (!g || !out || world < 2 || world > tc::MAX_WORLD) return MEL_EINVAL;
  for (int q = 0; q < world; ++q) out[q] = nullptr;
  if (g->precision == MEL_BF16 && (g->flags & (MEL_FLAG_NCCL_EXCHANGE | MEL_FLAG_NO_ZERO))) {
    fprintf(stderr, "mel_create_virtual: bf16 virtual ranks run the in-kernel exchange only\n");
    return MEL_EINVAL;
  }
  if (cudaSetDevice(cuda_device) != cudaSuccess) return MEL_ECUDA;
  VGroup* vg = new VGroup();
  vg->R = world;
  if (stream) {
    vg->stream = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&vg->stream, cudaStreamNonBlocking) != cudaSuccess) { delete vg; return MEL_ECUDA; }
    vg->own_stream = true;
  }
  int r = MEL_OK;
  auto cleanup = [&]() {
    for (int q = 0; q < world; ++q)
      if (out[q]) { mel_destroy(out[q]); out[q] = nullptr; }
  };
  for (int q = 0; q < world; ++q) {
    mel_ctx* c = new mel_ctx();
    c->rank = q; c->world = world; c->dev = cuda_device; c->virt = true; c->vg = vg;
    vg->cs[q] = c;
    vg->refs += 1;
    out[q] = c;
    r = create_impl(c, g, nullptr, vg->stream);
    if (r) {
      fprintf(stderr, "mel_create_virtual (rank %d): %s\n", q, c->err.c_str());
      cleanup();
      return r;
    }
  }
  mel_ctx* c = out[0];
  auto alloc_tab = [&](void** dst, const void* const* host) -> int {
    if (cudaMalloc(dst, sizeof(void*) * world) != cudaSuccess) return MEL_ENOMEM;
    if (cudaMemcpy(*dst, host, sizeof(void*) * world, cudaMemcpyHostToDevice) != cudaSuccess) return MEL_ECUDA;
    return MEL_OK;
  };
  const void* tg[tc::MAX_WORLD];
  const void* tr[tc::MAX_WORLD];
  const void* tn[tc::MAX_WORLD];
  for (int q = 0; q < world; ++q) {
    tg[q] = out[q]->d_g; tr[q] = &out[q]->d_sd->red[0]; tn[q] = &out[q]->d_sd->n_glob;
  }
  if ((r = alloc_tab((void**)&vg->d_tab_g, tg)) || (r = alloc_tab((void**)&vg->d_tab_red, tr)) ||
      (r = alloc_tab((void**)&vg->d_tab_nglob, tn))) {
    cleanup();
    return r;
  }
  if (g->precision == MEL_BF16) {
    // the in-kernel exchange between the members: every member's acc, counters and shadows
    // addressed directly (one device), K1 grid = #SMs / world CTAs per rank
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device);
    int G = sms / world;
    if (const char* e = getenv("MEL_VIRT_CTAS")) {       // diagnostics: fewer K1 CTAs per virtual rank
      const int v = atoi(e);
      if (v >= 1 && v < G) G = v;
    }
    if (cudaMalloc(&vg->d_desc, (size_t)tc::virt_desc_bytes() * world) != cudaSuccess) { cleanup(); return MEL_ENOMEM; }
    for (int q = 0; q < world; ++q) {
      mel_ctx* m = out[q];
      m->tcb.fwd_ctas = G < 160 ? G : 160;
      m->acc_bf16 = !(g->flags & MEL_FLAG_FP32_EXCHANGE) && m->Klast % 128 == 0;
      const size_t acc_bytes = (m->acc_bf16 ? 2 : 4) * m->Npad * m->Klast;
      if (cudaMalloc(&m->d_acc, acc_bytes) != cudaSuccess || cudaMemset(m->d_acc, 0, acc_bytes) != cudaSuccess ||
          cudaMalloc(&m->d_cnt, 4 * (m->Npad / 128)) != cudaSuccess ||
          cudaMemset(m->d_cnt, 0, 4 * (m->Npad / 128)) != cudaSuccess) {
        cleanup();
        return MEL_ENOMEM;
      }
    }
    for (int q = 0; q < world; ++q) {
      mel_ctx* m = out[q];
      for (int p = 0; p < world; ++p) {
        m->p_acc[p] = out[p]->d_acc; m->p_cnt[p] = out[p]->d_cnt;
        m->p_sh[0][p] = out[p]->d_shadow[0]; m->p_sh[1][p] = out[p]->d_shadow[1];
      }
      if (tc::prepare_peer(m->tcb, m->Klast, m->Npad, m->rank, world, m->p_acc, m->acc_bf16, m->p_sh[0], m->p_sh[1])) {
        fprintf(stderr, "mel_create_virtual: exchange tensor maps: %s\n", tc::last_error());
        cleanup();
        return MEL_ECUDA;
      }
      m->peer = true;
    }
  }
  if (cudaStreamSynchronize(vg->stream) != cudaSuccess) { cleanup(); return MEL_ECUDA; }
  (void)c;
  return MEL_OK;
}

int mel_param_layout(const mel_ctx* c, uint32_t* n_tensors, uint32_t* shapes, uint64_t* total) {
  if (!c) return MEL_EINVAL;
  if (n_tensors) *n_tensors = 2 * c->L;
  uint64_t t = 0;
  for (int l = 0; l < c->L; ++l) {
    if (shapes) {
      shapes[4 * l + 0] = c->dims[l + 1]; shapes[4 * l + 1] = c->dims[l];
      shapes[4 * l + 2] = c->dims[l + 1]; shapes[4 * l + 3] = 1;
    }
    t += (uint64_t)c->dims[l + 1] * c->dims[l] + c->dims[l + 1];
  }
  if (total) *total = t;
  return MEL_OK;
}

static int copy_tensors(mel_ctx* c, float* base, float* const* host, bool to_host) {
  for (int l = 0; l < c->L; ++l) {
    for (int w = 0; w < 2; ++w) {
      const uint64_t n = w == 0 ? (uint64_t)c->dims[l + 1] * c->dims[l] : c->dims[l + 1];
      float* d = base + c->off[2 * l + w];
      if (!host[2 * l + w]) continue;
      if (to_host) CK(cudaMemcpyAsync(host[2 * l + w], d, 4 * n, cudaMemcpyDeviceToHost, c->stream));
      else CK(cudaMemcpyAsync(d, host[2 * l + w], 4 * n, cudaMemcpyHostToDevice, c->stream));
    }
  }
  return MEL_OK;
}

static int refresh_shadow(mel_ctx* c) {
  int r0 = wait_shadow(c);
  if (r0) return r0;
  if (c->cfg.precision == MEL_BF16)
    to_bf16(c->d_p + c->off[2 * (c->L - 1)], c->d_shadow[c->shadow_cur], c->Npad * c->Klast, c->stream);
  return check_launch(c, "shadow");
}

int mel_set_params(mel_ctx* c, const float* const* t) {
  GUARD(c);
  if (!t) return fail(c, MEL_EINVAL, "null tensors");
  int r = copy_tensors(c, c->d_p, const_cast<float* const*>(t), false);
  if (r) return r;
  r = refresh_shadow(c);
  if (r) return r;
  CK(cudaStreamSynchronize(c->stream));
  return MEL_OK;
}

int mel_get_params(mel_ctx* c, float* const* t) {
  GUARD(c);
  if (!t) return fail(c, MEL_EINVAL, "null tensors");
  int r = gather_master(c, false);
  if (r) return r;
  r = copy_tensors(c, c->d_p, t, true);
  if (r) return r;
  CK(cudaStreamSynchronize(c->stream));
  return MEL_OK;
}

int mel_get_state(mel_ctx* c, mel_state_view* s) {
  GUARD(c);
  if (!s) return fail(c, MEL_EINVAL, "null state");
  int r = gather_master(c, true);
  if (r) return r;
  if (s->p && (r = copy_tensors(c, c->d_p, s->p, true))) return r;
  if (s->m && (r = copy_tensors(c, c->d_m, s->m, true))) return r;
  if (s->v && (r = copy_tensors(c, c->d_v, s->v, true))) return r;
  StepDev sd;
  CK(cudaMemcpyAsync(&sd, c->d_sd, sizeof sd, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  s->adam_step = sd.k;
  s->samples_seen = sd.S;
  return MEL_OK;
}

int mel_set_state(mel_ctx* c, const mel_state_view* s) {
  GUARD(c);
  if (!s || !s->p || !s->m || !s->v) return fail(c, MEL_EINVAL, "null state");
  int r;
  if ((r = copy_tensors(c, c->d_p, s->p, false))) return r;
  if ((r = copy_tensors(c, c->d_m, s->m, false))) return r;
  if ((r = copy_tensors(c, c->d_v, s->v, false))) return r;
  StepDev sd;
  CK(cudaMemcpyAsync(&sd, c->d_sd, sizeof sd, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  sd.k = s->adam_step;
  sd.S = s->samples_seen;
  CK(cudaMemcpyAsync(c->d_sd, &sd, sizeof sd, cudaMemcpyHostToDevice, c->stream));
  r = refresh_shadow(c);
  if (r) return r;
  CK(cudaStreamSynchronize(c->stream));
  return MEL_OK;
}

static int put_impl(mel_ctx* c, uint32_t sim, uint32_t t, const float X[5], const float* field, int on_device,
                    bool zero_copy);

int reservoir_put(mel_ctx* c, uint32_t sim, uint32_t t, const float X[5], const float* field, int on_device) {
  if (on_device < 0 || on_device > 2) return fail(c, MEL_EINVAL, "field_on_device must be 0, 1 or 2");
  return put_impl(c, sim, t, X, field, on_device, true);
}

static int put_impl(mel_ctx* c, uint32_t sim, uint32_t t, const float X[5], const float* field, int on_device,
                    bool zero_copy) {
  GUARD(c);
  if (!X || !field) return fail(c, MEL_EINVAL, "null X or field");
  if (c->closed) return fail(c, MEL_ECLOSED, "reservoir_put after reservoir_close");
  int r = ensure_ring_space(c);
  if (r) return r;
  const uint32_t S = c->cfg.staging_entries;
  const uint32_t e = (uint32_t)(c->tail % S);
  StMeta m{};
  m.sim = sim; m.t = t;
  for (int i = 0; i < 5; ++i) m.X[i] = X[i];
  // the mapped metadata entry is read by the commit kernel that consumes it; it is only
  // rewritten after that commit published its progress (ensure_ring_space)
  c->h_stmeta[e] = m;
  float* dst = const_cast<float*>(c->ra.st_field) + (uint64_t)e * c->Npad;
  c->h_stsrc[e] = nullptr;
  if (on_device == 2 && zero_copy && c->N % 4 == 0 && ((uintptr_t)field & 15) == 0) {
    // zero copy (opt-in): the commit that consumes this entry reads the caller's field in
    // stream order; the mel.h contract keeps it valid until that commit has run
    c->h_stsrc[e] = field;
  } else if (on_device) {
    CK(cudaMemcpyAsync(dst, field, 4ull * c->N, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    if (c->copy_fence) {
      CK(cudaEventRecord(c->ev_fence, c->stream));
      CK(cudaStreamWaitEvent(c->copy_stream, c->ev_fence, 0));
      c->copy_fence = false;
    }
    CK(cudaMemcpyAsync(dst, field, 4ull * c->N, cudaMemcpyHostToDevice, c->copy_stream));
    CK(cudaEventRecord(c->ev_copy, c->copy_stream));
    c->copy_pending = true;
  }
  c->tail += 1;
  return MEL_OK;
}

// releases the slots of ingest calls whose DMA has landed; with `block`, waits for the
// oldest one first
int ingest_retire(mel_ctx* c, bool block) {
  while (c->ing_n) {
    const uint32_t i = c->ing_head;
    if (block) {
      CK(cudaEventSynchronize(c->ing_ev[i]));
      block = false;
    } else {
      const cudaError_t q = cudaEventQuery(c->ing_ev[i]);
      if (q == cudaErrorNotReady) break;
      if (q != cudaSuccess) return fail(c, MEL_ECUDA, "ingest copy: %s", cudaGetErrorString(q));
    }
    for (uint32_t k = 0; k < c->ing_cnt[i]; ++k) mel_ingest_release(c->ing_handle);
    c->ing_head = (i + 1) % mel_ctx::ING_EVENTS;
    c->ing_n -= 1;
  }
  return MEL_OK;
}

int reservoir_ingest(mel_ctx* c, mel_ingest* g, uint32_t max_msgs, uint32_t timeout_us, uint32_t* n_put_host) {
  GUARD(c);
  if (!g) return fail(c, MEL_EINVAL, "null ingest handle");
  if (n_put_host) *n_put_host = 0;
  if (c->closed) return fail(c, MEL_ECLOSED, "reservoir_ingest after reservoir_close");
  if (g != c->ing_handle) {
    int r = ingest_retire(c, true);
    while (!r && c->ing_n) r = ingest_retire(c, true);
    if (r) return r;
    c->ing_handle = g;
  }
  void* base = nullptr;
  uint64_t bytes = 0;
  mel_ingest_segment(g, &base, &bytes);
  if (base != c->ing_base) {
    // page-lock the shared segment once, so each field is DMA-copied straight from the
    // client's slot into the staging ring (no bounce through pageable memory)
    if (c->ing_pinned) CK(cudaHostUnregister(c->ing_base));
    c->ing_base = base;
    c->ing_bytes = bytes;
    c->ing_pinned = cudaHostRegister(base, bytes, cudaHostRegisterDefault) == cudaSuccess;
    if (!c->ing_pinned) (void)cudaGetLastError();   // pageable copies still work, synchronously
  }
  if (!c->ing_ev[0])
    for (auto& e : c->ing_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // slots whose copies have landed go back to the clients; keep at most ING_EVENTS - 1
  // calls in flight
  int r = ingest_retire(c, c->ing_n == mel_ctx::ING_EVENTS);
  if (r) return r;
  uint32_t n = 0;
  bool eos = false;
  while (n < max_msgs) {
    r = ensure_ring_space(c);
    if (r == MEL_EAGAIN) break;                     // staging full: the caller samples (commit point)
    if (r) return r;
    mel_ingest_msg m;
    int q = mel_ingest_next(g, &m, 0u);
    if (q == MEL_EAGAIN && c->ing_n) {              // the ring may be waiting for our releases
      if ((r = ingest_retire(c, true))) return r;
      q = mel_ingest_next(g, &m, 0u);
    }
    if (q == MEL_EAGAIN && n == 0 && timeout_us) q = mel_ingest_next(g, &m, timeout_us);
    if (q == MEL_EAGAIN) break;
    if (q == MEL_EOS) { eos = true; break; }
    if (q != MEL_OK) return fail(c, q, "ingest ring: status %d", q);
    r = reservoir_put(c, m.sim_id, m.t, m.X, m.field, 0);
    if (r) return r;
    ++n;
  }
  if (n) {
    // the slots go back to the clients once this call's copies have landed
    const uint32_t i = (c->ing_head + c->ing_n) % mel_ctx::ING_EVENTS;
    CK(cudaEventRecord(c->ing_ev[i], c->copy_stream));
    c->ing_cnt[i] = n;
    c->ing_n += 1;
    if (!c->ing_pinned && (r = ingest_retire(c, true))) return r;
  }
  if (n_put_host) *n_put_host = n;
  return (eos && n == 0) ? MEL_EOS : MEL_OK;
}

int surrogate_train_offline(mel_ctx* c, mel_dataset* d, uint64_t seed, uint32_t epoch, uint32_t first_batch,
                            uint32_t n_batches, double* losses_host, uint32_t* steps_host) {
  GUARD(c);
  if (steps_host) *steps_host = 0;
  if (!d) return fail(c, MEL_EINVAL, "null dataset");
  if (c->cfg.policy != MEL_FIFO) return fail(c, MEL_EINVAL, "offline training needs mel_config.policy = MEL_FIFO");
  if (c->cfg.staging_entries < c->Bs) return fail(c, MEL_EINVAL, "offline training needs staging_entries >= batch");
  if (mel_dataset_n_field(d) != c->N) return fail(c, MEL_EINVAL, "dataset n_field %u != %u", mel_dataset_n_field(d), c->N);
  if (c->closed) return fail(c, MEL_ECLOSED, "offline training after reservoir_close");
  const uint64_t count = mel_dataset_count(d);
  const uint64_t nb_epoch = count / c->Bs;                   // the last partial batch is dropped (R24)
  if (first_batch >= nb_epoch) return MEL_OK;
  if (n_batches > nb_epoch - first_batch) n_batches = (uint32_t)(nb_epoch - first_batch);
  std::vector<uint32_t> perm(count);
  mel_dataset_epoch_order(count, seed, epoch, perm.data());
  const uint32_t* order = perm.data() + (uint64_t)first_batch * c->Bs;
  const uint64_t total = (uint64_t)n_batches * c->Bs;
  // records move in chunks through two pinned buffers: the loader threads read chunk q+1
  // while chunk q's fields are DMA-copied into the staging ring and the GPU trains
  if (!c->off_buf[0]) {
    c->off_chunk = c->Bs < 64 ? c->Bs : 64;
    for (int i = 0; i < 2; ++i) {
      CK(cudaHostAlloc((void**)&c->off_buf[i], (size_t)c->off_chunk * c->N * 4, cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&c->off_ev[i], cudaEventDisableTiming));
    }
  }
  const uint32_t chunk = c->off_chunk;
  const uint64_t n_chunks = (total + chunk - 1) / chunk;
  std::vector<uint32_t> sim(2 * chunk), tt(2 * chunk);
  std::vector<float> X(2 * 5 * chunk);
  auto load = [&](uint64_t q) {
    const int b = (int)(q & 1);
    const uint32_t n = (uint32_t)std::min<uint64_t>(chunk, total - q * chunk);
    return mel_dataset_read(d, order + q * chunk, n, sim.data() + b * chunk, tt.data() + b * chunk,
                            X.data() + 5 * b * chunk, c->off_buf[b], c->N);
  };
  std::future<int> fut = std::async(std::launch::async, load, (uint64_t)0);
  uint64_t put = 0;
  uint32_t steps = 0;
  uint64_t first_call = c->calls;
  for (uint64_t q = 0; q < n_chunks; ++q) {
    const int b = (int)(q & 1);
    int rl = fut.get();
    if (rl) return fail(c, MEL_ENOMEM, "dataset read failed (status %d)", rl);
    if (q + 1 < n_chunks) {
      CK(cudaEventSynchronize(c->off_ev[b ^ 1]));          // chunk q-1's copies out of that buffer
      fut = std::async(std::launch::async, load, q + 1);
    }
    const uint32_t n = (uint32_t)std::min<uint64_t>(chunk, total - q * chunk);
    for (uint32_t k = 0; k < n; ++k) {
      int r = reservoir_put(c, sim[b * chunk + k], tt[b * chunk + k], &X[5 * (b * chunk + k)],
                            c->off_buf[b] + (uint64_t)k * c->N, 0);
      if (r) return r;
      if (++put % c->Bs == 0) {
        // the FIFO hands out exactly the B records just put, in epoch order
        if ((r = reservoir_sample_batch(c, nullptr, nullptr))) return r;
        if ((r = surrogate_step(c, nullptr))) return r;
        if (losses_host && steps > 0)
          if ((r = surrogate_step_result(c, first_call + steps - 1, losses_host + steps - 1, nullptr))) return r;
        ++steps;
      }
    }
    CK(cudaEventRecord(c->off_ev[b], c->copy_stream));
  }
  if (losses_host && steps > 0) {
    int r = surrogate_step_result(c, first_call + steps - 1, losses_host + steps - 1, nullptr);
    if (r) return r;
  }
  if (steps_host) *steps_host = steps;
  return MEL_OK;
}

int reservoir_put_generated(mel_ctx* c, mel_heat* h, const uint32_t* sim, const float* X, const uint32_t* t,
                            uint32_t k, uint32_t* n_put_host) {
  GUARD(c);
  if (n_put_host) *n_put_host = 0;
  if (!h || !sim || !X || !t) return fail(c, MEL_EINVAL, "null generator argument");
  const uint32_t n = mel_heat_grid(h);
  if ((uint64_t)n * n != c->N) return fail(c, MEL_EINVAL, "generator grid %u^2 != n_field %u", n, c->N);
  if (c->closed) return fail(c, MEL_ECLOSED, "reservoir_put_generated after reservoir_close");
  const uint32_t kmax = 64;
  if (!c->d_gen) {
    DALLOC(c->d_gen, (size_t)kmax * c->N);
    DALLOC(c->d_gen_x, (size_t)kmax * 5);
    DALLOC(c->d_gen_t, kmax);
  }
  uint32_t done = 0;
  while (done < k) {
    const uint32_t m = std::min(kmax, k - done);
    for (uint32_t j = 0; j < m; ++j)
      if (t[done + j] >= mel_heat_tau(h)) return fail(c, MEL_EINVAL, "t = %u >= tau", t[done + j]);
    // the previous chunk's D2D copies out of the scratch are ordered before this on c->stream
    CK(cudaMemcpyAsync(c->d_gen_x, X + 5ull * done, 20ull * m, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_gen_t, t + done, 4ull * m, cudaMemcpyHostToDevice, c->stream));
    if (mel_heat_fields(h, c->d_gen_x, c->d_gen_t, m, c->d_gen, c->stream) != 0)
      return fail(c, MEL_ECUDA, "heat field generation failed");
    c->launches += 1;
    for (uint32_t j = 0; j < m; ++j) {
      // the scratch is reused by the next chunk before this entry's commit: copy it
      int r = put_impl(c, sim[done + j], t[done + j], X + 5ull * (done + j), c->d_gen + (uint64_t)j * c->N, 1, false);
      if (r == MEL_EAGAIN) {
        if (n_put_host) *n_put_host = done + j;
        return MEL_EAGAIN;
      }
      if (r) return r;
    }
    done += m;
  }
  if (n_put_host) *n_put_host = done;
  return MEL_OK;
}

int reservoir_close(mel_ctx* c) {
  GUARD(c);
  if (c->closed) return fail(c, MEL_EPROTO, "reservoir_close called twice");
  c->closed = true;
  return commit(c);
}

int reservoir_sample_batch(mel_ctx* c, int32_t* slots_host, uint32_t* n_host) {
  GUARD(c);
  int r;
  if (c->cfg.policy == MEL_RESERVOIR) {
    // commit control and the draws in one launch, then the commit's data plane
    const uint64_t max_e = c->tail - c->known_consumed;
    if (c->copy_pending) {
      CK(cudaStreamWaitEvent(c->stream, c->ev_copy, 0));
      c->copy_pending = false;
    }
    {
      Timer t(c, MEL_K_COMMIT, max_e ? 2 : 1);
      launch_commit_sample(c->ra, c->tail, c->closed ? 1u : 0u, (uint32_t)max_e, c->d_slots, c->Bs, c->stream);
    }
    r = check_launch(c, "commit + sample");
    if (r) return r;
  } else {
    r = commit(c);
    if (r) return r;
    {
      Timer t(c, MEL_K_SAMPLE, 1);
      launch_sample(c->ra, c->d_slots, c->Bs, c->stream);
    }
    r = check_launch(c, "sample");
    if (r) return r;
  }
  // During reception the fill phase never blocks (u <= p < C), so p = min(C, puts)
  // at every commit point and the watermark gate is host-decidable.
  bool need_sync = slots_host || n_host || c->closed;
  uint32_t n = c->Bs;
  if (!c->closed) {
    if (c->cfg.policy == MEL_RESERVOIR) {
      const uint64_t p = c->tail < c->C ? c->tail : c->C;
      if (p <= c->cfg.threshold) n = 0;
    } else {
      // FIFO / FIRO remove what they hand out: every accepted put is drawn, in the
      // buffer, or pending, and a commit fills the buffer up to C
      const uint64_t left = c->tail - c->drawn;
      const uint64_t p = left < c->C ? left : c->C;
      const uint64_t need = c->cfg.policy == MEL_FIFO ? c->Bs : (uint64_t)c->cfg.threshold + c->Bs;
      if (p < need) n = 0;
    }
  }
  if (need_sync) {
    r = sync_stream(c);
    if (r) return r;
    n = c->h_mirror->n_last;
  }
  c->batch_known = true;
  c->batch_n = n;
  c->drawn += n;
  if (n_host) *n_host = n;
  if (slots_host && n) CK(cudaMemcpy(slots_host, c->d_slots, 4ull * n, cudaMemcpyDeviceToHost));
  if (!c->closed && n == 0) return MEL_EAGAIN;
  return MEL_OK;
}

int surrogate_step(mel_ctx* c, double* loss_host) {
  GUARD(c);
  if (c->virt) return fail(c, MEL_EPROTO, "a virtual rank steps through surrogate_step_virtual");
  const bool local_has = c->batch_known && c->batch_n > 0;
  if (!c->batch_known) c->batch_n = 0;
  int r;
  if (c->world == 1 && c->batch_n == 0) {
    // no samples (watermark gate, drained, or no sample call): nothing to train on, so no
    // gather / forward / backward / Adam is launched and the parameters and the shadow stay
    // as they are; only the step's result (status 1, as step_finalize publishes it for an
    // empty step) is recorded in stream order for surrogate_step_result
    CK(cudaMemsetAsync(&c->d_st->n_last, 0, 4, c->stream));
    CK(cudaMemsetAsync(c->d_sd->red, 0, sizeof c->d_sd->red, c->stream));
    {
      Timer t(c, MEL_K_LOSS, 1);
      step_finalize(c->d_sd, (double)c->N, c->cfg.lr0, c->cfg.lr_min, c->cfg.lr_halving_samples, c->cfg.beta1,
                    c->cfg.beta2, c->d_mirror, c->d_st, c->stream, (uint32_t)(c->calls % MEL_RESULT_RING));
    }
    if ((r = check_launch(c, "empty step"))) return r;
    CK(cudaEventRecord(c->ev_call[c->calls % MEL_RESULT_RING], c->stream));
    c->calls += 1;
    c->batch_known = false;
    if ((r = sync_stream(c))) return r;
    const Mirror& m = *c->h_mirror;
    return (c->closed && m.over && m.p == 0) ? MEL_EOS : MEL_EAGAIN;
  }
  if ((r = step_front(c))) return r;
  r = c->cfg.precision == MEL_FP32 ? train_step_fp32(c) : train_step_bf16(c);
  if (r) return r;
  if ((r = head_backward(c))) return r;
  if ((r = world_exchange(c))) return r;
  if ((r = step_finish(c))) return r;
  const bool need_sync = loss_host || !local_has || c->closed;
  if (!need_sync) return MEL_OK;
  if ((r = sync_stream(c))) return r;
  const Mirror& m = *c->h_mirror;
  if (m.status == 3)
    return fail(c, MEL_ENONFINITE, "step skipped: non-finite inputs in a batch or a non-finite loss (%g)", m.loss);
  if (m.status == 1) {
    bool eos = c->closed && m.over && m.p == 0;
    if (c->world > 1) {
      // global EOS only when every rank is drained (reading Q11): n_total == 0 and
      // every rank closed; ranks agree on n_total, so agree on closed too
      int v = eos ? 1 : 0;
      int* dv;
      CK(cudaMalloc(&dv, 4));
      CK(cudaMemcpy(dv, &v, 4, cudaMemcpyHostToDevice));
      NK(ncclAllReduce(dv, dv, 1, ncclInt32, ncclMin, c->comm, c->stream));
      CK(cudaMemcpyAsync(&v, dv, 4, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      cudaFree(dv);
      eos = v == 1;
    }
    return eos ? MEL_EOS : MEL_EAGAIN;
  }
  if (loss_host) *loss_host = m.loss;
  if (!std::isfinite(m.loss)) return fail(c, MEL_ENONFINITE, "loss is not finite (%g)", m.loss);
  return MEL_OK;
}

// One collective step of a virtual-rank group (mel_create_virtual), ranks in order: the
// same per-rank kernels as surrogate_step, the NCCL all-reduces replaced by rank-ordered
// device sums (vsum_*) and K1 launched once over every rank's tiles.
int surrogate_step_virtual(mel_ctx* const* cs, int world, double* loss_host) {
  if (!cs || world < 2 || world > tc::MAX_WORLD) return MEL_EINVAL;
  VGroup* vg = cs[0] ? cs[0]->vg : nullptr;
  if (!vg || vg->R != world) return MEL_EINVAL;
  for (int q = 0; q < world; ++q) {
    if (!cs[q] || cs[q]->vg != vg || cs[q]->rank != q) return MEL_EINVAL;
    if (cs[q]->poisoned) return cs[q]->poisoned;
  }
  mel_ctx* c = cs[0];
  cudaSetDevice(c->dev);
  cudaStream_t s = c->stream;
  bool any_local = false, closed = false;
  int r;
  for (int q = 0; q < world; ++q) {
    any_local = any_local || (cs[q]->batch_known && cs[q]->batch_n > 0);
    closed = closed || cs[q]->closed;
    if ((r = step_front(cs[q]))) return r;
  }
  if (c->cfg.precision == MEL_FP32) {
    for (int q = 0; q < world; ++q)
      if ((r = train_step_fp32(cs[q]))) return r;
  } else {
    tc::OutTcArgs a[tc::MAX_WORLD];
    const tc::TcBuffers* tb[tc::MAX_WORLD];
    for (int q = 0; q < world; ++q) {
      bf16_args(cs[q], a[q]);
      tb[q] = &cs[q]->tcb;
      stage_count(cs[q]->d_sd, cs[q]->d_st, s);
    }
    vsum_f64(vg->d_tab_nglob, world, 1, s);                       // the global batch size
    for (int q = 0; q < world; ++q) bf16_prepare(cs[q]);
    int nparts;
    {
      Timer t(c, MEL_K_OUT_FWD_DW, 1);
      nparts = tc::launch_out_fwd_dw_virtual(a, tb, world, vg->d_desc, s);
    }
    if (nparts < 0) return fail(c, MEL_ECUDA, "virtual K1: %s", tc::last_error());
    for (int q = 0; q < world; ++q)
      if ((r = bf16_post_k1(cs[q], a[q], nparts))) return r;
  }
  for (int q = 0; q < world; ++q)
    if ((r = head_backward(cs[q]))) return r;
  {
    // the gradient exchange: the whole flat gradient (plain mode) or the small region (the
    // in-kernel exchange reduced W_L inside K1), plus [SSE, n]
    Timer t(c, MEL_K_ALLREDUCE, 2);
    const uint64_t n = c->peer ? c->off[2 * (c->L - 1)] : c->n_flat;
    vsum_f32(vg->d_tab_g, world, n, s);
    vsum_f64(vg->d_tab_red, world, 2, s);
  }
  if ((r = check_launch(c, "virtual exchange"))) return r;
  for (int q = 0; q < world; ++q)
    if ((r = step_finish(cs[q]))) return r;
  const bool need_sync = loss_host || !any_local || closed;
  if (!need_sync) return MEL_OK;
  CK(cudaStreamSynchronize(s));
  for (int q = 0; q < world; ++q) cs[q]->known_consumed = cs[q]->h_mirror->consumed;
  const Mirror& m = *c->h_mirror;
  if (m.status == 3)
    return fail(c, MEL_ENONFINITE, "step skipped: non-finite inputs in a batch or a non-finite loss (%g)", m.loss);
  if (m.status == 1) {
    bool eos = true;
    for (int q = 0; q < world; ++q) {
      const Mirror& mq = *cs[q]->h_mirror;
      eos = eos && cs[q]->closed && mq.over && mq.p == 0;
    }
    return eos ? MEL_EOS : MEL_EAGAIN;
  }
  if (loss_host) *loss_host = m.loss;
  if (!std::isfinite(m.loss)) return fail(c, MEL_ENONFINITE, "loss is not finite (%g)", m.loss);
  return MEL_OK;
}

int surrogate_step_result(mel_ctx* c, uint64_t call, double* loss_host, int* status_host) {
  GUARD(c);
  if (call >= c->calls || c->calls - call > (uint64_t)MEL_RESULT_RING)
    return fail(c, MEL_EINVAL, "step call %llu not among the last %d calls", (unsigned long long)call,
                MEL_RESULT_RING);
  const int slot = (int)(call % MEL_RESULT_RING);
  CK(cudaEventSynchronize(c->ev_call[slot]));               // that step only, not the stream
  const volatile Mirror* m = c->h_mirror;
  if (loss_host) *loss_host = m->ring_loss[slot];
  if (status_host) *status_host = m->ring_status[slot];
  return MEL_OK;
}

int surrogate_eval(mel_ctx* c, const float* X, const uint32_t* t, const float* fields, uint32_t n, double* mse,
                   float* pred) {
  GUARD(c);
  if (!X || !t || n == 0) return fail(c, MEL_EINVAL, "bad eval arguments");
  int rg = gather_master(c, false);   // full fp32 W_L (collective under ZeRO)
  if (rg) return rg;
  const uint32_t chunk = c->B;
  if (!c->d_eval_x) {
    DALLOC(c->d_eval_x, (size_t)chunk * 5); DALLOC(c->d_eval_t, chunk); DALLOC(c->d_eval_xn, (size_t)chunk * 8);
    DALLOC(c->d_eval_y, (size_t)chunk * c->Npad); DALLOC(c->d_eval_f, (size_t)chunk * c->N);
    for (int l = 0; l < c->L - 1; ++l) {
      DALLOC(c->d_eval_z[l], (size_t)chunk * c->dims[l + 1]);
      DALLOC(c->d_eval_h[l], (size_t)chunk * c->dims[l + 1]);
    }
  }
  double* d_part;
  DALLOC(d_part, 256);
  double total = 0.0;
  const float lo = c->cfg.temp_lo, span = c->cfg.temp_hi - c->cfg.temp_lo;
  // held-out fields already in this GPU's memory (unified addressing tells) are read in
  // place instead of being copied from the host
  bool fields_dev = false;
  if (fields) {
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, fields) == cudaSuccess)
      fields_dev = (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged) && pa.device == c->dev;
    else
      (void)cudaGetLastError();
  }
  std::vector<double> parts(256);
  for (uint32_t s0 = 0; s0 < n; s0 += chunk) {
    const uint32_t m = (n - s0) < chunk ? (n - s0) : chunk;
    CK(cudaMemcpyAsync(c->d_eval_x, X + 5ull * s0, 20ull * m, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_eval_t, t + s0, 4ull * m, cudaMemcpyHostToDevice, c->stream));
    eval_inputs(c->d_eval_x, c->d_eval_t, (int)m, c->cfg.steps_per_sim, lo, span, c->d_eval_xn, c->stream);
    head_forward(c, c->d_eval_xn, c->d_eval_z, c->d_eval_h, (int)m);
    const int L = c->L;
    sgemm(false, true, (int)m, (int)c->N, (int)c->Klast, c->d_eval_h[L - 2], (int)c->Klast, c->d_p + c->off[2 * (L - 1)],
          (int)c->Klast, c->d_eval_y, (int)c->Npad, EPI_BIAS, c->d_p + c->off[2 * (L - 1) + 1], nullptr, 0, 1, c->stream);
    c->launches += 2 + (L - 1) + 1;
    if (fields) {
      if (fields_dev) {
        normalise_fields(fields + (uint64_t)s0 * c->N, c->d_eval_f, (uint64_t)m * c->N, lo, span, c->stream);
      } else {
        CK(cudaMemcpyAsync(c->d_eval_f, fields + (uint64_t)s0 * c->N, 4ull * m * c->N, cudaMemcpyHostToDevice,
                           c->stream));
        normalise_fields(c->d_eval_f, c->d_eval_f, (uint64_t)m * c->N, lo, span, c->stream);
      }
      const int np = eval_mse_partial(c->d_eval_y, c->d_eval_f, (int)m, (int)c->N, (int)c->Npad, d_part, c->stream);
      c->launches += 2;
      CK(cudaMemcpyAsync(parts.data(), d_part, 8ull * np, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      for (int i = 0; i < np; ++i) total += parts[i];
    }
    if (pred) {
      std::vector<float> y((size_t)m * c->Npad);
      CK(cudaMemcpyAsync(y.data(), c->d_eval_y, 4ull * m * c->Npad, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      for (uint32_t i = 0; i < m; ++i)
        for (uint32_t j = 0; j < c->N; ++j) pred[(uint64_t)(s0 + i) * c->N + j] = y[(size_t)i * c->Npad + j] * span + lo;
    }
  }
  int r = check_launch(c, "eval");
  cudaFree(d_part);
  if (r) return r;
  CK(cudaStreamSynchronize(c->stream));
  if (mse) *mse = fields ? total / ((double)n * c->N) : NAN;
  return MEL_OK;
}

int reservoir_stats(mel_ctx* c, mel_stats* out) {
  GUARD(c);
  if (!out) return fail(c, MEL_EINVAL, "null stats");
  int r = sync_stream(c);
  if (r) return r;
  ResDev st;
  StepDev sd;
  CK(cudaMemcpy(&st, c->d_st, sizeof st, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&sd, c->d_sd, sizeof sd, cudaMemcpyDeviceToHost));
  memset(out, 0, sizeof *out);
  out->population = st.p; out->unseen = st.u; out->seen = st.p - st.u;
  out->puts = c->tail; out->committed = st.q; out->draws = st.d; out->evictions = st.evictions;
  out->pending = c->tail - st.consumed;
  out->steps = sd.k; out->samples = sd.S;
  for (int i = 0; i < MEL_HIST_BINS; ++i) out->hist[i] = st.hist[i];
  out->over = st.over; out->closed = c->closed;
  out->last_loss = sd.loss;
  return MEL_OK;
}

int reservoir_dump(mel_ctx* c, uint32_t* sim, uint32_t* t, float* X, uint32_t* seen, uint64_t* put_seq, void* payload) {
  GUARD(c);
  int r = sync_stream(c);
  if (r) return r;
  const uint32_t C = c->C;
  if (sim || t || X) {
    std::vector<SlotMeta> m(C);
    CK(cudaMemcpy(m.data(), c->ra.meta, sizeof(SlotMeta) * C, cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < C; ++i) {
      if (sim) sim[i] = m[i].sim;
      if (t) t[i] = m[i].t;
      if (X) for (int k = 0; k < 5; ++k) X[5 * i + k] = m[i].X[k];
    }
  }
  if (seen) CK(cudaMemcpy(seen, c->ra.seen, 4ull * C, cudaMemcpyDeviceToHost));
  if (put_seq) CK(cudaMemcpy(put_seq, c->ra.put_seq, 8ull * C, cudaMemcpyDeviceToHost));
  if (payload) {
    const size_t esz = c->cfg.storage == MEL_STORE_F32 ? 4 : 2;
    CK(cudaMemcpy2D(payload, esz * c->N, c->ra.payload, esz * c->Npad, esz * c->N, C, cudaMemcpyDeviceToHost));
  }
  return MEL_OK;
}

// ---------------------------------------------------------------------------------
// Reservoir checkpoint (include/mel.h reservoir_save / reservoir_load)
// ---------------------------------------------------------------------------------
namespace {
struct CkptHdr {
  char magic[8];                 // "MELRES01"
  uint32_t C, N, storage, policy, S, theta, batch, pad;
  uint64_t Npad, seed, tail, drawn, n_pending;
  uint32_t closed, pad2;
};
uint64_t ckpt_bytes(const mel_ctx* c, uint64_t n_pending) {
  const uint64_t C = c->C, W = (C + 31) / 32, esz = c->cfg.storage == MEL_STORE_F32 ? 4 : 2;
  return sizeof(CkptHdr) + sizeof(ResDev) + C * (sizeof(SlotMeta) + 4 + 8 + 4 + 4) + 4 * W + C * c->N * esz +
         n_pending * (sizeof(StMeta) + 4ull * c->N);
}
}  // namespace

int reservoir_checkpoint_bytes(mel_ctx* c, uint64_t* bytes) {
  GUARD(c);
  if (!bytes) return fail(c, MEL_EINVAL, "null bytes");
  int r = sync_stream(c);
  if (r) return r;
  ResDev st;
  CK(cudaMemcpy(&st, c->d_st, sizeof st, cudaMemcpyDeviceToHost));
  *bytes = ckpt_bytes(c, c->tail - st.consumed);
  return MEL_OK;
}

int reservoir_save(mel_ctx* c, void* blob) {
  GUARD(c);
  if (!blob) return fail(c, MEL_EINVAL, "null blob");
  int r = sync_stream(c);
  if (r) return r;
  CK(cudaStreamSynchronize(c->copy_stream));
  const uint32_t C = c->C, W = (C + 31) / 32, S = c->cfg.staging_entries;
  const size_t esz = c->cfg.storage == MEL_STORE_F32 ? 4 : 2;
  ResDev st;
  CK(cudaMemcpy(&st, c->d_st, sizeof st, cudaMemcpyDeviceToHost));
  CkptHdr h{};
  memcpy(h.magic, "MELRES01", 8);
  h.C = C; h.N = c->N; h.storage = c->cfg.storage; h.policy = c->cfg.policy; h.S = S;
  h.theta = c->cfg.threshold; h.batch = c->cfg.batch; h.Npad = c->Npad; h.seed = c->cfg.seed;
  h.tail = c->tail; h.drawn = c->drawn; h.n_pending = c->tail - st.consumed; h.closed = c->closed ? 1u : 0u;
  char* o = static_cast<char*>(blob);
  memcpy(o, &h, sizeof h); o += sizeof h;
  memcpy(o, &st, sizeof st); o += sizeof st;
  CK(cudaMemcpy(o, c->ra.meta, sizeof(SlotMeta) * C, cudaMemcpyDeviceToHost)); o += sizeof(SlotMeta) * C;
  CK(cudaMemcpy(o, c->ra.seen, 4ull * C, cudaMemcpyDeviceToHost)); o += 4ull * C;
  CK(cudaMemcpy(o, c->ra.put_seq, 8ull * C, cudaMemcpyDeviceToHost)); o += 8ull * C;
  CK(cudaMemcpy(o, c->ra.bitmap, 4ull * W, cudaMemcpyDeviceToHost)); o += 4ull * W;
  CK(cudaMemcpy(o, c->ra.pos, 4ull * C, cudaMemcpyDeviceToHost)); o += 4ull * C;
  CK(cudaMemcpy(o, c->ra.bad, 4ull * C, cudaMemcpyDeviceToHost)); o += 4ull * C;
  CK(cudaMemcpy2D(o, esz * c->N, c->ra.payload, esz * c->Npad, esz * c->N, C, cudaMemcpyDeviceToHost));
  o += esz * c->N * C;
  // the puts still pending in the staging ring: metadata + the fp32 field (from the ring, or
  // from the caller's buffer for a zero-copy put, which the reservoir_put contract keeps valid)
  for (uint64_t k = st.consumed; k < c->tail; ++k) {
    const uint32_t e = (uint32_t)(k % S);
    memcpy(o, &c->h_stmeta[e], sizeof(StMeta)); o += sizeof(StMeta);
    const float* src = c->h_stsrc[e] ? c->h_stsrc[e] : c->ra.st_field + (uint64_t)e * c->Npad;
    CK(cudaMemcpy(o, src, 4ull * c->N, cudaMemcpyDeviceToHost)); o += 4ull * c->N;
  }
  return MEL_OK;
}

int reservoir_load(mel_ctx* c, const void* blob) {
  GUARD(c);
  if (!blob) return fail(c, MEL_EINVAL, "null blob");
  CkptHdr h;
  const char* i = static_cast<const char*>(blob);
  memcpy(&h, i, sizeof h); i += sizeof h;
  if (memcmp(h.magic, "MELRES01", 8) != 0) return fail(c, MEL_EINVAL, "not a reservoir checkpoint");
  if (h.C != c->C || h.N != c->N || h.storage != c->cfg.storage || h.policy != c->cfg.policy ||
      h.S != c->cfg.staging_entries || h.theta != c->cfg.threshold || h.batch != c->cfg.batch || h.Npad != c->Npad ||
      h.seed != c->cfg.seed)
    return fail(c, MEL_EINVAL, "checkpoint of a different configuration");
  if (c->tail != 0) return fail(c, MEL_EPROTO, "reservoir_load after puts on this context");
  if (h.n_pending > c->cfg.staging_entries) return fail(c, MEL_EINVAL, "malformed checkpoint");
  int r = sync_stream(c);
  if (r) return r;
  const uint32_t C = c->C, W = (C + 31) / 32, S = c->cfg.staging_entries;
  const size_t esz = c->cfg.storage == MEL_STORE_F32 ? 4 : 2;
  ResDev st;
  memcpy(&st, i, sizeof st); i += sizeof st;
  if (h.tail - st.consumed != h.n_pending) return fail(c, MEL_EINVAL, "malformed checkpoint");
  CK(cudaMemcpy(c->d_st, &st, sizeof st, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->ra.meta, i, sizeof(SlotMeta) * C, cudaMemcpyHostToDevice)); i += sizeof(SlotMeta) * C;
  CK(cudaMemcpy(c->ra.seen, i, 4ull * C, cudaMemcpyHostToDevice)); i += 4ull * C;
  CK(cudaMemcpy(c->ra.put_seq, i, 8ull * C, cudaMemcpyHostToDevice)); i += 8ull * C;
  CK(cudaMemcpy(c->ra.bitmap, i, 4ull * W, cudaMemcpyHostToDevice)); i += 4ull * W;
  CK(cudaMemcpy(c->ra.pos, i, 4ull * C, cudaMemcpyHostToDevice)); i += 4ull * C;
  CK(cudaMemcpy(c->ra.bad, i, 4ull * C, cudaMemcpyHostToDevice)); i += 4ull * C;
  CK(cudaMemcpy2D(c->ra.payload, esz * c->Npad, i, esz * c->N, esz * c->N, C, cudaMemcpyHostToDevice));
  i += esz * c->N * C;
  for (uint64_t k = st.consumed; k < h.tail; ++k) {
    const uint32_t e = (uint32_t)(k % S);
    memcpy(&c->h_stmeta[e], i, sizeof(StMeta)); i += sizeof(StMeta);
    c->h_stsrc[e] = nullptr;
    CK(cudaMemcpy(const_cast<float*>(c->ra.st_field) + (uint64_t)e * c->Npad, i, 4ull * c->N, cudaMemcpyHostToDevice));
    i += 4ull * c->N;
  }
  Mirror& m = *c->h_mirror;
  m.consumed = st.consumed; m.q = st.q; m.d = st.d; m.evictions = st.evictions;
  m.p = st.p; m.u = st.u; m.over = st.over; m.n_last = 0;
  c->tail = h.tail;
  c->known_consumed = st.consumed;
  c->drawn = h.drawn;
  c->closed = h.closed != 0;
  c->batch_known = false;
  c->batch_n = 0;
  return MEL_OK;
}

int mel_params_copy(mel_ctx* dst, mel_ctx* src) {
  GUARD(src);
  mel_ctx* c = src;                               // errors are reported on (and poison) src
  if (!dst || dst == src) return fail(src, MEL_EINVAL, "bad destination context");
  if (dst->poisoned) return dst->poisoned;
  if (dst->n_flat != src->n_flat || dst->L != src->L || dst->N != src->N || dst->Npad != src->Npad)
    return fail(src, MEL_EINVAL, "parameter layouts differ");
  for (int l = 0; l < src->L; ++l)
    if (dst->dims[l] != src->dims[l]) return fail(src, MEL_EINVAL, "parameter layouts differ");
  int r = gather_master(src, false);              // full fp32 W_L on src (collective under ZeRO)
  if (r) return r;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, src->dev, dst->dev) == cudaSuccess && can) {
    // direct NVLink copy engine path (otherwise the driver stages through host memory)
    cudaError_t e = cudaDeviceEnablePeerAccess(dst->dev, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return fail(c, MEL_ECUDA, "peer access: %s",
                                                                                 cudaGetErrorString(e));
    (void)cudaGetLastError();
  }
  cudaEvent_t ready, copied;
  CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  CK(cudaEventRecord(ready, src->stream));
  cudaSetDevice(dst->dev);
  CK(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming));
  CK(cudaStreamWaitEvent(dst->stream, ready, 0));
  CK(cudaMemcpyPeerAsync(dst->d_p, dst->dev, src->d_p, src->dev, 4ull * src->n_flat, dst->stream));
  CK(cudaEventRecord(copied, dst->stream));
  r = refresh_shadow(dst);
  if (r) return r;
  cudaSetDevice(src->dev);
  // src's next update of its parameters waits until they have been read
  CK(cudaStreamWaitEvent(src->stream, copied, 0));
  cudaEventDestroy(ready);
  cudaEventDestroy(copied);
  return MEL_OK;
}

int mel_stream_wait_event(mel_ctx* c, void* cuda_event) {
  GUARD(c);
  if (!cuda_event) return fail(c, MEL_EINVAL, "null event");
  CK(cudaStreamWaitEvent(c->stream, (cudaEvent_t)cuda_event, 0));
  return MEL_OK;
}

int mel_sync(mel_ctx* c) {
  GUARD(c);
  if (c->comm_stream) CK(cudaStreamSynchronize(c->comm_stream));
  return sync_stream(c);
}

int mel_kernel_time(mel_ctx* c, int k, double* ms, uint64_t* launches) {
  GUARD(c);
  if (k < 0 || k >= MEL_K_COUNT) return fail(c, MEL_EINVAL, "bad kernel id");
  int r = sync_stream(c);
  if (r) return r;
  drain_timers(c);
  if (ms) *ms = c->kms[k];
  if (launches) *launches = c->klaunch[k];
  return MEL_OK;
}

int mel_kernel_time_reset(mel_ctx* c) {
  GUARD(c);
  int r = sync_stream(c);
  if (r) return r;
  drain_timers(c);
  for (int k = 0; k < MEL_K_COUNT; ++k) { c->kms[k] = 0; c->klaunch[k] = 0; }
  return MEL_OK;
}

int mel_debug_counters(mel_ctx* c, uint64_t* out, int n) {
  GUARD(c);
  if (!out || n <= 0) return fail(c, MEL_EINVAL, "bad counter buffer");
  int r = sync_stream(c);
  if (r) return r;
  if (tc::read_k1_profile(reinterpret_cast<unsigned long long*>(out), n)) return fail(c, MEL_ECUDA, "counter read failed");
  return MEL_OK;
}

int mel_set_flags(mel_ctx* c, uint32_t flags) {
  GUARD(c);
  c->cfg.flags = flags;
  return MEL_OK;
}

int mel_launch_count(const mel_ctx* c, uint64_t* n) {
  if (!c || !n) return MEL_EINVAL;
  *n = c->launches;
  return MEL_OK;
}

}  // extern "C"
