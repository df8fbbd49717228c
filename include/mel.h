/*
 * mel.h -- C ABI of the B200-native reservoir-fed surrogate trainer
 * (arXiv 2309.16743, Meyer et al., "High Throughput Training of Deep Surrogates
 * from Large Ensemble Runs").  Library: paper_2309_16743_b200/libmel.so.
 *
 * Citations are PAPER.md line numbers (P:n) with the section they fall in.
 *
 * The calls follow the paper's statement of the problem:
 *   reservoir_put          <- client `send` of one time step u_X^t (§3.1)
 *                             into the rank's training buffer (Alg. 1 put)
 *   reservoir_close        <- "finalize_communication" of the last client /
 *                             "the reception is over" (Alg. 1)
 *   reservoir_sample_batch <- the training thread building a batch with b gets
 *                             (Alg. 1 get, "with replacement")
 *   surrogate_step         <- forward, MSE, backward, gradient all-reduce, Adam
 *
 *   surrogate_eval         <- validation on held-out simulations
 *
 * Conventions (all calls):
 *   - Every call returns an int status (enum mel_status).  Negative = error;
 *     on error the context state is unchanged, except MEL_ECUDA / MEL_ENCCL which
 *     poison the context (every later call returns the same code).
 *     mel_last_error() returns a human-readable message for the last error.
 *   - Pointers named *_host are host memory owned by the caller, only read or
 *     written during the call.  Device pointers are accepted only where a
 *     `*_on_device` flag says so; they are read in stream order on the
 *     context's stream and must stay valid until the next mel_sync().
 *   - The context owns all device memory (reservoir slots, staging ring,
 *     weights, Adam moments, activations, scratch).  Nothing is allocated per
 *     step.
 *   - Threads: one thread per context at a time (the caller serialises the
 *     producer and consumer roles; the order of calls is the op-log, reading R4
 *     in DESIGN.md).
 *   - Layout of parameters: tensors in the order W_1, b_1, ..., W_L, b_L, with
 *     W_l row-major [out][in] fp32, dims = [6, hidden..., n_field].
 */
#ifndef MEL_H_
#define MEL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MEL_ABI_VERSION 2u
#define MEL_HIST_BINS 64
#define MEL_MAX_TENSORS 6

enum mel_status {
  MEL_OK = 0,
  MEL_EAGAIN = 1,     /* put: staging ring full | sample: p <= theta during reception
                          | step: no rank has a batch (nothing done)            */
  MEL_EOS = 2,        /* step: every rank is closed and drained                */
  MEL_EINVAL = -1,    /* bad argument or configuration                                 */
  MEL_ECLOSED = -2,   /* put after reservoir_close                                     */
  MEL_EPROTO = -3,    /* double close                                                  */
  MEL_ECUDA = -4,     /* CUDA error (context poisoned)                                 */
  MEL_ENCCL = -5,     /* NCCL error (context poisoned)                                 */
  MEL_ENOMEM = -6,    /* device allocation failed                                      */
  MEL_ENONFINITE = -7 /* step skipped: a batch held non-finite inputs, or the loss is not
                         finite (see surrogate_step)                                    */
};

enum mel_precision {
  MEL_FP32 = 0,  /* parity mode: every contraction in fp32 FFMA (SIMT kernels)        */
  MEL_BF16 = 1   /* bench mode: output layer on tcgen05 (bf16 operands, fp32 TMEM
                    accumulation), fp32 master weights / Adam / head               */
};

enum mel_storage {
  MEL_STORE_F32 = 0,  /* slot stores RN_f32((u - lo) / (hi - lo))                      */
  MEL_STORE_BF16 = 1  /* slot stores RNE_bf16 of the same fp32 value                    */
};

enum mel_policy {               /* the training buffer                  */
  MEL_RESERVOIR = 0, /* Algorithm 1: draws with replacement once p > theta, a put into a
                        full buffer evicts a random *seen* item (the paper's method)     */
  MEL_FIFO = 1,      /* queue: a batch is the B oldest items, removed when read; needs
                        p >= B during reception (B <= C); a full buffer suspends puts   */
  MEL_FIRO = 2       /* list: B random draws with removal once p >= theta + B (theta + B
                        <= C); threshold 0 after reservoir_close                         */
};

typedef struct mel_ctx mel_ctx;

typedef struct {
  uint32_t abi_version;        /* must be MEL_ABI_VERSION                                */
  uint32_t n_field;            /* N = n*n outputs ("output of 1M neurons")          */
  uint32_t hidden[2];          /* hidden widths; {256,256}; tiny {32,0}          */
  uint32_t capacity;           /* C, reservoir slots per rank (6000)              */
  uint32_t threshold;          /* theta, watermark (1000); require theta < C      */
  uint32_t batch;              /* B per rank (10; bench: 1024); any B >= 1 -- the
                                  bf16 kernels run it padded to whole 64-row chunks,
                                  the padding rows masked out of loss and gradients   */
  uint32_t steps_per_sim;      /* tau, used for the input t/tau (100)             */
  float temp_lo, temp_hi;      /* normalisation range, 100 / 500 K               */
  uint32_t precision;          /* enum mel_precision                                     */
  uint32_t storage;            /* enum mel_storage                                       */
  double lr0, lr_min;          /* 1e-3, 2.5e-4                            */
  uint64_t lr_halving_samples; /* 10000 global samples                           */
  double beta1, beta2, eps;    /* Adam 0.9, 0.999, 1e-8 (reading R15)                    */
  uint64_t seed;               /* Philox key for SAMPLE/EVICT/DRAIN/INIT streams */
  uint32_t staging_entries;    /* depth of the pending-put ring (>= 1)                   */
  uint32_t flags;              /* MEL_FLAG_*                                             */
  uint32_t policy;             /* enum mel_policy (ABI v2)                               */
  uint32_t pad;
} mel_config;

#define MEL_FLAG_TIMING 1u     /* record CUDA events around every kernel (bench roofline) */
#define MEL_FLAG_UNFUSED_ADAM 8u /* world == 1, bf16: run Adam of W_L as its own kernel over a
                                    stored gradient instead of inside the output-layer kernel's
                                    dW epilogue (the default there from batch 256 on; below
                                    it the separate kernel is already the default, DESIGN
                                    §7).  Read at mel_create only.                          */
#define MEL_FLAG_NCCL_EXCHANGE 16u /* world > 1, bf16: NCCL reduce-scatter of dW_L + sharded Adam
                                      kernel + shadow all-gather instead of the in-kernel NVLink
                                      exchange (the default when every GPU pair has peer access;
                                      DESIGN §10).  Read at mel_create only.                     */
#define MEL_FLAG_FP32_EXCHANGE 32u /* world > 1, bf16, in-kernel exchange: dW contributions travel
                                      over NVLink and accumulate at the owner in fp32 instead of
                                      the default bf16 (bf16 halves the NVLink bytes: each peer
                                      contribution is rounded once, with R > 2 the owner-side
                                      additions round too, reading R22).  Read at
                                      mel_create only.                                          */
#define MEL_FLAG_NO_ZERO 2u    /* world > 1, bf16: plain all-reduce + replicated Adam instead of
                                  reduce-scatter / sharded Adam / shadow all-gather            */

typedef struct {
  uint64_t population, unseen, seen;     /* p, u, s = p - u                            */
  uint64_t puts;                         /* accepted reservoir_put calls               */
  uint64_t committed;                    /* q: puts that reached a slot                */
  uint64_t draws;                        /* d: SAMPLE + DRAIN draws                    */
  uint64_t evictions;
  uint64_t pending;                      /* accepted but not committed (back-pressure) */
  uint64_t steps;                        /* optimiser steps taken (Adam k)             */
  uint64_t samples;                      /* global samples consumed (LR schedule S)    */
  uint64_t hist[MEL_HIST_BINS];          /* retired items by final seen count (Fig. 3) */
  uint32_t over;                         /* reception over and pending empty           */
  uint32_t closed;
  double last_loss;                      /* loss of the last completed step            */
} mel_stats;

/* Fills *cfg with the paper's defaults for the given output width and
 * batch.  Always succeeds for non-NULL cfg. */
int mel_config_default(mel_config* cfg, uint32_t n_field, uint32_t batch);

/* Writes a 128-byte NCCL unique id into out128 (host).  Call on rank 0 only, then
 * broadcast it to every rank (the Python binding uses torch.distributed).
 * Errors: MEL_ENCCL. */
int mel_nccl_unique_id(void* out128);

/* Creates a context on `cuda_device`.  world > 1 requires nccl_id (128 B from
 * mel_nccl_unique_id); world == 1 requires nccl_id == NULL.  cuda_stream: a
 * cudaStream_t to run on, or NULL for a library-owned stream.  Weights are
 * initialised from the Philox INIT stream (identical on every rank: reading R13)
 * unless mel_set_params is called.  Errors: MEL_EINVAL (bad config: n_field == 0,
 * theta >= C, batch == 0, bf16 mode with the last hidden width not a multiple
 * of 64, ...), MEL_ECUDA, MEL_ENCCL, MEL_ENOMEM. */
int mel_create(const mel_config* cfg, int rank, int world, const void* nccl_id,
               int cuda_device, void* cuda_stream, mel_ctx** out);
void mel_destroy(mel_ctx* ctx);
const char* mel_last_error(const mel_ctx* ctx);

/* Number of parameter tensors (2 per layer) and, if shapes != NULL, their
 * [rows, cols] (cols = 1 for biases).  Total element count in *total. */
int mel_param_layout(const mel_ctx* ctx, uint32_t* n_tensors, uint32_t* shapes /* 2*n */,
                     uint64_t* total);

/* Host fp32 parameters in / out (tensor order above).  set: all ranks must set
 * identical values; resets nothing else.  get synchronises the stream; with world > 1
 * in bf16 mode (row-sharded W_L optimiser state) get is COLLECTIVE (all-gather). */
int mel_set_params(mel_ctx* ctx, const float* const* tensors_host);
int mel_get_params(mel_ctx* ctx, float* const* tensors_host);

/* Full optimiser state (params, Adam first/second moments, step count k and
 * global samples S), host fp32.  Used by checkpointing and by the re-anchored
 * parity harness.  Synchronises; COLLECTIVE with world > 1 in bf16 mode. */
typedef struct {
  float* const* p;
  float* const* m;
  float* const* v;
  uint64_t adam_step;
  uint64_t samples_seen;
} mel_state_view;
int mel_get_state(mel_ctx* ctx, mel_state_view* out);
int mel_set_state(mel_ctx* ctx, const mel_state_view* in);

/* Alg. 1 put of one time step (sim_id, t, X[5] kelvin, field[N] fp32
 * kelvin -- the fp32 wire data of P:210).  The item enters the pending FIFO; it
 * is committed to a slot at the next commit point (start of
 * reservoir_sample_batch, or reservoir_close).  field_on_device = 0: field is
 * host memory, copied before return (pinned memory makes the copy asynchronous);
 * 1: device pointer on this context's GPU, copied into the staging ring on the context's
 * stream at the call (the buffer is free once the stream has passed that point: at once
 * for a caller on the same stream; a producer on another stream orders its writes first,
 * e.g. with mel_stream_wait_event); 2: device pointer, ZERO COPY -- the commit that
 * consumes the item reads the caller's field in stream order, which under back-pressure
 * (u == C) may be several sample calls later, so the buffer must stay valid and
 * unchanged until the item is committed AND that commit has run: until reservoir_stats
 * (which synchronises) reports pending == 0 (needs 16-byte alignment and n_field % 4 == 0,
 * else it is copied as with 1).  Errors: MEL_ECLOSED after close, MEL_EAGAIN when the
 * staging ring is full (the caller retries after sampling), MEL_EINVAL. */
int reservoir_put(mel_ctx* ctx, uint32_t sim_id, uint32_t t, const float X_host[5],
                  const float* field, int field_on_device);

/* Drains up to max_msgs first-copy time steps from an ingest ring (include/mel_ingest.h,
 * SURVEY §8(f) f2) into the buffer: each is a reservoir_put of the message's (sim_id, t,
 * X, field), the field DMA-copied straight from the shared segment (page-locked on first
 * use), in the ring's arrival order; a call's slots are released to the clients once
 * its copies have landed (checked at the next call, at most 7 calls in flight; the
 * ring must not be consumed elsewhere meanwhile, and must outlive the context or its
 * last reservoir_ingest).  Waits up to timeout_us for the first message only.  Stops early
 * when the staging ring is full (sample to reach a commit point) or nothing is published.
 * *n_put_host = messages put.  MEL_EOS when the ring reports every expected client
 * finalized and drained and nothing was put; MEL_ECLOSED after reservoir_close. */
#ifndef MEL_INGEST_TYPEDEF_
#define MEL_INGEST_TYPEDEF_
typedef struct mel_ingest mel_ingest;
#endif
int reservoir_ingest(mel_ctx* ctx, mel_ingest* ing, uint32_t max_msgs, uint32_t timeout_us,
                     uint32_t* n_put_host);

/* The offline baseline: trains on batches first_batch ..
 * first_batch + n_batches - 1 of epoch `epoch` of a file dataset (include/mel_dataset.h;
 * order = reading R24 with `seed`; the last partial batch of an epoch is dropped) on the
 * same trainer: each record is a reservoir_put of its field (read by the dataset's loader
 * threads into pinned chunk buffers, double-buffered against the DMA), and every B puts
 * are handed out by the FIFO buffer as one batch (reservoir_sample_batch) and trained
 * (surrogate_step).  Requires mel_config.policy = MEL_FIFO and staging_entries >= batch.
 * losses_host (NULL or >= n_batches doubles) receives each step's loss;
 * *steps_host = steps done. */
#ifndef MEL_DATASET_TYPEDEF_
#define MEL_DATASET_TYPEDEF_
typedef struct mel_dataset mel_dataset;
#endif
int surrogate_train_offline(mel_ctx* ctx, mel_dataset* ds, uint64_t seed, uint32_t epoch,
                            uint32_t first_batch, uint32_t n_batches, double* losses_host,
                            uint32_t* steps_host);

/* The on-device heat-equation client (include/mel_heat.h): generates the
 * k time steps u_{X_j}^{t_j} on this GPU from the generator's basis (fp32) and puts
 * them (reservoir_put with a device field) in order -- generation and training in one
 * allocation.  X_host [k][5] kelvin, sim_host / t_host [k] (t < tau).  *n_put_host = items
 * put; MEL_EAGAIN if the staging ring filled first (the rest was not put: sample, then
 * resubmit from n_put).  MEL_EINVAL if the generator's grid^2 != n_field. */
#ifndef MEL_HEAT_TYPEDEF_
#define MEL_HEAT_TYPEDEF_
typedef struct mel_heat mel_heat;
#endif
int reservoir_put_generated(mel_ctx* ctx, mel_heat* gen, const uint32_t* sim_host, const float* X_host,
                            const uint32_t* t_host, uint32_t k, uint32_t* n_put_host);

/* Signals that reception is over ("When all the simulation data have been
 * generated the blocking related to the threshold is lifted").  Commits pending
 * puts.  A second call returns MEL_EPROTO. */
int reservoir_close(mel_ctx* ctx);

/* Alg. 1 get x B, batch-atomic: commit point, watermark gate
 * (p <= theta -> MEL_EAGAIN during reception), then B Philox draws with
 * replacement, seen counters updated (unseen -> seen).  After
 * close the buffer drains: every draw removes its item, the batch may be shorter
 * than B, and 0 items means this rank is empty.  slots_host (int32[B], nullable)
 * and n_host (nullable) receive the slot ids / count; either being non-NULL
 * synchronises the stream, both NULL keeps the call asynchronous (during
 * reception the count is B). */
int reservoir_sample_batch(mel_ctx* ctx, int32_t* slots_host, uint32_t* n_host);

/* One training step on the batch of the last reservoir_sample_batch: forward,
 * MSE loss, backward, mean all-reduce of the gradients over the
 * `world` ranks (NCCL), Adam with the LR schedule.
 * COLLECTIVE when world > 1: every rank calls it the same number of times; a rank
 * without a batch contributes 0 samples.  loss_host (nullable): global mean loss
 * of this step (synchronises); NULL keeps the step asynchronous.
 * Returns MEL_OK, MEL_EAGAIN (no rank had samples: nothing done -- the parameters,
 * moments and step counters are unchanged; at world 1 the call launches no training
 * kernel at all, only the record of its status for surrogate_step_result, and
 * synchronises), MEL_EOS (every rank closed and drained), MEL_ENONFINITE, errors.
 * Non-finite values: a put whose X or field holds NaN / inf marks its slot at commit; a
 * step whose batch (on any rank) contains such a slot updates nothing -- parameters,
 * moments, step and sample counters unchanged -- and returns MEL_ENONFINITE (also reported
 * as status 3 by surrogate_step_result; not a poisoning error, the next step trains).  A
 * non-finite loss from finite inputs (arithmetic overflow) also returns MEL_ENONFINITE and
 * skips the update of the head and biases, but the output layer's Adam runs inside K1
 * before the global loss exists: there, elements whose updated second moment would not be
 * finite (a non-finite gradient, or one whose square overflows) keep p, m, v (every Adam
 * kernel applies that rule) and the rest are updated. */
int surrogate_step(mel_ctx* ctx, double* loss_host);

/* Result of an earlier surrogate_step call without draining the stream: `call` is the
 * 0-based index of that call on this context, one of the last 16.  Waits only until that
 * step's kernels have finished (so a producer loop can read step i-1's loss while step i
 * runs), then returns its global mean loss (loss_host) and status (status_host: 0 trained,
 * 1 no rank had samples, 3 skipped: non-finite inputs or loss, see surrogate_step).
 * MEL_EINVAL for a call index out of range. */
int surrogate_step_result(mel_ctx* ctx, uint64_t call, double* loss_host, int* status_host);

/* Forward-only validation of n samples given on the host: X_host n x 5
 * kelvin, t_host n, fields_host n x N fp32 kelvin (nullable: then no MSE; it may also
 * point into this context's GPU memory -- told apart by unified addressing -- and is then
 * read in place instead of copied from the host).
 * mse_host (nullable) receives the MSE in normalised units (reading Q13);
 * pred_host (nullable, n x N) the predictions de-normalised to kelvin.
 * Synchronises; COLLECTIVE with world > 1 in bf16 mode (gathers the W_L master). */
int surrogate_eval(mel_ctx* ctx, const float* X_host, const uint32_t* t_host,
                   const float* fields_host, uint32_t n, double* mse_host, float* pred_host);

/* Snapshot of the reservoir and trainer counters (synchronises). */
int reservoir_stats(mel_ctx* ctx, mel_stats* out);

/* Test/diagnostic view of the reservoir (synchronises).  Each output is nullable
 * and sized C (payload: C x n_field elements of 4 B for MEL_STORE_F32, 2 B for
 * MEL_STORE_BF16).  Empty slots report sim = 0xFFFFFFFF. */
int reservoir_dump(mel_ctx* ctx, uint32_t* sim_host, uint32_t* t_host, float* X_host /*C x 5*/,
                   uint32_t* seen_host, uint64_t* put_seq_host, void* payload_host);

/* Checkpoint of the rank's buffer (SPEC's ServerCheckpoint; with mel_get_state /
 * mel_set_state a full restart point of the step, P:183's fault tolerance): the slots
 * (payload, metadata, seen counters, put sequence), the counters (population, unseen,
 * commits q, Philox draws d, evictions, retired-count histogram, FIFO head, FIRO position
 * list, closed / over) and the puts still pending in the staging ring, so that a context
 * restored from it draws, evicts and trains exactly as the saved one would have.
 * reservoir_checkpoint_bytes: size of the blob (synchronises); reservoir_save: writes it to
 * host memory (synchronises); reservoir_load: restores it into a fresh context created with
 * the same configuration (n_field, capacity, threshold, batch, storage, policy,
 * staging_entries, seed) before its first put -- MEL_EINVAL on a mismatch or a malformed
 * blob, MEL_EPROTO after puts.  The ingest log (mel_ingest.h) is the ingest ring's own
 * state and is not part of this blob. */
int reservoir_checkpoint_bytes(mel_ctx* ctx, uint64_t* bytes_host);
int reservoir_save(mel_ctx* ctx, void* blob_host);
int reservoir_load(mel_ctx* ctx, const void* blob_host);

/* Validation on a dedicated GPU (validation stalls the consumer):
 * copies src's fp32 parameters (every layer; W_L gathered under ZeRO, collectively) into
 * dst, a context of the same layout on another GPU, over NVLink (cudaMemcpyPeerAsync), and
 * refreshes dst's bf16 shadow.  Asynchronous: dst's stream waits for src's work so far and
 * src's stream waits for the copy before any later parameter update, so surrogate_eval on
 * dst runs beside src's training.  MEL_EINVAL if the layouts differ.  The Adam moments and
 * step counters are not copied. */
int mel_params_copy(mel_ctx* dst, mel_ctx* src);

/* Waits for all work queued on the context's stream. */
int mel_sync(mel_ctx* ctx);

/* Orders the context's stream after a CUDA event (cudaEvent_t) recorded by the caller, e.g.
 * on the stream that produced a device field before reservoir_put(..., 1 or 2). */
int mel_stream_wait_event(mel_ctx* ctx, void* cuda_event);

/* Virtual ranks (test mode; "the locally computed vector of weight updates is
 * all-reduced", SURVEY 4.2 T3'): `world` (2..8) ranks on ONE device, so that the
 * data-parallel path -- in bf16 mode the in-kernel gradient exchange of the output layer
 * (dW tiles TMA-stored / reduce-added into the owner rank's buffer, owner-side fused Adam,
 * new shadow rows pushed to every rank) -- runs and is checked on a single GPU.  Creates
 * `world` contexts (out[world], rank order) on cuda_device sharing `stream` (NULL: one is
 * created), each a full rank (own reservoir, batch, replica); they are used with every call
 * above except surrogate_step.  Their collectives run as device-side rank-ordered sums, and
 * the output layer's K1 as ONE cooperative launch of world x floor(#SMs / world) CTAs over
 * every rank's tiles (the ranks' CTAs wait on one another, so they must be co-resident).
 * bf16 mode needs the in-kernel exchange (no MEL_FLAG_NCCL_EXCHANGE / MEL_FLAG_NO_ZERO);
 * fp32 mode all-reduces the flat gradient.  Release each context with mel_destroy.
 * MEL_EINVAL, MEL_ENOMEM, MEL_ECUDA (nothing created). */
int mel_create_virtual(const mel_config* cfg, int world, int cuda_device, void* stream, mel_ctx** out);

/* One collective surrogate_step over the virtual ranks ctxs[0..world) (rank order; each
 * rank's batch is its last reservoir_sample_batch).  Same semantics and statuses as
 * surrogate_step at `world` ranks; loss_host (nullable) receives the global loss. */
int surrogate_step_virtual(mel_ctx* const* ctxs, int world, double* loss_host);

/* Per-kernel timing (flag MEL_FLAG_TIMING): total milliseconds and launch count
 * of kernel class `k` (enum mel_kernel) since the last reset, measured with CUDA
 * events on the launching stream.  Synchronises. */
enum mel_kernel {
  MEL_K_COMMIT = 0, MEL_K_SAMPLE, MEL_K_GATHER, MEL_K_HEAD_FWD, MEL_K_OUT_FWD_DW,
  MEL_K_OUT_DH, MEL_K_HEAD_BWD, MEL_K_ALLREDUCE, MEL_K_ADAM, MEL_K_LOSS, MEL_K_COUNT
};
int mel_kernel_time(mel_ctx* ctx, int k, double* ms_host, uint64_t* launches_host);
int mel_kernel_time_reset(mel_ctx* ctx);
/* Replaces cfg.flags (MEL_FLAG_*) from the next call on.  Always MEL_OK. */
int mel_set_flags(mel_ctx* ctx, uint32_t flags);
/* Diagnostic: per-CTA wait-cycle counters of the output-layer kernel's warp roles
 * (layout documented in csrc/tc_out.cu).  Copies up to n uint64 values. */
int mel_debug_counters(mel_ctx* ctx, uint64_t* out_host, int n);
/* Number of library kernel launches since creation (bench "gpu_launches"). */
int mel_launch_count(const mel_ctx* ctx, uint64_t* n_host);

#ifdef __cplusplus
}
#endif
#endif /* MEL_H_ */
