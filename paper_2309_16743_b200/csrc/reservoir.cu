// Reservoir kernels (Algorithm 1) in the
// deterministic op-log form of DESIGN.md (readings R1-R9):
//   commit_ctrl  : one control CTA applies the pending puts in FIFO order under
//                  the put rule: fill phase slot = p + lane prefix;
//                  full phase evicts the r-th *seen* slot (r from Philox EVICT(q)),
//                  found by a block-wide rank-select over the seen bitmap in SMEM;
//                  stops when every slot is unseen (P:264 back-pressure).
//   commit_copy  : data plane, one CTA row per committed put, 16-byte vector
//                  loads of the fp32 staging entry, normalised on the fly and
//                  stored as fp32 or bf16 (P:210 wire data, reading R8).
//   sample_kernel: B Philox SAMPLE(d+b) draws with replacement,
//                  seen counters by atomicAdd (order-free), u -= #(0->1); after
//                  the reception is over, sequential DRAIN draws with removal.
//   commit_sample_kernel: reservoir_sample_batch's commit control and draws in one
//                  launch (Reservoir policy), before the commit's copy grid.
//   gather_inputs: normalised network inputs (X, t) of the batch (reading Q13).
// The comparison buffers of P:221-223 (reading R21) reuse the same put / staging /
// commit machinery: commit appends while p < C (FIFO at ring slot head + p, FIRO at
// list position p -> slot pos[p]); FIFO sampling takes the B oldest items, FIRO makes
// B DRAIN-stream draws with removal (swap with the last list position, in SMEM).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace mel {

namespace {

constexpr int CTRL_THREADS = 1024;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// exclusive block scan of one value per thread (CTRL_THREADS threads)
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = warp_incl_scan(v);
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t x = (lane < (int)(blockDim.x >> 5)) ? s_warp[lane] : 0u;
    uint32_t xi = warp_incl_scan(x);
    s_warp[lane] = xi - x;
  }
  __syncthreads();
  uint32_t r = s_warp[w] + incl - v;
  __syncthreads();
  return r;
}

// FIFO / FIRO commit: append the pending puts while the buffer has room
__device__ void commit_queue(const ResArgs& a, uint64_t tail, uint32_t closed) {
  ResDev* st = a.st;
  const uint32_t p = st->p, u = st->u, head = st->head;
  const uint64_t q = st->q, consumed = st->consumed;
  uint32_t cnt = 0;
  if (consumed < tail && p < a.C) {
    const uint64_t avail = tail - consumed, room = a.C - p;
    cnt = (uint32_t)(avail < room ? avail : room);
  }
  for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
    const uint32_t j = a.policy == 1 ? (head + p + i) % a.C : a.pos[p + i];
    const uint32_t e = (uint32_t)((consumed + i) % a.S);
    a.meta[j] = a.st_meta[e];
    a.seen[j] = 0;
    a.put_seq[j] = q + i;
    a.plan[i] = make_uint2(e, j);
    a.plan_src[i] = a.st_src[e];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    st->p = p + cnt; st->u = u + cnt; st->q = q + cnt; st->consumed = consumed + cnt; st->n_plan = cnt;
    if (closed && consumed + cnt == tail) st->over = 1;
    Mirror* m = a.mirror;
    m->consumed = consumed + cnt; m->q = q + cnt; m->p = p + cnt; m->u = u + cnt; m->over = st->over;
    m->evictions = st->evictions; m->d = st->d;
  }
}

// Reservoir commit control (one CTA of CTRL_THREADS): the body of commit_ctrl and of the
// first half of commit_sample_kernel
__device__ __forceinline__ void commit_reservoir(const ResArgs& a, uint64_t tail, uint32_t closed) {
  // Seen bitmap + exclusive prefix of its word popcounts in SMEM.  One warp plans the
  // puts in order (fill slots p, p+1, ...; full phase: evict the r-th seen slot, found by
  // a binary search over the prefix and a find-n-th-set-bit, then the prefix updated
  // lane-parallel); the whole block then applies the plan in parallel (metadata copy from
  // the mapped staging entries, seen / put_seq reset, retired-count histogram).
  extern __shared__ uint32_t s_dyn[];
  const uint32_t W = (a.C + 31) / 32;
  uint32_t* s_bits = s_dyn;                      // [W]
  uint32_t* s_pref = s_dyn + W;                  // [W + 1]
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_res[3];                  // p, u, n_plan after planning (thread 0 -> block)
  __shared__ uint32_t s_nev;
  // the first CC_PF pending entries' metadata and source pointers live in mapped host
  // memory: their loads are issued first, so the PCIe round trip overlaps the bitmap scan
  // and the planning instead of following them
  constexpr uint32_t CC_PF = 256;
  __shared__ StMeta s_meta[CC_PF];
  __shared__ const float* s_src[CC_PF];
  ResDev* st = a.st;
  const uint64_t c0 = st->consumed;
  const uint64_t n_pf = tail - c0 < CC_PF ? tail - c0 : CC_PF;
  if (threadIdx.x < n_pf) {
    const uint32_t e = (uint32_t)((c0 + threadIdx.x) % a.S);
    s_meta[threadIdx.x] = a.st_meta[e];
    s_src[threadIdx.x] = a.st_src[e];
  }
  for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) s_bits[i] = a.bitmap[i];
  uint32_t p = st->p, u = st->u;
  const uint64_t q0 = st->q;
  __syncthreads();
  {
    const uint32_t wpt = (W + blockDim.x - 1) / blockDim.x;   // words per thread
    const uint32_t w0 = threadIdx.x * wpt;
    uint32_t cnt = 0;
    for (uint32_t k = 0; k < wpt; ++k)
      if (w0 + k < W) cnt += __popc(s_bits[w0 + k]);
    uint32_t run = block_excl_scan(cnt, s_warp);
    for (uint32_t k = 0; k < wpt; ++k)
      if (w0 + k < W) { s_pref[w0 + k] = run; run += __popc(s_bits[w0 + k]); }
    if (w0 < W && w0 + wpt >= W) s_pref[W] = run;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    uint64_t consumed = c0;
    uint32_t n_plan = 0, n_ev = 0;
    while (consumed < tail && u < a.C) {                      // all unseen -> wait
      if (p < a.C) {                                          // fill phase: dense prefix
        const uint64_t avail = tail - consumed, room = (uint64_t)(a.C - p);
        const uint32_t cnt = (uint32_t)(avail < room ? avail : room);
        for (uint32_t i = lane; i < cnt; i += 32)
          a.plan[n_plan + i] = make_uint2((uint32_t)((consumed + i) % a.S), p + i);
        p += cnt; u += cnt; consumed += cnt; n_plan += cnt;
        continue;
      }
      // full phase: the r-th seen slot in ascending slot id, r ~ Philox EVICT(q)
      uint32_t w = 0, j = 0;
      if (lane == 0) {
        const uint32_t r = bounded(philox_r64(a.seed, TAG_EVICT, q0 + n_plan, a.rank), p - u);
        uint32_t lo = 0, hi = W;                              // largest w with pref[w] <= r
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (s_pref[mid] <= r) lo = mid; else hi = mid;
        }
        w = lo;
        j = w * 32 + __fns(s_bits[w], 0, (int)(r - s_pref[w]) + 1);
        s_bits[w] &= ~(1u << (j & 31));                       // the new item is unseen
      }
      w = __shfl_sync(0xffffffffu, w, 0);
      j = __shfl_sync(0xffffffffu, j, 0);
      for (uint32_t i = w + 1 + lane; i <= W; i += 32) s_pref[i] -= 1;
      if (lane == 0) a.plan[n_plan] = make_uint2((uint32_t)(consumed % a.S), j | 0x80000000u);
      __syncwarp();
      u += 1; consumed += 1; n_plan += 1; n_ev += 1;
    }
    if (lane == 0) { s_res[0] = p; s_res[1] = u; s_res[2] = n_plan; s_nev = n_ev; }
  }
  __syncthreads();
  p = s_res[0]; u = s_res[1];
  const uint32_t n_plan = s_res[2];
  const uint64_t q = q0 + n_plan, consumed = c0 + n_plan;
  for (uint32_t i = threadIdx.x; i < n_plan; i += blockDim.x) {
    const uint2 ej = a.plan[i];
    const uint32_t j = ej.y & 0x7FFFFFFFu;
    if (ej.y & 0x80000000u) {                                 // evictee retired with its count
      const uint32_t sc = a.seen[j];
      atomicAdd(reinterpret_cast<unsigned long long*>(&st->hist[sc < HIST_BINS ? sc : HIST_BINS - 1]), 1ull);
    }
    const StMeta m = i < CC_PF ? s_meta[i] : a.st_meta[ej.x];     // plan entry i is pending entry c0 + i
    a.meta[j] = m;
    a.bad[j] = (isfinite(m.X[0]) && isfinite(m.X[1]) && isfinite(m.X[2]) && isfinite(m.X[3]) && isfinite(m.X[4])) ? 0u : 1u;
    a.seen[j] = 0;
    a.put_seq[j] = q0 + i;
    a.plan[i] = make_uint2(ej.x, j);
    a.plan_src[i] = i < CC_PF ? s_src[i] : a.st_src[ej.x];
  }
  if (threadIdx.x == 0) st->evictions += s_nev;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) a.bitmap[i] = s_bits[i];
  if (threadIdx.x == 0) {
    st->p = p; st->u = u; st->q = q; st->consumed = consumed; st->n_plan = n_plan;
    if (closed && consumed == tail) st->over = 1;
    Mirror* m = a.mirror;
    m->consumed = consumed; m->q = q; m->p = p; m->u = u; m->over = st->over;
    m->evictions = st->evictions; m->d = st->d;
  }
}

__global__ void __launch_bounds__(CTRL_THREADS, 1)
commit_ctrl(ResArgs a, uint64_t tail, uint32_t closed) {
  pdl_enter();
  if (a.policy != 0) commit_queue(a, tail, closed);
  else commit_reservoir(a, tail, closed);
}

// data plane: blockIdx.y = plan index, 4 floats per thread per iteration
template <int STORAGE>
__global__ void __launch_bounds__(256)
commit_copy(ResArgs a) {
  pdl_enter();
  // a fixed grid strides over every committed entry (the host only knows an upper bound
  // on their number): 16-byte loads of the staged fp32 field (or, for a device put, of the
  // caller's own field: no staging copy), normalised on the fly
  const uint32_t n_plan = a.st->n_plan;
  const uint32_t n4 = (a.N + 3) / 4;
  for (uint32_t y = blockIdx.y; y < n_plan; y += gridDim.y) {     // gridDim.y entries at a time
    const uint2 ej = a.plan[y];
    const float* zc = a.plan_src[y];              // zero-copy device put: read the caller's field
    const float4* src = reinterpret_cast<const float4*>(zc ? zc : a.st_field + (uint64_t)ej.x * a.Npad);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
      float4 v = __ldg(src + i);
      float o[4] = {v.x, v.y, v.z, v.w};
      // a non-finite value marks the slot (its batches are skipped, surrogate_step ->
      // MEL_ENONFINITE); the padding lanes past N never count
      if (!(isfinite(v.x) || 4 * i >= a.N) || !(isfinite(v.y) || 4 * i + 1 >= a.N) ||
          !(isfinite(v.z) || 4 * i + 2 >= a.N) || !(isfinite(v.w) || 4 * i + 3 >= a.N))
        atomicOr(&a.bad[ej.y], 1u);
#pragma unroll
      for (int c = 0; c < 4; ++c) o[c] = (4 * i + c < a.N) ? normalise_rn(o[c], a.lo, a.span) : 0.f;
      if (STORAGE == 0) {
        float4* dst = reinterpret_cast<float4*>(static_cast<float*>(a.payload) + (uint64_t)ej.y * a.Npad);
        dst[i] = make_float4(o[0], o[1], o[2], o[3]);
      } else {
        __nv_bfloat162 lo = __floats2bfloat162_rn(o[0], o[1]);   // RNE
        __nv_bfloat162 hi = __floats2bfloat162_rn(o[2], o[3]);
        uint2 pk = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
        uint2* dst = reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.payload) + (uint64_t)ej.y * a.Npad);
        dst[i] = pk;
      }
    }
  }
}

constexpr int SAMPLE_THREADS = 1024;

// retire a FIFO / FIRO item: seen once, then removed (hist[1] counts it)
__device__ __forceinline__ void finish_queue_batch(const ResArgs& a, uint32_t p, uint32_t n, uint64_t d_new) {
  ResDev* st = a.st;
  st->hist[1] += n;
  st->u -= n;
  st->p = p - n;
  st->d = d_new;
  st->n_last = n;
  Mirror* m = a.mirror;
  m->p = p - n; m->u = st->u; m->d = d_new; m->n_last = n; m->over = st->over;
}

// FIFO: the n oldest items, n = B during reception (needs p >= B), min(B, p) after
__global__ void __launch_bounds__(SAMPLE_THREADS, 1)
fifo_sample_kernel(ResArgs a, int32_t* slots, uint32_t B) {
  pdl_enter();
  ResDev* st = a.st;
  const uint32_t p = st->p, head = st->head;
  const uint32_t n = st->over ? (p < B ? p : B) : (p >= B ? B : 0u);
  for (uint32_t b = threadIdx.x; b < n; b += blockDim.x) {
    const uint32_t j = (head + b) % a.C;
    slots[b] = (int32_t)j;
    a.seen[j] = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    st->head = (head + n) % a.C;
    finish_queue_batch(a, p, n, st->d + n);
  }
}

// FIRO: n draws k_b = bounded_DRAIN(d + b)(p - b) over the shrinking list, each
// removing its item by swapping it with the last list position.  The draws are computed
// in parallel (they depend only on p - b); the swap chain runs on one thread over the
// position permutation staged in SMEM (global memory when C does not fit).
constexpr uint32_t FIRO_SMEM_SLOTS = 48 * 1024;
__global__ void __launch_bounds__(SAMPLE_THREADS, 1)
firo_sample_kernel(ResArgs a, int32_t* slots, uint32_t B) {
  pdl_enter();
  extern __shared__ uint32_t s_pos[];
  ResDev* st = a.st;
  const uint32_t p = st->p;
  const uint64_t d = st->d;
  const uint32_t need = st->over ? 1u : a.theta + B;
  const uint32_t n = p >= need ? (p < B ? p : B) : 0u;
  const bool in_smem = a.C <= FIRO_SMEM_SLOTS;
  uint32_t* pos = in_smem ? s_pos : a.pos;
  if (in_smem)
    for (uint32_t i = threadIdx.x; i < a.C; i += blockDim.x) s_pos[i] = a.pos[i];
  for (uint32_t b = threadIdx.x; b < n; b += blockDim.x)
    slots[b] = (int32_t)bounded(philox_r64(a.seed, TAG_DRAIN, d + b, a.rank), p - b);   // k_b, for now
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t b = 0; b < n; ++b) {
      const uint32_t k = (uint32_t)slots[b], last = p - 1 - b;
      const uint32_t j = pos[k];
      pos[k] = pos[last];
      pos[last] = j;
      slots[b] = (int32_t)j;
    }
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < n; b += blockDim.x) a.seen[slots[b]] = 1;
  if (in_smem)
    for (uint32_t i = threadIdx.x; i < a.C; i += blockDim.x) a.pos[i] = s_pos[i];
  if (threadIdx.x == 0) finish_queue_batch(a, p, n, d + n);
}

// pos_smem: entries of pos[] the caller's dynamic shared memory holds (0: none)
__device__ __forceinline__ void sample_reservoir(const ResArgs& a, int32_t* slots, uint32_t B, uint32_t pos_smem) {
  __shared__ uint32_t s_cnt;
  ResDev* st = a.st;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const uint32_t p = st->p;
  const uint64_t d = st->d;
  if (!st->over) {
    if (p <= a.theta) {                          // P:242 watermark gate
      if (threadIdx.x == 0) { st->n_last = 0; a.mirror->n_last = 0; }
      return;
    }
    uint32_t local = 0;
    for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) {
      const uint32_t i = bounded(philox_r64(a.seed, TAG_SAMPLE, d + b, a.rank), p);
      slots[b] = (int32_t)i;
      const uint32_t old = atomicAdd(&a.seen[i], 1u);
      if (old == 0) { ++local; atomicOr(&a.bitmap[i >> 5], 1u << (i & 31)); }
    }
    if (local) atomicAdd(&s_cnt, local);
    __syncthreads();
    if (threadIdx.x == 0) {
      st->u -= s_cnt;
      st->d = d + B;
      st->n_last = B;
      Mirror* m = a.mirror;
      m->u = st->u; m->d = st->d; m->n_last = B; m->p = p; m->over = 0;
    }
    return;
  }
  // drain (P:249-258 with is_reception_over): n = min(B, p) draws, each removing its item.
  // Draw b is k_b = bounded(Philox(DRAIN, d + b), p - b) -- it depends only on b -- so the
  // draws run in parallel; the removal chain pos[k_b] <- pos[p - 1 - b] runs on one thread,
  // over pos[] staged in shared memory when it fits; the seen / histogram / u updates touch
  // distinct slots (no replacement) and run in parallel again.  Same result as drawing one
  // by one (the round-1 kernel did, on one thread, ~0.1 ms per 1024-draw batch).
  const uint32_t n = p < B ? p : B;
  for (uint32_t b = threadIdx.x; b < n; b += blockDim.x)
    slots[b] = (int32_t)bounded(philox_r64(a.seed, TAG_DRAIN, d + b, a.rank), p - b);
  extern __shared__ uint32_t s_dyn[];
  const bool in_smem = p <= pos_smem;
  uint32_t* pos = in_smem ? s_dyn : a.pos;
  if (in_smem)
    for (uint32_t i = threadIdx.x; i < p; i += blockDim.x) s_dyn[i] = a.pos[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t b = 0; b < n; ++b) {
      const uint32_t k = (uint32_t)slots[b];
      const uint32_t j = pos[k];
      pos[k] = pos[p - 1 - b];
      slots[b] = (int32_t)j;
    }
  }
  __syncthreads();
  if (in_smem)
    for (uint32_t i = threadIdx.x; i < p; i += blockDim.x) a.pos[i] = s_dyn[i];
  uint32_t zeros = 0;
  for (uint32_t b = threadIdx.x; b < n; b += blockDim.x) {
    const uint32_t j = (uint32_t)slots[b];
    const uint32_t sc = a.seen[j];
    a.seen[j] = sc + 1;
    if (sc == 0) ++zeros;
    atomicAdd(reinterpret_cast<unsigned long long*>(&st->hist[sc + 1 < HIST_BINS ? sc + 1 : HIST_BINS - 1]), 1ull);
  }
  if (zeros) atomicAdd(&s_cnt, zeros);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t u = st->u - s_cnt;
    st->p = p - n; st->u = u; st->d = d + n; st->n_last = n;
    Mirror* m = a.mirror;
    m->p = p - n; m->u = u; m->d = d + n; m->n_last = n; m->over = 1;
  }
}

__global__ void __launch_bounds__(SAMPLE_THREADS, 1)
sample_kernel(ResArgs a, int32_t* slots, uint32_t B) {
  pdl_enter();
  sample_reservoir(a, slots, B, 0u);
}

// reservoir_sample_batch's commit point and draw in one launch (Reservoir policy): the
// commit control, then -- after a block barrier, which orders the commit's global writes
// (p, u, bitmap, seen counters) before the draws -- the sample.  The commit's data plane
// (commit_copy) follows in the stream; the draws read only slot metadata, never payloads.
static_assert(CTRL_THREADS == SAMPLE_THREADS, "one block size for both halves");
__global__ void __launch_bounds__(CTRL_THREADS, 1)
commit_sample_kernel(ResArgs a, uint64_t tail, uint32_t closed, int32_t* slots, uint32_t B, uint32_t pos_smem) {
  pdl_enter();
  commit_reservoir(a, tail, closed);
  __syncthreads();                                  // (the commit is done with the shared memory)
  sample_reservoir(a, slots, B, pos_smem);
}

__global__ void gather_inputs(ResArgs a, const int32_t* slots, uint32_t B, uint32_t tau, float* xn) {
  pdl_enter();
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const uint32_t n = a.st->n_last;
  float out[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (b < n) {
    if (a.bad[slots[b]]) atomicOr(&a.st->bad_batch, 1u);     // reset by step_finalize
    const SlotMeta m = a.meta[slots[b]];
#pragma unroll
    for (int c = 0; c < 5; ++c) out[c] = normalise_rn(m.X[c], a.lo, a.span);
    out[5] = __fdiv_rn((float)m.t, (float)tau);
  }
  float4* dst = reinterpret_cast<float4*>(xn + (uint64_t)b * 8);
  dst[0] = make_float4(out[0], out[1], out[2], out[3]);
  dst[1] = make_float4(out[4], out[5], out[6], out[7]);
}

__global__ void init_res(ResArgs a) {
  pdl_enter();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.C; i += gridDim.x * blockDim.x) {
    a.pos[i] = i;
    a.seen[i] = 0;
    a.put_seq[i] = ~0ull;
    SlotMeta m; m.sim = 0xFFFFFFFFu; m.t = 0xFFFFFFFFu;
    for (int c = 0; c < 5; ++c) m.X[c] = 0.f;
    m.pad = 0;
    a.meta[i] = m;
  }
}

}  // namespace

void launch_commit(const ResArgs& a, uint64_t tail, uint32_t closed, uint32_t max_entries, cudaStream_t s) {
  const uint32_t W = (a.C + 31) / 32;
  const size_t smem = (size_t)(2 * W + 1) * 4;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(commit_ctrl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_pdl(commit_ctrl, dim3(1), dim3(CTRL_THREADS), smem, s, a, tail, closed);
  if (max_entries == 0) return;
  const uint32_t n4 = (a.N + 3) / 4;
  uint32_t gx = (n4 + 255) / 256;
#ifndef MEL_CC_ENTRIES
#define MEL_CC_ENTRIES 4   // entries whose copies run side by side (blockIdx.y)
#endif
  const uint32_t gy = max_entries < MEL_CC_ENTRIES ? max_entries : MEL_CC_ENTRIES;   // entries in flight
  const uint32_t cap = 148u * 4u * (max_entries < 4 ? max_entries : 4u);   // ~ one wave per 4 entries
  if (gx > cap) gx = cap;
  dim3 grid(gx, gy);
  if (a.storage == 0) launch_pdl(commit_copy<0>, dim3(grid), dim3(256), 0, s, a);
  else launch_pdl(commit_copy<1>, dim3(grid), dim3(256), 0, s, a);
}

void launch_commit_sample(const ResArgs& a, uint64_t tail, uint32_t closed, uint32_t max_entries, int32_t* slots,
                          uint32_t B, cudaStream_t s) {
  // dynamic shared memory: the commit's bitmap + prefix, then (drain) the position list
  const uint32_t W = (a.C + 31) / 32;
  constexpr uint32_t POS_SMEM_MAX = 50 * 1024;       // entries (200 KB); larger C drains from global
  const uint32_t pos_smem = a.C <= POS_SMEM_MAX ? a.C : 0u;
  const size_t smem = std::max((size_t)(2 * W + 1) * 4, (size_t)pos_smem * 4);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(commit_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_pdl(commit_sample_kernel, dim3(1), dim3(CTRL_THREADS), smem, s, a, tail, closed, slots, B, pos_smem);
  if (max_entries == 0) return;
  const uint32_t n4 = (a.N + 3) / 4;
  uint32_t gx = (n4 + 255) / 256;
  const uint32_t cap = 148u * 4u * (max_entries < 4 ? max_entries : 4u);
  if (gx > cap) gx = cap;
  const uint32_t gy = max_entries < MEL_CC_ENTRIES ? max_entries : MEL_CC_ENTRIES;
  if (a.storage == 0) launch_pdl(commit_copy<0>, dim3(gx, gy), dim3(256), 0, s, a);
  else launch_pdl(commit_copy<1>, dim3(gx, gy), dim3(256), 0, s, a);
}

void launch_sample(const ResArgs& a, int32_t* slots, uint32_t B, cudaStream_t s) {
  if (a.policy == 1) {
    launch_pdl(fifo_sample_kernel, dim3(1), dim3(SAMPLE_THREADS), 0, s, a, slots, B);
  } else if (a.policy == 2) {
    const size_t smem = a.C <= FIRO_SMEM_SLOTS ? (size_t)a.C * 4 : 0;
    if (smem > 48 * 1024) cudaFuncSetAttribute(firo_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(firo_sample_kernel, dim3(1), dim3(SAMPLE_THREADS), smem, s, a, slots, B);
  } else {
    launch_pdl(sample_kernel, dim3(1), dim3(SAMPLE_THREADS), 0, s, a, slots, B);
  }
}

void launch_gather(const ResArgs& a, const int32_t* slots, uint32_t B, uint32_t tau, float* xn, cudaStream_t s) {
  launch_pdl(gather_inputs, dim3((B + 127) / 128), dim3(128), 0, s, a, slots, B, tau, xn);
}

void launch_init_res(const ResArgs& a, cudaStream_t s) {
  launch_pdl(init_res, dim3(256), dim3(256), 0, s, a);
}

}  // namespace mel
