// Ingest channel (include/mel_ingest.h): simulation clients -> one shared-memory ring per
// server rank.  Host-only C++; built into libmel_ingest.so (clients) and libmel.so (server).
//
// Ring = bounded multi-producer / single-consumer queue of S fixed-size slots.  Slot k
// carries a sequence number that cycles  k -> (claimed, still k) -> k+1 (published) ->
// k+S (released, free for the ticket k+S).  A client claims ticket `pos` only when its slot
// is free for that lap (seq == pos, CAS on the shared enqueue counter), so a claim never
// waits; it then converts its fp64 field into the slot and publishes with a release
// store.  The server consumes tickets in order; a claimed-but-unpublished ticket whose
// claimant process is gone is skipped (the client restart case of P:183).
#include "mel_ingest.h"

#include <atomic>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <new>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include <fcntl.h>
#include <signal.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/statvfs.h>
#include <time.h>
#include <unistd.h>

namespace {

constexpr int ST_OK = 0, ST_EAGAIN = 1, ST_EOS = 2, ST_EINVAL = -1, ST_EPROTO = -3, ST_ENOMEM = -6;
constexpr uint64_t MAGIC = 0x53454e49474e454dull;   // "MENGINES" little-endian tag
constexpr uint32_t KIND_DATA = 0, KIND_FIN = 1;
constexpr uint64_t HDR_BYTES = 4096;
constexpr uint64_t SLOT_HDR_BYTES = 256;                // the field starts 256-byte aligned

struct RingHdr {
  std::atomic<uint64_t> magic;
  uint32_t version, n_field, slots, pad0;
  uint64_t slot_bytes, total_bytes;
  alignas(64) std::atomic<uint64_t> enq;   // next ticket to claim (clients)
  alignas(64) std::atomic<uint64_t> deq;   // next ticket the server will look at (informational)
};
static_assert(sizeof(RingHdr) <= HDR_BYTES, "ring header");

struct SlotHdr {
  std::atomic<uint64_t> seq;
  std::atomic<int32_t> pid;    // claimant (0 until the claimant writes it; cleared on release)
  uint32_t kind, sim, t;
  float X[5];
};
static_assert(sizeof(SlotHdr) <= SLOT_HDR_BYTES, "slot header");
static_assert(std::atomic<uint64_t>::is_always_lock_free, "address-free atomics needed across processes");

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

uint64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
}

// spin briefly, then sleep in 5 us steps; false once the deadline has passed
struct Waiter {
  uint64_t deadline;
  uint32_t spins = 0;
  explicit Waiter(uint32_t timeout_us) : deadline(now_ns() + 1000ull * timeout_us) {}
  bool again() {
    if (++spins < 256) return true;
    if (now_ns() >= deadline) return false;
    timespec ts{0, 5000};
    nanosleep(&ts, nullptr);
    return true;
  }
};

// backing file: $MEL_INGEST_DIR, else /dev/shm (tmpfs: page-lockable by cudaHostRegister)
std::string seg_path(const char* name, uint32_t rank) {
  const char* dir = getenv("MEL_INGEST_DIR");
  std::string d = dir && *dir ? dir : "/dev/shm";
  return d + "/mel_ingest." + name + "." + std::to_string(rank);
}

struct Mapping {
  uint8_t* base = nullptr;
  uint64_t bytes = 0;
  RingHdr* hdr() const { return reinterpret_cast<RingHdr*>(base); }
  SlotHdr* slot(uint64_t ticket) const {
    const RingHdr* h = hdr();
    return reinterpret_cast<SlotHdr*>(base + HDR_BYTES + (ticket % h->slots) * h->slot_bytes);
  }
  float* field(SlotHdr* s) const { return reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(s) + SLOT_HDR_BYTES); }
};

bool process_gone(int32_t pid) { return pid > 0 && kill(pid, 0) == -1 && errno == ESRCH; }

}  // namespace

struct mel_ingest {
  Mapping m;
  std::string path;
  uint32_t rank = 0, expected = 0;
  uint64_t head = 0;                                   // next ticket to examine
  struct Entry { uint64_t ticket; bool returned, done; };
  std::deque<Entry> pending;                           // examined, not yet released (ticket order)
  std::unordered_map<uint32_t, std::vector<uint64_t>> log;   // per client: bitmap over t
  std::set<uint32_t> finalized;
  mel_ingest_stats st{};
};

struct mel_client {
  std::vector<Mapping> rings;
  uint32_t id = 0, world = 0, n_field = 0;
  bool finalized = false;
  bool die_after_claim = false;   // fault injection for tests: MEL_INGEST_FAULT=die_after_claim
  bool die_after_pid = false;     //   ... MEL_INGEST_FAULT=die_after_pid (slot reserved, ticket not taken)
};

namespace {

void release_done_prefix(mel_ingest* g) {
  const uint32_t S = g->m.hdr()->slots;
  while (!g->pending.empty() && g->pending.front().done) {
    SlotHdr* s = g->m.slot(g->pending.front().ticket);
    s->pid.store(0, std::memory_order_relaxed);
    s->seq.store(g->pending.front().ticket + S, std::memory_order_release);
    g->pending.pop_front();
  }
}

bool log_test_and_set(mel_ingest* g, uint32_t sim, uint32_t t) {
  auto& bits = g->log[sim];
  const size_t w = t / 64;
  if (bits.size() <= w) bits.resize(w + 1, 0);
  const uint64_t b = 1ull << (t % 64);
  const bool seen = (bits[w] & b) != 0;
  bits[w] |= b;
  return seen;
}

int map_file(const std::string& path, bool create, uint64_t bytes, Mapping* out) {
  int fd;
  if (create) {
    unlink(path.c_str());
    fd = open(path.c_str(), O_RDWR | O_CREAT | O_EXCL, 0600);
    if (fd < 0) return ST_ENOMEM;
    if (ftruncate(fd, (off_t)bytes) != 0) { close(fd); unlink(path.c_str()); return ST_ENOMEM; }
  } else {
    fd = open(path.c_str(), O_RDWR);
    if (fd < 0) return ST_ENOMEM;
    struct stat sb;
    if (fstat(fd, &sb) != 0 || (uint64_t)sb.st_size < HDR_BYTES) { close(fd); return ST_EPROTO; }
    bytes = (uint64_t)sb.st_size;
  }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return ST_ENOMEM;
  out->base = static_cast<uint8_t*>(p);
  out->bytes = bytes;
  return ST_OK;
}

}  // namespace

extern "C" {

uint32_t mel_route(uint32_t client_id, uint32_t t, uint32_t world) {
  return world ? (uint32_t)(((uint64_t)client_id + t) % world) : 0u;
}

int mel_ingest_create(const char* name, uint32_t rank, uint32_t n_field, uint32_t slots, uint32_t expected_clients,
                      mel_ingest** out) {
  if (!name || !out || !*name || strlen(name) > 200 || strchr(name, '/') || n_field == 0 || slots < 2)
    return ST_EINVAL;
  *out = nullptr;
  const uint64_t slot_bytes = SLOT_HDR_BYTES + round_up(4ull * n_field, 256);
  const uint64_t bytes = HDR_BYTES + slot_bytes * slots;
  mel_ingest* g = new (std::nothrow) mel_ingest;
  if (!g) return ST_ENOMEM;
  g->path = seg_path(name, rank);
  int r = map_file(g->path, true, bytes, &g->m);
  if (r) { delete g; return r; }
  RingHdr* h = g->m.hdr();
  h->version = MEL_INGEST_VERSION; h->n_field = n_field; h->slots = slots; h->pad0 = 0;
  h->slot_bytes = slot_bytes; h->total_bytes = bytes;
  h->enq.store(0, std::memory_order_relaxed);
  h->deq.store(0, std::memory_order_relaxed);
  for (uint64_t k = 0; k < slots; ++k) {
    SlotHdr* s = g->m.slot(k);
    s->pid.store(0, std::memory_order_relaxed);
    s->seq.store(k, std::memory_order_relaxed);
  }
  h->magic.store(MAGIC, std::memory_order_release);   // clients attach only after this
  g->rank = rank;
  g->expected = expected_clients;
  *out = g;
  return ST_OK;
}

int mel_ingest_next(mel_ingest* g, mel_ingest_msg* out, uint32_t timeout_us) {
  if (!g || !out) return ST_EINVAL;
  RingHdr* h = g->m.hdr();
  Waiter w(timeout_us);
  for (;;) {
    SlotHdr* s = g->m.slot(g->head);
    const uint64_t seq = s->seq.load(std::memory_order_acquire);
    if (seq == g->head + 1) {                            // published
      const uint64_t ticket = g->head++;
      h->deq.store(g->head, std::memory_order_relaxed);
      if (s->kind == KIND_FIN) {
        g->finalized.insert(s->sim);
        g->st.finalized += 1;
        g->pending.push_back({ticket, false, true});
        release_done_prefix(g);
        continue;
      }
      if (g->log.find(s->sim) == g->log.end()) g->st.clients += 1;
      if (log_test_and_set(g, s->sim, s->t)) {           // already received: discard
        g->st.duplicates += 1;
        g->pending.push_back({ticket, false, true});
        release_done_prefix(g);
        continue;
      }
      g->pending.push_back({ticket, true, false});
      out->sim_id = s->sim;
      out->t = s->t;
      for (int i = 0; i < 5; ++i) out->X[i] = s->X[i];
      out->pad = 0;
      out->field = g->m.field(s);
      out->ticket = ticket;
      g->st.received += 1;
      g->st.bytes += 4ull * h->n_field;
      return ST_OK;
    }
    const bool claimed = h->enq.load(std::memory_order_acquire) > g->head;
    if (claimed && process_gone(s->pid.load(std::memory_order_relaxed)) &&
        s->seq.load(std::memory_order_acquire) != g->head + 1) {
      // the claimant died between its claim and its publish: skip the ticket
      g->st.abandoned += 1;
      g->pending.push_back({g->head++, false, true});
      h->deq.store(g->head, std::memory_order_relaxed);
      release_done_prefix(g);
      continue;
    }
    if (!claimed && g->expected && g->finalized.size() >= g->expected) return ST_EOS;
    if (!w.again()) return ST_EAGAIN;
  }
}

int mel_ingest_release(mel_ingest* g) {
  if (!g) return ST_EINVAL;
  for (auto& e : g->pending)
    if (e.returned && !e.done) {
      e.done = true;
      release_done_prefix(g);
      return ST_OK;
    }
  return ST_EPROTO;
}

uint32_t mel_ingest_outstanding(const mel_ingest* g) {
  if (!g) return 0;
  uint32_t n = 0;
  for (const auto& e : g->pending) n += (e.returned && !e.done) ? 1u : 0u;
  return n;
}

int mel_ingest_stats_get(const mel_ingest* g, mel_ingest_stats* out) {
  if (!g || !out) return ST_EINVAL;
  *out = g->st;
  return ST_OK;
}

int mel_ingest_segment(const mel_ingest* g, void** base, uint64_t* bytes) {
  if (!g || !base || !bytes) return ST_EINVAL;
  *base = g->m.base;
  *bytes = g->m.bytes;
  return ST_OK;
}

void mel_ingest_destroy(mel_ingest* g) {
  if (!g) return;
  if (g->m.base) munmap(g->m.base, g->m.bytes);
  unlink(g->path.c_str());
  delete g;
}

int mel_client_open(const char* name, uint32_t world, uint32_t client_id, mel_client** out) {
  if (!name || !out || !*name || strchr(name, '/') || world == 0) return ST_EINVAL;
  *out = nullptr;
  mel_client* c = new (std::nothrow) mel_client;
  if (!c) return ST_ENOMEM;
  c->id = client_id;
  c->world = world;
  const char* fault = getenv("MEL_INGEST_FAULT");
  c->die_after_claim = fault && strcmp(fault, "die_after_claim") == 0;
  c->die_after_pid = fault && strcmp(fault, "die_after_pid") == 0;
  for (uint32_t r = 0; r < world; ++r) {
    Mapping m;
    int st = map_file(seg_path(name, r), false, 0, &m);
    if (st == ST_OK) {
      const RingHdr* h = m.hdr();
      if (h->magic.load(std::memory_order_acquire) != MAGIC || h->version != MEL_INGEST_VERSION ||
          h->total_bytes != m.bytes || (c->n_field && h->n_field != c->n_field))
        st = ST_EPROTO;
      else
        c->n_field = h->n_field;
    }
    if (st != ST_OK) {
      if (m.base) munmap(m.base, m.bytes);
      mel_client_close(c);
      return st;
    }
    c->rings.push_back(m);
  }
  *out = c;
  return ST_OK;
}

}  // extern "C"

namespace {

// claim a free slot of ring r (never waits after the claim), fill it via `fill`, publish
template <typename F>
int client_push(mel_client* c, uint32_t r, uint32_t timeout_us, F&& fill) {
  Mapping& m = c->rings[r];
  RingHdr* h = m.hdr();
  Waiter w(timeout_us);
  uint64_t pos = h->enq.load(std::memory_order_relaxed);
  for (;;) {
    SlotHdr* s = m.slot(pos);
    const uint64_t seq = s->seq.load(std::memory_order_acquire);
    const int64_t dif = (int64_t)(seq - pos);
    if (dif == 0) {
      // reserve the slot with our pid first (a free slot has pid 0; a reservation left by a
      // process that died before taking the ticket is taken over), then take the ticket:
      // a claimed ticket therefore always names its claimant, so the server can tell a
      // claimant that died before publishing (mel_ingest_next skips its ticket)
      const int32_t me = (int32_t)getpid();
      int32_t cur = s->pid.load(std::memory_order_relaxed);
      if (cur != 0 && cur != me &&
          (!process_gone(cur) || h->enq.load(std::memory_order_acquire) != pos)) {
        // a live client's reservation, or a ticket a dead client took (the server skips it)
        pos = h->enq.load(std::memory_order_relaxed);
        continue;
      }
      if (!s->pid.compare_exchange_strong(cur, me, std::memory_order_acq_rel, std::memory_order_relaxed)) {
        pos = h->enq.load(std::memory_order_relaxed);
        continue;
      }
      if (c->die_after_pid) _exit(4);                     // a crash between reservation and ticket
      uint64_t expect = pos;
      if (h->enq.compare_exchange_strong(expect, pos + 1, std::memory_order_acq_rel, std::memory_order_relaxed)) {
        if (c->die_after_claim) _exit(3);                 // a client crash between claim and publish
        fill(s, m.field(s));
        s->seq.store(pos + 1, std::memory_order_release);
        return ST_OK;
      }
      int32_t mine = me;                                  // lost the ticket: drop the reservation
      s->pid.compare_exchange_strong(mine, 0, std::memory_order_acq_rel, std::memory_order_relaxed);
      pos = expect;
    } else if (dif < 0) {                                 // ring full: the slot is a lap behind
      if (!w.again()) return ST_EAGAIN;
      pos = h->enq.load(std::memory_order_relaxed);
    } else {
      pos = h->enq.load(std::memory_order_relaxed);
    }
  }
}

}  // namespace

extern "C" {

int mel_client_send(mel_client* c, uint32_t t, const float X[5], const double* field, uint32_t timeout_us) {
  if (!c || !X || !field) return ST_EINVAL;
  if (c->finalized) return ST_EPROTO;
  const uint32_t n = c->n_field, id = c->id;
  return client_push(c, mel_route(id, t, c->world), timeout_us, [&](SlotHdr* s, float* dst) {
    s->kind = KIND_DATA; s->sim = id; s->t = t;
    for (int i = 0; i < 5; ++i) s->X[i] = X[i];
    for (uint32_t i = 0; i < n; ++i) dst[i] = (float)field[i];   // fp64 -> fp32, RNE
  });
}

int mel_client_finalize(mel_client* c, uint32_t timeout_us) {
  if (!c) return ST_EINVAL;
  if (c->finalized) return ST_EPROTO;
  const uint32_t id = c->id;
  for (uint32_t r = 0; r < c->world; ++r) {
    int st = client_push(c, r, timeout_us, [&](SlotHdr* s, float*) {
      s->kind = KIND_FIN; s->sim = id; s->t = 0;
      for (int i = 0; i < 5; ++i) s->X[i] = 0.f;
    });
    if (st) return st;
  }
  c->finalized = true;
  return ST_OK;
}

void mel_client_close(mel_client* c) {
  if (!c) return;
  for (auto& m : c->rings)
    if (m.base) munmap(m.base, m.bytes);
  delete c;
}

}  // extern "C"
