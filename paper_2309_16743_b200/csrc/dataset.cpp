// Offline baseline data path (include/mel_dataset.h): a file dataset of
// page-aligned fp32 records, its epoch order (Fisher-Yates on the Philox stream, reading
// R24) and a positional reader that spreads one batch over several loader threads.
#include "mel_dataset.h"

#include <atomic>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

namespace {

constexpr int ST_OK = 0, ST_EINVAL = -1, ST_EPROTO = -3, ST_ENOMEM = -6;
constexpr uint64_t MAGIC = 0x315445534c454d4dull;   // "MMELSET1" tag
constexpr uint64_t HDR = 4096, PAGE = 4096;
constexpr uint32_t TAG_EPOCH = 5;                   // Philox stream tag (reading R24)

struct Header {
  uint64_t magic;
  uint32_t version, n_field;
  uint64_t count, field_stride, index_off, data_off;
};

struct Entry {
  uint32_t sim, t;
  float X[5];
  uint32_t pad;
};
static_assert(sizeof(Entry) == 32, "index entry");

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

bool pwrite_all(int fd, const void* buf, uint64_t n, uint64_t off) {
  const uint8_t* p = static_cast<const uint8_t*>(buf);
  while (n) {
    const ssize_t w = pwrite(fd, p, n, (off_t)off);
    if (w <= 0) {
      if (w < 0 && errno == EINTR) continue;
      return false;
    }
    p += w; n -= (uint64_t)w; off += (uint64_t)w;
  }
  return true;
}

bool pread_all(int fd, void* buf, uint64_t n, uint64_t off) {
  uint8_t* p = static_cast<uint8_t*>(buf);
  while (n) {
    const ssize_t r = pread(fd, p, n, (off_t)off);
    if (r <= 0) {
      if (r < 0 && errno == EINTR) continue;
      return false;
    }
    p += r; n -= (uint64_t)r; off += (uint64_t)r;
  }
  return true;
}

// Philox4x32-10 (Salmon et al., SC'11), the stream layout of reading Q8:
// key = (lo32 seed, hi32 seed), counter = (lo32 n, hi32 n, c2, tag), r64 = (o1 << 32) | o0
uint64_t philox_r64(uint64_t seed, uint32_t tag, uint64_t n, uint32_t c2) {
  uint32_t c0 = (uint32_t)n, c1 = (uint32_t)(n >> 32), cc2 = c2, c3 = tag;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * cc2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1, n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; cc2 = n2; c3 = n3;
  }
  return ((uint64_t)c1 << 32) | c0;
}

// floor(r * n / 2^64) without rejection (the library-wide bounded draw)
uint64_t bounded(uint64_t r, uint64_t n) { return (uint64_t)(((unsigned __int128)r * n) >> 64); }

}  // namespace

struct mel_dataset_writer {
  int fd = -1;
  Header h{};
  std::vector<Entry> index;
  std::vector<uint8_t> pad;
  bool failed = false;
};

struct mel_dataset {
  int fd = -1;
  Header h{};
  std::vector<Entry> index;
  uint32_t threads = 1;
};

extern "C" {

int mel_dataset_create(const char* path, uint32_t n_field, mel_dataset_writer** out) {
  if (!path || !out || n_field == 0) return ST_EINVAL;
  *out = nullptr;
  mel_dataset_writer* w = new (std::nothrow) mel_dataset_writer;
  if (!w) return ST_ENOMEM;
  w->fd = open(path, O_RDWR | O_CREAT | O_TRUNC, 0644);
  if (w->fd < 0) { delete w; return ST_ENOMEM; }
  w->h.magic = MAGIC;
  w->h.version = MEL_DATASET_VERSION;
  w->h.n_field = n_field;
  w->h.field_stride = round_up(4ull * n_field, PAGE);
  w->h.data_off = HDR;
  w->pad.assign(w->h.field_stride - 4ull * n_field, 0);
  *out = w;
  return ST_OK;
}

int mel_dataset_append(mel_dataset_writer* w, uint32_t sim, uint32_t t, const float X[5], const float* field) {
  if (!w || !X || !field) return ST_EINVAL;
  if (w->failed) return ST_ENOMEM;
  const uint64_t off = w->h.data_off + w->h.count * w->h.field_stride;
  const uint64_t nb = 4ull * w->h.n_field;
  if (!pwrite_all(w->fd, field, nb, off) || (!w->pad.empty() && !pwrite_all(w->fd, w->pad.data(), w->pad.size(), off + nb))) {
    w->failed = true;
    return ST_ENOMEM;
  }
  Entry e{};
  e.sim = sim; e.t = t;
  for (int i = 0; i < 5; ++i) e.X[i] = X[i];
  w->index.push_back(e);
  w->h.count += 1;
  return ST_OK;
}

int mel_dataset_finish(mel_dataset_writer* w) {
  if (!w) return ST_EINVAL;
  int st = w->failed ? ST_ENOMEM : ST_OK;
  if (!st) {
    w->h.index_off = w->h.data_off + w->h.count * w->h.field_stride;
    std::vector<uint8_t> hdr(HDR, 0);
    memcpy(hdr.data(), &w->h, sizeof(Header));
    if (!pwrite_all(w->fd, w->index.data(), w->index.size() * sizeof(Entry), w->h.index_off) ||
        !pwrite_all(w->fd, hdr.data(), HDR, 0) || fsync(w->fd) != 0)
      st = ST_ENOMEM;
  }
  close(w->fd);
  delete w;
  return st;
}

int mel_dataset_open(const char* path, uint32_t threads, mel_dataset** out) {
  if (!path || !out || threads == 0) return ST_EINVAL;
  *out = nullptr;
  mel_dataset* d = new (std::nothrow) mel_dataset;
  if (!d) return ST_ENOMEM;
  d->fd = open(path, O_RDONLY);
  if (d->fd < 0) { delete d; return ST_ENOMEM; }
  d->threads = threads;
  if (!pread_all(d->fd, &d->h, sizeof(Header), 0) || d->h.magic != MAGIC || d->h.version != MEL_DATASET_VERSION ||
      d->h.field_stride < 4ull * d->h.n_field) {
    close(d->fd);
    delete d;
    return ST_EPROTO;
  }
  d->index.resize(d->h.count);
  if (!pread_all(d->fd, d->index.data(), d->h.count * sizeof(Entry), d->h.index_off)) {
    close(d->fd);
    delete d;
    return ST_EPROTO;
  }
  *out = d;
  return ST_OK;
}

uint64_t mel_dataset_count(const mel_dataset* d) { return d ? d->h.count : 0; }
uint32_t mel_dataset_n_field(const mel_dataset* d) { return d ? d->h.n_field : 0; }

int mel_dataset_epoch_order(uint64_t count, uint64_t seed, uint32_t epoch, uint32_t* perm) {
  if (!perm || count > 0xFFFFFFFFull) return ST_EINVAL;
  for (uint64_t i = 0; i < count; ++i) perm[i] = (uint32_t)i;
  for (uint64_t i = count; i-- > 1;) {
    const uint64_t j = bounded(philox_r64(seed, TAG_EPOCH, i, epoch), i + 1);
    const uint32_t tmp = perm[i]; perm[i] = perm[j]; perm[j] = tmp;
  }
  return ST_OK;
}

int mel_dataset_read(mel_dataset* d, const uint32_t* idx, uint32_t n, uint32_t* sim, uint32_t* t, float* X,
                     float* fields, uint64_t ld) {
  if (!d || (!idx && n)) return ST_EINVAL;
  if (fields && ld < d->h.n_field) return ST_EINVAL;
  for (uint32_t k = 0; k < n; ++k) {
    if (idx[k] >= d->h.count) return ST_EINVAL;
    const Entry& e = d->index[idx[k]];
    if (sim) sim[k] = e.sim;
    if (t) t[k] = e.t;
    if (X) memcpy(X + 5ull * k, e.X, 5 * sizeof(float));
  }
  if (!fields || n == 0) return ST_OK;
  const uint32_t nt = d->threads < n ? d->threads : n;
  std::atomic<uint32_t> next{0};
  std::atomic<bool> ok{true};
  auto work = [&]() {
    for (uint32_t k; (k = next.fetch_add(1, std::memory_order_relaxed)) < n;)
      if (!pread_all(d->fd, fields + k * ld, 4ull * d->h.n_field, d->h.data_off + (uint64_t)idx[k] * d->h.field_stride))
        ok.store(false, std::memory_order_relaxed);
  };
  std::vector<std::thread> pool;
  for (uint32_t i = 1; i < nt; ++i) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  return ok.load() ? ST_OK : ST_ENOMEM;
}

void mel_dataset_close(mel_dataset* d) {
  if (!d) return;
  if (d->fd >= 0) close(d->fd);
  delete d;
}

}  // extern "C"
