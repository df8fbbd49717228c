/*
 * mel_dataset.h -- C ABI of the offline baseline's data path:
 * a file dataset of simulation time steps and a multi-threaded, epoch-shuffled reader.
 * Host-only code (no CUDA), built into libmel.so; surrogate_train_offline in mel.h
 * drives the trainer from it.
 *
 * What the paper fixes (§4.4 "Online versus multi-epoch Offline", P:425-469,
 * Table 2): the offline baseline trains on the same trainer from data written to disk
 * beforehand (one binary file per simulation there), over many epochs (100 on 250
 * simulations), read by several loader workers per GPU ("offline only manage to process
 * about 38 samples/sec, even when using 8 data loaders per GPU").  Epoch-wise shuffling
 * is the reading R24.
 *
 * File layout (little-endian): a 4096-byte header {magic "MELDSET1", version, n_field,
 * count, field_stride, index_off, data_off}; record i's fp32 kelvin field (n_field
 * values) at data_off + i * field_stride (data_off = 4096, field_stride = 4*n_field
 * rounded up to 4096: page-aligned records); after the last record, at index_off, the
 * `count` index entries of 32 bytes {u32 sim_id, u32 t, f32 X[5], u32 pad}.
 *
 * Epoch order (reading R24): a Fisher-Yates shuffle driven by the library's
 * Philox stream (reading Q8): for i = count-1 down to 1, j = bounded(r64(seed, TAG_EPOCH=5,
 * ctr = i, c2 = epoch), i + 1), swap(perm[i], perm[j]), starting from the identity.
 * Batches are consecutive runs of B entries of perm; the last partial batch is dropped.
 *
 * Conventions: int status (MEL_OK 0, MEL_EINVAL -1, MEL_EPROTO -3 not a dataset /
 * writer misuse, MEL_ENOMEM -6 open / write / read failure).  *_host pointers are read
 * or written during the call only.  One thread per handle (the reader's worker threads
 * are internal).
 */
#ifndef MEL_DATASET_H_
#define MEL_DATASET_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MEL_DATASET_VERSION 1u

#ifndef MEL_DATASET_TYPEDEF_
#define MEL_DATASET_TYPEDEF_
typedef struct mel_dataset mel_dataset;
#endif
typedef struct mel_dataset_writer mel_dataset_writer;

/* Creates (truncates) `path` for records of n_field fp32 values. */
int mel_dataset_create(const char* path, uint32_t n_field, mel_dataset_writer** out);
/* Appends one time step (sim_id, t, X[5] kelvin, field fp32 kelvin). */
int mel_dataset_append(mel_dataset_writer* w, uint32_t sim_id, uint32_t t, const float X_host[5],
                       const float* field_host);
/* Writes the index and header and closes the file (the writer is freed either way). */
int mel_dataset_finish(mel_dataset_writer* w);

/* Opens a dataset for reading; `threads` loader workers (>= 1) serve mel_dataset_read. */
int mel_dataset_open(const char* path, uint32_t threads, mel_dataset** out);
uint64_t mel_dataset_count(const mel_dataset* d);
uint32_t mel_dataset_n_field(const mel_dataset* d);
/* perm_host[0..count) = the epoch's order (reading R24). */
int mel_dataset_epoch_order(uint64_t count, uint64_t seed, uint32_t epoch, uint32_t* perm_host);
/* Reads records idx[0..n): metadata into sim/t/X (any may be NULL) and fields into
 * fields_host + k * ld (ld >= n_field floats; NULL skips the fields), the n reads
 * spread over the loader threads (positional reads of page-aligned records). */
int mel_dataset_read(mel_dataset* d, const uint32_t* idx_host, uint32_t n, uint32_t* sim_host,
                     uint32_t* t_host, float* X_host, float* fields_host, uint64_t ld);
void mel_dataset_close(mel_dataset* d);

#ifdef __cplusplus
}
#endif
#endif
