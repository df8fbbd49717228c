/*
 * mel_ingest.h -- C ABI of the ingest channel: the step before the training buffer
 * (SURVEY §8(f) row f2).  Host-only code (no CUDA), in libmel_ingest.so for the
 * simulation clients and inside libmel.so for the server side.
 *
 * What the paper fixes (PAPER.md line numbers, §3 "Framework architecture" and
 * §3.2.2 "Data distribution"):
 *   - clients are separate processes; "A first call is required to connect the client to
 *     the server (init_communication). A send is issued to transfer time steps u_X^t as
 *     soon as computed. Eventually, a client calls finialize_communication";
 *   - "they are gathered and then converted, typically from 64 to 32 bits" -- on the
 *     client, so the server is not loaded with the conversion;
 *   - "each client connects to all the ranks of the server and distributes the produced
 *     time steps u_X^t across all GPUs in a Round-Robin fashion. The destination of the
 *     first time step is chosen according to the client id";
 *   - "The server maintains a log of received messages per client, so in case of client
 *     restart, already received messages are discarded".
 *
 * B200-box design: one POSIX shared-memory ring per server rank
 * (/dev/shm/<name>.<rank>), a bounded multi-producer / single-consumer queue of
 * fixed-size slots [header | fp32 field], each slot cycling through the sequence
 * numbers ticket -> ticket+1 (published) -> ticket+S (free for the next lap).  Clients
 * claim a ticket with one atomic add, convert their fp64 field into the slot and
 * publish it with a release store; the server consumes tickets in order.  On the GPU
 * side (reservoir_ingest in mel.h) the segment is page-locked with cudaHostRegister and
 * each field is DMA-copied straight from the slot into the reservoir's staging ring.
 *
 * Reading R10: the round robin is a function of (client id, t) --
 * rank(c, t) = (c + t) mod R -- so a restarted client resends each time step to the
 * rank whose log already holds it, and the per-client log lives on that rank.
 * Reading R23: the log's key is (client id, t); a repeated key is discarded whatever
 * its payload; the messages a rank keeps are the first copies in arrival order.
 *
 * Conventions: every call returns an int status (MEL_OK = 0, MEL_EAGAIN = 1 "nothing
 * published yet / ring full", MEL_EOS = 2 "every client finalized and the ring is
 * drained", MEL_EINVAL = -1, MEL_EPROTO = -3 (a send after finalize, a segment of
 * another layout), MEL_ENOMEM = -6 (shm creation or mapping failed)).  Pointers
 * named *_host are read during the call only.  One thread per handle.
 */
#ifndef MEL_INGEST_H_
#define MEL_INGEST_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MEL_INGEST_VERSION 1u

#ifndef MEL_INGEST_TYPEDEF_
#define MEL_INGEST_TYPEDEF_
typedef struct mel_ingest mel_ingest;   /* server side: one rank's ring + per-client log */
#endif
typedef struct mel_client mel_client;   /* client side: connections to every rank's ring */

/* One published time step, as the server sees it.  `field` points into the shared
 * segment (fp32, n_field values, 256-byte aligned) and stays valid until the message
 * is released; messages are released in the order they were returned. */
typedef struct mel_ingest_msg {
  uint32_t sim_id;      /* the client id (one client per simulation)          */
  uint32_t t;           /* time step index                                            */
  float X[5];           /* the simulation's parameters (kelvin)                       */
  uint32_t pad;
  const float* field;   /* fp32 kelvin, converted by the client               */
  uint64_t ticket;      /* arrival order on this rank                                 */
} mel_ingest_msg;

typedef struct mel_ingest_stats {
  uint64_t received;      /* messages returned to the consumer (first copies)          */
  uint64_t duplicates;    /* messages discarded by the per-client log          */
  uint64_t abandoned;     /* tickets skipped because their client died before publishing */
  uint64_t finalized;     /* finalize markers seen                                     */
  uint64_t clients;       /* distinct clients seen                                     */
  uint64_t bytes;         /* fp32 payload bytes returned                               */
} mel_ingest_stats;

/* ---- server side ------------------------------------------------------------------ */

/* Creates (or re-creates: an old segment of that name is unlinked first) the ring of
 * `slots` messages of n_field fp32 values for server rank `rank`, shared-memory name
 * "/<name>.<rank>".  `expected_clients` = how many distinct clients must finalize before
 * mel_ingest_next returns MEL_EOS (0: never EOS).  Errors: MEL_EINVAL (slots < 2, n_field
 * 0, name too long), MEL_ENOMEM. */
int mel_ingest_create(const char* name, uint32_t rank, uint32_t n_field, uint32_t slots,
                      uint32_t expected_clients, mel_ingest** out);

/* Returns the next first-copy message in arrival order.  Duplicates ((sim_id, t)
 * already received on this rank) and finalize markers are consumed and released
 * internally, never returned.  Waits up to timeout_us for the next ticket to be
 * published; a ticket whose claiming process no longer exists is skipped (counted in
 * `abandoned`).  MEL_EAGAIN: nothing published in time.  MEL_EOS: expected_clients
 * finalized and every claimed ticket consumed. */
int mel_ingest_next(mel_ingest* ing, mel_ingest_msg* out_host, uint32_t timeout_us);

/* Releases the oldest returned, unreleased message (its slot becomes free for the
 * clients).  MEL_EPROTO if none is outstanding. */
int mel_ingest_release(mel_ingest* ing);

/* Number of returned, unreleased messages. */
uint32_t mel_ingest_outstanding(const mel_ingest* ing);

int mel_ingest_stats_get(const mel_ingest* ing, mel_ingest_stats* out_host);

/* The mapped segment (for page-locking by the GPU side) and its size in bytes. */
int mel_ingest_segment(const mel_ingest* ing, void** base, uint64_t* bytes);

/* Unmaps and unlinks the segment. */
void mel_ingest_destroy(mel_ingest* ing);

/* ---- client side ------------------------------------------------------------ */

/* init_communication: maps the rings "/<name>.0" ... "/<name>.<world-1>" (they must
 * exist).  MEL_EPROTO if a ring has another layout, MEL_ENOMEM if one is missing. */
int mel_client_open(const char* name, uint32_t world, uint32_t client_id, mel_client** out);

/* send: converts field_f64_host (n_field doubles, kelvin) to fp32 (round to nearest
 * even) into a slot of rank (client_id + t) mod world and publishes it.  Blocks while
 * that ring is full (up to timeout_us, then MEL_EAGAIN with nothing sent).
 * MEL_EPROTO after mel_client_finalize. */
int mel_client_send(mel_client* cl, uint32_t t, const float X_host[5], const double* field_f64_host,
                    uint32_t timeout_us);

/* finalize_communication: a finalize marker to every rank. */
int mel_client_finalize(mel_client* cl, uint32_t timeout_us);

/* Unmaps (without finalizing: a client that disappears is the restart case of P:183). */
void mel_client_close(mel_client* cl);

/* rank(c, t) of reading R10, exported so tests and the oracle can compare. */
uint32_t mel_route(uint32_t client_id, uint32_t t, uint32_t world);

#ifdef __cplusplus
}
#endif
#endif
