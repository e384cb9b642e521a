/* TEST INFRASTRUCTURE — the CPU oracle. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this library, and only as the
 * checker; the product (paper_1707_09414_b200/) never links or calls it.
 *
 * A plain-C restatement of the reference (bcastlab, /root/reference/proj) for
 * the broadcast hot path: chunking, the schedule generators with root
 * rotation, a sequential executor of the per-rank copy/forward loop over
 * per-pair FIFOs, the closed-form costs the tuner uses, tune/select and the
 * tuning-table CSV format. Every function cites the reference file:line it
 * restates. Parity is pinned against the reference itself: the golden
 * fixtures in tests/golden/ are produced by oracle/_ref/ref_harness (the
 * unmodified reference sources compiled by oracle/Makefile).
 */
#ifndef BCAST_ORACLE_H
#define BCAST_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_DIRECT = 0, ORC_CHAIN, ORC_KNOMIAL, ORC_SRA, ORC_CHAIN_PIPELINED,
       ORC_KNOMIAL_STAGED, ORC_ALGO_COUNT };
enum { ORC_SEND = 0, ORC_RECV = 1 };

typedef struct { uint32_t chunk_id; uint64_t offset; uint64_t length; } orc_chunk;
typedef struct { int32_t kind; int32_t peer; uint32_t chunk; uint32_t group; } orc_event;

typedef struct {
  int n, root;
  uint64_t message_bytes;
  int prologue;            /* 0 none, 1 self-send, 2 host staging */
  uint32_t n_chunks;
  orc_chunk* chunks;
  uint64_t* ev_off;        /* n + 1 offsets into events */
  orc_event* events;
} orc_schedule;

/* 0 on success, negative on a contract error (the reference throws
 * std::invalid_argument in every such case). */
int64_t orc_make_chunks(uint64_t message_bytes, uint64_t chunk_bytes,
                        orc_chunk* out, uint64_t cap);
int orc_make_schedule(int algo, int radix, uint64_t chunk_bytes, int n,
                      int root, uint64_t message_bytes, orc_schedule* out);
void orc_free_schedule(orc_schedule* s);
/* Runs every rank's event list against per-pair FIFO queues until all lists
 * are drained; buffers[r] has message_bytes bytes. 0 ok, <0 error. */
int orc_execute(const orc_schedule* s, uint8_t* const* buffers);
/* Convenience: schedule + execute. */
int orc_bcast(int algo, int radix, uint64_t chunk_bytes, int n, int root,
              uint64_t message_bytes, uint8_t* const* buffers);
/* bcastlab payload_for formula (mt19937_64 of seed*golden+size+1). */
void orc_payload(uint64_t seed, uint64_t size, uint8_t* out);
uint64_t orc_fnv1a(const uint8_t* p, uint64_t n);

/* Tuner. */
typedef struct { int32_t algorithm; int32_t radix_k; uint64_t chunk_bytes; } orc_config;
typedef struct { int32_t n; uint64_t msg_min, msg_max; orc_config config; double cost; } orc_entry;
double orc_cost(const orc_config* c, int n, uint64_t m, double startup,
                double bandwidth, double staging);
/* Returns entry count or negative on error; entries must hold
 * n_count * n_sizes. */
int64_t orc_tune(const int* n_list, int n_count, const uint64_t* sizes,
                 int n_sizes, const orc_config* cands, int n_cands,
                 const uint64_t* chunks, int n_chunks, double startup,
                 double bandwidth, double staging, orc_entry* out);
/* 0 ok, -1 empty table, -2 no tuned n <= n. */
int orc_select(const orc_entry* e, int64_t count, int n, uint64_t m,
               orc_config* out);
/* Writes the reference CSV text; returns bytes written (excl. NUL) or the
 * size needed when cap is too small. */
int64_t orc_save_table(const orc_entry* e, int64_t count, int oracle,
                       char* out, int64_t cap);
/* Parses reference CSV text. Returns entry count, or -(line number) on a
 * parse error (line 0 reported as -1000000). */
int64_t orc_load_table(const char* text, orc_entry* out, int64_t cap,
                       int* oracle_out);
/* std::to_chars(double) shortest form. */
int orc_format_double(double v, char* out, int cap);

#ifdef __cplusplus
}
#endif
#endif
