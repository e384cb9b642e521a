/* bcl.h — C-ABI of the B200-native pipelined-chain broadcast (libbcl.so).
 *
 * The reference (bcastlab, /root/reference/proj) exposes a C++ API; this is
 * the flat boundary a host in any language binds (see INTEGRATION.md for the
 * ctypes / cgo / JNI stubs). Plain pointers and sizes only. Every entry point
 * returns a bcl_status_t; on failure bcl_last_error() holds the message
 * (thread-local). Status codes map 1:1 onto the reference's exception classes
 * (proj/src/ sources; the CLI maps them to exit codes in
 * proj/tools/bcastlab.cpp:544-557):
 *   BCL_ERR_INVALID_ARGUMENT  std::invalid_argument (contract errors)
 *   BCL_ERR_RUNTIME           std::runtime_error (I/O, data errors)
 *   BCL_ERR_OUT_OF_RANGE      std::out_of_range (select, tuner.cpp:180-189)
 *   BCL_ERR_TABLE_PARSE       TableParseError (tuner.hpp:76-83), line in
 *                             bcl_last_error_line()
 *   BCL_ERR_CUDA              CUDA runtime failure (new: device path)
 *   BCL_ERR_TIMEOUT           a device wait exceeded the group timeout
 *   BCL_ERR_RANKS             AggregateRankError (runtime.hpp:51-63)
 */
#ifndef BCL_H
#define BCL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BCL_OK = 0,
  BCL_ERR_INVALID_ARGUMENT = 1,
  BCL_ERR_RUNTIME = 2,
  BCL_ERR_OUT_OF_RANGE = 3,
  BCL_ERR_TABLE_PARSE = 4,
  BCL_ERR_SYSTEM = 5,
  BCL_ERR_CUDA = 6,
  BCL_ERR_TIMEOUT = 7,
  BCL_ERR_RANKS = 8,
} bcl_status_t;

/* Algorithm ids in the reference enum order, which is also the tuner's
 * tie-break order (proj/include/bcastlab/core.hpp:27-34). */
typedef enum {
  BCL_DIRECT = 0,
  BCL_CHAIN = 1,
  BCL_KNOMIAL = 2,
  BCL_SCATTER_RING_ALLGATHER = 3,
  BCL_CHAIN_PIPELINED = 4,
  BCL_KNOMIAL_STAGED = 5,
} bcl_algorithm_t;

/* MPI_Datatype stand-in for bcl_bcast; the payload is moved bit-exactly. */
typedef enum {
  BCL_INT8 = 0, BCL_UINT8, BCL_INT32, BCL_UINT32, BCL_INT64, BCL_UINT64,
  BCL_FLOAT16, BCL_FLOAT32, BCL_FLOAT64, BCL_BFLOAT16,
} bcl_dtype_t;

/* AlgorithmConfig (core.hpp:45-53); unused parameters are 0. */
typedef struct {
  int32_t algorithm;
  int32_t radix_k;
  uint64_t chunk_bytes;
} bcl_config_t;

/* ChunkSpec (core.hpp:56-62). */
typedef struct {
  uint32_t chunk_id;
  uint64_t offset_bytes;
  uint64_t length_bytes;
} bcl_chunk_t;

/* Event (core.hpp:71-87); kind 0 = send, 1 = recv. */
typedef struct {
  int32_t kind;
  int32_t peer;
  uint32_t chunk;
  uint32_t group;
} bcl_event_t;

/* TuningEntry (tuner.hpp:21-29). */
typedef struct {
  int32_t n;
  uint64_t msg_min_bytes;
  uint64_t msg_max_bytes;
  bcl_config_t config;
  double predicted_cost_s;
} bcl_table_entry_t;

typedef struct bcl_schedule_s* bcl_schedule_t;
typedef struct bcl_table_s* bcl_table_t;
typedef struct bcl_comm_s* bcl_comm_t;

/* ---------------------------------------------------------------- errors */
const char* bcl_last_error(void);
size_t bcl_last_error_line(void);
const char* bcl_version(void);

/* ------------------------------------------- chunking and schedules (L1/L2) */
/* make_chunks (core.hpp:119-124): writes up to cap chunks, *count = total. */
bcl_status_t bcl_make_chunks(uint64_t message_bytes, uint64_t chunk_bytes,
                             bcl_chunk_t* out, size_t cap, size_t* count);
/* make_schedule (schedules.hpp:34-35). */
bcl_status_t bcl_schedule_create(const bcl_config_t* config, int n, int root,
                                 uint64_t message_bytes, bcl_schedule_t* out);
bcl_status_t bcl_schedule_destroy(bcl_schedule_t s);
/* prologue: 0 none, 1 self-send, 2 host staging (core.hpp:90-97). */
bcl_status_t bcl_schedule_info(bcl_schedule_t s, int* n, int* root,
                               uint64_t* message_bytes, int* prologue,
                               size_t* n_chunks);
bcl_status_t bcl_schedule_chunks(bcl_schedule_t s, bcl_chunk_t* out, size_t cap);
bcl_status_t bcl_schedule_rank_events(bcl_schedule_t s, int rank,
                                      bcl_event_t* out, size_t cap,
                                      size_t* count);
/* validate_schedule (core.hpp:133): BCL_OK when valid, else
 * BCL_ERR_INVALID_ARGUMENT with the violation in bcl_last_error(). */
bcl_status_t bcl_schedule_validate(bcl_schedule_t s);
/* to_text (core.hpp:136): *len = bytes needed incl. NUL. */
bcl_status_t bcl_schedule_text(bcl_schedule_t s, char* out, size_t cap, size_t* len);

/* ----------------------------------------------------------- tuner (L4) */
/* Closed-form cost (models.hpp:56-57) at NetworkParams {t_s, B, B_staging}. */
bcl_status_t bcl_model_cost(const bcl_config_t* config, int n, uint64_t message_bytes,
                            double startup_s, double link_Bps, double staging_Bps,
                            double* total_s);
/* Analytical tune (tuner.hpp:64-68); candidates' chunk_bytes are ignored
 * (chunk_pipelined fans out over chunks[]). */
bcl_status_t bcl_tune_analytical(const int* n_list, size_t n_count,
                                 const uint64_t* sizes, size_t n_sizes,
                                 const bcl_config_t* candidates, size_t n_cands,
                                 const uint64_t* chunks, size_t n_chunks,
                                 double startup_s, double link_Bps, double staging_Bps,
                                 bcl_table_t* out);
/* NetworkParams (core.hpp:16-25) plus, new on B200, a per-call constant a0
 * added to every algorithm's cost (Eq. 5 + a0 fits B200 measurements within
 * 1-3%; call_overhead_s = 0 is the reference model, bit-identical). */
typedef struct {
  double startup_s;
  double link_Bps;
  double staging_Bps;
  double call_overhead_s;
} bcl_network_params_t;
bcl_status_t bcl_model_cost_ex(const bcl_config_t* config, int n, uint64_t message_bytes,
                               const bcl_network_params_t* params, double* total_s);
bcl_status_t bcl_tune_analytical_ex(const int* n_list, size_t n_count, const uint64_t* sizes, size_t n_sizes,
                                    const bcl_config_t* candidates, size_t n_cands, const uint64_t* chunks,
                                    size_t n_chunks, const bcl_network_params_t* params, bcl_table_t* out);
/* Measured tune: cost(config, n, bytes, user) returns seconds (e.g. the
 * median device latency); NaN aborts with BCL_ERR_RUNTIME. */
typedef double (*bcl_cost_fn)(const bcl_config_t* config, int n, uint64_t bytes, void* user);
bcl_status_t bcl_tune_measured(const int* n_list, size_t n_count,
                               const uint64_t* sizes, size_t n_sizes,
                               const bcl_config_t* candidates, size_t n_cands,
                               const uint64_t* chunks, size_t n_chunks,
                               bcl_cost_fn cost, void* user, const char* provenance,
                               bcl_table_t* out);
/* load_table / save_table (tuner.hpp:88-91); *_text variants work on memory. */
bcl_status_t bcl_table_load(const char* path, bcl_table_t* out);
bcl_status_t bcl_table_load_text(const char* text, bcl_table_t* out);
bcl_status_t bcl_table_save(bcl_table_t t, const char* path);
bcl_status_t bcl_table_save_text(bcl_table_t t, char* out, size_t cap, size_t* len);
bcl_status_t bcl_table_builtin(bcl_table_t* out);
bcl_status_t bcl_table_destroy(bcl_table_t t);
/* oracle: 0 analytical, 1 simulated, 2 measured. */
bcl_status_t bcl_table_info(bcl_table_t t, int* oracle, size_t* n_entries);
bcl_status_t bcl_table_entries(bcl_table_t t, bcl_table_entry_t* out, size_t cap);
/* select (tuner.hpp:73-74). */
bcl_status_t bcl_table_select(bcl_table_t t, int n, uint64_t message_bytes,
                              bcl_config_t* out);

/* ------------------------------------- communicator (TransportFabric, L0/L3) */
/* One process drives n ranks; rank r runs on devices[r]. Several ranks may
 * share a GPU (they then run in one launch). out[r] is rank r's handle.
 * timeout_s <= 0 picks the default (20 s). */
bcl_status_t bcl_comm_init_all(int n, const int* devices, double timeout_s,
                               bcl_comm_t* out);
/* One process per GPU: create, exchange bcl_comm_export() blobs by any
 * out-of-band means (e.g. torch.distributed all_gather), then connect with
 * the n blobs ordered by rank. heap_bytes sizes the symmetric heap from which
 * bcl_mem_alloc serves broadcast buffers (peers map it via CUDA IPC). */
bcl_status_t bcl_comm_init_rank(int n, int rank, int device, size_t heap_bytes,
                                double timeout_s, bcl_comm_t* out);
/* The same with communicator options, "key=value" pairs separated by ','
 * (the BCL_* environment variables in lower case without the prefix, which
 * they override), e.g. "timeout_s=10,stage_bytes=8192,sys_scope=1":
 *   timeout_s      device wait bound (s)
 *   protocol       chain transport, as bcl_comm_set_protocol
 *   stage_bytes    TMA bulk-copy stage per copy warp (0 = 16-byte vector loads;
 *                  default 8192 across GPUs, 0 when every rank shares one GPU)
 *   sys_scope      1: system-scope flag polls and fences even when every rank
 *                  shares one GPU (the cross-GPU code path on one device)
 *   strict_sys     1 (default): system-scope fence in the publisher before
 *                  every flag batch (the PTX-model release); 0: the copy warps'
 *                  gpu-scope writer fence instead (faster for pull at n >= 3)
 *   writer_fence   with strict_sys=0: 0 publisher fences, 1 gpu scope, 2 the
 *                  call's scope
 *   ll128          -1 auto (ranks on distinct GPUs), 0 off, 1 also between
 *                  ranks sharing a GPU;  ll128_max, ll_chain_max, ll_max caps
 *   ll128_direct_min  `direct` calls from this size up to ll_max travel as
 *                  128-byte LL128 lines (every rank on its own GPU; 0 off,
 *                  without their landing areas either; default 131072; a
 *                  group's `direct` run holding such a call travels on
 *                  fused LL128 lines)
 *   nvls           NVLS multicast team: -1 auto (ranks on two or more GPUs with
 *                  multicast support), 0 off, 1 required (init fails without);
 *                  nvls_strict 1: system-scope fence before every counter bump
 *   window_bytes, min_slice, max_ctas, stages, poll_ns, host_piece, ll,
 *   eager_post, local_fused, local_ctas, local_item  (tuning knobs)
 * Unknown keys fail with BCL_ERR_INVALID_ARGUMENT. New on B200. */
bcl_status_t bcl_comm_init_all_opts(int n, const int* devices, const char* options, bcl_comm_t* out);
bcl_status_t bcl_comm_init_rank_opts(int n, int rank, int device, size_t heap_bytes, const char* options,
                                     bcl_comm_t* out);
bcl_status_t bcl_comm_export(bcl_comm_t c, void* blob, size_t cap, size_t* len);
bcl_status_t bcl_comm_connect(bcl_comm_t c, const void* blobs, size_t blob_len);
/* Buffer registration (one process per GPU; collective: every rank, same
 * order, NCCL-style). The device allocation (cudaMalloc / caching allocator
 * segment) holding [ptr, ptr + bytes) is exported with CUDA IPC: pass every
 * rank's blob, ordered by rank, to bcl_comm_register_connect. Afterwards
 * bcl_bcast works zero-copy on any buffer inside the registered allocations,
 * not only on bcl_mem_alloc buffers (the line protocols need neither). blob
 * == NULL only returns the blob size in *len. Up to
 * 255 registrations per communicator. One-process groups (bcl_comm_init_all)
 * need none: export returns *len = 0 and connect does nothing. */
bcl_status_t bcl_comm_register_export(bcl_comm_t c, void* ptr, size_t bytes, void* blob, size_t cap, size_t* len);
bcl_status_t bcl_comm_register_connect(bcl_comm_t c, const void* blobs, size_t blob_len);
bcl_status_t bcl_comm_destroy(bcl_comm_t c);
bcl_status_t bcl_comm_info(bcl_comm_t c, int* n, int* rank, int* device, int* lanes);
/* Largest message each line protocol takes on this communicator (bytes; 0 =
 * unavailable): LL for `direct`, LL and LL128 for the pipelined chain (LL128
 * needs every rank on its own GPU). New on B200; no reference counterpart. */
bcl_status_t bcl_comm_protocol_caps(bcl_comm_t c, uint64_t* ll_direct_max, uint64_t* ll_chain_max,
                                    uint64_t* ll128_max);
/* Tuning table consulted when a call passes config == NULL; the builtin
 * measured B200 table is used until one is set. The table is copied. */
bcl_status_t bcl_comm_set_table(bcl_comm_t c, bcl_table_t t);
/* The device lane plan of a call (identical on every rank): Q slices per
 * chunk, slice bytes, chunk count, CTAs per rank. Lane l serves slice l % Q of
 * chunks c with c % (lanes / Q) == l / Q. */
bcl_status_t bcl_comm_plan(bcl_comm_t c, const bcl_config_t* config, int root, uint64_t bytes, int* slices,
                           uint64_t* slice_bytes, uint32_t* n_chunks, int* ctas);
/* The device path a call of this shape would run (config NULL = tuned), as
 * text: "ll_kernel/direct", "ll128_kernel/direct", "ll_kernel/chain", "ll128_kernel",
 * "local_chain_kernel", "bcast_kernel/pull[/tma]", "bcast_kernel/push[/tma]",
 * "bcast_kernel/events", "nvls_kernel", "nvls_ll_kernel" or "none"; *len = bytes needed incl. NUL. */
bcl_status_t bcl_comm_path(bcl_comm_t c, const bcl_config_t* config, int root, uint64_t bytes, char* out,
                           size_t cap, size_t* len);
/* Pipelined-chain transport protocol: 0 auto (line protocols where the
 * tuning table's rules pick them -- LL128 when every rank has its own GPU, up
 * to the table's measured "# bcl-ll128-upto" rule (and the ll128_max option,
 * no limit by default: LL128 lines land in a bounded per-rank ring of 58 MB
 * with per-warp credits), else 16-byte LL lines up to ll_chain_max (default
 * 8 MiB) -- and above them the table's measured "# bcl-push-from" rule),
 * 1 pull (consumers load from the upstream buffer), 2 push (producers store
 * into the downstream buffer), 3 LL (flagged 16-byte lines forwarded hop by
 * hop), 4 LL128 (128-byte lines, 120 payload bytes each), 5 NVLS (the root
 * writes each piece once through a multicast address, the NVSwitch
 * replicates it to every GPU, receivers copy it out; any schedule -- in auto
 * mode NVLS carries the `direct` schedule above the LL threshold). 3 fails
 * above ll_chain_max, 4 above ll128_max or when ranks share a GPU without the
 * ll128=1 option, 5 when the communicator has no multicast team. */
bcl_status_t bcl_comm_set_protocol(bcl_comm_t c, int protocol);
/* Group fusion (NCCL-style ncclGroupStart/End; per calling thread, nestable).
 * bcl_bcast / bcl_bcast_all calls issued between start and end are deferred;
 * at the outermost end, runs of consecutive calls on one communicator that take
 * a line protocol (LL `direct`, LL or LL128 chain) with the same root and
 * stream are fused into one kernel launch carrying up to 32 messages (8 when
 * ranks share a GPU) on the run's most capable protocol (LL128 chain > LL
 * chain > LL direct), everything else launches as usual, in call order.
 * Every rank must issue the same calls between the same start/end (MPI
 * semantics), switching streams at the same calls (a stream change ends a
 * run); host-buffer and synchronous run_bcast calls cannot be grouped
 * (BCL_ERR_INVALID_ARGUMENT). The paper's caller broadcasts every layer of a
 * model (configs 4/5): grouped, ResNet-50's 161 per-tensor broadcasts run in
 * ~10 launches. New on B200; no reference counterpart. */
bcl_status_t bcl_group_start(void);
bcl_status_t bcl_group_end(void);
/* NVLS multicast team of this communicator: *available 1/0 and, when 0, why
 * (text, *len = bytes needed incl. NUL). Every rank agrees at init/connect.
 * New on B200; no reference counterpart. */
bcl_status_t bcl_comm_nvls(bcl_comm_t c, int* available, char* reason, size_t cap, size_t* len);
/* The config a NULL-config call would run for this size (select + clamp). */
bcl_status_t bcl_comm_choose(bcl_comm_t c, uint64_t message_bytes, bcl_config_t* out);
bcl_status_t bcl_mem_alloc(bcl_comm_t c, size_t bytes, void** ptr);
bcl_status_t bcl_mem_reset(bcl_comm_t c);

/* ------------------------------------------------------------ data plane */
/* MPI_Bcast-shaped per-rank call (north_star's bcast(buf, count, dtype,
 * root, comm)); semantics = execute_rank(make_schedule(select(table, n,
 * count*size(dtype)), n, root, M), rank, buf, fabric) (runtime.hpp:134-138).
 * In place on a device buffer, enqueued on `stream` (cudaStream_t, NULL =
 * legacy default stream); config NULL = tuned. Asynchronous: device errors
 * surface from bcl_comm_check(). Capturable into a CUDA graph (call epochs
 * live on the device; issue the call once before capturing so lazy
 * allocations are done); calls on one communicator must be stream-ordered. */
bcl_status_t bcl_bcast(void* buf, size_t count, bcl_dtype_t dtype, int root,
                       bcl_comm_t comm, const bcl_config_t* config, void* stream);
/* Same with a HOST buffer: H2D at the root, device broadcast, D2H elsewhere. */
bcl_status_t bcl_bcast_host(void* host_buf, size_t count, bcl_dtype_t dtype, int root,
                            bcl_comm_t comm, const bcl_config_t* config, void* stream);
/* All ranks of an init_all group in one call (bufs[r], streams[r] or NULL). */
bcl_status_t bcl_bcast_all(void* const* bufs, size_t count, bcl_dtype_t dtype, int root,
                           const bcl_comm_t* comms, int n, const bcl_config_t* config,
                           void* const* streams);
/* run_bcast (runtime.hpp:140-143): synchronous, all ranks, wall seconds. */
bcl_status_t bcl_run_bcast(int n, int root, void* const* device_bufs, uint64_t bytes,
                           const bcl_config_t* config, const bcl_comm_t* comms,
                           double* wall_s);
/* run_bcast over host spans, as the reference's (host-resident) buffers. */
bcl_status_t bcl_run_bcast_host(int n, int root, void* const* host_bufs, uint64_t bytes,
                                const bcl_config_t* config, const bcl_comm_t* comms,
                                double* wall_s);
/* Device-side barrier across the communicator (synchronised start). */
bcl_status_t bcl_barrier(bcl_comm_t comm, void* stream);
bcl_status_t bcl_barrier_all(const bcl_comm_t* comms, int n, void* const* streams);
/* Synchronize `stream` (NULL: the device) and report device-side failures. */
bcl_status_t bcl_comm_check(bcl_comm_t comm, void* stream);
/* Test hook: per-[src][chunk] byte counters (device memory, zeroed by the
 * caller) recording every pull this rank performs; NULL disables. */
bcl_status_t bcl_comm_set_provenance(bcl_comm_t comm, unsigned long long* counters);
/* Timeline hook: per lane, up to per_lane records of 4 %globaltimer stamps
 * (ns) {wait begin, data ready, copy done, published} for each pull, at
 * records[(lane * per_lane + i) * 4]; record i = the lane's i-th pull.
 * Device memory, zeroed by the caller; NULL disables. */
bcl_status_t bcl_comm_set_trace(bcl_comm_t comm, unsigned long long* records, uint32_t per_lane);
bcl_status_t bcl_comm_launches(bcl_comm_t comm, uint64_t* launches);

/* ------------------------------- device fabric (Transport / TransportFabric) */
/* A GPU-backed stand-in for the reference's message fabric
 * (proj/include/bcastlab/runtime.hpp:20-39): n ranks (threads of one
 * process), rank r on devices[r]. Same contract as the reference transports:
 * ordered and reliable per (src, dst) pair, eager send, blocking receive that
 * rejects an out-of-order chunk id (BCL_ERR_RUNTIME). The payload moves
 * through the GPUs: send stages it in the sender's GPU, receive pulls it into
 * the receiver's GPU with the library's copy kernel (NVLink P2P) and returns
 * it to the host. include/bcl_transport.hpp adapts it to the reference's
 * Transport / TransportFabric classes so execute_rank and run_bcast run on it.
 * Each endpoint (src for send, dst for receive) is used by one thread. */
typedef struct bcl_fabric_s* bcl_fabric_t;
bcl_status_t bcl_fabric_create(int n, const int* devices, bcl_fabric_t* out);
bcl_status_t bcl_fabric_destroy(bcl_fabric_t f);
bcl_status_t bcl_fabric_n_ranks(bcl_fabric_t f, int* n);
bcl_status_t bcl_fabric_send(bcl_fabric_t f, int src, int dst, uint32_t chunk, const void* data, size_t len);
/* Blocks for the next message src -> dst, checks its chunk id, returns its
 * length; bcl_fabric_recv then copies it into out (exactly len bytes). */
bcl_status_t bcl_fabric_recv_size(bcl_fabric_t f, int dst, int src, uint32_t chunk, size_t* len);
bcl_status_t bcl_fabric_recv(bcl_fabric_t f, int dst, int src, uint32_t chunk, void* out, size_t len);
/* Messages and payload bytes delivered src -> dst so far (schedule fidelity). */
bcl_status_t bcl_fabric_stats(bcl_fabric_t f, int src, int dst, uint64_t* messages, uint64_t* bytes);

#ifdef __cplusplus
}
#endif
#endif /* BCL_H */
