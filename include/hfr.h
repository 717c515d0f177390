/* hfr.h — C ABI of the B200-native HFReduce library (libhfr.so).
 *
 * HFReduce is the hierarchical, asynchronous gradient allreduce of
 * Fire-Flyer AI-HPC (arXiv 2408.14158), PAPER.md:296-398 (§4).  On one
 * 8xB200 NVSwitch box the GPUs play the role of the paper's nodes and every
 * transfer is an SM load/store over NVLink on CUDA-IPC-mapped memory; the
 * reduction is an fp32 fold on the SMs.
 *
 * Conventions for every function below
 *   - Returns an hfr_status_t; never aborts the process.
 *   - Pointers named buf / ptr are DEVICE pointers on the comm's CUDA device;
 *     all other pointers are host pointers.
 *   - A `stream` is a cudaStream_t passed as an opaque pointer (no CUDA types
 *     in this header).  0 is the legacy default stream.
 *   - Thread-compatible: one comm per process per device; calls on one comm
 *     must not race.
 *   - Collective calls (marked COLLECTIVE) must be made by every rank of the
 *     comm, in the same order, with matching arguments.
 */
#ifndef HFR_H_
#define HFR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HFR_MAX_RANKS 16

typedef struct hfr_comm_s* hfr_comm_t;
typedef struct hfr_req_s* hfr_req_t;
typedef void* hfr_stream_t; /* cudaStream_t */

/* Element types.  bf16, fp16 and FP8 are reduced with fp32 accumulation and
 * ONE final RNE rounding (reading R2; PAPER.md:404 lists
 * FP32/FP16/BF16/FP8).  FP8 (reading R20): OCP E4M3 "FN" (no Inf, max 448)
 * and E5M2 (IEEE-like, max 57344), one byte per element; a result that rounds
 * past the largest finite value is NaN (E4M3) or +-Inf (E5M2), as
 * torch.Tensor.to(float8_*).  FP8 runs every schedule except NVLS
 * (UNSUPPORTED: the switch has no fp32-accumulating FP8 reduction). */
typedef enum {
    HFR_FLOAT32 = 0,
    HFR_BFLOAT16 = 1,
    HFR_FLOAT16 = 2,
    HFR_FP8_E4M3 = 3,
    HFR_FP8_E5M2 = 4
} hfr_dtype_t;

/* Reduction operator.  The paper's only operator is the sum ("reduction add
 * operation"). */
typedef enum { HFR_SUM = 0 } hfr_op_t;

typedef enum {
    HFR_SUCCESS = 0,
    HFR_ERR_INVALID_ARGUMENT = 1, /* NULL buf with count > 0, bad rank/nranks, unknown enum, bad config */
    HFR_ERR_UNSUPPORTED = 2,      /* valid but not implemented (op != SUM, PAIR_DBT with odd n, ...) */
    HFR_ERR_CUDA = 3,             /* a CUDA runtime call failed; see hfr_last_cuda_error() */
    HFR_ERR_OUT_OF_MEMORY = 4,
    HFR_ERR_PROTOCOL = 5,         /* ranks disagree on count/dtype/op/algo/buffer/call order */
    HFR_ERR_TIMEOUT = 6,          /* a cross-rank spin wait exceeded timeout_ms */
    HFR_ERR_NOT_INITIALIZED = 7,  /* NULL or finalized comm / request */
    HFR_ERR_INTERNAL = 8
} hfr_status_t;

/* Allreduce schedules (the three subsystems of DESIGN.md §1).
 *   FLAT     reduce-scatter + all-gather in one fused pass: rank g pulls shard g
 *            of all n buffers over NVLink, folds in rank order 0..n-1 (fp32),
 *            scales, casts, and stores the result into all n buffers.  Result =
 *            rank-ascending fold (Algorithm 1 order).
 *   ONESHOT  small messages: every rank pushes its whole buffer into every
 *            peer's inbox, then folds all n copies locally in rank order.  Same
 *            result bits as FLAT; one cross-rank handoff instead of two.  For
 *            small messages the flag travels inside each 8-byte data word (LL
 *            form, no fence: ~5 us on 4 B200s).
 *   DBT      the paper's double binary tree (Algorithm 2) as
 *            a push-only P2P schedule over the GPUs; chunk c rides tree c mod 2.
 *   PAIR_DBT "HFReduce with NVLink": pair (2k,2k+1) reduce,
 *            tree over the n/2 pair partials per half, pair all-gather.
 *   CE       copy-engine two-shot (the paper's "No GPU Kernel Overhead",
 *            PAPER.md:375): peers' shards are PULLED by the copy engines,
 *            cross-rank ordering uses stream memory operations (no SM spins),
 *            and only a short local fold kernel runs on the SMs — for
 *            overlapping with compute (DDP).  Same result bits as FLAT.
 *            Runs on real and virtual comms alike (virtual ranks: the copy
 *            engines copy between the ranks' buffers on one GPU); at n = 1 or
 *            for messages under n * 16 KiB it runs FLAT (nothing to move).
 *   NVLS     ORDER-RELAXED NVLink SHARP path: the NVSwitch sums
 *            the n copies (multimem.ld_reduce) and multicasts the owner's
 *            scaled result (multimem.st).  The switch chooses the summation
 *            order, so results are NOT bit-exact: they are held to DESIGN.md
 *            reading R18 (fp32 |err| <= 1e-6 * sum|x|, bf16 <= 1 ulp + that).
 *            Needs hfr_config.nvls_bytes > 0 at init and a buffer from
 *            hfr_mem_alloc inside that arena; otherwise UNSUPPORTED (never a
 *            silent change of numerics).
 *   AUTO     ONESHOT (LL form) while each rank pushes <= 6 MiB of LL words
 *            ((n-1) * count * 8 bytes: bf16 <= 256 KiB at n=4, <= 1 MiB at n=2),
 *            FLAT above (never NVLS). */
typedef enum {
    HFR_ALGO_AUTO = 0,
    HFR_ALGO_FLAT = 1,
    HFR_ALGO_DBT = 2,
    HFR_ALGO_PAIR_DBT = 3,
    HFR_ALGO_ONESHOT = 4,
    HFR_ALGO_CE = 5,
    HFR_ALGO_NVLS = 6
} hfr_algo_t;

/* All-gather callback used ONLY by the collective setup calls (hfr_init,
 * hfr_mem_alloc, hfr_register, hfr_finalize) to exchange CUDA IPC handles:
 * gather `bytes` from every rank into recv[nranks*bytes] in rank order.
 * Returns 0 on success.  Typically a torch.distributed all_gather. */
typedef int (*hfr_allgather_fn)(const void* send, void* recv, size_t bytes, void* ctx);

typedef struct {
    int algo;             /* hfr_algo_t */
    size_t chunk_elems;   /* tree chunk size in elements (Alg. 1 "Chunk_Size");
                             multiple of 256; 0 -> 16384 at n=2, 32768 otherwise (measured best).
                             Changes DBT/PAIR_DBT bits (reading R8), never FLAT's. */
    int max_ctas;         /* CTAs per rank; 0 -> the schedule's measured default (FLAT with TMA
                             staging: 1 per SM (2 with virtual ranks), tree schedules: 2 per SM (fp32 DBT: 3), others: 1 per SM, never
                             more than the work needs).  Caps the SMs the comm uses. */
    int threads;          /* threads per CTA (128..512, multiple of 32); 0 -> the schedule's default
                             (256 for FLAT with TMA staging and the tree schedules, 512 otherwise) */
    float scale;          /* gradient scale, multiplies the fp32 total once (reading R3); 1.0 = sum */
    size_t scratch_bytes; /* per-rank library scratch (staging + tree partials); 0 -> 256 MiB */
    int timeout_ms;       /* cross-rank spin-wait timeout; 0 -> 60000 */
    size_t oneshot_max_bytes; /* ONESHOT inbox slot bytes, fixed at init (per-rank inbox =
                                 2 * nranks * this); the largest message for an explicit ONESHOT;
                                 the LL form needs 8 * count <= this.  0 -> 4 MiB */
    int stream_gate;      /* 1: before launching an SM schedule, make the stream wait (stream memory
                             operations in the copy-engine front end, no SM) until every rank has
                             reached this call, so no CTA spins on a late peer (overlap with compute);
                             real comms only.  0 (default): off. */
    size_t nvls_bytes;    /* > 0: at init, build an NVLS multicast arena of this many bytes per rank
                             (cuMulticast*, fixed at init); hfr_mem_alloc then hands out memory from
                             it (usable by every algo; required by NVLS).  Ignored for virtual comms.
                             If the box has no NVLS, init still succeeds and NVLS calls return
                             UNSUPPORTED.  0 (default): no arena. */
    int flat_staging;     /* FLAT kernel staging: 0 auto (TMA bulk copies into shared memory for n in
                             {2,4,8}, registers otherwise), 1 registers (no shared memory: small CTAs
                             can share an SM with a compute kernel, e.g. DDP overlap), 2 TMA.  Bits
                             are identical either way. */
    size_t ll_push_max;   /* AUTO: largest (n-1) * count * 8 bytes a rank pushes in the LL ONESHOT
                             form before FLAT takes over; 0 -> 6 MiB (the r01 crossover on 2 and 4
                             B200s).  Part of the call signature (it picks the schedule). */
    int pdl_off;          /* 1: launch the latency-bound kernels (ONESHOT, LL ONESHOT, barrier) of a
                             real comm as ordinary launches; 0 (default): programmatic dependent
                             launches (see hfr_allreduce).  Never changes results. */
    int tree_staging;     /* DBT / PAIR_DBT data movement: 0 auto (= 1, measured faster), 1 registers
                             (SM loads/stores, one flag and one system fence per chunk), 2 TMA (bulk
                             copies in and out of shared memory, one flag per tile of <= 4096 elements,
                             raised when the tile's bulk stores completed).  Bits are identical
                             either way.  Part of the call signature. */
} hfr_config_t;

/* Fill *cfg with the defaults above (algo AUTO, scale 1.0). */
void hfr_config_default(hfr_config_t* cfg);

/* COLLECTIVE.  Create a communicator for `rank` of `nranks` (1..HFR_MAX_RANKS)
 * processes, each driving one GPU of this box (`cuda_device`) — the paper's
 * set of GPUs that "require allreduce" together (§4 Alg. 1;
 * :323 "GPU_Count").  Allocates the peer-mapped signal pad and scratch,
 * exchanges CUDA IPC handles through `allgather(ctx)`, opens the peers'
 * mappings.  cfg may be NULL (defaults).  nranks = 1 needs no callback
 * (allgather may be NULL).
 * On success *comm is owned by the caller until hfr_finalize.
 * Errors: INVALID_ARGUMENT (comm NULL, rank out of range, nranks out of range,
 * allgather NULL with nranks > 1, bad cfg), CUDA, OUT_OF_MEMORY. */
hfr_status_t hfr_init(hfr_comm_t* comm, int rank, int nranks, int cuda_device,
                      hfr_allgather_fn allgather, void* ctx, const hfr_config_t* cfg);

/* Single-process communicator with `nranks` VIRTUAL ranks on one GPU: every
 * kernel launch runs all ranks' CTAs at once (cooperative launch), peer
 * "NVLink" accesses become local HBM accesses.  Same kernels, same protocol;
 * used for the 1-GPU bench line and the 1-GPU parity tests. */
hfr_status_t hfr_init_virtual(hfr_comm_t* comm, int nranks, int cuda_device, const hfr_config_t* cfg);

/* COLLECTIVE.  Change the configuration for subsequent calls
 * (scratch_bytes, timeout_ms, oneshot_max_bytes and nvls_bytes are fixed at
 * init and keep their init values). */
hfr_status_t hfr_comm_set_config(hfr_comm_t comm, const hfr_config_t* cfg);

/* Number of ranks this process drives: 1 for hfr_init comms, nranks for
 * virtual comms.  Also rank / nranks queries. */
int hfr_comm_local_ranks(hfr_comm_t comm);
int hfr_comm_rank(hfr_comm_t comm);
int hfr_comm_nranks(hfr_comm_t comm);

/* COLLECTIVE.  Allocate `bytes` of symmetric peer-mapped device memory.
 * ptrs receives hfr_comm_local_ranks(comm) pointers (one per local rank).
 * Buffers inside such memory are reduced zero-copy (no staging).  Freed by
 * hfr_mem_free (collective) or hfr_finalize. */
hfr_status_t hfr_mem_alloc(hfr_comm_t comm, size_t bytes, void** ptrs);
/* COLLECTIVE.  Release an hfr_mem_alloc allocation (ptr = the first pointer
 * hfr_mem_alloc returned).  Memory inside the NVLS arena is released only by
 * hfr_finalize (SUCCESS, no-op).  INVALID_ARGUMENT for unknown pointers. */
hfr_status_t hfr_mem_free(hfr_comm_t comm, void* ptr);

/* COLLECTIVE.  Make an existing cudaMalloc'ed range [ptr, ptr+bytes) peer
 * visible (its whole allocation is IPC-exported and opened by every peer).
 * Idempotent per allocation.  Real comms only (virtual comms: no-op). */
hfr_status_t hfr_register(hfr_comm_t comm, void* ptr, size_t bytes);

/* COLLECTIVE.  Undo hfr_register for the registered allocation containing
 * `ptr` (drains this device, then every peer closes its IPC mapping).  Call
 * before freeing registered memory: a later allocation at the same address
 * must not reuse stale peer mappings.  INVALID_ARGUMENT if `ptr` lies in no
 * registered range; virtual comms: no-op. */
hfr_status_t hfr_deregister(hfr_comm_t comm, void* ptr);

/* COLLECTIVE, asynchronous.  In-place sum-allreduce of `count` elements of
 * `dtype` at device pointer `buf` ("Dg: data need to allreduce",
 * :367 "Dg_i is allreduced").
 *   Ordering: starts after all work already enqueued on `stream`; returns to
 *   the host immediately.  If req != NULL the work runs on the comm's side
 *   stream and *req must be passed to hfr_wait exactly once; if req == NULL it
 *   runs on `stream` itself (completion is stream-ordered).  Real comms launch
 *   their small-message kernels as programmatic dependent launches: a kernel
 *   may become resident while the previous kernel on the stream finishes, but
 *   touches no memory before that kernel has completed (griddepcontrol.wait),
 *   so the ordering above is unchanged (config pdl_off = 1: ordinary launches).
 *   Result: every rank's buf holds identical bytes: the rank-ascending fold
 *   (FLAT), the tree-order fold (DBT) or the pair-first fold (PAIR_DBT), times
 *   scale, cast to dtype.  Buffers outside hfr_mem_alloc / hfr_register memory
 *   or not 16-byte aligned are staged through the scratch (correct, slower).
 *   Ownership: caller owns buf; it must stay allocated and untouched until
 *   completion.  All calls on one comm (allreduce, collectives, barrier; sync
 *   or async, on any streams) execute in issue order: each call's stream
 *   waits for the previous call's completion event.  Calls made during stream
 *   capture are ordered by the capturing stream only.
 *   Memory kind (peer-mapped zero-copy vs staged) is part of the collective
 *   contract: ranks must agree (a disagreement is PROTOCOL when the kernels
 *   meet, but the first call of a size may block in the scratch growth
 *   exchange until the allgather callback's own timeout).
 *   CUDA graphs: calls may be captured (stream capture) and replayed; launch
 *   epochs live in device memory.  The first call of a given size must run
 *   uncaptured (it may grow the scratch, which is collective); a captured
 *   call that would need more scratch returns UNSUPPORTED, and so does a
 *   captured HFR_ALGO_CE call (its stream-memop flags carry host epochs).
 *   Errors (returned now): NOT_INITIALIZED, INVALID_ARGUMENT (buf NULL with
 *   count > 0, unknown dtype), UNSUPPORTED (op != SUM), CUDA.  count == 0 is a
 *   successful no-op.  Cross-rank errors (PROTOCOL, TIMEOUT) surface at
 *   hfr_wait / hfr_comm_status. */
hfr_status_t hfr_allreduce(hfr_comm_t comm, void* buf, size_t count, hfr_dtype_t dtype,
                           hfr_op_t op, hfr_stream_t stream, hfr_req_t* req);

/* Virtual-comm form: bufs[r] is virtual rank r's buffer (all on the comm's
 * device).  Same semantics as hfr_allreduce. */
hfr_status_t hfr_allreduce_virtual(hfr_comm_t comm, void* const* bufs, size_t count, hfr_dtype_t dtype,
                                   hfr_op_t op, hfr_stream_t stream, hfr_req_t* req);

/* The other collectives HFReduce serves ("general reduce and broadcast",
 * PAPER.md:297; FSDP/ZeRO reduce-scatter and all-gather).  All
 * are in place on `buf` (count elements) and use the shard layout of
 * hfr_shard_range: shard g = [lo_g, hi_g).
 *   HFR_REDUCE_SCATTER  rank g's shard g := rank-ascending fold of shard g over all
 *                       ranks, times scale, cast; the rest of buf is unchanged.
 *   HFR_ALLGATHER       every rank's shard g := rank g's shard g (raw bytes, no scale).
 *   HFR_REDUCE          root's buf := the allreduce result; other ranks' buf unchanged.
 *   HFR_BROADCAST       every rank's buf := root's buf (raw bytes).
 *   HFR_ALLREDUCE       = hfr_allreduce (every schedule of hfr_config_t.algo).
 * The non-allreduce collectives run the FLAT kernel (bit-exact, same fold
 * order), except with hfr_config_t.algo == HFR_ALGO_NVLS on a buffer inside
 * the NVLS arena: then they run on the multicast object — ALLGATHER and
 * BROADCAST by multimem.st (bit-exact), REDUCE_SCATTER and REDUCE by
 * multimem.ld_reduce (order-relaxed, reading R18), UNSUPPORTED elsewhere.
 * root is ignored except for REDUCE / BROADCAST. */
typedef enum {
    HFR_ALLREDUCE = 0,
    HFR_REDUCE_SCATTER = 1,
    HFR_ALLGATHER = 2,
    HFR_REDUCE = 3,
    HFR_BROADCAST = 4
} hfr_coll_t;

hfr_status_t hfr_collective(hfr_comm_t comm, hfr_coll_t coll, void* buf, size_t count, hfr_dtype_t dtype,
                            hfr_op_t op, int root, hfr_stream_t stream, hfr_req_t* req);
hfr_status_t hfr_collective_virtual(hfr_comm_t comm, hfr_coll_t coll, void* const* bufs, size_t count,
                                    hfr_dtype_t dtype, hfr_op_t op, int root, hfr_stream_t stream, hfr_req_t* req);

/* Host-only: shard g of a count-element buffer of dtype over nranks ranks,
 * [*lo, *hi): 16-byte-vector granular, the ragged tail in the last shard. */
hfr_status_t hfr_shard_range(int nranks, size_t count, hfr_dtype_t dtype, int rank, size_t* lo, size_t* hi);


/* Complete a request — the paper's asynchronous allreduce returns at once and
 * its completion is awaited before the gradients are used (PAPER.md:309
 * "asynchronous", :451 "asynchronous allreduce ... overlap with the
 * computation", :367 "Dg_i is allreduced").  stream != NULL: make `stream`
 * wait for it (no host block; pass (hfr_stream_t)1 = cudaStreamLegacy for
 * the legacy default stream).  stream == NULL: block the host until done and
 * report PROTOCOL / TIMEOUT / CUDA errors raised by the kernels.  Releases
 * req (it must not be used again).  req == NULL (count == 0 calls): SUCCESS. */
hfr_status_t hfr_wait(hfr_req_t req, hfr_stream_t stream);

/* Non-blocking check: SUCCESS, or the sticky cross-rank error seen so far. */
hfr_status_t hfr_comm_status(hfr_comm_t comm);

/* COLLECTIVE.  Device-side barrier across all ranks, enqueued on `stream`
 * (used to align ranks before a timed region); ordered after the comm's
 * previous call like every other call. */
hfr_status_t hfr_barrier(hfr_comm_t comm, hfr_stream_t stream);

/* COLLECTIVE.  Tear down what hfr_init built (the communicator of PAPER.md:309,
 * §4 Alg. 1): synchronise this device, host barrier through the allgather
 * callback (no peer still reads or writes this rank's memory), close the
 * peers' IPC mappings, free the pad, scratch (including outgrown scratch
 * regions kept alive for in-flight kernels), hfr_mem_alloc memory and the
 * NVLS arena.  The comm handle is invalid afterwards.  Errors:
 * NOT_INITIALIZED (NULL comm). */
hfr_status_t hfr_finalize(hfr_comm_t comm);

/* Host-only query of the double binary tree the DBT schedule uses (reading
 * R9): for tree `which` (0 = A, 1 = B) over n ranks, fills parent[n] (-1 at
 * the root) and child0[n], child1[n] (children in ascending rank, -1 if
 * absent).  No GPU needed. */
hfr_status_t hfr_tree_query(int n, int which, int* parent, int* child0, int* child1);

/* Diagnostic: record per-CTA chunk timelines of the tree schedules into
 * `dev_buf` (device memory, >= 64 * 1024 * local_ranks bytes; capacity per CTA
 * = bytes / (64 * 1024 * local_ranks) events of 8 u64 {tag, t_wait, t_work,
 * t_stores_issued, t_done, 0, 0, 0} in globaltimer ns, CTA slot =
 * local_rank * 1024 + cta).  NULL turns tracing off.  Not for production use
 * (adds timer reads). */
hfr_status_t hfr_set_trace(hfr_comm_t comm, void* dev_buf, size_t bytes);

/* Kernel launches this comm has issued (for bench.py's gpu_launches). */
uint64_t hfr_comm_launches(hfr_comm_t comm);

const char* hfr_status_string(hfr_status_t s);
/* Text of the last CUDA error seen by this thread's calls (or ""). */
const char* hfr_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HFR_H_ */
