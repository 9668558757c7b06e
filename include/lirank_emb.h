/*
 * lirank_emb.h -- C ABI of the B200-native LiRank sparse-embedding hot path.
 *
 * The library (paper_2402_06859_b200/liblirank_emb.so, sm_100a) implements the
 * sparse-feature embedding path of LiRank (arXiv 2402.06859):
 *
 *   a2  pooled multi-hot lookup          PAPER.md:194 ("Sparse ID embedding features are
 *                                        transformed into dense embeddings through lookup in
 *                                        embedding tables"), PAPER.md:536-538 (features,
 *                                        "concatenated with all other dense features")
 *   a5  id dedup (radix sort)            BASELINE.json north_star; SURVEY.md §8(a)
 *   a6  segment-reduce of the gradient   PAPER.md:17 ("the global gradient")
 *   a7  global-norm clip to unit norm    PAPER.md:17 ("clip the global gradient to have
 *                                        unit norm for all experiments")
 *   a8  sparse AdaGrad on touched rows   PAPER.md:17, 516 ("we had to leverage AdaGrad for
 *                                        models where the number of sparse features was high")
 *   a9  middle-max row-wise 8-bit quant  PAPER.md:338-345 (X^middle, X^scale, X^int)
 *   a10 quantized-table pooled lookup    PAPER.md:341 (X^dequant = X^middle + X^int * X^scale)
 *   a1/a3/a4 all-to-all exchange (W>1)   PAPER.md:576 ("each GPU's input batch is
 *                                        all-to-all'ed ... lookups are all-to-all'ed to
 *                                        return the output")
 *
 * The exact arithmetic of every step (operation order, fp64 accumulations, rounding)
 * is SURVEY.md §8(c) with the readings listed in DESIGN.md §3.
 *
 * Conventions
 * -----------
 * - Memory ownership: the CALLER owns all device memory.  emb_plan() reports the byte
 *   sizes of the buffers a configuration needs; the caller allocates them (e.g. torch
 *   tensors) and passes them to emb_create().  The library owns only the handle and its
 *   host-side metadata (and, for world_size > 1, its NCCL communicator).  All device
 *   buffers must be 256-byte aligned and stay valid until emb_destroy().
 * - Streams: every call is enqueued on cfg.stream (a cudaStream_t; NULL = legacy default
 *   stream) and returns without waiting, unless it is documented to return host values.
 * - Pointers "host or device": ids, offsets, grad and out arguments may be device
 *   pointers or host pointers (detected with cudaPointerGetAttributes).  Host ids / offsets
 *   are copied into one of two library staging slots on an internal copy stream (the call's
 *   kernels wait for the copy; the copy waits only for the slot's previous readers, so the
 *   next call's transfer overlaps this call's kernels); a host grad is copied on the stream
 *   before the kernels; a host `out` is
 *   filled by a device-to-host copy after the kernels and the call then WAITS for the
 *   stream, so a host `out` is complete when the call returns.  Host inputs must stay
 *   valid until the call's work is done (a host-`out` call, emb_sync(), or a stream
 *   synchronisation).  Pinned host memory gives asynchronous copies; pageable memory works
 *   but copies synchronously.
 * - Errors: argument errors are returned synchronously and nothing is enqueued.  Data-
 *   dependent errors (out-of-range ids, non-finite gradient norm, non-finite table row
 *   at quantize) are recorded in a sticky device status word and reported (and cleared)
 *   by emb_sync().  CUDA launch/copy failures return EMB_ECUDA.
 * - Threading: one handle per (process, device); calls on a handle are not thread-safe.
 * - Multi-GPU (world_size > 1): every call is collective -- all ranks must issue the same
 *   sequence of calls.
 */
#ifndef LIRANK_EMB_H
#define LIRANK_EMB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMB_ABI_VERSION 2  /* 2: emb_config.table_cost, EMB_F_HOSTCOMM, emb_allreduce_f32 */

#if defined(__GNUC__)
#define EMB_API __attribute__((visibility("default")))
#else
#define EMB_API
#endif

typedef enum {
  EMB_OK = 0,
  EMB_EINVAL = 1,      /* bad argument (null pointer, size out of range, misalignment)   */
  EMB_ENOMEM = 2,      /* a supplied buffer is smaller than emb_plan() asked for; sticky
                          (sharded): a call's ids exceeded a planned receive capacity
                          (max_recv_nnz) -- the call was discarded on every rank        */
  EMB_ECUDA = 3,       /* a CUDA runtime call failed                                     */
  EMB_ENCCL = 4,       /* an NCCL call failed                                            */
  EMB_EIDRANGE = 5,    /* sticky: an id was < 0 or >= rows of its table (it was skipped) */
  EMB_ENONFINITE = 6,  /* sticky: non-finite global norm (update skipped) or non-finite
                          row at quantize (row stored as codes 0, middle 0, scale 0)      */
  EMB_ESTATE = 7       /* call out of order (backward before forward, q8 before quantize) */
} emb_status;

enum { EMB_POOL_SUM = 0, EMB_POOL_MEAN = 1 };
enum { EMB_ADAGRAD_ROWWISE = 0, EMB_ADAGRAD_ELEMENTWISE = 1 };
enum { EMB_SHARD_NONE = 0, EMB_SHARD_TABLE = 1, EMB_SHARD_ROW = 2 };

/* cfg.flags */
#define EMB_F_Q8 1u       /* allocate the int8 store (codes + per-row meta) for a9/a10       */
#define EMB_F_REQUANT 2u  /* (needs EMB_F_Q8) every AdaGrad update also re-quantizes the rows
                             it touched, so the q8 store tracks the fp32 tables between
                             full emb_quantize_mm8() passes                                   */
#define EMB_F_Q8_MINMAX 16u /* (needs EMB_F_Q8) NEXT-4: the q8 store holds MIN-MAX row-wise codes
                             (the baseline the paper contrasts middle-max with):
                             uint8 codes = clamp(round((x - min) / scale), 0, 255), meta {min,
                             scale} in place of {middle, scale}; a10 dequantizes
                             fmaf(code, scale, min).  Same row layout and kernels.             */
#define EMB_F_Q8_ONLY 32u  /* (needs EMB_F_Q8) SERVING handle (P:549-557 in-memory serving of the
                             quantized tables): no fp32 weights or accumulators exist
                             (weights_bytes = accum_bytes = 0; buf.weights / buf.accum may be
                             NULL) and no training workspace is planned.  Rows enter the q8
                             store through emb_quantize_block; emb_forward_q8 serves lookups.
                             Training / fp32 calls return EMB_ESTATE.  This is what lets the
                             1B-row Feed tables (96 GB as q8) be served from one GPU.          */
#define EMB_F_EXCHANGE 8u /* run the sharded exchange path even at world_size 1 (a 1-rank
                             communicator; exercises the transport on a single GPU)          */
#define EMB_F_P2P 64u     /* (sharded) FUSED EXCHANGE over peer memory (NVLink / NVSwitch): the
                             a1 ids are stored by one kernel at their final (compacted, source-
                             ordered) place in each owner's receive buffer; the owner's pooling
                             kernel stores every pooled row straight into the source rank's
                             buffer -- table-wise in its final [B][F][D] place, row-wise into a
                             per-owner slot summed in rank order -- and the backward's grad
                             rows are pushed into the owners' buffers by one kernel; stream-
                             ordered barriers (a 4-byte all-gather) replace the all-to-alls,
                             the reduce-scatter and the all-gather.  Peer mappings: CUDA IPC
                             of the workspace allocation (NCCL / host transports) or the other
                             handle's buffers (loopback), made by the first sharded forward
                             (collective); it returns EMB_ENCCL on EVERY rank if any rank
                             cannot map its peers (create again without the flag).  Workspace
                             grows by world * B * F * D floats (row-wise).
                             Without the flag the ids travel as an all-to-all of capacity-
                             padded slots (min(max_nnz, max_recv_nnz) ids per rank pair).
                             Either way no call of a sharded step reads a count on the host:
                             a sharded step can be captured as a CUDA graph.              */
#define EMB_F_LOOPBACK 4u /* (world_size > 1) TEST TRANSPORT: the ranks are threads of one
                             process sharing one device; cfg.nccl_unique_id is the hub from
                             emb_loopback_hub_create().  Every collective becomes a host
                             rendezvous + stream-ordered device copies (no kernel waits on
                             another rank).  Same exchange code path as NCCL otherwise.       */

#define EMB_F_HOSTCOMM 128u /* (world_size > 1) TEST TRANSPORT: one rank per PROCESS (e.g. several
                             processes sharing one GPU); cfg.nccl_unique_id points to an
                             emb_host_comm.  Every collective drains the stream and moves its
                             bytes through host memory with the caller's host all-gather; peer
                             memory (EMB_F_P2P) is mapped with CUDA IPC.  No kernel waits on
                             another rank.  Same exchange code path as NCCL otherwise.        */

/* The caller's host all-gather for EMB_F_HOSTCOMM: recv[r * bytes .. (r+1) * bytes) = the
 * `bytes` at send of rank r, for every rank r (a blocking collective over host memory, e.g.
 * torch.distributed.all_gather over gloo).  Returns 0 on success. */
typedef struct {
  void* ctx;
  int32_t (*allgather)(void* ctx, const void* send, void* recv, int64_t bytes);
} emb_host_comm;

typedef struct {
  uint32_t abi_version;          /* must be EMB_ABI_VERSION                                    */
  int32_t num_tables;            /* T >= 1                                                    */
  const int64_t* table_rows;     /* host [T]: rows of each (global, unsharded) table, < 2^31  */
  int32_t dim;                   /* D in [1, 1024]: embedding width, shared by all tables     */
  int32_t num_features;          /* F >= 1                                                    */
  const int32_t* feature_table;  /* host [F]: the table feature f reads.  Several features may
                                    share a table ("40 categorical features ...
                                    through 5 shared embedding matrices"); they then share its
                                    rows, and dedup merges their occurrences (reading 19).    */
  int32_t pooling;               /* EMB_POOL_SUM (default) or EMB_POOL_MEAN                   */
  int32_t adagrad_mode;          /* EMB_ADAGRAD_ROWWISE (default) or EMB_ADAGRAD_ELEMENTWISE  */
  float init_accumulator;        /* AdaGrad A0 (Keras default 0.1)                            */
  float eps;                     /* AdaGrad epsilon, outside the sqrt (Keras default 1e-7)    */
  float max_norm;                /* global-norm clip threshold (paper: 1.0)      */
  int64_t max_nnz;               /* capacity: ids per call on this rank, < 2^30               */
  int32_t max_batch;             /* capacity: local batch B per call                          */
  int32_t sharding;              /* EMB_SHARD_NONE (world_size 1), _TABLE or _ROW              */
  const int32_t* table_owner;    /* host [T] or NULL: explicit table-wise plan (owner rank)   */
  int32_t rank, world_size;      /* this process's rank and the number of ranks               */
  const void* nccl_unique_id;    /* 128-byte ncclUniqueId from rank 0 (NULL if world_size 1)  */
  void* stream;                  /* cudaStream_t every call is enqueued on                    */
  uint32_t flags;                /* EMB_F_*                                                   */
  int64_t max_recv_nnz;          /* sharded: capacity of occurrences this rank pools per call
                                    (its rows' share of every rank's ids); 0 = min(2, W) *
                                    max_nnz.  A call that exceeds it on any rank is discarded
                                    on every rank (zero outputs, no occurrences) with sticky
                                    EMB_ENOMEM (emb_sync).                                    */
  const double* table_cost;      /* host [T] or NULL: table-wise planning weight of each table,
                                    e.g. its expected bytes per step, B * L_t * (4 + row
                                    bytes) + B * row bytes with L_t the mean ids per sample
                                    on the table.  The automatic plan
                                    balances these; NULL balances rows.                     */
} emb_config;

typedef struct {
  int64_t weights_bytes;    /* fp32 [local_rows][row_pitch]                                    */
  int64_t accum_bytes;      /* fp32 [local_rows] (row-wise) or [local_rows][row_pitch]         */
  int64_t q8_codes_bytes;   /* q8 rows [local_rows][q8_pitch] (0 without EMB_F_Q8), each row =
                               [D int8 codes][pad to 8][fp32 middle][fp32 scale][pad]: one
                               contiguous run of whole 32-B sectors (D=64: 96 B), or of whole
                               64-B DRAM atoms with EMB_F_REQUANT (D=64: 128 B); every write
                               of a row rewrites all of it, pads as zero bytes                 */
  int64_t q8_meta_bytes;    /* 0 (metadata lives in the q8 rows; kept for ABI stability)       */
  int64_t workspace_bytes;  /* library scratch (staging, sort, segment partials, scalars)      */
  int64_t local_rows;       /* rows stored on this rank (sum over its local tables)            */
  int32_t row_pitch;        /* floats per stored fp32 row: round_up(D, 4) (16-B aligned rows)  */
  int32_t q8_pitch;         /* bytes per q8 row: round_up(round_up(D, 8) + 8, 32), or ... 64)
                               with EMB_F_REQUANT                                              */
} emb_sizes;

typedef struct {
  void* weights;    /* device; caller initialises it (layout: emb_local_layout) or uses
                       emb_write_rows                                                      */
  void* accum;      /* device; emb_create fills it with init_accumulator                   */
  void* q8_codes;   /* device (q8 rows) or NULL without EMB_F_Q8                           */
  void* q8_meta;    /* unused (may be NULL)                                                */
  void* workspace;  /* device                                                              */
} emb_buffers;

typedef struct emb_handle* emb_t;

EMB_API int32_t emb_abi_version(void);
EMB_API const char* emb_status_string(emb_status s);

/* Validate cfg and report buffer sizes (host-only; no CUDA calls).  For sharded
 * configurations it also fixes the plan: table-wise = cfg.table_owner if given, else a
 * greedy longest-processing-time assignment of tables by cfg.table_cost (by rows when
 * NULL): largest first, each to the least-loaded rank (ties to the lower rank);
 * row-wise = rank r owns rows [r*ceil(R/W), (r+1)*ceil(R/W)) of every table. */
EMB_API emb_status emb_plan(const emb_config* cfg, emb_sizes* out);

/* Per-table layout of this rank's weights buffer (host-only).  For each table t:
 * local_base[t] = first stored row of table t in `weights` (or -1 if t has no rows
 * here), row_lo[t] / row_hi[t] = the global rows [row_lo, row_hi) of t stored here.
 * Stored row (local_base[t] + (r - row_lo[t])) holds global row r of table t. */
EMB_API emb_status emb_local_layout(const emb_config* cfg, int64_t* local_base, int64_t* row_lo,
                            int64_t* row_hi);

/* Multi-GPU bootstrap (host-only).  Rank 0 calls emb_nccl_unique_id and distributes the
 * 128 bytes (e.g. a torch.distributed broadcast); every rank passes them as
 * cfg.nccl_unique_id.  NCCL is loaded at run time (libnccl.so.2, the copy PyTorch ships);
 * EMB_ENCCL if it is unavailable.  The loopback hub (EMB_F_LOOPBACK) is for tests. */
EMB_API emb_status emb_nccl_unique_id(void* out128);
EMB_API emb_status emb_loopback_hub_create(int32_t world, void** hub);
EMB_API emb_status emb_loopback_hub_destroy(void* hub);

/* Bind buffers, fill the accumulators with init_accumulator, clear the status word, and
 * (world_size > 1) create the communicator.  Enqueued on cfg.stream.
 * Sharded configurations (world_size > 1): every rank passes its own local batch B (the
 * same B on all ranks) to emb_forward; rows are exchanged with their owners (a1), pooled
 * there and returned (a3: table-wise all-to-all, row-wise reduce-scatter of partial sums),
 * and gradients flow back (a4) to the owners' a5-a8.  MEAN pooling is not supported when
 * sharded (EMB_EINVAL). */
EMB_API emb_status emb_create(const emb_config* cfg, const emb_buffers* buf, emb_t* out);

/* a2 (+ a1/a3 when sharded).  ids: int32 [nnz] feature-major, offsets: int32 [F*B+1]
 * with offsets[0] = 0 and offsets[F*B] = nnz; bag (f, b) is ids[offsets[f*B+b] ..
 * offsets[f*B+b+1]).  out: fp32 [B][F][D] (sample-major, feature order = feature index,
 * reading 20), 16-B aligned when D % 4 == 0.  Bag sums are taken in bag order; MEAN
 * divides by the bag length; an empty bag gives zeros.  An id outside [0, rows) of its
 * table is skipped (contributes 0, gets no gradient) and sets sticky EMB_EIDRANGE.
 * Also records this batch's (row, bag) occurrences for the next emb_backward_adagrad. */
EMB_API emb_status emb_forward(emb_t h, const int32_t* ids, const int32_t* offsets, int32_t batch,
                       int64_t nnz, float* out);

/* a5-a8 (+ a4 when sharded) for the batch of the most recent emb_forward (EMB_ESTATE if
 * none).  grad_out: fp32 [B][F][D] = dL/d(out) of that forward.  Dedups the occurrences by
 * (table, row), reduces G_u in fp64, forms the global squared norm
 * S = sum over ranks (rank order) of sum_u ||G_u||^2, + extra_sq_norm, the clip factor
 * c = min(1, max_norm / sqrt(S)), and applies AdaGrad (cfg.adagrad_mode) with step lr to
 * the touched rows only.  extra_sq_norm lets the caller fold the dense-tower gradient into
 * the global norm (pass 0 otherwise); it is added ONCE, not summed over ranks, so with
 * world_size > 1 every rank must pass the SAME value (the norm of the all-reduced dense
 * gradient, emb_allreduce_f32), or ranks would clip with different factors.  Non-finite S: no row is updated, sticky
 * EMB_ENONFINITE.  If sq_norm_out (host) is non-NULL the call waits for the step and
 * returns S there. */
EMB_API emb_status emb_backward_adagrad(emb_t h, const float* grad_out, float lr, double extra_sq_norm,
                                double* sq_norm_out);

/* Data-parallel dense side (NEXT-2, "Other layers ... processed in a data
 * parallel way"): data[0..count) (DEVICE fp32) = its sum over all ranks, in place, on the
 * library stream and transport (NCCL all-reduce; loopback / host transports sum in rank
 * order).  Every rank ends with identical values -- which is what makes the dense squared
 * norm a caller then passes as extra_sq_norm(_dev) identical on every rank, as the global
 * clip requires.  world_size 1: no-op.  (The loopback transport stages through a device
 * buffer it allocates on first use, so do not call it first inside a graph capture.) */
EMB_API emb_status emb_allreduce_f32(emb_t h, float* data, int64_t count);

/* As emb_backward_adagrad, with no host synchronisation for a dense side on the device
 * (NEXT-2, "global gradient clipped to unit norm" over sparse + dense; P:538 tower):
 * extra_sq_norm_dev (device fp64, optional) is the caller's dense squared gradient norm,
 * read on the stream when the global norm is formed; clip_out_dev (device fp32, optional)
 * receives the clip factor c the caller scales its dense gradients by (c = -1 when S is not
 * finite: the sparse update was skipped and the caller should skip its dense update);
 * sq_norm_out_dev (device fp64, optional) receives S.  Enqueued on cfg.stream; returns
 * without waiting. */
EMB_API emb_status emb_backward_adagrad_dev(emb_t h, const float* grad_out, float lr,
                                            const double* extra_sq_norm_dev, float* clip_out_dev,
                                            double* sq_norm_out_dev);

/* a9: quantize every local row (middle-max, 8 bits) into the q8 store.
 * The fp32 tables are kept.  EMB_ESTATE without EMB_F_Q8. */
EMB_API emb_status emb_quantize_mm8(emb_t h);

/* a10: like emb_forward, but reading the q8 store: out = sum in bag order of
 * fmaf(code, scale, middle).  EMB_ESTATE before the first emb_quantize_mm8 (unless
 * EMB_F_REQUANT has kept it current).  Does not record occurrences for backward.
 * ids == offsets == NULL: look up the batch of the most recent emb_forward (batch and nnz
 * must equal its, else EMB_EINVAL; EMB_ESTATE if there was none, or if its staging slot
 * has since been refilled by two later host-input calls) -- host inputs of that forward are
 * not copied again (its staged copy is used); device inputs must still hold the same values.
 * Sharded (W > 1 or EMB_F_EXCHANGE): if no other q8 lookup with fresh inputs came in between,
 * the forward's ids exchange (a1) is reused -- the owners look up the ids they already hold
 * (collective: every rank must make the same call, as always).                               */
EMB_API emb_status emb_forward_q8(emb_t h, const int32_t* ids, const int32_t* offsets, int32_t batch,
                          int64_t nnz, float* out);

/* Wait for the stream; return and clear the sticky status (EMB_OK if none). */
EMB_API emb_status emb_sync(emb_t h);

/* Synchronous introspection (waits for the stream).  Rows are GLOBAL row indices of
 * `table`; every requested row must be stored on this rank (EMB_EINVAL otherwise).
 * w: host fp32 [n][D]; acc: host fp32 [n] (row-wise) or [n][D] (element-wise), may be
 * NULL. */
EMB_API emb_status emb_read_rows(emb_t h, int32_t table, const int64_t* rows, int64_t n, float* w,
                         float* acc);
EMB_API emb_status emb_write_rows(emb_t h, int32_t table, const int64_t* rows, int64_t n,
                          const float* w, const float* acc);
/* codes: host int8 [n][D] (the raw bytes: uint8 codes under EMB_F_Q8_MINMAX); middle, scale:
 * host fp32 [n] (the row's min instead of its middle under EMB_F_Q8_MINMAX; either may be NULL). */
EMB_API emb_status emb_read_q8(emb_t h, int32_t table, const int64_t* rows, int64_t n, int8_t* codes,
                       float* middle, float* scale);

/* Synchronous: the dedup of the last backward (a5).  unique: host int32 [cap] local row
 * keys (stored-row indices, ascending); seg_offsets: host int32 [cap+1] CSR starts into
 * the sorted occurrence list; sorted_bags: host int32 [cap_occ] bag index (f*B+b) of each
 * sorted occurrence (may be NULL).  n_unique / n_valid receive U and the number of valid
 * occurrences.  EMB_ENOMEM if cap < U or cap_occ < n_valid. */
EMB_API emb_status emb_last_dedup(emb_t h, int32_t* unique, int32_t* seg_offsets, int64_t cap,
                          int32_t* sorted_bags, int64_t cap_occ, int64_t* n_unique,
                          int64_t* n_valid);

/* Synchronous: scalars of the last backward: global squared norm S (incl. extra and
 * other ranks), clip factor c, U on this rank. */
EMB_API emb_status emb_last_stats(emb_t h, double* sq_norm, float* clip, int64_t* n_unique);

/* Number of kernels this handle has launched so far (for launch accounting). */
EMB_API int64_t emb_kernel_launches(emb_t h);

/* Phase profiling with CUDA events recorded on cfg.stream around each phase of every
 * call (the kernels of one phase run back to back, so a phase's event pair times them).
 * emb_profile(h, 1) starts recording, (h, 0) stops.  emb_profile_read waits for the
 * stream, adds the elapsed times of all recorded phases into ms[EMB_PH_COUNT] (and the
 * number of recorded phase instances into count[EMB_PH_COUNT]; either may be NULL), and
 * with reset != 0 clears the accumulators first. */
enum {
  EMB_PH_FWD = 0,        /* a2 fp32 pooled lookup kernel                         */
  EMB_PH_SORT = 1,       /* a5 radix histogram + digit passes                    */
  EMB_PH_RLE = 2,        /* a5 run-length encode                                 */
  EMB_PH_SEGREDUCE = 3,  /* a6 chunk segment-reduce + fix-ups                    */
  EMB_PH_NORM = 4,       /* a7 norm partial (+ rank exchange) + clip factor      */
  EMB_PH_UPDATE = 5,     /* a8 clip + AdaGrad (+ fused re-quantize)              */
  EMB_PH_FWD_Q8 = 6,     /* a10 q8 pooled lookup kernel                          */
  EMB_PH_QUANTIZE = 7,   /* a9 full-table quantize                               */
  EMB_PH_COPY = 8,       /* host<->device staging copies                         */
  EMB_PH_EXCHANGE = 9,   /* a1/a3/a4 multi-GPU exchange                          */
  EMB_PH_COUNT = 10
};
EMB_API emb_status emb_profile(emb_t h, int32_t enable);
EMB_API emb_status emb_profile_read(emb_t h, double* ms, int64_t* count, int32_t reset);

/* Quantize (a9, the store's mode) a block of table rows given in fp32 into the q8 store:
 * rows[i * ld .. + D) holds row row0 + i of `table` (GLOBAL row index; every row of the block
 * must be stored on this rank), i < n.  rows is a DEVICE pointer, 16-B aligned, ld % 4 == 0,
 * ld >= D.  Enqueued on cfg.stream.  Marks the q8 store as filled (the caller is responsible
 * for covering every row it will look up).  Needs EMB_F_Q8; works with or without fp32
 * tables (with them, the block is NOT written to the fp32 table). */
EMB_API emb_status emb_quantize_block(emb_t h, int32_t table, int64_t row0, int64_t n,
                                      const float* rows, int64_t ld);

/* ---- NEXT-3: incremental training (Eq. 2-3) -----------------------------
 * Total loss = loss_D(w) + lambda_f/2 [alpha (w - w0)^T H0 (w - w0)
 *                                      + (1 - alpha)(w - w1)^T H1 (w - w1)],
 * H0, H1 the diagonal empirical-FIM approximations of the Hessian, w0 the cold-start
 * model, w1 = w_{t-1} (the prior model), alpha the "cold weight".
 *
 * emb_set_incremental: every later emb_backward_adagrad* adds the penalty gradient
 *   lambda_f [alpha H0 (w - w0) + (1 - alpha) H1 (w - w1)] (fp32, in this order) to the
 *   deduplicated gradient of the rows the step TOUCHES (untouched rows are not regularized:
 *   lazy, like the sparse update itself), before the global norm and the clip.  w0, H0, w1, H1
 *   are DEVICE fp32 arrays in the weights' layout ([local_rows][row_pitch], 16-B aligned),
 *   owned by the caller and read during each backward; a (w, H) pair may be NULL (both) to
 *   drop its term.  lambda_f = 0 or both pairs NULL turns the penalty off.  EMB_EINVAL for
 *   lambda_f < 0, alpha outside [0, 1], half a pair or host pointers.
 * emb_cold_weight_init: W = alpha w0 + (1 - alpha) w1 over all local rows ("initialized
 *   as alpha w0 + (1 - alpha) w_{t-1}"), fp32 fl(fl(alpha w0) + fl((1 - alpha) w1)); enqueued
 *   on cfg.stream.  The q8 store is not touched (call emb_quantize_mm8). */
EMB_API emb_status emb_set_incremental(emb_t h, const float* w0, const float* H0, const float* w1,
                                       const float* H1, float lambda_f, float alpha);
EMB_API emb_status emb_cold_weight_init(emb_t h, const float* w0, const float* w1, float alpha);

/* Release the handle (and its NCCL communicator).  Does not free caller buffers. */
EMB_API emb_status emb_destroy(emb_t h);

/* ---- NEXT-1: unlimited-dictionary ids (stateless; no handle) ------------------------------
 * PAPER.md:335 ("QR hashing ... a collision-resistant hashing function like MurmurHash",
 * "sum aggregation worked the best") and PAPER.md:602 ("mapped with ... Murmur hashing to a
 * space of int64 ... bitcast to convert this int64 to two numbers in int32 space (ranging
 * from 0 to 2^32-1), B and C which will look from independent sets of QR tables").
 * All pointers are DEVICE pointers (EMB_EINVAL otherwise); the work is enqueued on `stream`
 * (a cudaStream_t, NULL = legacy default stream) and the call returns without waiting.
 *
 * emb_hash_ids: hashes[i] = h1 of MurmurHash3 x64-128, seed 0, of the UTF-8 bytes
 *   bytes[str_offsets[i] .. str_offsets[i+1]) (i < n; offsets non-decreasing, int64).
 *
 * emb_qr_expand: one QR feature's tables live in ONE table of emb_qr_rows(R, Q, dual) rows,
 *   concatenated [quotient_B: Q][remainder_B: R] (+ [quotient_C: Q][remainder_C: R] when
 *   dual).  With n = low 32 bits of hashes[i] and n' = high 32 bits (unsigned), id i becomes
 *   the rows (in this order) (n / R) mod Q, Q + n mod R [, Q+R + (n'/R) mod Q, 2Q+R + n' mod R]
 *   at ids_out[k*i ..], k = 2 (single) or 4 (dual), and offsets_out[b] = k * offsets[b]
 *   (b <= nbags).  Pooling the expanded bags with SUM (emb_forward) is the paper's sum
 *   aggregation; their gradients flow to exactly the expanded rows (emb_backward_adagrad).
 *   Requires 1 <= R, 1 <= Q and emb_qr_rows(R, Q, dual) < 2^31 (EMB_EINVAL otherwise);
 *   ids_out holds k*nnz int32, offsets_out nbags+1 int32. */
EMB_API emb_status emb_hash_ids(const uint8_t* bytes, const int64_t* str_offsets, int64_t n,
                                uint64_t* hashes, void* stream);
EMB_API emb_status emb_qr_expand(const uint64_t* hashes, const int32_t* offsets, int64_t nbags,
                                 int64_t nnz, int32_t R, int64_t Q, int32_t dual,
                                 int32_t* ids_out, int32_t* offsets_out, void* stream);
/* rows of one feature's concatenated QR table: (dual ? 2 : 1) * (Q + R) */
EMB_API int64_t emb_qr_rows(int32_t R, int64_t Q, int32_t dual);

#ifdef __cplusplus
}
#endif
#endif /* LIRANK_EMB_H */
