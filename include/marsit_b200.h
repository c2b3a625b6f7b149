/*
 * marsit_b200.h — C-ABI of the B200-native Marsit sign-round path.
 *
 * This is the drop-in boundary for the reference's synchronisation path
 * (/root/reference/proj/include/marsit/, header-only C++20).  The reference
 * has no FFI; its public interface is a set of C++ functions, each of which
 * an entry point below replaces (file:line cited per function).  The C++
 * shim in include/marsit_b200/drop_in.hpp re-exposes the reference's exact
 * C++ signatures on top of this ABI; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "d_" pointers are CUDA device pointers,
 *    everything else is host memory.  `stream` is a cudaStream_t (NULL = the
 *    legacy default stream).
 *  - Every entry point returns a marsit_status; on failure the thread-local
 *    message is available from marsit_last_error().  Status codes map 1:1 to
 *    the reference exception taxonomy (errors.hpp:10-42).
 *  - Round entry points are asynchronous on `stream`.  Data-dependent errors
 *    that the reference raises mid-round (non_finite_error from
 *    DenseVector's constructor, dense_vector.hpp:25-29) are latched on the
 *    device and reported by marsit_ctx_check() (which synchronises the
 *    stream).  Validation errors are returned immediately.
 *  - One host thread per context; no global mutable state.
 *  - There is no CPU fallback: without a CUDA device every compute entry
 *    point returns MARSIT_ECUDA.
 */
#ifndef MARSIT_B200_H
#define MARSIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MARSIT_B200_ABI_VERSION 3

typedef enum marsit_status {
    MARSIT_OK = 0,
    MARSIT_EPARAM = 1,       /* marsit::parameter_error   errors.hpp:11-14 */
    MARSIT_ENONFINITE = 2,   /* marsit::non_finite_error  errors.hpp:19-22 */
    MARSIT_EPROTOCOL = 3,    /* marsit::protocol_error    errors.hpp:26-29 */
    MARSIT_EUNSUPPORTED = 4, /* marsit::unsupported_error errors.hpp:33-36 */
    MARSIT_ECUDA = 5,        /* CUDA runtime failure / no device        */
    MARSIT_ENCCL = 6         /* NCCL failure (multi-GPU contexts)       */
} marsit_status;

typedef enum marsit_dtype { MARSIT_F32 = 0, MARSIT_F64 = 1 } marsit_dtype;

/* schedule.hpp:12 Phase */
typedef enum marsit_phase { MARSIT_REDUCE = 0, MARSIT_GATHER = 1 } marsit_phase;

/* ------------------------------------------------------------------------
 * Schedules (host objects).  Replace marsit::Schedule and its builders.
 * ---------------------------------------------------------------------- */
typedef struct marsit_schedule marsit_schedule;

/* build_ring_schedule (schedule.hpp:61-94): m >= 2 else EPARAM. */
marsit_status marsit_schedule_ring(uint32_t m, marsit_schedule** out);
/* build_torus_schedule (schedule.hpp:110-196): rows, cols >= 2 else EPARAM. */
marsit_status marsit_schedule_torus(uint32_t rows, uint32_t cols, marsit_schedule** out);
/* An arbitrary Schedule given as flat tables (phase[steps];
 * send_to/recv_from/segment[steps*workers]); validated like
 * Schedule::validate (schedule.hpp:38-54) -> EPROTOCOL. */
marsit_status marsit_schedule_from_tables(uint32_t workers, uint32_t segments, uint32_t steps,
                                          const uint8_t* phase, const uint32_t* send_to,
                                          const uint32_t* recv_from, const uint32_t* segment,
                                          marsit_schedule** out);
marsit_status marsit_schedule_info(const marsit_schedule* s, uint32_t* workers,
                                   uint32_t* segments, uint32_t* steps);
marsit_status marsit_schedule_tables(const marsit_schedule* s, uint8_t* phase,
                                     uint32_t* send_to, uint32_t* recv_from, uint32_t* segment);
void marsit_schedule_destroy(marsit_schedule* s);

/* The compiled merge plan of one segment (host introspection, no device
 * needed).  Node ids 0..workers-1 are the workers' own packed segments;
 * node workers+k is the output of merge k.  offset_src is the index of the
 * previous merge of the same (receiver, segment) stream, whose draws this
 * merge continues (allreduce.hpp:167-177), or -1. */
typedef struct marsit_merge_info {
    uint32_t recv_node, local_node, receiver, c_recv, c_local;
    int32_t offset_src;
    uint32_t stage;
} marsit_merge_info;
marsit_status marsit_schedule_plan(const marsit_schedule* s, uint32_t segment,
                                   uint32_t capacity, marsit_merge_info* merges,
                                   uint32_t* n_merges, uint32_t* final_node,
                                   uint32_t* final_count);

/* ------------------------------------------------------------------------
 * Contexts.  A context binds (D, schedule, dtype, device, rank layout) and
 * owns all device scratch: per-segment packed-sign buffers, the compiled
 * merge plan, look-back flags, the NCCL communicator.
 * ---------------------------------------------------------------------- */
typedef struct marsit_ctx marsit_ctx;

/* How the packed segments move between ranks (nranks > 1).  The zero value
 * (the default of a zero-initialised descriptor) is the P2P transport, the
 * one exercised end to end across processes by the test suite; NCCL is
 * opt-in (see DESIGN.md section 5 for what has run on hardware). */
typedef enum marsit_transport {
    MARSIT_TRANSPORT_P2P = 0,       /* fused over peer memory (marsit_ctx_set_peers) */
    MARSIT_TRANSPORT_EXTERNAL = 1,  /* the caller moves the blocks between phases   */
    MARSIT_TRANSPORT_NCCL = 2       /* built in: grouped send/recv + all-gather     */
} marsit_transport;

typedef struct marsit_ctx_desc {
    uint64_t dim;                     /* D >= 1                                   */
    const marsit_schedule* schedule;  /* M workers, M segments                    */
    marsit_dtype dtype;               /* element type of grads / compensation      */
    int device;                       /* CUDA device ordinal                       */
    uint32_t nranks;                  /* processes sharing the M workers (>= 1)    */
    uint32_t rank;                    /* this process: workers [rank*M/nranks, ..) */
    const void* nccl_id;              /* 128-byte ncclUniqueId (NCCL, nranks > 1) */
    marsit_transport transport;
} marsit_ctx_desc;

marsit_status marsit_ctx_create(const marsit_ctx_desc* desc, marsit_ctx** out);
void marsit_ctx_destroy(marsit_ctx* ctx);
/* The worker ids resident on this rank: [*first, *first + *count). */
marsit_status marsit_ctx_local_workers(const marsit_ctx* ctx, uint32_t* first, uint32_t* count);

/* Sign round: the sign branch of marsit_round (sync.hpp:60-120, 91-118).
 *  d_grads[i], d_comp[i]: the i-th LOCAL worker's scaled gradient and
 *    compensation (D elements of dtype).
 *  d_comp_out[i]: receives c' = (g + c) - g_t; may equal d_comp[i] (in place).
 *  d_agg_bits (optional): aggregate_bits in the reference layout, ceil(D/64)
 *    little-endian u64 words, truncated to D (sync.hpp:103-112).
 *  d_update (optional): global_update g_t = +-eta_s (D elements of dtype). */
marsit_status marsit_sign_round(marsit_ctx* ctx, uint64_t t, double eta_s, uint64_t global_seed,
                                const void* const* d_grads, const void* const* d_comp,
                                void* const* d_comp_out, uint64_t* d_agg_bits, void* d_update,
                                void* stream);

/* Dense round (sync.hpp:78-87 -> allreduce_dense, allreduce.hpp:98-130):
 * d_mean = mean of (g + c) summed in schedule order; d_comp_out set to 0. */
marsit_status marsit_dense_round(marsit_ctx* ctx, uint64_t t, const void* const* d_grads,
                                 const void* const* d_comp, void* const* d_comp_out, void* d_mean,
                                 void* stream);

/* marsit_round (sync.hpp:60-120): dense iff period != 0 && t % period == 0,
 * else sign.  period == 0 means "never" (SyncConfig with no K).  d_update
 * receives g_t for both kinds of round (required for dense rounds).
 * *full_precision (optional, host) reports which branch ran. */
marsit_status marsit_round(marsit_ctx* ctx, uint64_t t, uint64_t period, double eta_s,
                           uint64_t global_seed, const void* const* d_grads,
                           const void* const* d_comp, void* const* d_comp_out,
                           uint64_t* d_agg_bits, void* d_update, int* full_precision,
                           void* stream);

/* allreduce_sign (allreduce.hpp:148-189) on already packed signs.
 *  d_signs: the LOCAL workers' packed segments, [local worker][segment][ceil(L/64)] u64
 *    with L = ceil(D/M) (the reference's PackedSignVector words).
 *  d_out: the consensus aggregate, [segment][ceil(L/64)] u64.
 *  counts (optional, host): [segment] contribution counts (all M for ring/torus). */
marsit_status marsit_allreduce_sign(marsit_ctx* ctx, uint64_t round, uint64_t global_seed,
                                    const uint64_t* d_signs, uint64_t* d_out, uint32_t* counts,
                                    void* stream);

/* External transport (or manual staging): a round split at its two exchange
 * points.  phase 0: sign extraction (or, for a dense round, u = g + c per
 * destination); the caller then moves block q of layout.send to rank q's
 * layout.recv (block r of recv comes from rank r).  phase 1: merge (dense:
 * sum) of this rank's owned segments into its own block of layout.gather;
 * the caller all-gathers the gather blocks.  phase 2: decode + compensation
 * (dense: mean out, compensation = 0).  Arguments as marsit_round. */
typedef struct marsit_exchange_layout {
    void* send;
    void* recv;
    uint64_t block_bytes;         /* per destination / source rank              */
    void* gather;
    uint64_t gather_block_bytes;  /* this rank's block is at rank*gather_block_bytes */
} marsit_exchange_layout;
marsit_status marsit_ctx_exchange_layout(const marsit_ctx* ctx, int dense,
                                         marsit_exchange_layout* out);
marsit_status marsit_round_phase(marsit_ctx* ctx, int phase, uint64_t t, uint64_t period,
                                 double eta_s, uint64_t global_seed, const void* const* d_grads,
                                 const void* const* d_comp, void* const* d_comp_out,
                                 uint64_t* d_agg_bits, void* d_update, int* full_precision,
                                 void* stream);

/* P2P transport (NVLink / NVSwitch peer memory, one process per GPU): no
 * exchange or all-gather phase.  The merge kernel reads its leaves straight
 * out of the peer ranks' packed-sign buffers and the decode reads every
 * aggregate segment from the rank that owns it; the dense round's owner sum
 * reads the peers' u blocks the same way.  Ordering is stream-ordered: after
 * each producing phase the stream writes this rank's epoch into its slot of
 * every peer's flag array, and before each consuming phase it waits
 * (cuStreamWaitValue64, on local memory) until every peer's slot reaches the
 * epoch — no kernel ever waits on another.  Every rank runs the same
 * sequence of rounds.
 * Setup: export this rank's buffers (marsit_ctx_p2p_buffers), map the peers'
 * (marsit_ipc_handle / marsit_ipc_open across processes), hand the table of
 * all ranks' mapped buffers (indexed by rank) to marsit_ctx_set_peers.
 * marsit_round_phase splits a round at the same points (0: extract + flag,
 * 1: wait + merge + flag, 2: wait + decode). */
typedef struct marsit_p2p_buffers {
    void* bits;        /* packed signs [S][local workers][words]          */
    void* agg;         /* aggregate bits [S][words] (owned segments)      */
    void* dense_send;  /* dense round: u [S][local workers][L]            */
    void* dense_mean;  /* dense round: mean [S * L] (owned segments)      */
    void* flags;       /* [2][nranks] u64 epochs reported by each rank   */
} marsit_p2p_buffers;
marsit_status marsit_ctx_p2p_buffers(const marsit_ctx* ctx, marsit_p2p_buffers* out);
marsit_status marsit_ctx_set_peers(marsit_ctx* ctx, const marsit_p2p_buffers* peers,
                                   uint32_t nranks);
/* CUDA IPC of one device allocation (64-byte handle) for the peer table. */
marsit_status marsit_ipc_handle(const void* d_ptr, void* handle_out);
marsit_status marsit_ipc_open(const void* handle, int device, void** d_ptr_out);
marsit_status marsit_ipc_close(void* d_ptr);

/* Error-compensated sign extraction alone (sync.hpp:71-76 + segmentation.hpp:32-53
 * + sign_vector.hpp:67-73): d_signs_out as in marsit_allreduce_sign's input. */
marsit_status marsit_sign_extract(marsit_ctx* ctx, const void* const* d_grads,
                                  const void* const* d_comp, uint64_t* d_signs_out,
                                  void* stream);

/* One merge_signs (merge.hpp:34-58) on the device, synchronous.  `key` is the
 * stream's constructor state (rng.hpp:30-38), `used` the draws it has already
 * produced; *consumed (host) receives the draws this merge consumed. */
marsit_status marsit_merge_signs(const uint64_t* d_recv, uint32_t c_recv, const uint64_t* d_local,
                                 uint32_t c_local, uint64_t len, uint64_t key, uint64_t used,
                                 uint64_t* d_out, uint64_t* consumed, int device, void* stream);

/* BitsAccount of one round (bits_account.hpp:15-40; allreduce.hpp:113, 182).
 * per_worker: [M] (optional). */
marsit_status marsit_bits_account(const marsit_ctx* ctx, int dense, uint64_t* per_worker,
                                  uint64_t* reduce_bits, uint64_t* gather_bits, uint64_t* total);

/* Synchronise `stream` and report latched device errors (non-finite values,
 * missing contributions).  Clears the latch. */
marsit_status marsit_ctx_check(marsit_ctx* ctx, void* stream);

/* Failure handling of multi-rank contexts (P2P, NCCL).  Every round enqueued
 * on such a context is watched by a host thread: if it has not completed
 * within the timeout (default 120000 ms, env MARSIT_WAIT_TIMEOUT_MS; 0 =
 * unbounded), if NCCL reports an asynchronous error (ncclCommGetAsyncError),
 * or if a peer announced an abort, the context is marked failed — P2P stream
 * waits are released (this rank's flags and its slots in the peers' flags are
 * set to the abort value, so the peers fail too instead of hanging), an NCCL
 * communicator is aborted — and every later call returns the latched status:
 * MARSIT_EPROTOCOL (a broken wire, protocol_error, errors.hpp:24-29) or
 * MARSIT_ENCCL.  marsit_ctx_status returns the latched status without
 * synchronising; marsit_ctx_check returns it after synchronising. */
marsit_status marsit_ctx_set_wait_timeout(marsit_ctx* ctx, uint64_t timeout_ms);
marsit_status marsit_ctx_status(const marsit_ctx* ctx);

/* Opt-in data consensus (consensus(), allreduce.hpp:32-43, called by
 * marsit_round at sync.hpp:101): after its merge every owner hashes its
 * aggregate segments (64-bit, order-independent XOR of SplitMix64 word
 * hashes) into a slot that travels with the segment; after the decode every
 * rank re-hashes all S segments as it reads them and compares.  A mismatch
 * is latched and reported by marsit_ctx_check as MARSIT_EPROTOCOL
 * ("consensus").  Off by default (two small kernels per round). */
marsit_status marsit_ctx_set_consensus(marsit_ctx* ctx, int enable);

/* Per-phase device timing (CUDA events on the launching stream).
 * Phases: 0 sign_extract, 1 exchange, 2 merge, 3 allgather, 4 decode_comp,
 * 5 export, 6 dense, 7 coins (coin precompute, on the context's side stream,
 * overlapping phase 0), 8 fused_round (small rounds: extract + merge + decode
 * in one cluster launch per segment), 9 spread_round (small rounds: coins,
 * extract, merge and decode in one launch over every SM).  ms[i]
 * accumulates; launches[i] counts kernel launches. */
#define MARSIT_N_PHASES 10
marsit_status marsit_ctx_set_timing(marsit_ctx* ctx, int enable);
marsit_status marsit_ctx_timing(marsit_ctx* ctx, float* ms, uint64_t* launches, int reset);

/* On-device round metrics.  Replaces the trainer's
 * per-round figures: matching_rate (analysis.hpp:244-253 against the mean of
 * u_w = g_w + c_w, trainer.hpp:241-251, 280-281), the round's BitsAccount
 * (bits_account.hpp:15-40) and the merge disagreement counters (coins drawn,
 * merge.hpp:44-53).  When enabled, the decode kernel forms the fp64 mean of u
 * over the workers and counts matches in the same pass (no extra HBM
 * traffic); the merge kernel's per-merge draw totals give the disagreements.
 * Matching needs every worker of the job on this context (G == 1); with an
 * NCCL communicator the disagreement counters are summed over the ranks
 * (marsit_ctx_metrics is then collective); with the external transport they
 * cover this rank's owned segments (rank_local = 1). */
typedef struct marsit_round_metrics {
    uint64_t round;             /* t of the last round run on the context */
    int32_t valid;              /* 0: no round has run yet */
    int32_t full_precision;     /* 1: the last round was dense (no sign metrics) */
    int32_t has_matching;       /* 1: matches / matching_rate are set */
    int32_t rank_local;         /* 1: disagreement counters cover this rank only */
    uint64_t dim;
    uint64_t matches;           /* coordinates with bit == (mean(u) >= 0) */
    double matching_rate;       /* matches / dim */
    uint64_t merges;            /* merges evaluated (one per reduce delivery) */
    uint64_t compared_bits;     /* merges * L */
    uint64_t disagreements;     /* coins drawn = sum over merges of popcount(r ^ l) */
    double disagreement_rate;   /* disagreements / compared_bits */
    uint64_t round_bits;        /* BitsAccount total of the last round */
} marsit_round_metrics;
marsit_status marsit_ctx_set_metrics(marsit_ctx* ctx, int enable);
/* Waits for `stream`, then reports the last round's metrics. */
marsit_status marsit_ctx_metrics(marsit_ctx* ctx, marsit_round_metrics* out, void* stream);

/* ------------------------------------------------------------------------
 * SSDM baseline collectives (the paper's comparison points).
 *   marsit_ssdm_compress   = ssdm_compress (ssdm.hpp:29-40) of one vector with
 *                            RngStream(seed, ssdm, worker, round, segment);
 *                            d_bits: ceil(len/64) u64 words; *norm_out on the
 *                            host (synchronises `stream`)
 *   marsit_ssdm_decompress = ssdm_decompress (ssdm.hpp:44-56)
 *   marsit_ssdm_allreduce  = cascading_allreduce (allreduce.hpp:205-262, mode
 *                            MARSIT_SSDM_CASCADING) or sum_ssdm_allreduce
 *                            (275-339, MARSIT_SSDM_SUM) over the context's
 *                            schedule: d_vectors[w] = worker w's D elements,
 *                            d_estimate = the D-element estimate every worker
 *                            ends with.  Ring schedules only
 *                            (MARSIT_EUNSUPPORTED otherwise, as the reference);
 *                            every worker on this context (G == 1).  The
 *                            BitsAccount outputs and max_abs_per_step[steps]
 *                            (sum mode) are optional host outputs; asking for
 *                            them in sum mode synchronises `stream`.
 * The l2 norm is summed in a fixed parallel order: equal to the reference's
 * sequential sum whenever that sum is exact, within a few ulps otherwise.
 * ---------------------------------------------------------------------- */
typedef enum marsit_ssdm_mode { MARSIT_SSDM_CASCADING = 0, MARSIT_SSDM_SUM = 1 } marsit_ssdm_mode;
marsit_status marsit_ssdm_compress(const void* d_v, uint64_t len, marsit_dtype dtype, uint64_t seed,
                                   uint64_t worker, uint64_t round, uint64_t segment,
                                   uint64_t* d_bits, double* norm_out, void* stream);
marsit_status marsit_ssdm_decompress(const uint64_t* d_bits, uint64_t len, double norm,
                                     marsit_dtype dtype, void* d_out, void* stream);
marsit_status marsit_ssdm_allreduce(marsit_ctx* ctx, int mode, uint64_t round, uint64_t seed,
                                    const void* const* d_vectors, void* d_estimate,
                                    uint64_t* bits_per_worker, uint64_t* reduce_bits,
                                    uint64_t* gather_bits, int64_t* max_abs_per_step,
                                    void* stream);

/* Synthetic input recipes generated on the device:
 * recipe 0 = dyadic, 1 = correlated.  d_out: D elements of dtype. */
marsit_status marsit_fill_recipe(int recipe, uint64_t seed, uint64_t worker, uint64_t round,
                                 uint64_t dim, marsit_dtype dtype, void* d_out, void* stream);

/* ------------------------------------------------------------------------
 * Multi-step sync driver: the per-round synchronisation part of the
 * reference trainer (trainer.hpp:184-307, Alg. 2) around marsit_round —
 * compensation state owned on the device and carried across rounds
 * (trainer.hpp:252), the round counter t, the dense cadence K, the identical
 * parameter update x_w -= g_t on every replica fused into the decode
 * (trainer.hpp:285-288), cumulative payload bits (trainer.hpp:278-279), and
 * bucketing for large models.
 *
 * Buckets: coordinates [b*bucket_elems, min((b+1)*bucket_elems, D)) form an
 * independent marsit_round with global seed
 *     seed_b = seed                                   if there is one bucket
 *     seed_b = mix(seed ^ ((b + 1) * 0x9e3779b97f4a7c15))  otherwise
 * where mix is the SplitMix64 finalizer of rng.hpp:66-70.  The reference
 * reproduces a bucketed round bucket by bucket with marsit_round(t, cfg,
 * grads[b], comp[b], sched, seed_b).
 * ---------------------------------------------------------------------- */
typedef struct marsit_driver marsit_driver;

typedef struct marsit_driver_desc {
    uint64_t dim;                     /* D                                         */
    const marsit_schedule* schedule;  /* M workers                                 */
    marsit_dtype dtype;
    int device;
    uint32_t nranks, rank;            /* as marsit_ctx_desc                        */
    const void* nccl_id;
    uint64_t bucket_elems;            /* 0 = one bucket of D                       */
    uint64_t period;                  /* K: dense every K-th round; 0 = never      */
    double eta_s;                     /* > 0                                       */
    uint64_t global_seed;
    uint64_t first_round;             /* t of the first step (trainer starts at 0) */
    marsit_transport transport;       /* nranks > 1: P2P (default) or NCCL         */
} marsit_driver_desc;

marsit_status marsit_driver_create(const marsit_driver_desc* desc, marsit_driver** out);
void marsit_driver_destroy(marsit_driver* drv);
/* One round t (then t += 1): d_grads[i] = local worker i's scaled gradient
 * (D elements).  d_params (optional): replica parameters, x -= g_t.
 * d_update (optional): receives g_t.  *full_precision (optional). */
marsit_status marsit_driver_step(marsit_driver* drv, const void* const* d_grads,
                                 void* const* d_params, void* d_update, int* full_precision,
                                 void* stream);
/* Device pointer to local worker i's compensation (D elements). */
marsit_status marsit_driver_compensation(marsit_driver* drv, uint32_t local_worker, void** d_comp);
/* Next round index, cumulative payload bits, number of buckets. */
marsit_status marsit_driver_state(const marsit_driver* drv, uint64_t* next_round,
                                  uint64_t* cum_bits, uint32_t* n_buckets);
/* Checkpoint / resume of the sync state (t, cumulative bits, every local
 * worker's compensation) — state the reference's params-only checkpoint
 * (checkpoint.hpp:18-91) does not keep.  Synchronises `stream`. */
marsit_status marsit_driver_save(marsit_driver* drv, const char* path, void* stream);
marsit_status marsit_driver_load(marsit_driver* drv, const char* path, void* stream);
/* P2P transport (desc.transport = MARSIT_TRANSPORT_P2P): every bucket owns a
 * context whose buffers the ranks exchange as for marsit_ctx_set_peers, once
 * per bucket, before the first step. */
marsit_status marsit_driver_p2p_buffers(const marsit_driver* drv, uint32_t bucket,
                                        marsit_p2p_buffers* out);
marsit_status marsit_driver_set_peers(marsit_driver* drv, uint32_t bucket,
                                      const marsit_p2p_buffers* peers, uint32_t nranks);
/* marsit_ctx_set_wait_timeout / marsit_ctx_set_consensus on every bucket. */
marsit_status marsit_driver_set_wait_timeout(marsit_driver* drv, uint64_t timeout_ms);
marsit_status marsit_driver_set_consensus(marsit_driver* drv, int enable);
/* Round metrics of the last step summed over the buckets (matching over all D
 * coordinates, as trainer.hpp:280-281 records it per round). */
marsit_status marsit_driver_set_metrics(marsit_driver* drv, int enable);
marsit_status marsit_driver_metrics(marsit_driver* drv, marsit_round_metrics* out, void* stream);

/* Parameters in the reference's checkpoint format (checkpoint.hpp:18-91:
 * "marsit-ckpt\0", u32 version 1, u64 D, D little-endian doubles), from / to
 * a device vector of dtype. */
marsit_status marsit_write_params_checkpoint(const char* path, const void* d_params, uint64_t dim,
                                             marsit_dtype dtype, void* stream);
marsit_status marsit_read_params_checkpoint(const char* path, void* d_params, uint64_t dim,
                                            marsit_dtype dtype, void* stream);

/* ncclGetUniqueId for multi-rank contexts (128 bytes). */
marsit_status marsit_nccl_unique_id(void* out128);

const char* marsit_last_error(void);
int marsit_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MARSIT_B200_H */
