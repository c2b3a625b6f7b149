// kernels.cuh — device-side data structures shared between the host runtime
// (runtime.cu) and the sm_100a kernels (kernels.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace marsit_b200 {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;  // rng.hpp:64
constexpr uint32_t kMaxLocalWorkers = 64;           // workers resident on one rank
constexpr int kMaxCachedMerges = 32;                // merge descriptors staged in smem per stage
constexpr int kMergeThreads = 256;
constexpr uint32_t kMaxLanes = 8;                   // independent chains per stage run side by side                   // 8 warps; a warp tile is 32 x WPT packed
                                                     // words, WPT in {1, 2} chosen per context
constexpr int kStreamThreads = 256;                  // sign_extract / decode
constexpr int kTaskWords = 16;                       // u32 words per warp task (512 elements)

// Source of a merge operand (16-bit code): [15:14] kind, [13:0] index.
enum : uint16_t { kSrcLeaf = 0u << 14, kSrcSlot = 1u << 14, kSrcGlobal = 2u << 14 };
constexpr uint16_t kNone = 0xFFFF;
constexpr uint16_t kFinal = 0xFFFE;

// One merge of a segment's compiled DAG (merge.hpp:34-58 applied by the
// receiver of a reduce step, allreduce.hpp:183-185).
struct DevMerge {
    uint64_t thresh11;   // ceil(p * 2^53) << 11: coin <=> mix(..) < thresh11
    uint64_t key;        // explicit stream key (key_mode == 1)
    uint64_t base_add;   // draws the stream had produced before this round's merges
    uint32_t receiver;   // stream owner; key = K(seed, merge, receiver, t, segment)
    uint16_t recv_src, local_src;
    uint16_t out_slot;   // shared-memory slot for same-stage consumers, or kNone
    uint16_t out_global; // global node index, kFinal (aggregate) or kNone
    int16_t offset_src;  // previous merge of the same stream (draw continuation) or -1
    uint8_t key_mode;    // 0: derive key from (seed, round); 1: explicit `key`
    uint8_t pad_;
    uint32_t segment;    // global segment id (stream key)
    uint32_t coin_words; // coin-buffer capacity of this merge: draws [0, 32*coin_words)
    uint64_t coin_off;   // u32-word offset of those bits in the coin buffer
    uint32_t coin_default;  // words precomputed while the merge has no history
    uint32_t pad2_;
};
static_assert(sizeof(DevMerge) == 64, "DevMerge layout");


// Cooperative merge (kernels.cu, K2): the tiles of one launch are
// co-resident; one grid barrier per merge step of the current plan stage.
struct CoopParams {
    const DevMerge* merges;       // owned segments' merges, stage-sorted per segment
    const uint32_t* seg_begin;    // [n_seg] first merge of each owned segment
    // merge ranges per (segment, stage, lane): [n_seg][n_stages][kMaxLanes+1];
    // a lane is an independent chain of the stage (torus: one per row), run
    // by its own tiles, so independent chains share the grid barriers
    const uint32_t* lane_begin;
    uint32_t n_stages, stage, k_steps;  // k_steps: max merges of a lane of this stage
    uint32_t n_lanes;             // lanes of this stage (grid = seg_cnt x n_lanes x part_tiles)
    uint32_t n_seg, s_first, tiles_per_seg, words_proc, wst, ml, max_slots;
    uint32_t tile_words;          // words per tile (<= 256 * WPT, multiple of max(WPT, 4))
    uint32_t part, n_parts, part_tile0, part_tiles;  // tiles of each segment in this launch
    uint32_t seg_lo, seg_cnt;     // owned segments [seg_lo, seg_lo + seg_cnt) in this launch
    uint32_t n_merges;
    uint64_t seg_bits;            // L
    const uint32_t* leaves;       // leaf(w, sl) = leaves + ((w/ml*n_seg + sl)*ml + w%ml)*wst
    // P2P transport: leaf(w, sl) = peer_bits[w/ml] + ((s_first + sl)*ml + w%ml)*wst,
    // i.e. straight out of the source rank's own [S][ml][wst] buffer
    const uint32_t* const* peer_bits;
    uint32_t* gnodes;             // [n_seg][gmax][wst] nodes crossing stages
    uint32_t gmax;
    uint32_t* agg;                // [S][agg_stride]
    uint32_t agg_stride;          // u32 words per aggregate row
    const uint32_t* coins;        // precomputed coin bitstreams
    uint64_t* flags;              // [k_steps][CTAs] popcount of each tile
    uint64_t* part_totals;        // [n_parts][n_merges] draws consumed per (part, merge)
    uint64_t seed, round;
    // adaptive coin budget: words the coin kernel computed per merge (this
    // buffer), and the draw index each merge ended at (written by its last
    // tile; the next round's coin kernel sizes its work from it)
    const uint32_t* coin_valid;
    uint64_t* coin_end;
    unsigned* seg_bars;           // per-segment barrier counters [seg_cnt x n_lanes] or null (grid barrier)
    int* err;                     // checked builds: bounds latch (bit 3)
};
cudaError_t launch_merge_coop(const CoopParams& p, int wpt, size_t smem, cudaStream_t st);
cudaError_t merge_coop_occupancy(int wpt, size_t smem, int* blocks_per_sm);

// Cluster merge (kernels.cu, K2): one thread-block cluster of csize CTAs per
// owned segment runs the segment's whole merge DAG in one launch.  A CTA owns
// a contiguous tile of tile_groups 4-word groups of the segment; its
// kClusterThreads threads own groups u * kClusterThreads + tid (NSUB of
// them).  The merges run level by level (a level = up to NL independent
// merges); per level: popcount of r ^ l, one CTA scan, each CTA pushes its
// per-merge totals into every CTA's shared memory (DSMEM) and one cluster
// barrier gives every CTA its draw offset — no grid-wide barrier, no global
// flags.  DAG intermediates stay in shared memory (slots); leaves are read
// from the extract's packed signs (or a peer rank's, P2P); the final node
// goes to the aggregate.  Clusters never wait on each other, so segments
// beyond one wave of resident clusters simply run later.
constexpr int kClusterThreads = 1024;
constexpr int kMaxClusterSize = 16;  // non-portable cluster size
constexpr int kMaxLevelMerges = 2;
constexpr int kMaxSegMerges = 64;    // merges of one segment staged in shared memory
struct ClusterParams {
    const DevMerge* merges;       // owned segments' merges, level order per segment
    const uint32_t* seg_begin;    // [n_seg + 1] first merge of each owned segment
    const uint32_t* lvl_start;    // [n_seg + 1] first entry of each segment in lvl_begin
    const uint32_t* lvl_begin;    // per segment: n_levels + 1 merge offsets (within the segment)
    uint32_t n_seg, s_first, seg_lo;  // this launch: owned segments [seg_lo, seg_lo + clusters)
    uint32_t csize;               // CTAs per cluster
    uint32_t tile_groups;         // 4-word groups per CTA tile
    uint32_t words_proc, wst, ml, n_slots;
    uint32_t stage;               // 1: pass 1 stages r and d in shared memory for pass 2
    uint32_t masks;               // 1 (needs stage): the deposit masks of d formed during the
                                  // barrier, [NL][4][tile_groups] uint4 after the staging
    uint64_t seg_bits;            // L
    const uint32_t* leaves;       // leaf(w, sl) = leaves + ((w/ml*n_seg + sl)*ml + w%ml)*wst
    const uint32_t* const* peer_bits;  // P2P: leaf(w, sl) = peer_bits[w/ml] + ((s_first+sl)*ml + w%ml)*wst
    uint32_t* agg;                // [S][agg_stride]
    uint32_t agg_stride;
    const uint32_t* coins;        // precomputed coin bitstreams (null: every draw inline)
    const uint32_t* coin_valid;   // words computed per merge (null: none)
    uint64_t* totals;             // [n_merges] draws consumed by each merge
    uint64_t* coin_end;           // [n_merges] stream index after each merge (adaptive coins)
    uint64_t seed, round;
    int* err;                     // checked builds: bounds latch (bit 3)
    // grid mode (merge_grid_kernel): csize = CTAs ("tiles") per segment, any
    // number; the per-merge CTA totals go through global memory, xch
    // [2][segments of the launch][csize][NL]: each word carries its launch
    // and level tag, and polling all of a segment's words replaces the
    // cluster barrier
    unsigned long long* xch;      // word = level tag << 32 | CTA total
    uint32_t prefetch;            // >0: the next level's local leaf tiles are prefetched into L1
                                  // (1 after the masks, 2 before them, 3 after the totals)
    uint32_t xch_tag;             // per launch (host counter; the level is the low 8 bits)
    unsigned* seg_bars;
    uint32_t coin_l1;             // 1: the likely coin window of pass 2 is prefetched into L1
    uint32_t solo_nm, solo_nlv;   // n_seg == 1: the segment's merges and levels (0: read seg_begin / lvl_start)
    uint32_t grid_coop;           // grid merge: launched with the cooperative attribute
    uint32_t coherent;            // 1: leaves and coins were written by this launch (spread
                                  // round): L2-coherent loads, no L1 prefetch
};
cudaError_t launch_merge_cluster(const ClusterParams& p, int nsub, int nl, uint32_t clusters,
                                 size_t smem, cudaStream_t st);

// Fused small round (one launch, G == 1): one cluster per segment extracts
// its tile of every worker into shared memory (K1), runs the segment's merge
// DAG with the cluster merge's level loop (K2), and decodes + updates the
// compensation of its tile (K3/K4; the re-read of g and c is L2-resident at
// these sizes).  Needs every worker local, M <= kFusedMaxWorkers, 16-byte
// aligned quads (L % 4 == 0).
constexpr uint32_t kFusedMaxWorkers = 16;
// 512 threads per CTA (up to 128 registers each): 8 fp32 (4 fp64) quads of g
// and of c in flight per lane in the streaming phases
constexpr int kFusedThreads = 512;

template <typename T>
struct FusedParams {
    const T* g[kFusedMaxWorkers];
    const T* c[kFusedMaxWorkers];
    T* c_out[kFusedMaxWorkers];
    uint32_t workers;
    uint64_t dim;
    T eta;
    T* update;   // optional g_t
    int* err;    // non-finite latch
    // TMEM stash (spread round; 0: off): u = g + c of the CTA's slice is parked in
    // tensor memory between the extract and the decode, thread-private (warp
    // w owns lanes 32 (w % 4) .. + 31 and columns (w / 4) * stash_cols ..
    // + stash_cols), so the decode reads only the aggregate bits; tmem_cols =
    // the allocation (a power of 2 >= 32)
    uint32_t stash_cols, tmem_cols;
};
template <typename T>
cudaError_t launch_round_cluster(const ClusterParams& p, const FusedParams<T>& f, int nsub, int nl,
                                 uint32_t clusters, size_t smem, cudaStream_t st);
template <typename T>
cudaError_t round_cluster_occupancy(int nsub, int nl, uint32_t csize, size_t smem, int* clusters);
// Spread small round (one launch, G == 1): the fused round over every SM
// instead of one cluster per segment.  Each CTA streams an equal slice of the
// (segment, 128-coordinate group) space: this round's coin chunks, then K1
// for every worker with the packed signs to global memory (L2); after the
// last CTA arrives, cluster s < n_seg runs segment s's merge DAG with the
// cluster level loop (leaves and coins through L2) and publishes it; each CTA
// then decodes its own slice (K3/K4, the re-read of g and c L2-resident).
// The synchronisation words are device state only (a self-resetting arrival
// count + generation), so rounds can be replayed from a CUDA graph.
constexpr uint32_t kSpreadMaxMerges = 256;  // coin streams per spread round
constexpr uint32_t kSpreadMaxTmaStages = 4;  // extract ring stages (TMA path)
// Coins: two buffers b = round & 1, each tagged with the (seed, round) it
// holds.  Round t uses buffer t & 1 and computes it first only when its tag
// misses; while the merge clusters run, the other CTAs compute round t + 1's
// coins into the other buffer and tag it.  The budget of both reads the
// stream ends the previous launch's merges wrote (cend[(t & 1) ^ 1]; this
// launch writes cend[t & 1]), so every CTA sizes the same work.
template <typename T>
struct SpreadParams {
    FusedParams<T> f;
    unsigned* sync;                 // [0] arrivals, [1] generation, [2 + s] segment s merged (generation)
    uint32_t n_merges;              // coin streams of the round: p.merges[0 .. n_merges)
    uint32_t* coins[2];             // coin buffers
    uint32_t* coin_valid[2];        // [n_merges] words computed per buffer
    unsigned long long* tag;        // [2][2]: (seed, round) each buffer holds, ~0 = none
    unsigned long long* cend;       // [2][n_merges] stream ends by round parity
    // extract through TMA (0: register loads): stages of one worker's slice,
    // g then c, tma_half bytes each (the largest slice of any CTA)
    uint32_t tma_stages, tma_half;
};
template <typename T>
cudaError_t launch_round_spread(const ClusterParams& p, const SpreadParams<T>& s, int nsub, int nl,
                                uint32_t ctas, size_t smem, bool cooperative, cudaStream_t st);
template <typename T>
cudaError_t round_spread_occupancy(int nsub, int nl, uint32_t csize, size_t smem, int* clusters);
// Concurrently resident clusters of csize CTAs with `smem` dynamic bytes (0 if unsupported).
cudaError_t merge_cluster_occupancy(int nsub, int nl, uint32_t csize, size_t smem, int* clusters);
// K2g: the same level loop over csize co-resident CTAs per segment (any
// number, cooperative launch of `segments` x csize CTAs of kClusterThreads).
// grid merge CTA size: kClusterThreads, or 256 / 512 threads for tiles of at most that many groups
cudaError_t launch_merge_grid(const ClusterParams& p, int nsub, int nl, uint32_t segments, size_t smem,
                              int nt, cudaStream_t st);
cudaError_t merge_grid_occupancy(int nsub, int nl, size_t smem, int nt, int* blocks_per_sm);

template <typename T>
struct StreamParams {
    const T* g[kMaxLocalWorkers];
    const T* c[kMaxLocalWorkers];
    T* c_out[kMaxLocalWorkers];
    uint32_t ml, n_seg;          // local workers, segments (all S)
    uint32_t seg0, n_proc;       // this launch: segments [seg0, seg0 + n_proc)
    uint64_t dim, seg_len;       // D, L
    uint32_t words_proc, wst;
    // walk the warp tasks from the last to the first: the decode walks them
    // opposite to the same round's extract, so it starts on the coordinates
    // the extract read last (still in L2 across the merge); the direction
    // alternates by round so consecutive rounds never share a cache warm-up
    uint32_t reverse;
    uint32_t* bits;              // extract output: [S][ml][wst]
    const uint32_t* agg;         // decode input: [S][wsa]
    uint32_t wsa;                // aggregate row stride (u32 words)
    // P2P transport: segment s is read from its owner's buffer agg_peers[s / s_own]
    const uint32_t* const* agg_peers;
    uint32_t s_own;
    T* update;                   // optional g_t (written by local worker 0)
    T* x[kMaxLocalWorkers];      // optional replica parameters: x -= g_t (trainer.hpp:285-288)
    T eta;
    int* err;
    // decode only: when set, the decode also counts the coordinates whose
    // aggregate bit equals (mean of u over the n_workers workers >= 0)
    unsigned long long* matches;
    uint32_t n_workers;
};

// Launch wrappers (kernels.cu).
template <typename T>
cudaError_t launch_extract(const StreamParams<T>& p, bool vec, int grid, cudaStream_t st);
template <typename T>
cudaError_t launch_decode(const StreamParams<T>& p, bool vec, int grid, cudaStream_t st);
cudaError_t stream_occupancy(bool f64, int* extract_blocks, int* decode_blocks);
// Precompute the coin bits of every merge: bit n of merge m's stream is
// (mix(key_m + (n+1)γ) < thresh11_m) for n < 32 * coin_words.  Data
// independent, so it runs concurrently with the HBM-bound extract.
cudaError_t launch_coins(const DevMerge* merges, uint32_t n_merges, uint64_t seed, uint64_t round,
                         const uint64_t* coin_end, uint32_t* coin_valid,
                         uint32_t* coins, int grid_x, cudaStream_t st);
cudaError_t launch_export_bits(const uint32_t* agg, uint32_t wst, uint64_t dim, uint64_t seg_len,
                               uint32_t* out_u32, cudaStream_t st,
                               const uint32_t* const* agg_peers = nullptr, uint32_t s_own = 1);
// P2P epoch flags: after everything before it on the stream, a system-wide
// fence then slots[i] = value (peer memory stores; fallback when the driver's
// stream write on peer memory is unavailable).
struct FlagSlots {
    unsigned long long* slot[kMaxLocalWorkers];
    uint32_t n;
};
cudaError_t launch_flag_write(const FlagSlots& s, unsigned long long value, cudaStream_t st);
// Opt-in data consensus (allreduce.hpp:32-43 on the device): the hash of an
// aggregate segment s is the XOR over its words wi < words_proc of
// mix64(((u64)wi << 32 | word) + (s + 1) * gamma) (order independent).
// seg_hash XORs the hashes of segments [s0, s0 + n_seg) into out[s] (out
// non-null) or into the segment's own hash slot, the u64 after its wst words
// in the aggregate row (out null; the slot must be zero).  Rows are read from
// agg_peers[s / s_own] when given, else from agg.  hash_compare latches
// err |= 2 for every segment whose slot (the owner's hash, as read here)
// differs from verify[s].
cudaError_t launch_seg_hash(const uint32_t* agg, const uint32_t* const* agg_peers, uint32_t s_own,
                            uint32_t wsa, uint32_t wst, uint32_t words_proc, uint32_t s0,
                            uint32_t n_seg, unsigned long long* out, cudaStream_t st);
cudaError_t launch_hash_compare(const uint32_t* agg, const uint32_t* const* agg_peers,
                                uint32_t s_own, uint32_t wsa, uint32_t wst, uint32_t n_seg,
                                const unsigned long long* verify, int* err, cudaStream_t st);
// Loads every kernel of the library (instead of lazily at first launch).
cudaError_t preload_kernels();
// x_w -= v for the local workers' parameter replicas (dense-round update).
template <typename T>
cudaError_t launch_sub_update(T* const* x, uint32_t ml, const T* v, uint64_t dim, int grid,
                              cudaStream_t st);
template <typename T>
cudaError_t launch_fill_recipe(int recipe, uint64_t seed, uint64_t worker, uint64_t round,
                               uint64_t dim, T* out, cudaStream_t st);

// Dense round (allreduce_dense, allreduce.hpp:98-130): per coordinate, the
// schedule's reduction tree of u = g + c evaluated in double.
struct DenseOp {
    uint16_t a, b;     // operand node ids (leaf w < M, else M + k)
    uint16_t pad0, pad1;
};
template <typename T>
struct DenseParams {
    const T* src[kMaxLocalWorkers * 2];  // leaves: g,c pairs (1 GPU) or exchanged u (multi)
    uint32_t mode;                       // 0: leaf w = g[w] + c[w]; 1: leaf w = u buffer
    const T* u_buf;                      // mode 1: [G][s_own][ml][L] u values
    const T* const* u_peers;             // mode 2 (P2P): rank q's own [S][ml][L] u buffer
    bool vec4;                           // mode 0 chain: 16-byte aligned quads throughout
    const uint16_t* chain;               // chain-of-chains plans: [n_seg][workers] leaf order
                                         // (null: general DAG)
    const uint64_t* chain_groups;        // [n_seg]: bit k set = a group chain ends at leaf k
    bool chain_multi;                    // some segment has more than one group (torus)
    T* c_zero[kMaxLocalWorkers];         // compensation reset c' = 0 fused into the pass
                                         // that reads g, c (sync.hpp:83-85); may alias c
    const DenseOp* ops;                  // [n_seg][n_ops]
    const uint16_t* final_node;          // [n_seg]
    uint32_t n_ops, n_seg, s_first, ml, workers;
    uint64_t dim, seg_len;
    double inv_m;
    T* mean;                              // [D] (full vector; owned segments written)
    int* err;
};
template <typename T>
cudaError_t launch_dense_reduce(const DenseParams<T>& p, int grid, cudaStream_t st);
template <typename T>
cudaError_t launch_dense_leaf(const T* const* g, const T* const* c, uint32_t ml, uint64_t dim,
                              uint64_t seg_len, uint32_t n_seg_total, uint32_t s_own,
                              T* u_send, int* err, int grid, cudaStream_t st,
                              T* const* c_zero = nullptr);

}  // namespace marsit_b200
