// internal.hpp — private runtime structures shared by runtime.cu (the
// C-ABI) and driver.cu (the multi-step sync driver).  Not installed.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/marsit_b200.h"
#include "kernels.cuh"
#include "plan.hpp"

struct marsit_schedule {
    marsit_b200::HostSchedule s;
    marsit_b200::Plan plan;
};

namespace marsit_b200 {

// Record the thread-local error message and return the status.
marsit_status fail(marsit_status st, const std::string& msg);


#define CUDA_TRY(expr)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(MARSIT_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define NCCL_TRY(expr)                                                                      \
    do {                                                                                    \
        ncclResult_t r_ = (expr);                                                           \
        if (r_ != ncclSuccess)                                                              \
            return fail(MARSIT_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
    } while (0)

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
inline uint64_t round_up(uint64_t a, uint64_t b) { return ceil_div(a, b) * b; }

inline int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

inline bool have_device() {
    int n = 0;
    return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
}

// Device-side plan of the merge DAGs (see DevMerge in kernels.cuh).
struct DevicePlan {
    std::vector<DevMerge> merges;
    std::vector<uint32_t> seg_begin, stage_begin;
    // [n_seg][n_stages][kMaxLanes+1] merge offsets (within the segment) of
    // each lane; n_lanes[stage] = lanes of the stage (max over segments)
    std::vector<uint32_t> lane_begin, n_lanes;
    uint32_t max_slots = 0, gmax = 0, n_stages = 1, n_merges = 0;
    // cluster plans (lower_cluster_plan): per owned segment the merges in
    // level order; lvl_begin holds each segment's level offsets (n_levels + 1
    // entries starting at lvl_start[sl]); seg_begin has n_seg + 1 entries
    std::vector<uint32_t> lvl_start, lvl_begin;
    uint32_t level_width = 1;  // most merges in one level
    // one lane per stage (plans built without the lane analysis)
    void single_lanes() {
        const size_t n_seg = seg_begin.size();
        lane_begin.assign(n_seg * n_stages * (kMaxLanes + 1), 0);
        n_lanes.assign(n_stages, 1);
        for (size_t sl = 0; sl < n_seg; ++sl)
            for (uint32_t st = 0; st < n_stages; ++st)
                for (uint32_t ln = 0; ln <= kMaxLanes; ++ln)
                    lane_begin[(sl * n_stages + st) * (kMaxLanes + 1) + ln] =
                        stage_begin[sl * (n_stages + 1) + st + (ln > 0 ? 1 : 0)];
    }
};

// Lower the owned segments' merge DAGs into the device plan (runtime.cu).
marsit_status lower_plan(const Plan& plan, uint32_t s_first, uint32_t n_seg, DevicePlan& dp);
// The same for the cluster merge: levels of independent merges, shared-memory slots.
marsit_status lower_cluster_plan(const Plan& plan, uint32_t s_first, uint32_t n_seg, DevicePlan& dp);

// The cooperative merge of a set of owned segments (K2).  Chooses the words
// per thread and splits each segment's tiles into parts so that one launch's
// tiles are co-resident; launches stage x part.
struct MergeRunner {
    DevicePlan dp;
    uint32_t n_seg = 0, s_first = 0, words_proc = 0, wst = 0, ml = 0, agg_stride = 0;
    uint64_t L = 0;
    int wpt = 1;
    size_t smem = 0;
    uint32_t seg_per_launch = 1;  // owned segments per cooperative launch
    uint32_t tiles_per_seg = 0, part_tiles = 0, n_parts = 1, tile_words = 0;
    std::vector<uint32_t> k_steps;  // per stage: max merges over segments
    DevMerge* d_merges = nullptr;
    uint32_t* d_seg_begin = nullptr;
    uint32_t* d_stage_begin = nullptr;  // the lane table (DevicePlan::lane_begin)
    uint32_t lanes_max = 1;
    uint32_t* gnodes = nullptr;
    uint64_t* flags = nullptr;  // [kmax][seg_per_launch * part_tiles]
    uint64_t* part_totals = nullptr;
    uint64_t* coin_end = nullptr;  // [n_merges] last round's end draw index per merge (~0: none)
    unsigned* seg_bars = nullptr;  // per-(segment, lane) barrier words (MARSIT_SEG_BARRIER)
    bool seg_barrier = env_int("MARSIT_SEG_BARRIER", 1) != 0;
    const uint32_t* const* peer_bits = nullptr;  // P2P transport: device table [G]
    int* err = nullptr;                          // the context's error latch (checked builds)
    // Merge kernel, MARSIT_MERGE_KERNEL:
    //   grid (default): the level loop over any number of co-resident
    //     1024-thread CTAs per segment (cooperative launch, tagged global
    //     totals; K2g) on the cluster plan;
    //   cluster: the same loop on one thread-block cluster per segment (DSMEM
    //     totals; K2c);
    //   coop: the cooperative stage/part merge (K2), also the fallback when
    //     the grid merge's tiles do not fit.
    bool cluster = [] {
        const char* e = std::getenv("MARSIT_MERGE_KERNEL");
        return !e || std::strcmp(e, "cluster") == 0 || std::strcmp(e, "grid") == 0;
    }();
    bool grid = [] {
        const char* e = std::getenv("MARSIT_MERGE_KERNEL");
        return !e || std::strcmp(e, "grid") == 0;
    }();
    unsigned long long* xch = nullptr;  // grid mode: [2][seg_per_launch][csize][level_width]
    uint32_t xch_epoch = 0;             // grid mode: launches so far (the words' launch tag)
    uint32_t grid_nt = kClusterThreads;  // grid mode: threads per CTA (256 / 512 for small tiles)
    uint32_t prefetch = uint32_t(env_int("MARSIT_MERGE_PREFETCH", 1));  // level loop: next leaves into L1
    // level loop, opt-in (MARSIT_COIN_L1=1): the likely coin window of pass 2
    // prefetched into L1 during the exchange.  Measured: C2 merge 101 -> 98
    // us, C4 98.6 -> 99.6, G = 8 rank 28.6 -> 30.7, G = 2 34.2 -> 36.4; the
    // C2 / C4 / C5 rounds unchanged within noise — off by default
    uint32_t coin_l1 = uint32_t(env_int("MARSIT_COIN_L1", 0) != 0);
    uint32_t grid_coop = uint32_t(env_int("MARSIT_GRID_COOP", 1) != 0);  // grid merge: cooperative attribute
    uint32_t csize = 16, tile_groups = 0, nsub = 1, stage = 0, masks = 0;
    size_t merge_smem = 0;  // merge_cluster_kernel's dynamic shared memory (smem minus the fused ring)
    // fused small rounds (round_cluster_kernel): extra shared memory per CTA
    // for every worker's packed tile + the aggregate; 0 = merge only
    uint32_t fused_arrays = 0;
    int fused_dtype = -1;  // element type of the fused kernel's occupancy query (0 f32, 1 f64)
    uint32_t* d_lvl_start = nullptr;
    uint32_t* d_lvl_begin = nullptr;

    MergeRunner() = default;
    MergeRunner(const MergeRunner&) = delete;
    MergeRunner& operator=(const MergeRunner&) = delete;
    ~MergeRunner() {
        for (void* p : {(void*)d_merges, (void*)d_seg_begin, (void*)d_stage_begin, (void*)gnodes,
                        (void*)flags, (void*)part_totals, (void*)coin_end, (void*)seg_bars,
                        (void*)d_lvl_start, (void*)d_lvl_begin, (void*)xch})
            if (p) cudaFree(p);
    }

    // seg_launch: owned segments per launch (1: per-segment pipeline);
    // cta_limit: CTAs per SM left to the merge (0: all it can get).
    // Lanes (independent chains side by side) halve the barrier steps of a
    // torus stage but multiply the tiles of a launch; when that costs extra
    // launches (one GPU, many segments: the tiles no longer fit one
    // co-resident grid) the stages run as single lanes instead.
    marsit_status configure(int sm_count, uint32_t seg_launch = 0, int cta_limit = 0) {
        if (grid && !fused_arrays) return configure_grid(sm_count, seg_launch ? seg_launch : n_seg);
        grid = false;
        if (cluster) return configure_cluster(seg_launch ? seg_launch : n_seg);
        marsit_status s = configure_once(sm_count, seg_launch, cta_limit);
        if (s || lanes_max == 1 || n_parts == 1) return s;
        const uint32_t parts_lanes = n_parts;
        DevicePlan keep = dp;
        dp.single_lanes();
        if ((s = configure_once(sm_count, seg_launch, cta_limit))) return s;
        if (n_parts < parts_lanes) return MARSIT_OK;
        dp = keep;
        return configure_once(sm_count, seg_launch, cta_limit);
    }

    // Cluster size and groups per thread: fewest waves of resident clusters
    // for the segments of one launch, then the smallest CTA tile (the
    // per-level deposit work of a CTA), + a fixed per-level sync cost.
    // MARSIT_MERGE_CSIZE forces the CTAs per cluster.
    marsit_status configure_cluster(uint32_t seg_launch) {
        seg_per_launch = seg_launch;
        n_parts = 1;
        const uint32_t total_groups = words_proc / 4;
        const int forced = env_int("MARSIT_MERGE_CSIZE", 0);
        uint64_t best = ~0ull;
        const uint32_t nl = dp.level_width;
        for (uint32_t cs : {16u, 14u, 12u, 10u, 8u, 6u, 4u, 2u, 1u}) {
            if (forced && cs != uint32_t(forced)) continue;
            const uint32_t tg = uint32_t(ceil_div(total_groups, cs));
            uint32_t ns = 0;
            const uint32_t threads = fused_arrays ? uint32_t(kFusedThreads) : uint32_t(kClusterThreads);
            for (uint32_t c : {1u, 2u, 4u, 8u, 16u})
                if (uint64_t(c) * threads >= tg && (nl == 1 || c <= 8)) {
                    ns = c;
                    break;
                }
            if (!ns) continue;
            // slots, + the level's staged r and d when they fit (pass 2 then
            // reads shared memory instead of re-loading the operands)
            const size_t base_sm = size_t(dp.max_slots + fused_arrays) * tg * 16;
            const size_t stage_sm = size_t(2) * nl * tg * 16;
            if (base_sm > 212 * 1024) continue;
            const size_t ring = 0;
            const size_t cap = fused_arrays ? 212 * 1024 : 200 * 1024;  // fused: 227 KB - static
            if (base_sm + ring > cap) continue;
            const uint32_t stg = base_sm + stage_sm + ring <= cap && env_int("MARSIT_MERGE_STAGE", 1) ? 1u : 0u;
            // + the deposit masks formed during the level barrier
            const size_t mask_sm = size_t(4) * nl * tg * 16;
            const uint32_t msk =
                stg && base_sm + stage_sm + mask_sm + ring <= cap && env_int("MARSIT_MERGE_MASKS", 1) ? 1u : 0u;
            const size_t sm = std::max<size_t>(base_sm + (stg ? stage_sm : 0) + (msk ? mask_sm : 0) + ring, 16);
            int occ = 0;
            if (fused_arrays && ns > 4) continue;  // the fused kernel's instantiations
            const cudaError_t oe =
                fused_arrays ? (fused_dtype == 1 ? round_cluster_occupancy<double>(int(ns), int(nl), cs, sm, &occ)
                                                 : round_cluster_occupancy<float>(int(ns), int(nl), cs, sm, &occ))
                             : merge_cluster_occupancy(int(ns), int(nl), cs, sm, &occ);
            if (oe != cudaSuccess || occ <= 0) {
                cudaGetLastError();
                continue;
            }
            const uint64_t waves = ceil_div(seg_per_launch, uint64_t(occ));
            const uint64_t cost = waves * (uint64_t(tg) + 400);
            if (env_int("MARSIT_MERGE_DEBUG", 0))
                fprintf(stderr, "merge cluster: csize %u groups/CTA %u nsub %u stage %u masks %u occ %d waves %llu cost %llu\n",
                        cs, tg, ns, stg, msk, occ, (unsigned long long)waves, (unsigned long long)cost);
            if (cost < best) {
                best = cost;
                csize = cs;
                tile_groups = tg;
                nsub = ns;
                smem = sm;
                merge_smem = sm - ring;
                stage = stg;
                masks = msk;
            }
        }
        if (best == ~0ull) return fail(MARSIT_EUNSUPPORTED, "merge clusters do not fit the device");
        return MARSIT_OK;
    }

    // Spread round (round_spread_kernel, 512-thread CTAs, one per SM): the
    // cluster size whose co-resident clusters give the most CTAs (ties: the
    // larger cluster), at least one cluster per owned segment; pairs only
    // when nothing larger fits (C1, measured: csize 4 / 132 CTAs 27.6 us per
    // round, 2 / 148 CTAs 33.6 us: the merge tile per CTA doubles); the merge
    // tiles of a cluster as in configure_cluster.  MARSIT_SPREAD_CSIZE forces it.
    marsit_status configure_spread(int dtype, uint32_t workers, uint32_t* ctas) {
        if (dp.n_merges > kSpreadMaxMerges) return fail(MARSIT_EUNSUPPORTED, "spread round: too many merges");
        seg_per_launch = n_seg;
        n_parts = 1;
        grid = false;
        const uint32_t total_groups = words_proc / 4;
        const uint32_t nl = dp.level_width;
        const int forced = env_int("MARSIT_SPREAD_CSIZE", 0);
        uint32_t best = 0;
        for (uint32_t cs : {16u, 8u, 4u, 2u}) {
            if (forced && cs != uint32_t(forced)) continue;
            const uint32_t tg = uint32_t(ceil_div(total_groups, cs));
            uint32_t ns = 0;
            for (uint32_t c : {1u, 2u, 4u})
                if (uint64_t(c) * kFusedThreads >= tg) {
                    ns = c;
                    break;
                }
            if (!ns) continue;
            const size_t cap = 200 * 1024;
            // the cluster's leaf tiles + its aggregate tile, then the slots
            const size_t base_sm = size_t(dp.max_slots + workers + 1) * tg * 16;
            const size_t stage_sm = size_t(2) * nl * tg * 16;
            const size_t mask_sm = size_t(4) * nl * tg * 16;
            if (base_sm > cap) continue;
            const uint32_t stg = base_sm + stage_sm <= cap && env_int("MARSIT_MERGE_STAGE", 1) ? 1u : 0u;
            const uint32_t msk =
                stg && base_sm + stage_sm + mask_sm <= cap && env_int("MARSIT_MERGE_MASKS", 1) ? 1u : 0u;
            const size_t sm = std::max<size_t>(base_sm + (stg ? stage_sm : 0) + (msk ? mask_sm : 0), 16);
            int occ = 0;
            const cudaError_t oe = dtype == 1 ? round_spread_occupancy<double>(int(ns), int(nl), cs, sm, &occ)
                                              : round_spread_occupancy<float>(int(ns), int(nl), cs, sm, &occ);
            if (oe != cudaSuccess || occ <= 0 || uint32_t(occ) < n_seg) {
                cudaGetLastError();
                continue;
            }
            if (env_int("MARSIT_MERGE_DEBUG", 0))
                fprintf(stderr, "spread: csize %u clusters %d groups/CTA %u nsub %u stage %u masks %u\n", cs, occ,
                        tg, ns, stg, msk);
            if (cs == 2 && best) continue;
            if (uint32_t(occ) * cs > best) {
                best = uint32_t(occ) * cs;
                csize = cs;
                tile_groups = tg;
                nsub = ns;
                smem = merge_smem = sm;
                stage = stg;
                masks = msk;
            }
        }
        if (!best) return fail(MARSIT_EUNSUPPORTED, "spread round does not fit the device");
        *ctas = best;
        return MARSIT_OK;
    }

    // Grid mode: every SM hosts one 1024-thread CTA; the segments of a
    // launch share the SMs evenly (csize tiles each); the smallest groups per
    // thread that cover a tile; r / d staging when the shared memory allows.
    marsit_status configure_grid(int sm_count, uint32_t seg_launch) {
        n_parts = 1;
        const uint32_t nl = dp.level_width;
        const uint32_t total_groups = words_proc / 4;
        int occ = 0;
        for (int attempt = 0; attempt < 2; ++attempt) {
            // MARSIT_MERGE_CSIZE forces the CTAs per segment (the segments
            // then run as several launches when they do not fit one)
            const uint32_t slots = uint32_t(sm_count) * std::max(occ, 1);
            const uint32_t forced = uint32_t(env_int("MARSIT_MERGE_CSIZE", 0));
            seg_per_launch = std::min<uint32_t>(seg_launch, forced ? std::max(1u, slots / forced) : slots);
            csize = forced ? forced : std::max<uint32_t>(1, slots / seg_per_launch);
            tile_groups = uint32_t(ceil_div(total_groups, csize));
            nsub = 0;
            for (uint32_t c : {1u, 2u, 4u, 8u, 16u})
                if (uint64_t(c) * kClusterThreads >= tile_groups && (nl == 1 || c <= 8)) {
                    nsub = c;
                    break;
                }
            if (!nsub) return fail(MARSIT_EUNSUPPORTED, "merge tiles too large for the grid merge");
            const size_t base_sm = size_t(dp.max_slots) * tile_groups * 16;
            const size_t stage_sm = size_t(2) * nl * tile_groups * 16;
            stage = base_sm + stage_sm <= 200 * 1024 && env_int("MARSIT_MERGE_STAGE", 1) ? 1u : 0u;
            const size_t mask_sm = size_t(4) * nl * tile_groups * 16;
            masks = stage && base_sm + stage_sm + mask_sm <= 200 * 1024 && env_int("MARSIT_MERGE_MASKS", 1) ? 1u : 0u;
            smem = merge_smem = std::max<size_t>(base_sm + (stage ? stage_sm : 0) + (masks ? mask_sm : 0), 16);
            if (smem > 200 * 1024) return fail(MARSIT_EUNSUPPORTED, "merge tiles do not fit shared memory");
            CUDA_TRY(merge_grid_occupancy(int(nsub), int(nl), smem, kClusterThreads, &occ));
            if (occ <= 0) return fail(MARSIT_EUNSUPPORTED, "grid merge does not fit an SM");
            if (uint64_t(seg_per_launch) * csize <= uint64_t(occ) * sm_count) break;
        }
        if (uint64_t(seg_per_launch) * csize > uint64_t(occ) * sm_count)
            return fail(MARSIT_EUNSUPPORTED, "grid merge CTAs are not co-resident");
        // tiles of <= 256 / 512 groups: CTAs of that many threads (one group
        // per thread; the same grid, so still one CTA per SM): G = 8 rank
        // merge 28.7 -> 24.8 us, torus 26.6 -> 22.7 us; MARSIT_GRID_SMALL=0
        // keeps 1024
        grid_nt = kClusterThreads;
        for (uint32_t nt : {256u, 512u})
            if (nsub == 1 && tile_groups <= nt && env_int("MARSIT_GRID_SMALL", 1)) {
                int occ_s = 0;
                if (merge_grid_occupancy(1, int(nl), smem, int(nt), &occ_s) == cudaSuccess &&
                    uint64_t(seg_per_launch) * csize <= uint64_t(occ_s) * sm_count) {
                    grid_nt = nt;
                    break;
                }
                cudaGetLastError();
            }
        if (env_int("MARSIT_MERGE_DEBUG", 0))
            fprintf(stderr, "merge grid: %u segments x %u CTAs of %u threads, groups/CTA %u nsub %u stage %u masks %u\n",
                    seg_per_launch, csize, grid_nt, tile_groups, nsub, stage, masks);
        return MARSIT_OK;
    }

    marsit_status configure_once(int sm_count, uint32_t seg_launch, int cta_limit) {
        seg_per_launch = seg_launch ? seg_launch : n_seg;
        k_steps.assign(dp.n_stages, 0);
        lanes_max = 1;
        for (uint32_t st = 0; st < dp.n_stages; ++st) lanes_max = std::max(lanes_max, dp.n_lanes[st]);
        for (uint32_t sl = 0; sl < n_seg; ++sl)
            for (uint32_t st = 0; st < dp.n_stages; ++st) {
                const uint32_t* lb = &dp.lane_begin[(size_t(sl) * dp.n_stages + st) * (kMaxLanes + 1)];
                for (uint32_t ln = 0; ln < kMaxLanes; ++ln)
                    k_steps[st] = std::max(k_steps[st], lb[ln + 1] - lb[ln]);
            }
        const uint64_t vsegs = uint64_t(seg_per_launch) * lanes_max;  // tile sets per launch
        // Tiling (measured on B200, tools/sweep_merge_balance.sh, merge alone):
        // fewest launches ("parts") first, then the lowest estimated step cost
        //   cost = WPT * (k + 1) + 6 * [k >= 3],   k = CTAs on the busiest SM.
        // Each merge step is a latency chain per thread that grows with the
        // words per thread (WPT), and the busiest SM's ALU work (coin deposit)
        // and the grid barrier grow with k.  Measured picks: G = 8 rank (1
        // segment) WPT 2, G = 2 rank (4 segments) WPT 4, one GPU C3 (8
        // segments) WPT 12.  MARSIT_MERGE_WPT forces the words per thread;
        // MARSIT_MERGE_BALANCE = k forces exactly k CTAs per SM when possible.
        const int forced = env_int("MARSIT_MERGE_WPT", 0);
        const int balance = env_int("MARSIT_MERGE_BALANCE", 0);
        uint64_t best_parts = ~0ull, best_cost = ~0ull;
        for (int w : {1, 2, 4, 8, 12, 16}) {
            if (forced && w != forced) continue;
            // slots + the deposit masks (4 words per packed word)
            const size_t sm = (size_t(std::max<uint32_t>(dp.max_slots, 1)) + 4) * w * kMergeThreads * 4;
            if (sm > 160 * 1024) continue;
            int occ = 0;
            CUDA_TRY(merge_coop_occupancy(w, sm, &occ));
            if (cta_limit > 0) occ = std::min(occ, cta_limit);
            const uint64_t cap = uint64_t(occ) * sm_count;
            const uint64_t tw_max = uint64_t(w) * kMergeThreads;
            const uint64_t gran = std::max(w, 4);  // a thread's words never straddle tiles
            const uint64_t tps_min = ceil_div(words_proc, tw_max);
            uint64_t tps = tps_min, tw = round_up(ceil_div(words_proc, tps), gran);
            if (balance > 0 && balance <= occ && (uint64_t(balance) * sm_count) % vsegs == 0) {
                // exactly `balance` CTAs on every SM; trailing tiles may be
                // empty: they only take part in the barriers
                const uint64_t t = uint64_t(balance) * sm_count / vsegs;
                const uint64_t tww = round_up(ceil_div(words_proc, t), gran);
                if (t >= tps_min && tww <= tw_max) {
                    tps = t;
                    tw = tww;
                }
            }
            const uint64_t pt = std::min<uint64_t>(tps, cap / vsegs);
            if (pt == 0) continue;
            const uint64_t parts = ceil_div(tps, pt);
            const uint64_t ctas = pt * vsegs;
            const uint64_t k = ceil_div(ctas, uint64_t(sm_count));
            const uint64_t cost = uint64_t(w) * (k + 1) + (k >= 3 ? 6 : 0);
            if (parts < best_parts || (parts == best_parts && cost < best_cost)) {
                best_parts = parts;
                best_cost = cost;
                wpt = w;
                smem = sm;
                tile_words = uint32_t(tw);
                tiles_per_seg = uint32_t(tps);
                part_tiles = uint32_t(pt);
                n_parts = uint32_t(parts);
            }
        }
        if (best_parts == ~0ull) return fail(MARSIT_EUNSUPPORTED, "merge tiles do not fit the device");
        return MARSIT_OK;
    }

    marsit_status upload() {
        const size_t nm = std::max<size_t>(dp.n_merges, 1);
        CUDA_TRY(cudaMalloc(&d_merges, sizeof(DevMerge) * nm));
        CUDA_TRY(cudaMemcpy(d_merges, dp.merges.data(), sizeof(DevMerge) * dp.n_merges,
                            cudaMemcpyHostToDevice));
        if (cluster) {
            auto put = [](uint32_t** d, const std::vector<uint32_t>& h) -> cudaError_t {
                cudaError_t e = cudaMalloc(d, sizeof(uint32_t) * std::max<size_t>(h.size(), 1));
                if (e == cudaSuccess && !h.empty())
                    e = cudaMemcpy(*d, h.data(), sizeof(uint32_t) * h.size(), cudaMemcpyHostToDevice);
                return e;
            };
            CUDA_TRY(put(&d_seg_begin, dp.seg_begin));
            CUDA_TRY(put(&d_lvl_start, dp.lvl_start));
            CUDA_TRY(put(&d_lvl_begin, dp.lvl_begin));
            CUDA_TRY(cudaMalloc(&part_totals, sizeof(uint64_t) * nm));
            CUDA_TRY(cudaMemset(part_totals, 0, sizeof(uint64_t) * nm));
            CUDA_TRY(cudaMalloc(&coin_end, sizeof(uint64_t) * nm));
            CUDA_TRY(cudaMemset(coin_end, 0xFF, sizeof(uint64_t) * nm));  // no history yet
            if (grid) {
                const size_t nx = size_t(2) * seg_per_launch * csize * dp.level_width;
                CUDA_TRY(cudaMalloc(&xch, sizeof(unsigned long long) * nx));
                CUDA_TRY(cudaMemset(xch, 0, sizeof(unsigned long long) * nx));
            }
            return MARSIT_OK;
        }
        CUDA_TRY(cudaMalloc(&d_seg_begin, sizeof(uint32_t) * dp.seg_begin.size()));
        CUDA_TRY(cudaMemcpy(d_seg_begin, dp.seg_begin.data(), sizeof(uint32_t) * dp.seg_begin.size(),
                            cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMalloc(&d_stage_begin, sizeof(uint32_t) * dp.lane_begin.size()));
        CUDA_TRY(cudaMemcpy(d_stage_begin, dp.lane_begin.data(),
                            sizeof(uint32_t) * dp.lane_begin.size(), cudaMemcpyHostToDevice));
        const uint32_t gmax = std::max<uint32_t>(dp.gmax, 1);
        CUDA_TRY(cudaMalloc(&gnodes, sizeof(uint32_t) * size_t(n_seg) * gmax * wst));
        uint32_t kmax = 1;
        for (uint32_t k : k_steps) kmax = std::max(kmax, k);
        const size_t nflags = size_t(kmax) * seg_per_launch * lanes_max * part_tiles;
        CUDA_TRY(cudaMalloc(&flags, sizeof(uint64_t) * nflags));
        CUDA_TRY(cudaMemset(flags, 0, sizeof(uint64_t) * nflags));
        CUDA_TRY(cudaMalloc(&part_totals, sizeof(uint64_t) * size_t(n_parts) * nm));
        CUDA_TRY(cudaMemset(part_totals, 0, sizeof(uint64_t) * size_t(n_parts) * nm));
        CUDA_TRY(cudaMalloc(&seg_bars, sizeof(unsigned) * size_t(seg_per_launch) * lanes_max));
        CUDA_TRY(cudaMemset(seg_bars, 0, sizeof(unsigned) * size_t(seg_per_launch) * lanes_max));
        CUDA_TRY(cudaMalloc(&coin_end, sizeof(uint64_t) * nm));
        CUDA_TRY(cudaMemset(coin_end, 0xFF, sizeof(uint64_t) * nm));  // no history yet
        return MARSIT_OK;
    }

    ClusterParams cluster_params(const uint32_t* leaves, uint32_t* agg, const uint32_t* coins,
                                 uint64_t seed, uint64_t round, uint32_t seg_lo,
                                 const uint32_t* coin_valid) const {
        ClusterParams c{};
        c.merges = d_merges;
        c.seg_begin = d_seg_begin;
        c.lvl_start = d_lvl_start;
        c.lvl_begin = d_lvl_begin;
        c.n_seg = n_seg;
        c.s_first = s_first;
        c.seg_lo = seg_lo;
        c.csize = csize;
        c.tile_groups = tile_groups;
        c.words_proc = words_proc;
        c.wst = wst;
        c.ml = ml;
        c.n_slots = dp.max_slots;
        c.stage = stage;
        c.masks = masks;
        c.prefetch = prefetch;
        c.coin_l1 = coin_l1;
        c.grid_coop = grid_coop;
        if (n_seg == 1 && dp.lvl_start.size() >= 2) {
            c.solo_nm = dp.n_merges;
            c.solo_nlv = dp.lvl_start[1] - dp.lvl_start[0] - 1;
        }
        c.seg_bits = L;
        c.leaves = leaves;
        c.peer_bits = peer_bits;
        c.agg = agg;
        c.agg_stride = agg_stride ? agg_stride : wst;
        c.coins = coins;
        c.coin_valid = coins ? coin_valid : nullptr;
        c.totals = part_totals;
        c.coin_end = coin_end;
        c.seed = seed;
        c.round = round;
        c.err = err;
        c.xch = xch;
        c.seg_bars = seg_bars;
        return c;
    }

    // Merge owned segments [seg_lo, seg_lo + seg_cnt) (seg_cnt <= seg_per_launch
    // per launch; more segments run as consecutive launches).
    marsit_status run(const uint32_t* leaves, uint32_t* agg, const uint32_t* coins, uint64_t seed,
                      uint64_t round, cudaStream_t st, uint64_t* n_launch, uint32_t seg_lo = 0,
                      uint32_t seg_cnt = ~0u, const uint32_t* coin_valid = nullptr) {
        if (seg_cnt == ~0u) seg_cnt = n_seg - seg_lo;
        if (cluster) {
            if (seg_cnt == 0) return MARSIT_OK;
            if (grid) {  // launches of at most seg_per_launch co-resident segments
                for (uint32_t s0 = seg_lo; s0 < seg_lo + seg_cnt; s0 += seg_per_launch) {
                    ClusterParams c = cluster_params(leaves, agg, coins, seed, round, s0, coin_valid);
                    if ((++xch_epoch & 0xFFFFFFu) == 0) ++xch_epoch;  // tag 0 = never written
                    c.xch_tag = xch_epoch;
                    CUDA_TRY(launch_merge_grid(c, int(nsub), int(dp.level_width),
                                               std::min(seg_per_launch, seg_lo + seg_cnt - s0), smem, int(grid_nt), st));
                    ++*n_launch;
                }
                return MARSIT_OK;
            }
            const ClusterParams c = cluster_params(leaves, agg, coins, seed, round, seg_lo, coin_valid);
            CUDA_TRY(launch_merge_cluster(c, int(nsub), int(dp.level_width), seg_cnt, merge_smem, st));
            ++*n_launch;
            return MARSIT_OK;
        }
        CoopParams c{};
        c.merges = d_merges;
        c.seg_begin = d_seg_begin;
        c.lane_begin = d_stage_begin;
        c.n_stages = dp.n_stages;
        c.n_seg = n_seg;
        c.s_first = s_first;
        c.tiles_per_seg = tiles_per_seg;
        c.tile_words = tile_words;
        c.words_proc = words_proc;
        c.wst = wst;
        c.ml = ml;
        c.max_slots = std::max<uint32_t>(dp.max_slots, 1);
        c.n_parts = n_parts;
        c.part_tiles = part_tiles;
        c.n_merges = dp.n_merges;
        c.seg_bits = L;
        c.leaves = leaves;
        c.peer_bits = peer_bits;
        c.gnodes = gnodes;
        c.gmax = std::max<uint32_t>(dp.gmax, 1);
        c.agg = agg;
        c.agg_stride = agg_stride ? agg_stride : wst;
        c.coins = coins;
        c.flags = flags;
        c.part_totals = part_totals;
        c.seed = seed;
        c.round = round;
        c.coin_valid = coins ? coin_valid : nullptr;
        c.coin_end = coin_end;
        c.seg_bars = seg_barrier ? seg_bars : nullptr;
        c.err = err;
        for (uint32_t s0 = seg_lo; s0 < seg_lo + seg_cnt; s0 += seg_per_launch) {
            c.seg_lo = s0;
            c.seg_cnt = std::min(seg_per_launch, seg_lo + seg_cnt - s0);
            for (uint32_t stage = 0; stage < dp.n_stages; ++stage) {
                if (k_steps[stage] == 0) continue;
                c.stage = stage;
                c.k_steps = k_steps[stage];
                c.n_lanes = dp.n_lanes[stage];
                for (uint32_t part = 0; part < n_parts; ++part) {
                    c.part = part;
                    c.part_tile0 = part * part_tiles;
                    CUDA_TRY(launch_merge_coop(c, wpt, smem, st));
                    ++*n_launch;
                }
            }
        }
        return MARSIT_OK;
    }
};

struct TimedPair {
    int phase;
    cudaEvent_t a, b;
};

// Device error latch bits (marsit_ctx::err, reported by marsit_ctx_check).
constexpr int kErrNonFinite = 1;  // DenseVector finiteness (dense_vector.hpp:25-29)
constexpr int kErrConsensus = 2;  // an aggregate segment differs from its owner's (allreduce.hpp:32-43)
constexpr int kErrBounds = 8;     // checked builds (MARSIT_CHECKED): an index failed its bound
constexpr int kErrSync = 16;      // spread round: a wait on the other CTAs ran past its bound

// P2P flag value that releases every stream wait: written by a watchdog that
// gave up (into its own flags and into its slot of every peer's flags) so no
// stream stays blocked; a peer that sees it reports the abort.  The stream
// waits compare (int64_t)(flag - epoch) >= 0, so the value is the largest
// positive int64 (all-ones would read as -1).
constexpr uint64_t kFlagAbort = 0x7FFFFFFFFFFFFFFFull;

// Bounded waits for multi-rank contexts (P2P epoch flags, NCCL collectives).
// The round entry points hand every enqueued round to this thread; if a round
// has not completed after the timeout (or NCCL reports an asynchronous error,
// or a peer posted kFlagAbort), the context is marked failed: P2P waits are
// released by writing kFlagAbort into the local flags and the peers' slots,
// NCCL communicators are aborted, and every later call on the context
// returns the latched status (EPROTOCOL / ENCCL) instead of hanging — the
// reference's contract for a broken wire is protocol_error (errors.hpp:24-29).
struct Watchdog {
    struct Item {
        cudaEvent_t ev;
        std::chrono::steady_clock::time_point t0;
        uint64_t epoch;
    };
    marsit_ctx* ctx = nullptr;
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<Item> pending;
    std::vector<cudaEvent_t> free_events;
    bool stop = false;
    cudaStream_t st = nullptr;        // private stream: flag reads and releases
    cudaEvent_t ev_poll = nullptr;
    uint64_t* h_flags = nullptr;      // pinned copy of the local flags [2][G]
    uint64_t* h_abort = nullptr;      // pinned [2][G] x kFlagAbort (the release values)

    explicit Watchdog(marsit_ctx* c);
    ~Watchdog();
    marsit_status watch(cudaStream_t s, uint64_t epoch);  // after a round was enqueued on s
    void loop();
    void give_up(marsit_status st, const std::string& msg);
};


}  // namespace marsit_b200

namespace marsit_b200 {
// Device scratch of the SSDM baselines (ssdm.cu), allocated on first use.
struct SsdmScratch {
    double* acc = nullptr;       // cascading accumulators [S][L]
    uint32_t* pk = nullptr;      // packets [M][S][wst]
    double* norms = nullptr;     // [M * S]
    double* partial = nullptr;   // [M * S][chunks]
    unsigned long long* hist = nullptr;  // [S][M][M+1]
    uint8_t* chain = nullptr;    // [S][M]
    ~SsdmScratch();
};
}  // namespace marsit_b200

struct marsit_ctx {
    int device = 0;
    marsit_dtype dtype = MARSIT_F32;
    size_t esize = 4;
    uint64_t D = 0, L = 0;
    uint32_t M = 0, S = 0, G = 1, rank = 0, ml = 0, s_own = 0, s_first = 0;
    uint32_t words64 = 0, words_proc = 0, wst = 0;
    int sm_count = 148;
    bool fused = false;  // small rounds: one round_cluster_kernel launch (runtime.cu fused_round)
    // small rounds over every SM: one round_spread_kernel launch (runtime.cu
    // spread_round); preferred to `fused` when it configures
    bool spread = false;
    bool spread_coop = true;           // + the cooperative attribute while accepted (MARSIT_SPREAD_COOP=0: off)
    uint32_t spread_ctas = 0;          // CTAs of the launch (co-resident clusters x csize)
    // spread round: TMEM columns per thread for the parked u (0: the decode
    // re-reads g, c) and the allocation per CTA
    uint32_t stash_cols = 0, tmem_cols = 0;
    // spread round: the extract's TMA ring (stages of one worker's slice, g
    // then c, tma_half bytes each; 0 stages = register loads) and the launch's
    // dynamic shared memory (max of that ring and the merge clusters' tiles)
    uint32_t tma_stages = 0, tma_half = 0;
    size_t spread_smem = 0;
    unsigned* spread_sync = nullptr;   // [2 + S]: arrivals, generation, per-segment merged flags
    uint32_t* spread_coins[2] = {nullptr, nullptr};  // coin buffers by round parity (SpreadParams)
    uint32_t* spread_valid[2] = {nullptr, nullptr};
    unsigned long long* spread_tag = nullptr;        // [2][2] (seed, round) per buffer
    unsigned long long* spread_cend = nullptr;       // [2][n_merges] stream ends by round parity
    // K1/K4 task order (StreamParams::reverse); MARSIT_L2_REUSE=0 disables
    bool l2_reuse = marsit_b200::env_int("MARSIT_L2_REUSE", 1) != 0;
    uint32_t task_dir = 0;
    bool vec_ok = false;
    marsit_b200::HostSchedule sched;
    marsit_b200::Plan plan;
    marsit_b200::MergeRunner merge;
    // device buffers
    uint32_t* bits = nullptr;  // [S][ml][wst]
    uint32_t* recv = nullptr;  // [G][s_own][ml][wst]   (G > 1)
    uint32_t* agg = nullptr;   // [S][wsa]: wst words, then the segment's u64 owner hash (consensus)
    uint32_t wsa = 0;          // aggregate row stride in u32 words (wst + 4)
    int* err = nullptr;
    int stream_grid = 0;   // generic grid-stride kernels
    int extract_grid = 0;  // persistent, one wave of resident CTAs
    int decode_grid = 0;
    int stats_grid = 0;   // decode with the fused matching count (metrics on)
    // dense round scratch
    void* dense_send = nullptr;  // [G][s_own][ml][L] of dtype
    void* dense_recv = nullptr;
    void* dense_mean = nullptr;  // [S*L] of dtype (G > 1)
    marsit_b200::DenseOp* d_dense_ops = nullptr;
    uint16_t* d_dense_final = nullptr;
    uint16_t* d_dense_chain = nullptr;  // chain-of-chains plans: [s_own][M] leaf order
    uint64_t* d_dense_groups = nullptr; // [s_own] group-end bits of that order
    bool dense_multi = false;           // more than one group in some segment
    uint32_t dense_n_ops = 0;
    // coin precompute on the aux stream; two buffers: this round's and the
    // next round's, computed speculatively for (seed, t + 1) during the decode
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr;
    uint32_t* coin_buf[2] = {nullptr, nullptr};
    uint32_t* coin_valid[2] = {nullptr, nullptr};  // [n_merges] words computed per merge
    cudaEvent_t ev_coin_done[2] = {nullptr, nullptr};
    struct CoinTag {
        bool valid = false;
        uint64_t seed = 0, round = 0;
    } coin_tag[2];
    int cur_coin = 0;
    bool coin_prefetch = true;
    bool coin_prefetch_at_extract = false;
    bool coins_pending = false;
    uint64_t coin_total_words = 0;
    // single GPU: per-segment merges (aux) pipelined with per-segment decodes
    bool pipeline = false;
    cudaEvent_t ev_extract = nullptr;
    std::vector<cudaEvent_t> ev_merge;
    int coin_grid_x = 1;
    // P2P transport (marsit_ctx_set_peers): device tables of the peers'
    // buffers, host copies of their flag words, this rank's epoch flags
    bool p2p = false, peers_set = false;
    bool flag_kernel = false;   // signal with flag_write_kernel instead of stream writes
    uint64_t* flags = nullptr;  // [2][G]: epoch each rank reported (data ready, results ready)
    uint64_t epoch = 0;         // rounds (sign or dense) run so far
    std::vector<const uint64_t*> peer_flags;
    std::vector<void*> peer_dense_mean;
    void** d_peer_tables = nullptr;  // [3][G]: bits, agg, dense_send
    // NCCL
    ncclComm_t comm = nullptr;
    bool owns_comm = true;
    // SSDM baselines (ssdm.cu)
    std::unique_ptr<marsit_b200::SsdmScratch> ssdm;
    // on-device round metrics (marsit_ctx_set_metrics)
    bool metrics = false;
    unsigned long long* d_metrics = nullptr;  // [0] matches, [1..2] NCCL sum scratch
    bool last_valid = false, last_dense = false, last_matching = false;
    uint64_t last_t = 0;
    // failure handling: a latched failure (status, message) makes every later
    // call return it; the watchdog bounds waits on peers / NCCL
    std::atomic<int> fail_status{0};
    mutable std::mutex fail_mu;
    std::string fail_msg;
    uint64_t wait_timeout_ms = uint64_t(marsit_b200::env_int("MARSIT_WAIT_TIMEOUT_MS", 120000));
    std::unique_ptr<marsit_b200::Watchdog> watchdog;
    // opt-in data consensus (allreduce.hpp:32-43): owners hash their aggregate
    // segments after the merge; after the decode every rank re-hashes all S
    // segments as it reads them and compares
    bool consensus = false;
    unsigned long long* d_verify = nullptr;  // [S] re-hashed segments
    cudaEvent_t ev_check = nullptr;          // marsit_ctx_check's stream poll
    uint64_t* h_check = nullptr;             // pinned: error latch, then the P2P flags [2][G]
    // timing
    bool timing = false;
    std::vector<marsit_b200::TimedPair> pending;
    std::vector<cudaEvent_t> event_pool;
    float ms[MARSIT_N_PHASES] = {};
    uint64_t launches[MARSIT_N_PHASES] = {};

    ~marsit_ctx();
    marsit_status begin_phase(cudaStream_t st, cudaEvent_t* a);
    marsit_status end_phase(int phase, cudaStream_t st, cudaEvent_t a, uint64_t n_launch);
};


namespace marsit_b200 {

// One sign round (sync.hpp:91-118) with the optional fused parameter update
// x_w -= g_t (params may be null).
marsit_status sign_round_impl(marsit_ctx* ctx, uint64_t t, double eta_s, uint64_t seed,
                              const void* const* grads, const void* const* comp,
                              void* const* comp_out, void* const* params, uint64_t* agg_bits,
                              void* update, cudaStream_t st);
// One dense round (sync.hpp:78-87); mean is required; params may be null.
marsit_status dense_round_any(marsit_ctx* ctx, uint64_t t, const void* const* grads, const void* const* comp,
                              void* const* comp_out, void* const* params, void* mean,
                              cudaStream_t st);
// cascading_allreduce / sum_ssdm_allreduce on the device (ssdm.cu).
marsit_status ssdm_allreduce_impl(marsit_ctx* ctx, int mode, uint64_t round, uint64_t seed,
                                  const void* const* d_vectors, void* d_estimate,
                                  uint64_t* bits_per_worker, uint64_t* reduce_bits,
                                  uint64_t* gather_bits, int64_t* max_abs_per_step,
                                  cudaStream_t st);
// marsit_ctx_create, optionally sharing an existing communicator (driver buckets).
marsit_status ctx_create_internal(const marsit_ctx_desc* desc, ncclComm_t shared_comm,
                                  marsit_ctx** out);
// Payload bits of one round (allreduce.hpp:113, 182).
uint64_t round_bits_total(const marsit_ctx* ctx, bool dense);
// The latched failure of a context (MARSIT_OK when healthy); sets the
// thread-local message.
marsit_status ctx_failed(const marsit_ctx* ctx);
void ctx_set_failed(marsit_ctx* ctx, marsit_status st, const std::string& msg);
// Hand the round just enqueued on `st` to the context's watchdog (no-op for
// single-rank contexts).
marsit_status watch_round(marsit_ctx* ctx, cudaStream_t st);

}  // namespace marsit_b200
