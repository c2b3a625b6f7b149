// runtime.cu — host runtime behind the C-ABI (include/marsit_b200.h).
//
// A marsit_ctx owns every device buffer of the path and the compiled merge
// plan; a sign round is a fixed sequence of launches on the caller's stream:
//
//   [aux: coins for (seed, t) unless prefetched]
//   extract -> (G > 1: NCCL exchange of packed segments to their owners)
//   -> cooperative merge (per plan stage x part) -> [aux: coins for t + 1]
//   -> (G > 1: NCCL all-gather of the owned aggregates) -> decode+comp
//
// Segments are owned by ranks in contiguous blocks (rank q owns segments
// [q*S/G, (q+1)*S/G)), so the exchange is an all-to-all of contiguous
// per-destination blocks and the all-gather is in place.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <functional>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.hpp"

using namespace marsit_b200;

namespace marsit_b200 {

namespace {
thread_local std::string g_last_error;
}  // namespace

marsit_status fail(marsit_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

// NVTX ranges around the host enqueue of each phase (MARSIT_NVTX=1; for
// profilers' range filters, e.g. ncu --nvtx --nvtx-include "marsit.merge/").
struct NvtxRange {
    bool on;
    explicit NvtxRange(const char* name) : on(nvtx_enabled()) {
        if (on) nvtxRangePushA(name);
    }
    ~NvtxRange() {
        if (on) nvtxRangePop();
    }
    static bool nvtx_enabled() {
        static const bool e = env_int("MARSIT_NVTX", 0) != 0;
        return e;
    }
};

marsit_status ctx_failed(const marsit_ctx* ctx) {
    const int st = ctx->fail_status.load();
    if (!st) return MARSIT_OK;
    std::lock_guard<std::mutex> lock(ctx->fail_mu);
    return fail(marsit_status(st), ctx->fail_msg);
}

void ctx_set_failed(marsit_ctx* ctx, marsit_status st, const std::string& msg) {
    std::lock_guard<std::mutex> lock(ctx->fail_mu);
    if (ctx->fail_status.load()) return;  // the first failure wins
    ctx->fail_msg = msg;
    ctx->fail_status.store(int(st));
}

// Wait for everything enqueued on `st` so far by polling an event (never
// blocking inside the driver: a thread blocked in a synchronous call can hold
// up the watchdog's own calls that would release the wait).
cudaError_t poll_stream(cudaStream_t st, cudaEvent_t ev) {
    cudaError_t e = cudaEventRecord(ev, st);
    if (e != cudaSuccess) return e;
    for (;;) {
        e = cudaEventQuery(ev);
        if (e != cudaErrorNotReady) return e;
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

// ---------------------------------------------------------------------------
// Watchdog (see internal.hpp)
// ---------------------------------------------------------------------------
Watchdog::Watchdog(marsit_ctx* c) : ctx(c) {
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&ev_poll, cudaEventDisableTiming);
    cudaHostAlloc(reinterpret_cast<void**>(&h_flags), 2 * size_t(ctx->G) * sizeof(uint64_t),
                  cudaHostAllocDefault);
    cudaHostAlloc(reinterpret_cast<void**>(&h_abort), 2 * size_t(ctx->G) * sizeof(uint64_t),
                  cudaHostAllocDefault);
    if (h_abort)
        for (size_t i = 0; i < 2 * size_t(ctx->G); ++i) h_abort[i] = kFlagAbort;
    th = std::thread([this] { loop(); });
}

Watchdog::~Watchdog() {
    {
        std::lock_guard<std::mutex> lock(mu);
        stop = true;
    }
    cv.notify_all();
    if (th.joinable()) th.join();
    for (auto& it : pending) cudaEventDestroy(it.ev);
    for (auto e : free_events) cudaEventDestroy(e);
    if (h_flags) cudaFreeHost(h_flags);
    if (h_abort) cudaFreeHost(h_abort);
    if (ev_poll) cudaEventDestroy(ev_poll);
    if (st) cudaStreamDestroy(st);
}

marsit_status Watchdog::watch(cudaStream_t s, uint64_t epoch) {
    cudaEvent_t ev = nullptr;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (!free_events.empty()) {
            ev = free_events.back();
            free_events.pop_back();
        }
    }
    if (!ev) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    if (cudaEventRecord(ev, s) != cudaSuccess) {
        std::lock_guard<std::mutex> lock(mu);
        free_events.push_back(ev);
        return fail(MARSIT_ECUDA, std::string("watchdog event: ") + cudaGetErrorString(cudaGetLastError()));
    }
    {
        std::lock_guard<std::mutex> lock(mu);
        pending.push_back({ev, std::chrono::steady_clock::now(), epoch});
    }
    cv.notify_all();
    return MARSIT_OK;
}

// Mark the context failed and unblock everything it enqueued: P2P stream
// waits are released (kFlagAbort in the local flags) and the peers are told
// (kFlagAbort in this rank's slots of their flags); NCCL is aborted.
void Watchdog::give_up(marsit_status status, const std::string& msg) {
    ctx_set_failed(ctx, status, msg);
    if (ctx->p2p && h_abort) {
        const size_t n = 2 * size_t(ctx->G);
        cudaMemcpyAsync(ctx->flags, h_abort, n * sizeof(uint64_t), cudaMemcpyHostToDevice, st);
        for (uint32_t q = 0; q < ctx->G && q < ctx->peer_flags.size(); ++q) {
            if (q == ctx->rank || !ctx->peer_flags[q]) continue;
            for (int which = 0; which < 2; ++which)
                cudaMemcpyAsync(const_cast<uint64_t*>(ctx->peer_flags[q]) + size_t(which) * ctx->G + ctx->rank,
                                h_abort, sizeof(uint64_t), cudaMemcpyHostToDevice, st);
        }
        poll_stream(st, ev_poll);
    }
    if (ctx->comm && ctx->owns_comm) {
        // frees the communicator and unblocks its kernels; the context only
        // returns the latched failure from now on
        ncclCommAbort(ctx->comm);
        ctx->owns_comm = false;
    }
    cudaGetLastError();
}

void Watchdog::loop() {
    cudaSetDevice(ctx->device);
    std::unique_lock<std::mutex> lock(mu);
    while (!stop) {
        if (pending.empty()) {
            cv.wait(lock, [this] { return stop || !pending.empty(); });
            continue;
        }
        Item it = pending.front();
        lock.unlock();
        const cudaError_t q = cudaEventQuery(it.ev);
        bool done = q == cudaSuccess;
        if (q != cudaSuccess && q != cudaErrorNotReady) {
            ctx_set_failed(ctx, MARSIT_ECUDA, std::string("round failed: ") + cudaGetErrorString(q));
            done = true;
        }
        if (!done && !ctx->fail_status.load()) {
            std::string why;
            marsit_status status = MARSIT_EPROTOCOL;
            if (ctx->comm) {
                ncclResult_t ar = ncclSuccess;
                if (ncclCommGetAsyncError(ctx->comm, &ar) == ncclSuccess && ar != ncclSuccess &&
                    ar != ncclInProgress) {
                    status = MARSIT_ENCCL;
                    why = std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar);
                }
            }
            const auto waited = std::chrono::duration_cast<std::chrono::milliseconds>(
                                    std::chrono::steady_clock::now() - it.t0).count();
            if (why.empty() && ctx->p2p) {
                // which peers are missing (or announced an abort)
                const size_t n = 2 * size_t(ctx->G);
                if (cudaMemcpyAsync(h_flags, ctx->flags, n * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                    st) == cudaSuccess &&
                    poll_stream(st, ev_poll) == cudaSuccess) {
                    std::string missing;
                    for (uint32_t r = 0; r < ctx->G; ++r) {
                        if (r == ctx->rank) continue;
                        for (int which = 0; which < 2; ++which) {
                            const uint64_t v = h_flags[size_t(which) * ctx->G + r];
                            if (v == kFlagAbort)
                                why = "P2P: peer rank " + std::to_string(r) + " aborted";
                            else if (v < it.epoch && missing.empty())
                                missing = "peer rank " + std::to_string(r) + " has not reported " +
                                          (which ? "its owned aggregates" : "its packed signs") +
                                          " for epoch " + std::to_string(it.epoch) + " (last " +
                                          std::to_string(v) + ")";
                        }
                    }
                    if (why.empty() && ctx->wait_timeout_ms && uint64_t(waited) > ctx->wait_timeout_ms)
                        why = "P2P: round did not complete within " +
                              std::to_string(ctx->wait_timeout_ms) + " ms" +
                              (missing.empty() ? std::string() : ": " + missing);
                }
                cudaGetLastError();
            } else if (why.empty() && ctx->wait_timeout_ms && uint64_t(waited) > ctx->wait_timeout_ms) {
                status = ctx->comm ? MARSIT_ENCCL : MARSIT_EPROTOCOL;
                why = "round did not complete within " + std::to_string(ctx->wait_timeout_ms) + " ms";
            }
            if (!why.empty()) give_up(status, why);
        }
        lock.lock();
        if (done) {
            pending.pop_front();
            free_events.push_back(it.ev);
            continue;
        }
        if (ctx->fail_status.load()) {
            // released: the stream drains; keep the events until they complete
            cv.wait_for(lock, std::chrono::milliseconds(5));
            continue;
        }
        cv.wait_for(lock, std::chrono::milliseconds(20));
    }
}

marsit_status watch_round(marsit_ctx* ctx, cudaStream_t st) {
    if (!ctx->watchdog) return MARSIT_OK;
    return ctx->watchdog->watch(st, ctx->epoch);
}

// Lower the owned segments' merge DAGs: execution order = (stage, schedule
// order); outputs consumed by a later merge of the same stage get a
// shared-memory slot (liveness-based reuse, read-before-write within a
// thread), outputs consumed by a later stage get a global node, the final
// node goes to the aggregate.
marsit_status lower_plan(const Plan& plan, uint32_t s_first, uint32_t n_seg, DevicePlan& dp) {
    const uint32_t W = plan.workers;
    dp = DevicePlan{};
    dp.n_stages = plan.n_stages;
    dp.seg_begin.resize(n_seg);
    dp.stage_begin.assign(size_t(n_seg) * (plan.n_stages + 1), 0);
    dp.lane_begin.assign(size_t(n_seg) * plan.n_stages * (kMaxLanes + 1), 0);
    dp.n_lanes.assign(plan.n_stages, 1);
    const bool lanes = env_int("MARSIT_MERGE_LANES", 1) != 0;
    for (uint32_t sl = 0; sl < n_seg; ++sl) {
        const SegmentPlan& sp = plan.seg[s_first + sl];
        const size_t n = sp.merges.size();
        if (sp.final_node < W) return fail(MARSIT_EUNSUPPORTED, "schedule performs no reduction");
        // lanes: the connected components of each stage's same-stage
        // dependencies (torus: one row chain each), numbered by first
        // appearance; MARSIT_MERGE_LANES=0 keeps one lane per stage
        std::vector<uint32_t> root(n), lane(n, 0);
        for (size_t k = 0; k < n; ++k) root[k] = uint32_t(k);
        std::function<uint32_t(uint32_t)> find = [&](uint32_t x) {
            return root[x] == x ? x : (root[x] = find(root[x]));
        };
        for (size_t k = 0; k < n; ++k)
            for (uint32_t in : {sp.merges[k].recv_node, sp.merges[k].local_node})
                if (in >= W && sp.merges[in - W].stage == sp.merges[k].stage)
                    root[find(uint32_t(k))] = find(in - W);
        if (lanes) {
            std::vector<int> lane_of_root(n, -1);
            std::vector<uint32_t> next_lane(plan.n_stages, 0);
            for (size_t k = 0; k < n; ++k) {
                const uint32_t rt = find(uint32_t(k));
                if (lane_of_root[rt] < 0)
                    lane_of_root[rt] = int(std::min(next_lane[sp.merges[k].stage]++, kMaxLanes - 1));
                lane[k] = uint32_t(lane_of_root[rt]);
            }
        }
        std::vector<uint32_t> order(n);
        for (size_t k = 0; k < n; ++k) order[k] = uint32_t(k);
        std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
            if (sp.merges[a].stage != sp.merges[b].stage)
                return sp.merges[a].stage < sp.merges[b].stage;
            return lane[a] < lane[b];
        });
        std::vector<uint32_t> pos(n);  // schedule index -> execution index
        for (size_t e = 0; e < n; ++e) pos[order[e]] = uint32_t(e);
        std::vector<int> last_same(n, -1);
        std::vector<bool> cross(n, false);
        for (size_t e = 0; e < n; ++e) {
            const MergeNode& m = sp.merges[order[e]];
            for (uint32_t in : {m.recv_node, m.local_node}) {
                if (in < W) continue;
                const uint32_t src = in - W;
                if (sp.merges[src].stage == m.stage)
                    last_same[src] = std::max(last_same[src], int(e));
                else
                    cross[src] = true;
            }
        }
        std::vector<uint16_t> slot_of(n, kNone), gidx_of(n, kNone);
        std::vector<bool> slot_busy;
        uint32_t gnext = 0;
        dp.seg_begin[sl] = uint32_t(dp.merges.size());
        for (size_t e = 0; e < n; ++e) {
            const uint32_t k = order[e];
            const MergeNode& m = sp.merges[k];
            DevMerge d{};
            d.thresh11 = coin_threshold(m.c_recv, m.c_local) << 11;
            d.receiver = m.receiver;
            d.segment = s_first + sl;
            d.key_mode = 0;
            d.offset_src = m.offset_src < 0 ? int16_t(-1) : int16_t(pos[m.offset_src]);
            auto encode = [&](uint32_t node) -> uint16_t {
                if (node < W) return uint16_t(kSrcLeaf | node);
                const uint32_t src = node - W;
                if (sp.merges[src].stage == m.stage) return uint16_t(kSrcSlot | slot_of[src]);
                return uint16_t(kSrcGlobal | gidx_of[src]);
            };
            d.recv_src = encode(m.recv_node);
            d.local_src = encode(m.local_node);
            for (uint32_t in : {m.recv_node, m.local_node})
                if (in >= W && last_same[in - W] == int(e) && slot_of[in - W] != kNone)
                    slot_busy[slot_of[in - W]] = false;
            if (last_same[k] >= 0) {
                uint32_t s = 0;
                while (s < slot_busy.size() && slot_busy[s]) ++s;
                if (s == slot_busy.size()) slot_busy.push_back(false);
                slot_busy[s] = true;
                slot_of[k] = uint16_t(s);
                dp.max_slots = std::max<uint32_t>(dp.max_slots, uint32_t(slot_busy.size()));
            }
            d.out_slot = slot_of[k];
            if (W + k == sp.final_node) {
                d.out_global = kFinal;
            } else if (cross[k]) {
                gidx_of[k] = uint16_t(gnext++);
                d.out_global = gidx_of[k];
            } else {
                d.out_global = kNone;
            }
            dp.merges.push_back(d);
        }
        dp.gmax = std::max(dp.gmax, gnext);
        for (uint32_t st = 0; st <= plan.n_stages; ++st) {
            uint32_t c = 0;
            for (size_t e = 0; e < n; ++e)
                if (sp.merges[order[e]].stage < st) ++c;
            dp.stage_begin[size_t(sl) * (plan.n_stages + 1) + st] = c;
        }
        for (uint32_t st = 0; st < plan.n_stages; ++st)
            for (uint32_t ln = 0; ln <= kMaxLanes; ++ln) {
                uint32_t c = 0, used = 0;
                for (size_t e = 0; e < n; ++e) {
                    const MergeNode& m = sp.merges[order[e]];
                    if (m.stage < st || (m.stage == st && lane[order[e]] < ln)) ++c;
                    if (m.stage == st) used = std::max(used, lane[order[e]] + 1);
                }
                dp.lane_begin[(size_t(sl) * plan.n_stages + st) * (kMaxLanes + 1) + ln] = c;
                dp.n_lanes[st] = std::max(dp.n_lanes[st], used);
            }
        if (slot_busy.size() > 64 || gnext > 0x3FFF)
            return fail(MARSIT_EUNSUPPORTED, "merge plan too large");
    }
    dp.n_merges = uint32_t(dp.merges.size());
    return MARSIT_OK;
}

// Cluster plans: one cluster runs a segment's whole DAG, so there are no
// stages.  Merges are grouped into levels (ASAP over their operands and the
// stream they continue, at most kMaxLevelMerges per level: a torus's row
// chains advance side by side); every merge output except the final node
// lives in a shared-memory slot, reused in place when its only reader is the
// merge that overwrites it (the ring's running aggregate) or freed after the
// level of its last reader.
marsit_status lower_cluster_plan(const Plan& plan, uint32_t s_first, uint32_t n_seg, DevicePlan& dp) {
    const uint32_t W = plan.workers;
    dp = DevicePlan{};
    dp.n_stages = 1;
    dp.seg_begin.assign(size_t(n_seg) + 1, 0);
    dp.lvl_start.assign(size_t(n_seg) + 1, 0);
    for (uint32_t sl = 0; sl < n_seg; ++sl) {
        const SegmentPlan& sp = plan.seg[s_first + sl];
        const size_t n = sp.merges.size();
        if (sp.final_node < W) return fail(MARSIT_EUNSUPPORTED, "schedule performs no reduction");
        if (n > size_t(kMaxSegMerges))
            return fail(MARSIT_EUNSUPPORTED, "merge plan too large (more than 64 merges per segment)");
        std::vector<int> lvl(n, 0);
        std::vector<uint32_t> width;
        for (size_t k = 0; k < n; ++k) {  // schedule order is topological
            const MergeNode& m = sp.merges[k];
            int L = 0;
            for (uint32_t in : {m.recv_node, m.local_node})
                if (in >= W) L = std::max(L, lvl[in - W] + 1);
            if (m.offset_src >= 0) L = std::max(L, lvl[m.offset_src] + 1);
            while (size_t(L) < width.size() && width[L] >= uint32_t(kMaxLevelMerges)) ++L;
            if (size_t(L) >= width.size()) width.resize(L + 1, 0);
            ++width[L];
            lvl[k] = L;
        }
        std::vector<uint32_t> order(n);
        for (size_t k = 0; k < n; ++k) order[k] = uint32_t(k);
        std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return lvl[a] < lvl[b]; });
        std::vector<uint32_t> pos(n);
        for (size_t e = 0; e < n; ++e) pos[order[e]] = uint32_t(e);
        // readers of every merge output: last level, count per level
        std::vector<int> last(n, -1);
        for (size_t k = 0; k < n; ++k)
            for (uint32_t in : {sp.merges[k].recv_node, sp.merges[k].local_node})
                if (in >= W) last[in - W] = std::max(last[in - W], lvl[k]);
        auto readers_at = [&](uint32_t node, int level) {
            int c = 0;
            for (size_t k = 0; k < n; ++k)
                if (lvl[k] == level)
                    for (uint32_t in : {sp.merges[k].recv_node, sp.merges[k].local_node})
                        c += in == W + node;
            return c;
        };
        std::vector<uint16_t> slot_of(n, kNone);
        std::vector<int> owner;  // slot -> node holding it (-1 free)
        dp.seg_begin[sl] = uint32_t(dp.merges.size());
        dp.lvl_start[sl] = uint32_t(dp.lvl_begin.size());
        size_t e = 0;
        for (int v = 0; v < int(width.size()); ++v) {
            dp.lvl_begin.push_back(uint32_t(e));
            dp.level_width = std::max(dp.level_width, width[v]);
            for (; e < n && lvl[order[e]] == v; ++e) {
                const uint32_t k = order[e];
                const MergeNode& m = sp.merges[k];
                DevMerge d{};
                d.thresh11 = coin_threshold(m.c_recv, m.c_local) << 11;
                d.receiver = m.receiver;
                d.segment = s_first + sl;
                d.key_mode = 0;
                d.offset_src = m.offset_src < 0 ? int16_t(-1) : int16_t(pos[m.offset_src]);
                auto encode = [&](uint32_t node) -> uint16_t {
                    if (node < W) return uint16_t(kSrcLeaf | node);
                    return uint16_t(kSrcSlot | slot_of[node - W]);
                };
                d.recv_src = encode(m.recv_node);
                d.local_src = encode(m.local_node);
                d.out_slot = kNone;
                d.out_global = kNone;
                if (W + k == sp.final_node) {
                    d.out_global = kFinal;
                } else {
                    uint16_t sl_out = kNone;
                    for (uint32_t in : {m.recv_node, m.local_node})  // in place
                        if (sl_out == kNone && in >= W && slot_of[in - W] != kNone &&
                            last[in - W] == v && readers_at(in - W, v) == 1)
                            sl_out = slot_of[in - W];
                    if (sl_out == kNone) {
                        size_t f = 0;
                        while (f < owner.size() && owner[f] >= 0) ++f;
                        if (f == owner.size()) owner.push_back(-1);
                        sl_out = uint16_t(f);
                    }
                    owner[sl_out] = int(k);
                    slot_of[k] = sl_out;
                    d.out_slot = sl_out;
                    dp.max_slots = std::max<uint32_t>(dp.max_slots, uint32_t(owner.size()));
                }
                dp.merges.push_back(d);
            }
            // slots whose node was last read at this level are free again
            for (size_t f = 0; f < owner.size(); ++f)
                if (owner[f] >= 0 && last[owner[f]] <= v) owner[f] = -1;
        }
        dp.lvl_begin.push_back(uint32_t(n));
        if (owner.size() > 0x3FFF) return fail(MARSIT_EUNSUPPORTED, "merge plan too large");
    }
    dp.seg_begin[n_seg] = uint32_t(dp.merges.size());
    dp.lvl_start[n_seg] = uint32_t(dp.lvl_begin.size());
    dp.n_merges = uint32_t(dp.merges.size());
    return MARSIT_OK;
}

}  // namespace marsit_b200

marsit_ctx::~marsit_ctx() {
    if (device >= 0) cudaSetDevice(device);
    watchdog.reset();  // joins the thread before any buffer it reads goes away
    for (void* p : {(void*)bits, (void*)recv, (void*)agg, (void*)err, dense_send, dense_recv,
                    dense_mean, (void*)d_dense_ops, (void*)d_dense_final, (void*)d_metrics,
                    (void*)d_verify,
                    (void*)d_dense_chain, (void*)d_dense_groups,
                    (void*)flags, (void*)d_peer_tables, (void*)spread_sync, (void*)spread_coins[0],
                    (void*)spread_coins[1], (void*)spread_valid[0], (void*)spread_valid[1],
                    (void*)spread_tag, (void*)spread_cend})
        if (p) cudaFree(p);
    for (auto& tp : pending) {
        cudaEventDestroy(tp.a);
        cudaEventDestroy(tp.b);
    }
    for (auto e : event_pool) cudaEventDestroy(e);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_check) cudaEventDestroy(ev_check);
    if (h_check) cudaFreeHost(h_check);
    if (ev_extract) cudaEventDestroy(ev_extract);
    for (auto e : ev_merge) cudaEventDestroy(e);
    for (int b = 0; b < 2; ++b) {
        if (ev_coin_done[b]) cudaEventDestroy(ev_coin_done[b]);
        if (coin_buf[b]) cudaFree(coin_buf[b]);
        if (coin_valid[b]) cudaFree(coin_valid[b]);
    }
    if (aux) cudaStreamDestroy(aux);
    if (comm && owns_comm) ncclCommDestroy(comm);
}

marsit_status marsit_ctx::begin_phase(cudaStream_t st, cudaEvent_t* a) {
    *a = nullptr;
    if (!timing) return MARSIT_OK;
    if (event_pool.empty()) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreate(&e));
        event_pool.push_back(e);
    }
    *a = event_pool.back();
    event_pool.pop_back();
    CUDA_TRY(cudaEventRecord(*a, st));
    return MARSIT_OK;
}

marsit_status marsit_ctx::end_phase(int phase, cudaStream_t st, cudaEvent_t a, uint64_t n_launch) {
    launches[phase] += n_launch;
    if (!timing || !a) return MARSIT_OK;
    cudaEvent_t b;
    if (event_pool.empty()) {
        CUDA_TRY(cudaEventCreate(&b));
    } else {
        b = event_pool.back();
        event_pool.pop_back();
    }
    CUDA_TRY(cudaEventRecord(b, st));
    pending.push_back({phase, a, b});
    return MARSIT_OK;
}

namespace {

enum Phase { kPhExtract = 0, kPhExchange, kPhMerge, kPhAllgather, kPhDecode, kPhExport, kPhDense,
             kPhCoins, kPhFused, kPhSpread };

template <typename T>
StreamParams<T> stream_params(marsit_ctx* ctx, const void* const* g, const void* const* c,
                              void* const* c_out, void* update, double eta,
                              void* const* params = nullptr) {
    StreamParams<T> p{};
    for (uint32_t w = 0; w < ctx->ml; ++w) {
        p.g[w] = static_cast<const T*>(g[w]);
        p.c[w] = static_cast<const T*>(c[w]);
        p.c_out[w] = c_out ? static_cast<T*>(c_out[w]) : nullptr;
        p.x[w] = params ? static_cast<T*>(params[w]) : nullptr;
    }
    p.ml = ctx->ml;
    p.n_seg = ctx->S;
    p.seg0 = 0;
    p.n_proc = ctx->S;
    p.dim = ctx->D;
    p.seg_len = ctx->L;
    p.words_proc = ctx->words_proc;
    p.wst = ctx->wst;
    p.bits = ctx->bits;
    p.agg = ctx->agg;
    p.wsa = ctx->wsa;
    p.update = static_cast<T*>(update);
    p.eta = T(eta);
    p.err = ctx->err;
    return p;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool vec_ok_ptrs(const marsit_ctx* ctx, const void* const* a, const void* const* b) {
    if (!ctx->vec_ok) return false;
    for (uint32_t w = 0; w < ctx->ml; ++w)
        if (!aligned16(a[w]) || !aligned16(b[w])) return false;
    return true;
}

marsit_status check_ptrs(const marsit_ctx* ctx, const void* const* a, const char* what) {
    if (!a) return fail(MARSIT_EPARAM, std::string(what) + " is null");
    for (uint32_t w = 0; w < ctx->ml; ++w)
        if (!a[w]) return fail(MARSIT_EPARAM, std::string(what) + " has a null worker pointer");
    return MARSIT_OK;
}

// K1 over all segments of the local workers.
marsit_status run_extract(marsit_ctx* ctx, const void* const* g, const void* const* c,
                          cudaStream_t st) {
    cudaEvent_t ev;
    marsit_status s = ctx->begin_phase(st, &ev);
    if (s) return s;
    const bool vec = vec_ok_ptrs(ctx, g, c);
    if (ctx->dtype == MARSIT_F32) {
        auto p = stream_params<float>(ctx, g, c, nullptr, nullptr, 0.0);
        p.reverse = ctx->task_dir;
        CUDA_TRY(launch_extract(p, vec, ctx->extract_grid, st));
    } else {
        auto p = stream_params<double>(ctx, g, c, nullptr, nullptr, 0.0);
        p.reverse = ctx->task_dir;
        CUDA_TRY(launch_extract(p, vec, ctx->extract_grid, st));
    }
    return ctx->end_phase(kPhExtract, st, ev, 1);
}

// NCCL all-to-all of the packed segments: destination q receives this rank's
// local workers' bits of the segments it owns (one contiguous block).
marsit_status run_exchange(marsit_ctx* ctx, cudaStream_t st) {
    if (ctx->G == 1 || !ctx->comm) return MARSIT_OK;  // external transport: the caller's
    cudaEvent_t ev;
    marsit_status s = ctx->begin_phase(st, &ev);
    if (s) return s;
    const size_t block = size_t(ctx->s_own) * ctx->ml * ctx->wst;  // u32 words per destination
    NCCL_TRY(ncclGroupStart());
    for (uint32_t q = 0; q < ctx->G; ++q) {
        NCCL_TRY(ncclSend(ctx->bits + q * block, block, ncclUint32, int(q), ctx->comm, st));
        NCCL_TRY(ncclRecv(ctx->recv + q * block, block, ncclUint32, int(q), ctx->comm, st));
    }
    NCCL_TRY(ncclGroupEnd());
    return ctx->end_phase(kPhExchange, st, ev, 0);
}

// Launch the coin kernel for (seed, round) into buffer b on the aux stream,
// forked from `st` at this point of its work.
marsit_status launch_coin_buffer(marsit_ctx* ctx, int b, uint64_t seed, uint64_t round,
                                 cudaStream_t st) {
    CUDA_TRY(cudaEventRecord(ctx->ev_fork, st));
    CUDA_TRY(cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0));
    cudaEvent_t ev;
    marsit_status s = ctx->begin_phase(ctx->aux, &ev);
    if (s) return s;
    CUDA_TRY(launch_coins(ctx->merge.d_merges, ctx->merge.dp.n_merges, seed, round,
                          ctx->merge.coin_end, ctx->coin_valid[b], ctx->coin_buf[b],
                          ctx->coin_grid_x, ctx->aux));
    if ((s = ctx->end_phase(kPhCoins, ctx->aux, ev, 1))) return s;
    CUDA_TRY(cudaEventRecord(ctx->ev_coin_done[b], ctx->aux));
    ctx->coin_tag[b] = {true, seed, round};
    return MARSIT_OK;
}

// Coins of this round: reuse the speculatively prefetched buffer when its tag
// matches (seed, round); otherwise compute them now, overlapping the extract.
// ---------------------------------------------------------------------------
// P2P transport: stream-ordered epoch flags (driver stream memory operations,
// resolved at run time so the library does not link libcuda).
// ---------------------------------------------------------------------------
using PfnStreamValue64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
struct StreamMemOps {
    PfnStreamValue64 wait = nullptr, write = nullptr;
};
const StreamMemOps& stream_memops() {
    static StreamMemOps ops;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            ops.wait = reinterpret_cast<PfnStreamValue64>(f);
        f = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            ops.write = reinterpret_cast<PfnStreamValue64>(f);
        cudaGetLastError();
    });
    return ops;
}

// Flags: every rank owns 2 x G u64 slots, flags[which * G + q] = the last
// epoch rank q reported for `which` (0: phase-0 data ready, 1: owned results
// ready).  A rank signals by writing its slot in every rank's array (remote
// stream writes, each preceded by a system-wide fence) and waits only on its
// own, local array — polling never crosses NVLink.
marsit_status p2p_signal(marsit_ctx* ctx, int which, cudaStream_t st) {
    if (!ctx->p2p) return MARSIT_OK;
    const StreamMemOps& m = stream_memops();
    FlagSlots fs{};
    for (uint32_t q = 0; q < ctx->G; ++q) {
        if (q == ctx->rank) continue;
        uint64_t* slot = const_cast<uint64_t*>(ctx->peer_flags[q]) + size_t(which) * ctx->G + ctx->rank;
        if (m.write && !ctx->flag_kernel) {
            const CUresult r = m.write(reinterpret_cast<CUstream>(st),
                                       reinterpret_cast<CUdeviceptr>(slot), ctx->epoch, 0);
            if (r == CUDA_SUCCESS) continue;
            ctx->flag_kernel = true;  // stream writes to peer memory unsupported: store from a kernel
        }
        fs.slot[fs.n++] = reinterpret_cast<unsigned long long*>(slot);
    }
    if (fs.n) CUDA_TRY(launch_flag_write(fs, ctx->epoch, st));
    return MARSIT_OK;
}

// The stream waits until every peer has reported this epoch for `which`.
marsit_status p2p_wait(marsit_ctx* ctx, int which, cudaStream_t st) {
    if (!ctx->p2p) return MARSIT_OK;
    const StreamMemOps& m = stream_memops();
    if (!m.wait) return fail(MARSIT_EUNSUPPORTED, "cuStreamWaitValue64 unavailable");
    for (uint32_t q = 0; q < ctx->G; ++q) {
        if (q == ctx->rank) continue;  // own work: stream order already holds
        const uint64_t* slot = ctx->flags + size_t(which) * ctx->G + q;
        const CUresult r = m.wait(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(slot),
                                  ctx->epoch, CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) return fail(MARSIT_ECUDA, "cuStreamWaitValue64 failed");
    }
    return MARSIT_OK;
}

const uint32_t* const* p2p_table(const marsit_ctx* ctx, int which) {
    return ctx->p2p ? reinterpret_cast<const uint32_t* const*>(ctx->d_peer_tables + size_t(which) * ctx->G)
                    : nullptr;
}

marsit_status run_coins(marsit_ctx* ctx, uint64_t seed, uint64_t round, cudaStream_t st) {
    if (ctx->coin_total_words == 0) return MARSIT_OK;
    for (int b = 0; b < 2; ++b)
        if (ctx->coin_tag[b].valid && ctx->coin_tag[b].seed == seed &&
            ctx->coin_tag[b].round == round) {
            ctx->cur_coin = b;
            // prefetched underneath the last decode: only the merge needs the
            // coins, so the extract may overlap the tail of the prefetch (small
            // rounds: the coin kernel outlasts the decode); run_merge waits
            ctx->coins_pending = true;
            return MARSIT_OK;
        }
    const int b = 1 - ctx->cur_coin;
    marsit_status s = launch_coin_buffer(ctx, b, seed, round, st);
    if (s) return s;
    ctx->cur_coin = b;
    ctx->coins_pending = true;
    return MARSIT_OK;
}

// After this round's merge is enqueued: precompute (seed, round + 1) into the
// other buffer; it runs underneath the HBM-bound decode.
marsit_status prefetch_coins(marsit_ctx* ctx, uint64_t seed, uint64_t round, cudaStream_t st) {
    if (ctx->coin_total_words == 0 || !ctx->coin_prefetch) return MARSIT_OK;
    return launch_coin_buffer(ctx, 1 - ctx->cur_coin, seed, round + 1, st);
}

marsit_status run_merge(marsit_ctx* ctx, uint64_t seed, uint64_t round, cudaStream_t st) {
    if (ctx->coins_pending) {
        CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_coin_done[ctx->cur_coin], 0));
        ctx->coins_pending = false;
    }
    cudaEvent_t ev;
    marsit_status s = ctx->begin_phase(st, &ev);
    if (s) return s;
    uint64_t n = 0;
    if ((s = ctx->merge.run(ctx->G == 1 ? ctx->bits : ctx->recv, ctx->agg,
                            ctx->coin_buf[ctx->cur_coin], seed, round, st, &n, 0, ~0u,
                            ctx->coin_valid[ctx->cur_coin])))
        return s;
    return ctx->end_phase(kPhMerge, st, ev, n);
}

marsit_status run_allgather(marsit_ctx* ctx, cudaStream_t st) {
    if (ctx->G == 1 || !ctx->comm) return MARSIT_OK;
    cudaEvent_t ev;
    marsit_status s = ctx->begin_phase(st, &ev);
    if (s) return s;
    const size_t block = size_t(ctx->s_own) * ctx->wsa;  // rows incl. the consensus hash slots
    NCCL_TRY(ncclAllGather(ctx->agg + ctx->rank * block, ctx->agg, block, ncclUint32, ctx->comm, st));
    return ctx->end_phase(kPhAllgather, st, ev, 0);
}

marsit_status run_decode(marsit_ctx* ctx, const void* const* g, const void* const* c,
                         void* const* c_out, void* const* params, void* update, double eta,
                         cudaStream_t st, uint32_t seg0 = 0, uint32_t n = 0) {
    cudaEvent_t ev;
    marsit_status s = ctx->begin_phase(st, &ev);
    if (s) return s;
    const bool vec = vec_ok_ptrs(ctx, g, c) && vec_ok_ptrs(ctx, (const void* const*)c_out, c) &&
                     (!params || vec_ok_ptrs(ctx, (const void* const*)params, c)) &&
                     (!update || aligned16(update));
    if (!n) n = ctx->S;
    // matching count fused into the decode (needs every worker local)
    unsigned long long* matches = nullptr;
    if (ctx->metrics && ctx->ml == ctx->M) {
        if (seg0 == 0) CUDA_TRY(cudaMemsetAsync(ctx->d_metrics, 0, sizeof(unsigned long long), st));
        matches = ctx->d_metrics;
        ctx->last_matching = true;
    }
    if (ctx->dtype == MARSIT_F32) {
        auto p = stream_params<float>(ctx, g, c, c_out, update, eta, params);
        p.seg0 = seg0;
        p.n_proc = n;
        p.matches = matches;
        p.n_workers = ctx->M;
        p.agg_peers = p2p_table(ctx, 1);
        p.s_own = ctx->s_own;
        p.reverse = ctx->l2_reuse ? ctx->task_dir ^ 1u : 0u;
        CUDA_TRY(launch_decode(p, vec, matches ? ctx->stats_grid : ctx->decode_grid, st));
    } else {
        auto p = stream_params<double>(ctx, g, c, c_out, update, eta, params);
        p.seg0 = seg0;
        p.n_proc = n;
        p.matches = matches;
        p.n_workers = ctx->M;
        p.agg_peers = p2p_table(ctx, 1);
        p.s_own = ctx->s_own;
        p.reverse = ctx->l2_reuse ? ctx->task_dir ^ 1u : 0u;
        CUDA_TRY(launch_decode(p, vec, matches ? ctx->stats_grid : ctx->decode_grid, st));
    }
    return ctx->end_phase(kPhDecode, st, ev, 1);
}

marsit_status run_export(marsit_ctx* ctx, uint64_t* out, cudaStream_t st) {
    if (!out) return MARSIT_OK;
    cudaEvent_t ev;
    marsit_status s = ctx->begin_phase(st, &ev);
    if (s) return s;
    CUDA_TRY(launch_export_bits(ctx->agg, ctx->wsa, ctx->D, ctx->L,
                                reinterpret_cast<uint32_t*>(out), st, p2p_table(ctx, 1), ctx->s_own));
    return ctx->end_phase(kPhExport, st, ev, 1);
}

marsit_status check_consensus(const marsit_ctx* ctx, bool need_full_count) {
    for (uint32_t s = 0; s < ctx->S; ++s) {
        const SegmentPlan& sp = ctx->plan.seg[s];
        if (!sp.consensus) return fail(MARSIT_EPROTOCOL, "consensus: workers disagree");
        if (need_full_count && sp.final_count != ctx->M)
            return fail(MARSIT_EPROTOCOL, "marsit_round: aggregate is missing contributions");
    }
    return MARSIT_OK;
}

// Dense round in three phases around the two exchange points (G > 1):
//   0: u = g + c of the local workers, laid out per destination rank
//   [exchange of u blocks]
//   1: owner-side schedule-order sum of the owned segments, x 1/M
//   [all-gather of the owned mean blocks]
//   2: mean out, compensation = 0 (sync.hpp:83-85), optional x -= mean
// With G == 1 phase 1 reads g and c directly and writes `mean`.
template <typename T>
marsit_status dense_phase(marsit_ctx* ctx, int phase, const void* const* g, const void* const* c,
                          void* const* c_out, void* const* params, void* mean, cudaStream_t st) {
    NvtxRange range(phase == 0 ? "marsit.dense.leaf" : phase == 1 ? "marsit.dense.sum" : "marsit.dense.out");
    cudaEvent_t ev;
    marsit_status s = ctx->begin_phase(st, &ev);
    if (s) return s;
    DenseParams<T> p{};
    p.chain = ctx->d_dense_chain;
    p.chain_groups = ctx->d_dense_groups;
    p.chain_multi = ctx->dense_multi;
    p.ops = ctx->d_dense_ops;
    p.final_node = ctx->d_dense_final;
    p.n_ops = ctx->dense_n_ops;
    p.n_seg = ctx->s_own;
    p.s_first = ctx->s_first;
    p.ml = ctx->ml;
    p.workers = ctx->M;
    p.dim = ctx->D;
    p.seg_len = ctx->L;
    p.inv_m = 1.0 / double(ctx->M);
    p.err = ctx->err;
    uint64_t launches = 0;
    if (phase == 1 && (s = p2p_wait(ctx, 0, st))) return s;
    if (phase == 2 && (s = p2p_wait(ctx, 1, st))) return s;
    if (phase == 0 && ctx->G > 1) {
        std::vector<const T*> gg(ctx->ml), cc(ctx->ml);
        std::vector<T*> zz(ctx->ml);
        for (uint32_t w = 0; w < ctx->ml; ++w) {
            gg[w] = static_cast<const T*>(g[w]);
            cc[w] = static_cast<const T*>(c[w]);
            zz[w] = static_cast<T*>(c_out[w]);  // c' = 0 (sync.hpp:83-85), fused
        }
        CUDA_TRY(launch_dense_leaf<T>(gg.data(), cc.data(), ctx->ml, ctx->D, ctx->L, ctx->S,
                                      ctx->s_own, static_cast<T*>(ctx->dense_send), ctx->err,
                                      ctx->stream_grid, st, zz.data()));
        ++launches;
    } else if (phase == 1) {
        if (ctx->G == 1) {
            p.mode = 0;
            for (uint32_t w = 0; w < ctx->ml; ++w) {
                p.src[2 * w] = static_cast<const T*>(g[w]);
                p.src[2 * w + 1] = static_cast<const T*>(c[w]);
                p.c_zero[w] = static_cast<T*>(c_out[w]);  // c' = 0 (sync.hpp:83-85), fused
            }
            p.mean = static_cast<T*>(mean);
            p.vec4 = ctx->L % 4 == 0 && ctx->D % 4 == 0 && aligned16(mean) &&
                     vec_ok_ptrs(ctx, g, c) && vec_ok_ptrs(ctx, (const void* const*)c_out, c);
        } else {
            p.mode = ctx->p2p ? 2 : 1;
            p.u_buf = static_cast<const T*>(ctx->dense_recv);
            p.u_peers = reinterpret_cast<const T* const*>(ctx->d_peer_tables + 2 * size_t(ctx->G));
            p.mean = static_cast<T*>(ctx->dense_mean);  // padded [S*L]; owned block written
            p.dim = uint64_t(ctx->S) * ctx->L;
        }
        CUDA_TRY(launch_dense_reduce(p, ctx->stream_grid, st));
        ++launches;
    } else if (phase == 2) {
        if (ctx->p2p) {  // every owner's block straight from its buffer (peer copies)
            const size_t block = size_t(ctx->s_own) * ctx->L;
            for (uint32_t q = 0; q < ctx->G; ++q) {
                const size_t off = q * block;
                if (off >= ctx->D) break;
                const size_t n = std::min<size_t>(block, ctx->D - off);
                CUDA_TRY(cudaMemcpyAsync(static_cast<T*>(mean) + off,
                                         static_cast<const T*>(ctx->peer_dense_mean[q]) + off,
                                         n * sizeof(T), cudaMemcpyDefault, st));
            }
        } else if (ctx->G > 1) {
            CUDA_TRY(cudaMemcpyAsync(mean, ctx->dense_mean, ctx->D * sizeof(T),
                                     cudaMemcpyDeviceToDevice, st));
        }
        if (params) {  // x_w -= mean (trainer.hpp:285-288)
            std::vector<T*> xs(ctx->ml);
            for (uint32_t w = 0; w < ctx->ml; ++w) xs[w] = static_cast<T*>(params[w]);
            CUDA_TRY(launch_sub_update<T>(xs.data(), ctx->ml, static_cast<const T*>(mean),
                                          ctx->D, ctx->stream_grid, st));
            ++launches;
        }
    }
    if ((s = ctx->end_phase(kPhDense, st, ev, launches))) return s;
    if (phase == 0) {
        if (ctx->p2p) ++ctx->epoch;  // after this rank's phase-0 launches
        return p2p_signal(ctx, 0, st);  // my u blocks are ready
    }
    if (phase == 1) return p2p_signal(ctx, 1, st);  // my owned mean block is ready
    return MARSIT_OK;
}

marsit_status dense_exchange(marsit_ctx* ctx, cudaStream_t st) {
    if (ctx->G == 1 || !ctx->comm) return MARSIT_OK;  // external transport: the caller's
    const size_t block = size_t(ctx->s_own) * ctx->ml * ctx->L;
    const ncclDataType_t dt = ctx->esize == 4 ? ncclFloat32 : ncclFloat64;
    NCCL_TRY(ncclGroupStart());
    for (uint32_t q = 0; q < ctx->G; ++q) {
        NCCL_TRY(ncclSend(static_cast<char*>(ctx->dense_send) + q * block * ctx->esize, block, dt,
                          int(q), ctx->comm, st));
        NCCL_TRY(ncclRecv(static_cast<char*>(ctx->dense_recv) + q * block * ctx->esize, block, dt,
                          int(q), ctx->comm, st));
    }
    NCCL_TRY(ncclGroupEnd());
    return MARSIT_OK;
}

marsit_status dense_allgather(marsit_ctx* ctx, cudaStream_t st) {
    if (ctx->G == 1 || !ctx->comm) return MARSIT_OK;
    const size_t seg_block = size_t(ctx->s_own) * ctx->L;
    const ncclDataType_t dt = ctx->esize == 4 ? ncclFloat32 : ncclFloat64;
    char* full = static_cast<char*>(ctx->dense_mean);
    NCCL_TRY(ncclAllGather(full + ctx->rank * seg_block * ctx->esize, full, seg_block, dt,
                           ctx->comm, st));
    return MARSIT_OK;
}

marsit_status dense_phase_any(marsit_ctx* ctx, int phase, const void* const* g,
                              const void* const* c, void* const* c_out, void* const* params,
                              void* mean, cudaStream_t st) {
    if (ctx->dtype == MARSIT_F32) return dense_phase<float>(ctx, phase, g, c, c_out, params, mean, st);
    return dense_phase<double>(ctx, phase, g, c, c_out, params, mean, st);
}

// Dense reduction tree of one segment (node < M: leaf; else op node - M)
// as groups of leaves: value = fold(fold(G_1), fold(G_2), ...) with
// fold(x_1, ..., x_n) = (((x_1 + x_2) + x_3) ... + x_n).  Returns false when
// the tree has another shape.  The order of the two operands of one add is
// immaterial (IEEE addition is commutative); the tree shape is reproduced
// exactly.
static bool chain_of_chains(const DenseOp* ops, uint32_t M, uint32_t fin,
                            std::vector<uint16_t>& order, uint64_t& group_ends) {
    order.clear();
    group_ends = 0;
    if (M > 64 || fin < M) return false;
    const uint32_t n_nodes = fin + 1;  // ops are in topological order: fin is the last
    auto leaf = [&](uint32_t n) { return n < M; };
    // chain[n]: n is a left-deep chain whose every add takes one leaf
    std::vector<uint8_t> chain(n_nodes, 0);
    for (uint32_t n = 0; n < n_nodes; ++n) {
        if (leaf(n)) {
            chain[n] = 1;
            continue;
        }
        const DenseOp& o = ops[n - M];
        if (o.a >= n || o.b >= n) return false;
        chain[n] = (leaf(o.b) && chain[o.a]) || (leaf(o.a) && chain[o.b]);
    }
    auto flatten = [&](uint32_t n, std::vector<uint16_t>& out) {
        std::vector<uint16_t> rev;
        while (!leaf(n)) {
            const DenseOp& o = ops[n - M];
            if (leaf(o.b) && chain[o.a]) {
                rev.push_back(o.b);
                n = o.a;
            } else {
                rev.push_back(o.a);
                n = o.b;
            }
        }
        rev.push_back(uint16_t(n));
        out.insert(out.end(), rev.rbegin(), rev.rend());
    };
    // dec[n]: n = fold over groups; the prefix operand of each outer add is
    // itself decomposable and the other operand is one group (a chain)
    std::vector<int8_t> dec(n_nodes, -1);
    std::vector<uint32_t> pre(n_nodes, 0), grp_of(n_nodes, 0);
    for (uint32_t n = 0; n < n_nodes; ++n) {
        if (chain[n]) {
            dec[n] = 1;
            pre[n] = ~0u;  // a single group
            continue;
        }
        const DenseOp& o = ops[n - M];
        dec[n] = 0;
        if (chain[o.b] && dec[o.a] == 1) {
            dec[n] = 1, pre[n] = o.a, grp_of[n] = o.b;
        } else if (chain[o.a] && dec[o.b] == 1) {
            dec[n] = 1, pre[n] = o.b, grp_of[n] = o.a;
        }
    }
    if (dec[fin] != 1) return false;
    std::vector<uint32_t> groups;  // group roots, last first
    uint32_t n = fin;
    while (pre[n] != ~0u) {
        groups.push_back(grp_of[n]);
        n = pre[n];
    }
    groups.push_back(n);
    std::vector<bool> seen(M, false);
    uint32_t k = 0;
    for (auto it = groups.rbegin(); it != groups.rend(); ++it) {
        const size_t before = order.size();
        flatten(*it, order);
        for (size_t i = before; i < order.size(); ++i) {
            if (seen[order[i]]) return false;  // every leaf exactly once
            seen[order[i]] = true;
        }
        k += uint32_t(order.size() - before);
        group_ends |= 1ull << (k - 1);
    }
    return order.size() == M;
}

// Coin precompute budget per merge: frac * L draws per use of its (receiver,
// segment) stream (a continuation merge starts after the earlier merges'
// draws).  Draws beyond it are computed inline by K2, so the budget only
// trades memory/ALU for the rare over-budget case.
void assign_coin_budget(DevicePlan& dp, uint32_t n_seg, uint64_t L, double frac,
                        uint64_t* total_words, uint64_t* max_words) {
    uint64_t off = 0, mx = 0;
    for (uint32_t sl = 0; sl < n_seg; ++sl) {
        const uint32_t mb = dp.seg_begin[sl];
        const uint32_t me = sl + 1 < n_seg ? dp.seg_begin[sl + 1] : dp.n_merges;
        for (uint32_t k = mb; k < me; ++k) {
            DevMerge& d = dp.merges[k];
            uint32_t depth = 0;
            for (int32_t src = d.offset_src; src >= 0; src = dp.merges[mb + src].offset_src) ++depth;
            // capacity: every draw the stream can make (the coin kernel
            // computes only what the last round's draw count calls for)
            const double want = frac * double(L) * (depth + 1);
            const uint64_t cap = frac > 0 ? ceil_div(L * (depth + 1), 32) : 0;
            uint64_t words = cap;
            d.coin_default = uint32_t(std::min<uint64_t>(cap, ceil_div(uint64_t(want) + 1, 32)));
            d.coin_words = uint32_t(words);
            d.coin_off = off;
            off += round_up(words, 64);  // whole 64-word chunks (coins_kernel)
            mx = std::max(mx, words);
        }
    }
    *total_words = off;
    *max_words = mx;
}

}  // namespace

namespace marsit_b200 {

// Opt-in consensus, owner side (after the merge, before the aggregates are
// published): the hash of every owned segment into its row's hash slot.
marsit_status consensus_own(marsit_ctx* ctx, cudaStream_t st) {
    if (!ctx->consensus) return MARSIT_OK;
    CUDA_TRY(cudaMemset2DAsync(ctx->agg + size_t(ctx->s_first) * ctx->wsa + ctx->wst,
                               size_t(ctx->wsa) * 4, 0, sizeof(uint64_t), ctx->s_own, st));
    CUDA_TRY(launch_seg_hash(ctx->agg, nullptr, 1, ctx->wsa, ctx->wst, ctx->words_proc,
                             ctx->s_first, ctx->s_own, nullptr, st));
    return MARSIT_OK;
}

// Reader side (after the decode): every segment re-hashed as this rank reads
// it and compared with its owner's hash (consensus, allreduce.hpp:32-43).
marsit_status consensus_verify(marsit_ctx* ctx, cudaStream_t st) {
    if (!ctx->consensus) return MARSIT_OK;
    if (!ctx->d_verify) CUDA_TRY(cudaMalloc(&ctx->d_verify, sizeof(unsigned long long) * ctx->S));
    CUDA_TRY(cudaMemsetAsync(ctx->d_verify, 0, sizeof(unsigned long long) * ctx->S, st));
    const uint32_t* const* peers = p2p_table(ctx, 1);
    CUDA_TRY(launch_seg_hash(ctx->agg, peers, ctx->s_own, ctx->wsa, ctx->wst, ctx->words_proc, 0,
                             ctx->S, ctx->d_verify, st));
    CUDA_TRY(launch_hash_compare(ctx->agg, peers, ctx->s_own, ctx->wsa, ctx->wst, ctx->S,
                                 ctx->d_verify, ctx->err, st));
    return MARSIT_OK;
}

// Sign round phases around the two exchange points:
//   0: coins (aux) + extract  ->  [exchange of packed segments]
//   1: merge of the owned segments (+ next round's coin prefetch)
//      ->  [all-gather of the owned aggregates]
//   2: decode + compensation (+ fused replica update) + export
marsit_status sign_phase(marsit_ctx* ctx, int phase, uint64_t t, double eta_s, uint64_t seed,
                         const void* const* d_grads, const void* const* d_comp,
                         void* const* d_comp_out, void* const* params, uint64_t* d_agg_bits,
                         void* d_update, cudaStream_t st) {
    marsit_status s = MARSIT_OK;
    NvtxRange range(phase == 0 ? "marsit.extract" : phase == 1 ? "marsit.merge" : "marsit.decode");
    // where the next round's coins run: underneath the decode by default;
    // underneath the extract when the metrics decode runs (its 3 CTAs/SM fill
    // the register file, so coins queued behind it would land on the next
    // round's extract instead: C3 metrics round 809 -> see DESIGN §11)
    const bool coins_at_extract = ctx->coin_prefetch_at_extract || (ctx->metrics && ctx->ml == ctx->M);
    if (phase == 0) {
        ctx->task_dir = ctx->l2_reuse ? uint32_t(t & 1) : 0;
        if ((s = run_coins(ctx, seed, t, st))) return s;
        // MARSIT_COIN_PREFETCH_AT=1: the next round's coins run underneath
        // this extract instead of this round's decode
        if (coins_at_extract && (s = prefetch_coins(ctx, seed, t, st))) return s;
        if ((s = run_extract(ctx, d_grads, d_comp, st))) return s;
        // the epoch advances only once this rank's phase-0 work is enqueued:
        // a failed launch above leaves the peers' view consistent
        if (ctx->p2p) ++ctx->epoch;
        return p2p_signal(ctx, 0, st);  // my packed signs are ready
    }
    if (phase == 1) {
        if ((s = p2p_wait(ctx, 0, st))) return s;  // every rank's packed signs
        if ((s = run_merge(ctx, seed, t, st))) return s;
        if ((s = consensus_own(ctx, st))) return s;
        if (!coins_at_extract && (s = prefetch_coins(ctx, seed, t, st))) return s;
        return p2p_signal(ctx, 1, st);  // my owned aggregates are ready
    }
    if ((s = p2p_wait(ctx, 1, st))) return s;  // every owner's aggregates
    if ((s = run_decode(ctx, d_grads, d_comp, d_comp_out, params, d_update, eta_s, st))) return s;
    if ((s = consensus_verify(ctx, st))) return s;
    return run_export(ctx, d_agg_bits, st);
}

void note_round(marsit_ctx* ctx, uint64_t t, bool dense) {
    ctx->last_valid = true;
    ctx->last_t = t;
    ctx->last_dense = dense;
    ctx->last_matching = false;  // set by the decode when it counts
}

marsit_status check_round_args(marsit_ctx* ctx, double eta_s, const void* const* d_grads,
                               const void* const* d_comp, void* const* d_comp_out,
                               void* const* params, bool sign) {
    if (!ctx) return fail(MARSIT_EPARAM, "ctx is null");
    marsit_status s;
    if ((s = ctx_failed(ctx))) return s;
    if (sign && !(eta_s > 0.0)) return fail(MARSIT_EPARAM, "SyncConfig: eta_s must be > 0");
    if ((s = check_ptrs(ctx, d_grads, "grads")) || (s = check_ptrs(ctx, d_comp, "comp")) ||
        (s = check_ptrs(ctx, (const void* const*)d_comp_out, "comp_out")) ||
        (params && (s = check_ptrs(ctx, (const void* const*)params, "params"))))
        return s;
    if ((s = check_consensus(ctx, sign))) return s;
    CUDA_TRY(cudaSetDevice(ctx->device));
    return MARSIT_OK;
}

// Small rounds on one GPU (ctx->fused): extract, merge and decode of a
// segment in one cluster launch (round_cluster_kernel), the coins of the next
// round prefetched underneath as usual.
template <typename T>
marsit_status fused_round(marsit_ctx* ctx, uint64_t t, double eta_s, uint64_t seed,
                          const void* const* g, const void* const* c, void* const* c_out,
                          uint64_t* d_agg_bits, void* d_update, cudaStream_t st) {
    marsit_status s;
    NvtxRange range("marsit.fused_round");
    if ((s = run_coins(ctx, seed, t, st))) return s;
    if (ctx->coins_pending) {
        CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_coin_done[ctx->cur_coin], 0));
        ctx->coins_pending = false;
    }
    // the next round's coins run beside this round's clusters (the other
    // buffer; their budget reads the draw ends of the round before, which
    // only sizes the work, never the bits)
    if ((s = prefetch_coins(ctx, seed, t, st))) return s;
    cudaEvent_t ev;
    if ((s = ctx->begin_phase(st, &ev))) return s;
    FusedParams<T> f{};
    for (uint32_t w = 0; w < ctx->M; ++w) {
        f.g[w] = static_cast<const T*>(g[w]);
        f.c[w] = static_cast<const T*>(c[w]);
        f.c_out[w] = static_cast<T*>(c_out[w]);
    }
    f.workers = ctx->M;
    f.dim = ctx->D;
    f.eta = T(eta_s);
    f.update = static_cast<T*>(d_update);
    f.err = ctx->err;
    const MergeRunner& mr = ctx->merge;
    const ClusterParams p = mr.cluster_params(nullptr, ctx->agg, ctx->coin_buf[ctx->cur_coin], seed, t, 0,
                                              ctx->coin_valid[ctx->cur_coin]);
    CUDA_TRY(launch_round_cluster<T>(p, f, int(mr.nsub), int(mr.dp.level_width), ctx->S, mr.smem, st));
    if ((s = ctx->end_phase(kPhFused, st, ev, 1))) return s;
    return run_export(ctx, d_agg_bits, st);
}

// Small rounds on one GPU over every SM (ctx->spread): coins, extract, merge
// and decode in one round_spread_kernel launch, which also computes the next
// round's coins while the merge clusters run (its own tagged coin buffers);
// no side stream, no host-side round state (the launch can be graph-captured).
template <typename T>
marsit_status spread_round(marsit_ctx* ctx, uint64_t t, double eta_s, uint64_t seed,
                           const void* const* g, const void* const* c, void* const* c_out,
                           uint64_t* d_agg_bits, void* d_update, cudaStream_t st) {
    marsit_status s;
    NvtxRange range("marsit.spread_round");
    cudaEvent_t ev;
    if ((s = ctx->begin_phase(st, &ev))) return s;
    SpreadParams<T> sp{};
    for (uint32_t w = 0; w < ctx->M; ++w) {
        sp.f.g[w] = static_cast<const T*>(g[w]);
        sp.f.c[w] = static_cast<const T*>(c[w]);
        sp.f.c_out[w] = static_cast<T*>(c_out[w]);
    }
    sp.f.workers = ctx->M;
    sp.f.dim = ctx->D;
    sp.f.eta = T(eta_s);
    sp.f.update = static_cast<T*>(d_update);
    sp.f.err = ctx->err;
    sp.sync = ctx->spread_sync;
    const MergeRunner& mr = ctx->merge;
    const bool coins = ctx->coin_total_words != 0;
    const int b = int(t & 1);
    sp.n_merges = coins ? mr.dp.n_merges : 0;
    for (int i = 0; i < 2; ++i) {
        sp.coins[i] = ctx->spread_coins[i];
        sp.coin_valid[i] = ctx->spread_valid[i];
    }
    sp.tag = ctx->spread_tag;
    sp.cend = ctx->spread_cend;
    sp.f.stash_cols = ctx->stash_cols;
    sp.f.tmem_cols = ctx->tmem_cols;
    sp.tma_stages = ctx->tma_stages;
    sp.tma_half = ctx->tma_half;
    ClusterParams p = mr.cluster_params(ctx->bits, ctx->agg, coins ? sp.coins[b] : nullptr, seed, t, 0,
                                        sp.coin_valid[b]);
    p.coin_end = reinterpret_cast<uint64_t*>(ctx->spread_cend) + size_t(b) * std::max<uint32_t>(mr.dp.n_merges, 1);
    p.coherent = 1;
    const int nsub = int(mr.nsub), nl = int(mr.dp.level_width);
    cudaError_t e = launch_round_spread<T>(p, sp, nsub, nl, ctx->spread_ctas, ctx->spread_smem, ctx->spread_coop, st);
    if (e != cudaSuccess && ctx->spread_coop) {
        // cooperative + cluster launch refused: the grid is sized to the
        // co-resident clusters, so a plain cluster launch keeps every CTA resident
        cudaGetLastError();
        ctx->spread_coop = false;
        e = launch_round_spread<T>(p, sp, nsub, nl, ctx->spread_ctas, ctx->spread_smem, false, st);
    }
    CUDA_TRY(e);
    if ((s = ctx->end_phase(kPhSpread, st, ev, 1))) return s;
    return run_export(ctx, d_agg_bits, st);
}

bool fused_eligible(const marsit_ctx* ctx, const void* const* g, const void* const* c,
                    void* const* c_out, void* const* params, void* update) {
    return ctx->fused && !ctx->metrics && !params && !ctx->pipeline &&
           vec_ok_ptrs(ctx, g, c) && vec_ok_ptrs(ctx, (const void* const*)c_out, c) &&
           (!update || aligned16(update));
}

marsit_status sign_round_impl(marsit_ctx* ctx, uint64_t t, double eta_s, uint64_t seed,
                              const void* const* d_grads, const void* const* d_comp,
                              void* const* d_comp_out, void* const* params, uint64_t* d_agg_bits,
                              void* d_update, cudaStream_t st) {
    marsit_status s = check_round_args(ctx, eta_s, d_grads, d_comp, d_comp_out, params, true);
    if (s) return s;
    if (ctx->G > 1 && !ctx->comm && !ctx->p2p)
        return fail(MARSIT_EUNSUPPORTED, "external-transport context: use marsit_round_phase");
    if (ctx->p2p && !ctx->peers_set) return fail(MARSIT_EPARAM, "P2P transport: call marsit_ctx_set_peers");
    note_round(ctx, t, false);
    if (ctx->spread && fused_eligible(ctx, d_grads, d_comp, d_comp_out, params, d_update))
        return ctx->dtype == MARSIT_F32
                   ? spread_round<float>(ctx, t, eta_s, seed, d_grads, d_comp, d_comp_out, d_agg_bits, d_update, st)
                   : spread_round<double>(ctx, t, eta_s, seed, d_grads, d_comp, d_comp_out, d_agg_bits, d_update, st);
    if (fused_eligible(ctx, d_grads, d_comp, d_comp_out, params, d_update))
        return ctx->dtype == MARSIT_F32
                   ? fused_round<float>(ctx, t, eta_s, seed, d_grads, d_comp, d_comp_out, d_agg_bits, d_update, st)
                   : fused_round<double>(ctx, t, eta_s, seed, d_grads, d_comp, d_comp_out, d_agg_bits, d_update, st);
    if (ctx->pipeline) {
        // st : coins? E ............ D0 D1 ... D(S-1)   (D_s waits M_s)
        // aux:           M0 M1 ... M(S-1) coins(t+1)      (after E)
        if ((s = run_coins(ctx, seed, t, st))) return s;
        if ((s = run_extract(ctx, d_grads, d_comp, st))) return s;
        CUDA_TRY(cudaEventRecord(ctx->ev_extract, st));
        CUDA_TRY(cudaStreamWaitEvent(ctx->aux, ctx->ev_extract, 0));
        ctx->coins_pending = false;  // aux is ordered after this round's coin kernel
        for (uint32_t sg = 0; sg < ctx->S; ++sg) {
            cudaEvent_t ev;
            if ((s = ctx->begin_phase(ctx->aux, &ev))) return s;
            uint64_t nl = 0;
            if ((s = ctx->merge.run(ctx->bits, ctx->agg, ctx->coin_buf[ctx->cur_coin], seed, t,
                                    ctx->aux, &nl, sg, 1, ctx->coin_valid[ctx->cur_coin])))
                return s;
            if ((s = ctx->end_phase(kPhMerge, ctx->aux, ev, nl))) return s;
            CUDA_TRY(cudaEventRecord(ctx->ev_merge[sg], ctx->aux));
        }
        if (ctx->coin_total_words && ctx->coin_prefetch) {  // aux is ordered after the merges
            const int b = 1 - ctx->cur_coin;
            cudaEvent_t ev;
            if ((s = ctx->begin_phase(ctx->aux, &ev))) return s;
            CUDA_TRY(launch_coins(ctx->merge.d_merges, ctx->merge.dp.n_merges, seed, t + 1,
                                  ctx->merge.coin_end, ctx->coin_valid[b], ctx->coin_buf[b],
                                  ctx->coin_grid_x, ctx->aux));
            if ((s = ctx->end_phase(kPhCoins, ctx->aux, ev, 1))) return s;
            CUDA_TRY(cudaEventRecord(ctx->ev_coin_done[b], ctx->aux));
            ctx->coin_tag[b] = {true, seed, t + 1};
        }
        for (uint32_t sg = 0; sg < ctx->S; ++sg) {
            CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_merge[sg], 0));
            if ((s = run_decode(ctx, d_grads, d_comp, d_comp_out, params, d_update, eta_s, st, sg,
                                1)))
                return s;
        }
        return run_export(ctx, d_agg_bits, st);  // st waited on the last merge
    }
    if ((s = sign_phase(ctx, 0, t, eta_s, seed, d_grads, d_comp, d_comp_out, params, d_agg_bits,
                        d_update, st)))
        return s;
    if ((s = run_exchange(ctx, st))) return s;
    if ((s = sign_phase(ctx, 1, t, eta_s, seed, d_grads, d_comp, d_comp_out, params, d_agg_bits,
                        d_update, st)))
        return s;
    if ((s = run_allgather(ctx, st))) return s;
    if ((s = sign_phase(ctx, 2, t, eta_s, seed, d_grads, d_comp, d_comp_out, params, d_agg_bits,
                        d_update, st)))
        return s;
    return watch_round(ctx, st);
}

marsit_status dense_round_any(marsit_ctx* ctx, uint64_t t, const void* const* d_grads,
                              const void* const* d_comp, void* const* d_comp_out,
                              void* const* params, void* d_mean, cudaStream_t st) {
    marsit_status s = check_round_args(ctx, 1.0, d_grads, d_comp, d_comp_out, params, false);
    if (s) return s;
    if (!d_mean) return fail(MARSIT_EPARAM, "mean is null");
    if (ctx->G > 1 && !ctx->comm && !ctx->p2p)
        return fail(MARSIT_EUNSUPPORTED, "external-transport context: use marsit_round_phase");
    if (ctx->p2p && !ctx->peers_set) return fail(MARSIT_EPARAM, "P2P transport: call marsit_ctx_set_peers");
    note_round(ctx, t, true);
    if ((s = dense_phase_any(ctx, 0, d_grads, d_comp, d_comp_out, params, d_mean, st))) return s;
    if ((s = dense_exchange(ctx, st))) return s;
    if ((s = dense_phase_any(ctx, 1, d_grads, d_comp, d_comp_out, params, d_mean, st))) return s;
    if ((s = dense_allgather(ctx, st))) return s;
    if ((s = dense_phase_any(ctx, 2, d_grads, d_comp, d_comp_out, params, d_mean, st))) return s;
    return watch_round(ctx, st);
}

uint64_t round_bits_total(const marsit_ctx* ctx, bool dense) {
    const uint64_t unit = dense ? 32ull * ctx->L : ctx->L;
    uint64_t t = 0;
    for (uint32_t w = 0; w < ctx->M; ++w) t += ctx->plan.sends_per_worker[w] * unit;
    return t;
}

}  // namespace marsit_b200

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* marsit_last_error(void) { return g_last_error.c_str(); }
int marsit_abi_version(void) { return MARSIT_B200_ABI_VERSION; }

static marsit_status finish_schedule(marsit_schedule* s, marsit_schedule** out) {
    s->plan = compile_plan(s->s);
    *out = s;
    return MARSIT_OK;
}

marsit_status marsit_schedule_ring(uint32_t m, marsit_schedule** out) {
    if (!out) return fail(MARSIT_EPARAM, "out is null");
    auto s = std::make_unique<marsit_schedule>();
    std::string msg;
    if (int rc = build_ring(m, s->s, &msg)) return fail(marsit_status(rc), msg);
    return finish_schedule(s.release(), out);
}

marsit_status marsit_schedule_torus(uint32_t rows, uint32_t cols, marsit_schedule** out) {
    if (!out) return fail(MARSIT_EPARAM, "out is null");
    auto s = std::make_unique<marsit_schedule>();
    std::string msg;
    if (int rc = build_torus(rows, cols, s->s, &msg)) return fail(marsit_status(rc), msg);
    return finish_schedule(s.release(), out);
}

marsit_status marsit_schedule_from_tables(uint32_t workers, uint32_t segments, uint32_t steps,
                                          const uint8_t* phase, const uint32_t* send_to,
                                          const uint32_t* recv_from, const uint32_t* segment,
                                          marsit_schedule** out) {
    if (!out) return fail(MARSIT_EPARAM, "out is null");
    if (workers == 0 || segments == 0) return fail(MARSIT_EPARAM, "empty schedule");
    if (steps && (!phase || !send_to || !recv_from || !segment))
        return fail(MARSIT_EPARAM, "null schedule table");
    auto s = std::make_unique<marsit_schedule>();
    s->s.topology = 2;
    s->s.workers = workers;
    s->s.segments = segments;
    const size_t n = size_t(steps) * workers;
    s->s.phase.assign(phase, phase + steps);
    s->s.send_to.assign(send_to, send_to + n);
    s->s.recv_from.assign(recv_from, recv_from + n);
    s->s.segment.assign(segment, segment + n);
    std::string msg;
    if (int rc = validate(s->s, &msg)) return fail(marsit_status(rc), msg);
    return finish_schedule(s.release(), out);
}

marsit_status marsit_schedule_info(const marsit_schedule* s, uint32_t* workers,
                                   uint32_t* segments, uint32_t* steps) {
    if (!s) return fail(MARSIT_EPARAM, "schedule is null");
    if (workers) *workers = s->s.workers;
    if (segments) *segments = s->s.segments;
    if (steps) *steps = s->s.steps();
    return MARSIT_OK;
}

marsit_status marsit_schedule_tables(const marsit_schedule* s, uint8_t* phase,
                                     uint32_t* send_to, uint32_t* recv_from, uint32_t* segment) {
    if (!s) return fail(MARSIT_EPARAM, "schedule is null");
    if (phase) std::copy(s->s.phase.begin(), s->s.phase.end(), phase);
    if (send_to) std::copy(s->s.send_to.begin(), s->s.send_to.end(), send_to);
    if (recv_from) std::copy(s->s.recv_from.begin(), s->s.recv_from.end(), recv_from);
    if (segment) std::copy(s->s.segment.begin(), s->s.segment.end(), segment);
    return MARSIT_OK;
}

void marsit_schedule_destroy(marsit_schedule* s) { delete s; }

marsit_status marsit_schedule_plan(const marsit_schedule* s, uint32_t segment, uint32_t capacity,
                                   marsit_merge_info* merges, uint32_t* n_merges,
                                   uint32_t* final_node, uint32_t* final_count) {
    if (!s) return fail(MARSIT_EPARAM, "schedule is null");
    if (segment >= s->plan.segments) return fail(MARSIT_EPARAM, "segment out of range");
    const SegmentPlan& sp = s->plan.seg[segment];
    if (n_merges) *n_merges = uint32_t(sp.merges.size());
    if (final_node) *final_node = sp.final_node;
    if (final_count) *final_count = sp.final_count;
    if (merges)
        for (size_t k = 0; k < sp.merges.size() && k < capacity; ++k) {
            const MergeNode& m = sp.merges[k];
            merges[k] = {m.recv_node, m.local_node, m.receiver, m.c_recv,
                         m.c_local,   m.offset_src, m.stage};
        }
    return MARSIT_OK;
}

marsit_status marsit_nccl_unique_id(void* out128) {
    if (!out128) return fail(MARSIT_EPARAM, "out is null");
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, sizeof(id));
    return MARSIT_OK;
}

marsit_status marsit_ctx_create(const marsit_ctx_desc* desc, marsit_ctx** out) {
    return ctx_create_internal(desc, nullptr, out);
}

}  // extern "C"

namespace marsit_b200 {

marsit_status ctx_create_internal(const marsit_ctx_desc* desc, ncclComm_t shared_comm,
                                  marsit_ctx** out) {
    if (!desc || !out) return fail(MARSIT_EPARAM, "null argument");
    *out = nullptr;
    if (!desc->schedule) return fail(MARSIT_EPARAM, "schedule is null");
    if (desc->dim == 0) return fail(MARSIT_EPARAM, "DenseVector: dimension must be >= 1");
    if (desc->dtype != MARSIT_F32 && desc->dtype != MARSIT_F64)
        return fail(MARSIT_EPARAM, "unknown dtype");
    const uint32_t G = desc->nranks ? desc->nranks : 1;
    const HostSchedule& hs = desc->schedule->s;
    if (hs.workers % G || hs.segments % G)
        return fail(MARSIT_EUNSUPPORTED, "workers and segments must be divisible by nranks");
    if (desc->rank >= G) return fail(MARSIT_EPARAM, "rank out of range");
    if (hs.workers / G > kMaxLocalWorkers)
        return fail(MARSIT_EUNSUPPORTED, "too many workers per rank (max 64)");
    if (G > kMaxLocalWorkers)  // P2P flag writes address G - 1 peers (FlagSlots)
        return fail(MARSIT_EUNSUPPORTED, "too many ranks (max 64)");
    const bool external = desc->transport == MARSIT_TRANSPORT_EXTERNAL;
    const bool p2p = G > 1 && desc->transport == MARSIT_TRANSPORT_P2P;
    if (desc->transport != MARSIT_TRANSPORT_NCCL && desc->transport != MARSIT_TRANSPORT_EXTERNAL &&
        desc->transport != MARSIT_TRANSPORT_P2P)
        return fail(MARSIT_EPARAM, "unknown transport");
    if (G > 1 && !external && !p2p && !desc->nccl_id && !shared_comm)
        return fail(MARSIT_EPARAM, "nccl_id required for nranks > 1");
    if (!have_device())
        return fail(MARSIT_ECUDA, "no CUDA device available (this library has no CPU path)");

    auto ctx = std::make_unique<marsit_ctx>();
    ctx->device = desc->device;
    CUDA_TRY(cudaSetDevice(desc->device));
    CUDA_TRY(preload_kernels());
    CUDA_TRY(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, desc->device));
    ctx->dtype = desc->dtype;
    ctx->esize = desc->dtype == MARSIT_F32 ? 4 : 8;
    ctx->sched = hs;
    ctx->plan = desc->schedule->plan;
    ctx->D = desc->dim;
    ctx->M = hs.workers;
    ctx->S = hs.segments;
    ctx->G = G;
    ctx->rank = desc->rank;
    ctx->ml = ctx->M / G;
    ctx->s_own = ctx->S / G;
    ctx->s_first = ctx->rank * ctx->s_own;
    ctx->L = ceil_div(ctx->D, ctx->S);  // segmentation.hpp:32-39
    if (ctx->L >= (1ull << 37)) return fail(MARSIT_EUNSUPPORTED, "segment too long");
    ctx->words64 = uint32_t(ceil_div(ctx->L, 64));
    ctx->words_proc = uint32_t(round_up(2ull * ctx->words64, 4));
    ctx->wst = uint32_t(round_up(ctx->words_proc, 32));
    ctx->wsa = ctx->wst + 4;  // + the segment's u64 consensus hash, rows 16 B aligned
    // vector kernels: every segment's quads 16 B-aligned (L % 4 == 0); other
    // lengths take the coalesced scalar kernels (all loads issued first)
    ctx->vec_ok = (ctx->L % 4) == 0;

    // merge plan, coin budget, tiling
    MergeRunner& mr = ctx->merge;
    // small one-GPU rounds run fused (one cluster launch: extract, merge,
    // decode; the decode's re-read of g and c stays in L2): every worker
    // local, L % 4 == 0, the inputs well inside L2 (MARSIT_FUSED=0 disables)
    ctx->fused = G == 1 && hs.workers <= kFusedMaxWorkers && ctx->vec_ok &&
                 uint64_t(hs.workers) * ctx->D * ctx->esize * 2 <= (96ull << 20) &&
                 env_int("MARSIT_FUSED", 1) != 0;
    const bool grid_default = mr.grid;
    const bool kernel_forced = std::getenv("MARSIT_MERGE_KERNEL") != nullptr;
    // ... and spread over every SM when the merge chain is short (M <= 8:
    // C1 27.9 vs 28.8-30.9 us, M = 8 at 1M 47.8 vs 58.9 us; at M = 16 the
    // cluster-per-segment kernel's 16-CTA merge levels win, 70.5 vs 90.8 us).
    // MARSIT_SPREAD=1 forces the spread round, 0 the cluster-per-segment one
    {
        const int sp = env_int("MARSIT_SPREAD", -1);
        ctx->spread = ctx->fused && (sp > 0 || (sp < 0 && hs.workers <= 8));
    }
    if (ctx->fused) {
        mr.cluster = true;
        mr.fused_arrays = ctx->spread ? 0 : hs.workers + 1;
        mr.fused_dtype = desc->dtype == MARSIT_F64 ? 1 : 0;
    }
    double frac = 0.53;
    if (const char* e = std::getenv("MARSIT_COIN_FRAC")) frac = std::atof(e);
    uint64_t max_words = 0;
    // lower the plan for the runner's merge kernel and size its coin budget
    auto lower = [&]() -> marsit_status {
        marsit_status ls = mr.cluster ? lower_cluster_plan(ctx->plan, ctx->s_first, ctx->s_own, mr.dp)
                                      : lower_plan(ctx->plan, ctx->s_first, ctx->s_own, mr.dp);
        if (!ls) assign_coin_budget(mr.dp, ctx->s_own, ctx->L, frac, &ctx->coin_total_words, &max_words);
        return ls;
    };
    marsit_status st = lower();
    if (st) return st;
    mr.n_seg = ctx->s_own;
    mr.s_first = ctx->s_first;
    mr.words_proc = ctx->words_proc;
    mr.wst = ctx->wst;
    mr.ml = ctx->ml;
    mr.L = ctx->L;
    mr.agg_stride = ctx->wsa;
    // single GPU with several segments: per-segment merge launches sized to
    // co-reside with the decode (MARSIT_PIPELINE=1 enables)
    ctx->pipeline = G == 1 && ctx->S >= 2 && env_int("MARSIT_PIPELINE", 0) != 0 &&
                    desc->transport != MARSIT_TRANSPORT_EXTERNAL;
    if (ctx->pipeline) {  // cooperative merges sized to share the SMs with the decode
        if (mr.grid && !ctx->fused) {
            mr.cluster = mr.grid = false;
            if ((st = lower())) return st;
        }
        if ((st = mr.configure(ctx->sm_count, 1, env_int("MARSIT_PIPE_MERGE_CTAS", 1)))) return st;
    } else {
        if (ctx->spread) {
            st = mr.configure_spread(mr.fused_dtype, hs.workers, &ctx->spread_ctas);
            if (st) {  // the spread round does not configure: the cluster-per-segment round
                cudaGetLastError();
                ctx->spread = false;
                mr.fused_arrays = hs.workers + 1;
                st = mr.configure(ctx->sm_count);
            }
        } else {
            st = mr.configure(ctx->sm_count);
        }
        if (st && ctx->fused) {  // the fused tiles do not fit: the merge kernel alone
            ctx->fused = false;
            mr.fused_arrays = 0;
            mr.grid = grid_default;
            st = mr.configure(ctx->sm_count);
        }
        // the grid merge's tiles do not fit (very long segments): the
        // cooperative merge, which runs them as several launch parts
        if (st && grid_default && mr.grid && !kernel_forced) {
            cudaGetLastError();
            mr.cluster = mr.grid = false;
            if ((st = lower())) return st;
            st = mr.configure(ctx->sm_count);
        }
        if (st) return st;
        // one GPU holding many segments: the cooperative merge when it runs
        // as one launch part (measured, B200: C3 merge 50.8 vs 53.1 us, round
        // 678-680 vs 687 us); the grid merge stays for a rank's few segments
        // (G = 2 / 4 / 8: 33.2 / 29.8 / 28.7 vs 40.9 / 34.8 / 30.6 us) and
        // wherever the cooperative merge needs several parts (C2, C4)
        if (mr.grid && !ctx->fused && !kernel_forced && G == 1 && ctx->s_own >= 8) {
            mr.cluster = mr.grid = false;
            if ((st = lower())) return st;
            st = mr.configure(ctx->sm_count);
            if (st || mr.n_parts > 1) {
                cudaGetLastError();
                mr.cluster = mr.grid = true;
                if ((st = lower())) return st;
                if ((st = mr.configure(ctx->sm_count))) return st;
            }
        }
    }
    if ((st = mr.upload())) return st;

    const size_t wst = ctx->wst;
    CUDA_TRY(cudaMalloc(&ctx->bits, sizeof(uint32_t) * ctx->S * ctx->ml * wst));
    CUDA_TRY(cudaMemset(ctx->bits, 0, sizeof(uint32_t) * ctx->S * ctx->ml * wst));
    CUDA_TRY(cudaMalloc(&ctx->agg, sizeof(uint32_t) * ctx->S * ctx->wsa));
    CUDA_TRY(cudaMemset(ctx->agg, 0, sizeof(uint32_t) * ctx->S * ctx->wsa));
    if (G > 1 && !p2p) {
        CUDA_TRY(cudaMalloc(&ctx->recv, sizeof(uint32_t) * ctx->S * ctx->ml * wst));
        CUDA_TRY(cudaMemset(ctx->recv, 0, sizeof(uint32_t) * ctx->S * ctx->ml * wst));
    }
    if (p2p) {
        ctx->p2p = true;
        ctx->flag_kernel = env_int("MARSIT_P2P_FLAG_KERNEL", 0) != 0;
        CUDA_TRY(cudaMalloc(&ctx->flags, 2 * size_t(G) * sizeof(uint64_t)));
        CUDA_TRY(cudaMemset(ctx->flags, 0, 2 * size_t(G) * sizeof(uint64_t)));
        CUDA_TRY(cudaMalloc(&ctx->d_peer_tables, 3 * size_t(G) * sizeof(void*)));
        CUDA_TRY(cudaMemset(ctx->d_peer_tables, 0, 3 * size_t(G) * sizeof(void*)));
    }
    CUDA_TRY(cudaMalloc(&ctx->err, sizeof(int)));
    CUDA_TRY(cudaMemset(ctx->err, 0, sizeof(int)));
    // TMEM stash of the spread round: a thread parks one quad of u per
    // (worker, step, group of the step) — 4 groups per step in fp32, 2 in
    // fp64 — in 4 (8) columns; a warp's quarter of the 512 columns is 128
    // per thread (MARSIT_STASH=0 disables).  C1: 30.8 -> 29.2 us per round.
    // (The cluster-per-segment round measured slower with it, 28.8 -> 30.9
    // us, and does not use it.)
    if (ctx->spread) {
        const uint64_t groups = ceil_div(uint64_t(ctx->S) * (ctx->words_proc / 4), ctx->spread_ctas);
        const uint64_t B = ctx->esize == 4 ? 4 : 2, step = uint64_t(kFusedThreads / 32) * B;
        const uint64_t cols = uint64_t(hs.workers) * ceil_div(groups, step) * B * ctx->esize;
        if (cols <= 128 && env_int("MARSIT_STASH", 1) != 0) {
            ctx->stash_cols = uint32_t(cols);
            uint32_t a = 32;
            while (a < 4 * cols) a *= 2;
            ctx->tmem_cols = a;
        }
    }
    if (ctx->spread) {
        // the extract's TMA ring (opt-in, MARSIT_SPREAD_TMA=1): 3 (else 2)
        // stages of a worker's slice when they fit next to the static shared
        // memory.  Measured slower than the register loads (C1 31.9 vs 27.9
        // us per round from a graph, M = 8 at 1M 54.1 vs 47.1): a stage is
        // consumed only once all of its bytes have landed
        ctx->spread_smem = mr.smem;
        {
            const uint64_t groups = ceil_div(uint64_t(ctx->S) * (ctx->words_proc / 4), ctx->spread_ctas);
            const uint64_t half = round_up(groups * 128 * ctx->esize, 16);
            for (uint32_t nst = std::min<uint32_t>(3, hs.workers); nst >= 2 && env_int("MARSIT_SPREAD_TMA", 0); --nst)
                if (nst * 2 * half <= 200 * 1024) {
                    ctx->tma_stages = nst;
                    ctx->tma_half = uint32_t(half);
                    ctx->spread_smem = std::max<size_t>(mr.smem, nst * 2 * half);
                    break;
                }
        }
        // the grid is sized to the co-resident clusters; the cooperative
        // attribute on top (same speed) also makes the driver guarantee that
        // residency when other kernels share the GPU (two spread contexts on
        // concurrent streams could otherwise starve each other's CTAs until
        // the bounded waits give up).  Nsight Compute fails such launches, so
        // under a profiler's injection (or MARSIT_SPREAD_COOP=0) the launch
        // is a plain cluster launch
        const bool profiled = std::getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") != nullptr ||
                              std::getenv("CUDA_INJECTION64_PATH") != nullptr;
        ctx->spread_coop = env_int("MARSIT_SPREAD_COOP", profiled ? 0 : 1) != 0;

        CUDA_TRY(cudaMalloc(&ctx->spread_sync, sizeof(unsigned) * (2 + ctx->S)));
        CUDA_TRY(cudaMemset(ctx->spread_sync, 0, sizeof(unsigned) * (2 + ctx->S)));
        const size_t nm = std::max<uint32_t>(mr.dp.n_merges, 1);
        for (int b = 0; b < 2; ++b) {
            CUDA_TRY(cudaMalloc(&ctx->spread_coins[b], sizeof(uint32_t) * (ctx->coin_total_words + 16)));
            CUDA_TRY(cudaMemset(ctx->spread_coins[b], 0, sizeof(uint32_t) * (ctx->coin_total_words + 16)));
            CUDA_TRY(cudaMalloc(&ctx->spread_valid[b], sizeof(uint32_t) * nm));
            CUDA_TRY(cudaMemset(ctx->spread_valid[b], 0, sizeof(uint32_t) * nm));
        }
        CUDA_TRY(cudaMalloc(&ctx->spread_tag, 4 * sizeof(unsigned long long)));
        CUDA_TRY(cudaMemset(ctx->spread_tag, 0xFF, 4 * sizeof(unsigned long long)));  // no buffer holds coins
        CUDA_TRY(cudaMalloc(&ctx->spread_cend, 2 * nm * sizeof(unsigned long long)));
        CUDA_TRY(cudaMemset(ctx->spread_cend, 0xFF, 2 * nm * sizeof(unsigned long long)));  // no history
    }
    mr.err = ctx->err;
    // marsit_ctx_check's pinned read-back (allocated here: cudaHostAlloc may
    // synchronise the device, which a blocked P2P stream would never allow)
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_check, cudaEventDisableTiming));
    CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_check),
                           sizeof(uint64_t) * (1 + 2 * size_t(G)), cudaHostAllocDefault));

    // coin buffers, aux stream
    CUDA_TRY(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    if (ctx->coin_total_words)
        for (int b = 0; b < 2; ++b) {
            CUDA_TRY(cudaMalloc(&ctx->coin_valid[b], sizeof(uint32_t) * std::max<uint32_t>(mr.dp.n_merges, 1)));
            CUDA_TRY(cudaMemset(ctx->coin_valid[b], 0, sizeof(uint32_t) * std::max<uint32_t>(mr.dp.n_merges, 1)));
            // + slack: a merge group reads its 5-word coin window whole
            CUDA_TRY(cudaMalloc(&ctx->coin_buf[b], sizeof(uint32_t) * (ctx->coin_total_words + 16)));
            CUDA_TRY(cudaMemset(ctx->coin_buf[b], 0, sizeof(uint32_t) * (ctx->coin_total_words + 16)));
            CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_coin_done[b], cudaEventDisableTiming));
        }
    ctx->coin_prefetch = env_int("MARSIT_COIN_PREFETCH", 1) != 0;
    ctx->coin_prefetch_at_extract = env_int("MARSIT_COIN_PREFETCH_AT", 0) != 0;
    if (ctx->pipeline) {
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_extract, cudaEventDisableTiming));
        ctx->ev_merge.resize(ctx->S);
        for (auto& e : ctx->ev_merge) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    {
        // MARSIT_COIN_CTAS (default 4) CTAs per SM in total, split across the
        // merges (one warp per 64-word chunk)
        const uint64_t coin_ctas = uint64_t(std::max(1, env_int("MARSIT_COIN_CTAS", 4)));
        ctx->coin_grid_x = int(std::max<uint64_t>(
            1, std::min<uint64_t>(ceil_div(max_words, 64 * 8),
                                  ceil_div(coin_ctas * ctx->sm_count,
                                           std::max<uint32_t>(mr.dp.n_merges, 1)))));
    }
    {
        // persistent grid-stride streaming kernels; MARSIT_{EXTRACT,DECODE}_CTAS
        // override the CTAs per SM.  The decode leaves SM room for the next
        // round's coin kernel running underneath it.  Measured (CUPTI, C3):
        // extract 247 us at 3 CTAs/SM vs 255 us at 4 and 274 us at 2
        // (tools/sweep_stream_ctas.sh, tools/ab_extract_ctas.sh).
        int ob_extract = 0, ob_decode = 0;
        CUDA_TRY(stream_occupancy(ctx->dtype == MARSIT_F64, &ob_extract, &ob_decode));
        // fp64: one decode CTA per SM leaves the coin prefetch room (C3 fp64
        // round 1420 -> 1334 us; at 2 the coins starve underneath the decode)
        // short extracts (a G = 8 rank reads 205 MB) lose less to their tail
        // with 4 CTAs/SM (34.0 -> 32.5 us); long ones run best at 3
        const uint64_t ext_bytes = uint64_t(ctx->ml) * ctx->D * ctx->esize * 2;
        const int want_e = env_int("MARSIT_EXTRACT_CTAS", ext_bytes < (512ull << 20) ? 4 : 3);
        const int want_d = env_int("MARSIT_DECODE_CTAS", ctx->dtype == MARSIT_F64 ? 1 : 2);
        ctx->extract_grid = std::max(1, std::min(ob_extract, want_e)) * ctx->sm_count;
        ctx->decode_grid = std::max(1, std::min(ob_decode, want_d)) * ctx->sm_count;
        // metrics on: the worker-inner decode keeps fewer loads in flight per
        // warp and runs best at 3 CTAs/SM (797 -> 785 us per C3 round)
        ctx->stats_grid = std::max(1, env_int("MARSIT_STATS_CTAS", 3)) * ctx->sm_count;
        ctx->stream_grid = 4 * ctx->sm_count;
    }

    // dense-round plan: per owned segment, the reduction tree (local + received)
    {
        std::vector<DenseOp> ops;
        std::vector<uint16_t> fin(ctx->s_own);
        uint32_t n_ops = 0;
        for (uint32_t sl = 0; sl < ctx->s_own; ++sl)
            n_ops = std::max<uint32_t>(n_ops, uint32_t(ctx->plan.seg[ctx->s_first + sl].merges.size()));
        if (ctx->M + n_ops > 2 * kMaxLocalWorkers)
            return fail(MARSIT_EUNSUPPORTED, "dense reduction tree too large");
        ops.resize(size_t(ctx->s_own) * std::max<uint32_t>(n_ops, 1));
        for (uint32_t sl = 0; sl < ctx->s_own; ++sl) {
            const SegmentPlan& sp = ctx->plan.seg[ctx->s_first + sl];
            for (uint32_t k = 0; k < n_ops; ++k) {
                DenseOp o{};
                if (k < sp.merges.size()) {
                    o.a = uint16_t(sp.merges[k].local_node);
                    o.b = uint16_t(sp.merges[k].recv_node);
                }
                ops[size_t(sl) * n_ops + k] = o;
            }
            fin[sl] = uint16_t(sp.final_node);
        }
        ctx->dense_n_ops = n_ops;
        // Chain-of-chains form (ring: one chain; torus: row chains, then a
        // chain over the row results): the register kernels evaluate it;
        // anything else keeps the general DAG kernels.
        bool chain = n_ops + 1 == ctx->M && env_int("MARSIT_DENSE_DAG", 0) == 0 && ctx->M <= 64;
        std::vector<uint16_t> order(size_t(ctx->s_own) * ctx->M);
        std::vector<uint64_t> groups(ctx->s_own);
        for (uint32_t sl = 0; sl < ctx->s_own && chain; ++sl) {
            std::vector<uint16_t> ord;
            uint64_t gm = 0;
            chain = chain_of_chains(&ops[size_t(sl) * n_ops], ctx->M, fin[sl], ord, gm);
            if (chain) {
                std::copy(ord.begin(), ord.end(), order.begin() + size_t(sl) * ctx->M);
                groups[sl] = gm;
                ctx->dense_multi |= gm != (1ull << (ctx->M - 1));
            }
        }
        if (chain && n_ops > 0) {
            CUDA_TRY(cudaMalloc(&ctx->d_dense_chain, sizeof(uint16_t) * order.size()));
            CUDA_TRY(cudaMemcpy(ctx->d_dense_chain, order.data(), sizeof(uint16_t) * order.size(),
                                cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMalloc(&ctx->d_dense_groups, sizeof(uint64_t) * groups.size()));
            CUDA_TRY(cudaMemcpy(ctx->d_dense_groups, groups.data(), sizeof(uint64_t) * groups.size(),
                                cudaMemcpyHostToDevice));
        }
        CUDA_TRY(cudaMalloc(&ctx->d_dense_ops, sizeof(DenseOp) * ops.size()));
        CUDA_TRY(cudaMemcpy(ctx->d_dense_ops, ops.data(), sizeof(DenseOp) * ops.size(),
                            cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMalloc(&ctx->d_dense_final, sizeof(uint16_t) * fin.size()));
        CUDA_TRY(cudaMemcpy(ctx->d_dense_final, fin.data(), sizeof(uint16_t) * fin.size(),
                            cudaMemcpyHostToDevice));
    }
    if (G > 1) {
        const size_t dense_elems = size_t(ctx->S) * ctx->ml * ctx->L;
        CUDA_TRY(cudaMalloc(&ctx->dense_send, ctx->esize * dense_elems));
        if (!p2p) CUDA_TRY(cudaMalloc(&ctx->dense_recv, ctx->esize * dense_elems));
        CUDA_TRY(cudaMalloc(&ctx->dense_mean, ctx->esize * size_t(ctx->S) * ctx->L));
        if (external || p2p) {
            ctx->comm = nullptr;  // the caller moves the blocks / peer memory
        } else if (shared_comm) {
            ctx->comm = shared_comm;
            ctx->owns_comm = false;
        } else {
            ncclUniqueId id;
            std::memcpy(&id, desc->nccl_id, sizeof(id));
            NCCL_TRY(ncclCommInitRank(&ctx->comm, int(G), id, int(desc->rank)));
        }
        if (ctx->comm) ctx->watchdog = std::make_unique<Watchdog>(ctx.get());
    }
    *out = ctx.release();
    return MARSIT_OK;
}

}  // namespace marsit_b200

extern "C" {

void marsit_ctx_destroy(marsit_ctx* ctx) { delete ctx; }

marsit_status marsit_ctx_local_workers(const marsit_ctx* ctx, uint32_t* first, uint32_t* count) {
    if (!ctx) return fail(MARSIT_EPARAM, "ctx is null");
    if (first) *first = ctx->rank * ctx->ml;
    if (count) *count = ctx->ml;
    return MARSIT_OK;
}

marsit_status marsit_sign_round(marsit_ctx* ctx, uint64_t t, double eta_s, uint64_t seed,
                                const void* const* d_grads, const void* const* d_comp,
                                void* const* d_comp_out, uint64_t* d_agg_bits, void* d_update,
                                void* stream) {
    return sign_round_impl(ctx, t, eta_s, seed, d_grads, d_comp, d_comp_out, nullptr, d_agg_bits,
                           d_update, static_cast<cudaStream_t>(stream));
}

marsit_status marsit_dense_round(marsit_ctx* ctx, uint64_t t, const void* const* d_grads,
                                 const void* const* d_comp, void* const* d_comp_out, void* d_mean,
                                 void* stream) {
    return dense_round_any(ctx, t, d_grads, d_comp, d_comp_out, nullptr, d_mean,
                           static_cast<cudaStream_t>(stream));
}

marsit_status marsit_round(marsit_ctx* ctx, uint64_t t, uint64_t period, double eta_s,
                           uint64_t seed, const void* const* d_grads, const void* const* d_comp,
                           void* const* d_comp_out, uint64_t* d_agg_bits, void* d_update,
                           int* full_precision, void* stream) {
    if (!ctx) return fail(MARSIT_EPARAM, "ctx is null");
    // SyncConfig::validate (sync.hpp:27-34); "never" is period == 0 here.
    if (!(eta_s > 0.0)) return fail(MARSIT_EPARAM, "SyncConfig: eta_s must be > 0");
    const bool dense = period != 0 && (t % period == 0);  // sync.hpp:78
    if (full_precision) *full_precision = dense ? 1 : 0;
    if (dense) {
        if (!d_update) return fail(MARSIT_EPARAM, "dense round needs d_update for the mean");
        return marsit_dense_round(ctx, t, d_grads, d_comp, d_comp_out, d_update, stream);
    }
    return marsit_sign_round(ctx, t, eta_s, seed, d_grads, d_comp, d_comp_out, d_agg_bits,
                             d_update, stream);
}

marsit_status marsit_ctx_exchange_layout(const marsit_ctx* ctx, int dense,
                                         marsit_exchange_layout* out) {
    if (!ctx || !out) return fail(MARSIT_EPARAM, "null argument");
    if (dense) {
        out->send = ctx->G > 1 ? ctx->dense_send : nullptr;
        out->recv = ctx->G > 1 ? ctx->dense_recv : nullptr;
        out->block_bytes = uint64_t(ctx->s_own) * ctx->ml * ctx->L * ctx->esize;
        out->gather = ctx->G > 1 ? ctx->dense_mean : nullptr;
        out->gather_block_bytes = uint64_t(ctx->s_own) * ctx->L * ctx->esize;
    } else {
        out->send = ctx->bits;
        out->recv = ctx->G > 1 ? ctx->recv : ctx->bits;
        out->block_bytes = uint64_t(ctx->s_own) * ctx->ml * ctx->wst * 4;
        out->gather = ctx->agg;
        out->gather_block_bytes = uint64_t(ctx->s_own) * ctx->wsa * 4;  // rows incl. hash slots
    }
    return MARSIT_OK;
}

marsit_status marsit_round_phase(marsit_ctx* ctx, int phase, uint64_t t, uint64_t period,
                                 double eta_s, uint64_t seed, const void* const* d_grads,
                                 const void* const* d_comp, void* const* d_comp_out,
                                 uint64_t* d_agg_bits, void* d_update, int* full_precision,
                                 void* stream) {
    if (phase < 0 || phase > 2) return fail(MARSIT_EPARAM, "phase must be 0, 1 or 2");
    if (!(eta_s > 0.0)) return fail(MARSIT_EPARAM, "SyncConfig: eta_s must be > 0");
    const bool dense = period != 0 && (t % period == 0);  // sync.hpp:78
    if (full_precision) *full_precision = dense ? 1 : 0;
    marsit_status s = check_round_args(ctx, eta_s, d_grads, d_comp, d_comp_out, nullptr, !dense);
    if (s) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (ctx->p2p && !ctx->peers_set) return fail(MARSIT_EPARAM, "P2P transport: call marsit_ctx_set_peers");
    if (phase == 0) note_round(ctx, t, dense);
    if (dense) {
        if (!d_update) return fail(MARSIT_EPARAM, "dense round needs d_update for the mean");
        s = dense_phase_any(ctx, phase, d_grads, d_comp, d_comp_out, nullptr, d_update, st);
    } else {
        s = sign_phase(ctx, phase, t, eta_s, seed, d_grads, d_comp, d_comp_out, nullptr,
                       d_agg_bits, d_update, st);
    }
    if (s || phase != 2) return s;
    return watch_round(ctx, st);
}

marsit_status marsit_sign_extract(marsit_ctx* ctx, const void* const* d_grads,
                                  const void* const* d_comp, uint64_t* d_signs_out, void* stream) {
    if (!ctx || !d_signs_out) return fail(MARSIT_EPARAM, "null argument");
    marsit_status s;
    if ((s = check_ptrs(ctx, d_grads, "grads")) || (s = check_ptrs(ctx, d_comp, "comp"))) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaSetDevice(ctx->device));
    if ((s = run_extract(ctx, d_grads, d_comp, st))) return s;
    const size_t row = size_t(ctx->words64) * 8;
    for (uint32_t w = 0; w < ctx->ml; ++w)
        CUDA_TRY(cudaMemcpy2DAsync(d_signs_out + size_t(w) * ctx->S * ctx->words64, row,
                                   ctx->bits + size_t(w) * ctx->wst, size_t(ctx->ml) * ctx->wst * 4,
                                   row, ctx->S, cudaMemcpyDeviceToDevice, st));
    return MARSIT_OK;
}

marsit_status marsit_allreduce_sign(marsit_ctx* ctx, uint64_t round, uint64_t seed,
                                    const uint64_t* d_signs, uint64_t* d_out, uint32_t* counts,
                                    void* stream) {
    if (!ctx || !d_signs || !d_out) return fail(MARSIT_EPARAM, "null argument");
    marsit_status s;
    if ((s = ctx_failed(ctx))) return s;
    // every worker's result is the consensus aggregate only for schedules
    // that end in consensus (ring, torus); the reference returns each
    // worker's own final state otherwise, which this entry point does not
    // materialise
    for (uint32_t sg = 0; sg < ctx->S; ++sg)
        if (!ctx->plan.seg[sg].consensus)
            return fail(MARSIT_EUNSUPPORTED,
                        "allreduce_sign: schedules whose workers do not end in consensus are not "
                        "supported (use ring / torus or a consensus-reaching table)");
    if (ctx->G > 1 && !ctx->comm)
        return fail(MARSIT_EUNSUPPORTED,
                    "allreduce_sign on a multi-rank context needs the NCCL transport "
                    "(P2P / external contexts: marsit_round_phase)");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaSetDevice(ctx->device));
    const size_t row = size_t(ctx->words64) * 8;
    for (uint32_t w = 0; w < ctx->ml; ++w)
        CUDA_TRY(cudaMemcpy2DAsync(ctx->bits + size_t(w) * ctx->wst, size_t(ctx->ml) * ctx->wst * 4,
                                   d_signs + size_t(w) * ctx->S * ctx->words64, row, row, ctx->S,
                                   cudaMemcpyDeviceToDevice, st));
    if ((s = run_coins(ctx, seed, round, st))) return s;
    if ((s = run_exchange(ctx, st))) return s;
    if ((s = run_merge(ctx, seed, round, st))) return s;
    if ((s = run_allgather(ctx, st))) return s;
    CUDA_TRY(cudaMemcpy2DAsync(d_out, row, ctx->agg, size_t(ctx->wsa) * 4, row, ctx->S,
                               cudaMemcpyDeviceToDevice, st));
    if (counts)
        for (uint32_t sg = 0; sg < ctx->S; ++sg) counts[sg] = ctx->plan.seg[sg].final_count;
    return MARSIT_OK;
}

// merge_signs (merge.hpp:34-58) as a one-merge plan through the same
// cooperative kernel: leaves = [received, local], explicit stream key, the
// stream's earlier draws as base, coins drawn inline.
marsit_status marsit_merge_signs(const uint64_t* d_recv, uint32_t c_recv, const uint64_t* d_local,
                                 uint32_t c_local, uint64_t len, uint64_t key, uint64_t used,
                                 uint64_t* d_out, uint64_t* consumed, int device, void* stream) {
    if (c_recv == 0 || c_local == 0)
        return fail(MARSIT_EPARAM, "merge_signs: aggregate count must be >= 1");
    if (!d_recv || !d_local || !d_out) return fail(MARSIT_EPARAM, "null argument");
    if (len == 0) {
        if (consumed) *consumed = 0;
        return MARSIT_OK;
    }
    if (!have_device())
        return fail(MARSIT_ECUDA, "no CUDA device available (this library has no CPU path)");
    CUDA_TRY(cudaSetDevice(device));
    int sm = 148;
    CUDA_TRY(cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t words64 = ceil_div(len, 64);
    MergeRunner mr;
    mr.n_seg = 1;
    mr.s_first = 0;
    mr.words_proc = uint32_t(round_up(2 * words64, 4));
    mr.wst = uint32_t(round_up(mr.words_proc, 32));
    mr.ml = 2;
    mr.L = len;
    DevMerge m{};
    m.thresh11 = coin_threshold(c_recv, c_local) << 11;
    m.key = key;
    m.base_add = used;
    m.key_mode = 1;
    m.recv_src = uint16_t(kSrcLeaf | 0);
    m.local_src = uint16_t(kSrcLeaf | 1);
    m.out_slot = kNone;
    m.out_global = kFinal;
    m.offset_src = -1;
    m.coin_words = 0;  // inline draws
    mr.dp.merges = {m};
    if (mr.cluster) {
        mr.dp.seg_begin = {0, 1};
        mr.dp.lvl_start = {0, 2};
        mr.dp.lvl_begin = {0, 1};
        mr.dp.level_width = 1;
        mr.dp.max_slots = 0;
    } else {
        mr.dp.seg_begin = {0};
        mr.dp.stage_begin = {0, 1};
        mr.dp.n_stages = 1;
        mr.dp.single_lanes();
    }
    mr.dp.n_merges = 1;
    marsit_status s;
    if ((s = mr.configure(sm)) || (s = mr.upload())) return s;
    struct Scratch {
        void* p = nullptr;
        ~Scratch() {
            if (p) cudaFree(p);
        }
    } scratch;
    const size_t leaves_b = sizeof(uint32_t) * 2 * mr.wst, agg_b = sizeof(uint32_t) * mr.wst;
    CUDA_TRY(cudaMalloc(&scratch.p, leaves_b + agg_b));
    uint32_t* leaves = static_cast<uint32_t*>(scratch.p);
    uint32_t* agg = leaves + 2 * mr.wst;
    CUDA_TRY(cudaMemsetAsync(scratch.p, 0, leaves_b + agg_b, st));
    CUDA_TRY(cudaMemcpyAsync(leaves, d_recv, words64 * 8, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(leaves + mr.wst, d_local, words64 * 8, cudaMemcpyDeviceToDevice, st));
    uint64_t n = 0;
    if ((s = mr.run(leaves, agg, nullptr, 0, 0, st, &n))) return s;
    CUDA_TRY(cudaMemcpyAsync(d_out, agg, words64 * 8, cudaMemcpyDeviceToDevice, st));
    std::vector<uint64_t> tot(mr.n_parts);
    CUDA_TRY(cudaMemcpyAsync(tot.data(), mr.part_totals, sizeof(uint64_t) * mr.n_parts,
                             cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (consumed) {
        uint64_t c = 0;
        for (uint64_t v : tot) c += v;
        *consumed = c;
    }
    return MARSIT_OK;
}

marsit_status marsit_bits_account(const marsit_ctx* ctx, int dense, uint64_t* per_worker,
                                  uint64_t* reduce_bits, uint64_t* gather_bits, uint64_t* total) {
    if (!ctx) return fail(MARSIT_EPARAM, "ctx is null");
    const uint64_t unit = dense ? 32ull * ctx->L : ctx->L;  // allreduce.hpp:113, 182
    uint64_t t = 0;
    for (uint32_t w = 0; w < ctx->M; ++w) {
        const uint64_t b = ctx->plan.sends_per_worker[w] * unit;
        if (per_worker) per_worker[w] = b;
        t += b;
    }
    if (reduce_bits) *reduce_bits = ctx->plan.reduce_sends * unit;
    if (gather_bits) *gather_bits = ctx->plan.gather_sends * unit;
    if (total) *total = t;
    return MARSIT_OK;
}

marsit_status marsit_ctx_check(marsit_ctx* ctx, void* stream) {
    if (!ctx) return fail(MARSIT_EPARAM, "ctx is null");
    CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // a stuck peer wait is released by the watchdog (bounded), so this returns
    // stream-ordered reads into pinned memory, completion by polling (no
    // legacy-stream or pageable copy that could wait on other streams)
    CUDA_TRY(cudaMemcpyAsync(ctx->h_check, ctx->err, sizeof(int), cudaMemcpyDeviceToHost, st));
    const bool read_flags = ctx->p2p && ctx->peers_set;
    if (read_flags)
        CUDA_TRY(cudaMemcpyAsync(ctx->h_check + 1, ctx->flags, 2 * sizeof(uint64_t) * ctx->G,
                                 cudaMemcpyDeviceToHost, st));
    if (ctx->watchdog) {
        CUDA_TRY(poll_stream(st, ctx->ev_check));
    } else {  // nothing has to release this stream: a blocking wait is fine
        CUDA_TRY(cudaEventRecord(ctx->ev_check, st));
        CUDA_TRY(cudaEventSynchronize(ctx->ev_check));
    }
    const int flag = *reinterpret_cast<const int*>(ctx->h_check);
    CUDA_TRY(cudaGetLastError());
    marsit_status s;
    if (read_flags && !ctx->fail_status.load()) {
        // a peer whose watchdog gave up released our waits with the abort
        // value: this rank's round read incomplete data
        const uint64_t* fl = ctx->h_check + 1;
        for (uint32_t q = 0; q < ctx->G; ++q)
            if (q != ctx->rank && (fl[q] == kFlagAbort || fl[ctx->G + q] == kFlagAbort)) {
                ctx_set_failed(ctx, MARSIT_EPROTOCOL, "P2P: peer rank " + std::to_string(q) + " aborted");
                break;
            }
    }
    if ((s = ctx_failed(ctx))) return s;
    if (flag) {
        CUDA_TRY(cudaMemsetAsync(ctx->err, 0, sizeof(int), st));
        CUDA_TRY(poll_stream(st, ctx->ev_check));
        if (flag & kErrBounds) return fail(MARSIT_ECUDA, "checked build: a device index failed its bound");
        if (flag & kErrSync)
            return fail(MARSIT_ECUDA, "spread round: CTAs were not co-resident (a wait timed out; results invalid)");
        if (flag & kErrNonFinite) return fail(MARSIT_ENONFINITE, "DenseVector: non-finite entry");
        return fail(MARSIT_EPROTOCOL, "consensus: an aggregate segment differs from its owner's");
    }
    return MARSIT_OK;
}

marsit_status marsit_ctx_p2p_buffers(const marsit_ctx* ctx, marsit_p2p_buffers* out) {
    if (!ctx || !out) return fail(MARSIT_EPARAM, "null argument");
    if (!ctx->p2p) return fail(MARSIT_EPARAM, "not a P2P-transport context (nranks > 1)");
    out->bits = ctx->bits;
    out->agg = ctx->agg;
    out->dense_send = ctx->dense_send;
    out->dense_mean = ctx->dense_mean;
    out->flags = ctx->flags;
    return MARSIT_OK;
}

marsit_status marsit_ctx_set_peers(marsit_ctx* ctx, const marsit_p2p_buffers* peers,
                                   uint32_t nranks) {
    if (!ctx || !peers) return fail(MARSIT_EPARAM, "null argument");
    if (!ctx->p2p) return fail(MARSIT_EPARAM, "not a P2P-transport context (nranks > 1)");
    if (nranks != ctx->G) return fail(MARSIT_EPARAM, "peer table must have one entry per rank");
    std::vector<void*> tab(3 * size_t(ctx->G));
    ctx->peer_flags.assign(ctx->G, nullptr);
    ctx->peer_dense_mean.assign(ctx->G, nullptr);
    for (uint32_t q = 0; q < ctx->G; ++q) {
        const marsit_p2p_buffers& b = peers[q];
        if (!b.bits || !b.agg || !b.dense_send || !b.dense_mean || !b.flags)
            return fail(MARSIT_EPARAM, "peer table: null buffer");
        tab[q] = b.bits;
        tab[ctx->G + q] = b.agg;
        tab[2 * size_t(ctx->G) + q] = b.dense_send;
        ctx->peer_flags[q] = static_cast<const uint64_t*>(b.flags);
        ctx->peer_dense_mean[q] = b.dense_mean;
    }
    CUDA_TRY(cudaSetDevice(ctx->device));
    CUDA_TRY(cudaMemcpy(ctx->d_peer_tables, tab.data(), tab.size() * sizeof(void*),
                        cudaMemcpyHostToDevice));
    ctx->merge.peer_bits = reinterpret_cast<const uint32_t* const*>(ctx->d_peer_tables);
    ctx->peers_set = true;
    if (!ctx->watchdog) ctx->watchdog = std::make_unique<Watchdog>(ctx);
    return MARSIT_OK;
}

marsit_status marsit_ipc_handle(const void* d_ptr, void* handle_out) {
    if (!d_ptr || !handle_out) return fail(MARSIT_EPARAM, "null argument");
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    std::memcpy(handle_out, &h, sizeof(h));
    return MARSIT_OK;
}

marsit_status marsit_ipc_open(const void* handle, int device, void** d_ptr_out) {
    if (!handle || !d_ptr_out) return fail(MARSIT_EPARAM, "null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    CUDA_TRY(cudaSetDevice(device));
    CUDA_TRY(cudaIpcOpenMemHandle(d_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
    return MARSIT_OK;
}

marsit_status marsit_ipc_close(void* d_ptr) {
    if (!d_ptr) return fail(MARSIT_EPARAM, "null argument");
    CUDA_TRY(cudaIpcCloseMemHandle(d_ptr));
    return MARSIT_OK;
}

marsit_status marsit_ctx_set_metrics(marsit_ctx* ctx, int enable) {
    if (!ctx) return fail(MARSIT_EPARAM, "ctx is null");
    CUDA_TRY(cudaSetDevice(ctx->device));
    if (enable && !ctx->d_metrics) {
        CUDA_TRY(cudaMalloc(&ctx->d_metrics, 4 * sizeof(unsigned long long)));
        CUDA_TRY(cudaMemset(ctx->d_metrics, 0, 4 * sizeof(unsigned long long)));
    }
    ctx->metrics = enable != 0;
    return MARSIT_OK;
}

marsit_status marsit_ctx_metrics(marsit_ctx* ctx, marsit_round_metrics* out, void* stream) {
    if (!ctx || !out) return fail(MARSIT_EPARAM, "null argument");
    CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    *out = marsit_round_metrics{};
    out->round = ctx->last_t;
    out->valid = ctx->last_valid ? 1 : 0;
    out->full_precision = ctx->last_dense ? 1 : 0;
    out->dim = ctx->D;
    marsit_bits_account(ctx, ctx->last_dense ? 1 : 0, nullptr, nullptr, nullptr, &out->round_bits);
    if (!ctx->last_valid || ctx->last_dense) return MARSIT_OK;
    if (ctx->last_matching) {
        unsigned long long m = 0;
        CUDA_TRY(cudaMemcpyAsync(&m, ctx->d_metrics, sizeof(m), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        out->has_matching = 1;
        out->matches = m;
        out->matching_rate = double(m) / double(ctx->D);
    }
    // per-merge draw totals of the owned segments, [part][merge]
    const MergeRunner& mr = ctx->merge;
    std::vector<uint64_t> tot(size_t(mr.n_parts) * mr.dp.n_merges);
    if (!tot.empty())
        CUDA_TRY(cudaMemcpyAsync(tot.data(), mr.part_totals, sizeof(uint64_t) * tot.size(),
                                 cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    unsigned long long agg[2] = {0, mr.dp.n_merges};
    for (uint64_t v : tot) agg[0] += v;
    if (ctx->G > 1 && ctx->comm) {
        if (!ctx->d_metrics) CUDA_TRY(cudaMalloc(&ctx->d_metrics, 4 * sizeof(unsigned long long)));
        CUDA_TRY(cudaMemcpyAsync(ctx->d_metrics + 1, agg, sizeof(agg), cudaMemcpyHostToDevice, st));
        NCCL_TRY(ncclAllReduce(ctx->d_metrics + 1, ctx->d_metrics + 1, 2, ncclUint64, ncclSum,
                               ctx->comm, st));
        CUDA_TRY(cudaMemcpyAsync(agg, ctx->d_metrics + 1, sizeof(agg), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    out->rank_local = (ctx->G > 1 && !ctx->comm) ? 1 : 0;
    out->disagreements = agg[0];
    out->merges = agg[1];
    out->compared_bits = agg[1] * ctx->L;
    out->disagreement_rate =
        out->compared_bits ? double(out->disagreements) / double(out->compared_bits) : 0.0;
    return MARSIT_OK;
}

marsit_status marsit_ctx_set_wait_timeout(marsit_ctx* ctx, uint64_t timeout_ms) {
    if (!ctx) return fail(MARSIT_EPARAM, "ctx is null");
    ctx->wait_timeout_ms = timeout_ms;
    return MARSIT_OK;
}

marsit_status marsit_ctx_set_consensus(marsit_ctx* ctx, int enable) {
    if (!ctx) return fail(MARSIT_EPARAM, "ctx is null");
    ctx->consensus = enable != 0;
    return MARSIT_OK;
}

marsit_status marsit_ctx_status(const marsit_ctx* ctx) {
    if (!ctx) return fail(MARSIT_EPARAM, "ctx is null");
    return ctx_failed(ctx);
}

marsit_status marsit_ctx_set_timing(marsit_ctx* ctx, int enable) {
    if (!ctx) return fail(MARSIT_EPARAM, "ctx is null");
    ctx->timing = enable != 0;
    return MARSIT_OK;
}

marsit_status marsit_ctx_timing(marsit_ctx* ctx, float* ms, uint64_t* launches, int reset) {
    if (!ctx) return fail(MARSIT_EPARAM, "ctx is null");
    CUDA_TRY(cudaSetDevice(ctx->device));
    for (auto& tp : ctx->pending) {
        CUDA_TRY(cudaEventSynchronize(tp.b));
        float e = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&e, tp.a, tp.b));
        ctx->ms[tp.phase] += e;
        ctx->event_pool.push_back(tp.a);
        ctx->event_pool.push_back(tp.b);
    }
    ctx->pending.clear();
    for (int i = 0; i < MARSIT_N_PHASES; ++i) {
        if (ms) ms[i] = ctx->ms[i];
        if (launches) launches[i] = ctx->launches[i];
        if (reset) {
            ctx->ms[i] = 0.f;
            ctx->launches[i] = 0;
        }
    }
    return MARSIT_OK;
}

marsit_status marsit_fill_recipe(int recipe, uint64_t seed, uint64_t worker, uint64_t round,
                                 uint64_t dim, marsit_dtype dtype, void* d_out, void* stream) {
    if (!d_out) return fail(MARSIT_EPARAM, "out is null");
    if (recipe != 0 && recipe != 1) return fail(MARSIT_EPARAM, "unknown recipe");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == MARSIT_F32)
        CUDA_TRY(launch_fill_recipe<float>(recipe, seed, worker, round, dim,
                                           static_cast<float*>(d_out), st));
    else
        CUDA_TRY(launch_fill_recipe<double>(recipe, seed, worker, round, dim,
                                            static_cast<double*>(d_out), st));
    return MARSIT_OK;
}

}  // extern "C"
