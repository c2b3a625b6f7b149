// drop_in.hpp — the reference's C++ sync API, executed by the B200 path.
//
// A maintainer of the reference (/root/reference/proj, header-only C++20)
// switches a call site from
//     marsit::marsit_round(t, cfg, grads, comp, sched, seed)        // sync.hpp:60-63
//     marsit::allreduce_sign(signs, sched, RoundContext{seed, t})   // allreduce.hpp:148-149
// to marsit::gpu::marsit_round / marsit::gpu::allreduce_sign with the SAME
// arguments and result types; likewise allreduce_dense (allreduce.hpp:98-130)
// and the SSDM baselines cascading_allreduce / sum_ssdm_allreduce
// (allreduce.hpp:205-339).  This header includes the reference's own
// headers for those types (marsit/sync.hpp), so it compiles inside the
// reference tree with -I<b200 repo>/include and links against
// libmarsit_b200.so and libcudart.
//
// Semantics match the reference exactly:
//  * inputs are doubles, so the device path runs the fp64 kernel
//    instantiation: u = g + c and c' = u - g_t are the same IEEE operations
//    as dense_vector.hpp:53-69, and the sign bits, the merge coins
//    (rng.hpp:28-54) and the aggregate are bit-identical;
//  * errors surface as the reference exception types (errors.hpp:10-42);
//  * value semantics: nothing is retained between calls except a cached
//    device context per (calling thread, D, schedule) (scratch buffers,
//    compiled plan) and pinned staging buffers per calling thread;
//  * re-entrant like the reference's pure functions: concurrent calls from
//    different host threads never share a context, scratch or staging
//    buffer (the C-ABI allows one host thread per context).
#pragma once

#include <marsit/allreduce.hpp>
#include <marsit/schedule.hpp>
#include <marsit/ssdm.hpp>
#include <marsit/sync.hpp>

#include <cuda_runtime.h>
#include <sys/mman.h>

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <bit>
#include <exception>
#include <optional>
#include <thread>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../marsit_b200.h"

#ifdef MARSIT_DROPIN_PROFILE
#include <chrono>
#include <cstdio>
#define MARSIT_DROPIN_T(v) const auto v = std::chrono::steady_clock::now()
#else
#define MARSIT_DROPIN_T(v)
#endif

namespace marsit::gpu {

namespace detail {

[[noreturn]] inline void raise(marsit_status st) {
    const std::string msg = std::string("marsit_b200: ") + marsit_last_error();
    switch (st) {
        case MARSIT_ENONFINITE: throw non_finite_error(msg);
        case MARSIT_EPARAM: throw parameter_error(msg);
        case MARSIT_EPROTOCOL: throw protocol_error(msg);
        case MARSIT_EUNSUPPORTED: throw unsupported_error(msg);
        default: throw std::runtime_error(msg);
    }
}

inline void check(marsit_status st) {
    if (st != MARSIT_OK) raise(st);
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device buffer with RAII.
struct DeviceBuffer {
    void* p = nullptr;
    explicit DeviceBuffer(size_t bytes) { cuda_check(cudaMalloc(&p, bytes ? bytes : 1), "cudaMalloc"); }
    ~DeviceBuffer() { cudaFree(p); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

// Grow-only device scratch reused across calls (per host thread): the
// value-semantics entry points stage their inputs here instead of allocating
// (and synchronously freeing) device memory on every call.
inline void* scratch(int slot, size_t bytes) {
    struct Pool {
        void* p[8] = {};
        size_t n[8] = {};
        ~Pool() {
            for (void* q : p)
                if (q) cudaFree(q);
        }
    };
    thread_local Pool pool;
    if (pool.n[slot] < bytes) {
        if (pool.p[slot]) cuda_check(cudaFree(pool.p[slot]), "cudaFree");
        pool.p[slot] = nullptr;
        pool.n[slot] = 0;
        cuda_check(cudaMalloc(&pool.p[slot], bytes ? bytes : 1), "cudaMalloc");
        pool.n[slot] = bytes;
    }
    return pool.p[slot];
}

// Pinned double-buffered staging per (calling thread, worker slot), grow-only:
// a helper thread copies a pageable vector chunk by chunk into pinned memory
// while the previous chunk's DMA runs on its own stream.
struct Staging {
    static constexpr size_t kChunk = size_t(16) << 20;  // bytes per buffer
    void* buf[2] = {nullptr, nullptr};
    cudaStream_t st = nullptr;
    cudaEvent_t done[2] = {nullptr, nullptr};
    Staging() {
        for (int b = 0; b < 2; ++b) {
            cuda_check(cudaHostAlloc(&buf[b], kChunk, cudaHostAllocDefault), "cudaHostAlloc");
            cuda_check(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming), "cudaEventCreate");
        }
        cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    // host (pageable) -> device, pipelined through the two pinned buffers
    void to_device(void* dst, const void* src, size_t bytes) {
        int b = 0;
        for (size_t off = 0; off < bytes; off += kChunk, b ^= 1) {
            const size_t n = std::min(kChunk, bytes - off);
            cuda_check(cudaEventSynchronize(done[b]), "staging");  // buffer b free again
            std::memcpy(buf[b], static_cast<const char*>(src) + off, n);
            cuda_check(cudaMemcpyAsync(static_cast<char*>(dst) + off, buf[b], n,
                                       cudaMemcpyHostToDevice, st), "H2D");
            cuda_check(cudaEventRecord(done[b], st), "staging");
        }
        cuda_check(cudaStreamSynchronize(st), "H2D");
    }
    // device -> freshly allocated host vector (written once, no zero fill)
    std::vector<double> to_host(const void* src, size_t count) {
        std::vector<double> out;
        out.reserve(count);
        const size_t bytes = count * sizeof(double);
#ifdef MADV_HUGEPAGE
        {  // fresh pages: ask for transparent huge pages (fewer first-touch faults)
            const uintptr_t a = reinterpret_cast<uintptr_t>(out.data());
            const uintptr_t lo = (a + (size_t(2) << 20) - 1) & ~((uintptr_t(2) << 20) - 1);
            const uintptr_t hi = (a + bytes) & ~((uintptr_t(2) << 20) - 1);
            if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
        }
#endif
        const size_t n0 = std::min(kChunk, bytes);
        cuda_check(cudaMemcpyAsync(buf[0], src, n0, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaEventRecord(done[0], st), "staging");
        int b = 0;
        for (size_t off = 0; off < bytes; off += kChunk, b ^= 1) {
            const size_t n = std::min(kChunk, bytes - off);
            if (off + n < bytes) {  // the next chunk's DMA under this chunk's copy-out
                const size_t n1 = std::min(kChunk, bytes - off - n);
                cuda_check(cudaMemcpyAsync(buf[b ^ 1], static_cast<const char*>(src) + off + n, n1,
                                           cudaMemcpyDeviceToHost, st), "D2H");
                cuda_check(cudaEventRecord(done[b ^ 1], st), "staging");
            }
            cuda_check(cudaEventSynchronize(done[b]), "staging");
            const double* p = static_cast<const double*>(buf[b]);
            out.insert(out.end(), p, p + n / sizeof(double));
        }
        return out;
    }
};
// `owner` is the thread that called the entry point (its helper threads use
// the owner's buffers), so concurrent callers never share a slot.
inline Staging& staging(std::thread::id owner, uint32_t slot) {
    static std::mutex mu;
    static std::map<std::pair<std::thread::id, uint32_t>, std::unique_ptr<Staging>> pool;
    std::lock_guard<std::mutex> lock(mu);
    auto& p = pool[{owner, slot}];
    if (!p) p = std::make_unique<Staging>();
    return *p;
}

// Run f(i) for i in [0, n) on n host threads (the per-worker staging: the
// pageable copies, the page faults of fresh result vectors and DenseVector's
// finiteness scan all scale with threads).
template <class F>
inline void parallel_for(uint32_t n, F&& f) {
    if (n <= 1) {
        if (n == 1) f(0u);
        return;
    }
    std::vector<std::thread> th;
    std::vector<std::exception_ptr> err(n);
    for (uint32_t i = 0; i < n; ++i)
        th.emplace_back([&, i] {
            try {
                f(i);
            } catch (...) {
                err[i] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

// marsit::Schedule (schedule.hpp:31-55) -> flat tables -> marsit_schedule.
struct ScheduleHandle {
    marsit_schedule* s = nullptr;
    explicit ScheduleHandle(const Schedule& sched) {
        const uint32_t W = sched.workers, K = static_cast<uint32_t>(sched.steps.size());
        std::vector<uint8_t> phase(K);
        std::vector<uint32_t> st(size_t(K) * W), rf(st.size()), sg(st.size());
        for (uint32_t k = 0; k < K; ++k) {
            phase[k] = sched.steps[k].phase == Phase::reduce ? MARSIT_REDUCE : MARSIT_GATHER;
            if (sched.steps[k].entries.size() != W) throw protocol_error("Schedule: step entry count != workers");
            for (uint32_t w = 0; w < W; ++w) {
                const ScheduleEntry& e = sched.steps[k].entries[w];
                st[size_t(k) * W + w] = e.send_to;
                rf[size_t(k) * W + w] = e.recv_from;
                sg[size_t(k) * W + w] = e.segment;
            }
        }
        check(marsit_schedule_from_tables(W, sched.segments, K, phase.data(), st.data(), rf.data(),
                                          sg.data(), &s));
    }
    ~ScheduleHandle() { marsit_schedule_destroy(s); }
};

// One cached context per (calling thread, D, schedule tables); fp64
// instantiation.  Thread-local: a context's device scratch (packed signs,
// aggregate, coin buffers, error latch) serves one round at a time.
struct CachedCtx {
    std::unique_ptr<ScheduleHandle> sched;
    marsit_ctx* ctx = nullptr;
    ~CachedCtx() { marsit_ctx_destroy(ctx); }
};

inline std::vector<uint32_t> schedule_key(const Schedule& s) {
    std::vector<uint32_t> k{s.workers, s.segments, static_cast<uint32_t>(s.steps.size())};
    for (const auto& step : s.steps) {
        k.push_back(step.phase == Phase::reduce ? 0u : 1u);
        for (const auto& e : step.entries) {
            k.push_back(e.send_to);
            k.push_back(e.recv_from);
            k.push_back(e.segment);
        }
    }
    return k;
}

inline marsit_ctx* context_for(size_t dim, const Schedule& sched) {
    thread_local std::map<std::pair<size_t, std::vector<uint32_t>>, std::unique_ptr<CachedCtx>> cache;
    auto key = std::make_pair(dim, schedule_key(sched));
    auto it = cache.find(key);
    if (it != cache.end()) return it->second->ctx;
    auto c = std::make_unique<CachedCtx>();
    c->sched = std::make_unique<ScheduleHandle>(sched);
    marsit_ctx_desc d{};
    d.dim = dim;
    d.schedule = c->sched->s;
    d.dtype = MARSIT_F64;
    d.device = 0;
    d.nranks = 1;
    d.rank = 0;
    check(marsit_ctx_create(&d, &c->ctx));
    marsit_ctx* out = c->ctx;
    cache.emplace(std::move(key), std::move(c));
    return out;
}

inline BitsAccount bits_account(marsit_ctx* ctx, uint32_t workers, bool dense) {
    BitsAccount b(workers);
    check(marsit_bits_account(ctx, dense ? 1 : 0, b.per_worker.data(), &b.reduce_bits,
                              &b.gather_bits, &b.total));
    return b;
}

}  // namespace detail

// sync.hpp:60-120, same signature and result.
inline MarsitRoundResult marsit_round(std::uint64_t t, const SyncConfig& cfg,
                                      const std::vector<DenseVector>& scaled_grads,
                                      const std::vector<CompensationState>& comp,
                                      const Schedule& sched, std::uint64_t global_seed) {
    cfg.validate();
    if (scaled_grads.size() != sched.workers || comp.size() != sched.workers)
        throw parameter_error("marsit_round: worker count mismatch");
    const size_t dim = scaled_grads[0].size();
    for (std::uint32_t w = 0; w < sched.workers; ++w)
        if (scaled_grads[w].size() != dim || comp[w].c.size() != dim)
            throw parameter_error("marsit_round: dimension mismatch");
    marsit_ctx* ctx = detail::context_for(dim, sched);
    const uint32_t W = sched.workers;
    const size_t bytes = dim * sizeof(double);
    struct Buf {
        void* p;
    };
    const Buf dg{detail::scratch(0, W * bytes)}, dc{detail::scratch(1, W * bytes)},
        dout{detail::scratch(2, W * bytes)}, dupd{detail::scratch(3, bytes)},
        dagg{detail::scratch(4, ((dim + 63) / 64) * 8)};
    std::vector<const void*> gp(W), cp(W);
    std::vector<void*> op(W);
    for (uint32_t w = 0; w < W; ++w) {
        gp[w] = static_cast<char*>(dg.p) + w * bytes;
        cp[w] = static_cast<char*>(dc.p) + w * bytes;
        op[w] = static_cast<char*>(dout.p) + w * bytes;
    }
    MARSIT_DROPIN_T(t0);
    const std::thread::id owner = std::this_thread::get_id();
    detail::parallel_for(2 * W, [&](uint32_t i) {  // one host thread and pinned pipeline per vector
        const uint32_t w = i / 2;
        if (i % 2 == 0)
            detail::staging(owner, i).to_device(const_cast<void*>(gp[w]), scaled_grads[w].values().data(), bytes);
        else
            detail::staging(owner, i).to_device(const_cast<void*>(cp[w]), comp[w].c.values().data(), bytes);
    });
    MARSIT_DROPIN_T(t1);
    const std::uint64_t period = cfg.full_precision_period ? *cfg.full_precision_period : 0;
    int full = 0;
    detail::check(::marsit_round(ctx, t, period, cfg.eta_s, global_seed, gp.data(), cp.data(),
                                 op.data(), static_cast<uint64_t*>(dagg.p), dupd.p, &full, nullptr));
    detail::check(marsit_ctx_check(ctx, nullptr));  // DenseVector finiteness (sync)
    MARSIT_DROPIN_T(t2);
    std::vector<double> upd(dim);
    detail::cuda_check(cudaMemcpy(upd.data(), dupd.p, bytes, cudaMemcpyDeviceToHost), "D2H");
    MarsitRoundResult out{DenseVector(std::move(upd)), {}, detail::bits_account(ctx, W, full != 0),
                          full != 0, std::nullopt};
    std::vector<std::optional<CompensationState>> cs(W);
    detail::parallel_for(W, [&](uint32_t w) {
        cs[w].emplace(CompensationState{DenseVector(detail::staging(owner, w).to_host(op[w], dim))});
    });
    out.compensation.reserve(W);
    for (auto& c : cs) out.compensation.push_back(std::move(*c));
    MARSIT_DROPIN_T(t3);
    if (!full) {
        PackedSignVector bits = PackedSignVector::zeros(dim);
        std::vector<std::uint64_t> words((dim + 63) / 64);
        detail::cuda_check(cudaMemcpy(words.data(), dagg.p, words.size() * 8, cudaMemcpyDeviceToHost), "D2H");
        for (size_t k = 0; k < words.size(); ++k)  // set bits only (the type has no word setter)
            for (std::uint64_t x = words[k]; x; x &= x - 1)
                bits.set_bit(k * 64 + static_cast<size_t>(std::countr_zero(x)), true);
        out.aggregate_bits = std::move(bits);
    }
    MARSIT_DROPIN_T(t4);
#ifdef MARSIT_DROPIN_PROFILE
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "drop-in: stage-in %.1f  round %.1f  results %.1f  bits %.1f ms\n",
                 ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4));
#endif
    return out;
}

// allreduce.hpp:148-189, same signature and result for schedules that end in
// consensus (ring, torus): every worker's state is the consensus aggregate.
// Schedules whose workers end in different states (e.g. reduce-only tables)
// raise unsupported_error: the device path materialises one aggregate per
// segment.
inline SignAllreduceResult allreduce_sign(const std::vector<std::vector<PackedSignVector>>& signs,
                                          const Schedule& sched, const RoundContext& rc) {
    if (signs.size() != sched.workers) throw parameter_error("allreduce_sign: worker count mismatch");
    const uint32_t W = sched.workers, S = sched.segments;
    for (uint32_t w = 0; w < W; ++w) {
        if (signs[w].size() != S) throw parameter_error("allreduce_sign: segment count mismatch");
        for (uint32_t s = 0; s < S; ++s)
            if (signs[w][s].size() != signs[0][0].size())
                throw protocol_error("allreduce_sign: segment length mismatch");
    }
    const size_t L = signs[0][0].size();
    const size_t nw = (L + 63) / 64;
    marsit_ctx* ctx = detail::context_for(L * S, sched);  // ceil(D/S) == L
    std::vector<std::uint64_t> host(size_t(W) * S * nw);
    for (uint32_t w = 0; w < W; ++w)
        for (uint32_t s = 0; s < S; ++s)
            std::copy(signs[w][s].words().begin(), signs[w][s].words().end(),
                      host.begin() + (size_t(w) * S + s) * nw);
    detail::DeviceBuffer din(host.size() * 8), dout(size_t(S) * nw * 8);
    detail::cuda_check(cudaMemcpy(din.p, host.data(), host.size() * 8, cudaMemcpyHostToDevice), "H2D");
    std::vector<uint32_t> counts(S);
    detail::check(marsit_allreduce_sign(ctx, rc.round, rc.global_seed,
                                        static_cast<const uint64_t*>(din.p),
                                        static_cast<uint64_t*>(dout.p), counts.data(), nullptr));
    std::vector<std::uint64_t> agg(size_t(S) * nw);
    detail::cuda_check(cudaMemcpy(agg.data(), dout.p, agg.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    std::vector<AggregateSign> consensus_state;
    for (uint32_t s = 0; s < S; ++s) {
        PackedSignVector v = PackedSignVector::zeros(L);
        for (size_t j = 0; j < L; ++j)
            if ((agg[size_t(s) * nw + (j >> 6)] >> (j & 63)) & 1u) v.set_bit(j, true);
        consensus_state.push_back(AggregateSign{std::move(v), counts[s]});
    }
    SignAllreduceResult out{std::vector<std::vector<AggregateSign>>(W, consensus_state),
                            detail::bits_account(ctx, W, false)};
    // BitsAccount of allreduce_sign counts L bits per send (allreduce.hpp:182)
    return out;
}

namespace detail {

inline void check_vectors(const std::vector<DenseVector>& v, const Schedule& sched) {
    // allreduce.hpp:75-84
    if (v.size() != sched.workers) throw parameter_error("allreduce: vector count != schedule workers");
    for (const DenseVector& x : v)
        if (x.size() != v[0].size()) throw parameter_error("allreduce: inconsistent dimensions");
}

// Upload M host vectors into one device buffer; returns the per-worker pointers.
inline std::vector<const void*> upload(const std::vector<DenseVector>& v, DeviceBuffer& buf) {
    const size_t bytes = v[0].size() * sizeof(double);
    std::vector<const void*> ptrs(v.size());
    for (size_t w = 0; w < v.size(); ++w) ptrs[w] = static_cast<char*>(buf.p) + w * bytes;
    const std::thread::id owner = std::this_thread::get_id();
    parallel_for(uint32_t(v.size()), [&](uint32_t w) {  // pinned pipeline per vector
        staging(owner, w).to_device(const_cast<void*>(ptrs[w]), v[w].values().data(), bytes);
    });
    return ptrs;
}

inline DenseVector download(const void* d, size_t n) {
    return DenseVector(staging(std::this_thread::get_id(), 0).to_host(d, n));
}

}  // namespace detail

// allreduce.hpp:98-130, same signature and result: the schedule-order sum
// scaled by 1/M at every worker.  Runs as a dense round whose compensation is
// -0.0 (x + -0.0 == x bit for bit, including x = -0.0).
inline DenseAllreduceResult allreduce_dense(const std::vector<DenseVector>& vectors,
                                            const Schedule& sched) {
    detail::check_vectors(vectors, sched);
    const size_t dim = vectors[0].size();
    const uint32_t W = sched.workers;
    marsit_ctx* ctx = detail::context_for(dim, sched);
    const size_t bytes = dim * sizeof(double);
    detail::DeviceBuffer dv(W * bytes), dz(bytes), dscr(W * bytes), dmean(bytes);
    std::vector<const void*> vp = detail::upload(vectors, dv);
    std::vector<double> negzero(dim, -0.0);
    detail::cuda_check(cudaMemcpy(dz.p, negzero.data(), bytes, cudaMemcpyHostToDevice), "H2D");
    std::vector<const void*> zp(W, dz.p);
    std::vector<void*> sp(W);
    for (uint32_t w = 0; w < W; ++w) sp[w] = static_cast<char*>(dscr.p) + w * bytes;
    detail::check(marsit_dense_round(ctx, 0, vp.data(), zp.data(), sp.data(), dmean.p, nullptr));
    detail::check(marsit_ctx_check(ctx, nullptr));
    DenseVector mean = detail::download(dmean.p, dim);
    return DenseAllreduceResult{std::vector<DenseVector>(W, mean), detail::bits_account(ctx, W, true)};
}

namespace detail {
inline std::pair<DenseVector, BitsAccount> ssdm(int mode, const std::vector<DenseVector>& vectors,
                                                const Schedule& sched, const RoundContext& rc,
                                                std::vector<std::int64_t>* max_abs) {
    if (sched.topology != Topology::ring)
        throw unsupported_error(mode == MARSIT_SSDM_CASCADING
                                    ? "cascading_allreduce: only ring schedules are supported"
                                    : "sum_ssdm_allreduce: only ring schedules are supported");
    check_vectors(vectors, sched);
    const size_t dim = vectors[0].size();
    const uint32_t W = sched.workers;
    marsit_ctx* ctx = context_for(dim, sched);
    DeviceBuffer dv(W * dim * sizeof(double)), dout(dim * sizeof(double));
    std::vector<const void*> vp = upload(vectors, dv);
    BitsAccount bits(W);
    std::vector<std::int64_t> mx(sched.steps.size() + 1);
    check(marsit_ssdm_allreduce(ctx, mode, rc.round, rc.global_seed, vp.data(), dout.p,
                                bits.per_worker.data(), &bits.reduce_bits, &bits.gather_bits,
                                mx.data(), nullptr));
    check(marsit_ctx_check(ctx, nullptr));
    bits.total = bits.reduce_bits + bits.gather_bits;
    if (max_abs) *max_abs = std::vector<std::int64_t>(mx.begin(), mx.begin() + sched.steps.size());
    return {download(dout.p, dim), std::move(bits)};
}
}  // namespace detail

// allreduce.hpp:205-262, same signature and result.  The l2 norms are summed
// in a fixed parallel order: bit-identical whenever the reference's
// sequential sums are exact, within its own rounding otherwise.
inline CascadingAllreduceResult cascading_allreduce(const std::vector<DenseVector>& vectors,
                                                    const Schedule& sched, const RoundContext& rc) {
    auto r = detail::ssdm(MARSIT_SSDM_CASCADING, vectors, sched, rc, nullptr);
    return CascadingAllreduceResult{std::vector<DenseVector>(sched.workers, r.first),
                                    std::move(r.second)};
}

// allreduce.hpp:275-339, same signature and result.
inline SumSsdmAllreduceResult sum_ssdm_allreduce(const std::vector<DenseVector>& vectors,
                                                 const Schedule& sched, const RoundContext& rc) {
    std::vector<std::int64_t> mx;
    auto r = detail::ssdm(MARSIT_SSDM_SUM, vectors, sched, rc, &mx);
    return SumSsdmAllreduceResult{std::vector<DenseVector>(sched.workers, r.first),
                                  std::move(r.second), std::move(mx)};
}

}  // namespace marsit::gpu
