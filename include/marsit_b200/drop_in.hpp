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
//    device context per (D, schedule) (scratch buffers, compiled plan).
#pragma once

#include <marsit/allreduce.hpp>
#include <marsit/schedule.hpp>
#include <marsit/ssdm.hpp>
#include <marsit/sync.hpp>

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../marsit_b200.h"

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

// One cached context per (D, schedule tables); fp64 instantiation.
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
    static std::mutex mu;
    static std::map<std::pair<size_t, std::vector<uint32_t>>, std::unique_ptr<CachedCtx>> cache;
    std::lock_guard<std::mutex> lock(mu);
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
    detail::DeviceBuffer dg(W * bytes), dc(W * bytes), dout(W * bytes), dupd(bytes),
        dagg(((dim + 63) / 64) * 8);
    std::vector<const void*> gp(W), cp(W);
    std::vector<void*> op(W);
    for (uint32_t w = 0; w < W; ++w) {
        char* g = static_cast<char*>(dg.p) + w * bytes;
        char* c = static_cast<char*>(dc.p) + w * bytes;
        detail::cuda_check(cudaMemcpy(g, scaled_grads[w].values().data(), bytes, cudaMemcpyHostToDevice), "H2D");
        detail::cuda_check(cudaMemcpy(c, comp[w].c.values().data(), bytes, cudaMemcpyHostToDevice), "H2D");
        gp[w] = g;
        cp[w] = c;
        op[w] = static_cast<char*>(dout.p) + w * bytes;
    }
    const std::uint64_t period = cfg.full_precision_period ? *cfg.full_precision_period : 0;
    int full = 0;
    detail::check(::marsit_round(ctx, t, period, cfg.eta_s, global_seed, gp.data(), cp.data(),
                                 op.data(), static_cast<uint64_t*>(dagg.p), dupd.p, &full, nullptr));
    detail::check(marsit_ctx_check(ctx, nullptr));  // DenseVector finiteness (sync)
    std::vector<double> upd(dim);
    detail::cuda_check(cudaMemcpy(upd.data(), dupd.p, bytes, cudaMemcpyDeviceToHost), "D2H");
    MarsitRoundResult out{DenseVector(std::move(upd)), {}, detail::bits_account(ctx, W, full != 0),
                          full != 0, std::nullopt};
    for (uint32_t w = 0; w < W; ++w) {
        std::vector<double> c(dim);
        detail::cuda_check(cudaMemcpy(c.data(), op[w], bytes, cudaMemcpyDeviceToHost), "D2H");
        out.compensation.push_back(CompensationState{DenseVector(std::move(c))});
    }
    if (!full) {
        PackedSignVector bits = PackedSignVector::zeros(dim);
        std::vector<std::uint64_t> words((dim + 63) / 64);
        detail::cuda_check(cudaMemcpy(words.data(), dagg.p, words.size() * 8, cudaMemcpyDeviceToHost), "D2H");
        for (size_t j = 0; j < dim; ++j)
            if ((words[j >> 6] >> (j & 63)) & 1u) bits.set_bit(j, true);
        out.aggregate_bits = std::move(bits);
    }
    return out;
}

// allreduce.hpp:148-189, same signature and result (every worker's state
// is the consensus aggregate, as for ring and torus schedules).
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
    for (size_t w = 0; w < v.size(); ++w) {
        char* d = static_cast<char*>(buf.p) + w * bytes;
        cuda_check(cudaMemcpy(d, v[w].values().data(), bytes, cudaMemcpyHostToDevice), "H2D");
        ptrs[w] = d;
    }
    return ptrs;
}

inline DenseVector download(const void* d, size_t n) {
    std::vector<double> h(n);
    cuda_check(cudaMemcpy(h.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    return DenseVector(std::move(h));
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
