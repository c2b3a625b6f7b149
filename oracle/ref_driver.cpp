// ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper around the UNMODIFIED reference headers
// (/root/reference/proj/include/marsit/*.hpp, compiled in place with
// -I, never copied).  Built by oracle/build_ref.sh into
// oracle/_ref/libmarsit_ref.so.  Used to (1) pin the C restatement in
// oracle/marsit_oracle.c, (2) generate tests/golden/ fixtures, and
// (3) time the reference's own CPU path as bench.py's reference arm.
//
// Status codes: 0 ok, 1 parameter_error, 2 non_finite_error,
// 3 protocol_error, 4 unsupported_error, 9 other exception.

#include <marsit/allreduce.hpp>
#include <marsit/analysis.hpp>
#include <marsit/merge.hpp>
#include <marsit/rng.hpp>
#include <marsit/schedule.hpp>
#include <marsit/ssdm.hpp>
#include <marsit/sync.hpp>

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <vector>

using namespace marsit;

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const non_finite_error&) {
        return 2;
    } catch (const parameter_error&) {
        return 1;
    } catch (const protocol_error&) {
        return 3;
    } catch (const unsupported_error&) {
        return 4;
    } catch (...) {
        return 9;
    }
}

Schedule make_schedule(int topology, std::uint32_t a, std::uint32_t b) {
    return topology == 0 ? build_ring_schedule(a) : build_torus_schedule(a, b);
}

PackedSignVector from_words(const std::uint64_t* words, std::size_t len) {
    PackedSignVector v = PackedSignVector::zeros(len);
    for (std::size_t j = 0; j < len; ++j)
        if ((words[j >> 6] >> (j & 63)) & 1u) v.set_bit(j, true);
    return v;
}

void to_words(const PackedSignVector& v, std::uint64_t* out) {
    const auto& w = v.words();
    std::memcpy(out, w.data(), w.size() * sizeof(std::uint64_t));
}

} // namespace

extern "C" {

// Schedule tables (schedule.hpp:61-196). Returns steps, or -status.
int ref_build_schedule(int topology, std::uint32_t a, std::uint32_t b, std::uint8_t* phase,
                       std::uint32_t* send_to, std::uint32_t* recv_from, std::uint32_t* segment) {
    Schedule s;
    int rc = guarded([&] { s = make_schedule(topology, a, b); });
    if (rc) return -rc;
    for (std::size_t k = 0; k < s.steps.size(); ++k) {
        phase[k] = s.steps[k].phase == Phase::reduce ? 0 : 1;
        for (std::uint32_t w = 0; w < s.workers; ++w) {
            const auto& e = s.steps[k].entries[w];
            send_to[k * s.workers + w] = e.send_to;
            recv_from[k * s.workers + w] = e.recv_from;
            segment[k * s.workers + w] = e.segment;
        }
    }
    return static_cast<int>(s.steps.size());
}

// First n next_u64() draws of RngStream(seed, purpose, w, t, s) (rng.hpp:28-43).
void ref_stream_draws(std::uint64_t seed, std::uint64_t purpose, std::uint64_t w, std::uint64_t t,
                      std::uint64_t s, std::size_t n, std::uint64_t* out) {
    RngStream rng(seed, static_cast<RngPurpose>(purpose), w, t, s);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng.next_u64();
}

int ref_pack_signs(const double* v, std::size_t len, std::uint64_t* words) {
    return guarded([&] {
        DenseVector d(std::vector<double>(v, v + len));
        to_words(pack_signs(d), words);
    });
}

// merge_signs (merge.hpp:34-58) on a stream that has already produced
// `skip` draws; returns the number of draws consumed in *consumed.
int ref_merge_signs(const std::uint64_t* recv, std::uint32_t c_recv, const std::uint64_t* local,
                    std::uint32_t c_local, std::size_t len, std::uint64_t seed, std::uint64_t w,
                    std::uint64_t t, std::uint64_t s, std::uint64_t skip, std::uint64_t* out,
                    std::uint64_t* consumed) {
    return guarded([&] {
        RngStream rng(seed, RngPurpose::merge, w, t, s);
        for (std::uint64_t i = 0; i < skip; ++i) rng.next_u64();
        AggregateSign r{from_words(recv, len), c_recv};
        AggregateSign l{from_words(local, len), c_local};
        AggregateSign o = merge_signs(r, l, rng);
        to_words(o.bits, out);
        // Count consumed draws by comparing with a fresh stream.
        RngStream probe(seed, RngPurpose::merge, w, t, s);
        RngStream after = rng;
        const std::uint64_t next = after.next_u64();
        std::uint64_t n = 0;
        while (probe.next_u64() != next) ++n;
        *consumed = n - skip;
    });
}

// allreduce_sign (allreduce.hpp:148-189) for a ring (topology 0, a=m) or
// torus (topology 1, a=rows, b=cols).  signs: [w][s][ceil(L/64)].
int ref_allreduce_sign(int topology, std::uint32_t a, std::uint32_t b, std::size_t seg_len,
                       const std::uint64_t* signs, std::uint64_t seed, std::uint64_t round,
                       std::uint64_t* out_state, std::uint32_t* out_counts,
                       std::uint64_t* bits_per_worker, std::uint64_t* reduce_bits,
                       std::uint64_t* gather_bits) {
    return guarded([&] {
        const Schedule sched = make_schedule(topology, a, b);
        const std::size_t nw = (seg_len + 63) / 64;
        std::vector<std::vector<PackedSignVector>> in(sched.workers);
        for (std::uint32_t w = 0; w < sched.workers; ++w)
            for (std::uint32_t s = 0; s < sched.segments; ++s)
                in[w].push_back(from_words(signs + (w * sched.segments + s) * nw, seg_len));
        SignAllreduceResult res = allreduce_sign(in, sched, RoundContext{seed, round});
        for (std::uint32_t w = 0; w < sched.workers; ++w) {
            bits_per_worker[w] = res.bits.per_worker[w];
            for (std::uint32_t s = 0; s < sched.segments; ++s) {
                to_words(res.per_worker[w][s].bits, out_state + (w * sched.segments + s) * nw);
                out_counts[w * sched.segments + s] = res.per_worker[w][s].count;
            }
        }
        *reduce_bits = res.bits.reduce_bits;
        *gather_bits = res.bits.gather_bits;
    });
}

// marsit_round (sync.hpp:60-120).  grads/comp: [M][D] doubles.
int ref_marsit_round(std::uint64_t t, int has_period, std::uint64_t period, double eta_s,
                     int topology, std::uint32_t a, std::uint32_t b, std::size_t dim,
                     const double* grads, const double* comp, std::uint64_t seed,
                     double* out_update, double* out_comp, std::uint64_t* out_agg_bits,
                     int* out_full_precision, std::uint64_t* bits_per_worker,
                     std::uint64_t* reduce_bits, std::uint64_t* gather_bits) {
    return guarded([&] {
        const Schedule sched = make_schedule(topology, a, b);
        SyncConfig cfg;
        if (has_period) cfg.full_precision_period = period;
        cfg.eta_s = eta_s;
        std::vector<DenseVector> g;
        std::vector<CompensationState> c;
        for (std::uint32_t w = 0; w < sched.workers; ++w) {
            g.emplace_back(std::vector<double>(grads + w * dim, grads + (w + 1) * dim));
            c.push_back(CompensationState{
                DenseVector(std::vector<double>(comp + w * dim, comp + (w + 1) * dim))});
        }
        MarsitRoundResult res = marsit_round(t, cfg, g, c, sched, seed);
        std::memcpy(out_update, res.global_update.values().data(), dim * sizeof(double));
        for (std::uint32_t w = 0; w < sched.workers; ++w)
            std::memcpy(out_comp + w * dim, res.compensation[w].c.values().data(),
                        dim * sizeof(double));
        *out_full_precision = res.full_precision ? 1 : 0;
        if (res.aggregate_bits) to_words(*res.aggregate_bits, out_agg_bits);
        for (std::uint32_t w = 0; w < sched.workers; ++w)
            bits_per_worker[w] = res.bits.per_worker[w];
        *reduce_bits = res.bits.reduce_bits;
        *gather_bits = res.bits.gather_bits;
    });
}

// The trainer's per-round matching figure: matching_rate (analysis.hpp:244-253)
// of the aggregate bits against the mean of u_w = add(g_w, c_w) summed in
// worker order and divided by W (trainer.hpp:241-251).  *matches receives
// the count (rate * dim, exact for dim < 2^53).
int ref_matching(const std::uint64_t* agg_words, std::size_t dim, std::uint32_t workers,
                 const double* grads, const double* comp, double* rate, std::uint64_t* matches) {
    return guarded([&] {
        std::vector<double> mean(dim, 0.0);
        for (std::uint32_t w = 0; w < workers; ++w) {
            const DenseVector g(std::vector<double>(grads + w * dim, grads + (w + 1) * dim));
            const DenseVector c(std::vector<double>(comp + w * dim, comp + (w + 1) * dim));
            const DenseVector u = add(g, c);
            for (std::size_t j = 0; j < dim; ++j) mean[j] += u[j];
        }
        for (double& v : mean) v /= static_cast<double>(workers);
        const double r = matching_rate(from_words(agg_words, dim), DenseVector(std::move(mean)));
        *rate = r;
        *matches = static_cast<std::uint64_t>(std::llround(r * static_cast<double>(dim)));
    });
}

// ---------------------------------------------------------------------------
// SSDM baselines (ssdm.hpp:29-56, allreduce.hpp:198-339).
// ---------------------------------------------------------------------------
// ssdm_compress of v with RngStream(seed, ssdm, w, t, s).
int ref_ssdm_compress(const double* v, std::size_t len, std::uint64_t seed, std::uint64_t w,
                      std::uint64_t t, std::uint64_t s, std::uint64_t* bits, double* norm) {
    return guarded([&] {
        RngStream rng(seed, RngPurpose::ssdm, w, t, s);
        SsdmPacket p = ssdm_compress(DenseVector(std::vector<double>(v, v + len)), rng);
        to_words(p.bits, bits);
        *norm = p.norm;
    });
}

// cascading_allreduce (mode 0) / sum_ssdm_allreduce (mode 1).  vectors:
// [M][D]; out: the consensus estimate (D); max_abs_per_step: [steps] (mode 1).
int ref_ssdm_allreduce(int mode, int topology, std::uint32_t a, std::uint32_t b, std::size_t dim,
                       const double* vectors, std::uint64_t seed, std::uint64_t round,
                       double* out, std::uint64_t* bits_per_worker, std::uint64_t* reduce_bits,
                       std::uint64_t* gather_bits, std::int64_t* max_abs_per_step) {
    return guarded([&] {
        const Schedule sched = make_schedule(topology, a, b);
        std::vector<DenseVector> in;
        for (std::uint32_t w = 0; w < sched.workers; ++w)
            in.emplace_back(std::vector<double>(vectors + w * dim, vectors + (w + 1) * dim));
        std::vector<DenseVector> per_worker;
        BitsAccount bits(sched.workers);
        if (mode == 0) {
            CascadingAllreduceResult r = cascading_allreduce(in, sched, RoundContext{seed, round});
            per_worker = std::move(r.per_worker);
            bits = r.bits;
        } else {
            SumSsdmAllreduceResult r = sum_ssdm_allreduce(in, sched, RoundContext{seed, round});
            per_worker = std::move(r.per_worker);
            bits = r.bits;
            for (std::size_t k = 0; k < r.max_abs_per_step.size(); ++k)
                max_abs_per_step[k] = r.max_abs_per_step[k];
        }
        const DenseVector& est = consensus(per_worker);
        std::memcpy(out, est.values().data(), dim * sizeof(double));
        for (std::uint32_t w = 0; w < sched.workers; ++w) bits_per_worker[w] = bits.per_worker[w];
        *reduce_bits = bits.reduce_bits;
        *gather_bits = bits.gather_bits;
    });
}

// ---------------------------------------------------------------------------
// CPU-baseline harness: inputs are built once (not timed); each call times
// exactly one marsit_round (sign round, K = never) with steady_clock and
// carries the compensation like trainer.hpp:252 does.
// ---------------------------------------------------------------------------
struct RefBench {
    Schedule sched;
    std::vector<DenseVector> grads;
    std::vector<CompensationState> comp;
    std::uint64_t seed = 0;
    std::size_t dim = 0;
};

void* ref_bench_create(int topology, std::uint32_t a, std::uint32_t b, std::size_t dim,
                       std::uint64_t seed) {
    auto* rb = new RefBench;
    rb->sched = make_schedule(topology, a, b);
    rb->seed = seed;
    rb->dim = dim;
    for (std::uint32_t w = 0; w < rb->sched.workers; ++w) {
        RngStream rng(seed, RngPurpose::trial, w, 1, 0);
        std::vector<double> v(dim);
        for (double& x : v)
            x = static_cast<double>(static_cast<std::int64_t>(rng.next_u64() >> 51) - 4096) *
                0x1.0p-20;
        rb->grads.emplace_back(std::move(v));
        rb->comp.push_back(CompensationState{DenseVector::zeros(dim)});
    }
    return rb;
}

// Returns the wall time of one marsit_round in milliseconds (or a negative status).
double ref_bench_round(void* h, std::uint64_t t) {
    auto* rb = static_cast<RefBench*>(h);
    SyncConfig cfg;
    cfg.eta_s = 0x1.0p-10;
    double ms = 0.0;
    int rc = guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        MarsitRoundResult res = marsit_round(t, cfg, rb->grads, rb->comp, rb->sched, rb->seed);
        const auto t1 = std::chrono::steady_clock::now();
        ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        rb->comp = std::move(res.compensation);
    });
    return rc ? -static_cast<double>(rc) : ms;
}

void ref_bench_destroy(void* h) { delete static_cast<RefBench*>(h); }

} // extern "C"
