// dropin_parity.cpp — runs the REFERENCE's marsit::marsit_round /
// marsit::allreduce_sign and the drop-in marsit::gpu:: versions (B200 path via
// the C-ABI) on identical inputs in one process and requires bit-identical
// results (compensation, global update, aggregate bits, bit accounting).
//
// Built here by `make -C tools dropin` against the read-only reference headers
// (test infrastructure: the binary carries the reference code, it does not
// read /root/reference at run time).  Exit status 0 = all cases identical.
#include <marsit/allreduce.hpp>
#include <marsit/rng.hpp>
#include <marsit/sync.hpp>

#include <marsit_b200/drop_in.hpp>

#include <cmath>
#include <chrono>
#include <cstdio>
#include <string>
#include <cstring>
#include <thread>
#include <vector>

using namespace marsit;

static int failures = 0;

static void expect(bool ok, const char* what, const char* tag) {
    if (!ok) {
        std::printf("MISMATCH %s: %s\n", tag, what);
        ++failures;
    }
}

static bool same(const DenseVector& a, const DenseVector& b) {
    return a.size() == b.size() &&
           std::memcmp(a.values().data(), b.values().data(), a.size() * sizeof(double)) == 0;
}

static std::vector<DenseVector> inputs(uint32_t W, size_t D, uint64_t seed, uint64_t t, int kind) {
    std::vector<DenseVector> out;
    for (uint32_t w = 0; w < W; ++w) {
        RngStream rng(seed, RngPurpose::trial, w, t, 0);
        std::vector<double> v(D);
        for (size_t j = 0; j < D; ++j) {
            if (kind == 0)
                v[j] = double(int64_t(rng.next_u64() >> 51) - 4096) * 0x1.0p-20;  // dyadic
            else
                v[j] = rng.next_gaussian() * 1e-3;                               // arbitrary doubles
            if (kind == 2 && j % 7 == 0) v[j] = (j % 14 == 0) ? 0.0 : -0.0;     // zeros
        }
        out.emplace_back(std::move(v));
    }
    return out;
}

static void run_case(const char* tag, const Schedule& sched, size_t D, std::optional<uint64_t> K,
                     int kind, int rounds) {
    SyncConfig cfg{K, 0x1.0p-10};
    std::vector<CompensationState> comp_ref(sched.workers, CompensationState{DenseVector::zeros(D)});
    std::vector<CompensationState> comp_gpu = comp_ref;
    for (int r = 0; r < rounds; ++r) {
        const uint64_t t = K ? uint64_t(r) : uint64_t(r + 1);
        auto g = inputs(sched.workers, D, 77, t, kind);
        MarsitRoundResult a = marsit::marsit_round(t, cfg, g, comp_ref, sched, 2026);
        MarsitRoundResult b = marsit::gpu::marsit_round(t, cfg, g, comp_gpu, sched, 2026);
        expect(a.full_precision == b.full_precision, "full_precision", tag);
        expect(same(a.global_update, b.global_update), "global_update", tag);
        for (uint32_t w = 0; w < sched.workers; ++w)
            expect(same(a.compensation[w].c, b.compensation[w].c), "compensation", tag);
        expect(a.aggregate_bits.has_value() == b.aggregate_bits.has_value(), "aggregate presence", tag);
        if (a.aggregate_bits && b.aggregate_bits)
            expect(*a.aggregate_bits == *b.aggregate_bits, "aggregate_bits", tag);
        expect(a.bits.per_worker == b.bits.per_worker && a.bits.total == b.bits.total &&
                   a.bits.reduce_bits == b.bits.reduce_bits && a.bits.gather_bits == b.bits.gather_bits,
               "BitsAccount", tag);
        comp_ref = a.compensation;
        comp_gpu = b.compensation;
    }
    std::printf("case %-28s D=%zu rounds=%d %s\n", tag, D, rounds, failures ? "" : "ok");
}

static void run_allreduce(const char* tag, const Schedule& sched, size_t L) {
    std::vector<std::vector<PackedSignVector>> signs(sched.workers);
    for (uint32_t w = 0; w < sched.workers; ++w) {
        RngStream rng(9, RngPurpose::trial, w, 3, 1);
        for (uint32_t s = 0; s < sched.segments; ++s) {
            PackedSignVector v = PackedSignVector::zeros(L);
            for (size_t j = 0; j < L; ++j)
                if (rng.next_u64() & 1u) v.set_bit(j, true);
            signs[w].push_back(std::move(v));
        }
    }
    RoundContext rc{31, 4};
    SignAllreduceResult a = marsit::allreduce_sign(signs, sched, rc);
    SignAllreduceResult b = marsit::gpu::allreduce_sign(signs, sched, rc);
    for (uint32_t w = 0; w < sched.workers; ++w)
        for (uint32_t s = 0; s < sched.segments; ++s)
            expect(a.per_worker[w][s] == b.per_worker[w][s], "AggregateSign", tag);
    expect(a.bits.total == b.bits.total && a.bits.per_worker == b.bits.per_worker, "bits", tag);
    std::printf("allreduce %-23s L=%zu %s\n", tag, L, failures ? "" : "ok");
}

static void run_dense(const char* tag, const Schedule& sched, size_t D, int kind) {
    auto v = inputs(sched.workers, D, 5, 1, kind);
    DenseAllreduceResult a = marsit::allreduce_dense(v, sched);
    DenseAllreduceResult b = marsit::gpu::allreduce_dense(v, sched);
    for (uint32_t w = 0; w < sched.workers; ++w) expect(same(a.per_worker[w], b.per_worker[w]), "mean", tag);
    expect(a.bits.per_worker == b.bits.per_worker && a.bits.total == b.bits.total, "dense bits", tag);
    std::printf("dense %-27s D=%zu %s\n", tag, D, failures ? "" : "ok");
}

// SSDM: bits exact; values exact for dyadic inputs in the sum variant (every
// norm is a first compression of exact data), else within 1e-9 relative.
static void run_ssdm(const char* tag, const Schedule& sched, size_t D, int kind) {
    auto v = inputs(sched.workers, D, 9, 2, kind);
    RoundContext rc{2026, 3};
    for (int mode = 0; mode < 2; ++mode) {
        std::vector<DenseVector> ea, eb;
        BitsAccount ba(sched.workers), bb(sched.workers);
        if (mode == 0) {
            auto a = marsit::cascading_allreduce(v, sched, rc);
            auto b = marsit::gpu::cascading_allreduce(v, sched, rc);
            ea = a.per_worker; eb = b.per_worker; ba = a.bits; bb = b.bits;
        } else {
            auto a = marsit::sum_ssdm_allreduce(v, sched, rc);
            auto b = marsit::gpu::sum_ssdm_allreduce(v, sched, rc);
            ea = a.per_worker; eb = b.per_worker; ba = a.bits; bb = b.bits;
            expect(a.max_abs_per_step == b.max_abs_per_step, "max_abs_per_step", tag);
        }
        bool ok = true;
        for (size_t j = 0; j < D; ++j) {
            const double x = ea[0][j], y = eb[0][j];
            if (mode == 1 && kind == 0) ok &= std::memcmp(&x, &y, 8) == 0;
            else ok &= std::signbit(x) == std::signbit(y) && std::fabs(x - y) <= 1e-9 * std::fabs(x);
        }
        expect(ok, mode ? "sum-ssdm estimate" : "cascading estimate", tag);
        expect(ba.per_worker == bb.per_worker && ba.reduce_bits == bb.reduce_bits &&
                   ba.gather_bits == bb.gather_bits, "ssdm bits", tag);
    }
    std::printf("ssdm %-28s D=%zu %s\n", tag, D, failures ? "" : "ok");
}

// Concurrency: several host threads call marsit::gpu::marsit_round with the
// same (D, schedule) at once (the reference's round is a pure function, and
// this file's own CPU baseline calls it from many threads); every result
// must equal the reference's serial result for that thread's inputs.
static void run_concurrent(const char* tag, uint32_t n_threads, size_t D) {
    const Schedule sched = build_ring_schedule(4);
    const SyncConfig cfg{std::nullopt, 0x1.0p-10};
    std::vector<std::vector<DenseVector>> g(n_threads);
    std::vector<MarsitRoundResult> want, got(n_threads, MarsitRoundResult{DenseVector::zeros(1), {}, BitsAccount(4), false, std::nullopt});
    std::vector<CompensationState> c0(4, CompensationState{DenseVector::zeros(D)});
    for (uint32_t i = 0; i < n_threads; ++i) {
        g[i] = inputs(4, D, 100 + i, 1, 1);
        want.push_back(marsit::marsit_round(1, cfg, g[i], c0, sched, 2026 + i));
    }
    std::vector<std::thread> th;
    std::vector<int> err(n_threads, 0);
    for (uint32_t i = 0; i < n_threads; ++i)
        th.emplace_back([&, i] {
            try {
                for (int rep = 0; rep < 3; ++rep)
                    got[i] = marsit::gpu::marsit_round(1, cfg, g[i], c0, sched, 2026 + i);
            } catch (...) {
                err[i] = 1;
            }
        });
    for (auto& t : th) t.join();
    for (uint32_t i = 0; i < n_threads; ++i) {
        expect(!err[i], "exception in a concurrent call", tag);
        if (err[i]) continue;
        expect(same(want[i].global_update, got[i].global_update), "concurrent global_update", tag);
        for (uint32_t w = 0; w < 4; ++w)
            expect(same(want[i].compensation[w].c, got[i].compensation[w].c), "concurrent compensation", tag);
        expect(want[i].aggregate_bits == got[i].aggregate_bits, "concurrent aggregate_bits", tag);
    }
    std::printf("concurrent %-22s threads=%u D=%zu %s\n", tag, n_threads, D, failures ? "" : "ok");
}

// --time D: wall time of one marsit_round through the reference's own API
// (host DenseVectors in, MarsitRoundResult out) — the reference's CPU round vs
// marsit::gpu::marsit_round (staging, device round, read-back) — ring 8, fp64
// Gaussian gradients, compensation carried over 3 timed rounds.
static int time_rounds(size_t D) {
    const Schedule sched = build_ring_schedule(8);
    const auto g = inputs(8, D, 7, 1, 1);
    std::vector<CompensationState> c_ref(8, CompensationState{DenseVector::zeros(D)}), c_gpu = c_ref;
    const SyncConfig cfg{std::nullopt, 0x1.0p-10};
    auto wall = [](auto&& fn) {
        const auto t0 = std::chrono::steady_clock::now();
        fn();
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    marsit::gpu::marsit_round(1, cfg, g, c_gpu, sched, 5);  // context + scratch warm-up
    c_gpu = c_ref;
    for (uint64_t t = 1; t <= 3; ++t) {
        std::optional<MarsitRoundResult> rr, rg;
        const double ms_ref = wall([&] { rr.emplace(marsit_round(t, cfg, g, c_ref, sched, 5)); });
        const double ms_gpu =
            wall([&] { rg.emplace(marsit::gpu::marsit_round(t, cfg, g, c_gpu, sched, 5)); });
        const bool same_bits = rr->aggregate_bits == rg->aggregate_bits;
        c_ref = rr->compensation;
        c_gpu = rg->compensation;
        std::printf("D=%zu round %llu: reference %.1f ms, marsit::gpu %.1f ms (%.1fx), bits %s\n", D,
                    (unsigned long long)t, ms_ref, ms_gpu, ms_ref / ms_gpu,
                    same_bits ? "identical" : "DIFFER");
        if (!same_bits) return 1;
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc == 3 && std::string(argv[1]) == "--time") return time_rounds(std::stoull(argv[2]));
    try {
        run_dense("ring4 gaussian", build_ring_schedule(4), 1001, 1);
        run_dense("torus2x4 zeros", build_torus_schedule(2, 4), 777, 2);
        run_dense("ring8 dyadic", build_ring_schedule(8), 8192, 0);
        run_ssdm("ring4 dyadic", build_ring_schedule(4), 4096, 0);
        run_ssdm("ring5 gaussian", build_ring_schedule(5), 333, 1);
        {  // torus: unsupported_error like the reference
            bool threw = false;
            try {
                marsit::gpu::cascading_allreduce(inputs(4, 10, 1, 1, 1), build_torus_schedule(2, 2),
                                                 RoundContext{1, 1});
            } catch (const unsupported_error&) {
                threw = true;
            }
            expect(threw, "unsupported_error for torus SSDM", "errors");
        }
        run_case("ring5 dyadic", build_ring_schedule(5), 37, std::nullopt, 0, 4);
        run_case("ring4 C1 dyadic", build_ring_schedule(4), 1000000, std::nullopt, 0, 2);
        run_case("ring8 gaussian", build_ring_schedule(8), 100003, std::nullopt, 1, 3);
        run_case("torus2x4 gaussian", build_torus_schedule(2, 4), 60201, std::nullopt, 1, 3);
        run_case("torus3x3 zeros", build_torus_schedule(3, 3), 5000, std::nullopt, 2, 2);
        run_case("ring4 dense K=3", build_ring_schedule(4), 777, uint64_t{3}, 1, 5);
        run_case("torus2x3 dense K=2", build_torus_schedule(2, 3), 61, uint64_t{2}, 1, 4);
        run_case("ring4 D<M", build_ring_schedule(4), 3, std::nullopt, 1, 2);
        run_allreduce("ring6", build_ring_schedule(6), 97);
        run_allreduce("torus2x3", build_torus_schedule(2, 3), 1000);
        run_allreduce("torus4x2", build_torus_schedule(4, 2), 65537);
        run_concurrent("ring4 same D", 6, 20011);
        {  // a reduce-only table ends without consensus: the reference returns
           // each worker's own state; the device path reports unsupported_error
            Schedule red = build_ring_schedule(4);
            red.steps.resize(3);
            bool threw = false;
            std::vector<std::vector<PackedSignVector>> signs(4, std::vector<PackedSignVector>(4, PackedSignVector::zeros(10)));
            try {
                marsit::gpu::allreduce_sign(signs, red, RoundContext{1, 1});
            } catch (const unsupported_error&) {
                threw = true;
            }
            expect(threw, "unsupported_error for a non-consensus schedule", "errors");
        }
        // error mapping: non-finite u (overflow) raises non_finite_error like the reference
        bool threw = false;
        try {
            std::vector<DenseVector> big(2, DenseVector(std::vector<double>(4, 1.5e308)));
            std::vector<CompensationState> c(2, CompensationState{DenseVector(std::vector<double>(4, 1.5e308))});
            marsit::gpu::marsit_round(1, SyncConfig{std::nullopt, 0.1}, big, c, build_ring_schedule(2), 1);
        } catch (const non_finite_error&) {
            threw = true;
        }
        expect(threw, "non_finite_error on overflow", "errors");
        threw = false;
        try {
            std::vector<DenseVector> g(2, DenseVector(std::vector<double>(4, 1.0)));
            std::vector<CompensationState> c(2, CompensationState{DenseVector::zeros(4)});
            marsit::gpu::marsit_round(1, SyncConfig{std::nullopt, 0.0}, g, c, build_ring_schedule(2), 1);
        } catch (const parameter_error&) {
            threw = true;
        }
        expect(threw, "parameter_error on eta_s <= 0", "errors");
    } catch (const std::exception& e) {
        std::printf("EXCEPTION %s\n", e.what());
        return 2;
    }
    std::printf("%s\n", failures ? "DROP-IN PARITY FAILED" : "DROP-IN PARITY OK (bit-identical)");
    return failures ? 1 : 0;
}
