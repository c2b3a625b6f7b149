// driver.cu — multi-step sync driver (include/marsit_b200.h, marsit_driver_*).
//
// The per-round synchronisation part of the reference trainer
// (trainer.hpp:184-307) around marsit_round, on the device: compensation
// carried in place across rounds (trainer.hpp:252), dense cadence K
// (sync.hpp:78), identical replica update x -= g_t fused into the decode
// (trainer.hpp:285-288), cumulative bits (trainer.hpp:278-279), buckets for
// very large models, and checkpoint / resume of that state.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "internal.hpp"

using namespace marsit_b200;

struct marsit_driver {
    struct Bucket {
        uint64_t off = 0, len = 0;
        marsit_ctx* ctx = nullptr;
    };
    std::vector<Bucket> buckets;
    uint64_t D = 0;
    marsit_dtype dtype = MARSIT_F32;
    size_t esize = 4;
    int device = 0;
    uint32_t M = 0, ml = 0, nranks = 1, rank = 0;
    uint64_t period = 0, seed = 0, t = 0, cum_bits = 0;
    double eta = 0.0;
    std::vector<void*> comp;  // [local worker] D elements, device
    void* scratch = nullptr;  // D elements: g_t of dense rounds when the caller wants none

    ~marsit_driver() {
        if (device >= 0) cudaSetDevice(device);
        for (auto& b : buckets) marsit_ctx_destroy(b.ctx);
        for (void* p : comp)
            if (p) cudaFree(p);
        if (scratch) cudaFree(scratch);
    }
};

namespace {

uint64_t mix64(uint64_t z) {  // rng.hpp:66-70
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

uint64_t bucket_seed(uint64_t seed, uint64_t b, size_t n_buckets) {
    return n_buckets == 1 ? seed : mix64(seed ^ ((b + 1) * 0x9e3779b97f4a7c15ull));
}

constexpr char kStateMagic[16] = {'m', 'a', 'r', 's', 'i', 't', '-', 'b', '2',
                                  '0', '0', '-', 's', 'y', 'n', 'c'};
constexpr uint32_t kStateVersion = 1;

struct StateHeader {
    char magic[16];
    uint32_t version, dtype;
    uint64_t dim;
    uint32_t workers, nranks, rank, local_workers;
    uint64_t next_round, cum_bits, period, seed, bucket_elems;
    double eta_s;
};

}  // namespace

extern "C" {

marsit_status marsit_driver_create(const marsit_driver_desc* desc, marsit_driver** out) {
    if (!desc || !out) return fail(MARSIT_EPARAM, "null argument");
    *out = nullptr;
    if (!desc->schedule) return fail(MARSIT_EPARAM, "schedule is null");
    if (desc->dim == 0) return fail(MARSIT_EPARAM, "DenseVector: dimension must be >= 1");
    if (!(desc->eta_s > 0.0)) return fail(MARSIT_EPARAM, "SyncConfig: eta_s must be > 0");
    if (!have_device())
        return fail(MARSIT_ECUDA, "no CUDA device available (this library has no CPU path)");
    auto drv = std::make_unique<marsit_driver>();
    drv->D = desc->dim;
    drv->dtype = desc->dtype;
    drv->esize = desc->dtype == MARSIT_F64 ? 8 : 4;
    drv->device = desc->device;
    drv->period = desc->period;
    drv->eta = desc->eta_s;
    drv->seed = desc->global_seed;
    drv->t = desc->first_round;
    drv->nranks = desc->nranks ? desc->nranks : 1;
    drv->rank = desc->rank;
    CUDA_TRY(cudaSetDevice(desc->device));
    const uint64_t be = desc->bucket_elems ? desc->bucket_elems : desc->dim;
    for (uint64_t off = 0; off < desc->dim; off += be) {
        marsit_driver::Bucket b;
        b.off = off;
        b.len = std::min<uint64_t>(be, desc->dim - off);
        marsit_ctx_desc cd{};
        cd.dim = b.len;
        cd.schedule = desc->schedule;
        cd.dtype = desc->dtype;
        cd.device = desc->device;
        cd.nranks = desc->nranks;
        cd.rank = desc->rank;
        cd.nccl_id = desc->nccl_id;
        cd.transport = desc->transport == MARSIT_TRANSPORT_NCCL ? MARSIT_TRANSPORT_NCCL
                                                                : MARSIT_TRANSPORT_P2P;
        // one NCCL communicator for all buckets (a unique id initialises one comm)
        marsit_status s = ctx_create_internal(
            &cd, drv->buckets.empty() ? nullptr : drv->buckets[0].ctx->comm, &b.ctx);
        if (s) return s;
        drv->buckets.push_back(b);
    }
    uint32_t first = 0;
    marsit_ctx_local_workers(drv->buckets[0].ctx, &first, &drv->ml);
    drv->M = drv->buckets[0].ctx->M;
    drv->comp.assign(drv->ml, nullptr);
    for (auto& p : drv->comp) {
        CUDA_TRY(cudaMalloc(&p, drv->esize * drv->D));
        CUDA_TRY(cudaMemset(p, 0, drv->esize * drv->D));
    }
    CUDA_TRY(cudaMalloc(&drv->scratch, drv->esize * drv->D));
    *out = drv.release();
    return MARSIT_OK;
}

void marsit_driver_destroy(marsit_driver* drv) { delete drv; }

marsit_status marsit_driver_step(marsit_driver* drv, const void* const* d_grads,
                                 void* const* d_params, void* d_update, int* full_precision,
                                 void* stream) {
    if (!drv) return fail(MARSIT_EPARAM, "driver is null");
    if (!d_grads) return fail(MARSIT_EPARAM, "grads is null");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaSetDevice(drv->device));
    const bool dense = drv->period != 0 && drv->t % drv->period == 0;  // sync.hpp:78
    const size_t nb = drv->buckets.size();
    std::vector<const void*> g(drv->ml);
    std::vector<void*> c(drv->ml), x(drv->ml);
    for (size_t bi = 0; bi < nb; ++bi) {
        const auto& b = drv->buckets[bi];
        const size_t boff = b.off * drv->esize;
        for (uint32_t w = 0; w < drv->ml; ++w) {
            g[w] = static_cast<const char*>(d_grads[w]) + boff;
            c[w] = static_cast<char*>(drv->comp[w]) + boff;
            x[w] = d_params ? static_cast<char*>(d_params[w]) + boff : nullptr;
        }
        void* upd = d_update ? static_cast<char*>(d_update) + boff : nullptr;
        marsit_status s;
        if (dense) {
            void* mean = upd ? upd : static_cast<char*>(drv->scratch) + boff;
            s = dense_round_any(b.ctx, drv->t, g.data(), (const void* const*)c.data(), c.data(),
                                d_params ? x.data() : nullptr, mean, st);
        } else {
            s = sign_round_impl(b.ctx, drv->t, drv->eta, bucket_seed(drv->seed, bi, nb), g.data(),
                                (const void* const*)c.data(), c.data(),
                                d_params ? x.data() : nullptr, nullptr, upd, st);
        }
        if (s) return s;
        drv->cum_bits += round_bits_total(b.ctx, dense);
    }
    if (full_precision) *full_precision = dense ? 1 : 0;
    ++drv->t;
    return MARSIT_OK;
}

marsit_status marsit_driver_compensation(marsit_driver* drv, uint32_t local_worker, void** d_comp) {
    if (!drv || !d_comp) return fail(MARSIT_EPARAM, "null argument");
    if (local_worker >= drv->ml) return fail(MARSIT_EPARAM, "local worker out of range");
    *d_comp = drv->comp[local_worker];
    return MARSIT_OK;
}

marsit_status marsit_driver_state(const marsit_driver* drv, uint64_t* next_round,
                                  uint64_t* cum_bits, uint32_t* n_buckets) {
    if (!drv) return fail(MARSIT_EPARAM, "driver is null");
    if (next_round) *next_round = drv->t;
    if (cum_bits) *cum_bits = drv->cum_bits;
    if (n_buckets) *n_buckets = uint32_t(drv->buckets.size());
    return MARSIT_OK;
}

marsit_status marsit_driver_p2p_buffers(const marsit_driver* drv, uint32_t bucket,
                                        marsit_p2p_buffers* out) {
    if (!drv) return fail(MARSIT_EPARAM, "driver is null");
    if (bucket >= drv->buckets.size()) return fail(MARSIT_EPARAM, "bucket out of range");
    return marsit_ctx_p2p_buffers(drv->buckets[bucket].ctx, out);
}

marsit_status marsit_driver_set_peers(marsit_driver* drv, uint32_t bucket,
                                      const marsit_p2p_buffers* peers, uint32_t nranks) {
    if (!drv) return fail(MARSIT_EPARAM, "driver is null");
    if (bucket >= drv->buckets.size()) return fail(MARSIT_EPARAM, "bucket out of range");
    return marsit_ctx_set_peers(drv->buckets[bucket].ctx, peers, nranks);
}

marsit_status marsit_driver_set_wait_timeout(marsit_driver* drv, uint64_t timeout_ms) {
    if (!drv) return fail(MARSIT_EPARAM, "driver is null");
    marsit_status s;
    for (auto& b : drv->buckets)
        if ((s = marsit_ctx_set_wait_timeout(b.ctx, timeout_ms))) return s;
    return MARSIT_OK;
}

marsit_status marsit_driver_set_consensus(marsit_driver* drv, int enable) {
    if (!drv) return fail(MARSIT_EPARAM, "driver is null");
    marsit_status s;
    for (auto& b : drv->buckets)
        if ((s = marsit_ctx_set_consensus(b.ctx, enable))) return s;
    return MARSIT_OK;
}

marsit_status marsit_driver_set_metrics(marsit_driver* drv, int enable) {
    if (!drv) return fail(MARSIT_EPARAM, "driver is null");
    marsit_status s;
    for (auto& b : drv->buckets)
        if ((s = marsit_ctx_set_metrics(b.ctx, enable))) return s;
    return MARSIT_OK;
}

marsit_status marsit_driver_metrics(marsit_driver* drv, marsit_round_metrics* out, void* stream) {
    if (!drv || !out) return fail(MARSIT_EPARAM, "null argument");
    *out = marsit_round_metrics{};
    out->has_matching = 1;
    marsit_status s;
    for (auto& b : drv->buckets) {
        marsit_round_metrics m{};
        if ((s = marsit_ctx_metrics(b.ctx, &m, stream))) return s;
        out->round = m.round;
        out->valid = m.valid;
        out->full_precision = m.full_precision;
        out->has_matching &= m.has_matching;
        out->rank_local |= m.rank_local;
        out->dim += m.dim;
        out->matches += m.matches;
        out->merges += m.merges;
        out->compared_bits += m.compared_bits;
        out->disagreements += m.disagreements;
        out->round_bits += m.round_bits;
    }
    if (!out->valid || out->full_precision) out->has_matching = 0;
    if (!out->has_matching) out->matches = 0;
    out->matching_rate = out->has_matching ? double(out->matches) / double(out->dim) : 0.0;
    out->disagreement_rate =
        out->compared_bits ? double(out->disagreements) / double(out->compared_bits) : 0.0;
    return MARSIT_OK;
}

marsit_status marsit_driver_save(marsit_driver* drv, const char* path, void* stream) {
    if (!drv || !path) return fail(MARSIT_EPARAM, "null argument");
    CUDA_TRY(cudaSetDevice(drv->device));
    CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    StateHeader h{};
    std::memcpy(h.magic, kStateMagic, sizeof(h.magic));
    h.version = kStateVersion;
    h.dtype = uint32_t(drv->dtype);
    h.dim = drv->D;
    h.workers = drv->M;
    h.nranks = drv->nranks;
    h.rank = drv->rank;
    h.local_workers = drv->ml;
    h.next_round = drv->t;
    h.cum_bits = drv->cum_bits;
    h.period = drv->period;
    h.seed = drv->seed;
    h.bucket_elems = drv->buckets.size() > 1 ? drv->buckets[0].len : 0;
    h.eta_s = drv->eta;
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) return fail(MARSIT_EPARAM, std::string("cannot open ") + path);
    f.write(reinterpret_cast<const char*>(&h), sizeof(h));
    std::vector<char> host(drv->esize * drv->D);
    for (uint32_t w = 0; w < drv->ml; ++w) {
        CUDA_TRY(cudaMemcpy(host.data(), drv->comp[w], host.size(), cudaMemcpyDeviceToHost));
        f.write(host.data(), std::streamsize(host.size()));
    }
    if (!f) return fail(MARSIT_EPARAM, std::string("write failed: ") + path);
    return MARSIT_OK;
}

marsit_status marsit_driver_load(marsit_driver* drv, const char* path, void* stream) {
    if (!drv || !path) return fail(MARSIT_EPARAM, "null argument");
    CUDA_TRY(cudaSetDevice(drv->device));
    CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    std::ifstream f(path, std::ios::binary);
    if (!f) return fail(MARSIT_EPARAM, std::string("cannot open ") + path);
    f.seekg(0, std::ios::end);
    const std::streamoff size = f.tellg();
    f.seekg(0, std::ios::beg);
    if (uint64_t(size) != sizeof(StateHeader) + uint64_t(drv->ml) * drv->D * drv->esize)
        return fail(MARSIT_EPARAM, "sync state file size does not match this driver");
    StateHeader h{};
    f.read(reinterpret_cast<char*>(&h), sizeof(h));
    if (!f || std::memcmp(h.magic, kStateMagic, sizeof(h.magic)) != 0)
        return fail(MARSIT_EPARAM, "not a marsit-b200 sync state file");
    if (h.version != kStateVersion) return fail(MARSIT_EUNSUPPORTED, "unsupported state version");
    if (h.dim != drv->D || h.dtype != uint32_t(drv->dtype) || h.workers != drv->M ||
        h.nranks != drv->nranks || h.rank != drv->rank || h.local_workers != drv->ml)
        return fail(MARSIT_EPARAM, "sync state does not match this driver (D, dtype, workers, ranks)");
    if (h.period != drv->period || h.seed != drv->seed || h.eta_s != drv->eta ||
        h.bucket_elems != (drv->buckets.size() > 1 ? drv->buckets[0].len : 0))
        return fail(MARSIT_EPARAM, "sync state was written with a different SyncConfig / seed / buckets");
    std::vector<char> host(drv->esize * drv->D);
    for (uint32_t w = 0; w < drv->ml; ++w) {
        f.read(host.data(), std::streamsize(host.size()));
        if (!f) return fail(MARSIT_EPARAM, "truncated sync state file");
        CUDA_TRY(cudaMemcpy(drv->comp[w], host.data(), host.size(), cudaMemcpyHostToDevice));
    }
    drv->t = h.next_round;
    drv->cum_bits = h.cum_bits;
    return MARSIT_OK;
}

// checkpoint.hpp:18-91 layout
marsit_status marsit_write_params_checkpoint(const char* path, const void* d_params, uint64_t dim,
                                             marsit_dtype dtype, void* stream) {
    if (!path || !d_params || dim == 0) return fail(MARSIT_EPARAM, "bad argument");
    CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    std::vector<double> v(dim);
    if (dtype == MARSIT_F64) {
        CUDA_TRY(cudaMemcpy(v.data(), d_params, dim * 8, cudaMemcpyDeviceToHost));
    } else {
        std::vector<float> f(dim);
        CUDA_TRY(cudaMemcpy(f.data(), d_params, dim * 4, cudaMemcpyDeviceToHost));
        for (uint64_t j = 0; j < dim; ++j) v[j] = f[j];
    }
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) return fail(MARSIT_EPARAM, std::string("cannot open ") + path);
    const char magic[12] = {'m', 'a', 'r', 's', 'i', 't', '-', 'c', 'k', 'p', 't', '\0'};
    const uint32_t version = 1;
    f.write(magic, 12);
    f.write(reinterpret_cast<const char*>(&version), 4);  // little-endian hosts only
    f.write(reinterpret_cast<const char*>(&dim), 8);
    f.write(reinterpret_cast<const char*>(v.data()), std::streamsize(dim * 8));
    if (!f) return fail(MARSIT_EPARAM, std::string("write failed: ") + path);
    return MARSIT_OK;
}

marsit_status marsit_read_params_checkpoint(const char* path, void* d_params, uint64_t dim,
                                            marsit_dtype dtype, void* stream) {
    if (!path || !d_params) return fail(MARSIT_EPARAM, "bad argument");
    std::ifstream f(path, std::ios::binary);
    if (!f) return fail(MARSIT_EPARAM, std::string("cannot open ") + path);
    // read_checkpoint (checkpoint.hpp:65-91): explicit little-endian header
    // fields and an exact file size of 24 + 8 * dim ("size mismatch")
    f.seekg(0, std::ios::end);
    const std::streamoff size = f.tellg();
    f.seekg(0, std::ios::beg);
    unsigned char hdr[24];
    if (size < 24 || !f.read(reinterpret_cast<char*>(hdr), 24))
        return fail(MARSIT_EPARAM, "read_checkpoint: truncated header");
    auto le = [&](int off, int bytes) {
        uint64_t v = 0;
        for (int i = 0; i < bytes; ++i) v |= uint64_t(hdr[off + i]) << (8 * i);
        return v;
    };
    const char want[12] = {'m', 'a', 'r', 's', 'i', 't', '-', 'c', 'k', 'p', 't', '\0'};
    if (std::memcmp(hdr, want, 12) != 0) return fail(MARSIT_EPARAM, "read_checkpoint: bad magic");
    if (le(12, 4) != 1) return fail(MARSIT_EUNSUPPORTED, "read_checkpoint: unsupported version");
    const uint64_t n = le(16, 8);
    if (uint64_t(size) != 24 + n * 8) return fail(MARSIT_EPARAM, "read_checkpoint: size mismatch");
    if (n != dim) return fail(MARSIT_EPARAM, "checkpoint dimension mismatch");
    std::vector<double> v(dim);
    f.read(reinterpret_cast<char*>(v.data()), std::streamsize(dim * 8));  // LE hosts (x86-64, aarch64)
    if (!f) return fail(MARSIT_EPARAM, "truncated checkpoint");
    for (double x : v)
        if (!std::isfinite(x)) return fail(MARSIT_ENONFINITE, "DenseVector: non-finite entry");
    CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    if (dtype == MARSIT_F64) {
        CUDA_TRY(cudaMemcpy(d_params, v.data(), dim * 8, cudaMemcpyHostToDevice));
    } else {
        std::vector<float> h(dim);
        for (uint64_t j = 0; j < dim; ++j) h[j] = float(v[j]);
        CUDA_TRY(cudaMemcpy(d_params, h.data(), dim * 4, cudaMemcpyHostToDevice));
    }
    return MARSIT_OK;
}

}  // extern "C"
