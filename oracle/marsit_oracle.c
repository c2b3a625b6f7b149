/*
 * marsit_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A deliberately literal, scalar restatement of the reference's sign-round
 * path.  Every function cites the reference lines it follows; paths are
 * relative to /root/reference/proj/include/marsit/.  See marsit_oracle.h.
 */
#include "marsit_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9e3779b97f4a7c15ull

/* rng.hpp:66-70 */
uint64_t orc_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* rng.hpp:30-38 */
uint64_t orc_stream_key(uint64_t seed, uint64_t purpose, uint64_t worker, uint64_t round,
                        uint64_t segment) {
    uint64_t h = orc_mix(seed ^ 0x6a09e667f3bcc909ull);
    h = orc_mix(h ^ (purpose * GAMMA));
    h = orc_mix(h ^ ((worker + 1) * GAMMA));
    h = orc_mix(h ^ ((round + 1) * GAMMA));
    h = orc_mix(h ^ ((segment + 1) * GAMMA));
    return h;
}

/* rng.hpp:40-43: state += gamma; return mix(state).  Draw n is therefore
 * mix(key + (n+1)*gamma). */
uint64_t orc_draw(uint64_t key, uint64_t n) { return orc_mix(key + (n + 1) * GAMMA); }

static uint32_t modu(int64_t x, uint32_t m) { return (uint32_t)(((x % m) + m) % m); }

/* schedule.hpp:38-54 */
int orc_validate_schedule(uint32_t workers, uint32_t segments, uint32_t steps,
                          const uint32_t* send_to, const uint32_t* recv_from,
                          const uint32_t* segment) {
    for (uint32_t k = 0; k < steps; ++k) {
        const uint32_t* st = send_to + (size_t)k * workers;
        const uint32_t* rf = recv_from + (size_t)k * workers;
        const uint32_t* sg = segment + (size_t)k * workers;
        for (uint32_t w = 0; w < workers; ++w) {
            if (st[w] >= workers || rf[w] >= workers || sg[w] >= segments) return ORC_EPROTOCOL;
            if (rf[st[w]] != w) return ORC_EPROTOCOL;
        }
    }
    return ORC_OK;
}

/* schedule.hpp:61-94 */
int orc_ring_schedule(uint32_t m, uint8_t* phase, uint32_t* send_to, uint32_t* recv_from,
                      uint32_t* segment) {
    if (m < 2) return -ORC_EPARAM;
    uint32_t k_out = 0;
    for (int ph = 0; ph < 2; ++ph) {
        for (uint32_t k = 0; k + 1 < m; ++k, ++k_out) {
            phase[k_out] = (uint8_t)ph;
            for (uint32_t w = 0; w < m; ++w) {
                size_t i = (size_t)k_out * m + w;
                send_to[i] = modu((int64_t)w + 1, m);
                recv_from[i] = modu((int64_t)w - 1, m);
                segment[i] = ph == 0 ? modu((int64_t)w - (int64_t)k, m)
                                     : modu((int64_t)w + 1 - (int64_t)k, m);
            }
        }
    }
    return (int)k_out;
}

/* schedule.hpp:110-196 */
int orc_torus_schedule(uint32_t rows, uint32_t cols, uint8_t* phase, uint32_t* send_to,
                       uint32_t* recv_from, uint32_t* segment) {
    if (rows < 2 || cols < 2) return -ORC_EPARAM;
    const uint32_t W = rows * cols;
    uint32_t n = 0;
#define ID(r, c) ((r) * cols + (c))
#define PUT(r, c, to, from, seg)                     \
    do {                                             \
        size_t i_ = (size_t)n * W + ID(r, c);        \
        send_to[i_] = (to);                          \
        recv_from[i_] = (from);                      \
        segment[i_] = (seg);                         \
    } while (0)
    /* Stage 1 (127-143) */
    for (uint32_t k = 0; k + 1 < cols; ++k)
        for (uint32_t q = 0; q < rows; ++q, ++n) {
            phase[n] = ORC_PHASE_REDUCE;
            for (uint32_t r = 0; r < rows; ++r)
                for (uint32_t c = 0; c < cols; ++c) {
                    uint32_t super = modu((int64_t)c - k, cols);
                    PUT(r, c, ID(r, modu((int64_t)c + 1, cols)), ID(r, modu((int64_t)c - 1, cols)),
                        super * rows + q);
                }
        }
    /* Stage 2 (147-174) */
    for (uint32_t k = 0; k + 1 < rows; ++k, ++n) {
        phase[n] = ORC_PHASE_REDUCE;
        for (uint32_t r = 0; r < rows; ++r)
            for (uint32_t c = 0; c < cols; ++c) {
                uint32_t owned = modu((int64_t)c + 1, cols);
                PUT(r, c, ID(modu((int64_t)r + 1, rows), c), ID(modu((int64_t)r - 1, rows), c),
                    owned * rows + modu((int64_t)r - k, rows));
            }
    }
    for (uint32_t k = 0; k + 1 < rows; ++k, ++n) {
        phase[n] = ORC_PHASE_GATHER;
        for (uint32_t r = 0; r < rows; ++r)
            for (uint32_t c = 0; c < cols; ++c) {
                uint32_t owned = modu((int64_t)c + 1, cols);
                PUT(r, c, ID(modu((int64_t)r + 1, rows), c), ID(modu((int64_t)r - 1, rows), c),
                    owned * rows + modu((int64_t)r + 1 - k, rows));
            }
    }
    /* Stage 3 (177-192) */
    for (uint32_t k = 0; k + 1 < cols; ++k)
        for (uint32_t q = 0; q < rows; ++q, ++n) {
            phase[n] = ORC_PHASE_GATHER;
            for (uint32_t r = 0; r < rows; ++r)
                for (uint32_t c = 0; c < cols; ++c) {
                    uint32_t super = modu((int64_t)c + 1 - k, cols);
                    PUT(r, c, ID(r, modu((int64_t)c + 1, cols)), ID(r, modu((int64_t)c - 1, cols)),
                        super * rows + q);
                }
        }
#undef PUT
#undef ID
    return (int)n;
}

/* sign_vector.hpp:67-73: bit = (v >= 0.0); storage padding stays 0 (15-18). */
void orc_pack_signs(const double* v, size_t len, uint64_t* words) {
    memset(words, 0, ((len + 63) / 64) * sizeof(uint64_t));
    for (size_t i = 0; i < len; ++i)
        if (v[i] >= 0.0) words[i >> 6] |= (uint64_t)1 << (i & 63);
}

static int get_bit(const uint64_t* w, size_t i) { return (int)((w[i >> 6] >> (i & 63)) & 1u); }

/* merge.hpp:34-58, bit-serial with the literal double compare of
 * rng.hpp:46-54 (next_uniform() < p). */
int orc_merge_signs(const uint64_t* recv, uint32_t c_recv, const uint64_t* local,
                    uint32_t c_local, size_t len, uint64_t key, uint64_t* used, uint64_t* out) {
    if (c_recv == 0 || c_local == 0) return ORC_EPARAM;
    const double p = (double)c_recv / ((double)c_recv + (double)c_local);
    const size_t nw = (len + 63) / 64;
    uint64_t* tmp = (uint64_t*)calloc(nw ? nw : 1, sizeof(uint64_t));
    uint64_t n = *used;
    for (size_t j = 0; j < len; ++j) {
        int r = get_bit(recv, j), l = get_bit(local, j);
        int res = r;
        if (r != l) {
            double u = (double)(orc_draw(key, n) >> 11) * 0x1.0p-53;
            ++n;
            res = (u < p) ? r : l;
        }
        if (res) tmp[j >> 6] |= (uint64_t)1 << (j & 63);
    }
    memcpy(out, tmp, nw * sizeof(uint64_t));
    free(tmp);
    *used = n;
    return ORC_OK;
}

/* allreduce.hpp:148-189 driving detail::run_schedule (51-73) and the lock-step
 * Transport (transport.hpp:18-47): every sender's payload is snapshotted
 * before any delivery of the step; deliveries happen in ascending sender order. */
/* statistics of the most recent orc_allreduce_sign call (orc_last_sign_stats) */
static uint64_t g_last_draws, g_last_merges;

void orc_last_sign_stats(uint64_t* draws, uint64_t* merges) {
    *draws = g_last_draws;
    *merges = g_last_merges;
}

int orc_allreduce_sign(uint32_t workers, uint32_t segments, size_t seg_len,
                       const uint64_t* signs, uint32_t steps, const uint8_t* phase,
                       const uint32_t* send_to, const uint32_t* recv_from,
                       const uint32_t* segment, uint64_t seed, uint64_t round,
                       uint64_t* out_state, uint32_t* out_counts, uint64_t* bits_per_worker,
                       uint64_t* reduce_bits, uint64_t* gather_bits) {
    int st = orc_validate_schedule(workers, segments, steps, send_to, recv_from, segment);
    if (st) return st;
    const size_t nw = (seg_len + 63) / 64;
    const size_t per_w = (size_t)segments * nw;
    uint64_t* state = out_state;
    memcpy(state, signs, (size_t)workers * per_w * sizeof(uint64_t));
    uint64_t* used = (uint64_t*)calloc((size_t)workers * segments, sizeof(uint64_t));
    uint64_t* inbox = (uint64_t*)malloc(((size_t)workers * nw + 1) * sizeof(uint64_t));
    uint32_t* inbox_count = (uint32_t*)malloc(workers * sizeof(uint32_t));
    for (size_t i = 0; i < (size_t)workers * segments; ++i) out_counts[i] = 1;
    for (uint32_t w = 0; w < workers; ++w) bits_per_worker[w] = 0;
    *reduce_bits = *gather_bits = 0;
    g_last_draws = g_last_merges = 0;

    for (uint32_t k = 0; k < steps; ++k) {
        const uint32_t* st_ = send_to + (size_t)k * workers;
        const uint32_t* sg = segment + (size_t)k * workers;
        /* make_payload snapshot + bits.add (allreduce.hpp:57-62, 182) */
        for (uint32_t w = 0; w < workers; ++w) {
            memcpy(inbox + (size_t)w * nw, state + (size_t)w * per_w + (size_t)sg[w] * nw,
                   nw * sizeof(uint64_t));
            inbox_count[w] = out_counts[(size_t)w * segments + sg[w]];
            bits_per_worker[w] += seg_len;
            if (phase[k] == ORC_PHASE_REDUCE) *reduce_bits += seg_len;
            else *gather_bits += seg_len;
        }
        /* deliver_step in ascending sender order (transport.hpp:27-35) */
        for (uint32_t from = 0; from < workers; ++from) {
            uint32_t to = st_[from], s = sg[from];
            uint64_t* dst = state + (size_t)to * per_w + (size_t)s * nw;
            uint32_t* cnt = &out_counts[(size_t)to * segments + s];
            if (phase[k] == ORC_PHASE_REDUCE) {
                /* stream_for(to, s): one lazily created stream per (receiver, segment)
                 * (allreduce.hpp:170-177); `used` carries its position. */
                uint64_t key = orc_stream_key(seed, ORC_PURPOSE_MERGE, to, round, s);
                int rc = orc_merge_signs(inbox + (size_t)from * nw, inbox_count[from], dst, *cnt,
                                         seg_len, key, &used[(size_t)to * segments + s], dst);
                if (rc) { st = rc; goto done; }
                *cnt = inbox_count[from] + *cnt;
                ++g_last_merges;
            } else {
                memcpy(dst, inbox + (size_t)from * nw, nw * sizeof(uint64_t));
                *cnt = inbox_count[from];
            }
        }
    }
done:
    /* every draw of a (receiver, segment) stream is one disagreeing coordinate */
    for (size_t i = 0; i < (size_t)workers * segments; ++i) g_last_draws += used[i];
    free(used);
    free(inbox);
    free(inbox_count);
    return st;
}

/* allreduce.hpp:98-130 (segments padded with 0.0, segmentation.hpp:32-53). */
int orc_allreduce_dense(uint32_t workers, uint32_t segments, size_t dim, const double* vectors,
                        uint32_t steps, const uint8_t* phase, const uint32_t* send_to,
                        const uint32_t* recv_from, const uint32_t* segment, double* out_mean,
                        uint64_t* bits_per_worker, uint64_t* reduce_bits,
                        uint64_t* gather_bits) {
    int st = orc_validate_schedule(workers, segments, steps, send_to, recv_from, segment);
    if (st) return st;
    const size_t L = (dim + segments - 1) / segments;
    const size_t per_w = (size_t)segments * L;
    double* state = (double*)calloc((size_t)workers * per_w, sizeof(double));
    double* inbox = (double*)malloc((size_t)workers * L * sizeof(double) + 8);
    for (uint32_t w = 0; w < workers; ++w)
        for (size_t j = 0; j < dim; ++j) state[(size_t)w * per_w + j] = vectors[(size_t)w * dim + j];
    for (uint32_t w = 0; w < workers; ++w) bits_per_worker[w] = 0;
    *reduce_bits = *gather_bits = 0;
    for (uint32_t k = 0; k < steps; ++k) {
        const uint32_t* st_ = send_to + (size_t)k * workers;
        const uint32_t* sg = segment + (size_t)k * workers;
        for (uint32_t w = 0; w < workers; ++w) {
            memcpy(inbox + (size_t)w * L, state + (size_t)w * per_w + (size_t)sg[w] * L,
                   L * sizeof(double));
            bits_per_worker[w] += (uint64_t)L * 32u;
            if (phase[k] == ORC_PHASE_REDUCE) *reduce_bits += (uint64_t)L * 32u;
            else *gather_bits += (uint64_t)L * 32u;
        }
        for (uint32_t from = 0; from < workers; ++from) {
            double* dst = state + (size_t)st_[from] * per_w + (size_t)sg[from] * L;
            const double* src = inbox + (size_t)from * L;
            if (phase[k] == ORC_PHASE_REDUCE) {
                /* add(state[to][s], p): a[i] + b[i]; DenseVector ctor checks finiteness */
                for (size_t j = 0; j < L; ++j) {
                    dst[j] = dst[j] + src[j];
                    if (!isfinite(dst[j])) { st = ORC_ENONFINITE; goto done; }
                }
            } else {
                memcpy(dst, src, L * sizeof(double));
            }
        }
    }
    {
        const double inv_m = 1.0 / (double)workers;
        /* consensus over per-worker results (sync.hpp:81 -> allreduce.hpp:32-43) */
        for (size_t j = 0; j < dim; ++j) {
            double v0 = state[j] * inv_m;
            for (uint32_t w = 1; w < workers; ++w)
                if (!(state[(size_t)w * per_w + j] * inv_m == v0)) { st = ORC_EPROTOCOL; goto done; }
            out_mean[j] = v0;
        }
    }
done:
    free(state);
    free(inbox);
    return st;
}

/* sync.hpp:60-120 */
int orc_marsit_round(uint64_t t, int has_period, uint64_t period, double eta_s,
                     uint32_t workers, uint32_t segments, size_t dim, const double* grads,
                     const double* comp, uint32_t steps, const uint8_t* phase,
                     const uint32_t* send_to, const uint32_t* recv_from,
                     const uint32_t* segment, uint64_t seed, double* out_update,
                     double* out_comp, uint64_t* out_agg_bits, int* out_full_precision,
                     uint64_t* bits_per_worker, uint64_t* reduce_bits, uint64_t* gather_bits) {
    /* SyncConfig::validate (27-34) */
    if (has_period && period == 0) return ORC_EPARAM;
    if (!(eta_s > 0.0)) return ORC_EPARAM;
    if (dim == 0) return ORC_EPARAM; /* DenseVector: dimension must be >= 1 */
    if (segments == 0) return ORC_EPARAM;
    const size_t n = (size_t)workers * dim;
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(grads[i]) || !isfinite(comp[i])) return ORC_ENONFINITE;
    /* u[w] = add(g[w], c[w]) (71-76) */
    double* u = (double*)malloc(n * sizeof(double));
    int st = ORC_OK;
    for (size_t i = 0; i < n; ++i) {
        u[i] = grads[i] + comp[i];
        if (!isfinite(u[i])) { free(u); return ORC_ENONFINITE; }
    }
    const int dense = has_period && (t % period == 0);
    *out_full_precision = dense;
    if (dense) {
        /* 78-87 */
        st = orc_allreduce_dense(workers, segments, dim, u, steps, phase, send_to, recv_from,
                                 segment, out_update, bits_per_worker, reduce_bits, gather_bits);
        if (!st) memset(out_comp, 0, n * sizeof(double));
        free(u);
        return st;
    }
    /* sign path (91-118) */
    const size_t L = (dim + segments - 1) / segments;
    const size_t nw = (L + 63) / 64;
    uint64_t* signs = (uint64_t*)calloc((size_t)workers * segments * nw, sizeof(uint64_t));
    uint64_t* state = (uint64_t*)calloc((size_t)workers * segments * nw, sizeof(uint64_t));
    uint32_t* counts = (uint32_t*)calloc((size_t)workers * segments, sizeof(uint32_t));
    double* part = (double*)malloc(L * sizeof(double));
    for (uint32_t w = 0; w < workers; ++w)
        for (uint32_t s = 0; s < segments; ++s) {
            for (size_t j = 0; j < L; ++j) {
                size_t src = (size_t)s * L + j;
                part[j] = src < dim ? u[(size_t)w * dim + src] : 0.0; /* segmentation.hpp:45-49 */
            }
            orc_pack_signs(part, L, signs + ((size_t)w * segments + s) * nw);
        }
    st = orc_allreduce_sign(workers, segments, L, signs, steps, phase, send_to, recv_from,
                            segment, seed, t, state, counts, bits_per_worker, reduce_bits,
                            gather_bits);
    if (st) goto done;
    /* consensus (101) */
    for (uint32_t w = 1; w < workers; ++w)
        for (uint32_t s = 0; s < segments; ++s) {
            if (counts[(size_t)w * segments + s] != counts[s] ||
                memcmp(state + ((size_t)w * segments + s) * nw, state + (size_t)s * nw,
                       nw * sizeof(uint64_t)) != 0) {
                st = ORC_EPROTOCOL;
                goto done;
            }
        }
    /* reassemble (103-112) */
    memset(out_agg_bits, 0, ((dim + 63) / 64) * sizeof(uint64_t));
    for (uint32_t s = 0; s < segments; ++s) {
        if (counts[s] != workers) { st = ORC_EPROTOCOL; goto done; }
        for (size_t j = 0; j < L; ++j) {
            size_t coord = (size_t)s * L + j;
            if (coord < dim && get_bit(state + (size_t)s * nw, j))
                out_agg_bits[coord >> 6] |= (uint64_t)1 << (coord & 63);
        }
    }
    /* unpack_to_update (sign_vector.hpp:77-89) and c' = u - g (116-118) */
    for (size_t j = 0; j < dim; ++j) out_update[j] = get_bit(out_agg_bits, j) ? eta_s : -eta_s;
    for (uint32_t w = 0; w < workers; ++w)
        for (size_t j = 0; j < dim; ++j) {
            double v = u[(size_t)w * dim + j] - out_update[j];
            if (!isfinite(v)) { st = ORC_ENONFINITE; goto done; }
            out_comp[(size_t)w * dim + j] = v;
        }
done:
    free(u);
    free(signs);
    free(state);
    free(counts);
    free(part);
    return st;
}

/* ---- SSDM baselines ---------------------------------------------------- */

#define ORC_PURPOSE_SSDM 4 /* rng.hpp:18 */

/* rng.hpp:46-54: next_uniform = (x >> 11) * 2^-53; next_bernoulli(p) = u < p */
static double uniform_of(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

/* ssdm.hpp:29-40 (DenseVector::l2_norm, dense_vector.hpp:41-45: acc += v*v) */
double orc_ssdm_compress(const double* v, size_t len, uint64_t key, uint64_t* bits) {
    double acc = 0.0;
    for (size_t j = 0; j < len; ++j) acc += v[j] * v[j];
    const double norm = sqrt(acc);
    memset(bits, 0, ((len + 63) / 64) * sizeof(uint64_t));
    const double denom = norm > 0.0 ? 2.0 * norm : 0.0;
    for (size_t j = 0; j < len; ++j) {
        const double p = denom > 0.0 ? 0.5 + v[j] / denom : 0.5;
        if (uniform_of(orc_draw(key, j)) < p) bits[j >> 6] |= (uint64_t)1 << (j & 63);
    }
    return norm;
}

/* ssdm.hpp:44-56 */
void orc_ssdm_decompress(const uint64_t* bits, size_t len, double norm, double* out) {
    for (size_t j = 0; j < len; ++j)
        out[j] = norm == 0.0 ? 0.0 : (get_bit(bits, j) ? norm : -norm);
}

/* elias.hpp:14-31: gamma length of zigzag(s) + 1 */
static uint64_t signed_sum_code_length(int64_t s) {
    const uint64_t z = ((uint64_t)s << 1) ^ (uint64_t)(s >> 63);
    uint64_t n = z + 1, width = 0;
    while (n) { ++width; n >>= 1; }
    return 2 * width - 1;
}

/* allreduce.hpp:205-262.  State per (worker, segment): the dense raw segment
 * (segmentation.hpp:32-53, value padding 0.0) and an optional packet. */
int orc_cascading_allreduce(uint32_t workers, uint32_t segments, size_t dim,
                            const double* vectors, uint32_t steps, const uint8_t* phase,
                            const uint32_t* send_to, const uint32_t* recv_from,
                            const uint32_t* segment, int is_ring, uint64_t seed, uint64_t round,
                            double* out_estimate, uint64_t* bits_per_worker,
                            uint64_t* reduce_bits, uint64_t* gather_bits) {
    if (!is_ring) return ORC_EUNSUPPORTED;
    int st = orc_validate_schedule(workers, segments, steps, send_to, recv_from, segment);
    if (st) return st;
    if (dim == 0) return ORC_EPARAM;
    const size_t L = (dim + segments - 1) / segments, nw = (L + 63) / 64;
    const size_t n_ws = (size_t)workers * segments;
    double* raw = (double*)calloc(n_ws * L, sizeof(double));
    uint64_t* pk_bits = (uint64_t*)calloc(n_ws * nw, sizeof(uint64_t));
    double* pk_norm = (double*)calloc(n_ws, sizeof(double));
    uint8_t* has = (uint8_t*)calloc(n_ws, 1);
    uint64_t* in_bits = (uint64_t*)malloc(((size_t)workers * nw + 1) * sizeof(uint64_t));
    double* in_norm = (double*)malloc(workers * sizeof(double));
    double* dec = (double*)malloc(L * sizeof(double));
    for (uint32_t w = 0; w < workers; ++w)
        for (size_t j = 0; j < dim; ++j)
            raw[(size_t)w * segments * L + j] = vectors[(size_t)w * dim + j];
    for (uint32_t w = 0; w < workers; ++w) bits_per_worker[w] = 0;
    *reduce_bits = *gather_bits = 0;
    for (uint32_t k = 0; k < steps; ++k) {
        const uint32_t* st_ = send_to + (size_t)k * workers;
        const uint32_t* sg = segment + (size_t)k * workers;
        for (uint32_t w = 0; w < workers; ++w) { /* make_payload: compress lazily */
            const size_t i = (size_t)w * segments + sg[w];
            if (!has[i]) {
                const uint64_t key = orc_stream_key(seed, ORC_PURPOSE_SSDM, w, round, sg[w]);
                pk_norm[i] = orc_ssdm_compress(raw + i * L, L, key, pk_bits + i * nw);
                has[i] = 1;
            }
            memcpy(in_bits + (size_t)w * nw, pk_bits + i * nw, nw * sizeof(uint64_t));
            in_norm[w] = pk_norm[i];
            bits_per_worker[w] += (uint64_t)L + 32u; /* bits.size() + 32 */
            if (phase[k] == ORC_PHASE_REDUCE) *reduce_bits += (uint64_t)L + 32u;
            else *gather_bits += (uint64_t)L + 32u;
        }
        for (uint32_t from = 0; from < workers; ++from) { /* deliver in sender order */
            const size_t i = (size_t)st_[from] * segments + sg[from];
            if (phase[k] == ORC_PHASE_REDUCE) {
                /* raw = add(ssdm_decompress(p), raw) */
                orc_ssdm_decompress(in_bits + (size_t)from * nw, L, in_norm[from], dec);
                for (size_t j = 0; j < L; ++j) {
                    raw[i * L + j] = dec[j] + raw[i * L + j];
                    if (!isfinite(raw[i * L + j])) { st = ORC_ENONFINITE; goto done; }
                }
            } else {
                memcpy(pk_bits + i * nw, in_bits + (size_t)from * nw, nw * sizeof(uint64_t));
                pk_norm[i] = in_norm[from];
                has[i] = 1;
            }
        }
    }
    {
        /* per worker: reassemble(scaled(ssdm_decompress(packet), 1/M)); consensus */
        const double inv_m = 1.0 / (double)workers;
        for (uint32_t w = 0; w < workers; ++w)
            for (uint32_t s = 0; s < segments; ++s) {
                const size_t i = (size_t)w * segments + s;
                if (!has[i]) { st = ORC_EPROTOCOL; goto done; }
                orc_ssdm_decompress(pk_bits + i * nw, L, pk_norm[i], dec);
                for (size_t j = 0; j < L && (size_t)s * L + j < dim; ++j) {
                    const double v = dec[j] * inv_m;
                    double* o = out_estimate + (size_t)s * L + j;
                    if (w == 0) *o = v;
                    else if (!(*o == v)) { st = ORC_EPROTOCOL; goto done; }
                }
            }
    }
done:
    free(raw); free(pk_bits); free(pk_norm); free(has); free(in_bits); free(in_norm); free(dec);
    return st;
}

/* allreduce.hpp:275-339 */
int orc_sum_ssdm_allreduce(uint32_t workers, uint32_t segments, size_t dim,
                           const double* vectors, uint32_t steps, const uint8_t* phase,
                           const uint32_t* send_to, const uint32_t* recv_from,
                           const uint32_t* segment, int is_ring, uint64_t seed, uint64_t round,
                           double* out_estimate, uint64_t* bits_per_worker,
                           uint64_t* reduce_bits, uint64_t* gather_bits,
                           int64_t* max_abs_per_step) {
    if (!is_ring) return ORC_EUNSUPPORTED;
    int st = orc_validate_schedule(workers, segments, steps, send_to, recv_from, segment);
    if (st) return st;
    if (dim == 0) return ORC_EPARAM;
    const size_t L = (dim + segments - 1) / segments, nw = (L + 63) / 64;
    const size_t n_ws = (size_t)workers * segments;
    uint64_t* pk_bits = (uint64_t*)calloc(n_ws * nw, sizeof(uint64_t));
    double* pk_norm = (double*)calloc(n_ws, sizeof(double));
    int64_t* sums = (int64_t*)malloc(n_ws * L * sizeof(int64_t));
    int64_t* inbox = (int64_t*)malloc(((size_t)workers * L + 1) * sizeof(int64_t));
    double* part = (double*)calloc(L, sizeof(double));
    double* dec = (double*)malloc(L * sizeof(double));
    for (uint32_t w = 0; w < workers; ++w)
        for (uint32_t s = 0; s < segments; ++s) { /* compress once, sums = +-1 */
            const size_t i = (size_t)w * segments + s;
            for (size_t j = 0; j < L; ++j) {
                const size_t src = (size_t)s * L + j;
                part[j] = src < dim ? vectors[(size_t)w * dim + src] : 0.0;
            }
            pk_norm[i] = orc_ssdm_compress(
                part, L, orc_stream_key(seed, ORC_PURPOSE_SSDM, w, round, s), pk_bits + i * nw);
            for (size_t j = 0; j < L; ++j) sums[i * L + j] = get_bit(pk_bits + i * nw, j) ? 1 : -1;
        }
    for (uint32_t w = 0; w < workers; ++w) bits_per_worker[w] = 0;
    *reduce_bits = *gather_bits = 0;
    for (uint32_t k = 0; k < steps; ++k) {
        const uint32_t* st_ = send_to + (size_t)k * workers;
        const uint32_t* sg = segment + (size_t)k * workers;
        int64_t step_max = 0;
        for (uint32_t w = 0; w < workers; ++w) {
            const size_t i = (size_t)w * segments + sg[w];
            uint64_t total = 32; /* norm side channel */
            for (size_t j = 0; j < L; ++j) {
                const int64_t v = sums[i * L + j];
                inbox[(size_t)w * L + j] = v;
                total += signed_sum_code_length(v);
                const int64_t mag = v < 0 ? -v : v;
                if (mag > step_max) step_max = mag;
            }
            bits_per_worker[w] += total;
            if (phase[k] == ORC_PHASE_REDUCE) *reduce_bits += total;
            else *gather_bits += total;
        }
        if (max_abs_per_step) max_abs_per_step[k] = step_max;
        for (uint32_t from = 0; from < workers; ++from) {
            int64_t* dst = sums + ((size_t)st_[from] * segments + sg[from]) * L;
            const int64_t* src = inbox + (size_t)from * L;
            if (phase[k] == ORC_PHASE_REDUCE) for (size_t j = 0; j < L; ++j) dst[j] += src[j];
            else memcpy(dst, src, L * sizeof(int64_t));
        }
    }
    {
        /* mean of the individually decompressed packets, worker order, * 1/M */
        const double inv_m = 1.0 / (double)workers;
        for (uint32_t s = 0; s < segments; ++s) {
            for (size_t j = 0; j < L; ++j) part[j] = 0.0;
            for (uint32_t w = 0; w < workers; ++w) {
                const size_t i = (size_t)w * segments + s;
                orc_ssdm_decompress(pk_bits + i * nw, L, pk_norm[i], dec);
                for (size_t j = 0; j < L; ++j) part[j] += dec[j];
            }
            for (size_t j = 0; j < L && (size_t)s * L + j < dim; ++j)
                out_estimate[(size_t)s * L + j] = part[j] * inv_m;
        }
    }
    free(pk_bits); free(pk_norm); free(sums); free(inbox); free(part); free(dec);
    return st;
}

void orc_gen_dyadic(uint64_t seed, uint64_t worker, uint64_t round, size_t dim, double* out) {
    uint64_t key = orc_stream_key(seed, ORC_PURPOSE_TRIAL, worker, round, 0);
    for (size_t j = 0; j < dim; ++j) {
        int64_t q = (int64_t)(orc_draw(key, j) >> 51) - 4096;
        out[j] = (double)q * 0x1.0p-20;
    }
}

void orc_gen_correlated(uint64_t seed, uint64_t worker, uint64_t round, size_t dim,
                        double* out) {
    uint64_t ka = orc_stream_key(seed, ORC_PURPOSE_TRIAL, 0xFFFF, round, 0);
    uint64_t kb = orc_stream_key(seed, ORC_PURPOSE_TRIAL, worker, round, 0);
    for (size_t j = 0; j < dim; ++j) {
        int64_t a = (int64_t)(orc_draw(ka, j) >> 52) - 2048;
        int64_t b = (int64_t)(orc_draw(kb, j) >> 53) - 1024;
        out[j] = (double)(a + b) * 0x1.0p-20;
    }
}
