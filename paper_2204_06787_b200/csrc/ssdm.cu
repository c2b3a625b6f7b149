// ssdm.cu — the reference's baseline collectives on the device (SURVEY §8f
// row 4): stochastic sign compression ssdm_compress / ssdm_decompress
// (ssdm.hpp:29-56), the cascading-compression all-reduce cascading_allreduce
// (allreduce.hpp:205-262) and the sum-accumulation all-reduce
// sum_ssdm_allreduce (allreduce.hpp:275-339), with every worker on one
// context (G == 1).
//
// Kernels (all HBM streaming or ALU work):
//   sumsq_raw / hop   fixed-order partial sums of v^2 per CTA chunk (the l2
//                     norm, dense_vector.hpp:41-45); `hop` also forms the
//                     cascading accumulator dec(packet) + raw (add, 53-58)
//   compress          bit j = (uniform_j < 1/2 + v_j / (2 norm)), uniform_j =
//                     draw j of RngStream(seed, ssdm, w, t, s) — one draw per
//                     coordinate, so the draws are random access
//   out_*             the estimate every worker ends with
//   hist              Elias-gamma payload accounting of the sum variant:
//                     histogram of the number of +1 signs among each chain
//                     prefix (bit-sliced counters), from which the code
//                     lengths of every partial sum follow exactly
//
// Norm: per-chunk partial sums, then one warp per item sums them in a fixed
// order, so the norm is deterministic; it equals the reference's sequential
// sum whenever that sum is exact (e.g. the dyadic recipe inputs) and is
// within a few ulps otherwise.  The Bernoulli draws avoid the division in
// all but ~2^-21 of the coordinates (ssdm_bit) and stay exact.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "internal.hpp"
#include "rng.cuh"

namespace marsit_b200 {
namespace {

constexpr int kSsThreads = 256;
constexpr uint32_t kSsChunk = kSsThreads * 32;  // coordinates per CTA in the norm passes
constexpr uint64_t kPurposeSsdm = 4;            // rng.hpp:18
constexpr uint32_t kSsMaxWorkers = 64;          // bit-sliced counters: 7 planes
constexpr unsigned kAll = 0xffffffffu;

struct SsdmParams {
    const void* vec[kMaxLocalWorkers];  // worker inputs, D elements of dtype
    uint32_t M, S, wst, nb;             // workers, segments, u32 words per packet, norm CTAs per item
    uint64_t D, L;
    uint64_t seed, round;
    const uint8_t* chain;  // [S][M]: worker at chain position k of segment s
    int k;                 // cascading hop
    int mode;              // 0 cascading, 1 sum
    int64_t key_w, key_s;  // standalone compress: explicit (worker, segment)
    double* acc;           // cascading accumulators [S][L]
    uint32_t* pk;          // packets: cascading [S][wst]; sum [M][S][wst]
    double* norms;         // per item
    double* partial;       // [item][nb]
    int* err;
};

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(kAll, v, o));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kSsThreads / 32; ++w) t = __dadd_rn(t, sh[w]);
    return t;  // valid in thread 0
}

__host__ __device__ __forceinline__ uint64_t ceil_div_d(uint64_t a, uint64_t b) {
    return (a + b - 1) / b;
}

template <typename T>
__device__ __forceinline__ double raw_at(const SsdmParams& p, uint32_t w, uint32_t s, uint64_t j) {
    const uint64_t gi = uint64_t(s) * p.L + j;
    return (j < p.L && gi < p.D) ? double(static_cast<const T*>(p.vec[w])[gi]) : 0.0;
}

// ssdm_decompress (ssdm.hpp:44-56) of coordinate j of a packet
__device__ __forceinline__ double dec_at(const uint32_t* pk, uint64_t j, double norm) {
    if (norm == 0.0) return 0.0;
    return ((pk[j >> 5] >> (j & 31)) & 1u) ? norm : -norm;
}

// Four consecutive coordinates j..j+3 of worker w's segment s in the input
// type (value padding beyond L / D reads 0).  VEC: quads fully inside both
// bounds are one 16-byte aligned vector load.
template <typename T, bool VEC>
__device__ __forceinline__ void raw_quad(const SsdmParams& p, uint32_t w, uint32_t s, uint64_t j,
                                         T (&v)[4]) {
    const uint64_t gi = uint64_t(s) * p.L + j;
    const T* src = static_cast<const T*>(p.vec[w]);
    if (VEC && j + 3 < p.L && gi + 3 < p.D) {
        if constexpr (sizeof(T) == 4) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(src + gi));
            v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
        } else {
            const double2 a = __ldg(reinterpret_cast<const double2*>(src + gi));
            const double2 b = __ldg(reinterpret_cast<const double2*>(src + gi) + 1);
            v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = (j + k < p.L && gi + k < p.D) ? src[gi + k] : T(0);
    }
}

// Sum of squares of the raw segments (sum variant: item = w * S + s).  A CTA
// owns a fixed chunk of kSsChunk coordinates (the summation order does not
// depend on the hardware); thread t takes quads t, t + 256, ... of it.
template <typename T, bool VEC>
__global__ void __launch_bounds__(kSsThreads) ssdm_sumsq_raw_kernel(const SsdmParams p) {
    __shared__ double sh[kSsThreads / 32];
    const uint32_t item = blockIdx.y, w = item / p.S, s = item % p.S;
    const uint64_t base = uint64_t(blockIdx.x) * kSsChunk;
    T v[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        raw_quad<T, VEC>(p, w, s, base + (uint64_t(i) * kSsThreads + threadIdx.x) * 4, v[i]);
    double ss = 0.0;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double x = double(v[i][k]);
            bad |= !isfinite(x);
            ss = __dadd_rn(ss, __dmul_rn(x, x));
        }
    if (bad) atomicExch(p.err, 1);  // DenseVector: non-finite entry (dense_vector.hpp:25-29)
    const double t = block_sum(ss, sh);
    if (threadIdx.x == 0) p.partial[uint64_t(item) * p.nb + blockIdx.x] = t;
}

// Cascading hop k for every segment (item = s): acc = raw (k = 0) or
// add(ssdm_decompress(packet of hop k-1), raw) (allreduce.hpp:240-242), and its
// sum of squares.
template <typename T, bool VEC>
__global__ void __launch_bounds__(kSsThreads) ssdm_hop_kernel(const SsdmParams p) {
    __shared__ double sh[kSsThreads / 32];
    const uint32_t s = blockIdx.y;
    const uint32_t w = p.chain[s * p.M + p.k];
    const uint32_t* pk = p.pk + uint64_t(s) * p.wst;
    const double nrm = p.k > 0 ? p.norms[s] : 0.0;
    double* acc = p.acc + uint64_t(s) * p.L;
    const uint64_t base = uint64_t(blockIdx.x) * kSsChunk;
    T r[8][4];
    uint32_t word[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint64_t j = base + (uint64_t(i) * kSsThreads + threadIdx.x) * 4;
        raw_quad<T, VEC>(p, w, s, j, r[i]);
        word[i] = (p.k > 0 && j < p.L) ? __ldg(pk + (j >> 5)) : 0u;
    }
    double ss = 0.0;
    bool bad = false;
    // acc rows start at s * L doubles: 16-byte aligned pairs iff L is even
    const bool pairs = VEC && (p.L % 2 == 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint64_t j = base + (uint64_t(i) * kSsThreads + threadIdx.x) * 4;
        double v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k] = double(r[i][k]);
            if (p.k > 0) {
                const double d = nrm == 0.0 ? 0.0 : (((word[i] >> ((j + k) & 31)) & 1u) ? nrm : -nrm);
                v[k] = __dadd_rn(d, v[k]);
            }
        }
        if (pairs && j + 3 < p.L) {
            reinterpret_cast<double2*>(acc + j)[0] = make_double2(v[0], v[1]);
            reinterpret_cast<double2*>(acc + j)[1] = make_double2(v[2], v[3]);
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (j + k < p.L) acc[j + k] = v[k];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (j + k < p.L) {
                bad |= !isfinite(v[k]);
                ss = __dadd_rn(ss, __dmul_rn(v[k], v[k]));
            }
    }
    if (bad) atomicExch(p.err, 1);
    const double t = block_sum(ss, sh);
    if (threadIdx.x == 0) p.partial[uint64_t(s) * p.nb + blockIdx.x] = t;
}

// The l2 norm of every item from its per-chunk partial sums, one warp per
// item, always the same order (lane l takes chunks l, l+32, ...; then a fixed
// butterfly), so every later use sees one deterministic value.
__global__ void ssdm_norm_kernel(const SsdmParams p, uint32_t items) {
    const uint32_t item = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (item >= items) return;
    double t = 0.0;
    for (uint32_t b = lane; b < p.nb; b += 32) t = __dadd_rn(t, p.partial[uint64_t(item) * p.nb + b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = __dadd_rn(t, __shfl_xor_sync(kAll, t, o));
    if (lane == 0) p.norms[item] = __dsqrt_rn(t);
}

// Bernoulli draw of ssdm_compress (ssdm.hpp:33-37): bit = (u < p), u = (x >> 11)
// * 2^-53, x = mix64(z), z = key + (j+1)γ, p = 1/2 + v / (2 norm).  Exact,
// without a division in the common case: P = p * 2^53 is known to +-2 units
// from one FMA (s53 = 2^52 / norm), and (x >> 11) < P is decided by the high
// word xh of x alone (x lies in [xh, xh+1) * 2^32, i.e. x >> 11 in
// [xh, xh+1) * 2^21) unless that interval is within 16 units of P — one
// value of xh in 2^32 — in which case the literal formula runs.
__device__ __forceinline__ bool ssdm_bit(uint64_t z, double v, double norm, double denom,
                                         double s53) {
    if (norm == 0.0) return mix64_hi(z) < 0x80000000u;  // p = 1/2 exactly
    const double pd = fma(v, s53, 0x1p52);
    const double lo = fma(double(mix64_hi(z)), 0x1p21, -pd);  // xh * 2^21 - P (exact)
    if (lo + 0x1p21 <= -16.0) return true;                     // whole block below P
    if (lo >= 16.0) return false;                              // whole block above P
    const double u = double(mix64(z) >> 11) * 0x1.0p-53;
    return u < __dadd_rn(0.5, __ddiv_rn(v, denom));
}

constexpr int kSsWordsPerWarp = 64;  // batches of 8 words, loads first

// ssdm_compress (ssdm.hpp:29-40) of every item; SRC: T for raw inputs (sum
// variant / standalone), double for the cascading accumulators.
template <typename SRC, bool CASCADE>
__global__ void __launch_bounds__(kSsThreads) ssdm_compress_kernel(const SsdmParams p) {
    const uint32_t item = blockIdx.y;
    uint32_t w, s;
    if (CASCADE) {
        s = item;
        w = p.chain[s * p.M + p.k];
    } else {
        w = item / p.S;
        s = item % p.S;
    }
    const double norm = p.norms[item];
    const double denom = norm > 0.0 ? __dmul_rn(2.0, norm) : 0.0;
    const double s53 = norm > 0.0 ? __ddiv_rn(0x1p52, norm) : 0.0;
    const uint64_t key =
        p.key_w >= 0 ? stream_key(p.seed, kPurposeSsdm, uint64_t(p.key_w), p.round, uint64_t(p.key_s))
                     : stream_key(p.seed, kPurposeSsdm, w, p.round, s);
    const int lane = threadIdx.x & 31;
    const uint32_t warp = blockIdx.x * (kSsThreads / 32) + (threadIdx.x >> 5);
    uint32_t* out = p.pk + uint64_t(item) * p.wst;
    const uint32_t q_end = min(p.wst, (warp + 1) * kSsWordsPerWarp);
    // this item's values: coordinates [0, valid) of the segment are real,
    // [valid, L) value padding (0)
    const uint64_t seg0 = uint64_t(s) * p.L;
    const uint64_t valid = CASCADE ? p.L : (p.D > seg0 ? min(p.L, p.D - seg0) : 0);
    const double* accs = p.acc + seg0;
    const SRC* raw = static_cast<const SRC*>(p.vec[w]) + seg0;
    for (uint32_t q0 = warp * kSsWordsPerWarp; q0 < q_end; q0 += 8) {
        double v[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const uint64_t j = uint64_t(q0 + b) * 32 + lane;
            if (j >= valid)
                v[b] = 0.0;
            else if (CASCADE)
                v[b] = accs[j];
            else
                v[b] = double(raw[j]);
        }
        uint64_t z = key + (uint64_t(q0) * 32 + lane + 1) * kGamma;  // draw j = 32 q + lane
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const uint64_t j = uint64_t(q0 + b) * 32 + lane;
            const bool bit = j < p.L && ssdm_bit(z, v[b], norm, denom, s53);
            z += 32 * kGamma;
            const uint32_t word = __ballot_sync(kAll, bit);
            if (lane == b && q0 + b < q_end) out[q0 + b] = word;
        }
    }
}

// Cascading estimate: reassemble(scaled(ssdm_decompress(final packet), 1/M))
// (allreduce.hpp:252-260).  A warp per packed word: the word is broadcast,
// lanes are coordinates (coalesced stores).
template <typename T>
__global__ void ssdm_out_cascade_kernel(const SsdmParams p, T* __restrict__ out) {
    const double inv_m = 1.0 / double(p.M);
    const uint32_t s = blockIdx.y;  // segment; warps stride over its packed words
    const uint64_t wps = ceil_div_d(p.L, 32);
    const int lane = threadIdx.x & 31;
    const double nrm = p.norms[s];
    const uint32_t* pk = p.pk + uint64_t(s) * p.wst;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x / 32);
    for (uint64_t q0 = (blockIdx.x * uint64_t(blockDim.x / 32) + (threadIdx.x >> 5)) * 4; q0 < wps;
         q0 += warps * 4) {
        uint32_t word[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) word[i] = q0 + i < wps ? __ldg(pk + q0 + i) : 0u;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint64_t j = (q0 + i) * 32 + lane, gi = uint64_t(s) * p.L + j;
            const double d = nrm == 0.0 ? 0.0 : (((word[i] >> lane) & 1u) ? nrm : -nrm);
            if (j < p.L && gi < p.D) out[gi] = T(__dmul_rn(d, inv_m));
        }
    }
}

// Sum variant estimate: mean of the M decompressed packets, summed in worker
// order from 0.0, times 1/M (allreduce.hpp:322-336).  A warp per packed word
// (lanes = coordinates); the packet words of 8 workers are loaded at once.
// +-norm is the norm with its sign bit set from the packet bit; a zero norm
// then contributes +-0.0 instead of +0.0, which leaves the sum unchanged (it
// starts at +0.0, and x + -0.0 == x for every x but -0.0).
template <typename T>
__global__ void ssdm_out_sum_kernel(const SsdmParams p, T* __restrict__ out) {
    __shared__ unsigned long long s_norm[kSsMaxWorkers];  // bit patterns
    const double inv_m = 1.0 / double(p.M);
    const uint32_t s = blockIdx.y;
    for (uint32_t w = threadIdx.x; w < p.M; w += blockDim.x)
        s_norm[w] = __double_as_longlong(p.norms[w * p.S + s]);
    __syncthreads();
    const uint64_t wps = ceil_div_d(p.L, 32);
    const uint64_t stride = uint64_t(p.S) * p.wst;  // worker w's row of segment s
    const int lane = threadIdx.x & 31;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x / 32);
    const uint64_t seg0 = uint64_t(s) * p.L;
    const uint64_t valid = p.D > seg0 ? min(p.L, p.D - seg0) : 0;
    for (uint64_t q = blockIdx.x * uint64_t(blockDim.x / 32) + (threadIdx.x >> 5); q < wps; q += warps) {
        const uint64_t j = q * 32 + lane;
        const uint32_t* row = p.pk + uint64_t(s) * p.wst + q;
        double a = 0.0;
        for (uint32_t w0 = 0; w0 < p.M; w0 += 8) {
            uint32_t word[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) word[i] = w0 + i < p.M ? __ldg(row + (w0 + i) * stride) : 0u;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (w0 + i >= p.M) break;
                const unsigned long long neg = uint64_t(((word[i] >> lane) & 1u) ^ 1u) << 63;
                a = __dadd_rn(a, __longlong_as_double(s_norm[w0 + i] | neg));
            }
        }
        if (j < valid) out[seg0 + j] = T(__dmul_rn(a, inv_m));
    }
}

// hist[s][k][c] += #coordinates of segment s with exactly c "+1" signs among
// chain positions 0..k (sum variant; L coordinates incl. value padding).
// The partial sum carried at that point is 2c - (k + 1).
__global__ void __launch_bounds__(kSsThreads) ssdm_hist_kernel(const SsdmParams p,
                                                               unsigned long long* hist) {
    extern __shared__ uint32_t sh_hist[];  // [M][M+1]
    const uint32_t s = blockIdx.y, M = p.M, H = M * (M + 1);
    for (uint32_t i = threadIdx.x; i < H; i += kSsThreads) sh_hist[i] = 0;
    __syncthreads();
    const uint32_t n_words = uint32_t((p.L + 31) / 32);
    for (uint32_t q = blockIdx.x * kSsThreads + threadIdx.x; q < n_words;
         q += gridDim.x * kSsThreads) {
        const uint64_t rem = p.L - uint64_t(q) * 32;
        const uint32_t valid = rem >= 32 ? kAll : ((1u << rem) - 1u);
        uint32_t c[7] = {0, 0, 0, 0, 0, 0, 0};  // bit-sliced counters, one per coordinate
        for (uint32_t k = 0; k < M; ++k) {
            const uint32_t w = p.chain[s * M + k];
            uint32_t carry = p.pk[(uint64_t(w) * p.S + s) * p.wst + q];
#pragma unroll
            for (int b = 0; b < 7; ++b) {
                const uint32_t t = c[b] & carry;
                c[b] ^= carry;
                carry = t;
            }
            for (uint32_t val = 0; val <= k + 1; ++val) {
                uint32_t eq = valid;
#pragma unroll
                for (int b = 0; b < 7; ++b) eq &= ((val >> b) & 1u) ? c[b] : ~c[b];
                const uint32_t n = __popc(eq);
                if (n) atomicAdd(&sh_hist[k * (M + 1) + val], n);
            }
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < H; i += kSsThreads)
        if (sh_hist[i]) atomicAdd(&hist[uint64_t(s) * H + i], (unsigned long long)sh_hist[i]);
}

template <typename T>
__global__ void ssdm_decompress_kernel(const uint32_t* __restrict__ pk, uint64_t len, double norm,
                                       T* __restrict__ out) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < len;
         j += uint64_t(gridDim.x) * blockDim.x)
        out[j] = T(dec_at(pk, j, norm));
}

// elias.hpp:14-31: gamma length of zigzag(v) + 1
uint64_t signed_sum_code_length(int64_t v) {
    const uint64_t z = (uint64_t(v) << 1) ^ uint64_t(v >> 63);
    uint64_t n = z + 1, width = 0;
    while (n) {
        ++width;
        n >>= 1;
    }
    return 2 * width - 1;
}


uint32_t compress_grid_x(uint32_t wst) {
    return uint32_t(ceil_div_d(wst, uint64_t(kSsThreads / 32) * kSsWordsPerWarp));
}


template <typename T>
marsit_status launch_pipeline(marsit_ctx* ctx, SsdmScratch& sc, SsdmParams& p, int mode,
                              void* d_out, bool want_hist, cudaStream_t st) {
    const dim3 blk(kSsThreads);
    const uint32_t cgx = compress_grid_x(p.wst);
    const uint32_t out_gx = uint32_t(std::max<uint64_t>(
        1, std::min<uint64_t>(ceil_div_d(ceil_div_d(p.L, 32), 8), ceil_div_d(uint64_t(ctx->sm_count) * 16, p.S))));
    // quads of a segment start at s * L: vector loads need L and D multiples
    // of 4 and 16-byte aligned inputs
    bool vec = p.L % 4 == 0;
    for (uint32_t w = 0; w < p.M; ++w) vec = vec && (reinterpret_cast<uintptr_t>(p.vec[w]) % 16 == 0);
    if (mode == 0) {
        for (uint32_t k = 0; k < p.M; ++k) {
            p.k = int(k);
            if (vec)
                ssdm_hop_kernel<T, true><<<dim3(p.nb, p.S), blk, 0, st>>>(p);
            else
                ssdm_hop_kernel<T, false><<<dim3(p.nb, p.S), blk, 0, st>>>(p);
            ssdm_norm_kernel<<<ceil_div_d(p.S, 8), 256, 0, st>>>(p, p.S);
            ssdm_compress_kernel<double, true><<<dim3(cgx, p.S), blk, 0, st>>>(p);
        }
        ssdm_out_cascade_kernel<T>
            <<<dim3(out_gx, p.S), 256, 0, st>>>(p, static_cast<T*>(d_out));
    } else {
        const uint32_t items = p.M * p.S;
        if (vec)
            ssdm_sumsq_raw_kernel<T, true><<<dim3(p.nb, items), blk, 0, st>>>(p);
        else
            ssdm_sumsq_raw_kernel<T, false><<<dim3(p.nb, items), blk, 0, st>>>(p);
        ssdm_norm_kernel<<<ceil_div_d(items, 8), 256, 0, st>>>(p, items);
        ssdm_compress_kernel<T, false><<<dim3(cgx, items), blk, 0, st>>>(p);
        ssdm_out_sum_kernel<T><<<dim3(out_gx, p.S), 256, 0, st>>>(p, static_cast<T*>(d_out));
        if (want_hist) {
            const size_t H = size_t(p.M) * (p.M + 1);
            CUDA_TRY(cudaMemsetAsync(sc.hist, 0, sizeof(unsigned long long) * H * p.S, st));
            const uint32_t n_w = uint32_t(ceil_div(p.L, 32));
            const uint32_t gx = std::max<uint32_t>(
                1, std::min<uint32_t>(ceil_div(n_w, kSsThreads), ceil_div(4u * ctx->sm_count, p.S)));
            ssdm_hist_kernel<<<dim3(gx, p.S), blk, H * sizeof(uint32_t), st>>>(p, sc.hist);
        }
    }
    CUDA_TRY(cudaGetLastError());
    return MARSIT_OK;
}

}  // namespace

marsit_status ssdm_allreduce_impl(marsit_ctx* ctx, int mode, uint64_t round, uint64_t seed,
                                  const void* const* d_vectors, void* d_estimate,
                                  uint64_t* bits_per_worker, uint64_t* reduce_bits,
                                  uint64_t* gather_bits, int64_t* max_abs_per_step,
                                  cudaStream_t st) {
    if (!ctx) return fail(MARSIT_EPARAM, "ctx is null");
    if (mode != MARSIT_SSDM_CASCADING && mode != MARSIT_SSDM_SUM)
        return fail(MARSIT_EPARAM, "ssdm mode must be cascading (0) or sum (1)");
    if (!d_vectors || !d_estimate) return fail(MARSIT_EPARAM, "null argument");
    const HostSchedule& hs = ctx->sched;
    // ring schedules (built, or explicit tables whose reduce phase is one
    // linear chain per segment — checked below); torus: as the reference
    if (hs.topology == 1)
        return fail(MARSIT_EUNSUPPORTED, mode == MARSIT_SSDM_CASCADING
                                             ? "cascading_allreduce: only ring schedules are supported"
                                             : "sum_ssdm_allreduce: only ring schedules are supported");
    if (ctx->G != 1 || ctx->ml != ctx->M)
        return fail(MARSIT_EUNSUPPORTED, "SSDM baselines run with every worker on one context");
    if (ctx->M > kSsMaxWorkers) return fail(MARSIT_EUNSUPPORTED, "SSDM baselines: at most 64 workers");
    for (uint32_t w = 0; w < ctx->M; ++w)
        if (!d_vectors[w]) return fail(MARSIT_EPARAM, "vectors: null pointer");
    CUDA_TRY(cudaSetDevice(ctx->device));
    const uint32_t M = ctx->M, S = ctx->S;
    const uint64_t L = ctx->L;

    // chain order of every segment, from the reduce deliveries
    // (allreduce.hpp:51-73): the receiver of each hop extends the sender's chain
    std::vector<std::vector<uint32_t>> chain(S);
    for (uint32_t k = 0; k < hs.steps(); ++k) {
        if (hs.phase[k] != 0) continue;
        for (uint32_t from = 0; from < M; ++from) {
            const uint32_t s = hs.segment[size_t(k) * M + from], to = hs.send_to[size_t(k) * M + from];
            if (chain[s].empty()) chain[s].push_back(from);
            if (chain[s].back() != from)
                return fail(MARSIT_EUNSUPPORTED, "SSDM baselines need linear reduce chains (ring)");
            chain[s].push_back(to);
        }
    }
    for (uint32_t s = 0; s < S; ++s)
        if (chain[s].size() != M) return fail(MARSIT_EUNSUPPORTED, "SSDM baselines: incomplete chain");

    if (!ctx->ssdm) ctx->ssdm.reset(new SsdmScratch());
    SsdmScratch& sc = *ctx->ssdm;
    const uint32_t wst = uint32_t(round_up(ceil_div(L, 32), 2));  // even: u64-compatible rows
    const uint32_t nb = uint32_t(ceil_div(L, kSsChunk));
    const size_t items = size_t(M) * S;
    if (!sc.chain) {
        CUDA_TRY(cudaMalloc(&sc.chain, size_t(S) * M));
        std::vector<uint8_t> flat(size_t(S) * M);
        for (uint32_t s = 0; s < S; ++s)
            for (uint32_t k = 0; k < M; ++k) flat[size_t(s) * M + k] = uint8_t(chain[s][k]);
        CUDA_TRY(cudaMemcpy(sc.chain, flat.data(), flat.size(), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMalloc(&sc.pk, sizeof(uint32_t) * items * wst));
        CUDA_TRY(cudaMalloc(&sc.norms, sizeof(double) * items));
        CUDA_TRY(cudaMalloc(&sc.partial, sizeof(double) * items * nb));
        CUDA_TRY(cudaMalloc(&sc.hist, sizeof(unsigned long long) * size_t(M) * (M + 1) * S));
    }
    if (mode == MARSIT_SSDM_CASCADING && !sc.acc)
        CUDA_TRY(cudaMalloc(&sc.acc, sizeof(double) * size_t(S) * L));

    SsdmParams p{};
    for (uint32_t w = 0; w < M; ++w) p.vec[w] = d_vectors[w];
    p.M = M;
    p.S = S;
    p.wst = wst;
    p.nb = nb;
    p.D = ctx->D;
    p.L = L;
    p.seed = seed;
    p.round = round;
    p.chain = sc.chain;
    p.mode = mode;
    p.key_w = -1;
    p.acc = sc.acc;
    p.pk = sc.pk;
    p.norms = sc.norms;
    p.partial = sc.partial;
    p.err = ctx->err;
    const bool want_hist =
        mode == MARSIT_SSDM_SUM && (bits_per_worker || reduce_bits || gather_bits || max_abs_per_step);
    marsit_status s = ctx->dtype == MARSIT_F32
                          ? launch_pipeline<float>(ctx, sc, p, mode, d_estimate, want_hist, st)
                          : launch_pipeline<double>(ctx, sc, p, mode, d_estimate, want_hist, st);
    if (s) return s;

    // BitsAccount (allreduce.hpp:232-235, 297-314): charged to the sender
    if (!(bits_per_worker || reduce_bits || gather_bits || max_abs_per_step)) return MARSIT_OK;
    const size_t H = size_t(M) * (M + 1);
    std::vector<unsigned long long> hist;
    std::vector<uint64_t> lensum(size_t(S) * M, 0);
    std::vector<int64_t> maxabs(size_t(S) * M, 0);
    if (want_hist) {
        hist.resize(H * S);
        CUDA_TRY(cudaMemcpyAsync(hist.data(), sc.hist, sizeof(unsigned long long) * hist.size(),
                                 cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        for (uint32_t sg = 0; sg < S; ++sg)
            for (uint32_t k = 0; k < M; ++k)
                for (uint32_t c = 0; c <= k + 1 && c <= M; ++c) {
                    const unsigned long long n = hist[sg * H + k * (M + 1) + c];
                    if (!n) continue;
                    const int64_t v = 2 * int64_t(c) - int64_t(k + 1);
                    lensum[size_t(sg) * M + k] += n * signed_sum_code_length(v);
                    maxabs[size_t(sg) * M + k] = std::max<int64_t>(maxabs[size_t(sg) * M + k],
                                                                   v < 0 ? -v : v);
                }
    }
    std::vector<uint64_t> bpw(M, 0);
    uint64_t rb = 0, gb = 0;
    std::vector<uint32_t> cnt(size_t(M) * S, 1);  // chain prefix length held per (worker, segment)
    for (uint32_t k = 0; k < hs.steps(); ++k) {
        const bool red = hs.phase[k] == 0;
        int64_t step_max = 0;
        for (uint32_t w = 0; w < M; ++w) {
            const uint32_t sg = hs.segment[size_t(k) * M + w];
            uint64_t b;
            if (mode == MARSIT_SSDM_CASCADING) {
                b = L + 32;  // bits.size() + 32-bit norm
            } else {
                const uint32_t pre = cnt[size_t(w) * S + sg];  // prefix length carried
                b = 32 + lensum[size_t(sg) * M + pre - 1];
                step_max = std::max(step_max, maxabs[size_t(sg) * M + pre - 1]);
            }
            bpw[w] += b;
            (red ? rb : gb) += b;
        }
        if (mode == MARSIT_SSDM_SUM && max_abs_per_step) max_abs_per_step[k] = step_max;
        for (uint32_t from = 0; from < M; ++from) {  // deliveries: counts follow the sums
            const uint32_t sg = hs.segment[size_t(k) * M + from], to = hs.send_to[size_t(k) * M + from];
            const uint32_t c_from = cnt[size_t(from) * S + sg];
            if (red)
                cnt[size_t(to) * S + sg] += c_from;
            else
                cnt[size_t(to) * S + sg] = c_from;
        }
    }
    if (bits_per_worker) std::copy(bpw.begin(), bpw.end(), bits_per_worker);
    if (reduce_bits) *reduce_bits = rb;
    if (gather_bits) *gather_bits = gb;
    return MARSIT_OK;
}

SsdmScratch::~SsdmScratch() {
    for (void* q : {(void*)acc, (void*)pk, (void*)norms, (void*)partial, (void*)hist, (void*)chain})
        if (q) cudaFree(q);
}

}  // namespace marsit_b200

using namespace marsit_b200;

extern "C" {

marsit_status marsit_ssdm_allreduce(marsit_ctx* ctx, int mode, uint64_t round, uint64_t seed,
                                    const void* const* d_vectors, void* d_estimate,
                                    uint64_t* bits_per_worker, uint64_t* reduce_bits,
                                    uint64_t* gather_bits, int64_t* max_abs_per_step,
                                    void* stream) {
    return ssdm_allreduce_impl(ctx, mode, round, seed, d_vectors, d_estimate, bits_per_worker,
                               reduce_bits, gather_bits, max_abs_per_step,
                               static_cast<cudaStream_t>(stream));
}

marsit_status marsit_ssdm_compress(const void* d_v, uint64_t len, marsit_dtype dtype, uint64_t seed,
                                   uint64_t worker, uint64_t round, uint64_t segment,
                                   uint64_t* d_bits, double* norm_out, void* stream) {
    if (!d_v || !d_bits || !norm_out) return fail(MARSIT_EPARAM, "null argument");
    if (len == 0) return fail(MARSIT_EPARAM, "DenseVector: dimension must be >= 1");
    if (dtype != MARSIT_F32 && dtype != MARSIT_F64) return fail(MARSIT_EPARAM, "unknown dtype");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SsdmParams p{};
    p.vec[0] = d_v;
    p.M = 1;
    p.S = 1;
    p.D = len;
    p.L = len;
    p.wst = uint32_t(round_up(ceil_div(len, 32), 2));
    p.nb = uint32_t(ceil_div(len, kSsChunk));
    p.seed = seed;
    p.round = round;
    p.key_w = int64_t(worker);
    p.key_s = int64_t(segment);
    p.pk = reinterpret_cast<uint32_t*>(d_bits);  // two u32 words per LE u64 word
    struct Scratch {
        void* q = nullptr;
        ~Scratch() {
            if (q) cudaFree(q);
        }
    } scr;
    CUDA_TRY(cudaMalloc(&scr.q, sizeof(double) * (p.nb + 1) + sizeof(int)));
    p.norms = static_cast<double*>(scr.q);
    p.partial = p.norms + 1;
    p.err = reinterpret_cast<int*>(p.partial + p.nb);
    CUDA_TRY(cudaMemsetAsync(p.err, 0, sizeof(int), st));
    const dim3 blk(kSsThreads);
    const uint32_t cgx = compress_grid_x(p.wst);
    if (dtype == MARSIT_F32)
        ssdm_sumsq_raw_kernel<float, false><<<dim3(p.nb, 1), blk, 0, st>>>(p);
    else
        ssdm_sumsq_raw_kernel<double, false><<<dim3(p.nb, 1), blk, 0, st>>>(p);
    ssdm_norm_kernel<<<1, 32, 0, st>>>(p, 1);
    if (dtype == MARSIT_F32)
        ssdm_compress_kernel<float, false><<<dim3(cgx, 1), blk, 0, st>>>(p);
    else
        ssdm_compress_kernel<double, false><<<dim3(cgx, 1), blk, 0, st>>>(p);
    CUDA_TRY(cudaGetLastError());
    int bad = 0;
    CUDA_TRY(cudaMemcpyAsync(norm_out, p.norms, sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&bad, p.err, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (bad) return fail(MARSIT_ENONFINITE, "DenseVector: non-finite entry");
    return MARSIT_OK;
}

marsit_status marsit_ssdm_decompress(const uint64_t* d_bits, uint64_t len, double norm,
                                     marsit_dtype dtype, void* d_out, void* stream) {
    if (!d_bits || !d_out) return fail(MARSIT_EPARAM, "null argument");
    if (len == 0) return fail(MARSIT_EPARAM, "ssdm_decompress: empty packet");
    if (!(norm >= 0.0)) return fail(MARSIT_EPARAM, "ssdm_decompress: negative norm");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int grid = int(std::min<uint64_t>(ceil_div(len, 256), 148 * 8));
    const uint32_t* pk = reinterpret_cast<const uint32_t*>(d_bits);
    if (dtype == MARSIT_F32)
        ssdm_decompress_kernel<float><<<grid, 256, 0, st>>>(pk, len, norm, static_cast<float*>(d_out));
    else if (dtype == MARSIT_F64)
        ssdm_decompress_kernel<double><<<grid, 256, 0, st>>>(pk, len, norm, static_cast<double*>(d_out));
    else
        return fail(MARSIT_EPARAM, "unknown dtype");
    CUDA_TRY(cudaGetLastError());
    return MARSIT_OK;
}

}  // extern "C"
