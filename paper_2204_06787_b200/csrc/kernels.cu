// kernels.cu — sm_100a kernels of the Marsit sign round.
//
//   K1 extract_kernel   u = g + c, bit = (u >= 0), packed per segment
//                       (sync.hpp:71-76, segmentation.hpp:32-53, sign_vector.hpp:67-73)
//   C  coins_kernel     the coin bits of every merge stream, precomputed on a
//                       side stream (data independent; rng.hpp:28-54)
//   K2 merge_coop_kernel the segments' merge DAGs, cooperative: one grid
//                       barrier + prefix sum per merge step for the coin
//                       stream offsets, parallel bit deposit of the coins
//                       (merge.hpp:34-58, allreduce.hpp:148-189)
//   K3/K4 decode_kernel g_t = +-eta_s from the aggregate bits and the
//                       compensation update c' = u - g_t fused in one pass
//                       (sync.hpp:103-118, sign_vector.hpp:77-89)
//   export_bits_kernel  aggregate bits in the reference's whole-vector layout
//   dense kernels       allreduce_dense in schedule order (allreduce.hpp:98-130)
//
// All of it is HBM / integer-ALU work: no tensor cores are involved.  The
// streaming kernels use 128-bit coalesced loads, warp ballots for packing and
// grids sized to the SM count; the merge kernel keeps every segment in L2.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "rng.cuh"

namespace marsit_b200 {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// The same finalizer with the 64-bit shifts of the xor-shifts moved onto the
// FMA pipe: for the low word, (lo >> s) == mulhi(lo, 2^(32-s)) and the bits
// carried in from the high word are hi * 2^(32-s).  Bit-identical to mix64;
// it only balances the ALU / FMA pipes (each issues every other cycle).
__device__ __forceinline__ uint64_t mix64f(uint64_t z) {
    uint32_t lo = uint32_t(z), hi = uint32_t(z >> 32);
    xorshr_fma(lo, hi, 1u << 2);  // >> 30
    uint64_t t = ((uint64_t(hi) << 32) | lo) * 0xbf58476d1ce4e5b9ull;
    lo = uint32_t(t);
    hi = uint32_t(t >> 32);
    xorshr_fma(lo, hi, 1u << 5);  // >> 27
    t = ((uint64_t(hi) << 32) | lo) * 0x94d049bb133111ebull;
    lo = uint32_t(t);
    hi = uint32_t(t >> 32);
    xorshr_fma(lo, hi, 1u << 1);  // >> 31
    return (uint64_t(hi) << 32) | lo;
}

// ---------------------------------------------------------------------------
// Checked builds (MARSIT_CHECKED, tools/gpu/checked.sh; compute-sanitizer is
// closed on this GPU pool): jitter() sleeps a pseudo-random time at the
// synchronisation points of the merge kernels so that any missing ordering
// shows up as a result that differs from the oracle; BOUNDS(cond, err) latches
// err |= 8 (reported by marsit_ctx_check) instead of making an access whose
// index failed its bound.  Both compile to nothing in the product build.
// ---------------------------------------------------------------------------
#ifdef MARSIT_CHECKED
__device__ __forceinline__ void jitter(uint32_t a) {
    const uint64_t h = mix64((uint64_t(blockIdx.x) << 40) ^ (uint64_t(a) << 20) ^ uint64_t(clock64()));
    if ((h & 3u) == 0) __nanosleep(uint32_t(h >> 8) & 4095u);
}
#define MARSIT_BOUNDS_OK(cond, errp) ((cond) ? true : (((errp) ? atomicOr((errp), 8) : 0), false))
#else
__device__ __forceinline__ void jitter(uint32_t) {}
#define MARSIT_BOUNDS_OK(cond, errp) true
#endif

// ---------------------------------------------------------------------------
// Memory helpers
// ---------------------------------------------------------------------------
// Streaming 128-bit loads that do not allocate in L1 (each byte is read once).
__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p));
    return v;
}

// Coherent variant for data the same kernel overwrites (in-place compensation).
__device__ __forceinline__ float4 ld_stream_rw(const float4* p) {
    float4 v;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_stream_rw(const double2* p) {
    double2 v;
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p));
    return v;
}

template <typename T>
struct Quad {
    T v[4];
};

// Four consecutive elements; `p` is 4-element aligned (16 B for float, 32 B for double).
__device__ __forceinline__ Quad<float> load4(const float* p) {
    float4 a = ld_stream(reinterpret_cast<const float4*>(p));
    return {{a.x, a.y, a.z, a.w}};
}
__device__ __forceinline__ Quad<double> load4(const double* p) {
    double2 a = ld_stream(reinterpret_cast<const double2*>(p));
    double2 b = ld_stream(reinterpret_cast<const double2*>(p) + 1);
    return {{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ Quad<float> load4_rw(const float* p) {
    float4 a = ld_stream_rw(reinterpret_cast<const float4*>(p));
    return {{a.x, a.y, a.z, a.w}};
}
__device__ __forceinline__ Quad<double> load4_rw(const double* p) {
    double2 a = ld_stream_rw(reinterpret_cast<const double2*>(p));
    double2 b = ld_stream_rw(reinterpret_cast<const double2*>(p) + 1);
    return {{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ void store4(float* p, const Quad<float>& q) {
    *reinterpret_cast<float4*>(p) = make_float4(q.v[0], q.v[1], q.v[2], q.v[3]);
}
__device__ __forceinline__ void store4(double* p, const Quad<double>& q) {
    reinterpret_cast<double2*>(p)[0] = make_double2(q.v[0], q.v[1]);
    reinterpret_cast<double2*>(p)[1] = make_double2(q.v[2], q.v[3]);
}

__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

template <typename T>
__device__ __forceinline__ bool finite(T x) {
    return isfinite(x);
}

// Word holding the sign bit in its top byte.
__device__ __forceinline__ uint32_t sign_word(float x) { return __float_as_uint(x); }
__device__ __forceinline__ uint32_t sign_word(double x) { return uint32_t(__double2hiint(x)); }

// bit k = (v_k >= 0) for values whose -0.0 has been folded to +0.0: the four
// sign bytes are gathered with byte permutes, inverted, and compacted to a
// nibble by one multiply-high (bits 7/15/23/31 -> 32/33/34/35).
template <typename T>
__device__ __forceinline__ uint32_t sign_nibble(T a, T b, T c, T d) {
    const uint32_t r1 = __byte_perm(sign_word(a), sign_word(b), 0x0073);
    const uint32_t r2 = __byte_perm(sign_word(c), sign_word(d), 0x7300);
    const uint32_t r = __byte_perm(r1, r2, 0x7610);
    return __umulhi(~r & 0x80808080u, 0x02040810u) & 0xFu;
}


// ---------------------------------------------------------------------------
// K1: error-compensated sign extraction.
//
// A warp task is 512 consecutive coordinates of one (worker, segment):
// 16 packed u32 words.  Vector path (L % 4 == 0): lane l holds coordinates
// 4l..4l+3 of each 128-coordinate sub-chunk (one 128-bit load per operand),
// packs them into a nibble, and 8-lane OR-shuffles assemble the words.
// Scalar path: lane l holds coordinate 32t + l of word t and a ballot is the
// word.  Coordinates j >= L are storage padding (bit
// 0, sign_vector.hpp:15-18); s*L + j >= D is value padding, 0.0, bit 1
// (segmentation.hpp:45-49 + sign_vector.hpp:70).
// ---------------------------------------------------------------------------
template <typename T, bool VEC>
__global__ void __launch_bounds__(kStreamThreads, sizeof(T) == 4 ? (VEC ? 4 : 3) : 2) extract_kernel(const StreamParams<T> p) {
    const int lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (kStreamThreads / 32);
    const uint32_t tasks_per_seg = (p.words_proc + kTaskWords - 1) / kTaskWords;
    const uint64_t n_tasks = uint64_t(tasks_per_seg) * p.n_proc * p.ml;
    bool bad = false;
    T fin = T(0);  // stays 0 unless some u = g + c is not finite
    for (uint64_t task = blockIdx.x * (kStreamThreads / 32) + (threadIdx.x >> 5); task < n_tasks;
         task += warps) {
        // p.reverse: walk the tasks from the end (see StreamParams::reverse)
        const uint64_t tk = p.reverse ? n_tasks - 1 - task : task;
        const uint32_t q = uint32_t(tk % tasks_per_seg);
        const uint64_t rest = tk / tasks_per_seg;
        const uint32_t s = p.seg0 + uint32_t(rest % p.n_proc);
        const uint32_t wl = uint32_t(rest / p.n_proc);
        const T* __restrict__ g = p.g[wl];
        const T* __restrict__ c = p.c[wl];
        const uint64_t seg0 = uint64_t(s) * p.seg_len;  // first global coordinate
        const uint64_t j0 = uint64_t(q) * (kTaskWords * 32);
        uint32_t word = 0;  // scalar path: lane t < 16 ends up holding word t of the task
        if (VEC) {
            // full task: every coordinate is real (no storage or value padding)
            const bool full = j0 + kTaskWords * 32 <= p.seg_len && seg0 + j0 + kTaskWords * 32 <= p.dim;
            Quad<T> gv[4], cv[4];
#pragma unroll
            for (int sub = 0; sub < 4; ++sub) {
                const uint64_t j = j0 + sub * 128 + lane * 4;
                const uint64_t gi = seg0 + j;
                if (full || (j < p.seg_len && gi + 3 < p.dim)) {
                    gv[sub] = load4(g + gi);
                    cv[sub] = load4(c + gi);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const bool in = (j + k < p.seg_len) && (gi + k < p.dim);
                        gv[sub].v[k] = in ? g[gi + k] : T(0);
                        cv[sub].v[k] = in ? c[gi + k] : T(0);
                    }
                }
            }
            // lane l's nibble = bits of coordinates 4l..4l+3; word q of the
            // sub-chunk is the concatenation of lanes 8q..8q+7's nibbles: an
            // OR-reduction over aligned groups of 8 lanes (3 shuffles).
#pragma unroll
            for (int sub = 0; sub < 4; ++sub) {
                T u[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    // + 0 turns -0.0 (only from -0.0 + -0.0) into +0.0, so the
                    // sign bit alone decides (u >= 0), sign_vector.hpp:70
                    u[k] = add_rn(add_rn(gv[sub].v[k], cv[sub].v[k]), T(0));
                    fin = fma_rn(u[k], T(0), fin);  // NaN iff some u is inf/NaN
                }
                uint32_t nib = sign_nibble(u[0], u[1], u[2], u[3]);
                if (!full) {
                    const uint64_t j = j0 + sub * 128 + lane * 4;
                    const uint64_t valid = j >= p.seg_len ? 0 : p.seg_len - j;  // storage padding -> 0
                    if (valid < 4) nib &= (1u << valid) - 1u;
                }
                uint32_t v = nib << ((lane & 7) * 4);
                v |= __shfl_xor_sync(kFull, v, 1);
                v |= __shfl_xor_sync(kFull, v, 2);
                v |= __shfl_xor_sync(kFull, v, 4);
                const uint32_t wi = q * kTaskWords + sub * 4 + (lane >> 3);
                if ((lane & 7) == 0 && wi < p.words_proc)
                    p.bits[(uint64_t(s) * p.ml + wl) * p.wst + wi] = v;
            }
        } else {
            // any segment length: lane-contiguous (coalesced) loads, all 32 of a
            // lane issued before the first is used
            // element t of this lane is coordinate j0 + 32 t + lane: real below
            // n_real, value padding (0.0, packs to 1) below n_seg, storage padding above
            const uint64_t first = j0 + lane;
            const uint64_t lim = p.dim > seg0 ? (p.dim - seg0 < p.seg_len ? p.dim - seg0 : p.seg_len) : 0;
            const int n_real = lim > first ? (lim - first > 4096 ? 4096 : int(lim - first)) : 0;
            const int n_seg = p.seg_len > first ? (p.seg_len - first > 4096 ? 4096 : int(p.seg_len - first)) : 0;
            const T* gb = g + seg0 + first;
            const T* cb = c + seg0 + first;
            T gv[kTaskWords], cv[kTaskWords];
#pragma unroll
            for (int t = 0; t < kTaskWords; ++t) {
                gv[t] = t * 32 < n_real ? gb[t * 32] : T(0);
                cv[t] = t * 32 < n_real ? cb[t * 32] : T(0);
            }
#pragma unroll
            for (int t = 0; t < kTaskWords; ++t) {
                const T u = add_rn(gv[t], cv[t]);
                fin = fma_rn(u, T(0), fin);  // NaN iff some u is inf/NaN (any non-finite g or c)
                const uint32_t w = __ballot_sync(kFull, t * 32 < n_seg && u >= T(0));
                if (lane == t) word = w;
            }
        }
        if (!VEC) {
            const uint32_t wi = q * kTaskWords + lane;
            if (lane < kTaskWords && wi < p.words_proc)
                p.bits[(uint64_t(s) * p.ml + wl) * p.wst + wi] = word;
        }
    }
    bad |= !(fin == fin);
    if (__any_sync(kFull, bad) && lane == 0) atomicOr(p.err, 1);
}

// ---------------------------------------------------------------------------
// K3+K4: decode the aggregate to +-eta_s and update the compensation,
// c' = (g + c) - g_t, in the same pass (sync.hpp:113-118).  Same task
// decomposition as K1, so each sub-chunk's bits are 4 aligned words.
// ---------------------------------------------------------------------------
// Aggregate row of segment s: local, or (P2P transport) the owner's buffer.
template <typename T>
__device__ __forceinline__ const uint32_t* agg_row(const StreamParams<T>& p, uint32_t s) {
    const uint32_t* base = p.agg_peers ? p.agg_peers[s / p.s_own] : p.agg;
    return base + uint64_t(s) * p.wsa;
}

// XU: the replica update x -= g_t is fused (its quads are loaded with g and c,
// so the read-modify-write of x is not a dependent round trip per sub-chunk)
template <typename T, bool VEC, bool XU>
__global__ void __launch_bounds__(kStreamThreads,
                                  (sizeof(T) == 4 && !XU) ? 3 : ((sizeof(T) == 8 && XU) ? 1 : 2))
    decode_kernel(const StreamParams<T> p) {
    const int lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (kStreamThreads / 32);
    const uint32_t tasks_per_seg = (p.words_proc + kTaskWords - 1) / kTaskWords;
    const uint64_t n_tasks = uint64_t(tasks_per_seg) * p.n_proc * p.ml;
    const T eta = p.eta;
    for (uint64_t task = blockIdx.x * (kStreamThreads / 32) + (threadIdx.x >> 5); task < n_tasks;
         task += warps) {
        // p.reverse: walk the tasks from the end (see StreamParams::reverse)
        const uint64_t tk = p.reverse ? n_tasks - 1 - task : task;
        const uint32_t q = uint32_t(tk % tasks_per_seg);
        const uint64_t rest = tk / tasks_per_seg;
        const uint32_t s = p.seg0 + uint32_t(rest % p.n_proc);
        const uint32_t wl = uint32_t(rest / p.n_proc);
        const T* __restrict__ g = p.g[wl];
        const T* c = p.c[wl];  // may alias c_out (in-place update): no __restrict__
        T* co = p.c_out[wl];
        T* upd = (wl == 0) ? p.update : nullptr;
        T* xp = p.x[wl];  // replica parameters (optional)
        const uint64_t seg0 = uint64_t(s) * p.seg_len;
        const uint64_t j0 = uint64_t(q) * (kTaskWords * 32);
        const uint32_t* aw = agg_row(p, s) + q * kTaskWords;
        if (VEC) {
            Quad<T> gv[4], cv[4], xv[XU ? 4 : 1];
            uint32_t nib[4];
#pragma unroll
            for (int sub = 0; sub < 4; ++sub) {
                const uint64_t j = j0 + sub * 128 + lane * 4;
                const uint64_t gi = seg0 + j;
                const uint32_t wi = q * kTaskWords + sub * 4 + (lane >> 3);
                const uint32_t word = (wi < p.words_proc) ? __ldg(aw + sub * 4 + (lane >> 3)) : 0u;
                nib[sub] = (word >> ((lane & 7) * 4)) & 0xFu;
                if (j < p.seg_len && gi + 3 < p.dim) {
                    gv[sub] = load4(g + gi);
                    cv[sub] = load4_rw(c + gi);
                    if (XU && xp) xv[XU ? sub : 0] = load4_rw(xp + gi);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const bool in = (j + k < p.seg_len) && (gi + k < p.dim);
                        gv[sub].v[k] = in ? g[gi + k] : T(0);
                        cv[sub].v[k] = in ? c[gi + k] : T(0);
                    }
                }
            }
#pragma unroll
            for (int sub = 0; sub < 4; ++sub) {
                const uint64_t j = j0 + sub * 128 + lane * 4;
                const uint64_t gi = seg0 + j;
                Quad<T> out, up;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const T gt = ((nib[sub] >> k) & 1u) ? eta : -eta;
                    out.v[k] = sub_rn(add_rn(gv[sub].v[k], cv[sub].v[k]), gt);
                    up.v[k] = gt;
                }
                if (j < p.seg_len && gi + 3 < p.dim) {
                    store4(co + gi, out);
                    if (upd) store4(upd + gi, up);
                    if (XU && xp) {
                        Quad<T>& xq = xv[XU ? sub : 0];
#pragma unroll
                        for (int k = 0; k < 4; ++k) xq.v[k] = sub_rn(xq.v[k], up.v[k]);
                        store4(xp + gi, xq);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if ((j + k < p.seg_len) && (gi + k < p.dim)) {
                            co[gi + k] = out.v[k];
                            if (upd) upd[gi + k] = up.v[k];
                            if (XU && xp) xp[gi + k] = sub_rn(xp[gi + k], up.v[k]);
                        }
                }
            }
        } else {
            // any segment length: lane-contiguous (coalesced) loads, all issued
            // before the first is used
            // element t of this lane is coordinate j0 + 32 t + lane (real below n_real)
            const uint64_t first = j0 + lane;
            const uint64_t lim = p.dim > seg0 ? (p.dim - seg0 < p.seg_len ? p.dim - seg0 : p.seg_len) : 0;
            const int n_real = lim > first ? (lim - first > 4096 ? 4096 : int(lim - first)) : 0;
            const uint64_t off = seg0 + first;
            T gv[kTaskWords], cv[kTaskWords], xv[XU ? kTaskWords : 1];
            // the task's 16 aggregate words: one load per lane, then broadcast
            const uint32_t wmine =
                (lane < kTaskWords && q * kTaskWords + lane < p.words_proc) ? __ldg(aw + lane) : 0u;
#pragma unroll
            for (int t = 0; t < kTaskWords; ++t) {
                gv[t] = t * 32 < n_real ? g[off + t * 32] : T(0);
                cv[t] = t * 32 < n_real ? c[off + t * 32] : T(0);
                if (XU) xv[XU ? t : 0] = (xp && t * 32 < n_real) ? xp[off + t * 32] : T(0);
            }
#pragma unroll
            for (int t = 0; t < kTaskWords; ++t) {
                const uint32_t wv = __shfl_sync(kFull, wmine, t);
                if (t * 32 < n_real) {
                    const T gt = ((wv >> lane) & 1u) ? eta : -eta;
                    co[off + t * 32] = sub_rn(add_rn(gv[t], cv[t]), gt);
                    if (upd) upd[off + t * 32] = gt;
                    if (XU && xp) xp[off + t * 32] = sub_rn(xv[XU ? t : 0], gt);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K3/K4 with the round's matching count fused in (analysis.hpp:244-253 on the
// input mean of trainer.hpp:241-251): every local worker of one coordinate
// block in the same task, so the fp64 sum of u_w = g_w + c_w in worker order
// is formed in registers while the decode reads g and c anyway — no extra
// HBM traffic.  matches += [aggregate bit == (sum / M >= 0)] over the D
// coordinates.  Needs every worker of the job local (p.ml == M).
// ---------------------------------------------------------------------------
// (sum / M >= 0) of the worker-order fp64 sum of u = g + c (trainer.hpp:249):
// for fp32 inputs every u and hence the exact sum is a multiple of 2^-149, so
// a negative rounded fp64 sum is at most -2^-149 and sum / M cannot round to
// -0: the sign of the sum decides without the division; fp64 u can be
// subnormal, so a negative sum still takes the literal division.
template <typename T>
__device__ __forceinline__ bool mean_nonneg(double sum, double m) {
    if (sum >= 0.0) return true;
    return sizeof(T) == 8 && __ddiv_rn(sum, m) >= 0.0;
}

// u in fp64 as the trainer forms it (add(g, c) on doubles, trainer.hpp:247):
// for fp32 inputs the exact sum of the two fp32 values, not the fp32-rounded u
// of the compensation update (the two can differ in the sign of the mean).
__device__ __forceinline__ double u64_of(float g, float c) { return __dadd_rn(double(g), double(c)); }
__device__ __forceinline__ double u64_of(double g, double c) { return __dadd_rn(g, c); }

template <typename T>
__device__ __forceinline__ void decode_one(const StreamParams<T>& p, uint32_t wl, uint64_t gi,
                                           T gt, double& u64) {
    const T g = p.g[wl][gi], c = p.c[wl][gi];
    const T u = add_rn(g, c);
    u64 = u64_of(g, c);
    p.c_out[wl][gi] = sub_rn(u, gt);
    if (wl == 0 && p.update) p.update[gi] = gt;
    if (p.x[wl]) p.x[wl][gi] = sub_rn(p.x[wl][gi], gt);
}

template <typename T, bool VEC>
// register cap: two CTAs per SM leave room for the coin precompute
// of the next round, which runs beside the decode on the side stream
__global__ void __maxnreg__(sizeof(T) == 4 ? 80 : 128) decode_stats_kernel(const StreamParams<T> p) {
    const int lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (kStreamThreads / 32);
    const uint32_t tasks_per_seg = (p.words_proc + kTaskWords - 1) / kTaskWords;
    const uint64_t n_tasks = uint64_t(tasks_per_seg) * p.n_proc;
    const T eta = p.eta;
    const double wm = double(p.n_workers);  // the mean divides by M (trainer.hpp:249)
    uint64_t matches = 0;
    for (uint64_t task = blockIdx.x * (kStreamThreads / 32) + (threadIdx.x >> 5); task < n_tasks;
         task += warps) {
        const uint32_t q = uint32_t(task % tasks_per_seg);
        const uint32_t s = p.seg0 + uint32_t(task / tasks_per_seg);
        const uint64_t seg0 = uint64_t(s) * p.seg_len;
        const uint64_t j0 = uint64_t(q) * (kTaskWords * 32);
        const uint32_t* aw = agg_row(p, s) + q * kTaskWords;
        // full task: all 512 coordinates real, 16-byte aligned quads
        const bool full = VEC && j0 + kTaskWords * 32 <= p.seg_len &&
                          seg0 + j0 + kTaskWords * 32 <= p.dim;
        if (full) {
            // two passes of two sub-chunks: 8 fp64 sums, and worker w + 1's
            // loads in flight while worker w is computed (the buffers of
            // different workers never overlap)
#pragma unroll 1
            for (int half = 0; half < 2; ++half) {
                uint32_t nib[2];
                double sum[2][4];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int sub = 2 * half + h;
                    const uint32_t word = __ldg(aw + sub * 4 + (lane >> 3));
                    nib[h] = (word >> ((lane & 7) * 4)) & 0xFu;
#pragma unroll
                    for (int k = 0; k < 4; ++k) sum[h][k] = 0.0;
                }
                const uint64_t gb = seg0 + j0 + half * 256 + lane * 4;  // + h * 128
                Quad<T> gv[2], cv[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    gv[h] = load4(p.g[0] + gb + h * 128);
                    cv[h] = load4_rw(p.c[0] + gb + h * 128);
                }
                for (uint32_t wl = 0; wl < p.ml; ++wl) {
                    Quad<T> gn[2], cn[2];
                    if (wl + 1 < p.ml) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            gn[h] = load4(p.g[wl + 1] + gb + h * 128);
                            cn[h] = load4_rw(p.c[wl + 1] + gb + h * 128);
                        }
                    }
                    T* xp = p.x[wl];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint64_t gi = gb + h * 128;
                        Quad<T> out, up;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const T gt = ((nib[h] >> k) & 1u) ? eta : -eta;
                            const T u = add_rn(gv[h].v[k], cv[h].v[k]);
                            sum[h][k] = __dadd_rn(sum[h][k], u64_of(gv[h].v[k], cv[h].v[k]));
                            out.v[k] = sub_rn(u, gt);
                            up.v[k] = gt;
                        }
                        store4(p.c_out[wl] + gi, out);
                        if (wl == 0 && p.update) store4(p.update + gi, up);
                        if (xp) {
                            Quad<T> xv = load4_rw(xp + gi);
#pragma unroll
                            for (int k = 0; k < 4; ++k) xv.v[k] = sub_rn(xv.v[k], up.v[k]);
                            store4(xp + gi, xv);
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        gv[h] = gn[h];
                        cv[h] = cn[h];
                    }
                }
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        matches += (((nib[h] >> k) & 1u) != 0) == mean_nonneg<T>(sum[h][k], wm);
            }
        } else {
            // ragged task (segment / vector tail or unaligned buffers): per coordinate
#pragma unroll 1
            for (int t = 0; t < kTaskWords; ++t) {
                const uint64_t j = j0 + t * 32 + lane;
                const uint64_t gi = seg0 + j;
                if (j < p.seg_len && gi < p.dim) {
                    const uint32_t bit = (__ldg(aw + t) >> lane) & 1u;
                    const T gt = bit ? eta : -eta;
                    double sum = 0.0;
                    for (uint32_t wl = 0; wl < p.ml; ++wl) {
                        double u;
                        decode_one(p, wl, gi, gt, u);
                        sum = __dadd_rn(sum, u);
                    }
                    matches += (bit != 0) == mean_nonneg<T>(sum, wm);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) matches += __shfl_xor_sync(kFull, matches, o);
    if (lane == 0 && matches) atomicAdd(p.matches, (unsigned long long)matches);
}

// ---------------------------------------------------------------------------
// K2: the merge DAG of every owned segment (merge.hpp:34-58 per merge).
//
// Per merge: d = r ^ l; the draw index of every disagreeing coordinate is
//   base(stream) + exclusive_prefix(popcount(d)) over the segment;
// the coin is (mix(key + (n+1)γ) >> 11) < ceil(p·2^53) (precomputed bit
// streams, coins_kernel) and out = r ^ (d & ~coin).  See merge_coop_kernel.
// ---------------------------------------------------------------------------
// Coins of one packed word: for each set bit of `d` (ascending), draw
// mix(z), z += gamma; keep the received bit where the draw is below th.
__device__ __forceinline__ uint32_t coin_word(uint32_t d, uint64_t& z, uint64_t th) {
    uint32_t keep = 0;
    while (d) {
        const uint32_t lsb = d & (0u - d);
        d ^= lsb;
        const uint64_t x = mix64f(z);
        z += kGamma;
        if (x < th) keep |= lsb;
    }
    return keep;
}

// K2: the merge DAG, cooperative.  One CTA per tile of 256 x WPT packed words;
// the tiles of one launch ("part": tiles [part_tile0, part_tile0+part_tiles)
// of every owned segment) are co-resident (cooperative launch).  Merge step
// k of the current plan stage: each tile publishes popcount(r ^ l), one
// grid-wide barrier, then every tile sums the published counts of the
// tiles before it (its exclusive draw offset; earlier parts contribute their
// totals), reads its precomputed coin bits and deposits them onto the set
// bits of r ^ l.  A continuation merge (torus stage 2) starts its stream
// after the complete draw total of the merge it continues (previous stage).
__device__ __forceinline__ uint32_t shl_fma(uint32_t x, uint32_t s) { return x * (1u << s); }
// Parallel bit deposit (PDEP): the low popcount(m) bits of x are placed,
// in order, at the set bits of m.  Byte-parallel form of the branch-free
// "expand" of Hacker's Delight §7-6: the four bytes of m are expanded side
// by side in three parallel-suffix rounds (shifts masked to stay inside a
// byte), and byte b of x is first fed from bit popcount(m's lower bytes) of
// x (an exclusive prefix of the byte popcounts, one multiply).  Split in
// two: the masks depend only on m (the disagreement word, known before the
// grid barrier, so they are formed while the other tiles arrive); the moves
// of x need the coin window (known after it).  expand_apply(x, masks(m)) & m
// == pdep(x, m) (checked against a bit-serial pdep on 200k random words and
// every byte pattern).
__device__ __forceinline__ void expand_masks(uint32_t m, uint32_t (&mv)[4]) {
    uint32_t pc = m - ((m >> 1) & 0x55555555u);
    pc = (pc & 0x33333333u) + ((pc >> 2) & 0x33333333u);
    pc = (pc + (pc >> 4)) & 0x0F0F0F0Fu;
    mv[3] = pc * 0x01010100u;  // byte b: popcount of bytes < b
    uint32_t mk = shl_fma(~m, 1) & 0xFEFEFEFEu;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        uint32_t mp = mk ^ (shl_fma(mk, 1) & 0xFEFEFEFEu);
        mp ^= shl_fma(mp, 2) & 0xFCFCFCFCu;
        mp ^= shl_fma(mp, 4) & 0xF0F0F0F0u;
        const uint32_t v = mp & m;
        m = (m ^ v) | (v >> (1 << i));
        mk &= ~mp;
        mv[i] = v;
    }
}
__device__ __forceinline__ uint32_t expand_apply(uint32_t x, const uint32_t (&mv)[4]) {
    const uint32_t ex = mv[3];
    uint32_t t = __byte_perm(x, x >> ((ex >> 8) & 0xFFu), 0x0040);
    t = __byte_perm(t, x >> ((ex >> 16) & 0xFFu), 0x0410);
    t = __byte_perm(t, x >> (ex >> 24), 0x4210);
    t = (t & ~mv[2]) | (shl_fma(t, 4) & mv[2]);
    t = (t & ~mv[1]) | (shl_fma(t, 2) & mv[1]);
    t = (t & ~mv[0]) | (shl_fma(t, 1) & mv[0]);
    return t;  // bits outside m are don't-care (the caller masks with d)
}

template <int WPT>
__device__ __forceinline__ void load_words(const uint32_t* p, uint32_t (&v)[WPT]) {
    if constexpr (WPT >= 4) {
#pragma unroll
        for (int q = 0; q < WPT / 4; ++q) {
            const uint4 x = __ldcg(reinterpret_cast<const uint4*>(p) + q);
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = x.z;
            v[4 * q + 3] = x.w;
        }
    } else if constexpr (WPT == 2) {
        const uint2 x = __ldcg(reinterpret_cast<const uint2*>(p));
        v[0] = x.x;
        v[1] = x.y;
    } else {
        v[0] = __ldcg(p);
    }
}

#if defined(MARSIT_COOP_PROF) || defined(MARSIT_FUSED_PROF)
}  // namespace
__device__ unsigned long long g_coop_prof[16];
namespace {
__device__ __forceinline__ uint64_t gtime_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define COOP_T(v) const uint64_t v = (threadIdx.x == 0 && blockIdx.x == 0) ? gtime_ns() : 0
#define COOP_ADD(slot_, val_) if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(&g_coop_prof[slot_], (unsigned long long)(val_))
#else
#define COOP_T(v)
#define COOP_ADD(i, x)
#endif

// Barrier over the n co-resident CTAs of one segment (the sense-reversing
// counter of cooperative groups' grid barrier on a per-segment word: the
// master adds 2^31 - (n - 1), the others 1, so every barrier flips bit 31
// and leaves the low bits at 0 for the next one).
__device__ __forceinline__ unsigned seg_barrier_arrive(unsigned* bar, bool master, unsigned n) {
    __syncthreads();
    unsigned old = 0;
    if (threadIdx.x == 0) {
        const unsigned nb = master ? 0x80000000u - (n - 1) : 1u;
        asm volatile("atom.add.release.gpu.u32 %0,[%1],%2;" : "=r"(old) : "l"(bar), "r"(nb) : "memory");
    }
    return old;
}
__device__ __forceinline__ void seg_barrier_wait(unsigned* bar, unsigned old) {
    if (threadIdx.x == 0) {
        unsigned cur;
        do {
            asm volatile("ld.acquire.gpu.u32 %0,[%1];" : "=r"(cur) : "l"(bar) : "memory");
        } while (((old ^ cur) & 0x80000000u) == 0);
    }
    __syncthreads();
}

template <int WPT>
__global__ void __launch_bounds__(kMergeThreads, WPT >= 12 ? 2 : (WPT >= 8 ? 3 : 4))
    merge_coop_kernel(const CoopParams p) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ uint32_t cslots[];  // [max_slots][WPT][kMergeThreads], then the
                                          // deposit masks [WPT][4][kMergeThreads]
    uint32_t* cmask = cslots + size_t(p.max_slots) * WPT * kMergeThreads;
    __shared__ uint32_t s_warp[kMergeThreads / 32];
    __shared__ uint64_t s_acc[kMergeThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t T = gridDim.x;  // CTAs in this launch
    const uint32_t vs = blockIdx.x / p.part_tiles, lt = blockIdx.x % p.part_tiles;
    const uint32_t sl = p.seg_lo + vs / p.n_lanes, chain = vs % p.n_lanes;
    const uint32_t tile = p.part_tile0 + lt;
    // a tile is tile_words (<= 256 * WPT, multiple of 4) consecutive words
    const uint32_t w0 = tile * p.tile_words + tid * WPT;
    const bool active = tile < p.tiles_per_seg && tid * WPT < p.tile_words && w0 < p.words_proc;
    // valid bits of my words: all 32 while rem >= 32 (bits beyond L stay 0)
    const int64_t rem0 = int64_t(p.seg_bits) - int64_t(w0) * 32;
    auto vmask = [&](int j) -> uint32_t {
        const int64_t rem = rem0 - 32 * j;
        return rem >= 32 ? kFull : (rem <= 0 ? 0u : ((1u << rem) - 1u));
    };
    const uint32_t mb = p.seg_begin[sl];
    const uint32_t* lb = p.lane_begin + (size_t(sl) * p.n_stages + p.stage) * (kMaxLanes + 1) + chain;
    const uint32_t kb = lb[0];
    const uint32_t nm = lb[1] - kb;
    const uint32_t sg = p.s_first + sl;
    // The stage's merge descriptors and the data-independent part of each
    // merge's draw base (draws before this round + earlier launch parts +
    // the continued stream's total, all written by earlier launches) are
    // staged in shared memory once, so no merge step starts with a dependent
    // global load (kMaxCachedMerges bounds the cache; longer stages read the
    // descriptors from global memory).
    __shared__ DevMerge s_m[kMaxCachedMerges];
    __shared__ uint64_t s_sbase[kMaxCachedMerges];
    __shared__ uint32_t s_valid[kMaxCachedMerges];
    const bool cached = nm <= kMaxCachedMerges;
    auto static_base = [&](uint32_t mi, const DevMerge& m) -> uint64_t {
        const uint32_t nmerges = p.n_merges;
        uint64_t base = m.base_add;  // draws of this stream before this merge
        for (uint32_t q = 0; q < p.part; ++q)  // earlier parts (earlier launches)
            base += __ldcg(p.part_totals + uint64_t(q) * nmerges + mb + mi);
        for (int32_t src = m.offset_src; src >= 0;) {  // continued stream (earlier stage)
            const DevMerge& pm = p.merges[mb + src];
            for (uint32_t q = 0; q < p.n_parts; ++q)
                base += __ldcg(p.part_totals + uint64_t(q) * nmerges + mb + src);
            base += pm.base_add;
            src = pm.offset_src;
        }
        return base;
    };
    if (cached && tid < nm) {
        const DevMerge m = p.merges[mb + kb + tid];
        s_m[tid] = m;
        s_sbase[tid] = static_base(kb + tid, m);
        s_valid[tid] = p.coin_valid ? p.coin_valid[mb + kb + tid] : 0u;
    }
    __syncthreads();
    auto merge_at = [&](uint32_t k) -> DevMerge { return cached ? s_m[k] : p.merges[mb + kb + k]; };
    // a thread's last words may pass the segment's end (WPT = 12): those are
    // loaded as 0 and never stored
    const bool tail = w0 + WPT > p.words_proc;
    auto load_row = [&](const uint32_t* row, uint32_t (&v)[WPT]) {
        if (!tail) {
            load_words<WPT>(row + w0, v);
        } else {
#pragma unroll
            for (int j = 0; j < WPT; ++j) v[j] = (w0 + j < p.words_proc) ? __ldcg(row + w0 + j) : 0u;
        }
    };
    auto load_src = [&](uint16_t src, uint32_t (&v)[WPT]) {
        const uint32_t idx = src & 0x3FFFu;
        if (!active) {
#pragma unroll
            for (int j = 0; j < WPT; ++j) v[j] = 0;
        } else if ((src & 0xC000u) == kSrcLeaf) {
            if (p.peer_bits)  // P2P: the source rank's buffer, over NVLink
                load_row(p.peer_bits[idx / p.ml] + (uint64_t(sg) * p.ml + idx % p.ml) * p.wst, v);
            else
                load_row(p.leaves + (uint64_t((idx / p.ml) * p.n_seg + sl) * p.ml + idx % p.ml) * p.wst,
                         v);
        } else if ((src & 0xC000u) == kSrcSlot) {
#pragma unroll
            for (int j = 0; j < WPT; ++j) v[j] = cslots[(idx * WPT + j) * kMergeThreads + tid];
        } else {
            load_row(p.gnodes + (uint64_t(sl) * p.gmax + idx) * p.wst, v);
        }
    };
    // the local operand of the next merge is prefetched when it is a leaf
    // (ring / torus: the received operand is the running aggregate)
    uint32_t pl[WPT];
    if (nm > 0) {
        const DevMerge m0 = merge_at(0);
        if ((m0.local_src & 0xC000u) == kSrcLeaf) load_src(m0.local_src, pl);
    }
    uint32_t r[WPT], d[WPT];
    for (uint32_t k = 0; k < p.k_steps; ++k) {
        COOP_T(t0);
        const bool live = k < nm;
        const uint32_t mi = kb + k;  // merge index within the segment
        DevMerge m{};
        uint32_t cnt = 0;
        if (live) {
            m = merge_at(k);
            load_src(m.recv_src, r);
            if ((m.local_src & 0xC000u) == kSrcLeaf) {
#pragma unroll
                for (int j = 0; j < WPT; ++j) d[j] = (r[j] ^ pl[j]) & vmask(j);
            } else {
                load_src(m.local_src, d);
#pragma unroll
                for (int j = 0; j < WPT; ++j) d[j] = (r[j] ^ d[j]) & vmask(j);
            }
            if (k + 1 < nm) {
                const DevMerge mn = merge_at(k + 1);
                if ((mn.local_src & 0xC000u) == kSrcLeaf) load_src(mn.local_src, pl);
            }
#pragma unroll
            for (int j = 0; j < WPT; ++j) cnt += __popc(d[j]);
        }
        // block scan: thread offset within the tile, tile total
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_warp[wid] = incl;
        __syncthreads();
        uint32_t warp_off = 0, tile_total = 0;
#pragma unroll
        for (int w = 0; w < kMergeThreads / 32; ++w) {
            const uint32_t v = s_warp[w];
            warp_off += w < wid ? v : 0u;
            tile_total += v;
        }
        // publish this tile's count for step k, then one grid-wide barrier
        uint64_t* flags = p.flags + uint64_t(k) * T;
        if (tid == 0) __stcg(reinterpret_cast<unsigned long long*>(flags + blockIdx.x),
                             (unsigned long long)tile_total);
        COOP_T(t1);
        // split barrier: the deposit masks of r ^ l are formed while the
        // other tiles arrive (they need d only, not the draw base).  With
        // p.seg_bars the barrier spans only this segment's tiles (its own
        // counter; the prefix never reads another segment's counts).
        unsigned seg_tok = 0;
        cg::grid_group::arrival_token token{};
        jitter(2 * k);
        if (p.seg_bars)
            seg_tok = seg_barrier_arrive(p.seg_bars + blockIdx.x / p.part_tiles, lt == 0, p.part_tiles);
        else
            token = grid.barrier_arrive();
        if (live) {
#pragma unroll
            for (int j = 0; j < WPT; ++j) {
                uint32_t mv[4];
                expand_masks(d[j], mv);
#pragma unroll
                for (int i = 0; i < 4; ++i) cmask[(j * 4 + i) * kMergeThreads + tid] = mv[i];
            }
        }
        if (p.seg_bars)
            seg_barrier_wait(p.seg_bars + blockIdx.x / p.part_tiles, seg_tok);
        else
            grid.barrier_wait(std::move(token));
        jitter(2 * k + 1);
        // exclusive draw offset: the counts of this segment's earlier tiles in
        // this launch, read block-wide (all loads in flight at once)
        const uint32_t seg_base = blockIdx.x - lt;
        uint64_t acc = 0;
        if (live)
            for (uint32_t i = tid; i < lt; i += kMergeThreads) acc += __ldcg(flags + seg_base + i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (lane == 0) s_acc[wid] = acc;
        __syncthreads();
        COOP_T(t2);
        // every thread sums the 8 warp partials itself (smem broadcast): no
        // second block barrier before the coin loads
        uint64_t pre = 0;
#pragma unroll
        for (int w = 0; w < kMergeThreads / 32; ++w) pre += s_acc[w];
        COOP_T(t3);
        if (live) {
            const uint64_t sbase = cached ? s_sbase[k] : static_base(mi, m);
            // the last tile of the part knows the part's total for this merge
            if (tid == 0 && (lt == p.part_tiles - 1 || tile + 1 == p.tiles_per_seg)) {
                p.part_totals[uint64_t(p.part) * p.n_merges + mb + mi] = pre + tile_total;
                if (p.coin_end && p.part + 1 == p.n_parts)  // the stream's end index
                    p.coin_end[mb + mi] = sbase + pre + tile_total;
            }
            const uint32_t valid =
                cached ? s_valid[k] : (p.coin_valid ? __ldcg(p.coin_valid + mb + mi) : 0u);
            const uint64_t n0 = sbase + pre + warp_off + (incl - cnt);  // my first coin's draw
            if (n0 + cnt <= uint64_t(valid) * 32) {
                const uint32_t* cw = p.coins + m.coin_off;
                uint64_t n = n0;
#pragma unroll
                for (int j = 0; j < WPT; ++j) {
                    const uint32_t pc = __popc(d[j]);
                    uint32_t window = 0;
                    if (pc) {
                        const uint64_t wi = n >> 5;
                        const uint32_t sh = uint32_t(n & 31);
                        if (!MARSIT_BOUNDS_OK(wi + 1 < uint64_t(m.coin_words) + 16, p.err)) break;
                        const uint32_t c0 = __ldg(cw + wi);
                        const uint32_t c1 = (sh + pc > 32) ? __ldg(cw + wi + 1) : 0u;
                        window = __funnelshift_r(c0, c1, sh);
                    }
                    uint32_t mv[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) mv[i] = cmask[(j * 4 + i) * kMergeThreads + tid];
                    r[j] = (r[j] ^ (d[j] & ~expand_apply(window, mv))) & vmask(j);
                    n += pc;
                }
            } else {
                // beyond the precomputed budget: draw inline (same stream, same indices)
                const uint64_t key =
                    m.key_mode ? m.key : stream_key(p.seed, 5, m.receiver, p.round, sg);
                uint64_t z = key + (n0 + 1) * kGamma;
#pragma unroll
                for (int j = 0; j < WPT; ++j)
                    r[j] = (r[j] ^ (d[j] & ~coin_word(d[j], z, m.thresh11))) & vmask(j);
            }
            if (active) {
                if (m.out_slot != kNone) {
#pragma unroll
                    for (int j = 0; j < WPT; ++j)
                        cslots[(m.out_slot * WPT + j) * kMergeThreads + tid] = r[j];
                }
                if (m.out_global == kFinal) {
                    uint32_t* dst = p.agg + uint64_t(sg) * p.agg_stride + w0;
#pragma unroll
                    for (int j = 0; j < WPT; ++j)
                        if (!tail || w0 + j < p.words_proc) dst[j] = r[j];
                } else if (m.out_global != kNone) {
                    uint32_t* dst = p.gnodes + (uint64_t(sl) * p.gmax + m.out_global) * p.wst + w0;
#pragma unroll
                    for (int j = 0; j < WPT; ++j)
                        if (!tail || w0 + j < p.words_proc) __stcg(dst + j, r[j]);
                }
            }
        }
        // no block barrier here: s_warp / s_acc are rewritten next step only
        // after the grid barrier, and slots / global nodes are read back by
        // the thread that wrote them
        COOP_T(t4);
        COOP_ADD(0, t1 - t0);
        COOP_ADD(1, t2 - t1);
        COOP_ADD(2, t3 - t2);
        COOP_ADD(3, t4 - t3);
        COOP_ADD(4, 1);
    }
}

// ---------------------------------------------------------------------------
// K2 (cluster): one thread-block cluster per owned segment runs the whole
// merge DAG of the segment (see ClusterParams).  Per level of up to NL
// independent merges:
//   pass 1  every thread: d = (r ^ l) & valid for its NSUB 4-word groups of
//           each merge, popcounts, warp scans;
//           CTA scan of the NL x NSUB columns (two block barriers);
//           each CTA stores its per-merge totals into slot [its rank] of
//           every cluster CTA's shared memory (st.shared::cluster), then
//           barrier.cluster arrive.release / wait.acquire;
//   prefix  the draw offset of a group = stream base (earlier merges of the
//           same stream, shared memory) + totals of the lower-ranked CTAs
//           (local shared memory after the barrier) + the CTA-local prefix;
//   pass 2  coins of the group's draws (precomputed bitstream, L2) deposited
//           onto the set bits of d; out = r ^ (d & ~coin) (merge.hpp:44-53):
//           a shared-memory slot for a later level, or the aggregate.
// The cluster totals double-buffer by level parity: a CTA overwrites slot
// [v & 1] of a peer only after the barrier of level v + 1, which the peer
// passes only after reading level v's values.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 64-bit store into CTA `rank`'s shared memory at the address of `local` (DSMEM)
__device__ __forceinline__ void st_cluster_u64(void* local, uint32_t rank, unsigned long long v) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local));
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.u64 [%0], %1;" :: "r"(ra), "l"(v) : "memory");
}

// The level loop of the cluster merge, shared by merge_cluster_kernel (leaves
// in global memory: the extract's packed signs or a peer's) and the fused
// small-round kernel (SMEM_LEAVES: every worker's packed tile in shared memory,
// leaf w at leaf_smem + w * tile_groups; the final node also to agg_smem).
// cl_slots: [n_slots][tile_groups] node values of this CTA's tile, then
// (p.stage) [NL][2][tile_groups] the level's r and d staged by pass 1.
// Static shared state of the cluster merge of one CTA.
template <int NSUB, int NL, int NT = kClusterThreads>
struct ClusterMergeShared {
    uint32_t wt[NL * NSUB][NT / 32];    // warp totals per column
    uint32_t wpre[NL * NSUB][NT / 32];  // exclusive warp prefix per column
    uint32_t ctot[NL * NSUB];                        // CTA total per column
    unsigned long long all[2][NL][kMaxClusterSize];  // CTA totals of the cluster (DSMEM)
    DevMerge m[kMaxSegMerges];
    const uint4* row[kMaxSegMerges][2];              // leaf operand rows (recv, local) or null
    unsigned long long tot[kMaxSegMerges];           // cluster-wide draws of each merge
    unsigned long long gx[NL][2];                    // grid mode: (lower CTAs', all CTAs') totals
    uint32_t valid[kMaxSegMerges];
    uint32_t lvl[kMaxSegMerges + 1];
};

// Prologue: stage the segment's merge descriptors, leaf rows and level table.
// The caller then needs one cluster barrier (every CTA of the cluster runs
// before the first remote store; it also publishes the staging to the CTA).
// The fused kernel stages before its extract and has that barrier after it.
template <int NSUB, int NL, bool SMEM_LEAVES, bool GRID = false, int NT = kClusterThreads>
__device__ __forceinline__ void cluster_merge_prologue(const ClusterParams& p,
                                                       ClusterMergeShared<NSUB, NL, NT>& sh,
                                                       const uint4* leaf_smem) {

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t cr = GRID ? blockIdx.x % p.csize : cluster_ctarank();
    const uint32_t sl = p.seg_lo + blockIdx.x / p.csize;
    const uint32_t sg = p.s_first + sl;
    // one owned segment (a G = S rank): its merge and level ranges come with
    // the launch, so the descriptor loads below do not wait on these
    const uint32_t mb = p.solo_nm ? 0u : p.seg_begin[sl], nm = p.solo_nm ? p.solo_nm : p.seg_begin[sl + 1] - mb;
    const uint32_t lb0 = p.solo_nm ? 0u : p.lvl_start[sl];
    const uint32_t nlv = p.solo_nm ? p.solo_nlv : p.lvl_start[sl + 1] - lb0 - 1;
    const uint32_t g_first = cr * p.tile_groups;
    for (uint32_t i = tid; i < nm; i += NT) {
        const DevMerge m = p.merges[mb + i];
        sh.m[i] = m;
        sh.tot[i] = 0;
        sh.valid[i] = p.coin_valid ? (p.coherent ? __ldcg(p.coin_valid + mb + i) : p.coin_valid[mb + i]) : 0u;
        // leaf rows resolved once (P2P: the source rank's buffer, over NVLink)
#pragma unroll
        for (int o = 0; o < 2; ++o) {
            const uint16_t src = o ? m.local_src : m.recv_src;
            const uint32_t w = src & 0x3FFFu;
            const uint4* row = nullptr;
            if ((src & 0xC000u) == kSrcLeaf) {
                if (SMEM_LEAVES)
                    row = leaf_smem + size_t(w) * p.tile_groups;
                else
                    row = reinterpret_cast<const uint4*>(
                              p.peer_bits ? p.peer_bits[w / p.ml] + (uint64_t(sg) * p.ml + w % p.ml) * p.wst
                                          : p.leaves + (uint64_t((w / p.ml) * p.n_seg + sl) * p.ml + w % p.ml) * p.wst) +
                          g_first;
            }
            sh.row[i][o] = row;
        }
    }
    for (uint32_t i = tid; i <= nlv; i += NT) sh.lvl[i] = p.lvl_begin[lb0 + i];
}

// The level loop (after cluster_merge_prologue).
template <int NSUB, int NL, bool SMEM_LEAVES, bool GRID = false, int NT = kClusterThreads>
__device__ __forceinline__ void cluster_merge_levels(const ClusterParams& p, ClusterMergeShared<NSUB, NL, NT>& sh,
                                                     uint4* cl_slots, const uint4* leaf_smem, uint4* agg_smem) {
    constexpr int NCOL = NL * NSUB;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t cr = GRID ? blockIdx.x % p.csize : cluster_ctarank();
    const uint32_t seg_in_launch = blockIdx.x / p.csize;
    const uint32_t sl = p.seg_lo + blockIdx.x / p.csize;
    const uint32_t sg = p.s_first + sl;
    const uint32_t mb = p.solo_nm ? 0u : p.seg_begin[sl];
    const uint32_t lb0 = p.solo_nm ? 0u : p.lvl_start[sl];
    const uint32_t nlv = p.solo_nm ? p.solo_nlv : p.lvl_start[sl + 1] - lb0 - 1;
    const uint32_t g_first = cr * p.tile_groups;

    const uint32_t total_groups = p.words_proc / 4;
    // groups of this CTA's tile that exist; those entirely below L need no mask
    const uint32_t n_here = total_groups > g_first ? min(p.tile_groups, total_groups - g_first) : 0u;
    const uint64_t full_groups = p.seg_bits / 128;  // groups whose 128 bits are all < L
    const bool peer = p.peer_bits != nullptr;
    const bool cg = peer || p.coherent;  // operands written by another SM of this launch / a peer
    uint4* const stage = cl_slots + size_t(p.n_slots) * p.tile_groups;  // valid when p.stage
    auto load_src = [&](uint32_t k, int o, uint32_t gl) -> uint4 {
        const uint4* row = sh.row[k][o];
        if (SMEM_LEAVES && row) return row[gl];
        if (row) return cg ? __ldcg(row + gl) : __ldg(row + gl);
        const uint16_t src = o ? sh.m[k].local_src : sh.m[k].recv_src;
        return cl_slots[size_t(src & 0x3FFFu) * p.tile_groups + gl];
    };
    // r (received operand) and d = (r ^ l) & valid of local group gl of merge k
    auto diff = [&](uint32_t k, uint32_t gl, uint4& r, uint4& d) {
        r = load_src(k, 0, gl);
        const uint4 b = load_src(k, 1, gl);
        d = make_uint4(r.x ^ b.x, r.y ^ b.y, r.z ^ b.z, r.w ^ b.w);
        const uint64_t g = uint64_t(g_first) + gl;
        if (g >= full_groups) {  // the segment's last bits: storage padding is 0
            uint32_t mk[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t rem = int64_t(p.seg_bits) - int64_t(g * 4 + j) * 32;
                mk[j] = rem >= 32 ? kFull : (rem <= 0 ? 0u : ((1u << rem) - 1u));
            }
            d.x &= mk[0], d.y &= mk[1], d.z &= mk[2], d.w &= mk[3];
        }
    };
    auto popc4 = [](const uint4& d) { return __popc(d.x) + __popc(d.y) + __popc(d.z) + __popc(d.w); };

    // the next level's local leaf tiles into L1 while this level finishes
    // (p.prefetch = where: 1 after the masks, 2 before them, 3 after the totals)
    auto prefetch_next = [&](uint32_t v, uint32_t where) {
        if (SMEM_LEAVES || cg || v + 1 >= nlv || p.prefetch != where) return;
        const uint32_t k1 = sh.lvl[v + 1], nk1 = sh.lvl[v + 2] - k1;
#pragma unroll
        for (int i = 0; i < NL; ++i)
#pragma unroll
            for (int u = 0; u < NSUB; ++u) {
                const uint32_t gl = uint32_t(u) * NT + tid;
                if (uint32_t(i) >= nk1 || gl >= n_here) continue;
#pragma unroll
                for (int o = 0; o < 2; ++o)
                    if (const uint4* row = sh.row[k1 + i][o]) asm volatile("prefetch.global.L1 [%0];" ::"l"(row + gl));
            }
    };

    for (uint32_t v = 0; v < nlv; ++v) {
#ifdef MARSIT_FUSED_PROF
        const uint64_t lv_t0 = (threadIdx.x == 0 && blockIdx.x == 0) ? gtime_ns() : 0;
#endif
        const uint32_t k0 = sh.lvl[v], nk = sh.lvl[v + 1] - k0;
        // pass 1: d, counts and warp scans (r and d staged for pass 2)
        uint32_t ex[NL][NSUB];
#pragma unroll
        for (int i = 0; i < NL; ++i)
#pragma unroll
            for (int u = 0; u < NSUB; ++u) {
                const uint32_t gl = uint32_t(u) * NT + tid;
                uint32_t c = 0;
                if (uint32_t(i) < nk && gl < n_here) {
                    uint4 r, d;
                    diff(k0 + i, gl, r, d);
                    c = popc4(d);
                    if (p.stage) {
                        stage[(i * 2) * p.tile_groups + gl] = r;
                        stage[(i * 2 + 1) * p.tile_groups + gl] = d;
                    }
                }
                uint32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += y;
                }
                ex[i][u] = incl - c;
                if (lane == 31) sh.wt[i * NSUB + u][wid] = incl;
            }
        __syncthreads();
        if (wid < NCOL) {  // NT / 32 <= 32 warp totals per column
            const uint32_t x = lane < NT / 32 ? sh.wt[wid][lane] : 0u;
            uint32_t incl = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane < NT / 32) sh.wpre[wid][lane] = incl - x;
            if (lane == 31) sh.ctot[wid] = incl;
        }
        __syncthreads();
        // this CTA's per-merge totals: cluster mode into every cluster CTA's
        // slot [v & 1][i][cr] (DSMEM); grid mode into global memory
        unsigned long long* const xch =
            GRID ? p.xch + (size_t(v & 1) * (gridDim.x / p.csize) + seg_in_launch) * p.csize * NL : nullptr;
        // grid mode: the total rides in one 64-bit word with the launch's
        // level tag, so the readers' polls are the barrier (no counter)
        const uint32_t tag = GRID ? (p.xch_tag << 8) | (v & 0xFFu) : 0u;
        if (GRID) {
            if (tid < NL) {
                unsigned long long t = 0;
#pragma unroll
                for (int u = 0; u < NSUB; ++u) t += sh.ctot[tid * NSUB + u];
                t |= uint64_t(tag) << 32;
                asm volatile("st.relaxed.gpu.global.u64 [%0],%1;" ::"l"(xch + size_t(cr) * NL + tid), "l"(t)
                             : "memory");
            }
        } else if (uint32_t(tid) < p.csize) {
#pragma unroll
            for (int i = 0; i < NL; ++i) {
                unsigned long long t = 0;
#pragma unroll
                for (int u = 0; u < NSUB; ++u) t += sh.ctot[i * NSUB + u];
                st_cluster_u64(&sh.all[v & 1][i][cr], uint32_t(tid), t);
            }
        }
        jitter(2 * v);
        // the coin words this CTA will most likely read in pass 2, into L1
        // while the other CTAs' totals arrive: the lower CTAs are assumed to
        // have drawn as many as this one (prefix ~ cr x own), +-slack; a wrong
        // estimate only wastes the prefetches (p.coin_l1)
        if (p.coin_l1 && p.coins && !p.coherent) {
            for (uint32_t i = 0; i < nk; ++i) {
                const DevMerge& m = sh.m[k0 + i];
                uint64_t base = m.base_add;
                for (int32_t src = m.offset_src; src >= 0; src = sh.m[src].offset_src)
                    base += sh.tot[src] + sh.m[src].base_add;
                uint64_t own = 0;
#pragma unroll
                for (int u = 0; u < NSUB; ++u) own += sh.ctot[i * NSUB + u];
                const uint64_t est = base + uint64_t(cr) * own, slack = 1024 + (own >> 3);
                const uint64_t w_lo = (est > slack ? est - slack : 0) >> 5;
                const uint64_t w_hi = min((est + own + slack) >> 5, uint64_t(sh.valid[k0 + i]));
                const uint32_t* cw = p.coins + m.coin_off;
                for (uint64_t line = (w_lo >> 5) + tid; line <= (w_hi >> 5) && w_lo < w_hi; line += NT)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(cw + line * 32));
            }
        }
#ifdef MARSIT_FUSED_PROF
        const uint64_t lv_t1 = (threadIdx.x == 0 && blockIdx.x == 0) ? gtime_ns() : 0;
#endif
        // split barrier: arrive, form the deposit masks of the staged d while
        // the other CTAs arrive (they depend on d only), then wait
        if (!GRID) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        prefetch_next(v, 2);
        if (p.masks) {
            uint4* const mreg = stage + size_t(2 * NL) * p.tile_groups;  // [NL][4 words][tg] x 4 masks
#pragma unroll
            for (int i = 0; i < NL; ++i)
#pragma unroll
                for (int u = 0; u < NSUB; ++u) {
                    const uint32_t gl = uint32_t(u) * NT + tid;
                    if (uint32_t(i) >= nk || gl >= n_here) continue;
                    const uint4 d = stage[(i * 2 + 1) * p.tile_groups + gl];
                    const uint32_t dd[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        uint32_t mv[4];
                        expand_masks(dd[j], mv);
                        mreg[size_t(i * 4 + j) * p.tile_groups + gl] = make_uint4(mv[0], mv[1], mv[2], mv[3]);
                    }
                }
        }
        prefetch_next(v, 1);
        if (GRID) {
            // warp i polls merge i's words of every CTA of the segment (all
            // of a lane's loads in flight at once, 8 per 256 CTAs) until each
            // carries this level's tag: the lower CTAs' sum is the tile's
            // draw offset, the sum over all the merge's total
            if (wid < NL && uint32_t(wid) < nk) {
                unsigned long long pre = 0, tot = 0;
                for (uint32_t q0 = 0; q0 < p.csize; q0 += 256) {
                    unsigned long long x[8];
                    for (;;) {
                        bool ok = true;
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const uint32_t q = q0 + e * 32 + lane;
                            x[e] = uint64_t(tag) << 32;
                            if (q < p.csize)
                                asm volatile("ld.relaxed.gpu.global.u64 %0,[%1];"
                                             : "=l"(x[e])
                                             : "l"(xch + size_t(q) * NL + wid)
                                             : "memory");
                        }
#pragma unroll
                        for (int e = 0; e < 8; ++e) ok &= uint32_t(x[e] >> 32) == tag;
                        if (__all_sync(kFull, ok)) break;
                    }
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const uint32_t q = q0 + e * 32 + lane;
                        const unsigned long long t = x[e] & 0xFFFFFFFFull;
                        pre += q < cr ? t : 0ull;
                        tot += t;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    pre += __shfl_xor_sync(kFull, pre, o);
                    tot += __shfl_xor_sync(kFull, tot, o);
                }
                if (lane == 0) sh.gx[wid][0] = pre, sh.gx[wid][1] = tot;
            }
            __syncthreads();
        } else {
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        }
        prefetch_next(v, 3);
        jitter(2 * v + 1);
#ifdef MARSIT_FUSED_PROF
        const uint64_t lv_t2 = (threadIdx.x == 0 && blockIdx.x == 0) ? gtime_ns() : 0;
#endif
        // pass 2: draw offsets, coins, deposit
#pragma unroll
        for (int i = 0; i < NL; ++i) {
            if (uint32_t(i) >= nk) continue;
            const uint32_t k = k0 + i;
            const DevMerge& m = sh.m[k];
            // lower-ranked CTAs' totals (the tile's draw offset) and the
            // cluster total: lane q holds CTA q's total, warp reductions
            unsigned long long pre = 0, tot = 0;
            if (GRID) {
                pre = sh.gx[i][0], tot = sh.gx[i][1];
            } else {
                const unsigned long long x = uint32_t(lane) < p.csize ? sh.all[v & 1][i][lane] : 0ull;
                pre = uint32_t(lane) < cr ? x : 0ull;
                tot = x;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    pre += __shfl_xor_sync(kFull, pre, o);
                    tot += __shfl_xor_sync(kFull, tot, o);
                }
            }
            // stream base: draws before this round's merges + the earlier
            // merges of the same (receiver, segment) stream (continuation)
            uint64_t base = m.base_add;
            for (int32_t src = m.offset_src; src >= 0; src = sh.m[src].offset_src)
                base += sh.tot[src] + sh.m[src].base_add;
            if (tid == 0) {
                sh.tot[k] = tot;  // read by later levels (after their block barriers)
                if (cr == 0) {
                    if (p.totals) p.totals[mb + k] = tot;
                    if (p.coin_end) p.coin_end[mb + k] = base + tot;
                }
            }
            const uint64_t valid_bits = uint64_t(sh.valid[k]) * 32;
            const uint32_t* cw = p.coins ? p.coins + m.coin_off : nullptr;
            uint64_t off = base + pre;  // + this CTA's earlier columns of merge i
            // two groups per batch: their operand and coin loads are issued
            // together (one round trip each) before the deposit ALU work
#pragma unroll
            for (int u0 = 0; u0 < NSUB; u0 += 2) {
                uint4 r[2], d[2];
                uint64_t n0[2];
                bool live[2], fast[2];
                uint32_t win[2][5];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int u = u0 + h;
                    const uint32_t gl = uint32_t(u) * NT + tid;
                    live[h] = u < NSUB && gl < n_here;
                    fast[h] = false;
                    if (u < NSUB) {
                        n0[h] = off + sh.wpre[i * NSUB + u][wid] + ex[i][u];
                        off += sh.ctot[i * NSUB + u];
                    }
                    if (!live[h]) continue;
                    if (p.stage) {
                        r[h] = stage[(i * 2) * p.tile_groups + gl];
                        d[h] = stage[(i * 2 + 1) * p.tile_groups + gl];
                    } else {
                        diff(k, gl, r[h], d[h]);
                    }
                    fast[h] = cw && n0[h] + popc4(d[h]) <= valid_bits;
                    if (fast[h] && !MARSIT_BOUNDS_OK((n0[h] >> 5) + 5 <= uint64_t(m.coin_words) + 16, p.err))
                        fast[h] = live[h] = false;
                    if (fast[h]) {
                        const uint32_t* c = cw + (n0[h] >> 5);
#pragma unroll
                        for (int q = 0; q < 5; ++q) win[h][q] = p.coherent ? __ldcg(c + q) : __ldg(c + q);
                    }
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (!live[h]) continue;
                    uint32_t rr[4] = {r[h].x, r[h].y, r[h].z, r[h].w};
                    const uint32_t dd[4] = {d[h].x, d[h].y, d[h].z, d[h].w};
                    if (fast[h]) {
                        // sliding 64-bit window over the 5 coin words: word j's
                        // coins start o bits into (lo, hi); at most one advance
                        // per word (popc <= 32)
                        uint32_t lo = win[h][0], hi = win[h][1], o = uint32_t(n0[h] & 31), a = 0;
                        const uint32_t glh = uint32_t(u0 + h) * NT + tid;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            uint32_t mv[4];
                            if (p.masks) {  // formed during the barrier
                                const uint4 q = (stage + size_t(2 * NL) * p.tile_groups)[size_t(i * 4 + j) * p.tile_groups + glh];
                                mv[0] = q.x, mv[1] = q.y, mv[2] = q.z, mv[3] = q.w;
                            } else {
                                expand_masks(dd[j], mv);
                            }
                            rr[j] ^= dd[j] & ~expand_apply(__funnelshift_r(lo, hi, o), mv);
                            o += __popc(dd[j]);
                            if (j < 3) {
                                // (lo, hi) = (win[a], win[a + 1]) after a advances
                                const bool adv = o >= 32;
                                uint32_t nx = win[h][2];
                                if (j >= 1) nx = a >= 1 ? win[h][3] : nx;
                                if (j >= 2) nx = a >= 2 ? win[h][4] : nx;
                                lo = adv ? hi : lo;
                                hi = adv ? nx : hi;
                                o -= adv ? 32u : 0u;
                                a += adv ? 1u : 0u;
                            }
                        }
                    } else {
                        // beyond the precomputed budget: draw inline (same stream, same indices)
                        const uint64_t key =
                            m.key_mode ? m.key : stream_key(p.seed, 5, m.receiver, p.round, sg);
                        uint64_t z = key + (n0[h] + 1) * kGamma;
#pragma unroll
                        for (int j = 0; j < 4; ++j) rr[j] ^= dd[j] & ~coin_word(dd[j], z, m.thresh11);
                    }
                    const uint4 out = make_uint4(rr[0], rr[1], rr[2], rr[3]);
                    const uint32_t gl = uint32_t(u0 + h) * NT + tid;
                    if (m.out_slot != kNone) cl_slots[size_t(m.out_slot) * p.tile_groups + gl] = out;
                    if (m.out_global == kFinal) {
                        reinterpret_cast<uint4*>(p.agg + uint64_t(sg) * p.agg_stride)[g_first + gl] = out;
                        if (SMEM_LEAVES) agg_smem[gl] = out;
                    }
                }
            }
        }
        // no block barrier here: slots and the staging are read back by the
        // threads that wrote them; sh.wt / sh.wpre / sh.ctot are rewritten by
        // the next level only after its first block barrier, which every
        // thread reaches after finishing this pass
#ifdef MARSIT_FUSED_PROF
        if (threadIdx.x == 0 && blockIdx.x == 0) {
            const uint64_t lv_t3 = gtime_ns();
            atomicAdd(&g_coop_prof[4], (unsigned long long)(lv_t1 - lv_t0));
            atomicAdd(&g_coop_prof[5], (unsigned long long)(lv_t2 - lv_t1));
            atomicAdd(&g_coop_prof[6], (unsigned long long)(lv_t3 - lv_t2));
            atomicAdd(&g_coop_prof[7], 1ull);
        }
#endif
    }
}

template <int NSUB, int NL>
__global__ void __launch_bounds__(kClusterThreads, 1) merge_cluster_kernel(const ClusterParams p) {
    extern __shared__ uint4 cl_dyn[];
    __shared__ ClusterMergeShared<NSUB, NL> sh;
    cluster_merge_prologue<NSUB, NL, false>(p, sh, nullptr);
    cluster_sync_all();
    cluster_merge_levels<NSUB, NL, false>(p, sh, cl_dyn, nullptr, nullptr);
}

// K2g: the level loop over csize co-resident CTAs per segment, cross-CTA
// totals through global memory and one release/acquire barrier per segment
// and level (cooperative launch).
// NT = 1024 (NSUB groups per thread), or 256 / 512 for tiles of at most that
// many groups (a rank's one or two segments over all SMs): 8 or 16 warps at
// each CTA barrier and scan instead of 32 of which most hold no group.
template <int NSUB, int NL, int NT = kClusterThreads>
__global__ void __launch_bounds__(NT, 1) merge_grid_kernel(const ClusterParams p) {
#ifdef MARSIT_FUSED_PROF
    const uint64_t gp_t0 = (threadIdx.x == 0 && blockIdx.x == 0) ? gtime_ns() : 0;
#endif
    extern __shared__ uint4 gr_dyn[];
    __shared__ ClusterMergeShared<NSUB, NL, NT> sh;
    cluster_merge_prologue<NSUB, NL, false, true, NT>(p, sh, nullptr);
    __syncthreads();
#ifdef MARSIT_FUSED_PROF
    const uint64_t gp_t1 = (threadIdx.x == 0 && blockIdx.x == 0) ? gtime_ns() : 0;
#endif
    cluster_merge_levels<NSUB, NL, false, true, NT>(p, sh, gr_dyn, nullptr, nullptr);
#ifdef MARSIT_FUSED_PROF
    if (threadIdx.x == 0 && blockIdx.x == 0) {  // slots 8-10: prologue, CTA 0's whole launch, launches
        atomicAdd(&g_coop_prof[8], (unsigned long long)(gp_t1 - gp_t0));
        atomicAdd(&g_coop_prof[9], (unsigned long long)(gtime_ns() - gp_t0));
        atomicAdd(&g_coop_prof[10], 1ull);
    }
#endif
}

// ---------------------------------------------------------------------------
// Fused small round (see FusedParams): K1 -> K2 -> K3/K4 of one segment per
// cluster in one launch.  A "task" is one worker's 128 coordinates of one
// 4-word group of this CTA's tile; a warp takes one task per step: lane l
// holds coordinates 4l..4l+3 (one 16-byte quad of g and of c), the four sign
// nibbles of a word meet by OR-shuffles over 8 lanes (as in K1), and the
// decode reads the group's aggregate words from shared memory.
// ---------------------------------------------------------------------------
// Tensor memory as a thread-private parking area (tcgen05.st / tcgen05.ld,
// 32x32b shape: thread i of the warp addresses TMEM lane base_lane + i).
__device__ __forceinline__ void tmem_put(uint32_t ta, const float (&u)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ta),
                 "r"(__float_as_uint(u[0])), "r"(__float_as_uint(u[1])), "r"(__float_as_uint(u[2])),
                 "r"(__float_as_uint(u[3]))
                 : "memory");
}
__device__ __forceinline__ void tmem_put(uint32_t ta, const double (&u)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(ta),
                 "r"(__double2loint(u[0])), "r"(__double2hiint(u[0])), "r"(__double2loint(u[1])),
                 "r"(__double2hiint(u[1])), "r"(__double2loint(u[2])), "r"(__double2hiint(u[2])),
                 "r"(__double2loint(u[3])), "r"(__double2hiint(u[3]))
                 : "memory");
}
__device__ __forceinline__ void tmem_get(uint32_t ta, float (&u)[4]) {
    uint32_t a, b, c, d;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(ta)
                 : "memory");
    u[0] = __uint_as_float(a), u[1] = __uint_as_float(b), u[2] = __uint_as_float(c), u[3] = __uint_as_float(d);
}
__device__ __forceinline__ void tmem_get(uint32_t ta, double (&u)[4]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta)
                 : "memory");
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = __hiloint2double(int(r[2 * k + 1]), int(r[2 * k]));
}
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_addr, uint32_t cols) {  // one warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     uint32_t(__cvta_generic_to_shared(smem_addr))),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
// every thread: after its last TMEM access; warp 0 frees the allocation
__device__ __forceinline__ void tmem_release(uint32_t addr, uint32_t cols) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if ((threadIdx.x >> 5) == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(cols) : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <typename T>
__device__ __forceinline__ bool quad_real(uint64_t j, uint64_t seg_len, uint64_t gi, uint64_t dim) {
    return j + 3 < seg_len && gi + 3 < dim;
}

template <typename T, int NSUB, int NL>
__global__ void __launch_bounds__(kFusedThreads, 1)
    round_cluster_kernel(const ClusterParams p, const FusedParams<T> f) {
#ifdef MARSIT_FUSED_PROF
    const uint64_t fp_t0 = (threadIdx.x == 0 && blockIdx.x == 0) ? gtime_ns() : 0;
#endif
    extern __shared__ uint4 fz_dyn[];  // [workers][tg] leaves, [tg] aggregate, then the merge's slots / staging
    __shared__ ClusterMergeShared<NSUB, NL, kFusedThreads> sh;
    const uint32_t tg = p.tile_groups;
    uint4* leaf = fz_dyn;
    uint4* aggs = leaf + size_t(f.workers) * tg;
    uint4* slots = aggs + tg;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr uint32_t NWARP = kFusedThreads / 32;
    const uint32_t cr = cluster_ctarank();
    const uint32_t sl = p.seg_lo + blockIdx.x / p.csize;
    const uint32_t g_first = cr * tg;
    const uint32_t total_groups = p.words_proc / 4;
    const uint32_t n_here = total_groups > g_first ? min(tg, total_groups - g_first) : 0u;
    const uint64_t seg0 = uint64_t(sl) * p.seg_bits;  // first coordinate of the segment (G == 1)
    // the merge's descriptors, loaded under the extract's streaming
    cluster_merge_prologue<NSUB, NL, true, false, kFusedThreads>(p, sh, leaf);
    constexpr int B = sizeof(T) == 4 ? 4 : 2;  // groups per warp step: 2B quad loads in flight per lane
    // K1: u = g + c, sign nibbles -> packed words in shared memory
    T fin = T(0);
    for (uint32_t w = 0; w < f.workers; ++w) {
        const T* __restrict__ gw = f.g[w];
        const T* __restrict__ cw = f.c[w];
        for (uint32_t gl0 = wid; gl0 < n_here; gl0 += NWARP * B) {
            Quad<T> gv[B], cv[B];
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint32_t gl = gl0 + b * NWARP;
                const uint64_t j = uint64_t(g_first + gl) * 128 + lane * 4;
                const uint64_t gi = seg0 + j;
                if (gl < n_here && quad_real<T>(j, p.seg_bits, gi, f.dim)) {
                    gv[b] = load4(gw + gi);
                    cv[b] = load4(cw + gi);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const bool in = gl < n_here && j + k < p.seg_bits && gi + k < f.dim;
                        gv[b].v[k] = in ? gw[gi + k] : T(0);
                        cv[b].v[k] = in ? cw[gi + k] : T(0);
                    }
                }
            }
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint32_t gl = gl0 + b * NWARP;
                if (gl >= n_here) break;
                const uint64_t j = uint64_t(g_first + gl) * 128 + lane * 4;
                T u[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    u[k] = add_rn(add_rn(gv[b].v[k], cv[b].v[k]), T(0));  // -0.0 -> +0.0 (sign_vector.hpp:70)
                    fin = fma_rn(u[k], T(0), fin);
                }
                uint32_t nib = sign_nibble(u[0], u[1], u[2], u[3]);
                const uint64_t valid = j >= p.seg_bits ? 0 : p.seg_bits - j;  // storage padding -> 0
                if (valid < 4) nib &= (1u << valid) - 1u;
                uint32_t v = nib << ((lane & 7) * 4);
                v |= __shfl_xor_sync(kFull, v, 1);
                v |= __shfl_xor_sync(kFull, v, 2);
                v |= __shfl_xor_sync(kFull, v, 4);
                if ((lane & 7) == 0) reinterpret_cast<uint32_t*>(leaf + size_t(w) * tg + gl)[lane >> 3] = v;
            }
        }
    }
    if (__any_sync(kFull, !(fin == fin)) && lane == 0) atomicOr(f.err, 1);
    cluster_sync_all();  // the tiles' leaves and the staged descriptors complete; cluster running
    // K2: the segment's merge DAG (cluster-wide draw offsets via DSMEM)
#ifdef MARSIT_FUSED_PROF
    const uint64_t fp_t1 = (threadIdx.x == 0 && blockIdx.x == 0) ? gtime_ns() : 0;
#endif
    cluster_merge_levels<NSUB, NL, true, false, kFusedThreads>(p, sh, slots, leaf, aggs);
    __syncthreads();
#ifdef MARSIT_FUSED_PROF
    const uint64_t fp_t2 = (threadIdx.x == 0 && blockIdx.x == 0) ? gtime_ns() : 0;
#endif
    // K3/K4: g_t = +-eta from the aggregate, c' = (g + c) - g_t
    for (uint32_t w = 0; w < f.workers; ++w) {
        const T* __restrict__ gw = f.g[w];
        const T* cw = f.c[w];  // may alias c_out (in place)
        T* co = f.c_out[w];
        T* upd = w == 0 ? f.update : nullptr;
        for (uint32_t gl0 = wid; gl0 < n_here; gl0 += NWARP * B) {
            Quad<T> gv[B], cv[B];
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint32_t gl = gl0 + b * NWARP;
                const uint64_t j = uint64_t(g_first + gl) * 128 + lane * 4;
                const uint64_t gi = seg0 + j;
                if (gl < n_here && quad_real<T>(j, p.seg_bits, gi, f.dim)) {
                    gv[b] = load4(gw + gi);
                    cv[b] = load4_rw(cw + gi);
                }
            }
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint32_t gl = gl0 + b * NWARP;
                if (gl >= n_here) break;
                const uint64_t j = uint64_t(g_first + gl) * 128 + lane * 4;
                const uint64_t gi = seg0 + j;
                const uint32_t word = reinterpret_cast<const uint32_t*>(aggs + gl)[lane >> 3];
                const uint32_t nib = (word >> ((lane & 7) * 4)) & 0xFu;
                if (quad_real<T>(j, p.seg_bits, gi, f.dim)) {
                    Quad<T> out, up;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const T gt = ((nib >> k) & 1u) ? f.eta : -f.eta;
                        out.v[k] = sub_rn(add_rn(gv[b].v[k], cv[b].v[k]), gt);
                        up.v[k] = gt;
                    }
                    store4(co + gi, out);
                    if (upd) store4(upd + gi, up);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (j + k < p.seg_bits && gi + k < f.dim) {
                            const T gt = ((nib >> k) & 1u) ? f.eta : -f.eta;
                            co[gi + k] = sub_rn(add_rn(gw[gi + k], cw[gi + k]), gt);
                            if (upd) upd[gi + k] = gt;
                        }
                }
            }
        }
    }
#ifdef MARSIT_FUSED_PROF
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const uint64_t fp_t3 = gtime_ns();
        atomicAdd(&g_coop_prof[0], (unsigned long long)(fp_t1 - fp_t0));
        atomicAdd(&g_coop_prof[1], (unsigned long long)(fp_t2 - fp_t1));
        atomicAdd(&g_coop_prof[2], (unsigned long long)(fp_t3 - fp_t2));
        atomicAdd(&g_coop_prof[3], 1ull);
    }
#endif
}

// ---------------------------------------------------------------------------
// Coin precompute: blockIdx.y = merge, warps stride over the merge's words;
// lane l draws n = 32*w + l and the warp ballot is coin word w.
// ---------------------------------------------------------------------------
// Coin of draw z: mix64(z) < th, decided on the high word of mix64 (exact
// unless it equals th's high word, probability 2^-32).  mix64_hi sends the
// first xor-shift to the ALU pipe and the second through the FMA pipe, and
// forms only the high word of the last product.
// Adaptive budget: a merge whose stream ended at draw E last round gets its
// coins up to E + E/16 + 4096 (capped by its buffer capacity); without a
// history (E = ~0), coin_default words.  The merge draws anything beyond
// coin_valid inline, so the budget changes the work, never the bits.
// Words of merge m's stream computed this round (and the chunks of 64 words
// that cover them), from the draw index its stream ended at last round.
__device__ __forceinline__ uint32_t coin_budget(const DevMerge& m, uint64_t e, uint32_t* chunks) {
    uint64_t want = m.coin_default;
    if (e != ~0ull) want = (e + e / 16 + 4096 + 31) / 32;
    const uint32_t words = uint32_t(want < m.coin_words ? want : m.coin_words);
    *chunks = (words + 63) / 64;  // 64 words = 2048 draws per chunk
    return *chunks * 64 < m.coin_words ? *chunks * 64 : m.coin_words;
}

// One warp: coin words [w0, w0 + NW) (NW = 32 or 64) of the stream with key
// `key`: lane l builds word w0 + l (and w0 + 32 + l, a second independent
// draw stream for ILP) bit by bit, then the words are stored coalesced.  The
// coin is decided on h2, the high word of mix64's last product (mix64_h2):
// its final xor-shift only flips bit 0, so h2 < th >> 32 decides unless h2
// agrees with th's high word above bit 0 (probability 2^-31 per draw) — that
// only raises a flag, and a word that saw one is redrawn with the full
// 64-bit compare (no per-draw branch).  (A ballot per word — lane l drawing
// bit l — measured slower: 151 vs 141 us per C3 coin launch.)
template <int NW>
__device__ __forceinline__ void coin_words(uint64_t key, uint64_t th, uint32_t* out, uint64_t w0, int lane) {
    static_assert(NW == 32 || NW == 64, "coin run of 32 or 64 words");
    constexpr bool TWO = NW == 64;
    const uint32_t thh = uint32_t(th >> 32), thh1 = thh >> 1;
    uint64_t za = key + ((w0 + uint64_t(lane)) * 32 + 1) * kGamma;
    uint64_t zb = za + 1024 * kGamma;
    const uint64_t za0 = za, zb0 = zb;
    uint32_t wa = 0, wb = 0;
    bool tie = false;
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
        const uint32_t xa = mix64_h2(za);
        wa |= uint32_t(xa < thh) << i;
        tie |= __umulhi(xa, 0x80000000u) == thh1;
        za += kGamma;
        if (TWO) {
            const uint32_t xb = mix64_h2(zb);
            wb |= uint32_t(xb < thh) << i;
            tie |= __umulhi(xb, 0x80000000u) == thh1;
            zb += kGamma;
        }
    }
    if (tie) {
        za = za0;
        zb = zb0;
        wa = wb = 0;
        for (int i = 0; i < 32; ++i) {
            if (mix64(za) < th) wa |= 1u << i;
            if (TWO && mix64(zb) < th) wb |= 1u << i;
            za += kGamma;
            zb += kGamma;
        }
    }
    __stcg(out + w0 + lane, wa);
    if (TWO) __stcg(out + w0 + 32 + lane, wb);
}

__global__ void __launch_bounds__(256) coins_kernel(const DevMerge* __restrict__ merges,
                                                    uint64_t seed, uint64_t round,
                                                    const uint64_t* __restrict__ coin_end,
                                                    uint32_t* __restrict__ coin_valid,
                                                    uint32_t* __restrict__ coins) {
    const DevMerge m = merges[blockIdx.y];
    uint32_t chunks;
    const uint32_t valid = coin_budget(m, coin_end ? coin_end[blockIdx.y] : ~0ull, &chunks);
    if (blockIdx.x == 0 && threadIdx.x == 0) coin_valid[blockIdx.y] = valid;
    if (chunks == 0) return;
    const int lane = threadIdx.x & 31;
    const uint64_t key = m.key_mode ? m.key : stream_key(seed, 5, m.receiver, round, m.segment);
    uint32_t* out = coins + m.coin_off;
    for (uint32_t c = blockIdx.x * 8 + (threadIdx.x >> 5); c < chunks; c += gridDim.x * 8)
        coin_words<64>(key, m.thresh11, out, uint64_t(c) * 64, lane);
}

// ---------------------------------------------------------------------------
// Spread small round (see SpreadParams): one launch, every SM streaming.
// A CTA owns groups [g_lo, g_hi) of the flattened (segment, group) space; a
// warp task is one worker's 128 coordinates of one group (lane l: quad l of g
// and of c), exactly as in the fused round.  Segment s is merged by cluster s.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Spin until *p == v (acquire).  Bounded (~2 s): every CTA of the launch is
// resident by construction (the grid is the co-resident cluster count), so a
// timeout means the device was shared beyond that — err |= 16 (reported by
// marsit_ctx_check) and the launch finishes instead of hanging the GPU.
__device__ __forceinline__ void wait_eq_u32(const unsigned* p, unsigned v, int* err) {
    for (uint32_t spin = 0; ld_acquire_u32(p) != v; ++spin) {
        if (spin == (1u << 22)) {
            atomicOr(err, 16);
            return;
        }
        __nanosleep(20);
    }
}


// The coins of round `round` into buffer cb, by CTAs [0, nctas) of the
// caller's choosing (cta = this CTA's index among them): warp 0 sizes every
// stream's chunks from the stream ends of the previous launch (lane-parallel loads,
// one scan per 32 streams), then the 32-word chunks go round robin over the
// CTAs first, one coin word per lane (short per-warp latency chains).
template <typename T>
__device__ __forceinline__ void spread_coins(const ClusterParams& p, const SpreadParams<T>& s, uint32_t* s_cbase,
                                             uint32_t cb, uint64_t round, uint32_t cta, uint32_t nctas) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr uint32_t NWARP = kFusedThreads / 32;
    // budgets from the stream ends of the launch before this one (cend of the
    // other parity than p.round's, which this launch's merges are writing):
    // stable for the whole launch, so every CTA sizes the same chunks
    const unsigned long long* cend = s.cend + size_t((p.round & 1) ^ 1) * s.n_merges;
    __syncthreads();  // s_cbase may still be read by an earlier call
    if (wid == 0) {
        uint32_t run = 0;
        for (uint32_t k0 = 0; k0 < s.n_merges; k0 += 32) {
            const uint32_t k = k0 + lane;
            uint32_t words = 0;
            if (k < s.n_merges) {
                uint32_t chunks;  // of 64 words: the budget rule of the coin kernel
                const uint32_t valid = coin_budget(p.merges[k], __ldcg(cend + k), &chunks);
                if (cta == 0) s.coin_valid[cb][k] = valid;
                words = chunks * 64;
            }
            const uint32_t units = words / 32;
            uint32_t incl = units;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += y;
            }
            if (k < s.n_merges) s_cbase[k] = run + incl - units;
            run += __shfl_sync(kFull, incl, 31);
        }
        if (lane == 0) s_cbase[s.n_merges] = run;
    }
    __syncthreads();
    const uint32_t nw = nctas * NWARP, total = s_cbase[s.n_merges];
    for (uint32_t i = wid * nctas + cta; i < total; i += nw) {
        uint32_t lo = 0, hi = s.n_merges;  // stream k with s_cbase[k] <= i < s_cbase[k + 1]
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (s_cbase[mid] <= i) lo = mid; else hi = mid;
        }
        const DevMerge& m = p.merges[lo];
        const uint64_t key = m.key_mode ? m.key : stream_key(p.seed, 5, m.receiver, round, m.segment);
        coin_words<32>(key, m.thresh11, s.coins[cb] + m.coin_off, uint64_t(i - s_cbase[lo]) * 32, lane);
    }
}

template <typename T, int NSUB, int NL>
__global__ void __launch_bounds__(kFusedThreads, 1)
    round_spread_kernel(const ClusterParams p, const SpreadParams<T> s) {
#ifdef MARSIT_FUSED_PROF
    const uint64_t fp_t0 = threadIdx.x == 0 ? gtime_ns() : 0;
#endif
    extern __shared__ uint4 sp_dyn[];  // merge clusters: [workers][tg] leaves, [tg] aggregate, slots / staging
    __shared__ ClusterMergeShared<NSUB, NL, kFusedThreads> sh;
    __shared__ unsigned s_gen;
    const FusedParams<T>& f = s.f;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr uint32_t NWARP = kFusedThreads / 32;
    // the generation before this CTA arrives (it cannot advance without us)
    if (tid == 0) s_gen = ld_acquire_u32(s.sync + 1);
    const uint32_t gps = p.words_proc / 4;  // groups per segment
    const uint64_t total = uint64_t(p.n_seg) * gps;
    const uint32_t g_lo = uint32_t(total * blockIdx.x / gridDim.x);
    const uint32_t g_hi = uint32_t(total * (blockIdx.x + 1) / gridDim.x);
    // this round's coins: computed here only when the buffer's tag misses
    const uint32_t cb = uint32_t(p.round & 1);
    __shared__ uint32_t s_cbase[kSpreadMaxMerges + 1];
    __shared__ int s_hit;
    __shared__ uint32_t s_tmem;
    // the buffer's tag: loaded now, compared after the extract (a miss
    // computes the coins then, before this CTA arrives)
    unsigned long long tag_seed = 0, tag_round = 0;
    if (tid == 0) {
        tag_seed = __ldcg(s.tag + 2 * cb);
        tag_round = __ldcg(s.tag + 2 * cb + 1);
    }
    const bool stash = f.stash_cols != 0;
    if (stash && wid == 0) tmem_alloc(&s_tmem, f.tmem_cols);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // this thread's parking area: lane quadrant wid % 4, column block wid / 4
    const uint32_t tbase = stash ? s_tmem + ((uint32_t(wid & 3) * 32) << 16) + uint32_t(wid >> 2) * f.stash_cols : 0u;
    constexpr uint32_t QCOLS = sizeof(T);  // TMEM columns (32-bit) per quad of u
    // the merge clusters stage their descriptors under the extract
    const uint32_t cl = blockIdx.x / p.csize;
    if (cl < p.n_seg) cluster_merge_prologue<NSUB, NL, true, false, kFusedThreads>(p, sh, sp_dyn);
#ifdef MARSIT_FUSED_PROF
    const bool prof = tid == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1);
    const int ps = blockIdx.x == 0 ? 8 : 12;  // slots 8..11: CTA 0, 12..15: the last CTA
    const uint64_t fp_tc = prof ? gtime_ns() : 0;
    if (prof) atomicAdd(&g_coop_prof[ps], (unsigned long long)(fp_tc - fp_t0));  // start: TMEM, descriptors
#endif
    constexpr int B = sizeof(T) == 4 ? 4 : 2;  // groups per warp step
    // K1: u = g + c, sign nibbles -> packed words of leaf (segment, worker)
    T fin = T(0);
    // The warp's tasks in order: t = (w * iters + it) * B + b is group
    // g_lo + wid + (it * B + b) * NWARP of worker w (also the TMEM column
    // order).
    const uint32_t iters = g_hi > g_lo + wid ? (g_hi - g_lo - wid + NWARP * B - 1) / (NWARP * B) : 0u;
    // one quad of worker w, group gg: u, the TMEM stash, the packed nibble
    auto consume = [&](uint32_t w, uint32_t gg, uint32_t col, const Quad<T>& gv, const Quad<T>& cv) {
        const uint32_t sl = gg / gps, gl = gg - sl * gps;
        const uint64_t j = uint64_t(gl) * 128 + lane * 4;
        T u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            u[k] = add_rn(add_rn(gv.v[k], cv.v[k]), T(0));  // -0.0 -> +0.0 (sign_vector.hpp:70)
            fin = fma_rn(u[k], T(0), fin);
        }
        if (stash) tmem_put(tbase + col, u);  // warp-uniform
        uint32_t nib = sign_nibble(u[0], u[1], u[2], u[3]);
        const uint64_t valid = j >= p.seg_bits ? 0 : p.seg_bits - j;  // storage padding -> 0
        if (valid < 4) nib &= (1u << valid) - 1u;
        uint32_t v = nib << ((lane & 7) * 4);
        v |= __shfl_xor_sync(kFull, v, 1);
        v |= __shfl_xor_sync(kFull, v, 2);
        v |= __shfl_xor_sync(kFull, v, 4);
        if ((lane & 7) == 0)
            const_cast<uint32_t*>(p.leaves)[(uint64_t(sl) * p.ml + w) * p.wst + uint64_t(gl) * 4 + (lane >> 3)] = v;
    };
    // a quad that is not whole (segment / vector end): element loads, value padding 0
    auto edge_quad = [&](uint32_t w, uint64_t j, uint64_t gi, Quad<T>& gv, Quad<T>& cv) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool in = j + k < p.seg_bits && gi + k < f.dim;
            gv.v[k] = in ? f.g[w][gi + k] : T(0);
            cv.v[k] = in ? f.c[w][gi + k] : T(0);
        }
    };
    if (s.tma_stages) {
        // TMA: one elected thread streams whole workers' slices (g, then c;
        // one bulk copy per segment piece) into a ring of tma_stages stages
        // of shared memory, each completing an mbarrier; the warps consume a
        // stage once its bytes have landed — up to tma_stages x 2 x the
        // slice in flight per SM, no registers held (the register path keeps
        // 64 KB per SM in flight, the loaded-latency limit of the extract)
        __shared__ __align__(8) unsigned long long s_full[kSpreadMaxTmaStages];
        const uint32_t nst = s.tma_stages;
        unsigned char* const ring = reinterpret_cast<unsigned char*>(sp_dyn);
        const uint32_t ring_s = uint32_t(__cvta_generic_to_shared(ring));
        if (tid == 0) {
            for (uint32_t q = 0; q < nst; ++q)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                                 uint32_t(__cvta_generic_to_shared(&s_full[q]))) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        // pieces of the slice: groups [a, b) inside one segment; the whole
        // quads of each (value / storage padding and partial quads are read
        // per element by the consumers)
        auto issue = [&](uint32_t w, uint32_t st) {
            const uint32_t bar = uint32_t(__cvta_generic_to_shared(&s_full[st]));
            uint32_t tx = 0;
            for (int pass = 0; pass < 2; ++pass) {
                if (pass == 1)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
                for (uint32_t a = g_lo; a < g_hi;) {
                    const uint32_t sl = a / gps, b = min(g_hi, (sl + 1) * gps);
                    const uint64_t j0 = uint64_t(a - sl * gps) * 128, seg0 = uint64_t(sl) * p.seg_bits;
                    uint64_t je = min(uint64_t(b - sl * gps) * 128, p.seg_bits);
                    je = min(je, f.dim > seg0 ? f.dim - seg0 : uint64_t(0));
                    const uint64_t n = je > j0 ? (je - j0) & ~3ull : 0;  // whole quads
                    const uint32_t bytes = uint32_t(n * sizeof(T));
                    if (bytes) {
                        if (pass == 0) {
                            tx += 2 * bytes;
                        } else {
                            const uint32_t off = st * 2 * s.tma_half + (a - g_lo) * 128 * uint32_t(sizeof(T));
                            asm volatile(
                                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                ::"r"(ring_s + off), "l"(f.g[w] + seg0 + j0), "r"(bytes), "r"(bar) : "memory");
                            asm volatile(
                                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                ::"r"(ring_s + off + s.tma_half), "l"(f.c[w] + seg0 + j0), "r"(bytes), "r"(bar)
                                : "memory");
                        }
                    }
                    a = b;
                }
            }
        };
        if (tid == 0)
            for (uint32_t w = 0; w < min(nst, f.workers); ++w) issue(w, w);
        for (uint32_t w = 0; w < f.workers; ++w) {
            const uint32_t st = w % nst, par = (w / nst) & 1u;
            const uint32_t bar = uint32_t(__cvta_generic_to_shared(&s_full[st]));
            asm volatile(
                "{\n\t.reg .pred P;\n"
                "WAIT_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
                "@!P bra WAIT_%=;\n}" ::"r"(bar), "r"(par) : "memory");
            const unsigned char* sg = ring + st * 2 * s.tma_half;
            const unsigned char* sc = sg + s.tma_half;
            uint32_t t0 = w * iters * B;
            for (uint32_t g0 = g_lo + wid; g0 < g_hi; g0 += NWARP * B, t0 += B) {
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const uint32_t gg = g0 + b * NWARP;
                    if (gg >= g_hi) break;
                    const uint32_t sl = gg / gps;
                    const uint64_t j = uint64_t(gg - sl * gps) * 128 + lane * 4;
                    const uint64_t gi = uint64_t(sl) * p.seg_bits + j;
                    Quad<T> gv, cv;
                    if (quad_real<T>(j, p.seg_bits, gi, f.dim)) {
                        const uint32_t o = ((gg - g_lo) * 128 + lane * 4) * uint32_t(sizeof(T));
                        gv = *reinterpret_cast<const Quad<T>*>(sg + o);
                        cv = *reinterpret_cast<const Quad<T>*>(sc + o);
                    } else {
                        edge_quad(w, j, gi, gv, cv);
                    }
                    consume(w, gg, (t0 + b) * QCOLS, gv, cv);
                }
            }
            if (w + nst < f.workers) {
                __syncthreads();  // every warp is done with stage st
                if (tid == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(w + nst, st);
                }
            }
        }
        __syncthreads();  // the ring's shared memory is reused by the merge staging
    } else {
        uint32_t t0 = 0;
        for (uint32_t w = 0; w < f.workers; ++w) {
            const T* __restrict__ gw = f.g[w];
            const T* __restrict__ cw = f.c[w];
            for (uint32_t g0 = g_lo + wid; g0 < g_hi; g0 += NWARP * B, t0 += B) {
                Quad<T> gv[B], cv[B];
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const uint32_t gg = g0 + b * NWARP;
                    const uint32_t sl = gg / gps;
                    const uint64_t j = uint64_t(gg - sl * gps) * 128 + lane * 4;
                    const uint64_t gi = uint64_t(sl) * p.seg_bits + j;
                    if (gg < g_hi && quad_real<T>(j, p.seg_bits, gi, f.dim)) {
                        gv[b] = load4(gw + gi);
                        cv[b] = load4(cw + gi);
                    } else if (gg < g_hi) {
                        edge_quad(w, j, gi, gv[b], cv[b]);
                    }
                }
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const uint32_t gg = g0 + b * NWARP;
                    if (gg >= g_hi) break;
                    consume(w, gg, (t0 + b) * QCOLS, gv[b], cv[b]);
                }
            }
        }
    }
    if (__any_sync(kFull, !(fin == fin)) && lane == 0) atomicOr(f.err, 1);
    if (stash) tmem_wait_st();
    if (tid == 0) s_hit = tag_seed == p.seed && tag_round == p.round;
    __syncthreads();
    if (!s_hit && s.n_merges) spread_coins(p, s, s_cbase, cb, p.round, blockIdx.x, gridDim.x);
    // arrive: the last CTA resets the count and advances the generation
    __syncthreads();
    jitter(100);  // checked builds: random arrival order
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(s.sync, 1u) == gridDim.x - 1) {
            s.sync[0] = 0;
            __threadfence();
            atomicAdd(s.sync + 1, 1u);
        }
    }
    const unsigned gen = s_gen + 1;
#ifdef MARSIT_FUSED_PROF
    const uint64_t fp_t1 = threadIdx.x == 0 ? gtime_ns() : 0;
#endif
    // K2: cluster cl < n_seg merges segment cl once every CTA has arrived;
    // meanwhile the other CTAs compute the next round's coins
    const uint32_t n_merge_ctas = p.n_seg * p.csize;
    if (cl >= p.n_seg && s.n_merges && gridDim.x > n_merge_ctas) {
        spread_coins(p, s, s_cbase, cb ^ 1u, p.round + 1, blockIdx.x - n_merge_ctas, gridDim.x - n_merge_ctas);
        if (blockIdx.x == n_merge_ctas && tid == 0) {  // read by the next launch only
            s.tag[2 * (cb ^ 1u)] = p.seed;
            s.tag[2 * (cb ^ 1u) + 1] = p.round + 1;
        }
    }
    if (cl < p.n_seg) {
        jitter(101);
        if (tid == 0) {
            wait_eq_u32(s.sync + 1, gen, f.err);
            // every CTA has read the tag: buffer cb now holds this round's
            // coins (computed above on a miss), tagged for later rounds
            if (blockIdx.x == 0 && s.n_merges) {
                s.tag[2 * cb] = p.seed;
                s.tag[2 * cb + 1] = p.round;
            }
        }
#ifdef MARSIT_FUSED_PROF
        if (prof) atomicAdd(&g_coop_prof[ps + 1], (unsigned long long)(gtime_ns() - fp_t1));  // wait: all arrived
#endif
        __syncthreads();
        // the coin words computed for this round's merges: written in this
        // launch on a tag miss, so read only now (the prologue ran earlier)
        {
            const uint32_t mb = p.seg_begin[cl], nm = p.seg_begin[cl + 1] - mb;
            for (uint32_t i = tid; i < nm; i += kFusedThreads)
                sh.valid[i] = p.coin_valid ? __ldcg(p.coin_valid + mb + i) : 0u;
        }
        // the cluster's tiles of the segment's leaves into shared memory (one
        // L2 round trip: every load of a thread in flight at once)
        const uint32_t tg = p.tile_groups, g_first = cluster_ctarank() * tg;
        const uint32_t n_here = gps > g_first ? min(tg, gps - g_first) : 0u;
        uint4* const leaf = sp_dyn;
        for (uint32_t w = 0; w < f.workers; ++w) {
            const uint4* src = reinterpret_cast<const uint4*>(p.leaves + (uint64_t(cl) * p.ml + w) * p.wst) + g_first;
            for (uint32_t gl = tid; gl < n_here; gl += kFusedThreads) leaf[size_t(w) * tg + gl] = __ldcg(src + gl);
        }
        cluster_sync_all();  // staged leaves and descriptors complete; the cluster runs
        cluster_merge_levels<NSUB, NL, true, false, kFusedThreads>(p, sh, leaf + size_t(f.workers + 1) * tg, leaf,
                                                                    leaf + size_t(f.workers) * tg);
        __syncthreads();
        if (tid == 0) __threadfence();
        cluster_sync_all();  // the segment's aggregate tiles are all written
        jitter(102);
        if (tid == 0 && cluster_ctarank() == 0) st_release_u32(s.sync + 2 + cl, gen);
    }
#ifdef MARSIT_FUSED_PROF
    const uint64_t fp_t2 = threadIdx.x == 0 ? gtime_ns() : 0;
#endif
    // K3/K4 of this CTA's slice once its segments' aggregates are published
    if (g_lo < g_hi) {
        jitter(103);
        if (tid == 0)
            for (uint32_t sl = g_lo / gps; sl <= (g_hi - 1) / gps; ++sl)
                wait_eq_u32(s.sync + 2 + sl, gen, f.err);
#ifdef MARSIT_FUSED_PROF
        if (prof) atomicAdd(&g_coop_prof[ps + 2], (unsigned long long)(gtime_ns() - fp_t2));  // wait: aggregates
#endif
        __syncthreads();
    }
    if (stash) {
        // K3/K4 from the parked u: c' = u - g_t (u's -0.0 was folded to +0.0,
        // which leaves u - g_t unchanged since g_t != 0)
        // the extract parked task (w * iters + it) * B + b at column task * QCOLS
        uint32_t it = 0;
        for (uint32_t g0 = g_lo + wid; g0 < g_hi; g0 += NWARP * B, ++it) {
            uint32_t word[B];  // the groups' aggregate words, once for every worker
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint32_t gg = g0 + b * NWARP;
                if (gg >= g_hi) break;
                const uint32_t sl = gg / gps, gl = gg - sl * gps;
                word[b] = __ldcg(p.agg + uint64_t(p.s_first + sl) * p.agg_stride + uint64_t(gl) * 4 + (lane >> 3));
            }
            for (uint32_t w = 0; w < f.workers; ++w) {
                T* co = f.c_out[w];
                T* upd = w == 0 ? f.update : nullptr;
                const uint32_t colw = (w * iters + it) * B * QCOLS;
                T u[B][4];
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    if (g0 + b * NWARP >= g_hi) break;
                    tmem_get(tbase + colw + b * QCOLS, u[b]);
                }
                tmem_wait_ld();
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const uint32_t gg = g0 + b * NWARP;
                    if (gg >= g_hi) break;
                    const uint32_t sl = gg / gps;
                    const uint64_t j = uint64_t(gg - sl * gps) * 128 + lane * 4;
                    const uint64_t gi = uint64_t(sl) * p.seg_bits + j;
                    const uint32_t nib = (word[b] >> ((lane & 7) * 4)) & 0xFu;
                    Quad<T> out, up;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        up.v[k] = ((nib >> k) & 1u) ? f.eta : -f.eta;
                        out.v[k] = sub_rn(u[b][k], up.v[k]);
                    }
                    if (quad_real<T>(j, p.seg_bits, gi, f.dim)) {
                        store4(co + gi, out);
                        if (upd) store4(upd + gi, up);
                    } else {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (j + k < p.seg_bits && gi + k < f.dim) {
                                co[gi + k] = out.v[k];
                                if (upd) upd[gi + k] = up.v[k];
                            }
                    }
                }
            }
        }
    }
    for (uint32_t w = 0; w < (stash ? 0u : f.workers); ++w) {
        const T* __restrict__ gw = f.g[w];
        const T* cw = f.c[w];  // may alias c_out (in place)
        T* co = f.c_out[w];
        T* upd = w == 0 ? f.update : nullptr;
        for (uint32_t g0 = g_lo + wid; g0 < g_hi; g0 += NWARP * B) {
            Quad<T> gv[B], cv[B];
            uint32_t word[B];
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint32_t gg = g0 + b * NWARP;
                const uint32_t sl = gg / gps, gl = gg - sl * gps;
                const uint64_t j = uint64_t(gl) * 128 + lane * 4;
                const uint64_t gi = uint64_t(sl) * p.seg_bits + j;
                word[b] = 0;
                if (gg < g_hi) {
                    word[b] = __ldcg(p.agg + uint64_t(p.s_first + sl) * p.agg_stride + uint64_t(gl) * 4 + (lane >> 3));
                    if (quad_real<T>(j, p.seg_bits, gi, f.dim)) {
                        gv[b] = load4(gw + gi);
                        cv[b] = load4_rw(cw + gi);
                    }
                }
            }
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const uint32_t gg = g0 + b * NWARP;
                if (gg >= g_hi) break;
                const uint32_t sl = gg / gps;
                const uint64_t j = uint64_t(gg - sl * gps) * 128 + lane * 4;
                const uint64_t gi = uint64_t(sl) * p.seg_bits + j;
                const uint32_t nib = (word[b] >> ((lane & 7) * 4)) & 0xFu;
                if (quad_real<T>(j, p.seg_bits, gi, f.dim)) {
                    Quad<T> out, up;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const T gt = ((nib >> k) & 1u) ? f.eta : -f.eta;
                        out.v[k] = sub_rn(add_rn(gv[b].v[k], cv[b].v[k]), gt);
                        up.v[k] = gt;
                    }
                    store4(co + gi, out);
                    if (upd) store4(upd + gi, up);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (j + k < p.seg_bits && gi + k < f.dim) {
                            const T gt = ((nib >> k) & 1u) ? f.eta : -f.eta;
                            co[gi + k] = sub_rn(add_rn(gw[gi + k], cw[gi + k]), gt);
                            if (upd) upd[gi + k] = gt;
                        }
                }
            }
        }
    }
    if (stash) tmem_release(s_tmem, f.tmem_cols);
#ifdef MARSIT_FUSED_PROF
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const uint64_t fp_t3 = gtime_ns();
        atomicAdd(&g_coop_prof[0], (unsigned long long)(fp_t1 - fp_t0));
        atomicAdd(&g_coop_prof[1], (unsigned long long)(fp_t2 - fp_t1));
        atomicAdd(&g_coop_prof[2], (unsigned long long)(fp_t3 - fp_t2));
        atomicAdd(&g_coop_prof[3], 1ull);
    }
    if (prof && blockIdx.x == gridDim.x - 1)
        atomicAdd(&g_coop_prof[ps + 3], (unsigned long long)(gtime_ns() - fp_t0));  // last CTA: whole launch
#endif
}

// ---------------------------------------------------------------------------
// Aggregate bits in the reference layout: bit j of the whole vector lives in
// segment j / L at offset j % L (sync.hpp:103-112).  One thread per output
// u32 word (two of them form one little-endian u64 word).
// ---------------------------------------------------------------------------
__global__ void export_bits_kernel(const uint32_t* __restrict__ agg, uint32_t wst, uint64_t dim,
                                   uint64_t seg_len, uint64_t n_out, uint32_t* __restrict__ out,
                                   const uint32_t* const* agg_peers, uint32_t s_own) {
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n_out;
         k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t j0 = k * 32;
        uint32_t val = 0;
        if (j0 < dim) {
            const uint32_t n = uint32_t(dim - j0 < 32 ? dim - j0 : 32);
            uint32_t pos = 0;
            while (pos < n) {
                const uint64_t j = j0 + pos;
                const uint64_t s = j / seg_len;
                const uint64_t o = j - s * seg_len;
                uint32_t take = n - pos;
                if (seg_len - o < take) take = uint32_t(seg_len - o);
                const uint32_t* a = (agg_peers ? agg_peers[s / s_own] : agg) + s * wst;
                const uint32_t wi = uint32_t(o >> 5), sh = uint32_t(o & 31);
                uint64_t window = a[wi];
                if (sh + take > 32) window |= uint64_t(a[wi + 1]) << 32;
                uint32_t bits = uint32_t(window >> sh);
                if (take < 32) bits &= (1u << take) - 1u;
                val |= bits << pos;
                pos += take;
            }
        }
        out[k] = val;
    }
}

// ---------------------------------------------------------------------------
// Consensus hashes (see launch_seg_hash): blockIdx.y = segment, grid-stride
// over its words, XOR-reduced per warp, one atomic per warp.
// ---------------------------------------------------------------------------
__global__ void seg_hash_kernel(const uint32_t* agg, const uint32_t* const* agg_peers,
                                uint32_t s_own, uint32_t wsa, uint32_t wst, uint32_t words_proc,
                                uint32_t s0, unsigned long long* out) {
    const uint32_t s = s0 + blockIdx.y;
    const uint32_t* row = (agg_peers ? agg_peers[s / s_own] : agg) + uint64_t(s) * wsa;
    const uint64_t salt = (uint64_t(s) + 1) * kGamma;
    uint64_t h = 0;
    for (uint32_t wi = blockIdx.x * blockDim.x + threadIdx.x; wi < words_proc;
         wi += gridDim.x * blockDim.x)
        h ^= mix64(((uint64_t(wi) << 32) | __ldcg(row + wi)) + salt);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h ^= __shfl_xor_sync(kFull, h, o);
    if ((threadIdx.x & 31) == 0 && h) {
        unsigned long long* dst =
            out ? out + s : reinterpret_cast<unsigned long long*>(const_cast<uint32_t*>(row) + wst);
        atomicXor(dst, (unsigned long long)h);
    }
}

__global__ void hash_compare_kernel(const uint32_t* agg, const uint32_t* const* agg_peers,
                                    uint32_t s_own, uint32_t wsa, uint32_t wst, uint32_t n_seg,
                                    const unsigned long long* verify, int* err) {
    for (uint32_t s = threadIdx.x; s < n_seg; s += blockDim.x) {
        const uint32_t* row = (agg_peers ? agg_peers[s / s_own] : agg) + uint64_t(s) * wsa;
        const unsigned long long stored =
            __ldcg(reinterpret_cast<const unsigned long long*>(row + wst));
        if (stored != verify[s]) atomicOr(err, 2);
    }
}

// x_w -= v (dense-round parameter update, trainer.hpp:285-288)
template <typename T>
__global__ void sub_update_kernel(StreamParams<T> p, const T* __restrict__ v) {
    const uint64_t n = p.dim * p.ml;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t w = uint32_t(i / p.dim);
        const uint64_t j = i - uint64_t(w) * p.dim;
        p.x[w][j] = sub_rn(p.x[w][j], v[j]);
    }
}

// ---------------------------------------------------------------------------
// Synthetic inputs: g_j from draw j of RngStream(seed,
// trial, w, t, 0).  recipe 0: ((x>>51) - 4096)·2^-20; recipe 1 (correlated):
// shared ((x_a>>52) - 2048) + per-worker ((x_b>>53) - 1024), ·2^-20.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void fill_recipe_kernel(int recipe, uint64_t seed, uint64_t worker, uint64_t round,
                                   uint64_t dim, T* __restrict__ out) {
    const uint64_t kb = stream_key(seed, 6, worker, round, 0);
    const uint64_t ka = stream_key(seed, 6, 0xFFFF, round, 0);
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < dim;
         j += uint64_t(gridDim.x) * blockDim.x) {
        int64_t q;
        if (recipe == 0) {
            q = int64_t(mix64(kb + (j + 1) * kGamma) >> 51) - 4096;
        } else {
            q = (int64_t(mix64(ka + (j + 1) * kGamma) >> 52) - 2048) +
                (int64_t(mix64(kb + (j + 1) * kGamma) >> 53) - 1024);
        }
        out[j] = T(double(q) * 0x1.0p-20);
    }
}

// ---------------------------------------------------------------------------
// Dense round.  dense_leaf_kernel (multi-rank): u = g + c of the local
// workers, laid out per destination rank for the exchange:
// u_send[q][sl][wl][L] (segment q*s_own + sl).  dense_reduce_kernel: per
// coordinate of an owned segment, evaluate the schedule's reduction tree in
// double (state[to][s] = add(state[to][s], p), allreduce.hpp:114-116),
// scale by 1/M (120-126).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void dense_leaf_kernel(const DenseParams<T> p, uint32_t s_own, uint32_t n_seg_total,
                                  T* __restrict__ u_send) {
    const uint64_t per_w = uint64_t(n_seg_total) * p.seg_len;
    const uint64_t n = per_w * p.ml;
    bool bad = false;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t wl = uint32_t(i / per_w);
        const uint64_t jj = i - uint64_t(wl) * per_w;  // padded coordinate
        const uint32_t s = uint32_t(jj / p.seg_len);
        const uint64_t o = jj - uint64_t(s) * p.seg_len;
        T u = T(0);
        if (jj < p.dim) {
            const T gg = p.src[2 * wl][jj], cc = p.src[2 * wl + 1][jj];
            u = add_rn(gg, cc);
            bad |= !(finite(gg) && finite(cc) && finite(u));
            if (p.c_zero[wl]) p.c_zero[wl][jj] = T(0);  // after the read (c may alias)
        }
        const uint32_t q = s / s_own, sl = s % s_own;
        u_send[((uint64_t(q) * s_own + sl) * p.ml + wl) * p.seg_len + o] = u;
    }
    if (bad) atomicOr(p.err, 1);
}

// Node values of the reduction tree live in shared memory
// ([node][kDenseThreads], conflict-free); a node index is data, so a
// register array would spill to local memory.
constexpr int kDenseThreads = 128;
template <typename T>
__global__ void __launch_bounds__(kDenseThreads) dense_reduce_kernel(const DenseParams<T> p) {
    extern __shared__ double dval[];  // [workers + n_ops][kDenseThreads]
    const int tid = threadIdx.x;
    const uint64_t n = uint64_t(p.n_seg) * p.seg_len;
    bool bad = false;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + tid; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t sl = uint32_t(i / p.seg_len);
        const uint64_t o = i - uint64_t(sl) * p.seg_len;
        const uint64_t j = uint64_t(p.s_first + sl) * p.seg_len + o;  // global coordinate
        if (p.mode == 0) {
            // loads in groups of 8 workers (16 independent loads in flight)
            const bool in = j < p.dim;
            for (uint32_t w0 = 0; w0 < p.workers; w0 += 8) {
                T gg[8], cc[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const bool ok = in && w0 + k < p.workers;
                    gg[k] = ok ? p.src[2 * (w0 + k)][j] : T(0);
                    cc[k] = ok ? p.src[2 * (w0 + k) + 1][j] : T(0);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (w0 + k >= p.workers) break;
                    const T uu = add_rn(gg[k], cc[k]);  // value padding: 0 + 0
                    bad |= !(finite(gg[k]) && finite(cc[k]) && finite(uu));
                    dval[(w0 + k) * kDenseThreads + tid] = double(uu);
                    if (in && p.c_zero[w0 + k]) p.c_zero[w0 + k][j] = T(0);  // after the read
                }
            }
        } else if (p.mode == 1) {
            for (uint32_t w = 0; w < p.workers; ++w) {
                const uint32_t src_rank = w / p.ml, wl = w % p.ml;
                dval[w * kDenseThreads + tid] = double(
                    p.u_buf[((uint64_t(src_rank) * p.n_seg + sl) * p.ml + wl) * p.seg_len + o]);
            }
        } else {  // P2P: straight out of the source rank's [S][ml][L] buffer
            for (uint32_t w = 0; w < p.workers; ++w) {
                const uint32_t src_rank = w / p.ml, wl = w % p.ml;
                dval[w * kDenseThreads + tid] = double(
                    p.u_peers[src_rank][((uint64_t(p.s_first) + sl) * p.ml + wl) * p.seg_len + o]);
            }
        }
        const DenseOp* ops = p.ops + uint64_t(sl) * p.n_ops;
        for (uint32_t k = 0; k < p.n_ops; ++k) {
            const double v = __dadd_rn(dval[ops[k].a * kDenseThreads + tid],
                                       dval[ops[k].b * kDenseThreads + tid]);
            bad |= !isfinite(v);
            dval[(p.workers + k) * kDenseThreads + tid] = v;
        }
        if (j < p.dim)
            p.mean[j] = T(__dmul_rn(dval[p.final_node[sl] * kDenseThreads + tid], p.inv_m));
    }
    if (bad) atomicOr(p.err, 1);
}

// Chain-of-chains plans (ring: one chain; torus: one chain per row, then a
// chain over the row results): the leaves of a segment are visited in
// `chain` order; within a group v_0 = u[c_0], v_k = u[c_k] + v_{k-1} (the
// receiver's state plus the received partial, allreduce.hpp:114-116, IEEE
// addition being commutative), and where bit k of `chain_groups` is set the
// group's value is folded into the outer chain the same way.  Leaves are
// loaded in chain order straight into registers (static indices) — no
// shared-memory staging — 16 loads in flight per group of 8 workers.  MODE 0: leaves
// g + c (one GPU), with the compensation reset fused; 1: exchanged u buffer;
// 2: peers' u buffers (P2P).
template <typename T, int MODE, bool MULTI>
__global__ void __launch_bounds__(256) dense_chain_kernel(const DenseParams<T> p) {
    const uint64_t n = uint64_t(p.n_seg) * p.seg_len;
    bool bad = false;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t sl = uint32_t(i / p.seg_len);
        const uint64_t o = i - uint64_t(sl) * p.seg_len;
        const uint64_t j = uint64_t(p.s_first + sl) * p.seg_len + o;  // global coordinate
        if (j >= p.dim) continue;  // value padding never reaches the output
        const uint16_t* ch = p.chain + uint64_t(sl) * p.workers;
        const uint64_t gm = MULTI ? p.chain_groups[sl] : (1ull << (p.workers - 1));
        double acc = 0.0, out = 0.0;
        bool first_in = true, first_out = true;
        for (uint32_t k0 = 0; k0 < p.workers; k0 += 8) {
            T u[8];
            if (MODE == 0) {
                T gg[8], cc[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const bool ok = k0 + k < p.workers;
                    const uint32_t w = ok ? ch[k0 + k] : 0u;
                    gg[k] = ok ? p.src[2 * w][j] : T(0);
                    cc[k] = ok ? p.src[2 * w + 1][j] : T(0);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    u[k] = add_rn(gg[k], cc[k]);
                    bad |= !(finite(gg[k]) && finite(cc[k]) && finite(u[k]));
                    if (k0 + k < p.workers) {
                        T* z = p.c_zero[ch[k0 + k]];
                        if (z) z[j] = T(0);  // after the read (c may alias)
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const bool ok = k0 + k < p.workers;
                    const uint32_t w = ok ? ch[k0 + k] : 0u;
                    const uint32_t src_rank = w / p.ml, wl = w % p.ml;
                    if (!ok)
                        u[k] = T(0);
                    else if (MODE == 1)
                        u[k] = p.u_buf[((uint64_t(src_rank) * p.n_seg + sl) * p.ml + wl) * p.seg_len + o];
                    else
                        u[k] = p.u_peers[src_rank][((uint64_t(p.s_first) + sl) * p.ml + wl) * p.seg_len + o];
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (k0 + k >= p.workers) break;
                acc = first_in ? double(u[k]) : __dadd_rn(double(u[k]), acc);
                bad |= !isfinite(acc);
                first_in = false;
                if ((gm >> (k0 + k)) & 1) {  // a group's chain ends: fold into the outer chain
                    out = first_out ? acc : __dadd_rn(acc, out);
                    bad |= !isfinite(out);
                    first_out = false;
                    first_in = true;
                }
            }
        }
        p.mean[j] = T(__dmul_rn(out, p.inv_m));
    }
    if (bad) atomicOr(p.err, 1);
}

// dense_chain_kernel, one-GPU leaves, 4 consecutive coordinates per thread
// (16-byte loads; needs L and D multiples of 4 and aligned g, c, c', mean).
template <typename T, bool MULTI>
__global__ void __launch_bounds__(256) dense_chain4_kernel(const DenseParams<T> p) {
    const uint64_t n4 = uint64_t(p.n_seg) * p.seg_len / 4;
    bool bad = false;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n4;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i0 = i * 4;
        const uint32_t sl = uint32_t(i0 / p.seg_len);
        const uint64_t o = i0 - uint64_t(sl) * p.seg_len;
        const uint64_t j = uint64_t(p.s_first + sl) * p.seg_len + o;
        if (j >= p.dim) continue;
        const uint16_t* ch = p.chain + uint64_t(sl) * p.workers;
        const uint64_t gm = MULTI ? p.chain_groups[sl] : (1ull << (p.workers - 1));
        double acc[4] = {0.0, 0.0, 0.0, 0.0}, out[4] = {0.0, 0.0, 0.0, 0.0};
        bool first_in = true, first_out = true;
        for (uint32_t k0 = 0; k0 < p.workers; k0 += 8) {
            Quad<T> gq[8], cq[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (k0 + k < p.workers) {
                    const uint32_t w = ch[k0 + k];
                    gq[k] = load4(p.src[2 * w] + j);
                    cq[k] = load4_rw(p.src[2 * w + 1] + j);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) gq[k].v[e] = cq[k].v[e] = T(0);
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (k0 + k >= p.workers) break;
                Quad<T> zero;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const T u = add_rn(gq[k].v[e], cq[k].v[e]);
                    bad |= !(finite(gq[k].v[e]) && finite(cq[k].v[e]) && finite(u));
                    acc[e] = first_in ? double(u) : __dadd_rn(double(u), acc[e]);
                    bad |= !isfinite(acc[e]);
                    zero.v[e] = T(0);
                }
                first_in = false;
                if ((gm >> (k0 + k)) & 1) {  // a group's chain ends: fold into the outer chain
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        out[e] = first_out ? acc[e] : __dadd_rn(acc[e], out[e]);
                        bad |= !isfinite(out[e]);
                    }
                    first_out = false;
                    first_in = true;
                }
                T* z = p.c_zero[ch[k0 + k]];
                if (z) store4(z + j, zero);  // after the read (c may alias)
            }
        }
        Quad<T> m;
#pragma unroll
        for (int e = 0; e < 4; ++e) m.v[e] = T(__dmul_rn(out[e], p.inv_m));
        store4(p.mean + j, m);
    }
    if (bad) atomicOr(p.err, 1);
}

// General reduction DAG (torus plans), one-GPU leaves, 4 consecutive
// coordinates per thread with 16-byte loads (same eligibility as
// dense_chain4_kernel); node values in shared memory as
// [node][coordinate of the quad][kDenseThreads] doubles (conflict-free).
template <typename T>
__global__ void __launch_bounds__(kDenseThreads) dense_dag4_kernel(const DenseParams<T> p) {
    extern __shared__ double dval[];  // [workers + n_ops][4][kDenseThreads]
    const int tid = threadIdx.x;
    const uint64_t n4 = uint64_t(p.n_seg) * p.seg_len / 4;
    bool bad = false;
    auto at = [&](uint32_t node, int e) -> double& { return dval[(node * 4 + e) * kDenseThreads + tid]; };
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + tid; i < n4;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i0 = i * 4;
        const uint32_t sl = uint32_t(i0 / p.seg_len);
        const uint64_t o = i0 - uint64_t(sl) * p.seg_len;
        const uint64_t j = uint64_t(p.s_first + sl) * p.seg_len + o;
        if (j >= p.dim) continue;  // value padding never reaches the output
        for (uint32_t w0 = 0; w0 < p.workers; w0 += 8) {
            Quad<T> gq[8], cq[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (w0 + k < p.workers) {
                    gq[k] = load4(p.src[2 * (w0 + k)] + j);
                    cq[k] = load4_rw(p.src[2 * (w0 + k) + 1] + j);
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (w0 + k >= p.workers) break;
                Quad<T> zero;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const T u = add_rn(gq[k].v[e], cq[k].v[e]);
                    bad |= !(finite(gq[k].v[e]) && finite(cq[k].v[e]) && finite(u));
                    at(w0 + k, e) = double(u);
                    zero.v[e] = T(0);
                }
                T* z = p.c_zero[w0 + k];
                if (z) store4(z + j, zero);  // after the read (c may alias)
            }
        }
        const DenseOp* ops = p.ops + uint64_t(sl) * p.n_ops;
        for (uint32_t k = 0; k < p.n_ops; ++k) {
            const DenseOp op = ops[k];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const double v = __dadd_rn(at(op.a, e), at(op.b, e));
                bad |= !isfinite(v);
                at(p.workers + k, e) = v;
            }
        }
        const uint32_t fin = p.final_node[sl];
        Quad<T> m;
#pragma unroll
        for (int e = 0; e < 4; ++e) m.v[e] = T(__dmul_rn(at(fin, e), p.inv_m));
        store4(p.mean + j, m);
    }
    if (bad) atomicOr(p.err, 1);
}

}  // namespace

// ---------------------------------------------------------------------------
// Launch wrappers
// ---------------------------------------------------------------------------
template <typename T>
cudaError_t launch_extract(const StreamParams<T>& p, bool vec, int grid, cudaStream_t st) {
    if (vec)
        extract_kernel<T, true><<<grid, kStreamThreads, 0, st>>>(p);
    else
        extract_kernel<T, false><<<grid, kStreamThreads, 0, st>>>(p);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_decode(const StreamParams<T>& p, bool vec, int grid, cudaStream_t st) {
    if (p.matches) {
        if (vec)
            decode_stats_kernel<T, true><<<grid, kStreamThreads, 0, st>>>(p);
        else
            decode_stats_kernel<T, false><<<grid, kStreamThreads, 0, st>>>(p);
    } else {
        bool xu = false;
        for (uint32_t w = 0; w < p.ml; ++w) xu |= p.x[w] != nullptr;
        if (xu) {
            if (vec)
                decode_kernel<T, true, true><<<grid, kStreamThreads, 0, st>>>(p);
            else
                decode_kernel<T, false, true><<<grid, kStreamThreads, 0, st>>>(p);
        } else if (vec)
            decode_kernel<T, true, false><<<grid, kStreamThreads, 0, st>>>(p);
        else
            decode_kernel<T, false, false><<<grid, kStreamThreads, 0, st>>>(p);
    }
    return cudaGetLastError();
}



template <int WPT>
static cudaError_t coop_attr() {  // dynamic shared memory beyond 48 KB (slots)
    static cudaError_t e = cudaFuncSetAttribute(merge_coop_kernel<WPT>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                200 * 1024);
    return e;
}

template <int WPT>
static cudaError_t coop_launch_t(const CoopParams& p, size_t smem, cudaStream_t st) {
    cudaError_t e = coop_attr<WPT>();
    if (e != cudaSuccess) return e;
    CoopParams q = p;
    void* args[] = {&q};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(merge_coop_kernel<WPT>),
                                       dim3(p.seg_cnt * p.n_lanes * p.part_tiles), dim3(kMergeThreads), args,
                                       smem, st);
}

template <int WPT>
static cudaError_t coop_occ_t(size_t smem, int* blocks) {
    cudaError_t e = coop_attr<WPT>();
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, merge_coop_kernel<WPT>,
                                                         kMergeThreads, smem);
}

cudaError_t launch_merge_coop(const CoopParams& p, int wpt, size_t smem, cudaStream_t st) {
    switch (wpt) {
        case 1: return coop_launch_t<1>(p, smem, st);
        case 2: return coop_launch_t<2>(p, smem, st);
        case 4: return coop_launch_t<4>(p, smem, st);
        case 8: return coop_launch_t<8>(p, smem, st);
        case 12: return coop_launch_t<12>(p, smem, st);
        case 16: return coop_launch_t<16>(p, smem, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t merge_coop_occupancy(int wpt, size_t smem, int* blocks) {
    switch (wpt) {
        case 1: return coop_occ_t<1>(smem, blocks);
        case 2: return coop_occ_t<2>(smem, blocks);
        case 4: return coop_occ_t<4>(smem, blocks);
        case 8: return coop_occ_t<8>(smem, blocks);
        case 12: return coop_occ_t<12>(smem, blocks);
        case 16: return coop_occ_t<16>(smem, blocks);
        default: return cudaErrorInvalidValue;
    }
}

template <int NSUB, int NL>
static cudaError_t cluster_attr(size_t smem) {
    auto k = merge_cluster_kernel<NSUB, NL>;
    static cudaError_t e = [&] {
        cudaError_t r = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        return r;
    }();
    (void)smem;
    return e;
}

template <int NSUB, int NL>
static cudaError_t cluster_launch_t(const ClusterParams& p, uint32_t clusters, size_t smem,
                                    cudaStream_t st) {
    cudaError_t e = cluster_attr<NSUB, NL>(smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(clusters * p.csize);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, merge_cluster_kernel<NSUB, NL>, p);
}

template <int NSUB, int NL>
static cudaError_t cluster_occ_t(uint32_t csize, size_t smem, int* clusters) {
    cudaError_t e = cluster_attr<NSUB, NL>(smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(csize);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(clusters, merge_cluster_kernel<NSUB, NL>, &cfg);
}

#define MARSIT_CLUSTER_DISPATCH(FN, ...)                                 \
    switch (nl * 100 + nsub) {                                           \
        case 101: return FN<1, 1>(__VA_ARGS__);                          \
        case 102: return FN<2, 1>(__VA_ARGS__);                          \
        case 104: return FN<4, 1>(__VA_ARGS__);                          \
        case 108: return FN<8, 1>(__VA_ARGS__);                          \
        case 116: return FN<16, 1>(__VA_ARGS__);                         \
        case 201: return FN<1, 2>(__VA_ARGS__);                          \
        case 202: return FN<2, 2>(__VA_ARGS__);                          \
        case 204: return FN<4, 2>(__VA_ARGS__);                          \
        case 208: return FN<8, 2>(__VA_ARGS__);                          \
        default: return cudaErrorInvalidValue;                           \
    }

template <typename T, int NSUB, int NL>
static cudaError_t fused_attr() {
    auto k = round_cluster_kernel<T, NSUB, NL>;
    static cudaError_t e = [&] {
        cudaError_t r = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncAttributes fa{};
        if (r == cudaSuccess) r = cudaFuncGetAttributes(&fa, k);
        // the opt-in maximum per CTA (227 KB on sm_100) less the static shared memory
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(232448 - fa.sharedSizeBytes));
        return r;
    }();
    return e;
}

template <typename T, int NSUB, int NL>
static cudaError_t fused_launch_t(const ClusterParams& p, const FusedParams<T>& f, uint32_t clusters,
                                  size_t smem, cudaStream_t st) {
    cudaError_t e = fused_attr<T, NSUB, NL>();
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(clusters * p.csize);
    cfg.blockDim = dim3(kFusedThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, round_cluster_kernel<T, NSUB, NL>, p, f);
}

template <typename T, int NSUB, int NL>
static cudaError_t fused_occ_t(uint32_t csize, size_t smem, int* clusters) {
    cudaError_t e = fused_attr<T, NSUB, NL>();
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(csize);
    cfg.blockDim = dim3(kFusedThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(clusters, round_cluster_kernel<T, NSUB, NL>, &cfg);
}

#define MARSIT_FUSED_DISPATCH(FN, ...)                                   \
    switch (nl * 100 + nsub) {                                           \
        case 101: return FN<T, 1, 1>(__VA_ARGS__);                       \
        case 102: return FN<T, 2, 1>(__VA_ARGS__);                       \
        case 104: return FN<T, 4, 1>(__VA_ARGS__);                       \
        case 201: return FN<T, 1, 2>(__VA_ARGS__);                       \
        case 202: return FN<T, 2, 2>(__VA_ARGS__);                       \
        case 204: return FN<T, 4, 2>(__VA_ARGS__);                       \
        default: return cudaErrorInvalidValue;                           \
    }

template <typename T>
cudaError_t launch_round_cluster(const ClusterParams& p, const FusedParams<T>& f, int nsub, int nl,
                                 uint32_t clusters, size_t smem, cudaStream_t st) {
    MARSIT_FUSED_DISPATCH(fused_launch_t, p, f, clusters, smem, st)
}

template <typename T>
cudaError_t round_cluster_occupancy(int nsub, int nl, uint32_t csize, size_t smem, int* clusters) {
    MARSIT_FUSED_DISPATCH(fused_occ_t, csize, smem, clusters)
}

template <typename T, int NSUB, int NL>
static cudaError_t spread_attr() {
    auto k = round_spread_kernel<T, NSUB, NL>;
    static cudaError_t e = [&] {
        cudaError_t r = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncAttributes fa{};
        if (r == cudaSuccess) r = cudaFuncGetAttributes(&fa, k);
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(232448 - fa.sharedSizeBytes));
        return r;
    }();
    return e;
}

template <typename T, int NSUB, int NL>
static cudaError_t spread_launch_t(const ClusterParams& p, const SpreadParams<T>& s, uint32_t ctas,
                                   size_t smem, bool cooperative, cudaStream_t st) {
    cudaError_t e = spread_attr<T, NSUB, NL>();
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kFusedThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cooperative ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, round_spread_kernel<T, NSUB, NL>, p, s);
}

template <typename T, int NSUB, int NL>
static cudaError_t spread_occ_t(uint32_t csize, size_t smem, int* clusters) {
    cudaError_t e = spread_attr<T, NSUB, NL>();
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(csize);
    cfg.blockDim = dim3(kFusedThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(clusters, round_spread_kernel<T, NSUB, NL>, &cfg);
}

template <typename T>
cudaError_t launch_round_spread(const ClusterParams& p, const SpreadParams<T>& s, int nsub, int nl,
                                uint32_t ctas, size_t smem, bool cooperative, cudaStream_t st) {
    MARSIT_FUSED_DISPATCH(spread_launch_t, p, s, ctas, smem, cooperative, st)
}

template <typename T>
cudaError_t round_spread_occupancy(int nsub, int nl, uint32_t csize, size_t smem, int* clusters) {
    MARSIT_FUSED_DISPATCH(spread_occ_t, csize, smem, clusters)
}

template <int NSUB, int NL, int NT = kClusterThreads>
static cudaError_t grid_attr() {
    static cudaError_t e = cudaFuncSetAttribute(merge_grid_kernel<NSUB, NL, NT>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return e;
}

template <int NSUB, int NL, int NT = kClusterThreads>
static cudaError_t grid_launch_t(const ClusterParams& p, uint32_t segments, size_t smem, cudaStream_t st) {
    cudaError_t e = grid_attr<NSUB, NL, NT>();
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(segments * p.csize);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = p.grid_coop ? 1 : 0;  // the grid is the co-resident CTA count either way
    return cudaLaunchKernelEx(&cfg, merge_grid_kernel<NSUB, NL, NT>, p);
}

template <int NSUB, int NL, int NT = kClusterThreads>
static cudaError_t grid_occ_t(size_t smem, int* blocks) {
    cudaError_t e = grid_attr<NSUB, NL, NT>();
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, merge_grid_kernel<NSUB, NL, NT>, NT, smem);
}

cudaError_t launch_merge_grid(const ClusterParams& p, int nsub, int nl, uint32_t segments, size_t smem,
                              int nt, cudaStream_t st) {
    if (nt == 256 || nt == 512) {
        if (nsub != 1) return cudaErrorInvalidValue;
        if (nt == 256)
            return nl == 1 ? grid_launch_t<1, 1, 256>(p, segments, smem, st) : grid_launch_t<1, 2, 256>(p, segments, smem, st);
        return nl == 1 ? grid_launch_t<1, 1, 512>(p, segments, smem, st) : grid_launch_t<1, 2, 512>(p, segments, smem, st);
    }
    MARSIT_CLUSTER_DISPATCH(grid_launch_t, p, segments, smem, st)
}

cudaError_t merge_grid_occupancy(int nsub, int nl, size_t smem, int nt, int* blocks) {
    if (nt == 256 || nt == 512) {
        if (nsub != 1) return cudaErrorInvalidValue;
        if (nt == 256) return nl == 1 ? grid_occ_t<1, 1, 256>(smem, blocks) : grid_occ_t<1, 2, 256>(smem, blocks);
        return nl == 1 ? grid_occ_t<1, 1, 512>(smem, blocks) : grid_occ_t<1, 2, 512>(smem, blocks);
    }
    MARSIT_CLUSTER_DISPATCH(grid_occ_t, smem, blocks)
}

cudaError_t launch_merge_cluster(const ClusterParams& p, int nsub, int nl, uint32_t clusters,
                                 size_t smem, cudaStream_t st) {
    MARSIT_CLUSTER_DISPATCH(cluster_launch_t, p, clusters, smem, st)
}

cudaError_t merge_cluster_occupancy(int nsub, int nl, uint32_t csize, size_t smem, int* clusters) {
    MARSIT_CLUSTER_DISPATCH(cluster_occ_t, csize, smem, clusters)
}

cudaError_t stream_occupancy(bool f64, int* extract_blocks, int* decode_blocks) {
    cudaError_t e;
    if (f64) {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(extract_blocks,
                                                          extract_kernel<double, true>,
                                                          kStreamThreads, 0);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(decode_blocks,
                                                              decode_kernel<double, true, false>,
                                                              kStreamThreads, 0);
    } else {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(extract_blocks,
                                                          extract_kernel<float, true>,
                                                          kStreamThreads, 0);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(decode_blocks,
                                                              decode_kernel<float, true, false>,
                                                              kStreamThreads, 0);
    }
    return e;
}


cudaError_t launch_coins(const DevMerge* merges, uint32_t n_merges, uint64_t seed, uint64_t round,
                         const uint64_t* coin_end, uint32_t* coin_valid,
                         uint32_t* coins, int grid_x, cudaStream_t st) {
    if (n_merges == 0) return cudaSuccess;
    coins_kernel<<<dim3(grid_x, n_merges), 256, 0, st>>>(merges, seed, round, coin_end, coin_valid,
                                                        coins);
    return cudaGetLastError();
}

cudaError_t launch_export_bits(const uint32_t* agg, uint32_t wst, uint64_t dim, uint64_t seg_len,
                               uint32_t* out_u32, cudaStream_t st,
                               const uint32_t* const* agg_peers, uint32_t s_own) {
    const uint64_t n_out = ((dim + 63) / 64) * 2;
    const int threads = 256;
    uint64_t blocks = (n_out + threads - 1) / threads;
    if (blocks > 148 * 8) blocks = 148 * 8;
    export_bits_kernel<<<int(blocks), threads, 0, st>>>(agg, wst, dim, seg_len, n_out, out_u32,
                                                        agg_peers, s_own);
    return cudaGetLastError();
}

cudaError_t launch_seg_hash(const uint32_t* agg, const uint32_t* const* agg_peers, uint32_t s_own,
                            uint32_t wsa, uint32_t wst, uint32_t words_proc, uint32_t s0,
                            uint32_t n_seg, unsigned long long* out, cudaStream_t st) {
    if (n_seg == 0) return cudaSuccess;
    uint32_t gx = (words_proc + 256 * 16 - 1) / (256 * 16);
    gx = gx < 1 ? 1 : (gx > 64 ? 64 : gx);
    seg_hash_kernel<<<dim3(gx, n_seg), 256, 0, st>>>(agg, agg_peers, s_own, wsa, wst, words_proc, s0,
                                                     out);
    return cudaGetLastError();
}

cudaError_t launch_hash_compare(const uint32_t* agg, const uint32_t* const* agg_peers,
                                uint32_t s_own, uint32_t wsa, uint32_t wst, uint32_t n_seg,
                                const unsigned long long* verify, int* err, cudaStream_t st) {
    hash_compare_kernel<<<1, 256, 0, st>>>(agg, agg_peers, s_own, wsa, wst, n_seg, verify, err);
    return cudaGetLastError();
}

__global__ void flag_write_kernel(const FlagSlots s, unsigned long long value) {
    __threadfence_system();  // the stream's earlier writes are visible system-wide first
    for (uint32_t i = threadIdx.x; i < s.n; i += blockDim.x)
        *reinterpret_cast<volatile unsigned long long*>(s.slot[i]) = value;
}

cudaError_t launch_flag_write(const FlagSlots& s, unsigned long long value, cudaStream_t st) {
    flag_write_kernel<<<1, 32, 0, st>>>(s, value);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_fill_recipe(int recipe, uint64_t seed, uint64_t worker, uint64_t round,
                               uint64_t dim, T* out, cudaStream_t st) {
    uint64_t blocks = (dim + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks == 0) blocks = 1;
    fill_recipe_kernel<T><<<int(blocks), 256, 0, st>>>(recipe, seed, worker, round, dim, out);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_sub_update(T* const* x, uint32_t ml, const T* v, uint64_t dim, int grid,
                              cudaStream_t st) {
    StreamParams<T> p{};
    for (uint32_t w = 0; w < ml; ++w) p.x[w] = x[w];
    p.ml = ml;
    p.dim = dim;
    sub_update_kernel<T><<<grid, 256, 0, st>>>(p, v);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_dense_reduce(const DenseParams<T>& p, int grid, cudaStream_t st) {
    if (p.chain) {
        if (p.chain_multi) {
            if (p.mode == 0 && p.vec4)
                dense_chain4_kernel<T, true><<<grid, 256, 0, st>>>(p);
            else if (p.mode == 0)
                dense_chain_kernel<T, 0, true><<<grid, 256, 0, st>>>(p);
            else if (p.mode == 1)
                dense_chain_kernel<T, 1, true><<<grid, 256, 0, st>>>(p);
            else
                dense_chain_kernel<T, 2, true><<<grid, 256, 0, st>>>(p);
        } else {
            if (p.mode == 0 && p.vec4)
                dense_chain4_kernel<T, false><<<grid, 256, 0, st>>>(p);
            else if (p.mode == 0)
                dense_chain_kernel<T, 0, false><<<grid, 256, 0, st>>>(p);
            else if (p.mode == 1)
                dense_chain_kernel<T, 1, false><<<grid, 256, 0, st>>>(p);
            else
                dense_chain_kernel<T, 2, false><<<grid, 256, 0, st>>>(p);
        }
        return cudaGetLastError();
    }
    if (p.mode == 0 && p.vec4) {
        const size_t smem4 = size_t(p.workers + p.n_ops) * 4 * kDenseThreads * sizeof(double);
        if (smem4 <= 200 * 1024) {
            if (smem4 > 48 * 1024) {
                cudaError_t e = cudaFuncSetAttribute(dense_dag4_kernel<T>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     int(smem4));
                if (e != cudaSuccess) return e;
            }
            dense_dag4_kernel<T><<<grid * 2, kDenseThreads, smem4, st>>>(p);
            return cudaGetLastError();
        }
    }
    const size_t smem = size_t(p.workers + p.n_ops) * kDenseThreads * sizeof(double);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(dense_reduce_kernel<T>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
    }
    dense_reduce_kernel<T><<<grid * 2, kDenseThreads, smem, st>>>(p);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_dense_leaf(const T* const* g, const T* const* c, uint32_t ml, uint64_t dim,
                              uint64_t seg_len, uint32_t n_seg_total, uint32_t s_own, T* u_send,
                              int* err, int grid, cudaStream_t st, T* const* c_zero) {
    DenseParams<T> p{};
    for (uint32_t w = 0; w < ml; ++w) {
        p.src[2 * w] = g[w];
        p.src[2 * w + 1] = c[w];
        p.c_zero[w] = c_zero ? c_zero[w] : nullptr;
    }
    p.ml = ml;
    p.dim = dim;
    p.seg_len = seg_len;
    p.err = err;
    dense_leaf_kernel<T><<<grid, 256, 0, st>>>(p, s_own, n_seg_total, u_send);
    return cudaGetLastError();
}

// Load every kernel of this library now (CUDA's default lazy loading would
// do it at first launch, which must wait for the device to go quiet — with
// P2P ranks whose streams wait on each other's flags inside one process, a
// first launch after such a wait was enqueued could never return).
cudaError_t preload_kernels() {
    // modules load per device: once for every device this process uses
    static std::mutex mu;
    static std::vector<int> done;
    int dev = 0;
    cudaError_t e0 = cudaGetDevice(&dev);
    if (e0 != cudaSuccess) return e0;
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(done.begin(), done.end(), dev) != done.end()) return cudaSuccess;
    const cudaError_t result = [] {
        const void* fns[] = {
            reinterpret_cast<const void*>(extract_kernel<float, true>),
            reinterpret_cast<const void*>(extract_kernel<float, false>),
            reinterpret_cast<const void*>(extract_kernel<double, true>),
            reinterpret_cast<const void*>(extract_kernel<double, false>),
            reinterpret_cast<const void*>(decode_kernel<float, true, false>),
            reinterpret_cast<const void*>(decode_kernel<float, false, false>),
            reinterpret_cast<const void*>(decode_kernel<double, true, false>),
            reinterpret_cast<const void*>(decode_kernel<double, false, false>),
            reinterpret_cast<const void*>(decode_kernel<float, true, true>),
            reinterpret_cast<const void*>(decode_kernel<float, false, true>),
            reinterpret_cast<const void*>(decode_kernel<double, true, true>),
            reinterpret_cast<const void*>(decode_kernel<double, false, true>),
            reinterpret_cast<const void*>(decode_stats_kernel<float, true>),
            reinterpret_cast<const void*>(decode_stats_kernel<float, false>),
            reinterpret_cast<const void*>(decode_stats_kernel<double, true>),
            reinterpret_cast<const void*>(decode_stats_kernel<double, false>),
            reinterpret_cast<const void*>(merge_coop_kernel<1>),
            reinterpret_cast<const void*>(merge_coop_kernel<2>),
            reinterpret_cast<const void*>(merge_coop_kernel<4>),
            reinterpret_cast<const void*>(merge_coop_kernel<8>),
            reinterpret_cast<const void*>(merge_coop_kernel<12>),
            reinterpret_cast<const void*>(merge_coop_kernel<16>),
            reinterpret_cast<const void*>(merge_grid_kernel<1, 1>),
            reinterpret_cast<const void*>(merge_grid_kernel<2, 1>),
            reinterpret_cast<const void*>(merge_grid_kernel<4, 1>),
            reinterpret_cast<const void*>(merge_grid_kernel<8, 1>),
            reinterpret_cast<const void*>(merge_grid_kernel<16, 1>),
            reinterpret_cast<const void*>(merge_grid_kernel<1, 2>),
            reinterpret_cast<const void*>(merge_grid_kernel<2, 2>),
            reinterpret_cast<const void*>(merge_grid_kernel<4, 2>),
            reinterpret_cast<const void*>(merge_grid_kernel<8, 2>),
            reinterpret_cast<const void*>(merge_grid_kernel<1, 1, 256>),
            reinterpret_cast<const void*>(merge_grid_kernel<1, 2, 256>),
            reinterpret_cast<const void*>(merge_grid_kernel<1, 1, 512>),
            reinterpret_cast<const void*>(merge_grid_kernel<1, 2, 512>),
            reinterpret_cast<const void*>(merge_cluster_kernel<1, 1>),
            reinterpret_cast<const void*>(merge_cluster_kernel<2, 1>),
            reinterpret_cast<const void*>(merge_cluster_kernel<4, 1>),
            reinterpret_cast<const void*>(merge_cluster_kernel<8, 1>),
            reinterpret_cast<const void*>(merge_cluster_kernel<16, 1>),
            reinterpret_cast<const void*>(merge_cluster_kernel<1, 2>),
            reinterpret_cast<const void*>(merge_cluster_kernel<2, 2>),
            reinterpret_cast<const void*>(merge_cluster_kernel<4, 2>),
            reinterpret_cast<const void*>(merge_cluster_kernel<8, 2>),
            reinterpret_cast<const void*>(round_cluster_kernel<float, 1, 1>),
            reinterpret_cast<const void*>(round_cluster_kernel<float, 2, 1>),
            reinterpret_cast<const void*>(round_cluster_kernel<float, 4, 1>),
            reinterpret_cast<const void*>(round_cluster_kernel<float, 1, 2>),
            reinterpret_cast<const void*>(round_cluster_kernel<float, 2, 2>),
            reinterpret_cast<const void*>(round_cluster_kernel<float, 4, 2>),
            reinterpret_cast<const void*>(round_cluster_kernel<double, 1, 1>),
            reinterpret_cast<const void*>(round_cluster_kernel<double, 2, 1>),
            reinterpret_cast<const void*>(round_cluster_kernel<double, 4, 1>),
            reinterpret_cast<const void*>(round_cluster_kernel<double, 1, 2>),
            reinterpret_cast<const void*>(round_cluster_kernel<double, 2, 2>),
            reinterpret_cast<const void*>(round_cluster_kernel<double, 4, 2>),
            reinterpret_cast<const void*>(coins_kernel),
            reinterpret_cast<const void*>(export_bits_kernel),
            reinterpret_cast<const void*>(flag_write_kernel),
            reinterpret_cast<const void*>(seg_hash_kernel),
            reinterpret_cast<const void*>(hash_compare_kernel),
            reinterpret_cast<const void*>(dense_leaf_kernel<float>),
            reinterpret_cast<const void*>(dense_leaf_kernel<double>),
            reinterpret_cast<const void*>(dense_reduce_kernel<float>),
            reinterpret_cast<const void*>(dense_reduce_kernel<double>),
            reinterpret_cast<const void*>(dense_chain_kernel<float, 0, false>),
            reinterpret_cast<const void*>(dense_chain_kernel<float, 1, false>),
            reinterpret_cast<const void*>(dense_chain_kernel<float, 2, false>),
            reinterpret_cast<const void*>(dense_chain4_kernel<float, false>),
            reinterpret_cast<const void*>(dense_chain_kernel<double, 0, false>),
            reinterpret_cast<const void*>(dense_chain_kernel<double, 1, false>),
            reinterpret_cast<const void*>(dense_chain_kernel<double, 2, false>),
            reinterpret_cast<const void*>(dense_chain4_kernel<double, false>),
            reinterpret_cast<const void*>(dense_chain_kernel<float, 0, true>),
            reinterpret_cast<const void*>(dense_chain_kernel<float, 1, true>),
            reinterpret_cast<const void*>(dense_chain_kernel<float, 2, true>),
            reinterpret_cast<const void*>(dense_chain4_kernel<float, true>),
            reinterpret_cast<const void*>(dense_chain_kernel<double, 0, true>),
            reinterpret_cast<const void*>(dense_chain_kernel<double, 1, true>),
            reinterpret_cast<const void*>(dense_chain_kernel<double, 2, true>),
            reinterpret_cast<const void*>(dense_chain4_kernel<double, true>),
            reinterpret_cast<const void*>(dense_dag4_kernel<float>),
            reinterpret_cast<const void*>(dense_dag4_kernel<double>),
            reinterpret_cast<const void*>(sub_update_kernel<float>),
            reinterpret_cast<const void*>(sub_update_kernel<double>),
        };
        cudaFuncAttributes a;
        for (const void* f : fns) {
            const cudaError_t e = cudaFuncGetAttributes(&a, f);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }();
    if (result == cudaSuccess) done.push_back(dev);
    return result;
}

#define MARSIT_INSTANTIATE(T)                                                                    \
    template cudaError_t launch_extract<T>(const StreamParams<T>&, bool, int, cudaStream_t);    \
    template cudaError_t launch_decode<T>(const StreamParams<T>&, bool, int, cudaStream_t);     \
    template cudaError_t launch_fill_recipe<T>(int, uint64_t, uint64_t, uint64_t, uint64_t, T*, \
                                               cudaStream_t);                                   \
    template cudaError_t launch_dense_reduce<T>(const DenseParams<T>&, int, cudaStream_t);      \
    template cudaError_t launch_sub_update<T>(T* const*, uint32_t, const T*, uint64_t, int,     \
                                              cudaStream_t);                                    \
    template cudaError_t launch_round_cluster<T>(const ClusterParams&, const FusedParams<T>&, int,  \
                                                 int, uint32_t, size_t, cudaStream_t);          \
    template cudaError_t round_cluster_occupancy<T>(int, int, uint32_t, size_t, int*);          \
    template cudaError_t launch_round_spread<T>(const ClusterParams&, const SpreadParams<T>&, int, \
                                                int, uint32_t, size_t, bool, cudaStream_t);      \
    template cudaError_t round_spread_occupancy<T>(int, int, uint32_t, size_t, int*);           \
    template cudaError_t launch_dense_leaf<T>(const T* const*, const T* const*, uint32_t,       \
                                              uint64_t, uint64_t, uint32_t, uint32_t, T*, int*,  \
                                              int, cudaStream_t, T* const*);
MARSIT_INSTANTIATE(float)
MARSIT_INSTANTIATE(double)

}  // namespace marsit_b200

// Test hook (not part of the public header): coin words [0, n_words) of the
// stream (key, th) through the production coin-word routine, 64 words per warp.
namespace marsit_b200 {
namespace {
__global__ void debug_coin_words_kernel(uint64_t key, uint64_t th, uint32_t n_chunks, uint32_t* out) {
    const uint32_t c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (c < n_chunks) coin_words<64>(key, th, out, uint64_t(c) * 64, threadIdx.x & 31);
}
}  // namespace
}  // namespace marsit_b200
extern "C" int marsit_debug_coin_words(uint64_t key, uint64_t th, uint32_t n_chunks, uint32_t* d_out) {
    marsit_b200::debug_coin_words_kernel<<<(n_chunks + 7) / 8, 256>>>(key, th, n_chunks, d_out);
    return int(cudaDeviceSynchronize());
}

#if defined(MARSIT_COOP_PROF) || defined(MARSIT_FUSED_PROF)
extern "C" void marsit_debug_coop_prof(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, marsit_b200::g_coop_prof, sizeof(marsit_b200::g_coop_prof));
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(marsit_b200::g_coop_prof, z, sizeof(z));
    }
}
#endif
