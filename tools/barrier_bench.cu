// Grid-barrier cost on B200: the cooperative merge pays one grid-wide
// barrier (plus a tile-count publish and a prefix read) per merge step.
// Compares cooperative_groups grid.sync with hand-rolled barriers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_bench barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>

namespace cg = cooperative_groups;

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// per-step work stand-in: publish a tile count, read the earlier tiles' counts
__device__ __forceinline__ uint64_t prefix_read(const uint64_t* flags, uint32_t lt) {
    uint64_t acc = 0;
    for (uint32_t i = threadIdx.x; i < lt; i += blockDim.x) acc += __ldcg(flags + i);
    return acc;
}

__global__ void k_cg(int iters, uint64_t* flags, unsigned long long* sink) {
    cg::grid_group g = cg::this_grid();
    uint64_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint64_t* f = flags + (it & 7) * gridDim.x;
        if (threadIdx.x == 0) __stcg(f + blockIdx.x, (uint64_t)it + blockIdx.x);
        g.sync();
        acc += prefix_read(f, blockIdx.x);
        __syncthreads();
    }
    if (acc == 42) *sink = acc;
}

// counter never reset within a launch: target = (it+1) * T
__global__ void k_custom(int iters, uint64_t* flags, unsigned* ctr, unsigned long long* sink) {
    uint64_t acc = 0;
    const unsigned T = gridDim.x;
    for (int it = 0; it < iters; ++it) {
        uint64_t* f = flags + (it & 7) * gridDim.x;
        __syncthreads();
        if (threadIdx.x == 0) {
            __stcg(f + blockIdx.x, (uint64_t)it + blockIdx.x);
            red_release_add(ctr, 1u);
            const unsigned target = (it + 1) * T;
            while (ld_acquire(ctr) < target) {
            }
        }
        __syncthreads();
        acc += prefix_read(f, blockIdx.x);
    }
    if (acc == 42) *sink = acc;
}

// same, but spin relaxed, one acquire fence after
__global__ void k_custom2(int iters, uint64_t* flags, unsigned* ctr, unsigned long long* sink) {
    uint64_t acc = 0;
    const unsigned T = gridDim.x;
    for (int it = 0; it < iters; ++it) {
        uint64_t* f = flags + (it & 7) * gridDim.x;
        __syncthreads();
        if (threadIdx.x == 0) {
            __stcg(f + blockIdx.x, (uint64_t)it + blockIdx.x);
            red_release_add(ctr, 1u);
            const unsigned target = (it + 1) * T;
            while (ld_relaxed(ctr) < target) {
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
        acc += prefix_read(f, blockIdx.x);
    }
    if (acc == 42) *sink = acc;
}

// cluster-hierarchical: barrier.cluster, one global arrival per cluster,
// leader spins, barrier.cluster
__global__ void k_cluster(int iters, uint64_t* flags, unsigned* ctr, unsigned long long* sink) {
    cg::cluster_group cl = cg::this_cluster();
    uint64_t acc = 0;
    const unsigned nclu = gridDim.x / cl.num_blocks();
    for (int it = 0; it < iters; ++it) {
        uint64_t* f = flags + (it & 7) * gridDim.x;
        if (threadIdx.x == 0) __stcg(f + blockIdx.x, (uint64_t)it + blockIdx.x);
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (cl.block_rank() == 0 && threadIdx.x == 0) {
            red_release_add(ctr, 1u);
            const unsigned target = (it + 1) * nclu;
            while (ld_acquire(ctr) < target) {
            }
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        acc += prefix_read(f, blockIdx.x);
        __syncthreads();
    }
    if (acc == 42) *sink = acc;
}

// no barrier: every tile waits only for the step-tagged counts of the tiles
// before it (flag = step << 32 | count)
__global__ void k_flags(int iters, uint64_t* flags, unsigned long long* sink) {
    __shared__ uint64_t s[8];
    uint64_t tot = 0;
    for (int it = 0; it < iters; ++it) {
        uint64_t* f = flags;  // [T] tagged words, reused every step
        if (threadIdx.x == 0) {
            const uint64_t v = (uint64_t(it + 1) << 32) | (blockIdx.x & 1023);
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(f + blockIdx.x), "l"(v) : "memory");
        }
        uint64_t acc = 0;
        for (uint32_t i = threadIdx.x; i < blockIdx.x; i += blockDim.x) {
            uint64_t v;
            do {
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(f + i) : "memory");
            } while ((v >> 32) < uint64_t(it + 1));
            acc += v & 0xffffffffu;
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
        if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0)
            for (int w = 0; w < 8; ++w) tot += s[w];
        __syncthreads();
    }
    if (tot == 42) *sink = tot;
}

int main() {
    uint64_t* flags;
    unsigned* ctr;
    unsigned long long* sink;
    cudaMalloc(&flags, 8 * 4096 * 8);
    cudaMalloc(&ctr, 4);
    cudaMalloc(&sink, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 2000;
    for (int T : {148, 196, 264, 296}) {
        auto time_it = [&](const char* name, auto launch) {
            cudaMemset(flags, 0, 8 * 4096 * 8);
            cudaMemset(ctr, 0, 4);
            launch();  // warm
            cudaMemset(flags, 0, 8 * 4096 * 8);
            cudaMemset(ctr, 0, 4);
            cudaDeviceSynchronize();
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaError_t e = cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("T=%d %-10s %7.3f us/step  %s\n", T, name, ms * 1e3 / iters,
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
        };
        time_it("cg", [&] {
            int it = iters;
            void* args[] = {&it, &flags, &sink};
            cudaLaunchCooperativeKernel((void*)k_cg, T, 256, args, 0, 0);
        });
        time_it("custom", [&] {
            cudaMemset(ctr, 0, 4);
            k_custom<<<T, 256>>>(iters, flags, ctr, sink);
        });
        time_it("custom2", [&] {
            cudaMemset(ctr, 0, 4);
            k_custom2<<<T, 256>>>(iters, flags, ctr, sink);
        });
        for (int cs : {2, 4, 8}) {
            if (T % cs) continue;
            char nm[32];
            snprintf(nm, sizeof nm, "cluster%d", cs);
            time_it(nm, [&] {
                cudaMemset(ctr, 0, 4);
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(T);
                cfg.blockDim = dim3(256);
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cs;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaError_t e = cudaLaunchKernelEx(&cfg, k_cluster, iters, flags, ctr, sink);
                if (e != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(e));
            });
        }
        time_it("flags", [&] {
            cudaMemset(flags, 0, 8 * 4096 * 8);
            k_flags<<<T, 256>>>(iters, flags, sink);
        });
    }
    return 0;
}
