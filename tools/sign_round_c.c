/*
 * sign_round_c.c — the C-ABI from plain C (no C++, no torch): the device-side
 * counterpart of the reference's samples/sign_sync_round.cpp tour.  Four
 * workers with different gradients, dense every 4th round, the compensation
 * carried in place on the device; after every sign round the defining
 * identity c' = (g + c) - g_t is checked bit for bit on the host, as the
 * reference sample does.
 *
 *   make -C tools sign_round_c && build/sign_round_c
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "marsit_b200.h"

#define CHECK(x)                                                                     \
    do {                                                                             \
        marsit_status s_ = (x);                                                      \
        if (s_ != MARSIT_OK) {                                                       \
            fprintf(stderr, "%s failed: %d %s\n", #x, (int)s_, marsit_last_error()); \
            return EXIT_FAILURE;                                                     \
        }                                                                            \
    } while (0)
#define CUDA(x)                                                                       \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));           \
            return EXIT_FAILURE;                                                      \
        }                                                                             \
    } while (0)

enum { kWorkers = 4, kDim = 1000 };

int main(void) {
    marsit_schedule* sched = NULL;
    CHECK(marsit_schedule_ring(kWorkers, &sched));
    marsit_ctx_desc desc;
    memset(&desc, 0, sizeof desc);
    desc.dim = kDim;
    desc.schedule = sched;
    desc.dtype = MARSIT_F64;
    desc.device = 0;
    desc.nranks = 1;
    desc.transport = MARSIT_TRANSPORT_P2P; /* the default; unused with one rank */
    marsit_ctx* ctx = NULL;
    CHECK(marsit_ctx_create(&desc, &ctx));

    static double g[kWorkers][kDim], c_prev[kWorkers][kDim], c_now[kWorkers][kDim];
    static double upd[kDim];
    void* d_g[kWorkers];
    void* d_c[kWorkers];
    for (int w = 0; w < kWorkers; ++w) {
        for (int j = 0; j < kDim; ++j)  /* locally scaled gradients, as in the sample */
            g[w][j] = (j % 2 == 0 ? 0.04 : -0.03) + 0.01 * w + 1e-5 * ((j * 7 + w) % 13);
        CUDA(cudaMalloc(&d_g[w], sizeof g[w]));
        CUDA(cudaMalloc(&d_c[w], sizeof g[w]));
        CUDA(cudaMemcpy(d_g[w], g[w], sizeof g[w], cudaMemcpyHostToDevice));
        CUDA(cudaMemset(d_c[w], 0, sizeof g[w]));
    }
    void* d_upd = NULL;
    uint64_t* d_bits = NULL;
    CUDA(cudaMalloc(&d_upd, sizeof upd));
    CUDA(cudaMalloc((void**)&d_bits, ((kDim + 63) / 64) * sizeof(uint64_t)));

    const uint64_t period = 4; /* dense every 4th round */
    const double eta_s = 0.05;
    for (uint64_t t = 0; t < 6; ++t) {
        for (int w = 0; w < kWorkers; ++w)
            CUDA(cudaMemcpy(c_prev[w], d_c[w], sizeof c_prev[w], cudaMemcpyDeviceToHost));
        int full = 0;
        CHECK(marsit_round(ctx, t, period, eta_s, /*seed*/ 1, (const void* const*)d_g,
                           (const void* const*)d_c, d_c /* in place */, d_bits, d_upd, &full,
                           NULL));
        CHECK(marsit_ctx_check(ctx, NULL));
        uint64_t per_worker[kWorkers], reduce_bits = 0, gather_bits = 0, total = 0;
        CHECK(marsit_bits_account(ctx, full, per_worker, &reduce_bits, &gather_bits, &total));
        CUDA(cudaMemcpy(upd, d_upd, sizeof upd, cudaMemcpyDeviceToHost));
        for (int w = 0; w < kWorkers; ++w)
            CUDA(cudaMemcpy(c_now[w], d_c[w], sizeof c_now[w], cudaMemcpyDeviceToHost));
        printf("round %llu  %-5s  bits %7llu  update[0] % .4f  comp[0][0] % .4f\n",
               (unsigned long long)t, full ? "dense" : "sign", (unsigned long long)total, upd[0],
               c_now[0][0]);
        if (!full)
            for (int w = 0; w < kWorkers; ++w)
                for (int j = 0; j < kDim; ++j) {
                    const double held = g[w][j] + c_prev[w][j];
                    if (c_now[w][j] != held - upd[j]) {
                        fprintf(stderr, "compensation identity broken at w=%d j=%d\n", w, j);
                        return EXIT_FAILURE;
                    }
                }
    }
    puts("sign rounds moved one bit per coordinate; the identity held exactly");
    for (int w = 0; w < kWorkers; ++w) {
        cudaFree(d_g[w]);
        cudaFree(d_c[w]);
    }
    cudaFree(d_upd);
    cudaFree(d_bits);
    marsit_ctx_destroy(ctx);
    marsit_schedule_destroy(sched);
    return EXIT_SUCCESS;
}
