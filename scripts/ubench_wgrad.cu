// Microbenchmark (diagnostic, not part of libnrc): tensor-pipe time of the
// MMA shapes of the training step, issued by an elected lane of a converged
// warp, one commit, clock64 from issue to the commit's mbarrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2106_12372_b200/csrc ubench_wgrad.cu
// Modes (per iteration):
//   0: wgrad  M64  N64 K128 (8 x K16, MN-major A and B)          one chain
//   1: wgrad  as 0 split into two K64 chains on two accumulators
//   2: six wgrad chains back to back (the step's six layers)
//   3: dgrad  M128 N64 K64  (4 x K16, A K-major, B MN-major)     one chain
//   4: fwd    M128 N64 K64  (4 x K16, K-major)                   one chain
//   5: wgrad  M128 N64 K128 (8 x K16, MN-major)  (twice the rows of 0)
//   6: wgrad  M64  N128 K128 (8 x K16, MN-major)
//   7: dgrad + wgrad (one round of the backward), one commit
#include <cstdio>
#include <cuda_runtime.h>

#include "nrc_device.cuh"

using namespace nrc;

__global__ void __launch_bounds__(128, 1) ubench(int mode, int iters, long long* out) {
    __shared__ __align__(1024) uint8_t sA[kTileBytes];
    __shared__ __align__(1024) uint8_t sB[kTileBytes];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    for (uint32_t o = tid * 16; o < kTileBytes; o += 128 * 16) {
        st_shared_v4(smem_u32(sA) + o, 0x3c003c00u, 0, 0, 0);
        st_shared_v4(smem_u32(sB) + o, 0x3c003c00u, 0, 0, 0);
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(&tslot, 512);
        tmem_relinquish();
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tslot;
    const uint32_t a = smem_u32(sA), b = smem_u32(sB);
    uint32_t phase = 0;
    long long total = 0;
    for (int it = 0; it < iters; ++it) {
        __syncthreads();
        long long t0 = clock64();
        if (warp == 0) {
            const uint32_t d = warp_uniform(tb);
            const uint64_t amn = warp_uniform(make_sdesc(a, kTileBytes, 1024u));
            const uint64_t bmn = warp_uniform(make_sdesc(b, kTileBytes, 1024u));
            const uint64_t ak = warp_uniform(desc_kmajor(a, 0));
            const uint64_t bk = warp_uniform(desc_kmajor(b, 0));
            const uint64_t bmn_w = warp_uniform(make_sdesc(b, 64u * 128u, 1024u));
            const uint32_t id_w = make_idesc(64, 64, 1, 1), id_w128 = make_idesc(128, 64, 1, 1),
                           id_wn = make_idesc(64, 128, 1, 1), id_d = make_idesc(128, 64, 0, 1),
                           id_f = make_idesc(128, 64, 0, 0);
            tc_fence_after();
            if (elect_one()) {
                if (mode == 0) {
                    umma_ss8<kMNmajStep, kMNmajStep>(d, amn, bmn, id_w, 0u);
                } else if (mode == 1) {
                    umma_ss4<kMNmajStep, kMNmajStep>(d, amn, bmn, id_w, 0u);
                    umma_ss4<kMNmajStep, kMNmajStep>(d + 64, amn + 4 * kMNmajStep, bmn + 4 * kMNmajStep, id_w, 0u);
                } else if (mode == 2) {
                    for (int l = 0; l < 6; ++l) umma_ss8<kMNmajStep, kMNmajStep>(d + 64 * l, amn, bmn, id_w, 0u);
                } else if (mode == 3) {
                    umma_ss4<kKmajStep, kMNmajStep>(d, ak, bmn_w, id_d, 0u);
                } else if (mode == 4) {
                    umma_ss4<kKmajStep, kKmajStep>(d, ak, bk, id_f, 0u);
                } else if (mode == 5) {
                    umma_ss8<kMNmajStep, kMNmajStep>(d, amn, bmn, id_w128, 0u);
                } else if (mode == 6) {
                    umma_ss8<kMNmajStep, kMNmajStep>(d, amn, bmn, id_wn, 0u);
                } else if (mode == 7) {
                    umma_ss4<kKmajStep, kMNmajStep>(d, ak, bmn_w, id_d, 0u);
                    umma_ss8<kMNmajStep, kMNmajStep>(d + 64, amn, bmn, id_w, 0u);
                }
                umma_commit(&bar);
            }
            __syncwarp();
        }
        mbar_wait(&bar, phase);
        phase ^= 1;
        tc_fence_after();
        total += clock64() - t0;
    }
    if (tid == 0) out[0] = total / iters;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    const char* names[] = {"wgrad M64 N64 K128 (8 MMA)", "wgrad split 2 x K64 chains", "6 wgrad chains",
                           "dgrad M128 N64 K64 (4 MMA)", "fwd M128 N64 K64 (4 MMA)", "wgrad M128 N64 K128",
                           "wgrad M64 N128 K128", "dgrad + wgrad (one round)"};
    for (int mode = 0; mode < 8; ++mode) {
        ubench<<<1, 128>>>(mode, 3, d);  // warm-up
        ubench<<<1, 128>>>(mode, 200, d);
        long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("mode %d %-32s %6lld cycles (issue -> commit arrival, mean)\n", mode, names[mode], c);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
