// Microbenchmark of the tcgen05 round trips the NRC kernels are built from
// (diagnostic, not part of libnrc).  One CTA of 128 threads, clock64 timing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2106_12372_b200/csrc ubench_tcgen05.cu
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
        tmem_alloc(&tslot, 128);
        tmem_relinquish();
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tslot;
    const uint32_t a = smem_u32(sA), b = smem_u32(sB);
    const uint32_t lane_off = (warp * 32u) << 16;
    const uint32_t idesc = make_idesc(128, 64, 0, 0);
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode == 5) {  // throughput: 16 layers back to back, one commit
            if (tid == 0) {
                tc_fence_after();
                for (int l = 0; l < 16; ++l)
                    for (int k = 0; k < 4; ++k) umma_f16(tb, desc_kmajor(a, k), desc_kmajor(b, k), idesc, k > 0);
                umma_commit(&bar);
            }
            mbar_wait(&bar, phase);
            phase ^= 1;
            continue;
        }
        if (mode == 7 || mode == 8 || mode == 9) {  // backward shapes
            if (tid == 0) {
                tc_fence_after();
                if (mode != 8)  // dgrad: M128 N64 K64, A K-major, B MN-major
                    for (int k = 0; k < 4; ++k)
                        umma_f16(tb, desc_kmajor(a, k), desc_mnmajor(b, k), make_idesc(128, 64, 0, 1), k > 0);
                if (mode != 7)  // wgrad: M64 N64 K128, A and B MN-major
                    for (int k = 0; k < 8; ++k)
                        umma_f16(tb + 64, desc_mnmajor(a, k), desc_mnmajor(b, k), make_idesc(64, 64, 1, 1), k > 0);
                umma_commit(&bar);
            }
            mbar_wait(&bar, phase);
            phase ^= 1;
            continue;
        }
        if (tid == 0) {
            tc_fence_after();
            if (mode == 1 || mode == 4) {
                for (int k = 0; k < 4; ++k) umma_f16_ta(tb, tb + 64 + 8 * k, desc_kmajor(b, k), idesc, k > 0);
            } else {
                for (int k = 0; k < 4; ++k) umma_f16(tb, desc_kmajor(a, k), desc_kmajor(b, k), idesc, k > 0);
            }
            umma_commit(&bar);
        }
        mbar_wait(&bar, phase);
        phase ^= 1;
        tc_fence_after();
        if (mode >= 2) {  // epilogue: drain, relu+cvt, write A back
            uint32_t hp[32];
            for (int half = 0; half < 2; ++half) {
                uint32_t v[32];
                tmem_ld32(tb + lane_off + 32 * half, v);
                for (int q = 0; q < 16; ++q)
                    hp[16 * half + q] = pack_h2_relu(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1]));
            }
            if (mode == 4) {
                tmem_st32(tb + lane_off + 64, hp);
            } else {
                for (int c = 0; c < 4; ++c)
                    st_shared_v4(a + swz(tid, c), hp[4 * c], hp[4 * c + 1], hp[4 * c + 2], hp[4 * c + 3]);
                fence_async_smem();
            }
            tc_fence_before();
            __syncthreads();
        } else if (mode == 6) {
            __syncthreads();
        }
    }
    long long t1 = clock64();
    if (tid == 0) out[0] = (t1 - t0) / iters;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 128);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    const char* names[] = {"mma SS + commit + wait", "mma TS + commit + wait", "round: SS mma + epi(smem)",
                           "round: SS mma + epi(smem) [same]", "round: TS mma + epi(tmem st)",
                           "16 layers back-to-back (per 16)", "SS mma + wait + syncthreads",
                           "dgrad M128N64K64 (B MN-major)", "wgrad M64N64K128 (A,B MN-major)", "dgrad + wgrad"};
    for (int mode = 0; mode < 10; ++mode) {
        ubench<<<1, 128>>>(mode, 2000, d);
        long long c = 0;
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("mode %d %-36s %lld cycles/iter  (%s)\n", mode, names[mode], c, cudaGetErrorString(e));
    }
    // all SMs at once (contention on nothing shared but L2/clock)
    ubench<<<148, 128>>>(0, 2000, d);
    cudaDeviceSynchronize();
    return 0;
}
