// Microbenchmark of the tcgen05 round trips the NRC kernels are built from
// (diagnostic, not part of libnrc).  One CTA of 128 threads, clock64 timing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2106_12372_b200/csrc ubench_tcgen05.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "nrc_device.cuh"

using namespace nrc;

__global__ void __launch_bounds__(128, 1) ubench(int mode, int iters, long long* out) {
    long long issue_sum = 0;
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
        if (mode == 16 || mode == 17) {  // warp-converged issue with elect.sync inside the asm
            if (warp == 0) {
                const uint32_t d_u = __shfl_sync(0xffffffffu, tb, 0);
                const uint32_t a_u = __shfl_sync(0xffffffffu, tb + 64, 0);
                const uint64_t b0 = desc_kmajor(b, 0);
                const uint32_t blo = __shfl_sync(0xffffffffu, uint32_t(b0), 0);
                const uint32_t bhi = __shfl_sync(0xffffffffu, uint32_t(b0 >> 32), 0);
                const uint64_t bd = (uint64_t(bhi) << 32) | blo;
                const uint32_t bar_u = __shfl_sync(0xffffffffu, smem_u32(&bar), 0);
                tc_fence_after();
                const long long a0 = clock64();
                if (mode == 16) {
                    asm volatile(
                        "{\n\t.reg .pred e, f, t;\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t"
                        "elect.sync _|e, 0xffffffff;\n\t"
                        "setp.ne.b32 f, 0, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
                        "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
                        "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t"
                        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, f;\n\t"
                        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, t;\n\t"
                        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, t;\n\t"
                        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, t;\n\t"
                        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n}" ::"r"(d_u),
                        "r"(a_u), "l"(bd), "r"(idesc), "r"(bar_u)
                        : "memory");
                } else {
                    if (elect_one()) umma_chain4_ta_commit(d_u, a_u, bd, idesc, &bar);
                }
                __syncwarp();
                if (tid == 0) issue_sum += clock64() - a0;
            }
            mbar_wait(&bar, phase);
            phase ^= 1;
            continue;
        }
        if (mode >= 10) {  // issue cost: clock around the issue of n MMAs + commit only
            if (tid == 0) {
                tc_fence_after();
                const long long a0 = clock64();
                const int nm = mode == 10 ? 4 : mode == 11 ? 1 : mode == 13 ? 2 : mode == 14 ? 16 : mode == 15 ? 64 : 4;
                for (int k = 0; k < nm; ++k) {
                    if (mode == 12)
                        umma_f16_ta(tb, tb + 64 + 8 * (k & 3), desc_kmajor(b, k & 3), idesc, k > 0);
                    else
                        umma_f16(tb, desc_kmajor(a, k & 3), desc_kmajor(b, k & 3), idesc, k > 0);
                }
                umma_commit(&bar);
                issue_sum += clock64() - a0;
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
    if (tid == 0 && mode >= 10) out[0] = issue_sum / iters;
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
                           "dgrad M128N64K64 (B MN-major)", "wgrad M64N64K128 (A,B MN-major)", "dgrad + wgrad",
                           "ISSUE ONLY: 4 SS mma + commit", "ISSUE ONLY: 1 SS mma + commit",
                           "ISSUE ONLY: 4 TS mma + commit", "ISSUE ONLY: 2 SS mma + commit",
                           "ISSUE ONLY: 16 SS mma + commit", "ISSUE ONLY: 64 SS mma + commit",
                           "ISSUE: warp elect.sync asm chain4 TS", "ISSUE: elect_one() + chain4 TS"};
    for (int mode = 0; mode < 18; ++mode) {
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
