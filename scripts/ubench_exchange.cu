// Microbenchmark (diagnostic, not part of libnrc): the per-step gradient
// exchange of a persistent training kernel -- every CTA writes an 86 KB fp32
// partial, a grid barrier, each CTA reduces its 1/G slice of the parameters
// over all G partials (8 fixed-order partial groups, every load in flight),
// a second grid barrier.  One CTA per SM (dynamic SMEM sized like the
// training kernel).  Prints ns per iteration for each mode.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ubench_exchange.cu -o /tmp/ubx && /tmp/ubx
// Modes: 0 two grid barriers; 1 barrier + slice reduction + barrier;
//        2 partial write + barrier + slice reduction + barrier
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kF4 = 5376;  // float4 per partial (21,504 floats)

__device__ __forceinline__ void grid_bar(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(384, 1) ubx(int mode, int iters, float4* parts, float4* outv, unsigned* ctr, long long* t_out) {
    extern __shared__ float4 sm[];
    const int G = gridDim.x, c = blockIdx.x, nt = blockDim.x;
    const int per = (kF4 + G - 1) / G;  // float4 of this CTA's slice
    const int f0 = c * per, f1 = min(kF4, f0 + per);
    const int items = 8 * (f1 - f0);
    unsigned gen = 0;
    long long t0 = 0;
    for (int it = 0; it < iters; ++it) {
        if (it == 1 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        if (mode == 2) {
            float4* my = parts + size_t(c) * kF4;
            for (int i = threadIdx.x; i < kF4; i += nt) my[i] = make_float4(it, c, i, 1.f);
        }
        grid_bar(ctr, (++gen) * G);
        if (mode >= 1) {
            for (int w = threadIdx.x; w < items; w += nt) {
                const int g = w / (f1 - f0), f = f0 + w % (f1 - f0);
                float4 v[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int p = g + 8 * k;
                    asm volatile("ld.global.relaxed.gpu.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v[k].x), "=f"(v[k].y), "=f"(v[k].z), "=f"(v[k].w) : "l"(parts + size_t(p) * kF4 + f));  // G = 128: 16 partials per group
                }
                float4 s = v[0];
#pragma unroll
                for (int k = 1; k < 16; ++k) s.x += v[k].x, s.y += v[k].y, s.z += v[k].z, s.w += v[k].w;
                sm[w] = s;
            }
            __syncthreads();
            for (int f = f0 + threadIdx.x; f < f1; f += nt) {
                float4 s = sm[f - f0];
                for (int g = 1; g < 8; ++g) {
                    const float4 u = sm[g * (f1 - f0) + f - f0];
                    s.x += u.x, s.y += u.y, s.z += u.z, s.w += u.w;
                }
                outv[f] = s;
            }
        }
        grid_bar(ctr, (++gen) * G);
    }
    if (threadIdx.x == 0 && c == 0) {
        long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        *t_out = t1 - t0;
    }
}

int main() {
    float4 *parts, *outv;
    unsigned* ctr;
    long long* t;
    cudaMalloc(&parts, size_t(148) * kF4 * 16);
    cudaMalloc(&outv, kF4 * 16);
    cudaMalloc(&ctr, 4);
    cudaMalloc(&t, 8);
    cudaMemset(parts, 0, size_t(148) * kF4 * 16);
    const int smem = 187 * 1024;
    cudaFuncSetAttribute(ubx, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 200;
    for (int grid : {128})
        for (int threads : {288, 384})
            for (int mode = 0; mode < 3; ++mode) {
                cudaMemset(ctr, 0, 4);
                ubx<<<grid, threads, smem>>>(mode, iters, parts, outv, ctr, t);
                cudaError_t e = cudaDeviceSynchronize();
                long long ns = 0;
                cudaMemcpy(&ns, t, 8, cudaMemcpyDeviceToHost);
                printf("grid %d threads %d mode %d: %.1f ns per iteration (%s)\n", grid, threads, mode,
                       double(ns) / (iters - 1), cudaGetErrorString(e));
            }
    return 0;
}
