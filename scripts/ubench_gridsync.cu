// Microbenchmark of the fused train kernel's inter-CTA phases (diagnostic,
// not part of libnrc): grid-barrier latency variants and the cross-CTA
// partial reduction (128 partials x 21,504 fp32) at several thread counts.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ubench_gridsync.cu -o ubench_gridsync
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kParam = 21504, kChunks = kParam / 4;

__device__ __forceinline__ long long gns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int MODE>
__device__ __forceinline__ void gsync(unsigned long long* ctr, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        if (MODE == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
        if (MODE == 2) __threadfence();
        if (MODE == 3) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        } else {
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        }
        unsigned long long v = 0;
        do {
            if (MODE == 3)
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
            else
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
            if (MODE == 2 && v < target) __nanosleep(32);
        } while (v < target);
        if (MODE == 3) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

// flag barrier: CTA b publishes epoch in its own 8-byte slot; warp 0 polls all slots
__device__ __forceinline__ void fsync(unsigned long long* flags, unsigned long long epoch) {
    __syncthreads();
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0)
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flags + blockIdx.x), "l"(epoch) : "memory");
        for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) {
            unsigned long long v;
            do {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + b) : "memory");
            } while (v < epoch);
        }
        __syncwarp();
    }
    __syncthreads();
}
__global__ void flag_bench(unsigned long long* flags, int iters, long long* out) {
    fsync(flags, 1);
    const long long t0 = gns();
    for (int i = 0; i < iters; ++i) fsync(flags, i + 2);
    const long long t1 = gns();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

template <int MODE>
__global__ void barrier_bench(unsigned long long* ctr, int iters, long long* out) {
    const unsigned long long G = gridDim.x;
    gsync<MODE>(ctr, G);
    const long long t0 = gns();
    for (int i = 0; i < iters; ++i) gsync<MODE>(ctr, G * (i + 2));
    const long long t1 = gns();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

// Each CTA reduces its balanced chunk slice over all G partials; BATCH loads
// in flight per thread (predicated tail), then a fixed-order group combine.
template <int BATCH>
__global__ void reduce_bench(const float4* __restrict__ P, float* __restrict__ outp, unsigned long long* ctr,
                             int iters, long long* out) {
    __shared__ float4 sred[1024];
    const int G = gridDim.x, T = blockDim.x, tid = threadIdx.x;
    const int c0 = blockIdx.x * kChunks / G, c1 = (blockIdx.x + 1) * kChunks / G, nch = c1 - c0;
    const int ng = nch >= T ? 1 : T / nch;
    gsync<0>(ctr, G);
    const long long t0 = gns();
    for (int it = 0; it < iters; ++it) {
        for (int t = tid; t < ng * nch; t += T) {
            const int c = t % nch, z = t / nch;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int p = z; p < G; p += BATCH * ng) {
                float4 x[BATCH];
#pragma unroll
                for (int u = 0; u < BATCH; ++u)
                    x[u] = (p + u * ng < G) ? __ldcg(P + size_t(p + u * ng) * kChunks + c0 + c)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int u = 0; u < BATCH; ++u) {
                    acc.x += x[u].x;
                    acc.y += x[u].y;
                    acc.z += x[u].z;
                    acc.w += x[u].w;
                }
            }
            sred[z * nch + c] = acc;
        }
        __syncthreads();
        for (int q = tid; q < nch; q += T) {
            float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int z = 0; z < ng; ++z) {
                g.x += sred[z * nch + q].x;
                g.y += sred[z * nch + q].y;
                g.z += sred[z * nch + q].z;
                g.w += sred[z * nch + q].w;
            }
            reinterpret_cast<float4*>(outp)[c0 + q] = g;
        }
        gsync<0>(ctr, G * (it + 2));
    }
    const long long t1 = gns();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

int main() {
    unsigned long long* ctr;
    long long* d;
    float4* P;
    float* o;
    cudaMalloc(&ctr, 8);
    cudaMalloc(&d, 8);
    cudaMalloc(&P, sizeof(float) * kParam * 148);
    cudaMalloc(&o, sizeof(float) * kParam);
    cudaMemset(P, 0, sizeof(float) * kParam * 148);
    long long ns = 0;
    for (int grid : {128, 148}) {
        cudaMemset(ctr, 0, 8);
        barrier_bench<0><<<grid, 160>>>(ctr, 1000, d);
        cudaDeviceSynchronize();
        cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        printf("barrier mode 0 (proxy fence + release/acquire) grid %d: %lld ns\n", grid, ns);
        cudaMemset(ctr, 0, 8);
        barrier_bench<1><<<grid, 160>>>(ctr, 1000, d);
        cudaDeviceSynchronize();
        cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        printf("barrier mode 1 (release/acquire)               grid %d: %lld ns\n", grid, ns);
        cudaMemset(ctr, 0, 8);
        barrier_bench<2><<<grid, 160>>>(ctr, 1000, d);
        cudaDeviceSynchronize();
        cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        printf("barrier mode 2 (threadfence + nanosleep)       grid %d: %lld ns\n", grid, ns);
        cudaMemset(ctr, 0, 8);
        barrier_bench<3><<<grid, 160>>>(ctr, 1000, d);
        cudaDeviceSynchronize();
        cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        printf("barrier mode 3 (fence.acq_rel + relaxed)       grid %d: %lld ns\n", grid, ns);
    }
    unsigned long long* flags;
    cudaMalloc(&flags, 8 * 256);
    for (int grid : {128, 148}) {
        cudaMemset(flags, 0, 8 * 256);
        flag_bench<<<grid, 160>>>(flags, 1000, d);
        cudaDeviceSynchronize();
        cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        printf("flag barrier (st.release / ld.acquire per CTA slot) grid %d: %lld ns\n", grid, ns);
    }
    for (int block : {160, 256, 512}) {
        cudaMemset(ctr, 0, 8);
        reduce_bench<8><<<128, block>>>(P, o, ctr, 200, d);
        cudaDeviceSynchronize();
        cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        printf("reduce+barrier BATCH 8  block %3d: %lld ns\n", block, ns);
        cudaMemset(ctr, 0, 8);
        reduce_bench<16><<<128, block>>>(P, o, ctr, 200, d);
        cudaDeviceSynchronize();
        cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        printf("reduce+barrier BATCH 16 block %3d: %lld ns\n", block, ns);
        cudaMemset(ctr, 0, 8);
        reduce_bench<32><<<128, block>>>(P, o, ctr, 200, d);
        cudaDeviceSynchronize();
        cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        printf("reduce+barrier BATCH 32 block %3d: %lld ns\n", block, ns);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
