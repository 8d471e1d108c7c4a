// nrc_kernels.cuh -- the sm_100a kernels of libnrc.
//
//   nrc_query_ts_kernel  fused encode -> tcgen05 layers (activations in TMEM)
//                        -> factorised output (P:L602-628 fully fused MLP;
//                        P:L874-878; Table 1)             nrc_query_ts.cuh
//   nrc_train_w_kernel   LCG gather -> encode -> forward (stash in SMEM) ->
//                        relative L2 loss gradient (Eq. 5) -> dgrad + wgrad on
//                        tcgen05 -> per-CTA fp32 partials (where
//                        the paper used CUTLASS split-k)   nrc_train_w.cuh
//   nrc_adam_w_kernel    deterministic partial reduction + Adam + EMA (Eq. 2)
//                        + fp16 operand images nrc_train_w.cuh
//   helpers (here)       image refresh, self-training targets, encode-only,
//                        tcgen05 layout selftest
#pragma once
#include "nrc_device.cuh"
#include "nrc_common.cuh"
#include "nrc_query_ts.cuh"
#include "nrc_train_w.cuh"
#include "nrc_train_ws.cuh"

namespace nrc {

// fp32 padded array -> fp16 operand image at hidden width W and depth nh.
template <int W>
__global__ void nrc_image_w_kernel(const float* __restrict__ w, uint8_t* __restrict__ img, int nh) {
    const NetRt<W> D(nh);
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= D.padded()) return;
    const int i = D.layer_of(j);
    const int rel = j - D.pad_off(i), r = rel / D.cols(i), c = rel % D.cols(i);
    *reinterpret_cast<__half*>(img + D.img_byte(i, r, c)) = __float2half_rn(w[j]);
}

// Self-training targets (nrc_assemble_targets): one thread per training path,
// back to front: acc = E + N + T * acc.
__global__ void nrc_targets_kernel(const uint32_t* __restrict__ first, const uint32_t* __restrict__ len,
                                   const uint32_t* __restrict__ flags, uint32_t n_paths,
                                   const float* __restrict__ vert, const float* __restrict__ tail,
                                   float* __restrict__ targets) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n_paths) return;
    const bool unbiased = (__ldg(flags + p) & 1u) != 0;
    float acc[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] = unbiased ? 0.0f : __ldg(tail + 3 * size_t(p) + c);
    const uint32_t f = __ldg(first + p), m = __ldg(len + p);
    for (uint32_t k = m; k-- > 0;) {
        const float* x = vert + 9 * size_t(f + k);
        float* t = targets + 3 * size_t(f + k);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            acc[c] = fmaf(__ldg(x + 6 + c), acc[c], __ldg(x + c) + __ldg(x + 3 + c));
            t[c] = acc[c];
        }
    }
}

// Encoding only (nrc_encode): one thread per record, logical feature order.
template <bool EXACT>
__global__ void nrc_encode_kernel(const float* __restrict__ rec, uint64_t n, EncodeParams ep, uint4* __restrict__ out,
                                  unsigned long long* degenerate) {
    __shared__ uint32_t scratch;
    if (threadIdx.x == 0) scratch = 0;
    __syncthreads();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    uint32_t deg = 0;
    if (i < n) {
        float r[16];
        load_record_global(rec + i * kRecFloats, r);
        uint32_t h[32];
        deg = encode_record<EXACT>(r, ep, h);
#pragma unroll
        for (int c = 0; c < 8; ++c) out[i * 8 + c] = make_uint4(h[4 * c], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]);
    }
    block_count_add(degenerate, deg, &scratch);
}

// ============================================================================ selftest
// One tile product per operand layout the fused kernels use (see nrc.h).
__global__ void __launch_bounds__(128, 1) nrc_selftest_kernel(int mode, const uint16_t* __restrict__ A,
                                                               const uint16_t* __restrict__ B, float* __restrict__ D) {
    __shared__ __align__(1024) uint8_t sA[kTileBytes];
    __shared__ __align__(1024) uint8_t sB[kTileBytes];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int blines = (mode == 2) ? 128 : (mode == 3) ? 16 : 64;
    const uint4* A4 = reinterpret_cast<const uint4*>(A);
    const uint4* B4 = reinterpret_cast<const uint4*>(B);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        uint4 x = A4[tid * 8 + c];
        st_shared_v4(smem_u32(sA) + swz(tid, c), x.x, x.y, x.z, x.w);
        if (int(tid) < blines) {
            uint4 y = B4[tid * 8 + c];
            st_shared_v4(smem_u32(sB) + swz(tid, c), y.x, y.y, y.z, y.w);
        }
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
    if (mode == 4) {  // A row of this thread -> TMEM columns 64..95 (2 fp16 per column)
        uint32_t row[32];
        const uint32_t* A32 = reinterpret_cast<const uint32_t*>(A);
#pragma unroll
        for (int q = 0; q < 32; ++q) row[q] = A32[tid * 32 + q];
        tmem_st32(tb + ((warp * 32u) << 16) + 64, row);
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    if (tid == 0) {
        const uint32_t a = smem_u32(sA), b = smem_u32(sB);
        if (mode == 4) {
            for (int k = 0; k < 4; ++k) umma_f16_ta(tb, tb + 64 + 8 * k, desc_kmajor(b, k), make_idesc(128, 64, 0, 0), k > 0);
        } else if (mode == 0) {
            for (int k = 0; k < 4; ++k) umma_f16(tb, desc_kmajor(a, k), desc_kmajor(b, k), make_idesc(128, 64, 0, 0), k > 0);
        } else if (mode == 1) {
            for (int k = 0; k < 4; ++k) umma_f16(tb, desc_kmajor(a, k), desc_mnmajor(b, k), make_idesc(128, 64, 0, 1), k > 0);
        } else if (mode == 2) {
            for (int k = 0; k < 8; ++k) umma_f16(tb, desc_mnmajor(a, k), desc_mnmajor(b, k), make_idesc(64, 64, 1, 1), k > 0);
        } else {
            for (int k = 0; k < 4; ++k) umma_f16(tb, desc_kmajor(a, k), desc_kmajor(b, k), make_idesc(128, 16, 0, 0), k > 0);
        }
        umma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    const uint32_t lane_off = (warp * 32u) << 16;
    if (mode == 2) {
        for (int half = 0; half < 2; ++half) {
            uint32_t v[32];
            tmem_ld32(tb + lane_off + 32 * half, v);
            const int o = int(warp) * 16 + int(lane);
            if (lane < 16)
                for (int q = 0; q < 32; ++q) D[o * 64 + 32 * half + q] = __uint_as_float(v[q]);
        }
    } else if (mode == 3) {
        uint32_t v[16];
        tmem_ld16(tb + lane_off, v);
        for (int q = 0; q < 16; ++q) D[tid * 16 + q] = __uint_as_float(v[q]);
    } else {
        for (int half = 0; half < 2; ++half) {
            uint32_t v[32];
            tmem_ld32(tb + lane_off + 32 * half, v);
            for (int q = 0; q < 32; ++q) D[tid * 64 + 32 * half + q] = __uint_as_float(v[q]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 128);
}

}  // namespace nrc
