// nrc_kernels.cuh -- the sm_100a kernels of libnrc.
//
//   nrc_query_kernel   fused encode -> 6 x tcgen05 layer -> factorised output
//                      (P:L602-628 fully fused MLP; Table 1)
//   nrc_train_kernel   fused encode -> forward (stash kept in SMEM) -> relative
//                      L2 loss gradient (Eq. 5) -> dgrad -> wgrad (both on
//                      tcgen05, accumulators in TMEM) -> per-CTA fp32 partials
//                      (where the paper used CUTLASS split-k)
//   nrc_adam_kernel    deterministic partial reduction + Adam + EMA (Eq. 2) +
//                      fp16 operand images
//   helpers            encode-only, partial reduction, image refresh, selftest
#pragma once
#include "nrc_device.cuh"
#include "nrc_fused_query.cuh"

namespace nrc {

// ============================================================================ train
struct TrainArgs {
    const float* rec;      // records (indexed through the gather below)
    const float* tgt;      // targets, 3 fp32 per record
    uint32_t n;            // rows in this batch
    uint32_t gather;       // 1: row k reads record lcg_perm(offset + k)
    uint64_t lcg_a, lcg_c, lcg_m, lcg_n, offset;
    const uint8_t* wimg;   // fp16 image of the TRAINING weights W_t
    EncodeParams ep;
    uint32_t flags;
    float loss_eps;
    float* partials;       // [gridDim.x][kParamPadded] fp32 un-normalised gradient sums
    float* loss_part;      // [gridDim.x] loss sums
    unsigned long long* bad_targets;
};

constexpr int kTrainSmemBytes = 1024 + kImgBytes + 7 * kTileBytes + 64 + 64;
constexpr uint32_t kTrainTmemCols = 512;  // acc 64 + 6 wgrad accumulators x 64

// One CTA per 128-row tile (persistent over tiles if n > 128 * grid).  The
// activation stash h0..h5 stays in SMEM (6 x 16 KB), each gradient g_i
// overwrites h_i in place once h_i's last reader (its wgrad MMA and the ReLU
// mask) has completed.  All six weight-gradient accumulators live in TMEM for
// the whole kernel and are written out once as this CTA's partial.
__global__ void __launch_bounds__(128, 1) nrc_train_kernel(TrainArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    const uint32_t tid = threadIdx.x, r = tid, warp = tid >> 5, lane = tid & 31;
    uint8_t* sW = smem;
    uint8_t* sSlot = smem + kImgBytes;                  // 6 tiles: h0..h5 (then g1..g5 in place)
    uint8_t* sG6 = smem + kImgBytes + 6 * kTileBytes;   // d loss / d y tile (cols 0..2 used)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kImgBytes + 7 * kTileBytes);
    uint64_t* wbar = &bars[0];
    uint64_t* mma_bar = &bars[1];
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
    float* red = reinterpret_cast<float*>(bars + 4);    // 4 floats + 4 u32

    if (tid == 0) {
        mbar_init(wbar, 1);
        mbar_init(mma_bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, kTrainTmemCols);
        tmem_relinquish();
    }
    // zero the dL/dy tile once: only chunk 0 of each line is rewritten per tile
    {
        const uint32_t base = smem_u32(sG6);
        for (uint32_t off = tid * 16; off < kTileBytes; off += 128 * 16) st_shared_v4(base + off, 0, 0, 0, 0);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (tid == 0) {
        mbar_arrive_expect_tx(wbar, kImgBytes);
        bulk_g2s(sW, a.wimg, kImgBytes, wbar);
    }

    const uint32_t sW_a = smem_u32(sW), sS_a = smem_u32(sSlot), sG6_a = smem_u32(sG6);
    const uint32_t lane_off = (warp * 32u) << 16;
    const uint32_t t_acc = tmem_base;                // 64 cols
    const uint32_t idesc_fwd = make_idesc(128, 64, 0, 0);
    const uint32_t idesc_out = make_idesc(128, 16, 0, 0);
    const uint32_t idesc_dgrad = make_idesc(128, 64, 0, 1);
    const uint32_t idesc_wgrad = make_idesc(64, 64, 1, 1);
    auto slot = [&](int i) -> uint32_t { return sS_a + i * kTileBytes; };
    auto t_wg = [&](int i) -> uint32_t { return tmem_base + 64u + 64u * i; };

    uint32_t phase = 0;
    float loss_sum = 0.0f;
    uint32_t bad = 0;
    bool first = true;
    const uint32_t ntiles = (a.n + kTile - 1) / kTile;
    mbar_wait(wbar, 0);

    auto mma_wait = [&]() {
        mbar_wait(mma_bar, phase);
        phase ^= 1;
        tc_fence_after();
    };
    auto sync_for_mma = [&]() {
        tc_fence_before();
        fence_async_smem();
        __syncthreads();
    };

#pragma unroll 1
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t row = tile * kTile + r;
        const bool valid = row < a.n;
        float rec[16];
        float tg[3] = {0.f, 0.f, 0.f};
        if (valid) {
            const uint64_t idx = a.gather ? lcg_perm(a.offset + row, a.lcg_n, a.lcg_a, a.lcg_c, a.lcg_m) : row;
            load_record_global(a.rec + idx * kRecFloats, rec);
#pragma unroll
            for (int c = 0; c < 3; ++c) tg[c] = __ldg(a.tgt + idx * 3 + c);
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) rec[i] = 0.0f;
        }
        {
            uint32_t h[32];
            encode_record(rec, a.ep, h);
            store_row_swz(slot(0), r, h);
        }
        sync_for_mma();

        // ---------------- forward: h_{i+1} = relu(W_i h_i), y = W5 h5
#pragma unroll 1
        for (int L = 0; L < 5; ++L) {
            if (tid == 0) {
                tc_fence_after();
                const uint32_t wl = sW_a + layer_off(L) * 2;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    umma_f16(t_acc, desc_kmajor(slot(L), k), desc_kmajor(wl, k), idesc_fwd, k > 0);
                umma_commit(mma_bar);
            }
            mma_wait();
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t v[32];
                tmem_ld32(t_acc + lane_off + 32 * half, v);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float* f = reinterpret_cast<const float*>(v) + 8 * c;
                    st_shared_v4(slot(L + 1) + swz(r, 4 * half + c), pack_h2_relu(f[0], f[1]),
                                 pack_h2_relu(f[2], f[3]), pack_h2_relu(f[4], f[5]), pack_h2_relu(f[6], f[7]));
                }
            }
            sync_for_mma();
        }
        if (tid == 0) {
            tc_fence_after();
            const uint32_t wl = sW_a + layer_off(5) * 2;
#pragma unroll
            for (int k = 0; k < 4; ++k) umma_f16(t_acc, desc_kmajor(slot(5), k), desc_kmajor(wl, k), idesc_out, k > 0);
            umma_commit(mma_bar);
        }
        mma_wait();
        // ---------------- relative L2 loss, Eq.(5) (R8-R10, R13)
        {
            uint32_t v[4];
            tmem_ld4(t_acc + lane_off, v);
            const bool use = valid && isfinite(tg[0]) && isfinite(tg[1]) && isfinite(tg[2]);
            if (valid && !use) ++bad;
            float yh[3], f[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                f[c] = (a.flags & 1u) ? rec[10 + c] + rec[13 + c] : 1.0f;
                yh[c] = __uint_as_float(v[c]) * f[c];
            }
            const float lam = 0.2126f * yh[0] + 0.7152f * yh[1] + 0.0722f * yh[2];
            const float den = lam * lam + a.loss_eps;
            const float inv3den = 1.0f / (3.0f * den);
            float gy[3], l = 0.0f;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float d = yh[c] - tg[c];
                l += d * d;
                gy[c] = use ? 2.0f * d * f[c] * inv3den : 0.0f;  // dl/dy_c, lambda stop-gradient
            }
            if (use) loss_sum += l * inv3den;
            st_shared_v4(sG6_a + swz(r, 0), pack_h2(gy[0], gy[1]), pack_h2(gy[2], 0.0f), 0u, 0u);
        }
        sync_for_mma();

        // ---------------- backward: layer 5
        if (tid == 0) {
            tc_fence_after();
            const uint32_t w5 = sW_a + layer_off(5) * 2;
            umma_f16(t_acc, desc_kmajor(sG6_a, 0), desc_mnmajor(w5, 0), idesc_dgrad, 0);  // delta5 = gy W5
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // G5 += gy^T h5
                umma_f16(t_wg(5), desc_mnmajor(sG6_a, kk), desc_mnmajor(slot(5), kk), idesc_wgrad,
                         (first && kk == 0) ? 0u : 1u);
            umma_commit(mma_bar);
        }
        mma_wait();
        // g_i = delta_i * 1[h_i > 0] written over h_i (ReLU'(0) = 0, R17)
        auto mask_epilogue = [&](int i) {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t v[32];
                tmem_ld32(t_acc + lane_off + 32 * half, v);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint32_t addr = slot(i) + swz(r, 4 * half + c);
                    const uint4 hv = ld_shared_v4(addr);
                    const float* f = reinterpret_cast<const float*>(v) + 8 * c;
                    st_shared_v4(addr, pack_h2(f[0], f[1]) & __vcmpne2(hv.x & 0x7FFF7FFFu, 0u),
                                 pack_h2(f[2], f[3]) & __vcmpne2(hv.y & 0x7FFF7FFFu, 0u),
                                 pack_h2(f[4], f[5]) & __vcmpne2(hv.z & 0x7FFF7FFFu, 0u),
                                 pack_h2(f[6], f[7]) & __vcmpne2(hv.w & 0x7FFF7FFFu, 0u));
                }
            }
        };
        mask_epilogue(5);
        sync_for_mma();
#pragma unroll 1
        for (int i = 4; i >= 0; --i) {
            if (tid == 0) {
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)  // G_i += g_{i+1}^T h_i
                    umma_f16(t_wg(i), desc_mnmajor(slot(i + 1), kk), desc_mnmajor(slot(i), kk), idesc_wgrad,
                             (first && kk == 0) ? 0u : 1u);
                if (i >= 1) {
                    const uint32_t wl = sW_a + layer_off(i) * 2;
#pragma unroll
                    for (int k = 0; k < 4; ++k)  // delta_i = g_{i+1} W_i
                        umma_f16(t_acc, desc_kmajor(slot(i + 1), k), desc_mnmajor(wl, k), idesc_dgrad, k > 0);
                }
                umma_commit(mma_bar);
            }
            mma_wait();
            if (i >= 1) {
                mask_epilogue(i);
                sync_for_mma();
            }
        }
        first = false;
    }

    // ---------------- write this CTA's gradient partial (M=64 TMEM layout:
    // row o lives in lane (o % 16) + 32 (o / 16); warp w holds o = 16 w + lane, lane < 16)
    float* part = a.partials + size_t(blockIdx.x) * kParamPadded;
#pragma unroll 1
    for (int i = 0; i < 6; ++i) {
        const int rows = (i < 5) ? 64 : kOutPad;
        const int o = int(warp) * 16 + int(lane);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            uint32_t v[32];
            tmem_ld32(t_wg(i) + lane_off + 32 * half, v);
            if (lane < 16 && o < rows) {
                float4* dst = reinterpret_cast<float4*>(part + layer_off(i) + o * 64 + 32 * half);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float4 x = first ? make_float4(0.f, 0.f, 0.f, 0.f)
                                     : make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                                   __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
                    dst[q] = x;
                }
            }
        }
    }
    // ---------------- loss sum (fixed-order reduction)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        loss_sum += __shfl_xor_sync(0xffffffffu, loss_sum, off);
        bad += __shfl_xor_sync(0xffffffffu, bad, off);
    }
    if (lane == 0) {
        red[warp] = loss_sum;
        reinterpret_cast<uint32_t*>(red + 4)[warp] = bad;
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
        a.loss_part[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
        const uint32_t* b = reinterpret_cast<const uint32_t*>(red + 4);
        const uint32_t nb = b[0] + b[1] + b[2] + b[3];
        if (nb) atomicAdd(a.bad_targets, (unsigned long long)nb);
    }
    if (warp == 0) tmem_dealloc(tmem_base, kTrainTmemCols);
}

// ============================================================================ Adam + EMA
struct AdamArgs {
    const float* src;        // gradient source
    int nsrc;                // number of padded partials (src_logical == 0)
    int src_logical;         // 1: src is a single logical-layout gradient sum
    float inv_n;             // 1 / N (batch mean, R10/R13)
    float *w, *m, *v, *ema;  // fp32 padded arrays
    uint8_t *wimg, *eimg;    // fp16 operand images
    float lr, b1, b2, eps, inv_bc1, inv_bc2;
    float ema_c1, ema_c2;    // W-bar = c1 W + c2 W-bar (Eq. 2 / R12)
    unsigned long long* bad_grads;
    const float* loss_part;  // optional: loss partial sums
    int nloss;
    float loss_scale;
    float* loss_out;
};

__device__ __forceinline__ void padded_coords(int j, int& layer, int& row, int& col) {
    layer = j < 20480 ? (j >> 12) : 5;
    const int rel = j - layer_off(layer);
    row = rel >> 6;
    col = rel & 63;
}
__device__ __forceinline__ uint32_t image_offset(int layer, int row, int col) {
    return uint32_t(layer_off(layer)) * 2u + uint32_t(row) * 128u + ((uint32_t(col >> 3) ^ uint32_t(row & 7)) << 4) +
           uint32_t(col & 7) * 2u;
}
__device__ __forceinline__ int logical_index(int layer, int row, int col) {
    if (layer < 5) return layer_off(layer) + row * 64 + col;
    return row < 3 ? 20480 + row * 64 + col : -1;
}

// Block-level fixed-order sum of partials[p][j] over p < np for the 32
// parameters j = 32*blockIdx.x + lane: warp w sums p = w, w+8, ... in
// ascending order, then warp 0 adds the 8 warp sums in warp order.  The same
// order in nrc_adam_kernel and nrc_reduce_kernel keeps nrc_train_step and
// nrc_train_backward + nrc_train_apply bitwise identical.
constexpr int kRedThreads = 256;
constexpr int kRedWarps = kRedThreads / 32;
__device__ __forceinline__ float block_partial_sum(const float* __restrict__ partials, int np, int j) {
    __shared__ float sred[kRedWarps][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float s = 0.0f;
    const float* p0 = partials + j;
#pragma unroll 4
    for (int p = w; p < np; p += kRedWarps) s += __ldcg(p0 + size_t(p) * kParamPadded);
    sred[w][lane] = s;
    __syncthreads();
    float t = 0.0f;
    if (w == 0) {
#pragma unroll
        for (int k = 0; k < kRedWarps; ++k) t += sred[k][lane];
    }
    return t;
}
__device__ __forceinline__ float warp_loss_sum(const float* __restrict__ part, int np) {
    float s = 0.0f;
    for (int p = threadIdx.x & 31; p < np; p += 32) s += part[p];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    return s;
}

// grid = kParamPadded / 32 blocks of kRedThreads; warp 0 updates 32 parameters.
__global__ void __launch_bounds__(kRedThreads) nrc_adam_kernel(AdamArgs a) {
    const int j = blockIdx.x * 32 + (threadIdx.x & 31);
    float g = 0.0f;
    if (!a.src_logical) g = block_partial_sum(a.src, a.nsrc, j);
    if (threadIdx.x >= 32) return;
    if (blockIdx.x == 0 && a.loss_out != nullptr) {
        const float s = warp_loss_sum(a.loss_part, a.nloss);
        if (threadIdx.x == 0) *a.loss_out = s * a.loss_scale;
    }
    int layer, row, col;
    padded_coords(j, layer, row, col);
    if (a.src_logical) {
        const int li = logical_index(layer, row, col);
        g = li >= 0 ? a.src[li] : 0.0f;
    }
    g *= a.inv_n;
    if (!isfinite(g)) {
        g = 0.0f;
        atomicAdd(a.bad_grads, 1ull);
    }
    float m = a.m[j], v = a.v[j], w = a.w[j], e = a.ema[j];
    m = a.b1 * m + (1.0f - a.b1) * g;
    v = a.b2 * v + (1.0f - a.b2) * g * g;
    w = w - a.lr * (m * a.inv_bc1) / (sqrtf(v * a.inv_bc2) + a.eps);
    e = a.ema_c1 * w + a.ema_c2 * e;
    a.m[j] = m;
    a.v[j] = v;
    a.w[j] = w;
    a.ema[j] = e;
    const uint32_t off = image_offset(layer, row, col);
    *reinterpret_cast<__half*>(a.wimg + off) = __float2half_rn(w);
    *reinterpret_cast<__half*>(a.eimg + off) = __float2half_rn(e);
}

// Rebuild an fp16 operand image from an fp32 padded array.
__global__ void nrc_image_kernel(const float* __restrict__ w, uint8_t* __restrict__ img) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= kParamPadded) return;
    int layer, row, col;
    padded_coords(j, layer, row, col);
    *reinterpret_cast<__half*>(img + image_offset(layer, row, col)) = __float2half_rn(w[j]);
}

// Sum the per-CTA partials in fixed order into a logical-layout gradient
// (nrc_train_backward), plus the loss sum.
// grid = kParamPadded / 32 blocks of kRedThreads (same order as Adam's sum).
__global__ void __launch_bounds__(kRedThreads) nrc_reduce_kernel(const float* __restrict__ partials, int np,
                                                                 float* __restrict__ grad,
                                                                 const float* __restrict__ loss_part,
                                                                 float* loss_sum) {
    const int j = blockIdx.x * 32 + (threadIdx.x & 31);
    const float g = block_partial_sum(partials, np, j);
    if (threadIdx.x >= 32) return;
    if (blockIdx.x == 0 && loss_sum != nullptr) {
        const float s = warp_loss_sum(loss_part, np);
        if (threadIdx.x == 0) *loss_sum = s;
    }
    int layer, row, col;
    padded_coords(j, layer, row, col);
    const int li = logical_index(layer, row, col);
    if (li >= 0) grad[li] = g;
}

// Encoding only (nrc_encode): one thread per record, logical feature order.
__global__ void nrc_encode_kernel(const float* __restrict__ rec, uint64_t n, EncodeParams ep, uint4* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float r[16];
    load_record_global(rec + i * kRecFloats, r);
    uint32_t h[32];
    encode_record(r, ep, h);
#pragma unroll
    for (int c = 0; c < 8; ++c) out[i * 8 + c] = make_uint4(h[4 * c], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]);
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
