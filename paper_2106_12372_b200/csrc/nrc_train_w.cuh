// nrc_train_w.cuh -- the training step at hidden width W in {32, 64, 128}
// (64 = the paper's network; 32 / 128 = the width ablation, BASELINE.json
// configs[3]): rows a0, a1, a4-a8 of SURVEY 8(a) (LCG gather
// P:L487-491 -> encode -> forward with the stash in SMEM -> Eq. 5 loss
// gradient P:L886-894 -> dgrad + wgrad on tcgen05), as one
// partials kernel per step followed by the reduce + Adam + EMA kernel
// (Eq. 2).
//
// Layout per CTA (one 128-row tile at a time, 4 row warps, warp 0 issues):
//  * stash: h0 (128 x 64 fp16) and h1..h5 (128 x W fp16, W/64 blocks of
//    128 lines of 128 B, SWIZZLE_128B; at W = 32 a line holds 32 values and
//    its other half stays zero).  The gradient g_j = delta_j * 1[h_j > 0]
//    overwrites h_j in place once dgrad_j and wgrad_j (the last readers of
//    h_j) have completed, so no separate gradient tiles exist.
//  * weights: W <= 64 keeps the whole fp16 image resident (one TMA load per
//    launch); W = 128 (151 KB image + 176 KB stash > 227 KB) streams one
//    layer (<= 32 KB) at a time into one buffer: W_{L+1} is fetched while
//    the epilogue of layer L runs, and W5 serves the forward and dgrad_5.
//  * TMEM: fwd / dgrad accumulator (max(W, 64) columns) + two wgrad
//    accumulators used alternately: G_{j+1} is drained to the CTA's fp32
//    partial while round j's MMAs run.
// MMA shapes (M x N x K, A/B majors):
//   forward L   128 x rows(L) x cols(L)      A = h_L K-major, B = W_L K-major
//   dgrad j     128 x max(W,64) x rows(j)    A = g_{j+1} K-major, B = W_j MN-major
//   wgrad j     M x N x 128 rows             A = g_{j+1}^T MN-major, B = h_j MN-major
//               M = 128 (W = 128, j < 5) else 64 (rows beyond W / 16 are 0)
//               N = 64 (j = 0) else max(W, 64) (columns beyond W are 0)
#pragma once
#include "nrc_common.cuh"

namespace nrc {

// Chunk-major layout of an fp32 gradient vector (CTA partials): layer i's
// block starts at pad_off(i) and holds element (o, c) at
// (c / 4) rows(i) + o float4s in, component c % 4.  A warp draining 16 / 32
// TMEM lanes (rows o) then stores one contiguous run per instruction, and the
// optimiser reads each float4 element of all partials with coalesced loads.
template <int W>
__device__ __forceinline__ int part_index(const NetRt<W>& D, int i, int o, int c) {
    return D.pad_off(i) + ((c >> 2) * D.rows(i) + o) * 4 + (c & 3);
}

template <int W>
struct TrainW {
    static constexpr bool kStream = W > 64;        // per-layer weight streaming
    static constexpr int kKB = (W + 63) / 64;      // 64-wide blocks of a hidden activation
    static constexpr int kNW = W > 64 ? W : 64;    // dgrad N, wgrad N (j >= 1), accumulator columns
    // depth variants: nh hidden layers, limited by the shared memory
    // of image + (nh + 1) stash slots + the dL/dy tile
    static constexpr int kMaxNh = W == 32 ? 8 : W == 64 ? 7 : 5;
    __host__ __device__ static constexpr int w_bytes(int nh) {
        return kStream ? kKB * W * 128 : (NetRt<W>(nh).img() + 1023) / 1024 * 1024;
    }
    __host__ __device__ static constexpr int stash_bytes(int nh) { return kTileBytes + nh * kKB * kTileBytes; }
    __host__ __device__ static constexpr int smem_bytes(int nh) {
        return 1024 + w_bytes(nh) + stash_bytes(nh) + kTileBytes + 96;
    }
    static constexpr uint32_t kTmemCols = 3 * kNW <= 256 ? 256u : 512u;
    __host__ __device__ static constexpr int slot_off(int i) { return i == 0 ? 0 : kTileBytes + (i - 1) * kKB * kTileBytes; }
    __host__ __device__ static constexpr int wg_n(int j) { return j == 0 ? 64 : kNW; }
};
static_assert(TrainW<32>::smem_bytes(TrainW<32>::kMaxNh) <= 232448 &&
                  TrainW<64>::smem_bytes(TrainW<64>::kMaxNh) <= 232448 &&
                  TrainW<128>::smem_bytes(TrainW<128>::kMaxNh) <= 232448,
              "227 KB of SMEM per CTA at the deepest supported network");

// SWIZZLE_128B descriptor with an explicit leading byte offset (the stride
// between 64-wide MN blocks of an MN-major operand, SBO = 8 lines = 1024 B).
__device__ __forceinline__ uint64_t desc_mn_lbo(uint32_t saddr, uint32_t lbo) { return make_sdesc(saddr, lbo, 1024u); }

// record + target of batch row `row` (zeros past the batch; row k of the
// step reads record lcg_perm(offset + k) when gathering, R15)
__device__ __forceinline__ void train_gather_row(const TrainArgs& a, uint32_t row, float (&rec)[16], float (&tg)[3]) {
    if (row < a.n) {
        const uint64_t k = row;
        const uint64_t idx = a.gather ? lcg_perm(a.offset + k, a.lcg_n, a.lcg_a, a.lcg_c, a.lcg_m) : k;
        const float* rsrc = a.rec + idx * kRecFloats;
        const float* tsrc = a.tgt + idx * 3;
        load_record_global(rsrc, rec);
#pragma unroll
        for (int c = 0; c < 3; ++c) tg[c] = __ldg(tsrc + c);
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) rec[i] = 0.0f;
#pragma unroll
        for (int c = 0; c < 3; ++c) tg[c] = 0.0f;
    }
}

// One training step's partials at width W: CTA c processes tiles c, c + grid,
// ... and writes its un-normalised fp32 gradient sum (padded layout of
// NetDims<W>) to partials[c] and its loss sum to loss_part[c].
// diagnostics (nrc_debug_set_trace): global-timer marks of each CTA at dbg[32 cta + k]
#define NRC_WTRC(k)                                                                     \
    do {                                                                                \
        if (a.dbg != nullptr && threadIdx.x == 0 && blockIdx.x < 127) a.dbg[32 * blockIdx.x + (k)] = global_ns(); \
    } while (0)
// EXACT: sin / Gaussian encoding primitives (NRC_EXACT_ENCODING, N4; width 64)
template <int W, bool EXACT = false>
__global__ void __launch_bounds__(128, 1) nrc_train_w_kernel(TrainArgs a) {
    const NetRt<W> D(int(a.nh));  // layer shapes / offsets at this depth (nh hidden layers)
    const int nh = D.nh;
    using T = TrainW<W>;
    const int wbytes = T::w_bytes(nh), stash_bytes = T::stash_bytes(nh);
    NRC_WTRC(0);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    const uint32_t tid = threadIdx.x, r = tid, warp = tid >> 5, lane = tid & 31;
    const uint32_t sW_a = smem_u32(smem);
    const uint32_t sH_a = sW_a + uint32_t(wbytes);
    const uint32_t sG6_a = sH_a + uint32_t(stash_bytes);  // dL/dy tile (columns 0..2 used)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + wbytes + stash_bytes + kTileBytes);
    uint64_t* wbar = &bars[0];
    uint64_t* wbar1 = &bars[10];  // resident image: W1 .. W_nh
    uint64_t* mma_bar = &bars[1];
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
    float* red = reinterpret_cast<float*>(bars + 3);  // 4 floats + 4 u32
    uint32_t* gmax = reinterpret_cast<uint32_t*>(bars + 7);  // per-warp max |dL/dy| (fp32 bits)
    uint32_t* deg_scratch = reinterpret_cast<uint32_t*>(bars + 9);

    if (tid == 0) {
        *deg_scratch = 0;
        mbar_init(wbar, 1);
        mbar_init(wbar1, 1);
        mbar_init(mma_bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, T::kTmemCols);
        tmem_relinquish();
    }
    // zero the dL/dy tile (only chunk 0 of a line is rewritten per tile) and, at
    // W < 64, the hidden slots (the upper half of each line is never written)
    {
        const uint32_t z0 = W < 64 ? sH_a + kTileBytes : sG6_a;
        for (uint32_t off = z0 + tid * 16; off < sG6_a + kTileBytes; off += 128 * 16) st_shared_v4(off, 0, 0, 0, 0);
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t lane_off = (warp * 32u) << 16;
    const uint32_t t_acc = tmem_base;
    auto t_g = [&](int j) -> uint32_t { return tmem_base + uint32_t(T::kNW) * (1u + uint32_t(j & 1)); };
    auto slot = [&](int i) -> uint32_t { return sH_a + uint32_t(T::slot_off(i)); };
    auto wl = [&](int L) -> uint32_t { return T::kStream ? sW_a : sW_a + uint32_t(D.img_off(L)); };
    // wgrad_j's M: the out-neuron rows (M = 64 holds rows 16 w + lane of warp w, lane < 16)
    auto wg_m = [&](int j) { return (j < nh && W > 64) ? 128 : 64; };

    uint32_t phase = 0, w_phase = 0;
    // weight bytes of layer L (streamed) or the whole image (resident), issued by thread 0
    // weight bytes of layer L (streamed), issued by thread 0; resident image
    // (L = 0): W0 on wbar and W1.. on wbar1, so layer 0 starts once its 8 KB land
    auto copy = [&](uint32_t off, uint32_t bytes, uint64_t* bar) {
        mbar_arrive_expect_tx(bar, bytes);
        for (uint32_t o = 0; o < bytes; o += 8192u) {
            const uint32_t b = bytes - o < 8192u ? bytes - o : 8192u;
            bulk_g2s(smem + (T::kStream ? 0u : off) + o, a.wimg + off + o, b, bar);
        }
    };
    auto fetch = [&](int L) {
        if (T::kStream) {
            copy(uint32_t(D.img_off(L)), uint32_t(D.img_off(L + 1) - D.img_off(L)), wbar);
        } else {
            copy(0u, uint32_t(D.img_off(1)), wbar);
            copy(uint32_t(D.img_off(1)), uint32_t(D.img() - D.img_off(1)), wbar1);
        }
    };
    auto wwait = [&]() {  // warp 0 only (the MMA issuer reads the weights)
        mbar_wait(wbar, w_phase);
        w_phase ^= 1;
    };
    auto mma_wait = [&]() {
        mbar_wait(mma_bar, phase);
        phase ^= 1;
        tc_fence_after();
    };
    auto sync_rows = [&]() {
        tc_fence_before();
        fence_async_smem();
        __syncthreads();
        tc_fence_after();
    };
    // forward layer L (whole warp 0, converged; one elected lane issues + commits)
    auto issue_fwd = [&](int L) {
        const uint32_t idesc = warp_uniform(make_idesc(128, D.rows(L), 0, 0));
        const uint64_t a0 = warp_uniform(desc_kmajor(slot(L), 0));
        const uint64_t a1 = warp_uniform(desc_kmajor(slot(L) + kTileBytes, 0));
        const uint64_t b0 = warp_uniform(desc_kmajor(wl(L), 0));
        const uint64_t b1 = warp_uniform(desc_kmajor(wl(L) + uint32_t(D.rows(L)) * 128u, 0));
        const uint32_t d = warp_uniform(t_acc);
        tc_fence_after();
        if (elect_one()) {
            if (D.cols(L) == 32) {
                umma_f16(d, a0, b0, idesc, 0u);
                umma_f16(d, a0 + 2, b0 + 2, idesc, 1u);
            } else {
                umma_ss4<kKmajStep, kKmajStep>(d, a0, b0, idesc, 0u);
                if (D.cols(L) == 128) umma_ss4<kKmajStep, kKmajStep>(d, a1, b1, idesc, 1u);
            }
            umma_commit(mma_bar);
        }
        __syncwarp();
    };
    // round j of the backward pass: dgrad_j (j >= 1) and wgrad_j, one commit
    auto issue_bwd = [&](int j) {
        const uint32_t gsrc = j == nh ? sG6_a : slot(j + 1);  // g_{j+1}
        const uint32_t d_acc = warp_uniform(t_acc), d_g = warp_uniform(t_g(j));
        // dgrad: delta_j = g_{j+1} W_j (K = rows(j) out-neurons)
        const uint32_t id_d = warp_uniform(make_idesc(128, T::kNW, 0, 1));
        const uint64_t da0 = warp_uniform(desc_kmajor(gsrc, 0));
        const uint64_t da1 = warp_uniform(desc_kmajor(gsrc + kTileBytes, 0));
        const uint64_t db = warp_uniform(desc_mn_lbo(wl(j), uint32_t(D.rows(j)) * 128u));
        // wgrad: G_j += g_{j+1}^T h_j (K = 128 rows)
        const uint32_t id_w = warp_uniform(make_idesc(wg_m(j), T::wg_n(j), 1, 1));
        const uint64_t wa = warp_uniform(desc_mn_lbo(gsrc, kTileBytes));
        const uint64_t wb = warp_uniform(desc_mn_lbo(slot(j), kTileBytes));
        tc_fence_after();
        if (elect_one()) {
            if (j >= 1) {
                if (j == nh) {
                    umma_f16(d_acc, da0, db, id_d, 0u);  // K = 16 (output layer, padded rows)
                } else if (W == 32) {
                    umma_f16(d_acc, da0, db, id_d, 0u);
                    umma_f16(d_acc, da0 + kKmajStep, db + kMNmajStep, id_d, 1u);
                } else {
                    umma_ss4<kKmajStep, kMNmajStep>(d_acc, da0, db, id_d, 0u);
                    if (W == 128) umma_ss4<kKmajStep, kMNmajStep>(d_acc, da1, db + 4 * kMNmajStep, id_d, 1u);
                }
            }
            umma_ss8<kMNmajStep, kMNmajStep>(d_g, wa, wb, id_w, 0u);
            umma_commit(mma_bar);
        }
        __syncwarp();
    };
    float* part = a.partials + size_t(blockIdx.x) * D.padded();
    // drain G_j (TMEM) into this CTA's partial (plain store on the first tile,
    // else add), undoing the tile's power-of-two dL/dy scale (exact in fp32);
    // chunk-major layout: for each store instruction the warp's rows write
    // consecutive 16-B chunks (one contiguous 256 / 512-B run)
    float inv_s = 1.0f;
    auto flush_g = [&](int j, bool first) {
        const int M = wg_m(j);
        const int o = M == 128 ? int(r) : int(warp) * 16 + int(lane);
        const int rows_pad = j < nh ? W : kOutPad;
        const bool valid = (M == 128 || lane < 16) && o < rows_pad;
        constexpr int kMaxParts32 = (W > 64 ? W : 64) / 32;
#pragma unroll
        for (int p = 0; p < kMaxParts32; ++p) {
            if (32 * p >= D.cols(j)) break;
            uint32_t v[32];
            tmem_ld32(t_g(j) + lane_off + 32u * p, v);
            if (valid) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int idx = part_index(D, j, o, 32 * p + 4 * q);
                    float4 x = make_float4(__uint_as_float(v[4 * q]) * inv_s, __uint_as_float(v[4 * q + 1]) * inv_s,
                                           __uint_as_float(v[4 * q + 2]) * inv_s, __uint_as_float(v[4 * q + 3]) * inv_s);
                    float4* dst = reinterpret_cast<float4*>(part + idx);
                    if (!first) {
                        const float4 y = *dst;
                        x.x += y.x, x.y += y.y, x.z += y.z, x.w += y.w;
                    }
                    *dst = x;
                }
            }
        }
    };
    // g_j = delta_j * 1[h_j > 0] written over h_j (ReLU'(0) = 0, R17)
    auto mask_epilogue = [&](int j) {
#pragma unroll
        for (int p = 0; p < W / 32; ++p) {
            uint32_t v[32];
            tmem_ld32(t_acc + lane_off + 32u * p, v);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t off = slot(j) + uint32_t(p >> 1) * kTileBytes + swz(r, uint32_t((p & 1) * 4 + q));
                const uint4 hv = ld_shared_v4(off);
                const float* f = reinterpret_cast<const float*>(v) + 8 * q;
                st_shared_v4(off, pack_h2(f[0], f[1]) & relu_mask(hv.x), pack_h2(f[2], f[3]) & relu_mask(hv.y),
                             pack_h2(f[4], f[5]) & relu_mask(hv.z), pack_h2(f[6], f[7]) & relu_mask(hv.w));
            }
        }
    };

    float loss_sum = 0.0f;
    uint32_t bad = 0, deg = 0;
    const uint32_t ntiles = (a.n + kTile - 1) / kTile;
    pdl_trigger();  // the optimiser kernel may launch (its griddepcontrol.wait covers this grid)
    bool first = true;
#pragma unroll 1
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const bool more = tile + gridDim.x < ntiles;
        const uint32_t row = tile * kTile + r;
        const bool valid = row < a.n;
        float rec[16], tg[3];
        train_gather_row(a, row, rec, tg);
        {
            uint32_t h[32];
            const uint32_t dg = encode_record<EXACT>(rec, a.ep, h);
            deg += valid ? dg : 0u;
            store_row_swz(slot(0), r, h);
        }
        if (first) {
            // the weights and this CTA's partial belong to the previous kernel
            // (launched with PDL) until it has completed
            NRC_WTRC(1);
            pdl_wait();
            NRC_WTRC(2);
            if (tid == 0) fetch(0);  // W0 (streamed) or the whole image
        }
        sync_rows();
        // ---------------- forward: h_{L+1} = relu(W_L h_L), y = W5 h5
#pragma unroll 1
        for (int L = 0; L <= nh; ++L) {
            if (warp == 0) {
                if (T::kStream || (L == 0 && first)) wwait();
                if (!T::kStream && L == 1 && first) mbar_wait(wbar1, 0);  // one launch = one image load
                issue_fwd(L);
            }
            mma_wait();
            if (nh == 5) NRC_WTRC(8 + L);
            if (T::kStream && L < nh && tid == 0) fetch(L + 1);  // the buffer is free
            if (L == nh) break;
#pragma unroll
            for (int p = 0; p < W / 32; ++p) {
                uint32_t v[32];
                tmem_ld32(t_acc + lane_off + 32u * p, v);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float* f = reinterpret_cast<const float*>(v) + 8 * q;
                    st_shared_v4(slot(L + 1) + uint32_t(p >> 1) * kTileBytes + swz(r, uint32_t((p & 1) * 4 + q)),
                                 pack_h2_relu(f[0], f[1]), pack_h2_relu(f[2], f[3]), pack_h2_relu(f[4], f[5]),
                                 pack_h2_relu(f[6], f[7]));
                }
            }
            sync_rows();
        }
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
                gy[c] = use ? 2.0f * d * f[c] * inv3den : 0.0f;
            }
            if (use) loss_sum += l * inv3den;
            if (a.pred != nullptr && valid) {
#pragma unroll
                for (int c = 0; c < 3; ++c) a.pred[size_t(row) * 3 + c] = yh[c];
            }
            // Per-tile power-of-two scale of dL/dy before the fp16 rounding
            // (R13, R25): the tile's largest |dL/dy| maps into [2^7, 2^8), so
            // HDR residuals (|dL/dy| up to ~1e7 at eps = 0.01) cannot overflow
            // fp16 and small ones keep full precision; undone exactly in fp32
            // when the weight gradients are drained (flush_g).
            {
                const uint32_t mx = __reduce_max_sync(
                    0xffffffffu, max(max(__float_as_uint(fabsf(gy[0])), __float_as_uint(fabsf(gy[1]))),
                                     __float_as_uint(fabsf(gy[2]))));
                if (lane == 0) gmax[warp] = mx;
                named_bar_sync(1, 128);
                const uint32_t tm = max(max(gmax[0], gmax[1]), max(gmax[2], gmax[3]));
                const int ex = int(tm >> 23);                  // biased exponent of the tile max
                const int k = min(max(134 - ex, -120), 120);   // 2^k * max in [2^7, 2^8)
                const float sc = __uint_as_float(uint32_t(127 + k) << 23);
                inv_s = __uint_as_float(uint32_t(127 - k) << 23);
#pragma unroll
                for (int c = 0; c < 3; ++c) gy[c] *= sc;
            }
            st_shared_v4(sG6_a + swz(r, 0), pack_h2(gy[0], gy[1]), pack_h2(gy[2], 0.0f), 0u, 0u);
        }
        sync_rows();
        NRC_WTRC(3);
        // ---------------- backward: round j = dgrad_j + wgrad_j, then
        // G_{j+1} drains while they run; g_j overwrites h_j after both complete
#pragma unroll 1
        for (int j = nh; j >= 1; --j) {
            if (warp == 0) {
                if (T::kStream && j < nh) wwait();  // W_j (the output layer is still resident from the forward)
                issue_bwd(j);
            }
            if (j < nh) flush_g(j + 1, first);
            if (nh == 5) NRC_WTRC(14 + 2 * (5 - j));
            mma_wait();
            if (nh == 5) NRC_WTRC(15 + 2 * (5 - j));
            if (T::kStream && tid == 0) {
                if (j > 1)
                    fetch(j - 1);
                else if (more)
                    fetch(0);  // the next tile's W0
            }
            mask_epilogue(j);
            if (nh == 5 && j >= 2) NRC_WTRC(24 + (5 - j));
            sync_rows();
            if (nh == 5 && j >= 2) NRC_WTRC(28 + (5 - j));
        }
        NRC_WTRC(4);
        if (warp == 0) issue_bwd(0);  // G_0 += g_1^T h_0 (no gradient w.r.t. the encoding)
        flush_g(1, first);
        mma_wait();
        flush_g(0, first);
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        NRC_WTRC(5);
        first = false;
    }
    // ---------------- this CTA's loss sum (fixed order over the 4 row warps)
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
    NRC_WTRC(6);
    block_count_add(a.degenerate, deg, deg_scratch);
    if (warp == 0) tmem_dealloc(tmem_base, T::kTmemCols);
}


// Reduce + Adam + EMA at width W.  Partials use the chunk-major layout
// (part_index): thread t of block b owns float4 element e = 32 b + lane of
// that layout, i.e. parameters (o, 4 c4 .. 4 c4 + 3) of one layer.
//   partials != nullptr: g = sum over p < np of partials[p][e] (ascending p
//   within each of the kAdamWarps warps, p = w mod kAdamWarps, then the warp sums in warp
//   order: deterministic for a given np);
//   tile_part != nullptr: the same over the peer table;
//   else g = grad_logical (logical layout = padded prefix; W5 pad rows 0).
//   grad_out: the reduced sum in the logical layout (nrc_train_backward).
//   apply: Adam (R11) + EMA (Eq. 2, R12) on g * inv_n, writing
//   the fp32 state and both fp16 operand images.
constexpr int kMaxDpTiles = 128;  // tiles per step in the fused peer all-reduce path
// 8 warps, 8 partial loads in flight per thread, ~84 registers: measured
// best against 16 warps or 16 loads in flight (one load round instead of two,
// but blocks that no longer fit beside the next step's partials CTAs) and
// against a 64-register bound that keeps two blocks beside a partials CTA
// (the next step's gather + encode then slows the reduction): 64.5 vs 72.7 /
// 72.7 / 68.6 us per 4-step frame
constexpr int kAdamWarps = 8;                  // warp w sums partials p = w mod kAdamWarps
constexpr int kAdamThreads = 32 * kAdamWarps;  // 32 float4 elements (128 parameters) per block
// a peer's (or our own) partial, read at system scope, not cached on this SM
__device__ __forceinline__ float ld_sys_f32(const float* p) {
    float v;
    asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ float4 ld_sys_v4(const float* p) {
    float4 v;
    asm volatile("ld.relaxed.sys.global.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
// Adam (R11) + EMA (Eq. 2, R12) of one parameter on the batch-mean
// gradient g; shared by the optimiser kernel and the fused optimiser stage
// so that both compile to the same arithmetic.  Returns 1 if g was
// non-finite (zeroed and counted).
struct AdamCoef {
    float lr, b1, b2, eps, inv_bc1, inv_bc2, ema_c1, ema_c2;
};
__device__ __forceinline__ uint32_t adam_ema(float g, const AdamCoef& k, float& m, float& v, float& w, float& e) {
    uint32_t bad = 0;
    if (!isfinite(g)) {
        g = 0.0f;
        bad = 1;
    }
    m = k.b1 * m + (1.0f - k.b1) * g;
    v = k.b2 * v + (1.0f - k.b2) * g * g;
    // sqrt.approx and the fast reciprocal-multiply division (relative error
    // <= 2 ulp on the update; the IEEE sqrtf / division slow paths, taken for
    // v = 0 entries, cost ~1.3 us on the step's critical path, DESIGN 5)
    w = w - __fdividef(k.lr * (m * k.inv_bc1), sqrt_approx(v * k.inv_bc2) + k.eps);
    e = k.ema_c1 * w + k.ema_c2 * e;
    return bad;
}
// L2 load kept in program order (not sunk below the partial loads)
__device__ __forceinline__ float4 ld_cg_v4(const float* p) {
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
// NVLink SHARP (NVLS): the sum over every rank's copy of a multicast-mapped
// buffer, reduced in the NVSwitch (fp32 accumulate) and returned to this SM
__device__ __forceinline__ float4 multimem_ld_reduce_v4(const float* mc) {
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(mc)
                 : "memory");
    return v;
}
__device__ __forceinline__ float multimem_ld_reduce_f32(const float* mc) {
    float v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc) : "memory");
    return v;
}
__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
struct AdamWArgs {
    const float* partials;
    int np;
    const float* grad_logical;
    float* grad_out;
    int apply;
    float inv_n;
    float *w, *m, *v, *ema;
    uint8_t *wimg, *eimg;
    float lr, b1, b2, eps, inv_bc1, inv_bc2, ema_c1, ema_c2;
    unsigned long long* bad_grads;
    const float* loss_part;  // optional: loss partial sums -> loss_out (x loss_scale)
    int nloss;
    float loss_scale;
    float* loss_out;
    long long* dbg;          // diagnostics: global-timer marks of blocks 0 and last at dbg[4088..4091]
    int nh;                  // hidden layers (depth variants)
    // peer mode (nrc_train_frame_dp_peer), if tile_part != nullptr: device
    // tables of np pointers -- partial p of the reduction is the tile-p partial
    // at tile_part[p] (in its owner's arena, possibly a peer's), loss partial p
    // at tile_loss[p].  (Tables in device memory keep the kernel parameters
    // small: a 2 KB parameter block measurably slowed every launch.)
    const float* const* tile_part;
    const float* const* tile_loss;
    // NVLS mode (nrc_train_apply_multimem), if grad_mc != nullptr: the
    // multicast address of every rank's [logical gradient sum | loss sum];
    // g = multimem.ld_reduce (the all-reduce done in the switch), loss likewise
    const float* grad_mc;
    // peer mode (nrc_train_apply_peers), if peer_grad != nullptr: a device
    // table of npeer pointers to every rank's [logical gradient sum | loss
    // sum] (peer memory over NVLink); g = their sum in rank order, identical
    // on every rank
    const float* const* peer_grad;
    int npeer;
};

#ifndef NRC_ADAM_BOUNDS
#define NRC_ADAM_BOUNDS __launch_bounds__(kAdamThreads, 1)
#endif
template <int W>
__global__ void NRC_ADAM_BOUNDS nrc_adam_w_kernel(AdamWArgs a) {
    const NetRt<W> D(a.nh);  // padded(nh) is a multiple of 128 for every width and depth
    __shared__ float4 sred[kAdamWarps][32];
    const int lane = int(threadIdx.x & 31), wp = int(threadIdx.x >> 5);
    const int e = int(blockIdx.x) * 32 + lane;  // float4 element of the chunk-major layout
    const int k = 4 * e;
    const int i = D.layer_of(k);  // one layer per block (layer sizes are multiples of 128)
    pdl_wait();  // launched as a programmatic dependent of the partials kernel
#ifndef NRC_ADAM_LATE_TRIGGER
    pdl_trigger();  // the next step's partials kernel may become resident (its griddepcontrol.wait covers this grid)
#endif
    const bool trc = a.dbg != nullptr && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x + 1 == gridDim.x);
    if (trc) a.dbg[4088 + 2 * (blockIdx.x != 0)] = global_ns();

    const int R = D.rows(i), C = D.cols(i);
    const int local = (k - D.pad_off(i)) >> 2;
    const int c4 = local / R, o = local - c4 * R;
    const int j0 = D.pad_off(i) + o * C + 4 * c4;  // row-major padded index of the 4 parameters
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    // the optimiser state (m, v, w, W-bar), one vector per warp 1..4, loaded
    // under the partial loads (one L2 round trip) and handed to warp 0 through
    // shared memory (4 registers per thread instead of 16: two optimiser
    // blocks fit on an SM beside a partials CTA)
    static_assert(kAdamWarps >= 5, "warps 1..4 load the optimiser state");
    __shared__ float4 sstate[4][32];
    float4 st = g;
    if (a.apply && wp >= 1 && wp <= 4) st = ld_cg_v4((wp == 1 ? a.m : wp == 2 ? a.v : wp == 3 ? a.w : a.ema) + j0);
    const bool from_partials = a.tile_part != nullptr || a.partials != nullptr;
    if (from_partials) {
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        const size_t stride = size_t(D.padded()) / 4;
        const float4* src = reinterpret_cast<const float4*>(a.partials) + e;
#ifndef NRC_ADAM_KIN
#define NRC_ADAM_KIN 8
#endif
        constexpr int kIn = NRC_ADAM_KIN;  // partial loads in flight per thread
        if (a.tile_part != nullptr) {  // fused all-reduce: NVLink loads for peers
#pragma unroll 1
            for (int p0 = wp; p0 < a.np; p0 += kAdamWarps * kIn) {
                float4 x[kIn];
#pragma unroll
                for (int u = 0; u < kIn; ++u) {
                    const int p = p0 + kAdamWarps * u;
                    x[u] = p >= a.np ? make_float4(0.f, 0.f, 0.f, 0.f) : ld_sys_v4(a.tile_part[p] + k);
                }
#pragma unroll
                for (int u = 0; u < kIn; ++u) s = f4_add(s, x[u]);
            }
        } else {
#pragma unroll 1
            for (int p0 = wp; p0 < a.np; p0 += kAdamWarps * kIn) {
                float4 x[kIn];
                const float4* sp = src + size_t(p0) * stride;
#pragma unroll
                for (int u = 0; u < kIn; ++u)
                    x[u] = p0 + kAdamWarps * u >= a.np ? make_float4(0.f, 0.f, 0.f, 0.f)
                                                       : __ldcg(sp + size_t(kAdamWarps * u) * stride);
#pragma unroll
                for (int u = 0; u < kIn; ++u) s = f4_add(s, x[u]);
            }
        }
        if (trc) a.dbg[4086 + (blockIdx.x != 0)] = global_ns();
        sred[wp][lane] = s;
    } else if (wp == 0 && a.peer_grad != nullptr) {
        if (j0 < D.logical()) {  // 4 consecutive logical entries; all ranks' loads in flight, then the sum in rank order
            float4 x[kMaxRanks];
#pragma unroll
            for (int p = 0; p < kMaxRanks; ++p) x[p] = p < a.npeer ? ld_sys_v4(a.peer_grad[p] + j0) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int p = 0; p < kMaxRanks; ++p)
                if (p < a.npeer) g = f4_add(g, x[p]);
        }
    } else if (wp == 0 && a.grad_mc != nullptr) {
        // 4 consecutive logical entries (j0 % 4 == 0; W5's pad rows are beyond logical)
        if (j0 < D.logical()) g = multimem_ld_reduce_v4(a.grad_mc + j0);
    } else if (wp == 0) {
        float gg[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) gg[q] = j0 + q < D.logical() ? a.grad_logical[j0 + q] : 0.0f;
        g = make_float4(gg[0], gg[1], gg[2], gg[3]);
    }
    if (wp >= 1 && wp <= 4) sstate[wp - 1][lane] = st;
    __syncthreads();
    if (trc) a.dbg[4084 + (blockIdx.x != 0)] = global_ns();
    if (wp == 0 && from_partials) {
#pragma unroll
        for (int q = 0; q < kAdamWarps; ++q) g = f4_add(g, sred[q][lane]);
    }
    if (wp == 1 && blockIdx.x == 0 && a.loss_out != nullptr) {
        // the batch loss, off warp 0's critical path: all loads in flight,
        // then each lane's sum in partial order and a butterfly
        float s = 0.0f;
        if (a.peer_grad != nullptr) {
            if (lane == 0)
                for (int p = 0; p < a.npeer; ++p) s += ld_sys_f32(a.peer_grad[p] + D.logical());
        } else if (a.grad_mc != nullptr) {
            if (lane == 0) s = multimem_ld_reduce_f32(a.grad_mc + D.logical());
        } else {
#pragma unroll 1
            for (int p0 = lane; p0 < a.nloss; p0 += 4 * 32) {
                float x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int p = p0 + 32 * u;
                    x[u] = p >= a.nloss ? 0.0f : a.tile_part != nullptr ? ld_sys_f32(a.tile_loss[p]) : __ldcg(a.loss_part + p);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (p0 + 32 * u < a.nloss) s += x[u];
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) *a.loss_out = s * a.loss_scale;
        return;
    }
    if (wp != 0) return;
    const float4 m = sstate[0][lane], v = sstate[1][lane], w = sstate[2][lane], em = sstate[3][lane];
    float gq[4] = {g.x, g.y, g.z, g.w};
    if (a.grad_out != nullptr) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (j0 + q < D.logical()) a.grad_out[j0 + q] = gq[q];
    }
    if (!a.apply) return;
    float mq[4] = {m.x, m.y, m.z, m.w}, vq[4] = {v.x, v.y, v.z, v.w}, wq[4] = {w.x, w.y, w.z, w.w},
          eq[4] = {em.x, em.y, em.z, em.w};
    const AdamCoef kc{a.lr, a.b1, a.b2, a.eps, a.inv_bc1, a.inv_bc2, a.ema_c1, a.ema_c2};
    uint32_t nbad = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) nbad += adam_ema(gq[q] * a.inv_n, kc, mq[q], vq[q], wq[q], eq[q]);
    if (nbad) atomicAdd(a.bad_grads, (unsigned long long)nbad);
    if (trc) a.dbg[4092 + (blockIdx.x != 0)] = global_ns();
    *reinterpret_cast<float4*>(a.m + j0) = make_float4(mq[0], mq[1], mq[2], mq[3]);
    *reinterpret_cast<float4*>(a.v + j0) = make_float4(vq[0], vq[1], vq[2], vq[3]);
    *reinterpret_cast<float4*>(a.w + j0) = make_float4(wq[0], wq[1], wq[2], wq[3]);
    *reinterpret_cast<float4*>(a.ema + j0) = make_float4(eq[0], eq[1], eq[2], eq[3]);
    // 4 consecutive columns = 8 contiguous bytes of one 16-B chunk of the image
    const uint32_t off = D.img_byte(i, o, 4 * c4);
    *reinterpret_cast<uint2*>(a.wimg + off) = make_uint2(pack_h2(wq[0], wq[1]), pack_h2(wq[2], wq[3]));
    *reinterpret_cast<uint2*>(a.eimg + off) = make_uint2(pack_h2(eq[0], eq[1]), pack_h2(eq[2], eq[3]));
    if (trc) a.dbg[4089 + 2 * (blockIdx.x != 0)] = global_ns();

}

// Fused peer all-reduce hand-off (nrc_train_frame_dp_peer), one thread: after
// this rank's partials kernel (stream order), publish them to every rank with
// a system-scope release add on its counter, then wait until all `world` ranks
// have published step `target / world` (acquire).  Bounded: after ~20 s it
// gives up and counts a timeout instead of hanging the GPU.
struct DpPeers {
    unsigned long long* ctr[kMaxRanks];  // every rank's hand-off counter (own included)
};
__global__ void nrc_dp_exchange_kernel(DpPeers peers, int world, unsigned long long* own, unsigned long long target,
                                       unsigned long long* timeouts) {
    pdl_trigger();  // the optimiser kernel may become resident (it waits for this grid)
    if (threadIdx.x != 0) return;
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int p = 0; p < world; ++p)
        asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(peers.ctr[p]) : "memory");
    const long long t0 = global_ns();
    unsigned long long v = 0;
    while (true) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(own) : "memory");
        if (v >= target) break;
        if (global_ns() - t0 > 20000000000ll) {
            atomicAdd(timeouts, 1ull);
            break;
        }
        __nanosleep(128);
    }
}

}  // namespace nrc
