// nrc_train_ws.cuh -- the training step's partials kernel with the weight
// gradients taken off the backward critical path (hidden width W <= 64,
// nh <= 6 hidden layers: the paper's network and the narrower / shallower
// variants).  Same arithmetic as nrc_train_w_kernel (rows a0, a1, a4-a7 of
// SURVEY 8(a)), different schedule:
//
//  * the gradient g_j = delta_j * 1[h_j > 0] goes to one of two g tiles
//    (g_j in gbuf[j & 1]) instead of over h_j, so wgrad_j (which reads h_j)
//    no longer has to finish before the mask epilogue of round j;
//  * round j issues dgrad_j -> commit(bar_d), wgrad_j -> commit(bar_w[j]);
//    the rows wait for bar_d only, so the mask epilogue of round j runs
//    while wgrad_j is on the tensor pipe (the in-order pipe finishes wgrad_j
//    before dgrad_{j-1}, whose commit therefore also covers gbuf reuse);
//  * every layer has its own TMEM accumulator G_j (64 + 64 (nh + 1) <= 512
//    columns) and four FLUSH warps (4..7, one per TMEM lane quadrant) drain
//    G_j into the CTA's fp32 partial once bar_w[j] has completed -- the rows
//    never touch the gradient accumulators;
//  * a dedicated ISSUER warp (8) issues every MMA chain: tcgen05.mma issue
//    blocks the issuing thread until the tensor pipe takes the instructions
//    (a round's 12 MMAs hold it for most of the round), so the row warps only
//    hand off (bar.arrive on named barrier 3; the issuer bar.syncs) and never
//    stall behind the pipe.
// One 128-row tile per CTA (batches of up to 128 x SMs rows, e.g. the
// paper's 16,384); larger batches use nrc_train_w_kernel.
#pragma once
#include "nrc_train_w.cuh"

namespace nrc {

#ifndef NRC_WS_MAXNREG
#define NRC_WS_MAXNREG __maxnreg__(112)
#endif
template <int W>
struct TrainWs {
    static_assert(W == 32 || W == 64, "the split schedule keeps one 64-column TMEM accumulator per layer");
    static constexpr int kMaxNh = 6;                 // 64 + 64 (nh + 1) <= 512 TMEM columns
    static constexpr int kThreads = 288;             // 4 row warps + 4 flush warps + the MMA issuer warp
    __host__ __device__ static constexpr int w_bytes(int nh) { return (NetRt<W>(nh).img() + 1023) / 1024 * 1024; }
    __host__ __device__ static constexpr int stash_bytes(int nh) { return kTileBytes + nh * kTileBytes; }
    // image + stash h0..h_nh + 2 g tiles + the dL/dy tile + barriers
    __host__ __device__ static constexpr int smem_bytes(int nh) {
        return 1024 + w_bytes(nh) + stash_bytes(nh) + 3 * kTileBytes + 256;
    }
};
static_assert(TrainWs<64>::smem_bytes(TrainWs<64>::kMaxNh) <= 232448, "227 KB of SMEM per CTA");

template <int W, bool EXACT = false>
__global__ void NRC_WS_MAXNREG nrc_train_ws_kernel(TrainArgs a) {
    const NetRt<W> D(int(a.nh));
    const int nh = D.nh;
    using T = TrainWs<W>;
    constexpr int kNW = 64;  // accumulator / wgrad N columns (W <= 64)
    const int wbytes = T::w_bytes(nh), stash_bytes = T::stash_bytes(nh);
    NRC_WTRC(0);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t r = tid & 127;  // row (row warps) / TMEM lane (flush warps)
    const uint32_t sW_a = smem_u32(smem);
    const uint32_t sH_a = sW_a + uint32_t(wbytes);
    const uint32_t sGb_a = sH_a + uint32_t(stash_bytes);        // gbuf[2]
    const uint32_t sG6_a = sGb_a + 2u * kTileBytes;              // dL/dy tile (columns 0..2 used)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + wbytes + stash_bytes + 3 * kTileBytes);
    uint64_t* wbar = &bars[0];
    uint64_t* wbar1 = &bars[1];
    uint64_t* mma_bar = &bars[2];   // forward layers
    uint64_t* bar_d = &bars[3];     // dgrad rounds
    uint64_t* bar_w = &bars[4];     // [nh + 1] wgrad_j
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
    float* red = reinterpret_cast<float*>(bars + 13);                 // 4 floats + 4 u32
    uint32_t* gmax = reinterpret_cast<uint32_t*>(bars + 17);          // per-warp max |dL/dy|
    uint32_t* deg_scratch = reinterpret_cast<uint32_t*>(bars + 19);
    float* inv_s_sh = reinterpret_cast<float*>(bars + 20);           // the tile's dL/dy scale, undone by the flush
    uint64_t* scale_bar = &bars[21];                                  // inv_s_sh written (thread 0 -> flush warps)

    if (tid == 0) {
        *deg_scratch = 0;
        mbar_init(wbar, 1);
        mbar_init(wbar1, 1);
        mbar_init(mma_bar, 1);
        mbar_init(bar_d, 1);
        for (int j = 0; j <= nh; ++j) mbar_init(&bar_w[j], 1);
        mbar_init(scale_bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    // zero the dL/dy tile (only chunk 0 of a line is rewritten per tile) and, at
    // W < 64, the hidden slots and g tiles (the upper half of each line is never written)
    {
        const uint32_t z0 = W < 64 ? sH_a + kTileBytes : sG6_a;
        for (uint32_t off = z0 + tid * 16; off < sG6_a + kTileBytes; off += T::kThreads * 16) st_shared_v4(off, 0, 0, 0, 0);
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_trigger();  // the optimiser kernel may launch (its griddepcontrol.wait covers this grid)
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t lane_off = warp_uniform(((warp & 3u) * 32u) << 16);  // (uniform register for tcgen05.ld)
    const uint32_t t_acc = tmem_base;
    const uint32_t t_accl = warp_uniform(t_acc + lane_off);  // this warp's lane quadrant of the accumulator
    auto t_g = [&](int j) -> uint32_t { return tmem_base + uint32_t(kNW) * (1u + uint32_t(j)); };
    auto slot = [&](int i) -> uint32_t { return sH_a + uint32_t(i) * kTileBytes; };
    auto gbuf = [&](int j) -> uint32_t { return sGb_a + uint32_t(j & 1) * kTileBytes; };
    auto gsrc = [&](int j) -> uint32_t { return j == nh ? sG6_a : gbuf(j + 1); };  // g_{j+1}
    auto wl = [&](int L) -> uint32_t { return sW_a + uint32_t(D.img_off(L)); };
    const uint32_t tile = blockIdx.x;  // grid = the batch's tiles

    auto issue_fwd = [&](int L) {
        const uint32_t idesc = warp_uniform(make_idesc(128, D.rows(L), 0, 0));
        const uint64_t a0 = warp_uniform(desc_kmajor(slot(L), 0));
        const uint64_t b0 = warp_uniform(desc_kmajor(wl(L), 0));
        const uint32_t d = warp_uniform(t_acc);
        tc_fence_after();
        if (elect_one()) {
            if (D.cols(L) == 32) {
                umma_f16(d, a0, b0, idesc, 0u);
                umma_f16(d, a0 + 2, b0 + 2, idesc, 1u);
            } else {
                umma_ss4<kKmajStep, kKmajStep>(d, a0, b0, idesc, 0u);
            }
            umma_commit(mma_bar);
        }
        __syncwarp();
    };
    // round j: dgrad_j (delta_j = g_{j+1} W_j, K = rows(j)) -> bar_d, then
    // wgrad_j (G_j = g_{j+1}^T h_j, K = 128 rows) -> bar_w[j]
    auto issue_bwd = [&](int j) {
        const uint32_t gs = gsrc(j);
        const uint32_t d_acc = warp_uniform(t_acc), d_g = warp_uniform(t_g(j));
        const uint32_t id_d = warp_uniform(make_idesc(128, kNW, 0, 1));
        const uint64_t da0 = warp_uniform(desc_kmajor(gs, 0));
        const uint64_t db = warp_uniform(desc_mn_lbo(wl(j), uint32_t(D.rows(j)) * 128u));
        const uint32_t id_w = warp_uniform(make_idesc(64, j == 0 ? 64 : kNW, 1, 1));
        const uint64_t wa = warp_uniform(desc_mn_lbo(gs, kTileBytes));
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
                }
                umma_commit(bar_d);
            }
            umma_ss8<kMNmajStep, kMNmajStep>(d_g, wa, wb, id_w, 0u);
            umma_commit(&bar_w[j]);
        }
        __syncwarp();
    };
    auto issuer_sync = [&]() {  // the rows' hand-off (their bar.arrive), then the MMAs may read
        named_bar_sync(3, 160);
        tc_fence_after();
    };

    if (warp == 8) {
        // ------------------------------------------------ MMA issuer warp
        issuer_sync();  // h0 encoded
        mbar_wait(wbar, 0);
        issue_fwd(0);
#pragma unroll 1
        for (int L = 1; L <= nh; ++L) {
            issuer_sync();  // h_L written
            if (L == 1) mbar_wait(wbar1, 0);
            issue_fwd(L);
        }
        issuer_sync();  // dL/dy written
#pragma unroll 1
        for (int j = nh; j >= 1; --j) {
            issue_bwd(j);
            issuer_sync();  // g_j written
        }
        issue_bwd(0);
    } else if (warp >= 4) {
        // ------------------------------------------------ flush warps
        // G_j (M = 64: out-neuron o = 16 q + lane in lanes 0..15 of quadrant q)
        // -> this CTA's partial (chunk-major, part_index), undoing the tile's
        // power-of-two dL/dy scale (exact in fp32); layers in the order their
        // wgrads finish.  The partial belongs to the previous kernel until it
        // has completed.
        pdl_wait();
        const uint32_t q = warp - 4u;
        float* part = a.partials + size_t(blockIdx.x) * D.padded();
        mbar_wait(scale_bar, 0);
        const float inv_s = *inv_s_sh;
        for (int j = nh; j >= 0; --j) {
            mbar_wait(&bar_w[j], 0);
            tc_fence_after();
#ifdef NRC_TRACE_FLUSH
            // diagnostics: global time at which wgrad_j completed (flush warp 4)
            if (a.dbg != nullptr && q == 0 && lane == 0 && blockIdx.x < 127)
                a.dbg[16384 + 32 * blockIdx.x + j] = global_ns();
#endif
            const int o = int(q) * 16 + int(lane);
            const bool valid = lane < 16 && o < D.rows(j);
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                if (32 * p >= D.cols(j)) break;
                uint32_t v[32];
                tmem_ld32(t_g(j) + lane_off + 32u * p, v);
                if (valid) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        float4* dst = reinterpret_cast<float4*>(part + part_index(D, j, o, 32 * p + 4 * c));
                        *dst = make_float4(__uint_as_float(v[4 * c]) * inv_s, __uint_as_float(v[4 * c + 1]) * inv_s,
                                           __uint_as_float(v[4 * c + 2]) * inv_s, __uint_as_float(v[4 * c + 3]) * inv_s);
                    }
                }
            }
        }
    } else {
        // ------------------------------------------------ row warps
        uint32_t phase = 0, d_phase = 0;
        auto copy = [&](uint32_t off, uint32_t bytes, uint64_t* bar) {
            mbar_arrive_expect_tx(bar, bytes);
            for (uint32_t o = 0; o < bytes; o += 8192u) {
                const uint32_t b = bytes - o < 8192u ? bytes - o : 8192u;
                bulk_g2s(smem + off + o, a.wimg + off + o, b, bar);
            }
        };
        auto mma_wait = [&]() {
            mbar_wait(mma_bar, phase);
            phase ^= 1;
            tc_fence_after();
        };
        // this thread's smem / TMEM work for the next MMA chain is done
        auto hand_off = [&]() {
            tc_fence_before();
            fence_async_smem();
            asm volatile("bar.arrive 3, 160;" ::: "memory");
        };
        // g_j = delta_j * 1[h_j > 0] -> gbuf[j & 1] (ReLU'(0) = 0, R17).  The
        // row's h_j chunks are loaded before the dgrad wait (mask_prefetch), so
        // no shared-memory round trip sits between the accumulator and the
        // hand-off; both accumulator halves are read before the first store.
        constexpr int kChunks = W / 8;  // 16-B chunks of a row
        auto mask_prefetch = [&](int j, uint4 (&hv)[kChunks]) {
    #pragma unroll
            for (int c = 0; c < kChunks; ++c) hv[c] = ld_shared_v4(slot(j) + swz(r, uint32_t(c)));
        };
        auto mask_epilogue = [&](int j, const uint4 (&hv)[kChunks]) {
            uint32_t v[W];
            tmem_ld32(t_accl, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
            if (W == 64) tmem_ld32(t_accl + 32u, *reinterpret_cast<uint32_t(*)[32]>(&v[W == 64 ? 32 : 0]));
            const float* f = reinterpret_cast<const float*>(v);
    #pragma unroll
            for (int c = 0; c < kChunks; ++c)
                st_shared_v4(gbuf(j) + swz(r, uint32_t(c)), pack_h2(f[8 * c], f[8 * c + 1]) & relu_mask(hv[c].x),
                             pack_h2(f[8 * c + 2], f[8 * c + 3]) & relu_mask(hv[c].y),
                             pack_h2(f[8 * c + 4], f[8 * c + 5]) & relu_mask(hv[c].z),
                             pack_h2(f[8 * c + 6], f[8 * c + 7]) & relu_mask(hv[c].w));
        };

        float loss_sum = 0.0f;
        uint32_t bad = 0, deg = 0;
        {
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
            NRC_WTRC(1);
            pdl_wait();  // the weights belong to the previous kernel until it completes
            NRC_WTRC(2);
            if (tid == 0) {
                copy(0u, uint32_t(D.img_off(1)), wbar);
                copy(uint32_t(D.img_off(1)), uint32_t(D.img() - D.img_off(1)), wbar1);
            }
            hand_off();
            // ---------------- forward: h_{L+1} = relu(W_L h_L), y = W_nh h_nh
    #pragma unroll 1
            for (int L = 0; L <= nh; ++L) {
                mma_wait();
                if (nh == 5) NRC_WTRC(8 + L);
                if (L == nh) break;
    #pragma unroll
                for (int p = 0; p < W / 32; ++p) {
                    uint32_t v[32];
                    tmem_ld32(t_accl + 32u * p, v);
    #pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float* f = reinterpret_cast<const float*>(v) + 8 * q;
                        st_shared_v4(slot(L + 1) + swz(r, uint32_t(p * 4 + q)), pack_h2_relu(f[0], f[1]),
                                     pack_h2_relu(f[2], f[3]), pack_h2_relu(f[4], f[5]), pack_h2_relu(f[6], f[7]));
                    }
                }
                hand_off();
            }
            // ---------------- relative L2 loss, Eq.(5) (R8-R10, R13, R25)
            {
                uint32_t v[4];
                tmem_ld4(t_accl, v);
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
                // per-tile power-of-two scale of dL/dy (R13, R25): the tile's largest
                // |dL/dy| maps into [2^7, 2^8); undone in fp32 by the flush warps
                const uint32_t mx = __reduce_max_sync(
                    0xffffffffu, max(max(__float_as_uint(fabsf(gy[0])), __float_as_uint(fabsf(gy[1]))),
                                     __float_as_uint(fabsf(gy[2]))));
                if (lane == 0) gmax[warp] = mx;
                named_bar_sync(2, 128);
                {
                    const uint32_t tm = max(max(gmax[0], gmax[1]), max(gmax[2], gmax[3]));
                    const int ex = int(tm >> 23);
                    const int ks = min(max(134 - ex, -120), 120);
                    if (tid == 0) {
                        *inv_s_sh = __uint_as_float(uint32_t(127 - ks) << 23);
                        mbar_arrive(scale_bar);
                    }
                    const float sc = __uint_as_float(uint32_t(127 + ks) << 23);
    #pragma unroll
                    for (int c = 0; c < 3; ++c) gy[c] *= sc;
                }
                st_shared_v4(sG6_a + swz(r, 0), pack_h2(gy[0], gy[1]), pack_h2(gy[2], 0.0f), 0u, 0u);
            }
            hand_off();
            NRC_WTRC(3);
            // ---------------- backward
    #pragma unroll 1
            for (int j = nh; j >= 1; --j) {
                if (nh == 5) NRC_WTRC(14 + 2 * (5 - j));
                uint4 hv[kChunks];
                mask_prefetch(j, hv);
                mbar_wait(bar_d, d_phase);
                d_phase ^= 1;
                tc_fence_after();
                if (nh == 5) NRC_WTRC(15 + 2 * (5 - j));
                mask_epilogue(j, hv);
                if (nh == 5 && j >= 2) NRC_WTRC(24 + (5 - j));
                hand_off();  // (wgrad_0 = g_1^T h_0 follows round 1 on the issuer: no gradient w.r.t. the encoding)
                if (nh == 5 && j >= 2) NRC_WTRC(28 + (5 - j));
            }
            NRC_WTRC(4);
            NRC_WTRC(5);
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
        {
            const uint32_t sdeg = __reduce_add_sync(0xffffffffu, deg);
            if (lane == 0 && sdeg != 0) atomicAdd(deg_scratch, sdeg);
        }
        named_bar_sync(1, 128);
        if (tid == 0) {
            a.loss_part[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
            const uint32_t* b = reinterpret_cast<const uint32_t*>(red + 4);
            const uint32_t nb = b[0] + b[1] + b[2] + b[3];
            if (nb) atomicAdd(a.bad_targets, (unsigned long long)nb);
            if (*deg_scratch != 0 && a.degenerate != nullptr) atomicAdd(a.degenerate, (unsigned long long)*deg_scratch);
        }
        NRC_WTRC(6);
    }
    // both roles meet here: the flush warps are done with the TMEM
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem_base, 512);
}

}  // namespace nrc
