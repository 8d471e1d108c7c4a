// nrc_query_ts.cuh -- fused cache query with the activations in TMEM
// (rows a1-a3 of SURVEY 8(a)).
//
// Why: with the A operand in shared memory, every 128-row layer moves
// 40 KB through the SM's shared-memory port (MMA reads A 16 KB + W 8 KB, the
// epilogue writes A 16 KB), ~250 KB per tile, which bounded a round-1 SMEM
// variant at ~2k cycles per tile.  Here the encoder and the
// ReLU epilogue write the fp16 activations straight into tensor memory
// (tcgen05.st) and the MMA reads A from TMEM (".kind::f16 [d], [a], b_desc"),
// so shared memory only feeds the 8 KB weight tile per layer.
//
// TMEM per in-flight tile: fp32 accumulator D (64 columns) + fp16 A
// (128 rows x 64 halves = 32 columns) -> 5 tiles per SM in 480 of 512
// columns.  Layer L reads A at column a and writes D; its epilogue reads D
// and writes the next A over the dead A (same columns).
#pragma once
#include "nrc_common.cuh"

namespace nrc {

// TMEM columns per in-flight tile at hidden width W: accumulator W + fp16 A
// (the 64-wide input for layer 0, W wide after) max(64, W) / 2.
template <int W>
__host__ __device__ constexpr int ts_slot_cols() {
    return W + (W > 64 ? W : 64) / 2;
}
template <int W>
__host__ __device__ constexpr int ts_max_slots() {
    return 512 / ts_slot_cols<W>();
}

template <int G, int W = 64>
__host__ __device__ int query_ts_smem_bytes_nh(int nh) {
    return 1024 + NetRt<W>(nh).img() + G * kRecTileBytes + 8 * (1 + 2 * G) + 16;
}

// One layer's K chain (K/16 MMAs, A in TMEM at a + 8 k, B K-major blocks of
// 64: b0 for k < 4, b1 for k >= 4), then a commit.  Elected lane only.
template <int NK>
__device__ __forceinline__ void umma_ta_chain_commit(uint32_t d, uint32_t a, uint64_t b0, uint64_t b1, uint32_t idesc,
                                                     uint64_t* bar) {
    static_assert(NK == 2 || NK == 4 || NK == 8, "K = 32, 64 or 128");
    if (NK == 4) {
        umma_chain4_ta_commit(d, a, b0, idesc, bar);
        return;
    }
    umma_f16_ta(d, a, b0, idesc, 0u);
    umma_f16_ta(d, a + 8, b0 + 2, idesc, 1u);
    if (NK == 8) {
        umma_f16_ta(d, a + 16, b0 + 4, idesc, 1u);
        umma_f16_ta(d, a + 24, b0 + 6, idesc, 1u);
        umma_f16_ta(d, a + 32, b1, idesc, 1u);
        umma_f16_ta(d, a + 40, b1 + 2, idesc, 1u);
        umma_f16_ta(d, a + 48, b1 + 4, idesc, 1u);
        umma_f16_ta(d, a + 56, b1 + 6, idesc, 1u);
    }
    umma_commit(bar);
}

// G independent 4-warp groups per CTA, one 128-row tile in flight per group,
// hidden width W, NH hidden layers fixed at compile time (0: args.nh at run
// time, the depth variants), EXACT: sin / Gaussian encoding primitives (N4).
// Per tile a group runs straight-line code: encode -> TMEM A; then per layer
// L the issuer lane's K chain + commit, the group waits, drains the fp32
// accumulator and writes relu(fp16) back as the next A, group barrier; the
// output layer's epilogue writes RGB.  The other groups' tiles fill the MMA
// round trips.
template <int G, int W = 64, int NH = 5, bool EXACT = false>
__global__ void __launch_bounds__(128 * G, 1) nrc_query_ts_kernel(QueryArgs args) {
    static_assert(G <= ts_max_slots<W>(), "TMEM holds 512 columns");
    const NetRt<W> D(NH > 0 ? NH : int(args.nh));  // layer shapes / offsets at this depth
    const int nh = D.nh, img = D.img();
    constexpr uint32_t kACols = (W > 64 ? W : 64) / 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    const uint32_t tid = threadIdx.x;
    const uint32_t g = tid >> 7, r = tid & 127, warp = tid >> 5, wq = warp & 3;
    // the group's MMA / TMA issuer: warp g % 4 of the group (an elected lane
    // issues), so the issuers of the groups sit on different SM sub-partitions
    const bool issuer_warp = wq == (g & 3u);
    const bool issuer = r == 32u * (g & 3u);
    uint8_t* sW = smem;
    const float* sRec = reinterpret_cast<const float*>(smem + img + g * kRecTileBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + img + G * kRecTileBytes);
    uint64_t* wbar = &bars[0];
    uint64_t* mma_bar = &bars[1 + 2 * g];
    uint64_t* rec_bar = &bars[2 + 2 * g];
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 1 + 2 * G);
    uint32_t* deg_scratch = tmem_slot + 1;
    uint32_t deg = 0;  // zero-length omega / n vectors this thread encoded

    if (tid == 0) {
        *deg_scratch = 0;
        for (int i = 0; i < 1 + 2 * G; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (tid == 0) {
        mbar_arrive_expect_tx(wbar, uint32_t(img));
        bulk_g2s(sW, args.wimg, uint32_t(img), wbar);
    }

    const uint64_t n = args.n;
    const uint64_t ntiles = (n + kTile - 1) / kTile;
    const uint64_t Q = uint64_t(gridDim.x) * G;  // this group's tiles: blockIdx.x G + g + k Q
    auto issue_records = [&](uint64_t t) {
        const uint64_t row0 = t * kTile;
        const uint64_t nv = (n - row0) < uint64_t(kTile) ? (n - row0) : uint64_t(kTile);
        const uint32_t bytes = uint32_t(nv) * kRecFloats * 4;
        mbar_arrive_expect_tx(rec_bar, bytes);
        bulk_g2s(const_cast<float*>(sRec), args.rec + row0 * kRecFloats, bytes, rec_bar);
    };
    uint64_t t = uint64_t(blockIdx.x) * G + g;
    if (issuer && t < ntiles) issue_records(t);
    mbar_wait(wbar, 0);

    const uint32_t sW_a = smem_u32(sW);
    const uint32_t lane_off = (wq * 32u) << 16;
    const uint32_t t_d = tmem_base + uint32_t(W) * g;               // fp32 accumulator
    const uint32_t t_a = tmem_base + uint32_t(W * G) + kACols * g;  // fp16 A operand
    // this warp's lane quadrant, warp-uniform (kept in uniform registers for tcgen05.ld / st)
    const uint32_t t_dl = warp_uniform(t_d + lane_off), t_al = warp_uniform(t_a + lane_off);
    // called by the whole issuer warp (converged)
    auto issue_layer = [&](int L) {
        // the weight tile's address made warp-uniform first: the descriptor
        // arithmetic then stays inside the issuer warp (not hoisted into all)
        const uint32_t wl = warp_uniform(sW_a + uint32_t(D.img_off(L)));
        const uint32_t idesc = make_idesc(128, D.rows(L), 0, 0);
        const uint32_t d = warp_uniform(t_d), a = warp_uniform(t_a);
        const uint64_t b0 = desc_kmajor(wl, 0);
        const uint64_t b1 = desc_kmajor(wl + uint32_t(D.rows(L)) * 128u, 0);
        tc_fence_after();
        if (elect_one()) {
            if (D.cols(L) == 32)
                umma_ta_chain_commit<2>(d, a, b0, b1, idesc, mma_bar);
            else if (D.cols(L) == 64)
                umma_ta_chain_commit<4>(d, a, b0, b1, idesc, mma_bar);
            else
                umma_ta_chain_commit<8>(d, a, b0, b1, idesc, mma_bar);
        }
        __syncwarp();
    };
    uint32_t rec_phase = 0, phase = 0;
    auto mma_wait = [&]() {
        mbar_wait(mma_bar, phase);
        phase ^= 1u;
        tc_fence_after();
    };
    // h_{L+1} = relu(acc) -> fp16, written over h_L in the group's TMEM A
    auto hidden_epilogue = [&]() {
#pragma unroll
        for (int part = 0; part < W / 32; ++part) {
            uint32_t v[32];
            tmem_ld32(t_dl + 32 * part, v);
            uint32_t hp[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) hp[q] = pack_h2_relu(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1]));
            tmem_st16_nowait(t_al + 16 * part, hp);
        }
        tmem_wait_st();
        tc_fence_before();
        named_bar_sync(1 + g, 128);
    };

#pragma unroll 1
    for (; t < ntiles; t += Q) {
        mbar_wait(rec_bar, rec_phase);
        rec_phase ^= 1u;
        const uint64_t row = t * kTile + r;
        const bool valid = row < n;
        float rec[16];
        {
            const float4* src = reinterpret_cast<const float4*>(sRec + r * kRecFloats);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float4 v = valid ? src[c] : make_float4(0.f, 0.f, 0.f, 0.f);
                rec[4 * c + 0] = v.x;
                rec[4 * c + 1] = v.y;
                rec[4 * c + 2] = v.z;
                rec[4 * c + 3] = v.w;
            }
        }
        float fac[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) fac[c] = (args.flags & 1u) ? rec[10 + c] + rec[13 + c] : 1.0f;
        {
            uint32_t h[32];
            const uint32_t dg = encode_record<EXACT>(rec, args.ep, h);
            deg += valid ? dg : 0u;
            tmem_st32(t_al, h);  // includes tcgen05.wait::st
        }
        fence_async_smem();  // record reads before the next TMA overwrite
        tc_fence_before();
        named_bar_sync(1 + g, 128);  // A written; records consumed; the previous tile's TMEM reads done
        if (issuer_warp) {
            if (issuer && t + Q < ntiles) issue_records(t + Q);
            __syncwarp();
            issue_layer(0);
        }
        if constexpr (NH > 0) {
#pragma unroll
            for (int L = 0; L < NH; ++L) {
                mma_wait();
                hidden_epilogue();
                if (issuer_warp) issue_layer(L + 1);
            }
        } else {
#pragma unroll 1
            for (int L = 0; L < nh; ++L) {
                mma_wait();
                hidden_epilogue();
                if (issuer_warp) issue_layer(L + 1);
            }
        }
        // output: q = max(0, y * (alpha + beta))
        mma_wait();
        uint32_t v[4];
        tmem_ld4(t_dl, v);
        tc_fence_before();
        if (valid) {
            float qv[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                qv[c] = __uint_as_float(v[c]) * fac[c];
                if (args.flags & 2u) qv[c] = fmaxf(qv[c], 0.0f);
            }
            if (args.image == nullptr) {
                float* o = args.out + row * 3;
#pragma unroll
                for (int c = 0; c < 3; ++c) o[c] = qv[c];
            } else {  // pixel += throughput * radiance
                float* px = args.image + size_t(__ldg(args.pix + row)) * 3;
                const float* th = args.thr + row * 3;
#pragma unroll
                for (int c = 0; c < 3; ++c) atomicAdd(px + c, __ldg(th + c) * qv[c]);
            }
        }
    }
    tc_fence_before();
    block_count_add(args.degenerate, deg, deg_scratch);  // includes __syncthreads
    if (warp == 0) tmem_dealloc(tmem_base, 512);
}

}  // namespace nrc
