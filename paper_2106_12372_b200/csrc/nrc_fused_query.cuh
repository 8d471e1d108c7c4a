// nrc_fused_query.cuh -- the fused cache-query kernel (rows a1-a3 of SURVEY 8(a)):
// encode (Table 1) -> 6 tcgen05 layers
// -> reflectance factorisation and clamp, EMA weights.
//
// Design notes: a layer's MMA round trip (issue -> commit ->
// mbarrier -> TMEM drain) is ~650 cycles against ~175 cycles of tensor work
// (scripts/ubench_tcgen05.cu), so each SM keeps 8 tiles in flight (TMEM holds
// 8 fp32 accumulators of 64 columns).  Warp-specialised variants (dedicated
// encoder / epilogue / MMA-issuer warps with mbarrier or atomic hand-offs)
// were measured slower than this "every warp does everything" layout on the
// 1080p query (151.6 us vs 184-456 us): the hot path is latency-bound, and
// 16 interchangeable warps per SM hide more latency than role-split ones.
#pragma once
#include "nrc_device.cuh"

namespace nrc {

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

struct QueryArgs {
    const float* rec;    // n records x 16 fp32
    float* out;          // n x 3 fp32
    uint64_t n;
    const uint8_t* wimg; // fp16 operand image (43,008 B), EMA or raw
    EncodeParams ep;
    uint32_t flags;      // NRC_FACTORIZE | NRC_CLAMP_QUERY
    long long* dbg;      // per-round clock64 trace (builds with -DNRC_TRACE_QUERY only), else unused
    // fused pixel reconstruction (nrc_query_accumulate, TMEM kernel only): if
    // image != nullptr, image[3 pix[i] + c] += thr[3 i + c] * q_c instead of out
    const uint32_t* pix;
    const float* thr;
    float* image;
    uint32_t nh;         // hidden layers (5; depth variants in the TMEM kernel only)
};

constexpr int kRecTileBytes = kTile * kRecFloats * 4;  // 8 KB of records per tile

template <int G, int S>
__host__ __device__ constexpr int query_smem_bytes() {
    return 1024 + kImgBytes + G * S * kTileBytes + G * kRecTileBytes + 8 * (1 + (S + 1) * G) +
           16;
}
template <int G, int S>
__host__ __device__ constexpr uint32_t query_tmem_cols() {
    return (G * S * 64 <= 128) ? 128 : (G * S * 64 <= 256) ? 256 : 512;
}

// Persistent: one CTA per SM, G independent 4-warp groups sharing one SMEM
// copy of the weight image.  A group keeps S 128-row tiles in
// flight (each with its own SMEM activation tile and TMEM accumulator) and
// round-robins over them: while the tensor pipe runs slot s's layer, the
// group's threads drain slot s^1's accumulator (ReLU + fp16) or encode its
// next tile.  Thread r of a group owns row r (TMEM lane r); thread 0 of the
// group issues the tcgen05.mma chain and the TMA bulk copies of the records.
template <int G, int S>
__global__ void __launch_bounds__(128 * G, 1) nrc_query_kernel(QueryArgs args) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    const uint32_t tid = threadIdx.x;
    const uint32_t g = tid >> 7, r = tid & 127, warp = tid >> 5, wq = warp & 3;
    uint8_t* sW = smem;
    uint8_t* sH0 = smem + kImgBytes + g * S * kTileBytes;
    const float* sRec = reinterpret_cast<const float*>(smem + kImgBytes + G * S * kTileBytes + g * kRecTileBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kImgBytes + G * S * kTileBytes + G * kRecTileBytes);
    uint64_t* wbar = &bars[0];
    uint64_t* mma_bar = &bars[1 + (S + 1) * g];  // [S]
    uint64_t* rec_bar = &bars[1 + (S + 1) * g + S];
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 1 + (S + 1) * G);

    if (tid == 0) {
        for (int i = 0; i < 1 + (S + 1) * G; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, query_tmem_cols<G, S>());
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (tid == 0) {
        mbar_arrive_expect_tx(wbar, kImgBytes);
        bulk_g2s(sW, args.wimg, kImgBytes, wbar);
    }

    const uint64_t n = args.n;
    const uint64_t ntiles = (n + kTile - 1) / kTile;
    const uint64_t q0 = uint64_t(blockIdx.x) * G + g;   // this group's k-th tile is q0 + k * Q
    const uint64_t Q = uint64_t(gridDim.x) * G;
    uint64_t k_next = 0;
    uint32_t rec_phase = 0;

    auto issue_records = [&](uint64_t t) {
        const uint64_t row0 = t * kTile;
        const uint64_t nv = (n - row0) < uint64_t(kTile) ? (n - row0) : uint64_t(kTile);
        const uint32_t bytes = uint32_t(nv) * kRecFloats * 4;
        mbar_arrive_expect_tx(rec_bar, bytes);
        bulk_g2s(const_cast<float*>(sRec), args.rec + row0 * kRecFloats, bytes, rec_bar);
    };
    if (r == 0 && q0 < ntiles) issue_records(q0);
    mbar_wait(wbar, 0);

    const uint32_t sW_a = smem_u32(sW), sH_a = smem_u32(sH0);
    auto issue_layer = [&](int s, int L) {
        const uint32_t wl = sW_a + layer_off(L) * 2;
        const uint32_t idesc = (L < 5) ? make_idesc(128, 64, 0, 0) : make_idesc(128, 16, 0, 0);
        const uint32_t a = sH_a + s * kTileBytes;
        const uint32_t d = tmem_base + (g * S + s) * 64;
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_f16(d, desc_kmajor(a, k), desc_kmajor(wl, k), idesc, k > 0);
        umma_commit(&mma_bar[s]);
    };

    // per-slot state (uniform across the group; registers after full unroll)
    uint64_t row[S];
    float fac[S][3];
    int layer[S];
    bool active[S];
    uint32_t phase[S];

    // encode the group's next tile into slot s and start its layer chain
    auto start_tile = [&](int s) -> bool {
        const uint64_t t = q0 + k_next * Q;
        if (t >= ntiles) return false;
        mbar_wait(rec_bar, rec_phase);
        rec_phase ^= 1;
        row[s] = t * kTile + r;
        const bool valid = row[s] < n;
        float rec[16];
        const float4* src = reinterpret_cast<const float4*>(sRec + r * kRecFloats);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float4 v = valid ? src[c] : make_float4(0.f, 0.f, 0.f, 0.f);
            rec[4 * c + 0] = v.x;
            rec[4 * c + 1] = v.y;
            rec[4 * c + 2] = v.z;
            rec[4 * c + 3] = v.w;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) fac[s][c] = (args.flags & 1u) ? rec[10 + c] + rec[13 + c] : 1.0f;
        {
            uint32_t h[32];
            encode_record(rec, args.ep, h);
            store_row_swz(sH_a + s * kTileBytes, r, h);
        }
        fence_async_smem();
        named_bar_sync(1 + g, 128);  // tile written; records consumed; previous TMEM reads of slot s done
        ++k_next;
        if (r == 0) {
            const uint64_t tn = q0 + k_next * Q;
            if (tn < ntiles) issue_records(tn);
            issue_layer(s, 0);
        }
        return true;
    };

#pragma unroll
    for (int s = 0; s < S; ++s) {
        phase[s] = 0;
        layer[s] = 0;
        active[s] = start_tile(s);
    }
    bool any = active[0];
#pragma unroll
    for (int s = 1; s < S; ++s) any = any || active[s];

#pragma unroll 1
    while (any) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (!active[s]) continue;
            mbar_wait(&mma_bar[s], phase[s]);
            phase[s] ^= 1;
            tc_fence_after();
            const uint32_t t_row = tmem_base + (g * S + s) * 64 + ((wq * 32u) << 16);
            if (layer[s] < 5) {
                // h_{L+1} = relu(acc) -> fp16, written over h_L in the slot's A tile
                const uint32_t a = sH_a + s * kTileBytes;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    uint32_t v[32];
                    tmem_ld32(t_row + 32 * half, v);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float* f = reinterpret_cast<const float*>(v) + 8 * c;
                        st_shared_v4(a + swz(r, 4 * half + c), pack_h2_relu(f[0], f[1]), pack_h2_relu(f[2], f[3]),
                                     pack_h2_relu(f[4], f[5]), pack_h2_relu(f[6], f[7]));
                    }
                }
                tc_fence_before();
                fence_async_smem();
                named_bar_sync(1 + g, 128);
                ++layer[s];
                if (r == 0) issue_layer(s, layer[s]);
            } else {
                // output: q = max(0, y * (alpha + beta))
                uint32_t v[4];
                tmem_ld4(t_row, v);
                tc_fence_before();
                if (row[s] < n) {
                    float* o = args.out + row[s] * 3;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        float qv = __uint_as_float(v[c]) * fac[s][c];
                        if (args.flags & 2u) qv = fmaxf(qv, 0.0f);
                        o[c] = qv;
                    }
                }
                layer[s] = 0;
                active[s] = start_tile(s);
            }
        }
        any = active[0];
#pragma unroll
        for (int s = 1; s < S; ++s) any = any || active[s];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, query_tmem_cols<G, S>());
}

}  // namespace nrc
