// nrc_train.cuh -- the fused training kernel (rows a0, a1, a4-a8 of SURVEY 8(a)):
// LCG-gathered records -> encode -> forward with the activation
// stash kept in SMEM -> relative-L2 loss gradient (Eq. 5) ->
// dgrad and wgrad on tcgen05 -> per-CTA fp32 weight-gradient partials ->
// (fused mode) deterministic reduction + Adam + EMA on row slices, all s
// optimisation steps of a frame in one persistent launch.
// The paper wrote activations to global memory and ran the weight-gradient
// GEMMs as separate CUTLASS split-k launches; here everything for
// a 128-row tile stays on chip and the wgrad MMAs run behind the dgrad chain.
#pragma once
#include "nrc_fused_query.cuh"

namespace nrc {

constexpr int kMaxFusedSteps = 8;
constexpr int kMaxParts = 8;  // ranks of one box
struct StepCoef {
    float inv_bc1, inv_bc2;  // Adam bias corrections 1/(1-b^t)
    float ema_c1, ema_c2;    // W-bar = c1 W + c2 W-bar (Eq. 2 / R12)
};

struct TrainArgs {
    const float* rec;      // records (indexed through the gather below)
    // peer mode (nrc_train_frame_parts): record i lives in part i / part_n at
    // row i % part_n of rec_parts / tgt_parts (peer pointers), if n_parts > 0
    const float* rec_parts[kMaxParts];
    const float* tgt_parts[kMaxParts];
    uint32_t n_parts, part_n;
    const float* tgt;      // targets, 3 fp32 per record
    uint32_t n;            // rows per step
    uint32_t gather;       // 1: row k of step j reads record lcg_perm(offset + j n + k); 0: record j n + k
    uint64_t lcg_a, lcg_c, lcg_m, lcg_n, offset;
    const uint8_t* wimg;   // fp16 image of the TRAINING weights W_t
    EncodeParams ep;
    uint32_t flags;
    float loss_eps;
    float* partials;       // [gridDim.x][kParamPadded] fp32 un-normalised gradient sums (partial_index layout)
    float* loss_part;      // [gridDim.x] loss sums
    unsigned long long* bad_targets;
    long long* dbg;        // optional phase timestamps of CTA 0 (diagnostics), else nullptr
    // ---- fused mode (cooperative launch): Adam + EMA between steps
    uint32_t fused;        // 0: one step, partials only (multi-GPU / backward path)
    uint32_t nsteps;       // steps in this launch (<= kMaxFusedSteps)
    float inv_n, lr, b1, b2, adam_eps;
    StepCoef coef[kMaxFusedSteps];
    float *w, *m, *v, *ema;   // fp32 padded state
    uint8_t *wimg_out, *eimg; // fp16 operand images rewritten by the optimiser
    unsigned long long* bad_grads;
    float* losses;            // nsteps batch-mean losses (optional)
    unsigned long long* gbar; // grid-barrier counter (monotonic across launches)
    unsigned long long gbar_base;
    unsigned long long* gbarA;  // arrivals of CTAs whose W3..W5 partials are written (phase A)
    unsigned long long gbarA_base;
    uint32_t nh;              // hidden layers (nrc_train_w_kernel; the fused kernel is built for 5)
};

// SMEM: weight image | h0..h5 stash (6 tiles) | 3 rotating gradient tiles |
// dL/dy tile | barriers.  The stash is immutable during the backward pass, so
// wgrad_i (which reads h_i and g_{i+1}) can still be in flight while the
// epilogue of a later round writes another gradient buffer.  In fused mode
// the stash + gradient tiles (144 KB) double as the optimiser's staging area.
constexpr int kPhaseAScratch = 4096;  // helper-warp group sums (phase A)
constexpr int kTrainSmemBytes = 1024 + kImgBytes + 10 * kTileBytes + 64 + 64 + kPhaseAScratch;
constexpr int kHelpThreads = 224;      // warps 5..11
constexpr int kChunkSplit = 3 * 4096 / 4;  // chunks of W0..W2 (phase B) | W3..W5 (phase A)
constexpr uint32_t kTrainTmemCols = 512;  // acc 64 + 6 wgrad accumulators x 64
constexpr int kTrainThreads = 160;        // tile threads: 4 row warps + 1 wgrad-issue warp
constexpr int kTrainBlock = 384;          // + 7 warps that only join the fused optimiser
constexpr int kParamChunks = kParamPadded / 4;  // 5376 16-byte chunks of a partial

// Position of padded parameter (layer, row o, column k) inside a CTA's
// gradient partial: rows of 64 fp32, 16-byte chunks XOR-swizzled by o % 16.
__host__ __device__ __forceinline__ int partial_index(int layer, int o, int k) {
    return layer_off(layer) + o * 64 + ((((k >> 2) ^ (o & 15))) << 2) + (k & 3);
}
// inverse of partial_index(): padded parameter index stored at partial position pp
__device__ __forceinline__ int partial_to_param(int pp) {
    const int row = pp >> 6;  // padded rows of 64: layer_off(l) = 64 * (first row of l)
    const int o = row < 320 ? (row & 63) : row - 320;
    return row * 64 + (((((pp >> 2) & 15) ^ (o & 15))) << 2) + (pp & 3);
}
__device__ __forceinline__ float ld_global_f32(const float* p) {  // not sunk past the partial loads
    float v;
    asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void padded_coords(int j, int& layer, int& row, int& col) {
    layer = j < 20480 ? (j >> 12) : 5;
    const int rel = j - layer_off(layer);
    row = rel >> 6;
    col = rel & 63;
}
// byte offset of parameter (layer, row, col) in an fp16 operand image
__device__ __forceinline__ uint32_t image_offset(int layer, int row, int col) {
    return uint32_t(layer_off(layer)) * 2u + uint32_t(row) * 128u + ((uint32_t(col >> 3) ^ uint32_t(row & 7)) << 4) +
           uint32_t(col & 7) * 2u;
}
// Adam (R11) + EMA (Eq. 2; R12) of padded parameter j with the
// batch-mean gradient g; writes fp32 state and both fp16 operand images.
struct OptParams {
    float lr, b1, b2, eps, inv_bc1, inv_bc2, ema_c1, ema_c2;
};
__device__ __forceinline__ void adam_ema_apply(int j, float g, const OptParams& o, float m, float v, float w, float e,
                                               float* __restrict__ w_, float* __restrict__ m_, float* __restrict__ v_,
                                               float* __restrict__ e_, uint8_t* wimg, uint8_t* eimg,
                                               unsigned long long* bad_grads) {
    if (!isfinite(g)) {  // non-finite gradient entries are zeroed and counted
        g = 0.0f;
        atomicAdd(bad_grads, 1ull);
    }
    m = o.b1 * m + (1.0f - o.b1) * g;
    v = o.b2 * v + (1.0f - o.b2) * g * g;
    w = w - o.lr * (m * o.inv_bc1) / (sqrtf(v * o.inv_bc2) + o.eps);
    e = o.ema_c1 * w + o.ema_c2 * e;
    m_[j] = m;
    v_[j] = v;
    w_[j] = w;
    e_[j] = e;
    int layer, row, col;
    padded_coords(j, layer, row, col);
    const uint32_t off = image_offset(layer, row, col);
    *reinterpret_cast<__half*>(wimg + off) = __float2half_rn(w);
    *reinterpret_cast<__half*>(eimg + off) = __float2half_rn(e);
}
__device__ __forceinline__ void adam_ema_update(int j, float g, const OptParams& o, float* __restrict__ w_,
                                                float* __restrict__ m_, float* __restrict__ v_,
                                                float* __restrict__ e_, uint8_t* wimg, uint8_t* eimg,
                                                unsigned long long* bad_grads) {
    adam_ema_apply(j, g, o, m_[j], v_[j], w_[j], e_[j], w_, m_, v_, e_, wimg, eimg, bad_grads);
}

// 0xFFFF in each 16-bit half whose fp16 activation is > 0 (ReLU'(0) = 0, R17)
__device__ __forceinline__ uint32_t relu_mask(uint32_t h2bits) {
    __half2 h;
    memcpy(&h, &h2bits, 4);
    return __hgt2_mask(h, __float2half2_rn(0.0f));
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// Grid-wide barrier of a cooperative launch: monotonic counter, release /
// acquire at GPU scope; `target` = value once every CTA has arrived.
__device__ __forceinline__ void grid_sync(unsigned long long* ctr, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // bulk (async-proxy) stores before the release
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned long long v = 0;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

__device__ __forceinline__ long long global_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// per-CTA global-timer marks of step 1 at dbg[256 + 8 cta + k] (diagnostics)
#define NRC_GTRC(k)                                                                           \
    do {                                                                                      \
        if (a.dbg != nullptr && step == 1 && threadIdx.x == 0) a.dbg[256 + 8 * blockIdx.x + (k)] = global_ns(); \
    } while (0)
// Called by a whole converged warp: one elected lane issues a chain of 4 (or
// 8) MMAs and, if bar != nullptr, commits them to bar (see elect_one()).
template <int AS, int BS, int NCHAIN>
__device__ __forceinline__ void warp_issue(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc0,
                                           uint64_t* bar) {
    d = warp_uniform(d);
    a = warp_uniform(a);
    b = warp_uniform(b);
    acc0 = warp_uniform(acc0);
    tc_fence_after();
    if (elect_one()) {
        if (NCHAIN == 8)
            umma_ss8<AS, BS>(d, a, b, idesc, acc0);
        else if (NCHAIN == 4)
            umma_ss4<AS, BS>(d, a, b, idesc, acc0);
        else
            umma_f16(d, a, b, idesc, acc0);
        if (bar != nullptr) umma_commit(bar);
    }
    __syncwarp();
}

// Spin until *ctr >= target: relaxed polls with a short back-off (acquire
// polls hammer L2 and the SM's memory pipe while other warps compute), then
// one acquire fence.
__device__ __forceinline__ void wait_counter(unsigned long long* ctr, unsigned long long target) {
    unsigned long long v = 0;
    while (true) {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        if (v >= target) break;
        __nanosleep(64);
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

#define NRC_TRC(i)                                                                          \
    do {                                                                                    \
        if (a.dbg != nullptr && blockIdx.x == 0 && threadIdx.x == 0) a.dbg[trc + (i)] = clock64(); \
    } while (0)

// One CTA per 128-row tile (persistent over tiles if n > 128 * grid).  Warps
// 0-3 own the rows (thread r = row r = TMEM lane r): gather, encode, the
// forward / loss / mask epilogues, and the forward + dgrad MMA issue (thread
// 0).  Warp 4 issues the weight-gradient MMAs on its own commit barrier, so
// the issuing thread's stall on those 48 small MMAs never delays an epilogue.
// Partial-only mode is launched with programmatic dependent launch:
// everything before griddepcontrol.wait (barriers, TMEM, record gather,
// encode of the first tile) overlaps the previous kernel.  Fused mode is a
// cooperative launch that runs all steps with two grid barriers per step:
// partials -> [barrier] -> each CTA reduces its slice of parameter rows over
// all partials in fixed CTA order and applies Adam + EMA -> [barrier] ->
// reload the new weight image.
template <bool EXACT>
__global__ void __launch_bounds__(kTrainBlock, 1) nrc_train_kernel(TrainArgs a) {
    uint32_t trc = 0;  // trace slot base: 32 per step
    NRC_TRC(0);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    const uint32_t tid = threadIdx.x, r = tid, warp = tid >> 5, lane = tid & 31;
    constexpr uint32_t kBarRows = 1, kBarDgrad = 2, kBarG1 = 3, kBarHelp = 4, kBarTile = 5;  // named barriers
    uint8_t* sW = smem;
    const uint32_t sW_a = smem_u32(sW);
    const uint32_t sH_a = sW_a + kImgBytes;              // h0..h5
    const uint32_t sGb_a = sH_a + 6 * kTileBytes;        // g buffers (g_i in buffer i % 3)
    const uint32_t sG6_a = sGb_a + 3 * kTileBytes;       // dL/dy (cols 0..2 used)
    float* sOpt = reinterpret_cast<float*>(smem + kImgBytes);  // fused-mode group sums (stash area)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kImgBytes + 10 * kTileBytes);
    uint64_t* wbar = &bars[0];     // weight image loads
    uint64_t* mma_bar = &bars[1];  // forward / dgrad commits (thread 0)
    uint64_t* wg_bar = &bars[2];   // wgrad commits (warp 4)
    uint64_t* staged_bar = &bars[3];  // rows -> warp 5: a W3..W5 partial is staged in SMEM
    float* sHelp = reinterpret_cast<float*>(smem + kImgBytes + 10 * kTileBytes + 128);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
    float* red = reinterpret_cast<float*>(bars + 5);    // 4 floats + 4 u32

    if (tid == 0) {
        mbar_init(wbar, 1);
        mbar_init(mma_bar, 1);
        mbar_init(wg_bar, 1);
        mbar_init(staged_bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(tmem_slot, kTrainTmemCols);
        tmem_relinquish();
    }
    // zero the dL/dy tile once: only chunk 0 of each line is rewritten per tile
    for (uint32_t off = tid * 16; off < kTileBytes; off += kTrainBlock * 16) st_shared_v4(sG6_a + off, 0, 0, 0, 0);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    NRC_TRC(1);
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t lane_off = ((warp & 3) * 32u) << 16;
    const uint32_t t_acc = tmem_base;  // 64 columns: forward / dgrad accumulator
    auto t_wg = [&](int i) -> uint32_t { return tmem_base + 64u + 64u * i; };
    auto hs = [&](int i) -> uint32_t { return sH_a + i * kTileBytes; };
    auto gb = [&](int i) -> uint32_t { return sGb_a + (i % 3) * kTileBytes; };
    const uint32_t idesc_fwd = make_idesc(128, 64, 0, 0);
    const uint32_t idesc_out = make_idesc(128, 16, 0, 0);
    const uint32_t idesc_dgrad = make_idesc(128, 64, 0, 1);
    const uint32_t idesc_wgrad = make_idesc(64, 64, 1, 1);

    uint32_t phase = 0, wg_phase = 0, w_phase = 0, st_phase = 0;
    float loss_sum = 0.0f;
    uint32_t bad = 0;
    bool first = true;
    bool weights_ready = false;
    const uint32_t ntiles = (a.n + kTile - 1) / kTile;
    float* part = a.partials + size_t(blockIdx.x) * kParamPadded;

    auto load_weights = [&]() {
        if (tid == 0) {
            asm volatile("fence.proxy.async;" ::: "memory");  // generic writes of the image -> TMA read
            mbar_arrive_expect_tx(wbar, kImgBytes);
#pragma unroll
            for (int q = 0; q < 6; ++q)  // several copies in flight
                bulk_g2s(sW + q * (kImgBytes / 6), a.wimg + q * (kImgBytes / 6), kImgBytes / 6, wbar);
        }
        if (warp < 4) {  // only the row warps read the image through their MMAs' descriptors
            mbar_wait(wbar, w_phase);
            w_phase ^= 1;
        }
    };
    auto mma_wait = [&]() {
        mbar_wait(mma_bar, phase);
        phase ^= 1;
        tc_fence_after();
    };
    auto wg_wait = [&]() {
        mbar_wait(wg_bar, wg_phase);
        wg_phase ^= 1;
        tc_fence_after();
    };
    auto sync_rows = [&]() {  // warps 0-3: make SMEM / TMEM work visible to the next MMA
        tc_fence_before();
        fence_async_smem();
        named_bar_sync(kBarRows, 128);
    };
    // wgrad of layer i (M=64 over outputs o, N=64 over inputs k, K=128 rows):
    // G_i += g_{i+1}^T h_i, both operands MN-major views of the stored tiles
    // (whole warp 4; commit to wg_bar if commit)
    auto issue_wgrad = [&](int i, uint32_t g_next, bool commit) {
        warp_issue<kMNmajStep, kMNmajStep, 8>(t_wg(i), desc_mnmajor(g_next, 0), desc_mnmajor(hs(i), 0), idesc_wgrad,
                                              first ? 0u : 1u, commit ? wg_bar : nullptr);
    };
    // Stage layer i's fp32 gradient (64 x 64, or 16 x 64 for W5) from TMEM into
    // the dead stash slot i (h_i's last readers -- its mask epilogue and
    // wgrad_i -- have completed) in the partials layout (partial_index(): row
    // o's 16-B chunk c at chunk c ^ (o % 16), so the 16 rows a warp stages in
    // one step hit distinct banks).  M=64 TMEM layout: row o lives in lane
    // (o % 16) + 32 (o / 16), so warp w holds o = 16 w + lane for lane < 16.
    // The TMA engine then writes the block to global.
    auto stage_partial = [&](int i) {
        const int rows = (i < 5) ? 64 : kOutPad;
        const int o = int(warp) * 16 + int(lane);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            uint32_t v[32];
            tmem_ld32(t_wg(i) + lane_off + 32 * half, v);
            if (lane < 16 && o < rows) {
                const uint32_t row_base = hs(i) + uint32_t(o) * 256u;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t c = uint32_t(8 * half + q) ^ uint32_t(o & 15);
                    st_shared_v4(row_base + 16u * c, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                }
            }
        }
    };
    // after a barrier that follows stage_partial(i) + fence.proxy.async
    auto store_partial = [&](int i) {
        if (tid == 0) {
            bulk_s2g(part + layer_off(i), hs(i), uint32_t((i < 5 ? 64 : kOutPad) * 64 * 4));
            bulk_commit();
        }
    };
    // g_i = delta_i * 1[h_i > 0] -> gradient buffer i % 3 (ReLU'(0) = 0, R17)
    auto mask_epilogue = [&](int i) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            uint32_t v[32];
            tmem_ld32(t_acc + lane_off + 32 * half, v);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t off = swz(r, 4 * half + c);
                const uint4 hv = ld_shared_v4(hs(i) + off);
                const float* f = reinterpret_cast<const float*>(v) + 8 * c;
                st_shared_v4(gb(i) + off, pack_h2(f[0], f[1]) & relu_mask(hv.x), pack_h2(f[2], f[3]) & relu_mask(hv.y),
                             pack_h2(f[4], f[5]) & relu_mask(hv.z), pack_h2(f[6], f[7]) & relu_mask(hv.w));
            }
        }
    };

    // record + target of batch row `row` of step `step` (zeros past the batch)
    auto gather_row = [&](uint32_t step_, uint32_t row, float (&rec)[16], float (&tg)[3]) {
        if (row < a.n) {
            const uint64_t k = uint64_t(step_) * a.n + row;
            const uint64_t idx = a.gather ? lcg_perm(a.offset + k, a.lcg_n, a.lcg_a, a.lcg_c, a.lcg_m) : k;
            const float* rsrc = a.rec + idx * kRecFloats;
            const float* tsrc = a.tgt + idx * 3;
            if (a.n_parts > 0) {  // the owner's buffer (a peer GPU's memory over NVLink)
                const uint32_t p = uint32_t(idx / a.part_n);
                const uint64_t o = idx - uint64_t(p) * a.part_n;
                rsrc = a.rec_parts[p] + o * kRecFloats;
                tsrc = a.tgt_parts[p] + o * 3;
            }
            load_record_global(rsrc, rec);
#pragma unroll
            for (int c = 0; c < 3; ++c) tg[c] = __ldg(tsrc + c);
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) rec[i] = 0.0f;
#pragma unroll
            for (int c = 0; c < 3; ++c) tg[c] = 0.0f;
        }
    };
    // fused mode: the rows gather and encode the next step's first tile while
    // the grid waits at barrier 2 (the records do not depend on the weights)
    bool have_next = false;
    float rec_n[16], tg_n[3];

#pragma unroll 1
    for (uint32_t step = 0; step < a.nsteps; ++step) {
        first = true;
        trc = 32u * step;
        NRC_GTRC(6);
#pragma unroll 1
        for (uint32_t tile = blockIdx.x; warp < 6 && tile < ntiles; tile += gridDim.x) {
            const bool last = tile + gridDim.x >= ntiles;
            if (warp == 5) {
                // ---------------- partial-store warp: TMA-store G5, G4, G3 as the rows
                // stage them, then (fused mode) announce that they are globally written
                if (last) {
#pragma unroll 1
                    for (int i = 3; i >= 1; --i) {
                        mbar_wait(staged_bar, st_phase);
                        st_phase ^= 1;
                        if (lane == 0) {
                            bulk_s2g(part + layer_off(i + 2), hs(i + 2), uint32_t((i + 2 < 5 ? 64 : kOutPad) * 64 * 4));
                            bulk_commit();
                        }
                        __syncwarp();
                    }
                    if (lane == 0) {
                        bulk_wait_all();
                        if (a.fused) {
                            asm volatile("fence.proxy.async.global;" ::: "memory");
                            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.gbarA) : "memory");
                        }
                    }
                    __syncwarp();
                }
                continue;
            }
            if (warp == 4) {
                // ---------------- wgrad issue warp: G_{i+1} right after dgrad_i is queued
#pragma unroll 1
                for (int i = 4; i >= 1; --i) {
                    named_bar_sync(kBarDgrad, 64);
                    issue_wgrad(i + 1, i == 4 ? sG6_a : gb(i + 2), true);  // G_{i+1} += g_{i+2}^T h_{i+1}
                }
                named_bar_sync(kBarG1, kTrainThreads);  // g_1 written
                issue_wgrad(1, gb(2), false);  // G_1 += g_2^T h_1
                issue_wgrad(0, gb(1), true);   // G_0 += g_1^T h_0 (no gradient w.r.t. the encoding)
                first = false;
                continue;
            }
            const uint32_t row = tile * kTile + r;
            const bool valid = row < a.n;
            float rec[16];
            float tg[3] = {0.f, 0.f, 0.f};
            if (have_next && tile == blockIdx.x) {
                // gathered and encoded into h0 during the previous step's barrier wait
#pragma unroll
                for (int i = 0; i < 16; ++i) rec[i] = rec_n[i];
#pragma unroll
                for (int c = 0; c < 3; ++c) tg[c] = tg_n[c];
                have_next = false;
            } else {
                gather_row(step, row, rec, tg);
                NRC_TRC(2);
                uint32_t h[32];
                encode_record<EXACT>(rec, a.ep, h);
                store_row_swz(hs(0), r, h);
            }
            if (!weights_ready) {
                // the weight image (and the partials buffer) belong to the previous
                // kernel in the stream until it has completed
                pdl_wait();
                load_weights();
                weights_ready = true;
                NRC_TRC(3);
            }
            sync_rows();
            NRC_TRC(4);

            // ---------------- forward: h_{i+1} = relu(W_i h_i), y = W5 h5
#pragma unroll 1
            for (int L = 0; L < 5; ++L) {
                if (warp == 0)
                    warp_issue<kKmajStep, kKmajStep, 4>(t_acc, desc_kmajor(hs(L), 0),
                                                        desc_kmajor(sW_a + layer_off(L) * 2, 0), idesc_fwd, 0u,
                                                        mma_bar);
                mma_wait();
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    uint32_t v[32];
                    tmem_ld32(t_acc + lane_off + 32 * half, v);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float* f = reinterpret_cast<const float*>(v) + 8 * c;
                        st_shared_v4(hs(L + 1) + swz(r, 4 * half + c), pack_h2_relu(f[0], f[1]),
                                     pack_h2_relu(f[2], f[3]), pack_h2_relu(f[4], f[5]), pack_h2_relu(f[6], f[7]));
                    }
                }
                sync_rows();
                NRC_TRC(5 + L);
            }
            if (warp == 0)
                warp_issue<kKmajStep, kKmajStep, 4>(t_acc, desc_kmajor(hs(5), 0), desc_kmajor(sW_a + layer_off(5) * 2, 0),
                                                    idesc_out, 0u, mma_bar);
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
            sync_rows();
            NRC_TRC(10);
            if (last && !a.fused) pdl_trigger();  // the optimiser kernel may begin launching

            // ---------------- backward.  Round i: thread 0 queues
            // dgrad_i and commits it, then warp 4 queues wgrad_{i+1} behind it; the
            // rows wait for dgrad_i only.  G_{i+2} is staged and bulk-stored in
            // round i (its wgrad was queued a round earlier).
            if (warp == 0)  // delta5 = gy W5 (one K=16 step)
                warp_issue<0, 0, 1>(t_acc, desc_kmajor(sG6_a, 0), desc_mnmajor(sW_a + layer_off(5) * 2, 0), idesc_dgrad,
                                    0u, mma_bar);
            mma_wait();
            mask_epilogue(5);
            sync_rows();
            NRC_TRC(11);
#pragma unroll 1
            for (int i = 4; i >= 1; --i) {
                if (warp == 0) {  // delta_i = g_{i+1} W_i
                    warp_issue<kKmajStep, kMNmajStep, 4>(t_acc, desc_kmajor(gb(i + 1), 0),
                                                         desc_mnmajor(sW_a + layer_off(i) * 2, 0), idesc_dgrad, 0u,
                                                         mma_bar);
                    named_bar_arrive(kBarDgrad, 64);  // warp 4 may queue wgrad_{i+1} now
                }
                if (i <= 3) {
                    // wgrad_{i+2} (queued before dgrad_i) done: g_{i+3}'s buffer and
                    // slot i+2 are dead; G_{i+2} is staged while dgrad_i runs
                    wg_wait();
                    if (last) stage_partial(i + 2);
                }
                mma_wait();
                mask_epilogue(i);
                sync_rows();
                if (last && i <= 3 && tid == 0) mbar_arrive(staged_bar);  // warp 5 stores G_{i+2}
                NRC_TRC(16 - i);
            }
            named_bar_arrive(kBarG1, kTrainThreads);  // warp 4 may queue wgrad_1, wgrad_0
            wg_wait();  // wgrad_2
            if (last) stage_partial(2);
            wg_wait();  // wgrad_1, wgrad_0
            NRC_TRC(16);
            if (last) {
                stage_partial(1);
                stage_partial(0);
                fence_async_smem();
                named_bar_sync(kBarRows, 128);
                store_partial(2);
                store_partial(1);
                store_partial(0);
            }
            first = false;
        }
        const unsigned long long G = gridDim.x;
        const StepCoef sc = a.coef[step];
        const OptParams op{a.lr, a.b1, a.b2, a.adam_eps, sc.inv_bc1, sc.inv_bc2, sc.ema_c1, sc.ema_c2};
        // Deterministic reduction of partial chunks [cA, cB) over the G partials
        // + Adam + EMA, by threads t < T of a thread set that syncs with sync().
        // ng == 1: each thread owns whole chunks; else thread t sums chunk t % nch
        // over partials p = z, z + ng, ... (z = t / nch) and the group sums are
        // added in group order through scratch.  The order depends only on G.
        auto reduce_apply = [&](int cA, int cB, int t, int T, float* scratch, auto&& sync) {
            const int nch = cB - cA, per = 4 * nch;
            const int ng = nch >= T ? 1 : T / nch;
            const float4* P4 = reinterpret_cast<const float4*>(a.partials) + cA;
            auto sum_chunk = [&](int c, int z) {
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
                for (int p = z; p < int(G); p += 16 * ng) {  // 16 loads in flight (predicated tail)
                    float4 x[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        x[u] = (p + u * ng < int(G)) ? __ldcg(P4 + size_t(p + u * ng) * kParamChunks + c)
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        acc.x += x[u].x;
                        acc.y += x[u].y;
                        acc.z += x[u].z;
                        acc.w += x[u].w;
                    }
                }
                return acc;
            };
            if (ng == 1) {
                for (int c = t; c < nch; c += T) {
                    const float4 g4 = sum_chunk(c, 0);
                    const float g[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        adam_ema_update(partial_to_param(4 * (cA + c) + e), g[e] * a.inv_n, op, a.w, a.m, a.v, a.ema,
                                        a.wimg_out, a.eimg, a.bad_grads);
                }
                return;
            }
            // Adam state of the first two owned parameters, loaded under the partial loads
            float st0[4] = {0.f, 0.f, 0.f, 0.f}, st1[4] = {0.f, 0.f, 0.f, 0.f};  // m, v, w, e
            if (t < per) {
                const int j = partial_to_param(4 * cA + t);
                st0[0] = ld_global_f32(a.m + j), st0[1] = ld_global_f32(a.v + j);
                st0[2] = ld_global_f32(a.w + j), st0[3] = ld_global_f32(a.ema + j);
            }
            if (t + T < per) {
                const int j = partial_to_param(4 * cA + t + T);
                st1[0] = ld_global_f32(a.m + j), st1[1] = ld_global_f32(a.v + j);
                st1[2] = ld_global_f32(a.w + j), st1[3] = ld_global_f32(a.ema + j);
            }
            if (t < ng * nch) reinterpret_cast<float4*>(scratch)[t] = sum_chunk(t % nch, t / nch);
            sync();
            for (int q = t, u = 0; q < per; q += T, ++u) {
                float g = 0.0f;
                for (int z = 0; z < ng; ++z) g += scratch[z * per + q];
                const int j = partial_to_param(4 * cA + q);
                if (u < 2) {
                    const float* stv = u == 0 ? st0 : st1;
                    adam_ema_apply(j, g * a.inv_n, op, stv[0], stv[1], stv[2], stv[3], a.w, a.m, a.v, a.ema,
                                   a.wimg_out, a.eimg, a.bad_grads);
                } else {
                    adam_ema_update(j, g * a.inv_n, op, a.w, a.m, a.v, a.ema, a.wimg_out, a.eimg, a.bad_grads);
                }
            }
        };
        if (first && warp < 4) {  // no tile for this CTA: contribute zeros
            pdl_wait();
            for (int j = tid; j < kParamPadded; j += 128) part[j] = 0.0f;
        }
        NRC_GTRC(0);
        if (tid == 0) bulk_wait_all();  // partials globally written
        NRC_TRC(30);
        NRC_GTRC(1);
        // ---------------- this CTA's loss sum (fixed-order reduction over the 4 row warps)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            loss_sum += __shfl_xor_sync(0xffffffffu, loss_sum, off);
            bad += __shfl_xor_sync(0xffffffffu, bad, off);
        }
        if (lane == 0 && warp < 4) {
            red[warp] = loss_sum;
            reinterpret_cast<uint32_t*>(red + 4)[warp] = bad;
        }
        tc_fence_before();
        if (warp < 5) named_bar_sync(kBarTile, kTrainThreads);  // rows + warp 4 (helpers are not involved)
        if (tid == 0) {
            a.loss_part[blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
            const uint32_t* b = reinterpret_cast<const uint32_t*>(red + 4);
            const uint32_t nb = b[0] + b[1] + b[2] + b[3];
            if (nb) atomicAdd(a.bad_targets, (unsigned long long)nb);
        }
        loss_sum = 0.0f;
        bad = 0;
        if (!a.fused) break;

        // ---------------- optimiser (fused mode).  Grid barrier 1: thread 0
        // arrives once this CTA's partials and loss are written; the helper
        // warps meanwhile reduce W3..W5 (phase A) and join before phase B.
        if (warp >= 5) {
            // ---------------- phase A (helper warps): W3..W5 as soon as every CTA
            // has written them, overlapping the rows' last backward round
            if (tid == 160) wait_counter(a.gbarA, a.gbarA_base + G * (step + 1));
            named_bar_sync(kBarHelp, kHelpThreads);
            const int n_a = kParamChunks - kChunkSplit;
            reduce_apply(kChunkSplit + int(blockIdx.x * uint32_t(n_a) / uint32_t(G)),
                         kChunkSplit + int((blockIdx.x + 1) * uint32_t(n_a) / uint32_t(G)), int(tid) - 160,
                         kHelpThreads, sHelp, [&]() { named_bar_sync(kBarHelp, kHelpThreads); });
        }
        if (tid == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.gbar) : "memory");
            wait_counter(a.gbar, a.gbar_base + G * (2 * step + 1));
        }
        __syncthreads();
        NRC_TRC(17);
        NRC_GTRC(2);
        {
            // phase B: W0..W2, this CTA's balanced slice of chunks [0, kChunkSplit),
            // all 384 threads, group sums staged in the (now free) stash
            reduce_apply(int(blockIdx.x * uint32_t(kChunkSplit) / uint32_t(G)),
                         int((blockIdx.x + 1) * uint32_t(kChunkSplit) / uint32_t(G)), int(tid), kTrainBlock,
                         sOpt + 4 * kTileBytes / 4,  // stash slot 4 (slot 0 takes the next h0)
                         [&]() { __syncthreads(); });
            NRC_TRC(18);
            if (blockIdx.x == 0 && warp == 4 && a.losses != nullptr) {
                float x[8];  // G <= 256 partials, all loads in flight
#pragma unroll
                for (int u = 0; u < 8; ++u) x[u] = (lane + 32 * u < G) ? __ldcg(a.loss_part + lane + 32 * u) : 0.0f;
                float s = 0.0f;
#pragma unroll
                for (int u = 0; u < 8; ++u) s += x[u];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
                if (lane == 0) a.losses[step] = s * a.inv_n;
            }
        }
        NRC_TRC(19);
        NRC_GTRC(3);
        // grid barrier 2: arrive, gather + encode the next step's first tile
        // while the other CTAs finish their slices, then wait
        __syncthreads();
        if (tid == 0) {
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.gbar) : "memory");
        }
        if (step + 1 < a.nsteps && warp < 4 && blockIdx.x < ntiles) {
            gather_row(step + 1, blockIdx.x * kTile + r, rec_n, tg_n);
            uint32_t h[32];
            encode_record<EXACT>(rec_n, a.ep, h);
            store_row_swz(hs(0), r, h);
            fence_async_smem();
            have_next = true;
        }
        if (tid == 0) {
            wait_counter(a.gbar, a.gbar_base + G * (2 * step + 2));
        }
        __syncthreads();
        NRC_TRC(20);
        NRC_GTRC(4);
        if (step + 1 < a.nsteps) load_weights();  // W_{t+1}
        NRC_TRC(21);
        NRC_GTRC(5);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, kTrainTmemCols);
    NRC_TRC(31);
}
#undef NRC_TRC
#undef NRC_GTRC

}  // namespace nrc
