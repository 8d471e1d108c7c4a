// nrc_common.cuh -- argument blocks and small device helpers shared by the
// query kernel (nrc_query_ts.cuh) and the training kernels (nrc_train_w.cuh).
#pragma once
#include "nrc_device.cuh"

namespace nrc {

constexpr int kMaxRanks = 8;  // GPUs of one box (multi-GPU paths)

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// ----------------------------------------------------------------- query
struct QueryArgs {
    const float* rec;    // n records x 16 fp32
    float* out;          // n x 3 fp32
    uint64_t n;
    const uint8_t* wimg; // fp16 operand image, EMA or raw
    EncodeParams ep;
    uint32_t flags;      // NRC_FACTORIZE | NRC_CLAMP_QUERY
    long long* dbg;      // unused by the query kernel (diagnostics hook of the training kernels)
    // fused pixel reconstruction (nrc_query_accumulate): if image != nullptr,
    // image[3 pix[i] + c] += thr[3 i + c] * q_c instead of out
    const uint32_t* pix;
    const float* thr;
    float* image;
    uint32_t nh;                     // hidden layers
    unsigned long long* degenerate;  // += number of zero-length omega / n vectors encoded (R7)
};

constexpr int kRecTileBytes = kTile * kRecFloats * 4;  // 8 KB of records per tile

// ----------------------------------------------------------------- training
struct StepCoef {
    float inv_bc1, inv_bc2;  // Adam bias corrections 1/(1-b^t)
    float ema_c1, ema_c2;    // W-bar = c1 W + c2 W-bar (Eq. 2 / R12)
};

struct TrainArgs {
    const float* rec;      // records (indexed through the gather below)
    const float* tgt;      // targets, 3 fp32 per record
    uint32_t n;            // rows per step
    uint32_t gather;       // 1: row k reads record lcg_perm(offset + k); 0: record k
    uint64_t lcg_a, lcg_c, lcg_m, lcg_n, offset;
    const uint8_t* wimg;   // fp16 image of the TRAINING weights W_t
    EncodeParams ep;
    uint32_t flags;
    float loss_eps;
    float* partials;       // [gridDim.x][padded] fp32 un-normalised gradient sums (chunk-major, part_index)
    float* loss_part;      // [gridDim.x] loss sums
    unsigned long long* bad_targets;
    unsigned long long* degenerate;  // zero-length omega / n vectors encoded (R7)
    float* pred;           // optional: the training forward's factored prediction y * (alpha + beta), n x 3
    long long* dbg;        // optional phase timestamps (diagnostics), else nullptr
    uint32_t nh;           // hidden layers
};

__device__ __forceinline__ float ld_global_f32(const float* p) {  // not sunk past the partial loads
    float v;
    asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}

// 0xFFFF in each 16-bit half whose fp16 activation is > 0 (ReLU'(0) = 0, R17)
__device__ __forceinline__ uint32_t relu_mask(uint32_t h2bits) {
    __half2 h;
    memcpy(&h, &h2bits, 4);
    return __hgt2_mask(h, __float2half2_rn(0.0f));
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ long long global_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Sum of a per-thread counter over the CTA, added once to *ctr (thread 0).
// All threads of the block must call it.
__device__ __forceinline__ void block_count_add(unsigned long long* ctr, uint32_t mine, uint32_t* scratch) {
    uint32_t s = __reduce_add_sync(0xffffffffu, mine);
    if ((threadIdx.x & 31) == 0 && s != 0) atomicAdd(scratch, s);
    __syncthreads();
    if (threadIdx.x == 0 && *scratch != 0 && ctr != nullptr) atomicAdd(ctr, (unsigned long long)*scratch);
}

}  // namespace nrc
