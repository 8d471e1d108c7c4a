// nrc_device.cuh -- sm_100a device primitives for libnrc: PTX wrappers for
// mbarriers, 1-D TMA bulk copies, tcgen05 (UMMA, TMEM alloc/ld, commit), the
// 128B-swizzled operand layout, and the input encoding (Table 1).
//
// Operand layout: every 64-wide fp16 tile (activations,
// gradients, weights) is stored as 128-byte lines, line r holding 64 fp16
// values whose 16-byte chunk c sits at chunk position c ^ (r & 7) -- the
// SWIZZLE_128B atom (8 lines x 128 B, 1024-B aligned).  The same bytes are a
// K-major operand when a line is an M/N row and an MN-major operand when a
// line is a K row, so one stored tile serves forward, dgrad and wgrad.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace nrc {

// ----------------------------------------------------------------- constants
constexpr int kW = 64;                    // hidden width
constexpr int kTile = 128;                // rows per tile (one TMEM lane per row)
constexpr int kNumLayers = 6;             // W0..W5 (reading R1)
constexpr int kOutPad = 16;               // W5 padded to 16 rows (UMMA N granularity)
constexpr int kParamLogical = 5 * 64 * 64 + 3 * 64;   // 20,672
constexpr int kParamPadded = 5 * 64 * 64 + 16 * 64;   // 21,504
constexpr int kParamPaddedEnd = kParamPadded;
// start of layer i in the padded parameter layout (i = 6: end)
__host__ __device__ constexpr int layer_off(int i) { return i < 6 ? i * 4096 : kParamPaddedEnd; }
constexpr int kImgBytes = kParamPadded * 2;           // 43,008 B fp16 image

// Hidden width W in {32, 64, 128} (width ablation; W = 64 is the
// paper's network and the layout above).  Layer i has rows(i) outputs (W,
// W5 padded to 16) and cols(i) inputs (64 for W0, else W).
//  * fp32 padded arrays: element (i, r, c) at pad_off(i) + r cols(i) + c.
//  * fp16 operand image: layer i is cols(i)/64 (rounded up) K-blocks of
//    rows(i) 128-byte lines (64 halves, SWIZZLE_128B chunk order c ^ (r % 8)).
template <int W>
struct NetDims {
    static_assert(W == 32 || W == 64 || W == 128, "hidden width 32, 64 or 128");
    __host__ __device__ static constexpr int rows(int i) { return i < 5 ? W : kOutPad; }
    __host__ __device__ static constexpr int cols(int i) { return i == 0 ? 64 : W; }
    __host__ __device__ static constexpr int kblocks(int i) { return (cols(i) + 63) / 64; }
    __host__ __device__ static constexpr int pad_off(int i) {
        return i == 0 ? 0 : i <= 5 ? 64 * W + (i - 1) * W * W : 64 * W + 4 * W * W + kOutPad * W;
    }
    // sum over j < i of kblocks(j) rows(j) 128 (closed form: no recursion at run time)
    __host__ __device__ static constexpr int img_off(int i) {
        return i == 0 ? 0
                      : i <= 5 ? W * 128 + (i - 1) * ((W + 63) / 64) * W * 128
                               : W * 128 + 4 * ((W + 63) / 64) * W * 128 + ((W + 63) / 64) * kOutPad * 128;
    }
    static constexpr int kPadded = 64 * W + 4 * W * W + kOutPad * W;
    static constexpr int kLogical = 64 * W + 4 * W * W + 3 * W;
    static constexpr int kImg = img_off(6);
    __host__ __device__ static constexpr uint32_t img_byte(int i, int r, int c) {
        return uint32_t(img_off(i) + (c >> 6) * rows(i) * 128 + r * 128) +
               ((uint32_t((c & 63) >> 3) ^ uint32_t(r & 7)) << 4) + uint32_t(c & 7) * 2u;
    }
};
static_assert(NetDims<64>::kPadded == kParamPadded && NetDims<64>::kImg == kImgBytes, "W=64 layout");

// NetDims<W> with a run-time number of hidden layers nh (SURVEY N4 depth
// variants; nh = 5 gives NetDims<W>): layers 0..nh, layer nh is the output
// layer (rows padded to 16); the same padded fp32 and fp16 image layouts.
template <int W>
struct NetRt {
    int nh;
    __host__ __device__ constexpr explicit NetRt(int nh_) : nh(nh_) {}
    __host__ __device__ constexpr int rows(int i) const { return i < nh ? W : kOutPad; }
    __host__ __device__ static constexpr int cols(int i) { return i == 0 ? 64 : W; }
    __host__ __device__ static constexpr int kblocks(int i) { return (cols(i) + 63) / 64; }
    __host__ __device__ constexpr int pad_off(int i) const {
        return i == 0 ? 0 : i <= nh ? 64 * W + (i - 1) * W * W : 64 * W + (nh - 1) * W * W + kOutPad * W;
    }
    __host__ __device__ constexpr int img_off(int i) const {
        return i == 0 ? 0
                      : i <= nh ? W * 128 + (i - 1) * ((W + 63) / 64) * W * 128
                                : W * 128 + (nh - 1) * ((W + 63) / 64) * W * 128 + ((W + 63) / 64) * kOutPad * 128;
    }
    __host__ __device__ constexpr int padded() const { return pad_off(nh + 1); }
    __host__ __device__ constexpr int logical() const { return 64 * W + (nh - 1) * W * W + 3 * W; }
    __host__ __device__ constexpr int img() const { return img_off(nh + 1); }
    __host__ __device__ constexpr uint32_t img_byte(int i, int r, int c) const {
        return uint32_t(img_off(i) + (c >> 6) * rows(i) * 128 + r * 128) +
               ((uint32_t((c & 63) >> 3) ^ uint32_t(r & 7)) << 4) + uint32_t(c & 7) * 2u;
    }
    // layer of padded parameter j
    __host__ __device__ constexpr int layer_of(int j) const {
        int i = 0;
        while (i < nh && j >= pad_off(i + 1)) ++i;
        return i;
    }
};
constexpr int kTileBytes = kTile * 128;               // 16 KB per 128x64 fp16 tile
constexpr int kRecFloats = 16;                        // 64-B record

// ----------------------------------------------------------------- misc PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "NRC_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra NRC_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 1-D TMA bulk copy shared -> global (bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src_saddr, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src_saddr), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// Generic-proxy smem writes -> visible to the async proxy (tensor core reads).
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ----------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem], kind::f16 (fp16 in, fp32 accumulate).
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Same with the A operand read from TMEM (lane = row, 2 fp16 per column, K-major).
__device__ __forceinline__ void umma_f16_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// One lane of a converged warp (elect.sync).  Issuing tcgen05.mma from an
// elected lane of a converged warp, with operands made warp-uniform by
// __shfl_sync, lets ptxas keep the descriptors in uniform registers: ~170
// cycles for a 4-MMA chain + commit instead of ~650 from a lone divergent
// thread (scripts/ubench_tcgen05.cu modes 10/17).
__device__ __forceinline__ bool elect_one() {
    uint32_t p = 0;
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n}" : "=r"(p));
    return p != 0;
}
__device__ __forceinline__ uint32_t warp_uniform(uint32_t x) { return __shfl_sync(0xffffffffu, x, 0); }
__device__ __forceinline__ uint64_t warp_uniform(uint64_t x) {
    const uint32_t lo = __shfl_sync(0xffffffffu, uint32_t(x), 0), hi = __shfl_sync(0xffffffffu, uint32_t(x >> 32), 0);
    return (uint64_t(hi) << 32) | lo;
}
// K chains of 4 or 8 MMAs with both operands in shared memory; operand
// descriptors advance by ASTEP / BSTEP (16-byte units) per K=16 step.  The
// first MMA accumulates iff acc0 != 0.  Issue from an elected lane of a
// converged warp (see elect_one), then umma_commit from the same lane.
template <int ASTEP, int BSTEP>
__device__ __forceinline__ void umma_ss4(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc0) {
    asm volatile(
        "{\n\t.reg .pred p, t;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
        "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
        "add.u64 a1, %1, %5;\n\tadd.u64 a2, %1, %6;\n\tadd.u64 a3, %1, %7;\n\t"
        "add.u64 b1, %2, %8;\n\tadd.u64 b2, %2, %9;\n\tadd.u64 b3, %2, %10;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, t;\n}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc0), "n"(ASTEP), "n"(2 * ASTEP), "n"(3 * ASTEP), "n"(BSTEP),
        "n"(2 * BSTEP), "n"(3 * BSTEP)
        : "memory");
}
template <int ASTEP, int BSTEP>
__device__ __forceinline__ void umma_ss8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc0) {
    umma_ss4<ASTEP, BSTEP>(d_tmem, a, b, idesc, acc0);
    umma_ss4<ASTEP, BSTEP>(d_tmem, a + 4 * ASTEP, b + 4 * BSTEP, idesc, 1u);
}
// descriptor K-step increments (16-byte units): K-major +32 B, MN-major +2048 B
constexpr int kKmajStep = 2, kMNmajStep = 128;

// One 64-deep K chain (4 x K=16) with A in TMEM and B a K-major SWIZZLE_128B
// smem tile, then a commit to `bar`, in ONE asm block: the K steps are
// a + 8 columns and b_desc + 2 (32 B) computed inside, so ptxas materialises
// the uniform operands once instead of re-broadcasting six registers per MMA
// (each re-broadcast waits for the previous tcgen05.mma to read its operands).
__device__ __forceinline__ void umma_chain4_ta_commit(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                                      uint32_t idesc, uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred f, t;\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t"
        "setp.ne.b32 f, 0, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
        "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
        "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, f;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, t;\n\t"
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(smem_u32(bar))
        : "memory");
}
// Arrive on an mbarrier once all previously issued tcgen05 ops of this thread
// have completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// Instruction descriptor, kind::f16: D fp32, A/B fp16, majors, N>>3, M>>4.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int a_mn_major, int b_mn_major) {
    return (1u << 4) | (uint32_t(a_mn_major) << 15) | (uint32_t(b_mn_major) << 16) | (uint32_t(N >> 3) << 17) |
           (uint32_t(M >> 4) << 24);
}
// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version field = 1.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFFu);
    d |= uint64_t((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
// K-major operand (line = M/N row, 64 K values per line); K step of 16 = +32 B.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t tile_saddr, int kstep) {
    return make_sdesc(tile_saddr + 32u * kstep, 16u, 1024u);
}
// MN-major operand (line = K row, 64 M/N values per line); K step of 16 = +2048 B.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t tile_saddr, int kstep) {
    return make_sdesc(tile_saddr + 2048u * kstep, 8192u, 1024u);
}

// 32 lanes x 32 bit, 32 / 16 / 4 consecutive columns.  The wait takes the
// registers as in/out operands so no use can be scheduled before it.
#define NRC_R8(o) "=r"(r[o + 0]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3]), "=r"(r[o + 4]), "=r"(r[o + 5]), \
                  "=r"(r[o + 6]), "=r"(r[o + 7])
#define NRC_W8(o) "+r"(r[o + 0]), "+r"(r[o + 1]), "+r"(r[o + 2]), "+r"(r[o + 3]), "+r"(r[o + 4]), "+r"(r[o + 5]), \
                  "+r"(r[o + 6]), "+r"(r[o + 7])
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : NRC_R8(0), NRC_R8(8), NRC_R8(16), NRC_R8(24)
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" : NRC_W8(0), NRC_W8(8), NRC_W8(16), NRC_W8(24)::"memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : NRC_R8(0), NRC_R8(8)
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" : NRC_W8(0), NRC_W8(8)::"memory");
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3])::"memory");
}
#define NRC_S8(o) "r"(r[o + 0]), "r"(r[o + 1]), "r"(r[o + 2]), "r"(r[o + 3]), "r"(r[o + 4]), "r"(r[o + 5]), \
                  "r"(r[o + 6]), "r"(r[o + 7])
// 32 lanes x 32 bit store of 32 consecutive columns, then wait for completion.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        NRC_S8(0), NRC_S8(8), NRC_S8(16), NRC_S8(24)
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// 16 consecutive columns, no wait (pair with tmem_wait_st before the data is used)
__device__ __forceinline__ void tmem_st16_nowait(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        NRC_S8(0), NRC_S8(8)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
#undef NRC_S8
#undef NRC_R8
#undef NRC_W8

// ----------------------------------------------------------------- fp16 packing
// (lo, hi) -> f16x2 with round-to-nearest-even (cvt puts its FIRST source in
// the upper half).
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
    uint32_t d;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
    return d;
}
// Same with ReLU fused into the conversion (cvt.rn.relu).
__device__ __forceinline__ uint32_t pack_h2_relu(float lo, float hi) {
    uint32_t d;
    asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
    return d;
}
// Byte offset of 16-B chunk c of line r inside a SWIZZLE_128B tile.
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t c) { return r * 128u + ((c ^ (r & 7u)) << 4); }

__device__ __forceinline__ void st_shared_v4(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(saddr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t saddr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(saddr)
                 : "memory");
    return v;
}

// ----------------------------------------------------------------- encoding
// Position normalisation constants: v = fp32(fp32(p - lo) * inv) (reading R3).
struct EncodeParams {
    float lo[3];
    float inv[3];
    uint32_t exact;  // 1: sin / Gaussian primitives (NRC_EXACT_ENCODING, N4) instead of tri / quartic
};

// 1.0f if a >= b else 0.0f (one FSET)
__device__ __forceinline__ float set_ge(float a, float b) {
    float r;
    asm("set.ge.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
// quartic(x) = 15/16 (1 - x^2)^2 on |x| <= 1, else 0: clamping
// 1 - x^2 at 0 gives the compact support without a compare; 1 - x^2 <= 1, so
// the clamp is a saturate folded into the FFMA (FFMA.SAT, same value).
__device__ __forceinline__ float quartic_f(float x) {
    const float t = __saturatef(fmaf(-x, x, 1.0f));
    return (0.9375f * t) * t;
}
// One-blob, k = 4, centres (i + 1/2)/4, width 1/4, clamp to [0,1] (R6).
__device__ __forceinline__ void one_blob4(float s, float* o) {
    s = __saturatef(s);
    float x = 4.0f * s;
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = quartic_f(x - (float(i) + 0.5f));
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float r;
    asm("ex2.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// atan2(y, x) with IEEE sign conventions (atan2(+-0, x<0) = +-pi, atan2(+-0,
// -0) = +-pi: the sign bit of x decides), |error| <= 1.2e-7 rad: atan(a) =
// a P(a^2) on [0,1] (degree-7 minimax fit, fp32 Horner).
__device__ __forceinline__ float atan2_fast(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    const float a = mx > 0.0f ? __fdividef(mn, mx) : 0.0f;
    const float s = a * a;
    float p = -0.004053147975355387f;
    p = fmaf(p, s, 0.021859295666217804f);
    p = fmaf(p, s, -0.05590952932834625f);
    p = fmaf(p, s, 0.09642207622528076f);
    p = fmaf(p, s, -0.13908733427524567f);
    p = fmaf(p, s, 0.19946610927581787f);
    p = fmaf(p, s, -0.3332986831665039f);
    p = fmaf(p, s, 0.9999993443489075f);
    float r = a * p;
    if (ay > ax) r = 1.57079632679489662f - r;
    if (__float_as_uint(x) >> 31) r = 3.14159265358979323846f - r;
    return copysignf(r, y);
}
// sph (Table 1 caption; reading R7): (acos(u_z / |u|)/pi,
// (atan2(u_y, u_x) + pi)/(2 pi)), computed without normalising u:
// acos(z / |u|) = atan2(sqrt(x^2 + y^2), z) for u != 0 (the same angle, but
// well conditioned at the poles, where acos of a rounded z / |u| is not:
// d acos / dz = -1 / sin(theta)).  Returns 1 for a zero-length (degenerate)
// vector, read as (0,0,1) and counted.
__device__ __forceinline__ uint32_t sph_f(float x, float y, float z, float& th, float& ph) {
    const float r2 = x * x + y * y;
    const float l2 = fmaf(z, z, r2);
    const uint32_t degenerate = !(l2 > 0.0f) ? 1u : 0u;
    if (degenerate) {
        x = 0.0f;
        y = 0.0f;
        z = 1.0f;
    }
    th = atan2_fast(sqrt_approx(degenerate ? 0.0f : r2), z) * 0.318309886183790672f;  // 1/pi
    ph = (atan2_fast(y, x) + 3.14159265358979323846f) * 0.159154943091895336f;  // 1/(2 pi)
    return degenerate;
}

// Encodes one record into 64 fp16 features packed as 32 f16x2 words, in the
// order of reading R5 / Table 1: freq(x) 36 | ob(sph(w)) 8 | ob(sph(n)) 8 |
// ob(1-e^-r) 4 | alpha 3 | beta 3 | 1, 1.
// Exact primitives (readings R21/R22): sin(pi 2^d v) with
// sinpif's exact range reduction (2^d v is exact in fp32), and the Gaussian
// one-blob exp(-x^2/2)/sqrt(2 pi) at the bin centres.
__device__ __forceinline__ uint32_t encode_record_exact(const float* rec, const EncodeParams& ep, uint32_t (&h)[32]) {
    float e[64];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float v = __fmul_rn(__fsub_rn(rec[a], ep.lo[a]), ep.inv[a]);
#pragma unroll
        for (int d = 0; d < 12; ++d) e[12 * a + d] = sinpif(ldexpf(v, d));
    }
    auto ob = [](float s, float* o) {
        s = fminf(fmaxf(s, 0.0f), 1.0f);
        const float x = 4.0f * s;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float t = x - (float(i) + 0.5f);
            o[i] = 0.3989422804014327f * __expf(-0.5f * t * t);
        }
    };
    float th, ph;
    uint32_t deg = sph_f(rec[3], rec[4], rec[5], th, ph);
    ob(th, e + 36);
    ob(ph, e + 40);
    deg += sph_f(rec[6], rec[7], rec[8], th, ph);
    ob(th, e + 44);
    ob(ph, e + 48);
    ob(1.0f - ex2_approx(-1.44269504088896341f * fmaxf(rec[9], 0.0f)), e + 52);
#pragma unroll
    for (int c = 0; c < 6; ++c) e[56 + c] = rec[10 + c];
    e[62] = 1.0f;
    e[63] = 1.0f;
#pragma unroll
    for (int j = 0; j < 32; ++j) h[j] = pack_h2(e[2 * j], e[2 * j + 1]);
    return deg;
}

__device__ __forceinline__ uint32_t encode_record_cheap(const float* rec, const EncodeParams& ep, uint32_t (&h)[32]);
// EXACT selects the primitives at compile time (kernels are instantiated per
// variant, so the cheap path carries no trace of the exact one).
// Returns the number (0..2) of zero-length direction / normal vectors (R7).
template <bool EXACT = false>
__device__ __forceinline__ uint32_t encode_record(const float* rec, const EncodeParams& ep, uint32_t (&h)[32]) {
    if constexpr (EXACT) {
        return encode_record_exact(rec, ep, h);
    } else {
        return encode_record_cheap(rec, ep, h);
    }
}
__device__ __forceinline__ uint32_t encode_record_cheap(const float* rec, const EncodeParams& ep, uint32_t (&h)[32]) {
    float e[64];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        // tri is even (tri(-x) = tri(x)), so work on |v|: then v - 2 floor(v / 2)
        // is exact in fp32 (for v < 0 it is not: the result may need a finer
        // ulp than v, and the doublings below would amplify the rounding)
        const float v = fabsf(__fmul_rn(__fsub_rn(rec[a], ep.lo[a]), ep.inv[a]));
        // m_d = 2^d v mod 2 by exact doubling: m_{d+1} = 2 u_d with
        // u_d = m_d - [m_d >= 1] (exact); tri(2^d v) = 2 |m_d - 1| - 1
        // (P:L678), bit-identical to the direct form.  Per value: t = RN(2 u - 1)
        // (= RN(m - 1)), e, the 0/1 step [u >= 1/2] (one FSET) and u' = 2 u - step.
        const float m0 = v - 2.0f * floorf(v * 0.5f);
        float u = m0 - set_ge(m0, 1.0f);
#pragma unroll
        for (int d = 0; d < 12; ++d) {
            const float t = d == 0 ? m0 - 1.0f : fmaf(2.0f, u, -1.0f);
            e[12 * a + d] = fmaf(2.0f, fabsf(t), -1.0f);
            if (d > 0) u = fmaf(2.0f, u, -set_ge(u, 0.5f));
        }
    }
    float th, ph;
    uint32_t deg = sph_f(rec[3], rec[4], rec[5], th, ph);
    one_blob4(th, e + 36);
    one_blob4(ph, e + 40);
    deg += sph_f(rec[6], rec[7], rec[8], th, ph);
    one_blob4(th, e + 44);
    one_blob4(ph, e + 48);
    one_blob4(1.0f - ex2_approx(-1.44269504088896341f * fmaxf(rec[9], 0.0f)), e + 52);  // 1 - e^{-r}
#pragma unroll
    for (int c = 0; c < 6; ++c) e[56 + c] = rec[10 + c];
    e[62] = 1.0f;
    e[63] = 1.0f;
#pragma unroll
    for (int j = 0; j < 32; ++j) h[j] = pack_h2(e[2 * j], e[2 * j + 1]);
    return deg;
}

// Writes a packed 64-feature row into line `row` of a SWIZZLE_128B tile.
__device__ __forceinline__ void store_row_swz(uint32_t tile_saddr, uint32_t row, const uint32_t (&h)[32]) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
        st_shared_v4(tile_saddr + swz(row, c), h[4 * c + 0], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]);
}

// Fetch 16 floats of a record (64 B, 16-B aligned) from global memory.
__device__ __forceinline__ void load_record_global(const float* __restrict__ src, float* rec) {
    const float4* s = reinterpret_cast<const float4*>(src);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float4 v = __ldg(s + i);
        rec[4 * i + 0] = v.x;
        rec[4 * i + 1] = v.y;
        rec[4 * i + 2] = v.z;
        rec[4 * i + 3] = v.w;
    }
}

// LCG permutation of reading R15: f(i) = (a i + c) mod m, iterated
// until < n (cycle walking).
__device__ __forceinline__ uint64_t lcg_perm(uint64_t i, uint64_t n, uint64_t a, uint64_t c, uint64_t m) {
    uint64_t x = i;
    do {
        x = (a * x + c) & (m - 1);
    } while (x >= n);
    return x;
}

}  // namespace nrc
