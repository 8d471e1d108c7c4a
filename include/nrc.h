/*
 * nrc.h -- C ABI of libnrc, a B200-native (sm_100a) implementation of the
 * data-parallel hot path of Neural Radiance Caching (Mueller, Rousselle,
 * Novak, Keller, "Real-time Neural Radiance Caching for Path Tracing",
 * SIGGRAPH 2021, arXiv 2106.12372).
 *
 * Citations: "P:L<n>" = line n of the paper source; "S:L<n>" =
 * line n of SPEC.md; "R<k>" = reading k in DESIGN.md section 3.
 *
 * The calls follow the paper's statement of the problem: a radiance cache
 * that maps cache-query records (Table 1) to scattered radiance
 * (Eq. 1) through a fully fused 64-wide MLP (P:L602-628,
 * P:L692-698), trained online every frame from (record, target) pairs with
 * the relative L2 loss (Eq. 5) and Adam, with
 * EMA-averaged weights for queries (Eq. 2), on s batches of l
 * LCG-shuffled records.
 *
 * Conventions
 *  - All functions have C linkage, never throw and never exit.  They return
 *    nrc_status; on failure nrc_last_error(handle) holds a message.
 *  - Pointers named d_* are CUDA device pointers (e.g. torch tensors'
 *    data_ptr()); h_* are host pointers.  The caller owns every buffer,
 *    including the state arena passed to nrc_init.  The library never calls
 *    cudaMalloc/cudaFree.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Device-side calls are stream-ordered and asynchronous: results
 *    are valid once the stream has been synchronised.  nrc_get_params,
 *    nrc_set_params and nrc_get_stats are synchronous (device-wide sync).
 *  - Validation failures (NULL or misaligned pointers, n > max_batch, bad
 *    config) return NRC_ERR_INVALID_ARGUMENT / NRC_ERR_UNSUPPORTED and
 *    enqueue nothing.  n == 0 is a valid no-op.
 *  - Data-dependent problems never fail a call: non-finite gradient entries
 *    are zeroed and counted; records with a non-finite target are
 *    masked out of loss and gradient and counted.
 *  - A handle is not thread-safe.  Train calls on one handle must not
 *    overlap each other; queries may run concurrently with training only on
 *    another stream and only if the caller orders them against the EMA
 *    update (they read the fp16 EMA image that train steps rewrite).
 */
#ifndef NRC_H_
#define NRC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NRC_ABI_VERSION 2u

/* One cache query (Table 1): 16 fp32 = 64 bytes.
 * Arrays of records must be 16-byte aligned.  Domain: pos is any finite point
 * (inside or outside the AABB; the triangle waves are defined on all reals,
 * R3/R4); dir and normal need not be unit length (they are renormalised, R7;
 * |u|^2 must be a normal fp32 number or exactly 0, i.e. |u| in [1e-18, 1e18]
 * or u = 0); a zero vector reads as (0,0,1) and is counted
 * (nrc_get_stats); roughness < 0 reads as 0; reflectances are any finite
 * values (alpha + beta = 0 gives a zero query and zero gradient). */
typedef struct nrc_record {
    float pos[3];      /* x in world space; normalised by the config AABB (R3) */
    float dir[3];      /* scattered direction omega                              */
    float normal[3];   /* surface normal n(x)                                    */
    float roughness;   /* r(x, omega) >= 0 (negative values read as 0)           */
    float diffuse[3];  /* diffuse reflectance alpha                              */
    float specular[3]; /* specular reflectance beta                              */
} nrc_record;

typedef enum nrc_status {
    NRC_OK = 0,
    NRC_ERR_INVALID_ARGUMENT = 1,
    NRC_ERR_UNSUPPORTED = 2,
    NRC_ERR_OUT_OF_MEMORY = 3, /* state arena too small */
    NRC_ERR_CUDA = 4,          /* a CUDA call failed; see nrc_last_error */
    NRC_ERR_NCCL = 5,          /* reserved; not returned by this version */
    NRC_ERR_STATE = 6          /* handle not initialised / wrong device  */
} nrc_status;

/* Parameter sets readable/writable through nrc_get_params/nrc_set_params. */
typedef enum nrc_param_set {
    NRC_PARAMS_TRAIN = 0, /* fp32 master weights W_t             */
    NRC_PARAMS_EMA = 1,   /* EMA weights W-bar_t used by queries */
    NRC_ADAM_M = 2,       /* Adam first moment                            */
    NRC_ADAM_V = 3        /* Adam second moment                           */
} nrc_param_set;

/* nrc_config.flags */
enum {
    NRC_FACTORIZE = 1u,         /* multiply the output by alpha+beta       */
    NRC_CLAMP_QUERY = 2u,       /* clamp query radiance at 0 (R2)                        */
    NRC_EMA_PRINTED_FORM = 4u,  /* Eq.(2) exactly as printed instead of R12's form      */
    NRC_QUERY_RAW_WEIGHTS = 8u, /* queries read W_t instead of W-bar_t                  */
    NRC_EXACT_ENCODING = 16u    /* sin / Gaussian encoding primitives instead of the
                                 * cheap tri / quartic ones (
                                 * readings R21, R22)                       */
};

typedef struct nrc_config {
    uint32_t abi_version;      /* must equal NRC_ABI_VERSION                          */
    uint32_t hidden_width;     /* 64 ("five hidden layers have 64 neurons");
                                * 32 or 128 for the width ablation (BASELINE configs[3]),
                                * query and training alike.  nrc_param_count() gives
                                * 64 W + 4 W^2 + 3 W (logical layout: W0 W x 64,
                                * W1..W4 W x W, W5 3 x W, row-major [out][in]).        */
    uint32_t n_hidden_layers;  /* 5; depth variants: 1..8 / 1..7 / 1..5
                                * at hidden_width 32 / 64 / 128 (training-kernel shared
                                * memory), query and training alike; parameters
                                * 64 W + (n-1) W^2 + 3 W                              */
    uint32_t reserved0;        /* 0 (alignment of max_batch)                          */
    uint64_t max_batch;        /* largest n accepted by query/train calls, <= 2^40    */
    float aabb_min[3];         /* position normalisation domain (R3)           */
    float aabb_max[3];
    float learning_rate;       /* 1e-2 (R11; paper: "high learning-rate")     */
    float adam_beta1;          /* 0.9  (R11)                                          */
    float adam_beta2;          /* 0.99 (R11)                                          */
    float adam_eps;            /* 1e-8 (R11), added outside the square root           */
    float loss_eps;            /* 0.01 (Eq. 5)                                */
    float ema_alpha;           /* 0.99; 0 => W-bar == W                      */
    uint32_t flags;            /* default NRC_FACTORIZE | NRC_CLAMP_QUERY             */
    uint64_t seed;             /* Glorot-uniform init stream (R16)                    */
    int32_t device;            /* CUDA device ordinal the state lives on              */
} nrc_config;

typedef struct nrc_handle nrc_handle;

/* Fills *cfg with the paper's defaults (width 64, 5 hidden layers, unit-cube
 * AABB, lr 1e-2, betas 0.9/0.99, eps 1e-8, loss eps 0.01, EMA 0.99, seed 1,
 * max_batch 8,294,400 = one 4K frame, device 0). */
void nrc_default_config(nrc_config* cfg);

/* Bytes of device memory the caller must provide to nrc_init (weights,
 * Adam state, EMA, fp16 weight images, gradient partials, counters).
 * Returns 0 for an invalid config. */
size_t nrc_state_bytes(const nrc_config* cfg);

/* Validates cfg, carves the state out of d_state (device memory of at least
 * nrc_state_bytes(cfg) bytes, 256-byte aligned, owned by the caller and kept
 * alive until nrc_destroy), writes the seeded Glorot-uniform weights (R16),
 * W-bar = W, m = v = 0, step = 0.  Synchronous.  *out receives a host-side
 * handle (freed by nrc_destroy). */
nrc_status nrc_init(const nrc_config* cfg, void* d_state, size_t state_bytes, nrc_handle** out);

nrc_status nrc_destroy(nrc_handle* h);

/* Cache query: d_rgb[3i+c] = max(0, y_c(e(rec_i)) *
 * (alpha_c + beta_c)) with the EMA weights, for i < n.  d_rec: n
 * records (16-byte aligned); d_rgb: 3n fp32 (4-byte aligned).  One fused
 * kernel: encode -> 6 tcgen05 layers -> factorisation epilogue. */
nrc_status nrc_query(nrc_handle* h, const nrc_record* d_rec, uint64_t n, float* d_rgb, void* stream);

/* Query with the pixel reconstruction fused into the epilogue (
 * SURVEY 8(f) N2): the rendering path of pixel d_pixel[i] ends in cache query
 * i, whose radiance q_i (as nrc_query computes it) reaches the pixel through
 * the path throughput d_thr[3i..3i+2]:  d_image[3 d_pixel[i] + c] += d_thr[3i + c] q_ic.
 * d_image is an fp32 RGB image the caller owns and zeroes; the adds are
 * atomic (deterministic when the pixel indices are distinct, the one-query-
 * per-pixel case).  No radiance array is written. */
nrc_status nrc_query_accumulate(nrc_handle* h, const nrc_record* d_rec, uint64_t n, const uint32_t* d_pixel,
                                const float* d_thr, float* d_image, void* stream);

/* One optimisation step on a batch: forward, relative
 * L2 loss (Eq. 5) of the factored prediction, backward, Adam on the batch-
 * mean gradient, EMA update.  d_rec: n records; d_tgt: 3n fp32 targets;
 * d_loss (optional, 1 fp32): the batch-mean loss.  n <= max_batch.  Two
 * kernel launches: the partials kernel (min(#SMs, ceil(n/128)) CTAs) and the
 * reduce + Adam + EMA kernel, chained with programmatic dependent launch.
 * dL/dy is back-propagated in fp16 with a per-128-row power-of-two scale that
 * is undone exactly in fp32 (R13, R25), so HDR targets cannot overflow it. */
nrc_status nrc_train_step(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n, float* d_loss,
                          void* stream);

/* Multi-GPU split of nrc_train_step.  nrc_train_backward writes the UN-
 * normalised gradient sum over the n_local records into d_grad
 * (nrc_param_count() fp32, logical layout: W0 Wx64, W1..W4 WxW, W5 3xW,
 * row-major [out][in]) and, if d_loss_sum != NULL, the loss sum (1 fp32).
 * d_pred (optional, 3 n_local fp32): the training forward's (a4) factored
 * prediction y * (alpha + beta) of each record, unclamped -- the quantity the
 * loss sees (R9); with the same weights it equals nrc_query's radiance bit
 * for bit when the query reads W_t without the clamp.  The caller all-reduces
 * (SUM) d_grad (and the loss sum) across ranks, then nrc_train_apply runs
 * Adam + EMA with g = d_grad_sum / n_global and, if d_loss_sum and d_loss are
 * both given, writes the batch-mean loss *d_loss = *d_loss_sum / n_global
 * (R10).  Deterministic: equal inputs give bitwise-equal replicas on every
 * rank. */
nrc_status nrc_train_backward(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n_local,
                              float* d_grad, float* d_loss_sum, float* d_pred, void* stream);
nrc_status nrc_train_apply(nrc_handle* h, const float* d_grad_sum, uint32_t n_global, const float* d_loss_sum,
                           float* d_loss, void* stream);

/* A frame's training: records are shuffled by the LCG
 * permutation of nrc_lcg_params(n_total, shuffle_seed) (R15) and split into
 * s disjoint batches of l records (P:L350 footnote); batch j is records
 * perm(j*l + k), k < l, gathered inside the kernel (nothing materialised).
 * If s*l > n_total, l shrinks to n_total / s.  d_losses: s fp32
 * (optional).  Equivalent (bitwise) to s nrc_train_step calls on the
 * gathered batches; two launches per step. */
nrc_status nrc_train_frame(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n_total, uint32_t s,
                           uint32_t l, uint64_t shuffle_seed, float* d_losses, void* stream);

/* Data-parallel shard of batch j of a frame (multi-GPU nrc_train_frame): the
 * un-normalised gradient sum and loss sum over records perm(j*l + k) for
 * row_begin <= k < row_end, with perm the LCG permutation of
 * nrc_lcg_params(n_total, shuffle_seed), gathered in-kernel.  Rank r of P
 * takes k in [r*l/P, (r+1)*l/P); all-reduce d_grad, then nrc_train_apply
 * with n_global = l.  d_grad / d_loss_sum as in nrc_train_backward. */
nrc_status nrc_train_frame_backward(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n_total,
                                    uint32_t l, uint64_t shuffle_seed, uint32_t j, uint32_t row_begin,
                                    uint32_t row_end, float* d_grad, float* d_loss_sum, void* stream);

/* Data-parallel frame training with the gradient all-reduce fused into the
 * optimiser over peer memory (SURVEY 8(e) mitigation 2, 8(f) N3 (ii); no NCCL
 * call).  `world` <= 8 ranks hold identically initialised caches and the
 * same (replicated) frame records d_rec / d_tgt (n_total records, shuffled
 * and split as in nrc_train_frame).  A step's l rows form T = ceil(l / 128)
 * tiles (T <= 128, i.e. l <= 16,384); rank r computes the fp32 gradient
 * partials of tiles [r T / world, (r+1) T / world) into its own state arena
 * (two slot halves by step parity), a one-thread hand-off kernel adds 1 to
 * every rank's counter (system-scope release; peer memory over NVLink) and
 * waits until all ranks have published the step, then the optimiser kernel
 * reduces the T tile partials in tile order straight from their owners'
 * arenas (peer loads) and applies Adam + EMA.  Every rank ends bitwise equal
 * to single-GPU nrc_train_frame on the same records (same tiles, same
 * partials, same summation order).  peer_state: host array of `world` device
 * pointers to every rank's state arena in rank order (this rank's own
 * d_state at index rank; peers' mapped with nrc_ipc_import).  All ranks must
 * make the same sequence of calls; the hand-off gives up after ~20 s
 * (counted by nrc_dp_timeouts) instead of hanging.  d_losses: s fp32
 * (optional).  NRC_ERR_UNSUPPORTED if T > 128. */
nrc_status nrc_train_frame_dp_peer(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n_total,
                                   uint32_t s, uint32_t l, uint64_t shuffle_seed, uint32_t rank, uint32_t world,
                                   void* const* peer_state, float* d_losses, void* stream);
/* Number of nrc_train_frame_dp_peer / nrc_peer_barrier hand-offs that timed
 * out (synchronous). */
nrc_status nrc_dp_timeouts(nrc_handle* h, uint64_t* count);

/* Data-parallel Adam + EMA step with the gradient all-reduce done in the
 * NVSwitch (NVLink SHARP; SURVEY 8(e) mitigation 2 / 8(f) N3 (ii); the step
 * of P:L896-902 on the batch of P:L491 split over the ranks).  mc_grad: the
 * MULTICAST address (16-byte aligned) of a buffer that every rank holds in
 * symmetric memory, laid out [logical gradient sum (nrc_param_count floats) |
 * loss sum (1 float)] as written by nrc_train_backward /
 * nrc_train_frame_backward.  The optimiser kernel reads every entry with
 * multimem.ld_reduce.add.f32 (the sum over all ranks' copies, fp32 in the
 * switch) and applies Adam + EMA on sum / n_global; d_loss (optional, 1
 * float) receives loss sum / n_global.  The caller orders the call after
 * every rank's gradient is written (nrc_peer_barrier) and keeps the buffer
 * untouched until every rank's call has completed (e.g. two buffers used by
 * step parity).  Not bitwise equal to single-GPU training (the switch's
 * summation order).  Increments the step counter. */
nrc_status nrc_train_apply_multimem(nrc_handle* h, const float* mc_grad, uint32_t n_global, float* d_loss,
                                    void* stream);

/* Data-parallel Adam + EMA step with the all-reduce folded into the
 * optimiser's loads over peer memory (SURVEY 8(e) mitigation 2 without NVLS;
 * P:L896-902 on the batch of P:L491 split over the ranks).  peer_bufs: host
 * array of `world` device pointers (16-byte aligned), rank order, each rank's
 * [logical gradient sum (nrc_param_count floats) | loss sum] as written by
 * nrc_train_frame_backward -- this rank's own buffer and its peers' (mapped
 * over NVLink, e.g. a symmetric-memory buffer).  Every gradient entry is
 * summed over the ranks in rank order, so every rank applies the same
 * gradient (replicas stay bitwise identical; not bitwise equal to one GPU,
 * the per-rank sums add in another order).  The caller orders the call after
 * every rank's buffer is written (nrc_peer_barrier) and keeps the buffers
 * untouched until every rank's call has completed (two buffer sets by step
 * parity).  d_loss (optional) receives the loss sum / n_global.  Increments
 * the step counter. */
nrc_status nrc_train_apply_peers(nrc_handle* h, const float* const* peer_bufs, uint32_t world, uint32_t n_global,
                                 float* d_loss, void* stream);

/* A single-process NVLS buffer on `device` (multicast object with this one
 * device bound; driver multicast support required, else
 * NRC_ERR_UNSUPPORTED): *d_uc = its ordinary (unicast) address, *d_mc = its
 * multicast address, both >= bytes (rounded up to the multicast
 * granularity), zero-filled.  For nrc_train_apply_multimem with one rank
 * (the code path of the N-rank NVLS step on a one-GPU system; N ranks use
 * symmetric memory from the framework, e.g. torch).  nrc_multicast_free
 * takes the unicast address. */
nrc_status nrc_multicast_alloc(int device, size_t bytes, void** d_uc, void** d_mc);
nrc_status nrc_multicast_free(void* d_uc);

/* Cross-rank barrier on the stream (one 32-thread kernel): adds 1 to every
 * rank's counter (system-scope release; peer_counters: `world` device
 * pointers, each rank's own u64 counter mapped into this process -- peer
 * memory over NVLink, e.g. a symmetric-memory buffer -- in rank order,
 * 8-byte aligned, zero before the first call) and waits until its own counter
 * (peer_counters[rank]) reaches world x (number of calls so far).  All ranks
 * must make the same sequence of calls; gives up after ~20 s (counted by
 * nrc_dp_timeouts) instead of hanging. */
nrc_status nrc_peer_barrier(nrc_handle* h, void* const* peer_counters, uint32_t rank, uint32_t world, void* stream);

/* CUDA IPC for nrc_train_frame_dp_peer.  nrc_ipc_export: the 64-byte handle of
 * the device allocation that contains d_ptr and d_ptr's offset in it;
 * nrc_ipc_import (another process): maps it, *d_ptr = mapped base + offset;
 * nrc_ipc_close: unmaps (pass the imported pointer and its offset).  A
 * process cannot import its own handle. */
nrc_status nrc_ipc_export(const void* d_ptr, uint8_t* handle, uint64_t* offset);
nrc_status nrc_ipc_import(const uint8_t* handle, uint64_t offset, void** d_ptr);
nrc_status nrc_ipc_close(void* d_ptr, uint64_t offset);

/* Host helper: the LCG constants of reading R15 (m = 2^ceil(log2 n), a = 1
 * mod 4, c odd, from the splitmix64 stream of seed). */
nrc_status nrc_lcg_params(uint64_t n, uint64_t seed, uint64_t* a, uint64_t* c, uint64_t* m);

/* The input encoding alone (Table 1 + padding):
 * d_out[64 i + j] = fp16 bits of feature j of record i (row-major, logical
 * order).  Same device function the fused kernels use. */
nrc_status nrc_encode(nrc_handle* h, const nrc_record* d_rec, uint64_t n, uint16_t* d_out, void* stream);

/* Self-training targets.  Training
 * path p owns vertices d_first[p] .. d_first[p] + d_len[p] - 1 (camera side
 * first); d_vert holds 9 fp32 per vertex: emitted radiance E, next-event
 * estimate N and throughput T towards the next vertex (RGB each).  d_tail:
 * 3 fp32 per path, the cache's radiance at the path's terminal vertex (e.g.
 * from nrc_query on the tail records); ignored for paths with bit 0 of
 * d_flags set (the unbiased fraction u = 1/16 terminated by Russian roulette
 * only).  Writes d_targets (3 fp32 per vertex):
 *   target(last) = E + N + T * tail,  target(v_i) = E_i + N_i + T_i * target(v_{i+1})
 * in fp32 (fmaf).  All pointers device, 4-byte aligned; vertex ranges must lie
 * in [0, n_vertices).  One kernel launch (one thread per path). */
nrc_status nrc_assemble_targets(nrc_handle* h, const uint32_t* d_first, const uint32_t* d_len,
                                const uint32_t* d_flags, uint32_t n_paths, const float* d_vert,
                                const float* d_tail, float* d_targets, void* stream);

/* Parameter I/O in the logical layout (nrc_param_count() fp32 host floats).
 * nrc_set_params(NRC_PARAMS_TRAIN) also refreshes the fp16 image of W;
 * nrc_set_params(NRC_PARAMS_EMA) refreshes the fp16 image of W-bar.
 * Synchronous. */
nrc_status nrc_get_params(nrc_handle* h, nrc_param_set which, float* h_out, size_t n);
nrc_status nrc_set_params(nrc_handle* h, nrc_param_set which, const float* h_in, size_t n);

/* Adam step count t, the non-finite counters (gradient entries zeroed,
 * records with a non-finite target masked) and the number of zero-length
 * direction / normal vectors encoded so far by queries, training and
 * nrc_encode (read as (0,0,1)).  Any output may be
 * NULL.  Synchronous. */
nrc_status nrc_get_stats(nrc_handle* h, uint64_t* step, uint64_t* nonfinite_grads, uint64_t* nonfinite_targets,
                         uint64_t* degenerate_vectors);

/* 20,672 at width 64 (5*64*64 + 3*64; reading R1). */
size_t nrc_param_count(const nrc_handle* h);

const char* nrc_status_string(nrc_status s);
const char* nrc_last_error(const nrc_handle* h);

/* End-to-end frame with HOST buffers (for pinned host memory): copies the
 * query records and the training records/targets into d_scratch (at least
 * nrc_frame_scratch_bytes(n_query, n_train) bytes of device memory), runs
 * nrc_query (EMA weights from before this frame's training) and
 * nrc_train_frame, and copies the radiance (3 n_query fp32) and the s losses
 * back.  Asynchronous on `stream`; the caller synchronises. */
size_t nrc_frame_scratch_bytes(uint64_t n_query, uint32_t n_train);
nrc_status nrc_frame_host(nrc_handle* h, const nrc_record* h_query, uint64_t n_query, float* h_rgb,
                          const nrc_record* h_train, const float* h_tgt, uint32_t n_train, uint32_t s, uint32_t l,
                          uint64_t shuffle_seed, float* h_losses, void* d_scratch, size_t scratch_bytes,
                          void* stream);

/* Diagnostic: one tcgen05 tile product in each operand layout the kernels
 * use, on plain row-major fp16 inputs (mode 0: D[128x64] = A[128x64] B[64x64]^T;
 * mode 1: D[128x64] = A[128x64] B[64x64]; mode 2: D[64x64] = A[128x64]^T
 * B[128x64]; mode 3: D[128x16] = A[128x64] B[16x64]^T; mode 4: as mode 0 with
 * A read from tensor memory).  D is fp32
 * row-major.  Synchronous. */
nrc_status nrc_selftest_umma(int mode, const uint16_t* d_a, const uint16_t* d_b, float* d_d);

/* Number of kernel launches the most recent call on this handle enqueued
 * (used by bench.py to report gpu_launches). */
uint32_t nrc_last_launch_count(const nrc_handle* h);

#ifdef __cplusplus
}
#endif

#endif /* NRC_H_ */
