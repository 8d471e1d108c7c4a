// nrc_api.cu -- host side of libnrc: the C ABI declared in include/nrc.h.
// Argument validation, state-arena layout, launch configuration.  All
// arithmetic of the method runs in the kernels of nrc_kernels.cuh.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "nrc.h"
#include "nrc_kernels.cuh"

using namespace nrc;

namespace {

// Query-kernel launchers: the TMEM-activation kernel with G
// tile groups per CTA and one tile in flight per group, per width / encoding.
struct QueryEntry {
    cudaError_t (*set_smem)();
    void (*launch)(int, const QueryArgs&, cudaStream_t);
    int groups;
};
// One TMEM-activation configuration per width and encoding (N4):
// G groups; the paper's depth (5 hidden layers) is compiled straight-line, the
// depth variants (N4) run the same kernel with a run-time layer loop.
template <int G, int W, bool EXACT = false>
struct QueryLauncherW {
    static cudaError_t set_smem() {
        const int bytes = query_ts_smem_bytes_nh<G, W>(TrainW<W>::kMaxNh);
        cudaError_t e = cudaFuncSetAttribute(nrc_query_ts_kernel<G, W, 5, EXACT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) return e;
        return cudaFuncSetAttribute(nrc_query_ts_kernel<G, W, 0, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    bytes);
    }
    static void launch(int grid, const QueryArgs& qa, cudaStream_t st) {
        const int smem = query_ts_smem_bytes_nh<G, W>(int(qa.nh));
        if (qa.nh == 5)
            nrc_query_ts_kernel<G, W, 5, EXACT><<<grid, 128 * G, smem, st>>>(qa);
        else
            nrc_query_ts_kernel<G, W, 0, EXACT><<<grid, 128 * G, smem, st>>>(qa);
    }
};
#ifndef NRC_Q64_G
#define NRC_Q64_G 5
#endif
const QueryEntry kQuery64 = {&QueryLauncherW<NRC_Q64_G, 64>::set_smem, &QueryLauncherW<NRC_Q64_G, 64>::launch, NRC_Q64_G};
const QueryEntry kQueryExact = {&QueryLauncherW<5, 64, true>::set_smem, &QueryLauncherW<5, 64, true>::launch, 5};
#ifndef NRC_W32_G
#define NRC_W32_G 7  // 7 groups: 82 us vs 90 us with 5 at 1080p (round 1, 5 / 7 groups at width 32)
#endif
const QueryEntry kQueryW32 = {&QueryLauncherW<NRC_W32_G, 32>::set_smem, &QueryLauncherW<NRC_W32_G, 32>::launch,
                              NRC_W32_G};
const QueryEntry kQueryW128 = {&QueryLauncherW<2, 128>::set_smem, &QueryLauncherW<2, 128>::launch, 2};
constexpr int kMaxPartials = 256; // train-kernel grid cap (>= SM count)

// Runtime view of NetRt<W> (nrc_device.cuh) for the host code: width W,
// nh hidden layers (layers 0..nh, nh = the output layer).
constexpr int kMaxLayers = 9;  // nh <= 8
struct WidthInfo {
    int W = 64, nh = 5, padded = 0, logical = 0, img = 0;
    int pad_off[kMaxLayers + 1] = {}, rows[kMaxLayers] = {}, cols[kMaxLayers] = {};
};
template <int W>
WidthInfo width_info_t(int nh) {
    const NetRt<W> D(nh);
    WidthInfo w;
    w.W = W;
    w.nh = nh;
    w.padded = D.padded();
    w.logical = D.logical();
    w.img = D.img();
    for (int i = 0; i <= nh + 1; ++i) w.pad_off[i] = D.pad_off(i);
    for (int i = 0; i <= nh; ++i) {
        w.rows[i] = i < nh ? W : 3;  // logical rows (the output layer has 3)
        w.cols[i] = D.cols(i);
    }
    return w;
}
bool width_supported(uint32_t W) { return W == 32 || W == 64 || W == 128; }
// depth variants: 1..TrainW<W>::kMaxNh hidden layers (shared memory of the training kernel)
int max_hidden_layers(uint32_t W) {
    return W == 32 ? TrainW<32>::kMaxNh : W == 128 ? TrainW<128>::kMaxNh : TrainW<64>::kMaxNh;
}
WidthInfo width_info(int W, int nh) {
    return W == 32 ? width_info_t<32>(nh) : W == 128 ? width_info_t<128>(nh) : width_info_t<64>(nh);
}

struct StateLayout {
    size_t w, m, v, ema, wimg, eimg, partials, loss_part, counters, dp_tables, peer_tab, total;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

StateLayout layout(int W, int nh) {
    const WidthInfo wi = width_info(W, nh);
    StateLayout L{};
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t at = o;
        o = align_up(o + bytes, 256);
        return at;
    };
    const size_t pf = sizeof(float) * size_t(wi.padded);
    L.w = take(pf);
    L.m = take(pf);
    L.v = take(pf);
    L.ema = take(pf);
    L.wimg = take(size_t(wi.img));
    L.eimg = take(size_t(wi.img));
    // training scratch: per-CTA fp32 gradient partials (padded layout of the width)
    L.partials = take(sizeof(float) * size_t(wi.padded) * kMaxPartials);
    L.loss_part = take(sizeof(float) * kMaxPartials);
    // [0] non-finite gradients, [1] non-finite targets, [2] zero-length
    // omega / n vectors encoded, [4] fused peer all-reduce hand-off, [5] its timeouts
    L.counters = take(sizeof(unsigned long long) * 8);
    // nrc_train_frame_dp_peer: per step parity, kMaxDpTiles partial + loss pointers
    L.dp_tables = take(sizeof(const float*) * 2 * 2 * kMaxDpTiles);
    // nrc_train_apply_peers: two tables of kMaxRanks peer-buffer pointers
    L.peer_tab = take(sizeof(const float*) * 2 * kMaxRanks);
    L.total = o;
    return L;
}

uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

}  // namespace

struct nrc_handle {
    nrc_config cfg;
    uint8_t* state;
    StateLayout L;
    int num_sms;
    uint64_t step;
    EncodeParams ep;
    std::string err;
    uint32_t launches;
    long long* dbg = nullptr;  // diagnostics only (nrc_debug_set_trace)
    unsigned long long dp_expect = 0;  // hand-off counter value after the last nrc_train_frame_dp_peer step
    unsigned long long bar_expect = 0; // nrc_peer_barrier: this rank's counter value after the last barrier
    // nrc_train_apply_peers: host copies of the two device pointer tables
    const float* peer_tab_host[2][kMaxRanks] = {};
    uint32_t peer_tab_world[2] = {0, 0};
    int peer_tab_next = 0;
    uint64_t dp_seq = 0;               // steps done by nrc_train_frame_dp_peer (partial-slot parity)
    WidthInfo wi;                 // hidden width (64 unless the C4 width ablation)
    int query_ctas = 0;           // cap on the query grid (0: all SMs)
    bool train_legacy = false;    // NRC_TRAIN_LEGACY=1: nrc_train_w_kernel for one-tile batches too
    // nrc_train_frame as one CUDA graph (2 s kernel nodes with programmatic
    // edges), captured once per (rows per step, steps) and replayed with the
    // per-call arguments; NRC_TRAIN_GRAPH=0 launches on the stream instead
    bool train_graph = true;
    struct TrainGraph {
        uint32_t n = 0, nsteps = 0;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        std::vector<cudaGraphNode_t> nodes;  // P_0, A_0, P_1, A_1, ...
    } tgraph;
    cudaStream_t capture = nullptr;
    int train_ctas = 0;           // cap on the train grid (0: one CTA per tile up to all SMs)
    // nrc_frame_host pipelining: host->device and device->host copy streams and events
    cudaStream_t copy_in = nullptr, copy_out = nullptr;
    std::vector<cudaEvent_t> events;
    ~nrc_handle() {
        if (tgraph.exec) cudaGraphExecDestroy(tgraph.exec);
        if (tgraph.graph) cudaGraphDestroy(tgraph.graph);
        if (capture) cudaStreamDestroy(capture);
        for (cudaEvent_t e : events) cudaEventDestroy(e);
        if (copy_in) cudaStreamDestroy(copy_in);
        if (copy_out) cudaStreamDestroy(copy_out);
    }
    cudaEvent_t event(size_t i) {  // lazily created, reused across frames
        while (events.size() <= i) {
            cudaEvent_t e = nullptr;
            cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            events.push_back(e);
        }
        return events[i];
    }
    float* d_w() { return reinterpret_cast<float*>(state + L.w); }
    float* d_m() { return reinterpret_cast<float*>(state + L.m); }
    float* d_v() { return reinterpret_cast<float*>(state + L.v); }
    float* d_ema() { return reinterpret_cast<float*>(state + L.ema); }
    uint8_t* d_wimg() { return state + L.wimg; }
    uint8_t* d_eimg() { return state + L.eimg; }
    float* d_partials() { return reinterpret_cast<float*>(state + L.partials); }
    float* d_loss_part() { return reinterpret_cast<float*>(state + L.loss_part); }
    unsigned long long* d_counters() { return reinterpret_cast<unsigned long long*>(state + L.counters); }
};

static nrc_status fail(nrc_handle* h, nrc_status s, const std::string& msg) {
    if (h) h->err = msg;
    return s;
}
static nrc_status cuda_check(nrc_handle* h, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return NRC_OK;
    return fail(h, NRC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define NRC_CUDA(h, call)                                          \
    do {                                                           \
        nrc_status _s = cuda_check((h), (call), #call);            \
        if (_s != NRC_OK) return _s;                               \
    } while (0)
#define NRC_LAUNCHED(h, what)                                      \
    do {                                                           \
        nrc_status _s = cuda_check((h), cudaGetLastError(), what); \
        if (_s != NRC_OK) return _s;                               \
        ++(h)->launches;                                           \
    } while (0)

static bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// Launch with programmatic dependent launch (PDL): the kernel may start while
// its predecessor in the stream drains; it calls griddepcontrol.wait before
// touching anything the predecessor writes.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}
template <int W>
static void launch_images(nrc_handle* h, cudaStream_t st) {
    const int blocks = (h->wi.padded + 255) / 256;
    nrc_image_w_kernel<W><<<blocks, 256, 0, st>>>(h->d_w(), h->d_wimg(), h->wi.nh);
    nrc_image_w_kernel<W><<<blocks, 256, 0, st>>>(h->d_ema(), h->d_eimg(), h->wi.nh);
}

extern "C" {

void nrc_default_config(nrc_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof(*c));
    c->abi_version = NRC_ABI_VERSION;
    c->hidden_width = 64;
    c->n_hidden_layers = 5;
    c->max_batch = 3840u * 2160u;
    for (int i = 0; i < 3; ++i) {
        c->aabb_min[i] = 0.0f;
        c->aabb_max[i] = 1.0f;
    }
    c->learning_rate = 1e-2f;
    c->adam_beta1 = 0.9f;
    c->adam_beta2 = 0.99f;
    c->adam_eps = 1e-8f;
    c->loss_eps = 0.01f;
    c->ema_alpha = 0.99f;
    c->flags = NRC_FACTORIZE | NRC_CLAMP_QUERY;
    c->seed = 1;
    c->device = 0;
}

static nrc_status validate_config(const nrc_config* c, std::string* why) {
    if (!c) {
        *why = "config is NULL";
        return NRC_ERR_INVALID_ARGUMENT;
    }
    if (c->abi_version != NRC_ABI_VERSION) {
        *why = "ABI version mismatch";
        return NRC_ERR_UNSUPPORTED;
    }
    if ((c->flags & NRC_EXACT_ENCODING) && c->hidden_width != 64) {
        *why = "NRC_EXACT_ENCODING is built for hidden_width 64";
        return NRC_ERR_UNSUPPORTED;
    }
    if (!width_supported(c->hidden_width)) {
        *why = "hidden_width must be 32, 64 (P:L694) or 128 (width ablation)";
        return NRC_ERR_UNSUPPORTED;
    }
    if (c->n_hidden_layers < 1 || int(c->n_hidden_layers) > max_hidden_layers(c->hidden_width)) {
        *why = "n_hidden_layers must be 5 (P:L694) or, for the depth variants, 1..8 / 1..7 / 1..5 at width 32 / 64 / 128";
        return NRC_ERR_UNSUPPORTED;
    }
    if (c->max_batch == 0 || c->max_batch > (1ull << 40)) {
        *why = "max_batch must be in [1, 2^40]";
        return NRC_ERR_INVALID_ARGUMENT;
    }
    for (int i = 0; i < 3; ++i) {
        const float ext = c->aabb_max[i] - c->aabb_min[i];
        if (!(ext > 0.0f) || !std::isfinite(ext)) {
            *why = "degenerate AABB";
            return NRC_ERR_INVALID_ARGUMENT;
        }
    }
    if (!(c->learning_rate > 0.0f) || !(c->adam_beta1 >= 0.0f && c->adam_beta1 < 1.0f) ||
        !(c->adam_beta2 >= 0.0f && c->adam_beta2 < 1.0f) || !(c->adam_eps >= 0.0f) || !(c->loss_eps > 0.0f) ||
        !(c->ema_alpha >= 0.0f && c->ema_alpha < 1.0f)) {
        *why = "optimiser hyper-parameter out of range";
        return NRC_ERR_INVALID_ARGUMENT;
    }
    return NRC_OK;
}

size_t nrc_state_bytes(const nrc_config* cfg) {
    std::string why;
    if (validate_config(cfg, &why) != NRC_OK) return 0;
    return layout(int(cfg->hidden_width), int(cfg->n_hidden_layers)).total;
}

const char* nrc_status_string(nrc_status s) {
    switch (s) {
        case NRC_OK: return "NRC_OK";
        case NRC_ERR_INVALID_ARGUMENT: return "NRC_ERR_INVALID_ARGUMENT";
        case NRC_ERR_UNSUPPORTED: return "NRC_ERR_UNSUPPORTED";
        case NRC_ERR_OUT_OF_MEMORY: return "NRC_ERR_OUT_OF_MEMORY";
        case NRC_ERR_CUDA: return "NRC_ERR_CUDA";
        case NRC_ERR_NCCL: return "NRC_ERR_NCCL";
        case NRC_ERR_STATE: return "NRC_ERR_STATE";
    }
    return "NRC_ERR_UNKNOWN";
}

const char* nrc_last_error(const nrc_handle* h) { return h ? h->err.c_str() : "NULL handle"; }
uint32_t nrc_last_launch_count(const nrc_handle* h) { return h ? h->launches : 0; }
size_t nrc_param_count(const nrc_handle* h) { return h ? size_t(h->wi.logical) : size_t(kParamLogical); }

nrc_status nrc_lcg_params(uint64_t n, uint64_t seed, uint64_t* a, uint64_t* c, uint64_t* m) {
    if (!a || !c || !m || n == 0) return NRC_ERR_INVALID_ARGUMENT;
    uint64_t mm = 1;
    while (mm < n) mm <<= 1;
    const uint64_t x0 = splitmix64(seed), x1 = splitmix64(seed + 0x9E3779B97F4A7C15ull);
    uint64_t aa = ((x0 & (mm - 1)) & ~uint64_t(3)) | 1u;
    if (mm >= 8 && aa == 1) aa = 5;
    *a = aa;
    *c = (x1 & (mm - 1)) | 1u;
    *m = mm;
    return NRC_OK;
}

static nrc_status refresh_images(nrc_handle* h, cudaStream_t st) {
    if (h->wi.W == 32)
        launch_images<32>(h, st);
    else if (h->wi.W == 128)
        launch_images<128>(h, st);
    else
        launch_images<64>(h, st);
    nrc_status s = cuda_check(h, cudaGetLastError(), "nrc_image_w_kernel");
    if (s == NRC_OK) h->launches += 2;
    return s;
}

nrc_status nrc_init(const nrc_config* cfg, void* d_state, size_t state_bytes, nrc_handle** out) {
    std::string why;
    if (!out) return NRC_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    nrc_status s = validate_config(cfg, &why);
    if (s != NRC_OK) {
        std::fprintf(stderr, "nrc_init: %s\n", why.c_str());
        return s;
    }
    const StateLayout L = layout(int(cfg->hidden_width), int(cfg->n_hidden_layers));
    if (!d_state || !aligned(d_state, 256)) return NRC_ERR_INVALID_ARGUMENT;
    if (state_bytes < L.total) return NRC_ERR_OUT_OF_MEMORY;

    nrc_handle* h = new nrc_handle();
    h->cfg = *cfg;
    h->state = static_cast<uint8_t*>(d_state);
    h->L = L;
    h->wi = width_info(int(cfg->hidden_width), int(cfg->n_hidden_layers));
    h->step = 0;
    h->launches = 0;
    for (int i = 0; i < 3; ++i) {
        // reading R3: inv = fp32(1 / fp32(hi - lo))
        volatile float ext = cfg->aabb_max[i] - cfg->aabb_min[i];
        volatile float inv = 1.0f / ext;
        h->ep.lo[i] = cfg->aabb_min[i];
        h->ep.inv[i] = inv;
    }
    h->ep.exact = (cfg->flags & NRC_EXACT_ENCODING) ? 1u : 0u;
    auto bail = [&](nrc_status st) {
        std::fprintf(stderr, "nrc_init: %s\n", h->err.c_str());
        delete h;
        return st;
    };
    if ((s = cuda_check(h, cudaSetDevice(cfg->device), "cudaSetDevice")) != NRC_OK) return bail(s);
    if ((s = cuda_check(h, cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, cfg->device),
                        "cudaDeviceGetAttribute")) != NRC_OK)
        return bail(s);
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, cfg->device);
    if (major != 10) {
        h->err = "libnrc is built for sm_100a (B200); device compute capability major = " + std::to_string(major);
        return bail(NRC_ERR_UNSUPPORTED);
    }
    // diagnostics / probes only: cap the query or train grid
    if (const char* e = std::getenv("NRC_QUERY_CTAS")) h->query_ctas = std::atoi(e);
    if (const char* e = std::getenv("NRC_TRAIN_CTAS")) h->train_ctas = std::atoi(e);
    // diagnostics / A-B only: the single-schedule partials kernel for every batch
    if (const char* e = std::getenv("NRC_TRAIN_LEGACY")) h->train_legacy = std::atoi(e) != 0;
    if (const char* e = std::getenv("NRC_TRAIN_GRAPH")) h->train_graph = std::atoi(e) != 0;
    if ((s = cuda_check(h, kQuery64.set_smem(), "cudaFuncSetAttribute(query)")) != NRC_OK) return bail(s);
    if ((s = cuda_check(h, kQueryW32.set_smem(), "cudaFuncSetAttribute(query w32)")) != NRC_OK) return bail(s);
    if ((s = cuda_check(h, kQueryW128.set_smem(), "cudaFuncSetAttribute(query w128)")) != NRC_OK) return bail(s);
    if ((s = cuda_check(h, kQueryExact.set_smem(), "cudaFuncSetAttribute(query exact)")) != NRC_OK) return bail(s);
    if ((s = cuda_check(h, cudaFuncSetAttribute(nrc_train_w_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                TrainW<32>::smem_bytes(TrainW<32>::kMaxNh)),
                        "cudaFuncSetAttribute(train w32)")) != NRC_OK ||
        (s = cuda_check(h, cudaFuncSetAttribute(nrc_train_w_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                TrainW<64>::smem_bytes(TrainW<64>::kMaxNh)),
                        "cudaFuncSetAttribute(train w64)")) != NRC_OK ||
        (s = cuda_check(h, cudaFuncSetAttribute(nrc_train_w_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                TrainW<128>::smem_bytes(TrainW<128>::kMaxNh)),
                        "cudaFuncSetAttribute(train w128)")) != NRC_OK ||
        (s = cuda_check(h, cudaFuncSetAttribute(nrc_train_w_kernel<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                TrainW<64>::smem_bytes(TrainW<64>::kMaxNh)),
                        "cudaFuncSetAttribute(train w64 exact)")) != NRC_OK ||
        (s = cuda_check(h, cudaFuncSetAttribute(nrc_train_ws_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                TrainWs<32>::smem_bytes(TrainWs<32>::kMaxNh)),
                        "cudaFuncSetAttribute(train ws32)")) != NRC_OK ||
        (s = cuda_check(h, cudaFuncSetAttribute(nrc_train_ws_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                TrainWs<64>::smem_bytes(TrainWs<64>::kMaxNh)),
                        "cudaFuncSetAttribute(train ws64)")) != NRC_OK ||
        (s = cuda_check(h, cudaFuncSetAttribute(nrc_train_ws_kernel<64, true>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                TrainWs<64>::smem_bytes(TrainWs<64>::kMaxNh)),
                        "cudaFuncSetAttribute(train ws64 exact)")) != NRC_OK)
        return bail(s);

    // Glorot-uniform init from the counter-based splitmix64 stream (R16):
    // counter (layer << 32 | r * fan_in + c), bound sqrt(6 / (fan_in + fan_out)).
    const WidthInfo& wi = h->wi;
    std::vector<float> w(size_t(wi.padded), 0.0f);
    for (int i = 0; i <= wi.nh; ++i) {  // layer wi.nh is the output layer
        const int rows = wi.rows[i], cols = wi.cols[i];
        const double bound = std::sqrt(6.0 / (double(cols) + double(rows)));
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) {
                const uint64_t ctr = (uint64_t(i) << 32) | uint64_t(r * cols + c);
                const double u = double(splitmix64(cfg->seed ^ ctr) >> 11) * (1.0 / 9007199254740992.0);
                w[size_t(wi.pad_off[i]) + size_t(r) * cols + c] = float((2.0 * u - 1.0) * bound);
            }
    }
    const size_t pf = sizeof(float) * size_t(wi.padded);
    if ((s = cuda_check(h, cudaMemset(h->state, 0, L.total), "cudaMemset(state)")) != NRC_OK) return bail(s);
    if ((s = cuda_check(h, cudaMemcpy(h->d_w(), w.data(), pf, cudaMemcpyHostToDevice), "cudaMemcpy(w)")) != NRC_OK)
        return bail(s);
    if ((s = cuda_check(h, cudaMemcpy(h->d_ema(), w.data(), pf, cudaMemcpyHostToDevice), "cudaMemcpy(ema)")) != NRC_OK)
        return bail(s);
    if ((s = refresh_images(h, 0)) != NRC_OK) return bail(s);
    if ((s = cuda_check(h, cudaDeviceSynchronize(), "nrc_init sync")) != NRC_OK) return bail(s);
    *out = h;
    return NRC_OK;
}

nrc_status nrc_destroy(nrc_handle* h) {
    delete h;
    return NRC_OK;
}

static nrc_status check_train_width(nrc_handle* h) {
    if (width_supported(uint32_t(h->wi.W))) return NRC_OK;
    return fail(h, NRC_ERR_UNSUPPORTED, "unsupported hidden width for training");
}
static nrc_status check_handle(nrc_handle* h) {
    if (!h || !h->state) return NRC_ERR_STATE;
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != h->cfg.device) return cuda_check(h, cudaSetDevice(h->cfg.device), "cudaSetDevice");
    return NRC_OK;
}

static nrc_status query_impl(nrc_handle* h, const nrc_record* d_rec, uint64_t n, float* d_rgb, const uint32_t* d_pix,
                             const float* d_thr, float* d_image, void* stream) {
    QueryArgs qa{};
    qa.rec = reinterpret_cast<const float*>(d_rec);
    qa.out = d_rgb;
    qa.n = n;
    const bool raw = (h->cfg.flags & NRC_QUERY_RAW_WEIGHTS) || h->cfg.ema_alpha == 0.0f;
    qa.wimg = raw ? h->d_wimg() : h->d_eimg();
    qa.ep = h->ep;
    qa.flags = h->cfg.flags & (NRC_FACTORIZE | NRC_CLAMP_QUERY);
    qa.dbg = h->dbg;
    qa.pix = d_pix;
    qa.thr = d_thr;
    qa.image = d_image;
    qa.nh = uint32_t(h->wi.nh);
    qa.degenerate = h->d_counters() + 2;
    const QueryEntry& qe = h->ep.exact        ? kQueryExact
                           : h->wi.W == 32   ? kQueryW32
                           : h->wi.W == 128  ? kQueryW128
                                             : kQuery64;
    const uint64_t ntiles = (n + kTile - 1) / kTile;
    const uint64_t G = uint64_t(qe.groups);
    const uint64_t ctas = (ntiles + G - 1) / G;  // one tile stream per group
    const uint64_t cap = h->query_ctas > 0 && h->query_ctas < h->num_sms ? uint64_t(h->query_ctas) : uint64_t(h->num_sms);
    const int grid = int(ctas < cap ? ctas : cap);
    qe.launch(grid, qa, static_cast<cudaStream_t>(stream));
    NRC_LAUNCHED(h, "nrc_query_ts_kernel");
    return NRC_OK;
}

nrc_status nrc_query(nrc_handle* h, const nrc_record* d_rec, uint64_t n, float* d_rgb, void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    h->launches = 0;
    if (n == 0) return NRC_OK;
    if (!d_rec || !d_rgb || !aligned(d_rec, 16) || !aligned(d_rgb, 4))
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_query: NULL or misaligned pointer");
    if (n > h->cfg.max_batch) return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_query: n > max_batch");
    return query_impl(h, d_rec, n, d_rgb, nullptr, nullptr, nullptr, stream);
}

nrc_status nrc_query_accumulate(nrc_handle* h, const nrc_record* d_rec, uint64_t n, const uint32_t* d_pixel,
                                const float* d_thr, float* d_image, void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    h->launches = 0;
    if (n == 0) return NRC_OK;
    if (!d_rec || !d_pixel || !d_thr || !d_image || !aligned(d_rec, 16) || !aligned(d_pixel, 4) ||
        !aligned(d_thr, 4) || !aligned(d_image, 4))
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_query_accumulate: NULL or misaligned pointer");
    if (n > h->cfg.max_batch) return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_query_accumulate: n > max_batch");
    return query_impl(h, d_rec, n, nullptr, d_pixel, d_thr, d_image, stream);
}

struct Gather {
    bool on;
    uint64_t a, c, m, n, offset;
};

// Adam bias corrections and EMA coefficients of optimisation step t >= 1
static StepCoef step_coef(const nrc_config& c, uint64_t t) {
    StepCoef k{};
    k.inv_bc1 = float(1.0 / (1.0 - std::pow(double(c.adam_beta1), double(t))));
    k.inv_bc2 = float(1.0 / (1.0 - std::pow(double(c.adam_beta2), double(t))));
    // Eq.(2): eta_t = 1 - a^t.  R12: W-bar = [(1-a) W + a eta_{t-1} W-bar] / eta_t
    const double al = c.ema_alpha;
    const double eta_t = 1.0 - std::pow(al, double(t));
    const double eta_p = 1.0 - std::pow(al, double(t - 1));
    if (al == 0.0) {
        k.ema_c1 = 1.0f;
        k.ema_c2 = 0.0f;
    } else if (c.flags & NRC_EMA_PRINTED_FORM) {
        k.ema_c1 = float((1.0 - al) / eta_t);
        k.ema_c2 = float(al * eta_p);
    } else {
        k.ema_c1 = float((1.0 - al) / eta_t);
        k.ema_c2 = float(al * eta_p / eta_t);
    }
    return k;
}

static TrainArgs train_args(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n,
                            const Gather& gth) {
    TrainArgs ta{};
    ta.rec = reinterpret_cast<const float*>(d_rec);
    ta.tgt = d_tgt;
    ta.n = n;
    ta.gather = gth.on ? 1u : 0u;
    ta.lcg_a = gth.a;
    ta.lcg_c = gth.c;
    ta.lcg_m = gth.m;
    ta.lcg_n = gth.n;
    ta.offset = gth.offset;
    ta.wimg = h->d_wimg();
    ta.ep = h->ep;
    ta.flags = h->cfg.flags & NRC_FACTORIZE;
    ta.loss_eps = h->cfg.loss_eps;
    ta.partials = h->d_partials();
    ta.loss_part = h->d_loss_part();
    ta.bad_targets = h->d_counters() + 1;
    ta.degenerate = h->d_counters() + 2;
    ta.dbg = h->dbg;
    ta.nh = uint32_t(h->wi.nh);
    return ta;
}
static int train_grid(const nrc_handle* h, uint32_t n) {
    const uint32_t ntiles = (n + kTile - 1) / kTile;
    int grid = int(ntiles);
    int cap = h->num_sms < kMaxPartials ? h->num_sms : kMaxPartials;
    if (h->train_ctas > 0 && h->train_ctas < cap) cap = h->train_ctas;
    return grid > cap ? cap : grid;
}
// The partials kernel for this handle's width / encoding, one tile per CTA up to `grid`.
static cudaError_t launch_train_w_grid(nrc_handle* h, const TrainArgs& ta, int grid, cudaStream_t st) {
    const int nh = h->wi.nh;
    // one tile per CTA at width <= 64, depth <= 6: the split schedule
    // (nrc_train_ws_kernel, wgrads off the backward critical path)
    const bool one_tile = uint64_t(grid) * kTile >= uint64_t(ta.n);
    if (one_tile && nh <= TrainWs<64>::kMaxNh && h->wi.W <= 64 && !h->train_legacy) {
        if (h->wi.W == 32)
            return launch_pdl(nrc_train_ws_kernel<32>, dim3(grid), dim3(TrainWs<32>::kThreads),
                              TrainWs<32>::smem_bytes(nh), st, ta);
        if (h->ep.exact)
            return launch_pdl(nrc_train_ws_kernel<64, true>, dim3(grid), dim3(TrainWs<64>::kThreads),
                              TrainWs<64>::smem_bytes(nh), st, ta);
        return launch_pdl(nrc_train_ws_kernel<64>, dim3(grid), dim3(TrainWs<64>::kThreads), TrainWs<64>::smem_bytes(nh),
                          st, ta);
    }
    if (h->wi.W == 32)
        return launch_pdl(nrc_train_w_kernel<32>, dim3(grid), dim3(128), TrainW<32>::smem_bytes(nh), st, ta);
    if (h->wi.W == 128)
        return launch_pdl(nrc_train_w_kernel<128>, dim3(grid), dim3(128), TrainW<128>::smem_bytes(nh), st, ta);
    if (h->ep.exact)  // NRC_EXACT_ENCODING (width 64 only, validate_config)
        return launch_pdl(nrc_train_w_kernel<64, true>, dim3(grid), dim3(128), TrainW<64>::smem_bytes(nh), st, ta);
    return launch_pdl(nrc_train_w_kernel<64>, dim3(grid), dim3(128), TrainW<64>::smem_bytes(nh), st, ta);
}
// One step's partials over n rows.
static nrc_status launch_train_w(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n,
                                 const Gather& gth, cudaStream_t st, int* nparts, float* d_pred = nullptr) {
    TrainArgs ta = train_args(h, d_rec, d_tgt, n, gth);
    ta.pred = d_pred;
    if (h->dbg) ta.dbg = h->dbg + 4096 * (h->step % 4);  // diagnostics: one 4096-slot block per step
    const int grid = train_grid(h, n);
    *nparts = grid;
    NRC_CUDA(h, launch_train_w_grid(h, ta, grid, st));
    NRC_LAUNCHED(h, "nrc_train_w_kernel");
    return NRC_OK;
}
static AdamWArgs adam_w_args(nrc_handle* h) {
    AdamWArgs aa{};
    const nrc_config& c = h->cfg;
    aa.w = h->d_w();
    aa.m = h->d_m();
    aa.v = h->d_v();
    aa.ema = h->d_ema();
    aa.wimg = h->d_wimg();
    aa.eimg = h->d_eimg();
    aa.lr = c.learning_rate;
    aa.b1 = c.adam_beta1;
    aa.b2 = c.adam_beta2;
    aa.eps = c.adam_eps;
    const StepCoef k = step_coef(c, h->step);  // already incremented
    aa.inv_bc1 = k.inv_bc1;
    aa.inv_bc2 = k.inv_bc2;
    aa.ema_c1 = k.ema_c1;
    aa.ema_c2 = k.ema_c2;
    aa.bad_grads = h->d_counters() + 0;
    aa.loss_part = h->d_loss_part();
    if (h->dbg) aa.dbg = h->dbg + 4096 * ((h->step + 3) % 4);  // the step's block (step already incremented)
    aa.nh = h->wi.nh;
    return aa;
}
static nrc_status launch_adam_w(nrc_handle* h, const AdamWArgs& aa, cudaStream_t st) {
    const dim3 grid(unsigned(h->wi.padded / 128)), block(kAdamThreads);  // 128 parameters per block
    if (h->wi.W == 32)
        NRC_CUDA(h, launch_pdl(nrc_adam_w_kernel<32>, grid, block, 0, st, aa));
    else if (h->wi.W == 128)
        NRC_CUDA(h, launch_pdl(nrc_adam_w_kernel<128>, grid, block, 0, st, aa));
    else
        NRC_CUDA(h, launch_pdl(nrc_adam_w_kernel<64>, grid, block, 0, st, aa));
    NRC_LAUNCHED(h, "nrc_adam_w_kernel");
    return NRC_OK;
}

// nsteps optimisation steps of n rows each (step k gathers rows offset + k n
// when gathering): per step the partials kernel, then reduce + Adam + EMA.
static nrc_status train_steps_graph(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n,
                                    const Gather& gth, float* d_losses, uint32_t nsteps, cudaStream_t st);
static nrc_status train_steps(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n,
                              const Gather& gth, float* d_losses, uint32_t nsteps, cudaStream_t st) {
    if (nsteps >= 2 && h->train_graph && !h->dbg) return train_steps_graph(h, d_rec, d_tgt, n, gth, d_losses, nsteps, st);
    uint32_t launches = 0;
    for (uint32_t k = 0; k < nsteps; ++k) {
        Gather g = gth;
        g.offset = gth.offset + uint64_t(k) * n;
        int np = 0;
        nrc_status s = launch_train_w(h, d_rec, d_tgt, n, g, st, &np);
        if (s != NRC_OK) return s;
        h->step += 1;
        AdamWArgs aa = adam_w_args(h);
        aa.partials = h->d_partials();
        aa.np = np;
        aa.apply = 1;
        aa.inv_n = float(1.0 / double(n));
        aa.nloss = np;
        aa.loss_scale = aa.inv_n;
        aa.loss_out = d_losses ? d_losses + k : nullptr;
        if ((s = launch_adam_w(h, aa, st)) != NRC_OK) return s;
        launches += 2;
    }
    h->launches = launches;
    return NRC_OK;
}
// The same launches as one CUDA graph: the graph of (n, nsteps) is captured
// once on a private stream (programmatic edges between the kernels, as on the
// stream) and replayed with this call's kernel arguments
// (cudaGraphExecKernelNodeSetParams); saves the per-launch gaps of the chain.
static nrc_status train_steps_graph(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n,
                                    const Gather& gth, float* d_losses, uint32_t nsteps, cudaStream_t st) {
    const int grid = train_grid(h, n);
    std::vector<TrainArgs> pa(nsteps);
    std::vector<AdamWArgs> aa(nsteps);
    for (uint32_t k = 0; k < nsteps; ++k) {
        Gather g = gth;
        g.offset = gth.offset + uint64_t(k) * n;
        pa[k] = train_args(h, d_rec, d_tgt, n, g);
        h->step += 1;
        aa[k] = adam_w_args(h);
        aa[k].partials = h->d_partials();
        aa[k].np = grid;
        aa[k].apply = 1;
        aa[k].inv_n = float(1.0 / double(n));
        aa[k].nloss = grid;
        aa[k].loss_scale = aa[k].inv_n;
        aa[k].loss_out = d_losses ? d_losses + k : nullptr;
    }
    auto& tg = h->tgraph;
    if (tg.exec == nullptr || tg.n != n || tg.nsteps != nsteps) {
        if (tg.exec) cudaGraphExecDestroy(tg.exec);
        if (tg.graph) cudaGraphDestroy(tg.graph);
        tg = nrc_handle::TrainGraph{};
        if (!h->capture) NRC_CUDA(h, cudaStreamCreateWithFlags(&h->capture, cudaStreamNonBlocking));
        NRC_CUDA(h, cudaStreamBeginCapture(h->capture, cudaStreamCaptureModeThreadLocal));
        for (uint32_t k = 0; k < nsteps; ++k) {
            cudaError_t e = launch_train_w_grid(h, pa[k], grid, h->capture);
            if (e == cudaSuccess) {
                const uint64_t saved = h->launches;
                nrc_status st2 = launch_adam_w(h, aa[k], h->capture);
                h->launches = uint32_t(saved);
                if (st2 != NRC_OK) e = cudaErrorUnknown;
            }
            if (e != cudaSuccess) {
                cudaGraph_t dead = nullptr;
                cudaStreamEndCapture(h->capture, &dead);
                if (dead) cudaGraphDestroy(dead);
                return fail(h, NRC_ERR_CUDA, "nrc_train_frame: graph capture failed");
            }
        }
        NRC_CUDA(h, cudaStreamEndCapture(h->capture, &tg.graph));
        // the captured chain in launch order: from the root along its single
        // dependent each time (the programmatic edges are graph edges too)
        size_t count = 0;
        NRC_CUDA(h, cudaGraphGetRootNodes(tg.graph, nullptr, &count));
        if (count != 1) return fail(h, NRC_ERR_CUDA, "nrc_train_frame: unexpected graph shape");
        cudaGraphNode_t node = nullptr;
        NRC_CUDA(h, cudaGraphGetRootNodes(tg.graph, &node, &count));
        while (node != nullptr) {
            cudaGraphNodeType t;
            NRC_CUDA(h, cudaGraphNodeGetType(node, &t));
            if (t != cudaGraphNodeTypeKernel) return fail(h, NRC_ERR_CUDA, "nrc_train_frame: unexpected graph node");
            tg.nodes.push_back(node);
            size_t nd = 0;
            NRC_CUDA(h, cudaGraphNodeGetDependentNodes_v2(node, nullptr, nullptr, &nd));
            if (nd > 1) return fail(h, NRC_ERR_CUDA, "nrc_train_frame: unexpected graph shape");
            cudaGraphNode_t next = nullptr;
            cudaGraphEdgeData edge{};
            if (nd == 1) NRC_CUDA(h, cudaGraphNodeGetDependentNodes_v2(node, &next, &edge, &nd));
            node = next;
        }
        if (tg.nodes.size() != size_t(2) * nsteps)
            return fail(h, NRC_ERR_CUDA, "nrc_train_frame: unexpected graph shape");
        NRC_CUDA(h, cudaGraphInstantiate(&tg.exec, tg.graph, 0));
        tg.n = n;
        tg.nsteps = nsteps;
    } else {
        for (uint32_t i = 0; i < 2 * nsteps; ++i) {
            cudaKernelNodeParams p{};
            NRC_CUDA(h, cudaGraphKernelNodeGetParams(tg.nodes[i], &p));
            void* args[1] = {(i & 1) ? static_cast<void*>(&aa[i / 2]) : static_cast<void*>(&pa[i / 2])};
            p.kernelParams = args;
            p.extra = nullptr;
            NRC_CUDA(h, cudaGraphExecKernelNodeSetParams(tg.exec, tg.nodes[i], &p));
        }
    }
    NRC_CUDA(h, cudaGraphLaunch(tg.exec, st));
    h->launches = 2 * nsteps;
    return NRC_OK;
}

// partials -> logical gradient sum + loss sum (multi-GPU backward)
static nrc_status reduce_partials(nrc_handle* h, int np, float* d_grad, float* d_loss_sum, cudaStream_t st) {
    AdamWArgs aa = adam_w_args(h);
    aa.partials = h->d_partials();
    aa.np = np;
    aa.grad_out = d_grad;
    aa.apply = 0;
    aa.nloss = np;
    aa.loss_scale = 1.0f;
    aa.loss_out = d_loss_sum;
    return launch_adam_w(h, aa, st);
}

static nrc_status check_train_args(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint64_t n,
                                   const char* who) {
    if (!d_rec || !d_tgt || !aligned(d_rec, 16) || !aligned(d_tgt, 4))
        return fail(h, NRC_ERR_INVALID_ARGUMENT, std::string(who) + ": NULL or misaligned pointer");
    if (n > h->cfg.max_batch) return fail(h, NRC_ERR_INVALID_ARGUMENT, std::string(who) + ": n > max_batch");
    return NRC_OK;
}

nrc_status nrc_train_step(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n, float* d_loss,
                          void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    if ((s = check_train_width(h)) != NRC_OK) return s;
    h->launches = 0;
    if (n == 0) return NRC_OK;
    if ((s = check_train_args(h, d_rec, d_tgt, n, "nrc_train_step")) != NRC_OK) return s;
    if (d_loss && !aligned(d_loss, 4)) return fail(h, NRC_ERR_INVALID_ARGUMENT, "misaligned d_loss");
    Gather g{false, 0, 0, 0, 0, 0};
    return train_steps(h, d_rec, d_tgt, n, g, d_loss, 1, static_cast<cudaStream_t>(stream));
}

nrc_status nrc_train_backward(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n_local,
                              float* d_grad, float* d_loss_sum, float* d_pred, void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    if ((s = check_train_width(h)) != NRC_OK) return s;
    h->launches = 0;
    if (!d_grad || !aligned(d_grad, 4)) return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_backward: bad d_grad");
    if (d_pred && !aligned(d_pred, 4)) return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_backward: bad d_pred");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n_local == 0) {  // contributes a zero gradient to the all-reduce
        NRC_CUDA(h, cudaMemsetAsync(d_grad, 0, sizeof(float) * size_t(h->wi.logical), st));
        if (d_loss_sum) NRC_CUDA(h, cudaMemsetAsync(d_loss_sum, 0, sizeof(float), st));
        return NRC_OK;
    }
    if ((s = check_train_args(h, d_rec, d_tgt, n_local, "nrc_train_backward")) != NRC_OK) return s;
    int np = 0;
    Gather g{false, 0, 0, 0, 0, 0};
    if ((s = launch_train_w(h, d_rec, d_tgt, n_local, g, st, &np, d_pred)) != NRC_OK) return s;
    return reduce_partials(h, np, d_grad, d_loss_sum, st);
}

nrc_status nrc_train_frame_backward(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n_total,
                                    uint32_t l, uint64_t shuffle_seed, uint32_t j, uint32_t row_begin,
                                    uint32_t row_end, float* d_grad, float* d_loss_sum, void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    if ((s = check_train_width(h)) != NRC_OK) return s;
    h->launches = 0;
    if (!d_grad || !aligned(d_grad, 4)) return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_frame_backward: bad d_grad");
    if (row_begin > row_end || row_end > l || uint64_t(j + 1) * l > n_total)
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_frame_backward: rows outside batch j");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint32_t n = row_end - row_begin;
    if (n == 0) {
        NRC_CUDA(h, cudaMemsetAsync(d_grad, 0, sizeof(float) * size_t(h->wi.logical), st));
        if (d_loss_sum) NRC_CUDA(h, cudaMemsetAsync(d_loss_sum, 0, sizeof(float), st));
        return NRC_OK;
    }
    if ((s = check_train_args(h, d_rec, d_tgt, n, "nrc_train_frame_backward")) != NRC_OK) return s;
    Gather g{true, 0, 0, 0, n_total, uint64_t(j) * l + row_begin};
    nrc_lcg_params(n_total, shuffle_seed, &g.a, &g.c, &g.m);
    int np = 0;
    if ((s = launch_train_w(h, d_rec, d_tgt, n, g, st, &np)) != NRC_OK) return s;
    return reduce_partials(h, np, d_grad, d_loss_sum, st);
}

nrc_status nrc_train_apply(nrc_handle* h, const float* d_grad_sum, uint32_t n_global, const float* d_loss_sum,
                           float* d_loss, void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    if ((s = check_train_width(h)) != NRC_OK) return s;
    h->launches = 0;
    if (n_global == 0) return NRC_OK;
    if (!d_grad_sum || !aligned(d_grad_sum, 4)) return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_apply: bad grad");
    if ((d_loss_sum && !aligned(d_loss_sum, 4)) || (d_loss && !aligned(d_loss, 4)))
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_apply: misaligned loss pointer");
    h->step += 1;
    AdamWArgs aw = adam_w_args(h);
    aw.grad_logical = d_grad_sum;
    aw.apply = 1;
    aw.inv_n = float(1.0 / double(n_global));
    if (d_loss_sum && d_loss) {  // batch-mean loss = all-reduced loss sum / n_global (R10)
        aw.loss_part = d_loss_sum;
        aw.nloss = 1;
        aw.loss_scale = aw.inv_n;
        aw.loss_out = d_loss;
    } else {
        aw.loss_part = nullptr;
        aw.nloss = 0;
    }
    return launch_adam_w(h, aw, static_cast<cudaStream_t>(stream));
}

static nrc_status train_frame_impl(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n_total,
                                   uint32_t s_, uint32_t l, uint64_t shuffle_seed, float* d_losses, Gather g,
                                   cudaStream_t st) {
    if (uint64_t(s_) * l > n_total) l = n_total / s_;  // batches shrink proportionally
    if (l == 0) return NRC_OK;
    if (l > h->cfg.max_batch) return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_frame: l > max_batch");
    g.on = true;
    g.n = n_total;
    g.offset = 0;
    nrc_lcg_params(n_total, shuffle_seed, &g.a, &g.c, &g.m);
    return train_steps(h, d_rec, d_tgt, l, g, d_losses, s_, st);
}

nrc_status nrc_train_frame(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n_total, uint32_t s_,
                           uint32_t l, uint64_t shuffle_seed, float* d_losses, void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    if ((s = check_train_width(h)) != NRC_OK) return s;
    h->launches = 0;
    if (n_total == 0 || s_ == 0 || l == 0) return NRC_OK;
    if (!d_rec || !d_tgt || !aligned(d_rec, 16) || !aligned(d_tgt, 4))
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_frame: NULL or misaligned pointer");
    if (d_losses && !aligned(d_losses, 4)) return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_frame: misaligned d_losses");
    Gather g{true, 0, 0, 0, n_total, 0};
    return train_frame_impl(h, d_rec, d_tgt, n_total, s_, l, shuffle_seed, d_losses, g,
                            static_cast<cudaStream_t>(stream));
}


nrc_status nrc_train_frame_dp_peer(nrc_handle* h, const nrc_record* d_rec, const float* d_tgt, uint32_t n_total,
                                   uint32_t s_, uint32_t l, uint64_t shuffle_seed, uint32_t rank, uint32_t world,
                                   void* const* peer_state, float* d_losses, void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    if ((s = check_train_width(h)) != NRC_OK) return s;
    h->launches = 0;
    if (world == 0 || world > uint32_t(kMaxRanks) || rank >= world || !peer_state)
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_frame_dp_peer: 1..8 ranks, rank < world, peer_state");
    if (peer_state[rank] != h->state)
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_frame_dp_peer: peer_state[rank] must be this cache's arena");
    for (uint32_t p = 0; p < world; ++p)
        if (!peer_state[p] || !aligned(peer_state[p], 256))
            return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_frame_dp_peer: NULL or misaligned peer arena");
    if (n_total == 0 || s_ == 0 || l == 0) return NRC_OK;
    if (!d_rec || !d_tgt || !aligned(d_rec, 16) || !aligned(d_tgt, 4))
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_frame_dp_peer: NULL or misaligned pointer");
    if (uint64_t(s_) * l > n_total) l = n_total / s_;
    if (l == 0) return NRC_OK;
    const uint32_t T = (l + kTile - 1) / kTile;  // tiles per step
    if (T > uint32_t(kMaxDpTiles) || int(T) > h->num_sms)
        return fail(h, NRC_ERR_UNSUPPORTED, "nrc_train_frame_dp_peer: at most 128 tiles (16,384 rows) per step");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto t_lo = [&](uint32_t k) { return k * T / world; };  // rank k owns tiles [t_lo(k), t_lo(k + 1))
    Gather g{true, 0, 0, 0, n_total, 0};
    nrc_lcg_params(n_total, shuffle_seed, &g.a, &g.c, &g.m);
    DpPeers peers{};
    for (uint32_t p = 0; p < world; ++p)
        peers.ctr[p] = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(peer_state[p]) + h->L.counters) + 4;
    const size_t pad = size_t(h->wi.padded);
    // reduction tables of both slot parities: [parity][partials | losses][tile]
    const float** d_tab = reinterpret_cast<const float**>(h->state + h->L.dp_tables);
    {
        std::vector<const float*> tab(size_t(2) * 2 * kMaxDpTiles, nullptr);
        for (uint32_t par = 0; par < 2; ++par)
            for (uint32_t k = 0; k < world; ++k) {
                const float* part = reinterpret_cast<const float*>(static_cast<uint8_t*>(peer_state[k]) + h->L.partials);
                const float* loss = reinterpret_cast<const float*>(static_cast<uint8_t*>(peer_state[k]) + h->L.loss_part);
                for (uint32_t t = t_lo(k); t < t_lo(k + 1); ++t) {
                    const size_t slot = size_t(par) * kMaxDpTiles + (t - t_lo(k));
                    tab[(par * 2 + 0) * kMaxDpTiles + t] = part + slot * pad;
                    tab[(par * 2 + 1) * kMaxDpTiles + t] = loss + slot;
                }
            }
        // pageable source: staged before the call returns, so `tab` may go
        NRC_CUDA(h, cudaMemcpyAsync(d_tab, tab.data(), sizeof(const float*) * tab.size(), cudaMemcpyHostToDevice, st));
    }
    uint32_t launches = 0;
    for (uint32_t j = 0; j < s_; ++j) {
        const uint32_t parity = uint32_t(h->dp_seq & 1u);
        // 1. this rank's tiles of batch j -> per-tile partials in slot half `parity`
        const uint32_t r0 = t_lo(rank) * kTile, r1 = std::min(t_lo(rank + 1) * kTile, l);
        if (r1 > r0) {
            g.offset = uint64_t(j) * l + r0;
            TrainArgs ta = train_args(h, d_rec, d_tgt, r1 - r0, g);
            ta.partials = h->d_partials() + size_t(parity) * kMaxDpTiles * pad;
            ta.loss_part = h->d_loss_part() + size_t(parity) * kMaxDpTiles;
            const int grid = int(t_lo(rank + 1) - t_lo(rank));  // one tile per CTA: CTA c -> tile t_lo(rank) + c
            NRC_CUDA(h, launch_train_w_grid(h, ta, grid, st));
            NRC_LAUNCHED(h, "nrc_train_w_kernel");
            ++launches;
        }
        // 2. publish to every rank, wait for every rank (system-scope counters)
        h->dp_expect += world;
        nrc_dp_exchange_kernel<<<1, 32, 0, st>>>(peers, int(world), h->d_counters() + 4, h->dp_expect,
                                                  h->d_counters() + 5);
        NRC_LAUNCHED(h, "nrc_dp_exchange_kernel");
        // 3. reduce all T tile partials in tile order from their owners' arenas + Adam + EMA
        h->step += 1;
        AdamWArgs aa = adam_w_args(h);
        aa.tile_part = d_tab + (parity * 2 + 0) * kMaxDpTiles;
        aa.tile_loss = d_tab + (parity * 2 + 1) * kMaxDpTiles;
        aa.np = int(T);
        aa.nloss = int(T);
        aa.apply = 1;
        aa.inv_n = float(1.0 / double(l));
        aa.loss_scale = aa.inv_n;
        aa.loss_out = d_losses ? d_losses + j : nullptr;
        if ((s = launch_adam_w(h, aa, st)) != NRC_OK) return s;
        launches += 2;
        h->dp_seq += 1;
    }
    h->launches = launches;
    return NRC_OK;
}

nrc_status nrc_train_apply_multimem(nrc_handle* h, const float* mc_grad, uint32_t n_global, float* d_loss,
                                    void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    if ((s = check_train_width(h)) != NRC_OK) return s;
    h->launches = 0;
    if (n_global == 0) return NRC_OK;
    if (!mc_grad || !aligned(mc_grad, 16) || (d_loss && !aligned(d_loss, 4)))
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_apply_multimem: NULL or misaligned pointer");
    h->step += 1;
    AdamWArgs aw = adam_w_args(h);
    aw.grad_mc = mc_grad;
    aw.apply = 1;
    aw.inv_n = float(1.0 / double(n_global));
    aw.loss_scale = aw.inv_n;
    aw.loss_out = d_loss;
    return launch_adam_w(h, aw, static_cast<cudaStream_t>(stream));
}

nrc_status nrc_train_apply_peers(nrc_handle* h, const float* const* peer_bufs, uint32_t world, uint32_t n_global,
                                 float* d_loss, void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    if ((s = check_train_width(h)) != NRC_OK) return s;
    h->launches = 0;
    if (!peer_bufs || world == 0 || world > uint32_t(kMaxRanks))
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_apply_peers: 1..8 peer buffers");
    for (uint32_t p = 0; p < world; ++p)
        if (!peer_bufs[p] || !aligned(peer_bufs[p], 16))
            return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_apply_peers: NULL or misaligned peer buffer");
    if (d_loss && !aligned(d_loss, 4)) return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_train_apply_peers: misaligned d_loss");
    if (n_global == 0) return NRC_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the pointer table in device memory: reuse one of two slots when it holds
    // the same pointers (buffers alternate by step parity), else refill one
    const float** d_tab = reinterpret_cast<const float**>(h->state + h->L.peer_tab);
    int slot = -1;
    for (int q = 0; q < 2 && slot < 0; ++q)
        if (h->peer_tab_world[q] == world &&
            std::equal(peer_bufs, peer_bufs + world, static_cast<const float* const*>(h->peer_tab_host[q])))
            slot = q;
    if (slot < 0) {
        slot = h->peer_tab_next;
        h->peer_tab_next ^= 1;
        std::copy(peer_bufs, peer_bufs + world, h->peer_tab_host[slot]);
        h->peer_tab_world[slot] = world;
        // pageable source: staged before the call returns
        NRC_CUDA(h, cudaMemcpyAsync(d_tab + slot * kMaxRanks, h->peer_tab_host[slot], sizeof(const float*) * world,
                                    cudaMemcpyHostToDevice, st));
    }
    h->step += 1;
    AdamWArgs aw = adam_w_args(h);
    aw.peer_grad = d_tab + slot * kMaxRanks;
    aw.npeer = int(world);
    aw.apply = 1;
    aw.inv_n = float(1.0 / double(n_global));
    aw.loss_scale = aw.inv_n;
    aw.loss_out = d_loss;
    return launch_adam_w(h, aw, st);
}

nrc_status nrc_peer_barrier(nrc_handle* h, void* const* peer_counters, uint32_t rank, uint32_t world, void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    h->launches = 0;
    if (!peer_counters || world == 0 || world > uint32_t(kMaxRanks) || rank >= world)
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_peer_barrier: 1..8 ranks, rank < world");
    DpPeers peers{};
    for (uint32_t p = 0; p < world; ++p) {
        if (!peer_counters[p] || !aligned(peer_counters[p], 8))
            return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_peer_barrier: NULL or misaligned counter");
        peers.ctr[p] = static_cast<unsigned long long*>(peer_counters[p]);
    }
    h->bar_expect += world;
    nrc_dp_exchange_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
        peers, int(world), peers.ctr[rank], h->bar_expect, h->d_counters() + 5);
    NRC_LAUNCHED(h, "nrc_dp_exchange_kernel");
    return NRC_OK;
}

}  // extern "C"
// ---- single-process NVLS multicast buffer (driver API through the runtime's
// entry-point query: no link-time libcuda dependency)
namespace {
template <typename F>
F driver_fn(const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
    return reinterpret_cast<F>(fn);
}
struct McBuf {
    CUmemGenericAllocationHandle mem = 0, mc = 0;
    CUdeviceptr uc = 0, mcp = 0;
    size_t size = 0;
    int device = 0;
};
std::vector<McBuf> g_mc;  // live buffers (nrc_multicast_free releases)
}  // namespace
extern "C" {

nrc_status nrc_multicast_alloc(int device, size_t bytes, void** d_uc, void** d_mc) {
    if (!d_uc || !d_mc || bytes == 0) return NRC_ERR_INVALID_ARGUMENT;
    *d_uc = *d_mc = nullptr;
    using GetGran = CUresult (*)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
    using McCreate = CUresult (*)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
    using McAdd = CUresult (*)(CUmemGenericAllocationHandle, CUdevice);
    using McBind = CUresult (*)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                                unsigned long long);
    using MemCreate = CUresult (*)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
    using Reserve = CUresult (*)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
    using Map = CUresult (*)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    using Access = CUresult (*)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
    using DevGet = CUresult (*)(CUdevice*, int);
    using Attr = CUresult (*)(int*, CUdevice_attribute, CUdevice);
    auto get_gran = driver_fn<GetGran>("cuMulticastGetGranularity");
    auto mc_create = driver_fn<McCreate>("cuMulticastCreate");
    auto mc_add = driver_fn<McAdd>("cuMulticastAddDevice");
    auto mc_bind = driver_fn<McBind>("cuMulticastBindMem");
    auto mem_create = driver_fn<MemCreate>("cuMemCreate");
    auto reserve = driver_fn<Reserve>("cuMemAddressReserve");
    auto map = driver_fn<Map>("cuMemMap");
    auto access = driver_fn<Access>("cuMemSetAccess");
    auto dev_get = driver_fn<DevGet>("cuDeviceGet");
    auto attr = driver_fn<Attr>("cuDeviceGetAttribute");
    if (!get_gran || !mc_create || !mc_add || !mc_bind || !mem_create || !reserve || !map || !access || !dev_get || !attr)
        return NRC_ERR_UNSUPPORTED;
    if (cudaSetDevice(device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess) return NRC_ERR_CUDA;
    CUdevice dev;
    if (dev_get(&dev, device) != CUDA_SUCCESS) return NRC_ERR_CUDA;
    int mc_ok = 0;
    if (attr(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS || !mc_ok) return NRC_ERR_UNSUPPORTED;
    CUmulticastObjectProp prop{};
    prop.numDevices = 1;
    prop.size = bytes;
    size_t gran = 0;
    if (get_gran(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || gran == 0) return NRC_ERR_CUDA;
    McBuf b;
    b.device = device;
    b.size = (bytes + gran - 1) / gran * gran;
    prop.size = b.size;
    if (mc_create(&b.mc, &prop) != CUDA_SUCCESS) return NRC_ERR_UNSUPPORTED;
    if (mc_add(b.mc, dev) != CUDA_SUCCESS) return NRC_ERR_CUDA;
    CUmemAllocationProp mp{};
    mp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    mp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    mp.location.id = device;
    if (mem_create(&b.mem, b.size, &mp, 0) != CUDA_SUCCESS) return NRC_ERR_OUT_OF_MEMORY;
    if (mc_bind(b.mc, 0, b.mem, 0, b.size, 0) != CUDA_SUCCESS) return NRC_ERR_CUDA;
    CUmemAccessDesc ad{};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = device;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (reserve(&b.uc, b.size, gran, 0, 0) != CUDA_SUCCESS || map(b.uc, b.size, 0, b.mem, 0) != CUDA_SUCCESS ||
        access(b.uc, b.size, &ad, 1) != CUDA_SUCCESS)
        return NRC_ERR_CUDA;
    if (reserve(&b.mcp, b.size, gran, 0, 0) != CUDA_SUCCESS || map(b.mcp, b.size, 0, b.mc, 0) != CUDA_SUCCESS ||
        access(b.mcp, b.size, &ad, 1) != CUDA_SUCCESS)
        return NRC_ERR_CUDA;
    if (cudaMemset(reinterpret_cast<void*>(b.uc), 0, b.size) != cudaSuccess) return NRC_ERR_CUDA;
    *d_uc = reinterpret_cast<void*>(b.uc);
    *d_mc = reinterpret_cast<void*>(b.mcp);
    g_mc.push_back(b);
    return NRC_OK;
}

nrc_status nrc_multicast_free(void* d_uc) {
    using Unmap = CUresult (*)(CUdeviceptr, size_t);
    using Free = CUresult (*)(CUdeviceptr, size_t);
    using Release = CUresult (*)(CUmemGenericAllocationHandle);
    using Unbind = CUresult (*)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
    using DevGet = CUresult (*)(CUdevice*, int);
    auto unmap = driver_fn<Unmap>("cuMemUnmap");
    auto afree = driver_fn<Free>("cuMemAddressFree");
    auto release = driver_fn<Release>("cuMemRelease");
    auto unbind = driver_fn<Unbind>("cuMulticastUnbind");
    auto dev_get = driver_fn<DevGet>("cuDeviceGet");
    for (size_t i = 0; i < g_mc.size(); ++i) {
        McBuf& b = g_mc[i];
        if (reinterpret_cast<void*>(b.uc) != d_uc) continue;
        if (!unmap || !afree || !release || !unbind || !dev_get) return NRC_ERR_UNSUPPORTED;
        cudaDeviceSynchronize();
        CUdevice dev;
        dev_get(&dev, b.device);
        unmap(b.mcp, b.size);
        afree(b.mcp, b.size);
        unmap(b.uc, b.size);
        afree(b.uc, b.size);
        unbind(b.mc, dev, 0, b.size);
        release(b.mc);
        release(b.mem);
        g_mc.erase(g_mc.begin() + long(i));
        return NRC_OK;
    }
    return NRC_ERR_INVALID_ARGUMENT;
}

nrc_status nrc_dp_timeouts(nrc_handle* h, uint64_t* count) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    if (!count) return NRC_ERR_INVALID_ARGUMENT;
    unsigned long long c = 0;
    NRC_CUDA(h, cudaDeviceSynchronize());
    NRC_CUDA(h, cudaMemcpy(&c, h->d_counters() + 5, sizeof(c), cudaMemcpyDeviceToHost));
    *count = c;
    return NRC_OK;
}

nrc_status nrc_ipc_export(const void* d_ptr, uint8_t* handle, uint64_t* offset) {
    if (!d_ptr || !handle || !offset) return NRC_ERR_INVALID_ARGUMENT;
    // driver entry point through the runtime (no link-time libcuda dependency)
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = nullptr;
    if (!get_range) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return NRC_ERR_CUDA;
        get_range = reinterpret_cast<GetRange>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS) return NRC_ERR_CUDA;
    cudaIpcMemHandle_t hd;
    if (cudaIpcGetMemHandle(&hd, reinterpret_cast<void*>(base)) != cudaSuccess) return NRC_ERR_CUDA;
    std::memcpy(handle, &hd, sizeof(hd));
    *offset = uint64_t(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
    return NRC_OK;
}

nrc_status nrc_ipc_import(const uint8_t* handle, uint64_t offset, void** d_ptr) {
    if (!handle || !d_ptr) return NRC_ERR_INVALID_ARGUMENT;
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, handle, sizeof(hd));
    void* base = nullptr;
    if (cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return NRC_ERR_CUDA;
    *d_ptr = static_cast<uint8_t*>(base) + offset;
    return NRC_OK;
}

nrc_status nrc_ipc_close(void* d_ptr, uint64_t offset) {
    if (!d_ptr) return NRC_ERR_INVALID_ARGUMENT;
    return cudaIpcCloseMemHandle(static_cast<uint8_t*>(d_ptr) - offset) == cudaSuccess ? NRC_OK : NRC_ERR_CUDA;
}

nrc_status nrc_encode(nrc_handle* h, const nrc_record* d_rec, uint64_t n, uint16_t* d_out, void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    h->launches = 0;
    if (n == 0) return NRC_OK;
    if (!d_rec || !d_out || !aligned(d_rec, 16) || !aligned(d_out, 16))
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_encode: NULL or misaligned pointer");
    const unsigned blocks = unsigned((n + 127) / 128);
    if (h->ep.exact)
        nrc_encode_kernel<true><<<blocks, 128, 0, static_cast<cudaStream_t>(stream)>>>(
            reinterpret_cast<const float*>(d_rec), n, h->ep, reinterpret_cast<uint4*>(d_out), h->d_counters() + 2);
    else
        nrc_encode_kernel<false><<<blocks, 128, 0, static_cast<cudaStream_t>(stream)>>>(
            reinterpret_cast<const float*>(d_rec), n, h->ep, reinterpret_cast<uint4*>(d_out), h->d_counters() + 2);
    NRC_LAUNCHED(h, "nrc_encode_kernel");
    return NRC_OK;
}

nrc_status nrc_assemble_targets(nrc_handle* h, const uint32_t* d_first, const uint32_t* d_len,
                                const uint32_t* d_flags, uint32_t n_paths, const float* d_vert,
                                const float* d_tail, float* d_targets, void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    h->launches = 0;
    if (n_paths == 0) return NRC_OK;
    if (!d_first || !d_len || !d_flags || !d_vert || !d_tail || !d_targets || !aligned(d_first, 4) ||
        !aligned(d_len, 4) || !aligned(d_flags, 4) || !aligned(d_vert, 4) || !aligned(d_tail, 4) ||
        !aligned(d_targets, 4))
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_assemble_targets: NULL or misaligned pointer");
    nrc_targets_kernel<<<(n_paths + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
        d_first, d_len, d_flags, n_paths, d_vert, d_tail, d_targets);
    NRC_LAUNCHED(h, "nrc_targets_kernel");
    return NRC_OK;
}

static float* param_ptr(nrc_handle* h, nrc_param_set which) {
    switch (which) {
        case NRC_PARAMS_TRAIN: return h->d_w();
        case NRC_PARAMS_EMA: return h->d_ema();
        case NRC_ADAM_M: return h->d_m();
        case NRC_ADAM_V: return h->d_v();
    }
    return nullptr;
}

// logical <-> padded: only W5's rows 3..15 are padding (W0..W4 identical)
static void logical_to_padded(const WidthInfo& wi, const float* lg, float* pd) {
    std::memset(pd, 0, sizeof(float) * size_t(wi.padded));
    std::memcpy(pd, lg, sizeof(float) * size_t(wi.logical));
}
static void padded_to_logical(const WidthInfo& wi, const float* pd, float* lg) {
    std::memcpy(lg, pd, sizeof(float) * size_t(wi.logical));
}

nrc_status nrc_get_params(nrc_handle* h, nrc_param_set which, float* h_out, size_t n) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    float* src = param_ptr(h, which);
    if (!src || !h_out || n < size_t(h->wi.logical)) return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_get_params");
    std::vector<float> pd(size_t(h->wi.padded));
    NRC_CUDA(h, cudaDeviceSynchronize());
    NRC_CUDA(h, cudaMemcpy(pd.data(), src, sizeof(float) * pd.size(), cudaMemcpyDeviceToHost));
    padded_to_logical(h->wi, pd.data(), h_out);
    return NRC_OK;
}

nrc_status nrc_set_params(nrc_handle* h, nrc_param_set which, const float* h_in, size_t n) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    float* dst = param_ptr(h, which);
    if (!dst || !h_in || n < size_t(h->wi.logical)) return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_set_params");
    std::vector<float> pd(size_t(h->wi.padded));
    logical_to_padded(h->wi, h_in, pd.data());
    NRC_CUDA(h, cudaDeviceSynchronize());
    NRC_CUDA(h, cudaMemcpy(dst, pd.data(), sizeof(float) * pd.size(), cudaMemcpyHostToDevice));
    h->launches = 0;
    if ((s = refresh_images(h, 0)) != NRC_OK) return s;
    NRC_CUDA(h, cudaDeviceSynchronize());
    return NRC_OK;
}

nrc_status nrc_get_stats(nrc_handle* h, uint64_t* step, uint64_t* nonfinite_grads, uint64_t* nonfinite_targets,
                         uint64_t* degenerate_vectors) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    unsigned long long c[4] = {0, 0, 0, 0};
    NRC_CUDA(h, cudaDeviceSynchronize());
    NRC_CUDA(h, cudaMemcpy(c, h->d_counters(), sizeof(c), cudaMemcpyDeviceToHost));
    if (step) *step = h->step;
    if (nonfinite_grads) *nonfinite_grads = c[0];
    if (nonfinite_targets) *nonfinite_targets = c[1];
    if (degenerate_vectors) *degenerate_vectors = c[2];
    return NRC_OK;
}

size_t nrc_frame_scratch_bytes(uint64_t n_query, uint32_t n_train) {
    return align_up(n_query * sizeof(nrc_record), 256) + align_up(n_query * 3 * sizeof(float), 256) +
           align_up(size_t(n_train) * sizeof(nrc_record), 256) + align_up(size_t(n_train) * 3 * sizeof(float), 256) +
           256;
}

nrc_status nrc_frame_host(nrc_handle* h, const nrc_record* h_query, uint64_t n_query, float* h_rgb,
                          const nrc_record* h_train, const float* h_tgt, uint32_t n_train, uint32_t s_, uint32_t l,
                          uint64_t shuffle_seed, float* h_losses, void* d_scratch, size_t scratch_bytes,
                          void* stream) {
    nrc_status s = check_handle(h);
    if (s != NRC_OK) return s;
    if (!d_scratch || !aligned(d_scratch, 256) || scratch_bytes < nrc_frame_scratch_bytes(n_query, n_train))
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_frame_host: scratch too small or misaligned");
    if ((n_query && (!h_query || !h_rgb)) || (n_train && (!h_train || !h_tgt)))
        return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_frame_host: NULL host buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* p = static_cast<uint8_t*>(d_scratch);
    nrc_record* dq = reinterpret_cast<nrc_record*>(p);
    p += align_up(n_query * sizeof(nrc_record), 256);
    float* drgb = reinterpret_cast<float*>(p);
    p += align_up(n_query * 3 * sizeof(float), 256);
    nrc_record* dt = reinterpret_cast<nrc_record*>(p);
    p += align_up(size_t(n_train) * sizeof(nrc_record), 256);
    float* dtg = reinterpret_cast<float*>(p);
    p += align_up(size_t(n_train) * 3 * sizeof(float), 256);
    float* dloss = reinterpret_cast<float*>(p);  // up to 64 losses
    if (s_ > 64) return fail(h, NRC_ERR_INVALID_ARGUMENT, "nrc_frame_host: s > 64");
    // Pipelined: the query batch moves in chunks; chunk k's
    // host->device copy (stream copy_in) overlaps the query of chunk k-1 (the
    // caller's stream) and the device->host copy of chunk k-2's RGB (stream
    // copy_out).  The training data (small) goes first; training runs after
    // the last query chunk, so queries see the EMA weights of the previous
    // frame as in the unpipelined order.  The caller's stream finally waits
    // for copy_out, so synchronising it covers every copy.
    if (!h->copy_in) NRC_CUDA(h, cudaStreamCreateWithFlags(&h->copy_in, cudaStreamNonBlocking));
    if (!h->copy_out) NRC_CUDA(h, cudaStreamCreateWithFlags(&h->copy_out, cudaStreamNonBlocking));
    constexpr uint64_t kChunk = 262144;  // records per chunk (16.8 MB in, 3.1 MB out)
    const uint64_t nchunks = (n_query + kChunk - 1) / kChunk;
    uint32_t launches = 0;
    size_t ev = 0;
    cudaEvent_t e_start = h->event(ev++);
    NRC_CUDA(h, cudaEventRecord(e_start, st));  // earlier work on the caller's stream (scratch reuse)
    NRC_CUDA(h, cudaStreamWaitEvent(h->copy_in, e_start, 0));
    NRC_CUDA(h, cudaStreamWaitEvent(h->copy_out, e_start, 0));
    cudaEvent_t e_train = h->event(ev++);
    if (n_train) {
        NRC_CUDA(h, cudaMemcpyAsync(dt, h_train, size_t(n_train) * sizeof(nrc_record), cudaMemcpyHostToDevice,
                                    h->copy_in));
        NRC_CUDA(h, cudaMemcpyAsync(dtg, h_tgt, size_t(n_train) * 3 * sizeof(float), cudaMemcpyHostToDevice,
                                    h->copy_in));
    }
    NRC_CUDA(h, cudaEventRecord(e_train, h->copy_in));
    for (uint64_t k = 0; k < nchunks; ++k) {
        const uint64_t r0 = k * kChunk, nr = (n_query - r0) < kChunk ? (n_query - r0) : kChunk;
        cudaEvent_t e_in = h->event(ev++), e_q = h->event(ev++);
        NRC_CUDA(h, cudaMemcpyAsync(dq + r0, h_query + r0, nr * sizeof(nrc_record), cudaMemcpyHostToDevice,
                                    h->copy_in));
        NRC_CUDA(h, cudaEventRecord(e_in, h->copy_in));
        NRC_CUDA(h, cudaStreamWaitEvent(st, e_in, 0));
        if ((s = nrc_query(h, dq + r0, nr, drgb + 3 * r0, stream)) != NRC_OK) return s;
        launches += h->launches;
        NRC_CUDA(h, cudaEventRecord(e_q, st));
        NRC_CUDA(h, cudaStreamWaitEvent(h->copy_out, e_q, 0));
        NRC_CUDA(h, cudaMemcpyAsync(h_rgb + 3 * r0, drgb + 3 * r0, nr * 3 * sizeof(float), cudaMemcpyDeviceToHost,
                                    h->copy_out));
    }
    NRC_CUDA(h, cudaStreamWaitEvent(st, e_train, 0));
    if ((s = nrc_train_frame(h, dt, dtg, n_train, s_, l, shuffle_seed, dloss, stream)) != NRC_OK) return s;
    launches += h->launches;
    if (h_losses && s_) NRC_CUDA(h, cudaMemcpyAsync(h_losses, dloss, s_ * sizeof(float), cudaMemcpyDeviceToHost, st));
    cudaEvent_t e_out = h->event(ev++);
    NRC_CUDA(h, cudaEventRecord(e_out, h->copy_out));
    NRC_CUDA(h, cudaStreamWaitEvent(st, e_out, 0));
    h->launches = launches;
    return NRC_OK;
}

// Undocumented diagnostic hook (not part of nrc.h): a device buffer of >= 64
// int64 receives clock64 phase timestamps of the train kernel's CTA 0.
nrc_status nrc_debug_set_trace(nrc_handle* h, long long* d_buf) {
    if (!h) return NRC_ERR_STATE;
    h->dbg = d_buf;
    return NRC_OK;
}

nrc_status nrc_selftest_umma(int mode, const uint16_t* d_a, const uint16_t* d_b, float* d_d) {
    if (mode < 0 || mode > 4 || !d_a || !d_b || !d_d || !aligned(d_a, 16) || !aligned(d_b, 16))
        return NRC_ERR_INVALID_ARGUMENT;
    nrc_selftest_kernel<<<1, 128>>>(mode, d_a, d_b, d_d);
    if (cudaGetLastError() != cudaSuccess) return NRC_ERR_CUDA;
    if (cudaDeviceSynchronize() != cudaSuccess) return NRC_ERR_CUDA;
    return NRC_OK;
}

}  // extern "C"
