// C ABI of the B200 render path: context / scene / tape management and the
// launch sequence (include/gvr_cuda.h documents the contract).
//
//   gvr_scene_set : H2D (or D2D) FP64 upload + K0 validate  [1 sync: error code]
//   gvr_render    : K1 project + bin (per-tile lists, atomics) -> tile order ->
//                   K3a select (per-tile smem sort) -> order -> K3b blend;
//                   fully asynchronous (no host synchronisation)
//   gvr_scalar_loss, gvr_backward : K4 per-pixel backward -> K5 object space
#include "../../include/gvr_cuda.h"
#include "backward.cuh"
#include "fit.cuh"
#include "forward.cuh"
#include "project.cuh"
#include "sampler.cuh"
#include "blocks.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

using namespace gvrk;

namespace {

// Forward tile = 8x8 pixels = one default coarse cell (64 threads, 2 warps):
// small CTAs balance the very uneven per-tile work and keep 8 CTAs per SM.
constexpr int kFwdTile = 8;
constexpr int kMaxKPrime = 128;

struct Buf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = bytes > 0 ? bytes + bytes / 4 : 256;
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

bool is_device_ptr(const void* ptr) {
    if (!ptr) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

// Tape flags buffer (ints): [0] dropped_behind, [1] nonfinite, [2..3] loss (double),
// [kListStats .. +3] tile-list stats of the last render (list_offsets),
// [kMaskTotal] mask-rectangle tiles requested by the last render (project_kernel).
constexpr int kListStats = 8, kMaskTotal = 12;

#ifndef GVR_LOSS_CTAS_PER_SM
#define GVR_LOSS_CTAS_PER_SM 4
#endif
constexpr unsigned kLossBlocks = 148u * GVR_LOSS_CTAS_PER_SM;  // loss kernel grid (grid-stride; 2 / 8 / 16 per SM: slower)

enum Stage {
    ST_PROJECT, ST_EMIT, ST_RANGES, ST_SELECT, ST_BLEND, ST_LOSS, ST_BACKWARD, ST_OBJECT, ST_COUNT
};

struct gvr_context {
    int device = 0;
    // optional per-stage timing (events around each launch, summed at query time)
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_pending;
    double stage_ms[ST_COUNT] = {0};
    int64_t stage_n[ST_COUNT] = {0};
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    std::string err;
    int64_t launches = 0;   // kernels of this library
    int64_t capture_launch0 = 0;  // launches when the current capture began
    int64_t lib_calls = 0;  // CUB device-wide calls (scan, radix sort)
    double guard = 0.02;
    bool precise = false;  // verification mode of the blend (gvr_context_set_precise)
    bool tile_profile = false;  // record per-tile selection cycles (gvr_context_set_tile_profile)
    int list_smem = kSelListSmem;  // test hook: longest list sorted in shared memory
    long long pool_override = 0;  // tile-list pool capacity in entries (test hook); 0 = automatic
    bool capturing = false;  // stream capture in progress: no host syncs, no allocations, no timers
    bool async = false;      // host-buffer calls enqueue their copies and return (gvr_context_set_async)
    Buf flags;  // [0] dropped_behind (int), [1] nonfinite (int), [2..3] first_error (u64), [4..5] loss (double)
    int* h_flags = nullptr;  // pinned mirror (64 B)
    Buf scratch[4];           // staging of host inputs / outputs of the helper entry points
    // multi-view calls: views run on worker streams forked from / joined into `stream`
    std::vector<cudaStream_t> workers;
    std::vector<cudaEvent_t> join_ev;
    cudaEvent_t fork_ev = nullptr;
    Buf ptr_table;
    gvr_tape* aux_tape = nullptr;  // render behind gvr_sample_attributes
    // async host-buffer mode: device->host copies of a call's outputs drain on this
    // stream while the context stream runs the next call (out_begin / out_end)
    cudaStream_t out_stream = nullptr;
    cudaEvent_t out_fork = nullptr;
};

struct gvr_graph {
    gvr_context* ctx = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;  // kernels of this library captured (counted again on every replay)
};

struct gvr_scene {
    gvr_context* ctx = nullptr;
    int K = 0, D = 0;
    double tau = 1.0;
    uint64_t version = 0;
    bool valid = false;
    bool deferred = false;  // last upload by gvr_scene_set_deferred: gvr_scene_check reads the device flag
    Buf centers, inv_cov, attr;
    Buf vflag;  // deferred validation: first error (kernel << 2 | code), ~0 = none
};

struct gvr_tape {
    gvr_context* ctx = nullptr;
    const gvr_scene* scene = nullptr;
    uint64_t scene_version = 0;
    bool valid = false;
    bool has_upstream = false;
    gvr_camera cam{};
    gvr_selection cfg{};
    CameraP camp{};
    SelP selp{};
    int K = 0, D = 0, H = 0, W = 0, tile = 16, tiles_x = 0, tiles_y = 0;
    int dropped_behind = 0;
    // per kernel
    Buf rec32, rec64;
    // per-tile candidate lists
    Buf tile_count, tile_off, tile_fill, pool, sorted_pool, tile_cycles;
    // pending device->host output copies on the context's out_stream, per call kind
    // (0 render, 1 loss, 2 backward): the next call of that kind rewrites their sources
    cudaEvent_t out_ev[3] = {nullptr, nullptr, nullptr};
    bool out_pending[3] = {false, false, false};
    // LPT cost hint: the selection cycles per tile of the last render, valid for the
    // same camera and tile layout (hint_cam, hint_shard) -- repeated renders of a view
    Buf tile_hint;
    bool hint_valid = false;
    CameraP hint_cam{};
    int hint_tiles = 0, hint_shard = -1, hint_nshards = 0;
    long long pool_hint = 0;  // entries the last observed render listed (grow-only sizing)
    bool profiled = false;    // the last render recorded tile cycles
    Buf sched;  // [0] n_order (selected tiles), [1] n_all, order[tiles], tile_done[tiles]
    // per pixel
    Buf topk, count, image, alpha, depth, topk_w, tape_t, ent, ent_a;
    Buf d_image, d_alpha;
    // gradients
    Buf acc, attr_fb, d_attr, d_center, d_inv_cov, d_rt;
    // deterministic backward: per-kernel mask rectangles (render), entry adjoints, CTA partials
    Buf kinfo, masks, slot_off, app, bent, bkey, rays, pieces, kcount, rt_part, tickets, loss_part;
    long long mask_hint = 0;
    // host copy-out staging
    Buf stage_i, stage_w;
    // [0] dropped_behind (int), [1] nonfinite (int), [2..3] loss (double); pinned mirror
    Buf flags;
    int* h_flags = nullptr;
};

namespace {

int set_err(gvr_context* ctx, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf;
    return code;
}

#define CUDA_TRY(ctx, expr)                                                                             \
    do {                                                                                                \
        cudaError_t e_ = (expr);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            return set_err((ctx), GVR_ERR_RUNTIME, "CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), \
                           __FILE__, __LINE__, cudaGetErrorString(e_));                                 \
    } while (0)

#define LAUNCH_CHECK(ctx)                  \
    do {                                   \
        ++(ctx)->launches;                 \
        CUDA_TRY((ctx), cudaGetLastError()); \
    } while (0)

// Camera::validate (types.cpp:44-63), same messages.
const char* camera_error(const gvr_camera* c) {
    if (!c) return "camera is null";
    for (int i = 0; i < 9; ++i)
        if (!std::isfinite(c->rotation[i])) return "camera extrinsics have non-finite values";
    for (int i = 0; i < 3; ++i)
        if (!std::isfinite(c->translation[i]))
            return "camera extrinsics have non-finite values";
    const double* r = c->rotation;
    double worst = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += r[3 * k + i] * r[3 * k + j];
            worst = std::fmax(worst, std::fabs(acc - (i == j ? 1.0 : 0.0)));
        }
    if (worst > 1e-6) return "camera rotation is not orthonormal";
    const double det = r[0] * (r[4] * r[8] - r[5] * r[7]) - r[1] * (r[3] * r[8] - r[5] * r[6]) +
                       r[2] * (r[3] * r[7] - r[4] * r[6]);
    if (std::fabs(det - 1.0) > 1e-6) return "camera rotation determinant is not +1";
    if (!(c->focal > 0.0) || !std::isfinite(c->focal))
        return "camera focal length must be > 0";
    if (c->height < 1 || c->width < 1) return "camera image size must be at least 1x1";
    if (!std::isfinite(c->ox) || !std::isfinite(c->oy))
        return "camera principal point has non-finite values";
    return nullptr;
}

int validate_camera(gvr_context* ctx, const gvr_camera* c) {
    const char* e = camera_error(c);
    return e ? set_err(ctx, GVR_ERR_VALIDATION, "%s", e) : GVR_OK;
}

// SelectionConfig::validate (tracer.cpp:8-18), same messages.
int validate_cfg_ref(gvr_context* ctx, const gvr_selection* s) {
    if (!s) return set_err(ctx, GVR_ERR_VALIDATION, "selection config is null");
    if (!(s->eta > 0.0 && s->eta < 1.0)) return set_err(ctx, GVR_ERR_VALIDATION, "selection eta must be in (0, 1)");
    if (s->k_prime < 1) return set_err(ctx, GVR_ERR_VALIDATION, "selection k_prime must be >= 1");
    if (s->coarse_downsample < 1) return set_err(ctx, GVR_ERR_VALIDATION, "coarse downsample must be >= 1");
    return GVR_OK;
}

// ... plus the render path's K' limit.
int validate_cfg(gvr_context* ctx, const gvr_selection* s) {
    if (int rc = validate_cfg_ref(ctx, s)) return rc;
    if (s->k_prime > kMaxKPrime)
        return set_err(ctx, GVR_ERR_RUNTIME, "k_prime %d exceeds the CUDA backend limit of %d", s->k_prime, kMaxKPrime);
    return GVR_OK;
}

int copy_in(gvr_context* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return GVR_OK;
    const cudaMemcpyKind kind = is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CUDA_TRY(ctx, cudaMemcpyAsync(dst, src, bytes, kind, ctx->stream));
    return GVR_OK;
}

// Returns true in *host if a D2H copy was enqueued (caller must synchronise).
// Host destinations go on `hs` (the out stream of an async call, else the context stream).
int copy_out(gvr_context* ctx, void* dst, const void* src, size_t bytes, bool* host, cudaStream_t hs = nullptr) {
    if (!dst || bytes == 0) return GVR_OK;
    const bool dev = is_device_ptr(dst);
    CUDA_TRY(ctx, cudaMemcpyAsync(dst, src, bytes, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                  dev || !hs ? ctx->stream : hs));
    if (!dev) *host = true;
    return GVR_OK;
}

// Async host-buffer mode: the host copies of a call's outputs are forked onto the
// context's out stream (after everything the context stream has enqueued), so the
// next call of the step does not queue behind them; out_end records their event on
// the tape and out_wait makes the next call of the same kind (which rewrites the
// copied buffers) wait for it. Synchronous mode and graph capture: the context stream.
int out_begin(gvr_context* ctx, cudaStream_t* hs) {
    *hs = ctx->stream;
    if (!ctx->async || ctx->capturing) return GVR_OK;
    if (!ctx->out_stream) {
        CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->out_stream, cudaStreamNonBlocking));
        CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->out_fork, cudaEventDisableTiming));
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->out_fork, ctx->stream));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->out_stream, ctx->out_fork, 0));
    *hs = ctx->out_stream;
    return GVR_OK;
}

int out_end(gvr_context* ctx, gvr_tape* t, int kind, cudaStream_t hs) {
    if (hs == ctx->stream) return GVR_OK;
    if (!t->out_ev[kind]) CUDA_TRY(ctx, cudaEventCreateWithFlags(&t->out_ev[kind], cudaEventDisableTiming));
    CUDA_TRY(ctx, cudaEventRecord(t->out_ev[kind], hs));
    t->out_pending[kind] = true;
    return GVR_OK;
}

int out_wait(gvr_context* ctx, gvr_tape* t, int kind) {
    // (a capture cannot wait on work recorded before it: the caller synchronises first)
    if (!t->out_pending[kind] || ctx->capturing) return GVR_OK;
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, t->out_ev[kind], 0));
    t->out_pending[kind] = false;
    return GVR_OK;
}

cudaEvent_t take_event(gvr_context* ctx) {
    if (!ctx->ev_pool.empty()) {
        cudaEvent_t e = ctx->ev_pool.back();
        ctx->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// RAII bracket: records events around the enclosed launches when timing is on.
struct StageTimer {
    gvr_context* ctx;
    int stage;
    cudaEvent_t a = nullptr, b = nullptr;
    StageTimer(gvr_context* c, int st) : ctx(c), stage(st) {
        if (ctx->timing && !ctx->capturing) {
            a = take_event(ctx);
            b = take_event(ctx);
            cudaEventRecord(a, ctx->stream);
        }
    }
    ~StageTimer() {
        if (a) {
            cudaEventRecord(b, ctx->stream);
            ctx->ev_pending.push_back({stage, {a, b}});
        }
    }
};

void harvest_timings(gvr_context* ctx) {
    for (auto& pe : ctx->ev_pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, pe.second.first, pe.second.second) == cudaSuccess) {
            ctx->stage_ms[pe.first] += ms;
            ctx->stage_n[pe.first] += 1;
        }
        ctx->ev_pool.push_back(pe.second.first);
        ctx->ev_pool.push_back(pe.second.second);
    }
    ctx->ev_pending.clear();
    cudaGetLastError();
}

unsigned blocks_for(long long n, int threads) { return (unsigned)((n + threads - 1) / threads); }

template <int KMAX>
int launch_forward(gvr_context* ctx, const FwdParams& fp, int tiles) {
    const size_t list_smem = sizeof(unsigned long long) * (size_t)kSelListSmem;
    if (KMAX <= 32) {
        auto kern = select_warp_kernel<KMAX>;
        const size_t smem = sizeof(unsigned long long) * (size_t)kSelListSmem +
                            sizeof(unsigned long long) * (8 / GVR_SEL_SPLIT) * kWarpListCap;  // + per-warp lists
        CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        StageTimer st(ctx, ST_SELECT);
        kern<<<tiles * GVR_SEL_SPLIT, 256 / GVR_SEL_SPLIT, smem, ctx->stream>>>(fp);
    } else {
        constexpr int NT = 64;
        const size_t smem = sizeof(Cand) * NT + 12ull * KMAX * NT + list_smem;
        auto kern = select_kernel<KMAX>;
        CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        StageTimer st(ctx, ST_SELECT);
        kern<<<tiles, NT, smem, ctx->stream>>>(fp);
    }
    LAUNCH_CHECK(ctx);
    {
        const size_t smem = 32ull * KMAX * (64 / GVR_BLEND_SPLIT) + kBlendStageBytes;
        auto kern = blend_kernel<KMAX>;
        CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        StageTimer st(ctx, ST_BLEND);
        FwdParams bp = fp;
        if (KMAX > 32) bp.tile_done = nullptr;  // the CTA selection does not hand off per tile
        // with the per-tile hand-off the blend is a programmatic dependent of the
        // selection: its CTAs start on the SMs the selection's last wave leaves idle
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(tiles * GVR_BLEND_SPLIT);
        cfg.blockDim = dim3(256 / GVR_BLEND_SPLIT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = bp.tile_done ? 1 : 0;
        CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, kern, bp));
    }
    LAUNCH_CHECK(ctx);
    return GVR_OK;
}

template <int KMAX>
int launch_backward(gvr_context* ctx, const BwdParams& bp, int tiles) {
    const size_t smem = 36ull * KMAX * (64 / GVR_BWD_SPLIT);
    auto kern = backward_pixels_kernel<KMAX>;
    CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    {
        StageTimer st(ctx, ST_BACKWARD);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(tiles * GVR_BWD_SPLIT);
        cfg.blockDim = dim3(256 / GVR_BWD_SPLIT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;  // programmatic dependent of offsets_kernel (griddepcontrol.wait before the records)
        CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, kern, bp));
    }
    LAUNCH_CHECK(ctx);
    return GVR_OK;
}

// Grow-only buffer whose contents must start at zero (cleared when reallocated).
int ensure_zeroed(gvr_context* ctx, Buf& b, size_t bytes) {
    const void* before = b.p;
    CUDA_TRY(ctx, b.ensure(bytes));
    if (b.p != before) CUDA_TRY(ctx, cudaMemsetAsync(b.p, 0, b.cap, ctx->stream));
    return GVR_OK;
}

int sync_and_check(gvr_context* ctx) {
    if (ctx->capturing)
        return set_err(ctx, GVR_ERR_RUNTIME, "operation needs a host synchronisation; not allowed while capturing a graph");
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->out_stream) CUDA_TRY(ctx, cudaStreamSynchronize(ctx->out_stream));
    if (!ctx->ev_pending.empty()) harvest_timings(ctx);
    return GVR_OK;
}

// K0 on an uploaded scene (GaussianKernel::validate, types.cpp:17-29); one sync.
int decode_validation(gvr_context* ctx, unsigned long long h) {
    if (h == ~0ull) return GVR_OK;
    const long long k = (long long)(h >> 2);
    switch ((int)(h & 3)) {
        case 1: return set_err(ctx, GVR_ERR_VALIDATION, "kernel has non-finite values (kernel %lld)", k);
        case 2: return set_err(ctx, GVR_ERR_VALIDATION, "inv_cov is not symmetric (kernel %lld)", k);
        default: return set_err(ctx, GVR_ERR_VALIDATION, "inv_cov is not positive-definite (kernel %lld)", k);
    }
}

int validate_uploaded(gvr_context* ctx, gvr_scene* s) {
    const int K = s->K, D = s->D;
    if (K > 0) {
        unsigned long long* first = reinterpret_cast<unsigned long long*>(ctx->flags.as<int>() + 2);
        CUDA_TRY(ctx, cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), ctx->stream));
        validate_scene_kernel<<<blocks_for(K, 256), 256, 0, ctx->stream>>>(K, D, s->centers.as<double>(),
                                                                           s->inv_cov.as<double>(),
                                                                           s->attr.as<double>(), first);
        LAUNCH_CHECK(ctx);
        unsigned long long h = 0;
        CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_flags + 2, first, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
        if (int rc = sync_and_check(ctx)) return rc;
        std::memcpy(&h, ctx->h_flags + 2, sizeof h);
        return decode_validation(ctx, h);
    }
    return GVR_OK;
}

// Calibration: a long chain of independent FMAs per thread (8 chains) on the
// FP32 (kind 0) or FP64 (kind 1) pipe; returns achieved FLOP/s (FMA = 2).
template <typename T>
__global__ void fma_peak_kernel(T* out, int iters, T a, T b) {
    T x0 = (T)threadIdx.x, x1 = x0 + (T)1, x2 = x0 + (T)2, x3 = x0 + (T)3;
    T x4 = x0 + (T)4, x5 = x0 + (T)5, x6 = x0 + (T)6, x7 = x0 + (T)7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
            x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

}  // namespace

static int backward_impl(gvr_context* ctx, gvr_tape* t, const double* d_image, const double* d_alpha,
                         const gvr_grad_flags* flags, const gvr_gradients* out, bool accumulate,
                         double* packed = nullptr, double* packed_rt = nullptr);

extern "C" {

#ifndef GVR_SOURCE_HASH
#define GVR_SOURCE_HASH "unknown"
#endif
const char* gvr_build_hash(void) { return GVR_SOURCE_HASH; }

int gvr_context_create(int device, gvr_context** out) {
    if (!out) return GVR_ERR_RUNTIME;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) {
        cudaGetLastError();
        return GVR_ERR_RUNTIME;
    }
    if (cudaSetDevice(device) != cudaSuccess) return GVR_ERR_RUNTIME;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major < 10) return GVR_ERR_RUNTIME;
    auto* ctx = new gvr_context();
    ctx->device = device;
    if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return GVR_ERR_RUNTIME;
    }
    ctx->stream = ctx->own_stream;
    if (ctx->flags.ensure(64) != cudaSuccess || cudaMallocHost(&ctx->h_flags, 64) != cudaSuccess) {
        delete ctx;
        return GVR_ERR_RUNTIME;
    }
    *out = ctx;
    return GVR_OK;
}

void gvr_context_destroy(gvr_context* ctx) {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    harvest_timings(ctx);
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    ctx->flags.release();
    for (Buf& b : ctx->scratch) b.release();
    ctx->ptr_table.release();
    for (cudaStream_t w : ctx->workers) cudaStreamDestroy(w);
    for (cudaEvent_t e : ctx->join_ev) cudaEventDestroy(e);
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
    if (ctx->out_stream) {
        cudaStreamSynchronize(ctx->out_stream);
        cudaStreamDestroy(ctx->out_stream);
    }
    if (ctx->out_fork) cudaEventDestroy(ctx->out_fork);
    if (ctx->aux_tape) gvr_tape_destroy(ctx->aux_tape);
    if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

const char* gvr_last_error(const gvr_context* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int gvr_context_set_stream(gvr_context* ctx, void* s) {
    if (!ctx) return GVR_ERR_RUNTIME;
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
    return GVR_OK;
}

void* gvr_context_stream(gvr_context* ctx) { return ctx ? ctx->stream : nullptr; }

int gvr_context_synchronize(gvr_context* ctx) {
    if (!ctx) return GVR_ERR_RUNTIME;
    return sync_and_check(ctx);
}

int64_t gvr_context_launch_count(const gvr_context* ctx) { return ctx ? ctx->launches : 0; }
int64_t gvr_context_library_call_count(const gvr_context* ctx) { return ctx ? ctx->lib_calls : 0; }

int gvr_context_enable_timing(gvr_context* ctx, int on) {
    if (!ctx) return GVR_ERR_RUNTIME;
    if (int rc = sync_and_check(ctx)) return rc;
    ctx->timing = on != 0;
    for (int i = 0; i < ST_COUNT; ++i) {
        ctx->stage_ms[i] = 0.0;
        ctx->stage_n[i] = 0;
    }
    return GVR_OK;
}

int gvr_context_stage_times(gvr_context* ctx, double* ms, int64_t* count, int n) {
    if (!ctx) return GVR_ERR_RUNTIME;
    if (int rc = sync_and_check(ctx)) return rc;
    for (int i = 0; i < n && i < ST_COUNT; ++i) {
        if (ms) ms[i] = ctx->stage_ms[i];
        if (count) count[i] = ctx->stage_n[i];
    }
    return GVR_OK;
}

int gvr_measure_pipe_peak(gvr_context* ctx, int kind, double* flops) {
    if (!ctx || !flops) return GVR_ERR_RUNTIME;
    cudaDeviceProp prop;
    CUDA_TRY(ctx, cudaGetDeviceProperties(&prop, ctx->device));
    const int threads = 512, blocks = prop.multiProcessorCount * 4;
    const int iters = kind == 0 ? 4096 : 1024;
    void* out = nullptr;
    CUDA_TRY(ctx, cudaMalloc(&out, sizeof(double) * threads * blocks));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a, ctx->stream);
        if (kind == 0)
            fma_peak_kernel<float><<<blocks, threads, 0, ctx->stream>>>((float*)out, iters, 0.999f, 0.001f);
        else
            fma_peak_kernel<double><<<blocks, threads, 0, ctx->stream>>>((double*)out, iters, 0.999, 0.001);
        cudaEventRecord(b, ctx->stream);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    CUDA_TRY(ctx, cudaGetLastError());
    *flops = 2.0 * 8 * 16 * (double)iters * threads * blocks / (best * 1e-3);
    return GVR_OK;
}

// ---------------------------------------------------------------- ADAM (fit.cpp:20-42)

int gvr_adam_step_guarded(gvr_context* ctx, double* params, const double* grads, double* m, double* v, int64_t n,
                          int64_t step, double lr, double beta1, double beta2, double eps, const double* loss,
                          int32_t* diverged) {
    if (!ctx || step < 1 || n < 0 || !params || !grads || !m || !v) return GVR_ERR_RUNTIME;
    if (n == 0) return GVR_OK;
    if ((loss == nullptr) != (diverged == nullptr) || (loss && (!is_device_ptr(loss) || !is_device_ptr(diverged))))
        return set_err(ctx, GVR_ERR_RUNTIME, "gvr_adam_step_guarded needs device loss and diverged pointers");
    const double bc1 = 1.0 - std::pow(beta1, static_cast<double>(step));
    const double bc2 = 1.0 - std::pow(beta2, static_cast<double>(step));
    // host arrays (the C++ drop-in's AdamState) are staged through the context scratch
    double* arr[4] = {params, const_cast<double*>(grads), m, v};
    double* dev[4];
    bool host[4];
    const size_t bytes = sizeof(double) * (size_t)n;
    for (int i = 0; i < 4; ++i) {
        host[i] = !is_device_ptr(arr[i]);
        dev[i] = arr[i];
        if (host[i]) {
            if (ctx->capturing) return set_err(ctx, GVR_ERR_RUNTIME, "gvr_adam_step with host arrays is not capturable");
            CUDA_TRY(ctx, ctx->scratch[i].ensure(bytes));
            dev[i] = ctx->scratch[i].as<double>();
            CUDA_TRY(ctx, cudaMemcpyAsync(dev[i], arr[i], bytes, cudaMemcpyHostToDevice, ctx->stream));
        }
    }
    adam_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(n, dev[0], dev[1], dev[2], dev[3], lr, beta1, beta2, eps,
                                                             bc1, bc2, loss, diverged);
    LAUNCH_CHECK(ctx);
    bool any = false;
    for (int i : {0, 2, 3})
        if (host[i]) {
            CUDA_TRY(ctx, cudaMemcpyAsync(arr[i], dev[i], bytes, cudaMemcpyDeviceToHost, ctx->stream));
            any = true;
        }
    return any ? sync_and_check(ctx) : GVR_OK;
}

int gvr_adam_step(gvr_context* ctx, double* params, const double* grads, double* m, double* v, int64_t n,
                  int64_t step, double lr, double beta1, double beta2, double eps) {
    return gvr_adam_step_guarded(ctx, params, grads, m, v, n, step, lr, beta1, beta2, eps, nullptr, nullptr);
}

// ---------------------------------------------------------------- CUDA graphs

int gvr_graph_begin(gvr_context* ctx) {
    if (!ctx || ctx->capturing) return GVR_ERR_RUNTIME;
    if (int rc = sync_and_check(ctx)) return rc;
    CUDA_TRY(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    ctx->capturing = true;
    ctx->capture_launch0 = ctx->launches;
    return GVR_OK;
}

int gvr_graph_end(gvr_context* ctx, gvr_graph** out) {
    if (!ctx || !ctx->capturing || !out) return GVR_ERR_RUNTIME;
    ctx->capturing = false;
    cudaGraph_t g = nullptr;
    CUDA_TRY(ctx, cudaStreamEndCapture(ctx->stream, &g));
    auto* gr = new gvr_graph();
    gr->ctx = ctx;
    gr->graph = g;
    gr->launches = ctx->launches - ctx->capture_launch0;
    cudaError_t e = cudaGraphInstantiate(&gr->exec, g, 0);
    if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        delete gr;
        return set_err(ctx, GVR_ERR_RUNTIME, "graph instantiation failed: %s", cudaGetErrorString(e));
    }
    *out = gr;
    return GVR_OK;
}

int gvr_graph_launch(gvr_context* ctx, gvr_graph* g) {
    if (!ctx || !g || g->ctx != ctx) return GVR_ERR_RUNTIME;
    CUDA_TRY(ctx, cudaGraphLaunch(g->exec, ctx->stream));
    ctx->launches += g->launches;
    return GVR_OK;
}

void gvr_graph_destroy(gvr_graph* g) {
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
}

int gvr_context_set_tile_capacity(gvr_context* ctx, int cap) {
    if (!ctx || cap < 0) return GVR_ERR_RUNTIME;
    ctx->pool_override = cap;
    return GVR_OK;
}

int gvr_context_set_list_smem(gvr_context* ctx, int n) {
    if (!ctx || n < 0) return GVR_ERR_RUNTIME;
    ctx->list_smem = std::min(n, kSelListSmem);
    return GVR_OK;
}

int gvr_context_set_async(gvr_context* ctx, int on) {
    if (!ctx) return GVR_ERR_RUNTIME;
    if (int rc = sync_and_check(ctx)) return rc;
    ctx->async = on != 0;
    return GVR_OK;
}

int gvr_context_set_precise(gvr_context* ctx, int on) {
    if (!ctx) return GVR_ERR_RUNTIME;
    ctx->precise = on != 0;
    return GVR_OK;
}

int gvr_camera_validate(const gvr_camera* camera, char* msg, int32_t msg_cap) {
    const char* e = camera_error(camera);
    if (!e) return GVR_OK;
    if (msg && msg_cap > 0) std::snprintf(msg, (size_t)msg_cap, "%s", e);
    return GVR_ERR_VALIDATION;
}

int gvr_context_set_tile_profile(gvr_context* ctx, int on) {
    if (!ctx) return GVR_ERR_RUNTIME;
    ctx->tile_profile = on != 0;
    return GVR_OK;
}

int gvr_context_set_prefilter_guard(gvr_context* ctx, double guard) {
    if (!ctx || !(guard >= 0.0)) return GVR_ERR_RUNTIME;
    ctx->guard = guard;
    return GVR_OK;
}

// ---------------------------------------------------------------- scene

int gvr_scene_create(gvr_context* ctx, gvr_scene** out) {
    if (!ctx || !out) return GVR_ERR_RUNTIME;
    auto* s = new gvr_scene();
    s->ctx = ctx;
    *out = s;
    return GVR_OK;
}

void gvr_scene_destroy(gvr_scene* s) {
    if (!s) return;
    cudaStreamSynchronize(s->ctx->stream);
    s->centers.release();
    s->inv_cov.release();
    s->attr.release();
    s->vflag.release();
    delete s;
}

int32_t gvr_scene_size(const gvr_scene* s) { return s ? s->K : 0; }
int32_t gvr_scene_attr_dim(const gvr_scene* s) { return s ? s->D : 0; }

int gvr_scene_set(gvr_context* ctx, gvr_scene* s, int32_t K, int32_t D, double tau, const double* centers,
                  const double* inv_cov, const double* attr) {
    if (!ctx || !s) return GVR_ERR_RUNTIME;
    if (ctx->async) return gvr_scene_set_deferred(ctx, s, K, D, tau, centers, inv_cov, attr);
    s->valid = false;
    s->deferred = false;
    ++s->version;
    if (K < 0 || D < 0) return set_err(ctx, GVR_ERR_VALIDATION, "scene sizes must be >= 0");
    // GaussianScene::validate order: tau first, then kernels (types.cpp:31-42)
    if (tau < 0.0 || !std::isfinite(tau)) return set_err(ctx, GVR_ERR_VALIDATION, "tau must be finite and >= 0");
    if (K > 0 && (!centers || !inv_cov || (D > 0 && !attr)))
        return set_err(ctx, GVR_ERR_RUNTIME, "scene arrays must not be null");
    CUDA_TRY(ctx, s->centers.ensure(sizeof(double) * 3 * (size_t)K));
    CUDA_TRY(ctx, s->inv_cov.ensure(sizeof(double) * 9 * (size_t)K));
    CUDA_TRY(ctx, s->attr.ensure(sizeof(double) * (size_t)D * K));
    if (int rc = copy_in(ctx, s->centers.p, centers, sizeof(double) * 3 * (size_t)K)) return rc;
    if (int rc = copy_in(ctx, s->inv_cov.p, inv_cov, sizeof(double) * 9 * (size_t)K)) return rc;
    if (int rc = copy_in(ctx, s->attr.p, attr, sizeof(double) * (size_t)D * K)) return rc;
    s->K = K;
    s->D = D;
    s->tau = tau;
    if (int rc = validate_uploaded(ctx, s)) return rc;
    s->valid = true;
    return GVR_OK;
}

int gvr_scene_set_deferred(gvr_context* ctx, gvr_scene* s, int32_t K, int32_t D, double tau, const double* centers,
                           const double* inv_cov, const double* attr) {
    if (!ctx || !s) return GVR_ERR_RUNTIME;
    s->valid = false;
    s->deferred = false;
    ++s->version;
    if (K < 0 || D < 0) return set_err(ctx, GVR_ERR_VALIDATION, "scene sizes must be >= 0");
    if (tau < 0.0 || !std::isfinite(tau)) return set_err(ctx, GVR_ERR_VALIDATION, "tau must be finite and >= 0");
    if (K > 0 && (!centers || !inv_cov || (D > 0 && !attr)))
        return set_err(ctx, GVR_ERR_RUNTIME, "scene arrays must not be null");
    const size_t need[4] = {sizeof(double) * 3 * (size_t)K, sizeof(double) * 9 * (size_t)K, sizeof(double) * (size_t)D * K,
                            sizeof(unsigned long long)};
    Buf* bufs[4] = {&s->centers, &s->inv_cov, &s->attr, &s->vflag};
    for (int b = 0; b < 4; ++b) {
        if (ctx->capturing && bufs[b]->cap < need[b])
            return set_err(ctx, GVR_ERR_RUNTIME, "scene buffers must be sized by an uncaptured call first");
        CUDA_TRY(ctx, bufs[b]->ensure(need[b]));
    }
    if (int rc = copy_in(ctx, s->centers.p, centers, need[0])) return rc;
    if (int rc = copy_in(ctx, s->inv_cov.p, inv_cov, need[1])) return rc;
    if (int rc = copy_in(ctx, s->attr.p, attr, need[2])) return rc;
    s->K = K;
    s->D = D;
    s->tau = tau;
    CUDA_TRY(ctx, cudaMemsetAsync(s->vflag.p, 0xff, sizeof(unsigned long long), ctx->stream));
    if (K > 0) {
        validate_scene_kernel<<<blocks_for(K, 256), 256, 0, ctx->stream>>>(
            K, D, s->centers.as<double>(), s->inv_cov.as<double>(), s->attr.as<double>(),
            s->vflag.as<unsigned long long>());
        LAUNCH_CHECK(ctx);
    }
    s->valid = true;  // provisional: gvr_scene_check reports the validation result
    s->deferred = true;
    return GVR_OK;
}

int gvr_scene_check(gvr_context* ctx, gvr_scene* s) {
    if (!ctx || !s) return GVR_ERR_RUNTIME;
    // the flag is re-read on every check: a captured upload re-validates on every replay
    if (!s->deferred) return s->valid ? GVR_OK : set_err(ctx, GVR_ERR_RUNTIME, "scene is not valid");
    if (ctx->capturing)
        return set_err(ctx, GVR_ERR_RUNTIME, "operation needs a host synchronisation; not allowed while capturing a graph");
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_flags + 2, s->vflag.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                  ctx->stream));
    if (int rc = sync_and_check(ctx)) return rc;
    unsigned long long h = 0;
    std::memcpy(&h, ctx->h_flags + 2, sizeof h);
    const int rc = decode_validation(ctx, h);
    s->valid = rc == GVR_OK;
    return rc;
}

// ---------------------------------------------------------------- tape / forward

int gvr_tape_create(gvr_context* ctx, gvr_tape** out) {
    if (!ctx || !out) return GVR_ERR_RUNTIME;
    auto* t = new gvr_tape();
    t->ctx = ctx;
    if (t->flags.ensure(64) != cudaSuccess || cudaMallocHost(&t->h_flags, 64) != cudaSuccess) {
        t->flags.release();
        delete t;
        return set_err(ctx, GVR_ERR_RUNTIME, "tape allocation failed");
    }
    std::memset(t->h_flags, 0, 64);
    *out = t;
    return GVR_OK;
}

void gvr_tape_destroy(gvr_tape* t) {
    if (!t) return;
    cudaStreamSynchronize(t->ctx->stream);
    Buf* bufs[] = {&t->rec32, &t->rec64, &t->tile_count, &t->tile_off, &t->tile_fill, &t->pool, &t->sorted_pool,
                   &t->tile_cycles, &t->tile_hint, &t->sched, &t->topk, &t->count, &t->image, &t->alpha,
                   &t->depth, &t->topk_w, &t->tape_t, &t->ent, &t->ent_a, &t->d_image, &t->d_alpha, &t->acc, &t->d_attr, &t->d_center,
                   &t->d_inv_cov, &t->d_rt, &t->stage_i, &t->stage_w, &t->flags, &t->attr_fb, &t->kinfo,
                   &t->masks, &t->slot_off, &t->app, &t->bent, &t->bkey, &t->rays, &t->pieces, &t->kcount, &t->rt_part, &t->tickets,
                   &t->loss_part};
    for (Buf* b : bufs) b->release();
    if (t->h_flags) cudaFreeHost(t->h_flags);
    if (t->ctx->out_stream) cudaStreamSynchronize(t->ctx->out_stream);
    for (cudaEvent_t e : t->out_ev)
        if (e) cudaEventDestroy(e);
    delete t;
}

int gvr_tape_shape(const gvr_tape* t, int32_t* h, int32_t* w, int32_t* kp, int32_t* d) {
    if (!t || !t->valid) return GVR_ERR_RUNTIME;
    if (h) *h = t->H;
    if (w) *w = t->W;
    if (kp) *kp = t->cfg.k_prime;
    if (d) *d = t->D;
    return GVR_OK;
}

int gvr_render(gvr_context* ctx, const gvr_scene* scene, const gvr_camera* camera, const gvr_selection* cfg,
               gvr_tape* tape, const gvr_render_outputs* out) {
    return gvr_render_shard(ctx, scene, camera, cfg, tape, out, 0, 1);
}

}  // extern "C"

// Enqueues one render on ctx->stream. Host outputs are copied asynchronously;
// *host_out is set when the caller must synchronise (then check the tape's
// nonfinite flag, mirrored into tape->h_flags[1]).
static int render_impl(gvr_context* ctx, const gvr_scene* scene, const gvr_camera* camera, const gvr_selection* cfg,
                       gvr_tape* tape, const gvr_render_outputs* out, int32_t shard, int32_t nshards, bool* host_out) {
    *host_out = false;
    if (!ctx || !scene || !tape) return GVR_ERR_RUNTIME;
    if (nshards < 1 || shard < 0 || shard >= nshards)
        return set_err(ctx, GVR_ERR_RUNTIME, "bad tile shard %d of %d", shard, nshards);
    if (tape->ctx != ctx || scene->ctx != ctx) return set_err(ctx, GVR_ERR_RUNTIME, "objects belong to another context");
    if (!scene->valid) return set_err(ctx, GVR_ERR_VALIDATION, "scene has not been validated");
    if (int rc = validate_camera(ctx, camera)) return rc;
    if (int rc = validate_cfg(ctx, cfg)) return rc;
    if (int rc = out_wait(ctx, tape, 0)) return rc;  // the last render's host copies read image / alpha / depth
    tape->valid = false;
    tape->has_upstream = false;

    const int K = scene->K, D = scene->D, H = camera->height, W = camera->width;
    const int Dc = D > 1 ? D : 1;
    const int kp = cfg->k_prime;
    const long long P = (long long)H * W;
    const int tile = kFwdTile;
    const int tiles_x = (W + tile - 1) / tile, tiles_y = (H + tile - 1) / tile;
    const int tiles = tiles_x * tiles_y;

    tape->scene = scene;
    tape->scene_version = scene->version;
    tape->cam = *camera;
    tape->cfg = *cfg;
    tape->K = K;
    tape->D = D;
    tape->H = H;
    tape->W = W;
    tape->tile = tile;
    tape->tiles_x = tiles_x;
    tape->tiles_y = tiles_y;

    CameraP cp;
    std::memcpy(cp.R, camera->rotation, sizeof cp.R);
    std::memcpy(cp.T, camera->translation, sizeof cp.T);
    cp.focal = camera->focal;
    cp.ox = camera->ox;
    cp.oy = camera->oy;
    cp.H = H;
    cp.W = W;
    SelP sp;
    sp.eta = cfg->eta;
    sp.log_eta = std::log(cfg->eta);
    sp.chi = 2.0 * std::log(1.0 / cfg->eta);
    sp.kp = kp;
    sp.coarse = cfg->coarse_enabled ? 1 : 0;
    sp.ds = cfg->coarse_downsample;
    tape->camp = cp;
    tape->selp = sp;

    CUDA_TRY(ctx, tape->rec32.ensure(sizeof(Rec32) * (size_t)(K > 0 ? K : 1)));
    CUDA_TRY(ctx, tape->rec64.ensure(sizeof(Rec64) * (size_t)(K > 0 ? K : 1)));
    // Tile lists live in one pool laid out by a count pass + scan. Its size is
    // not known on the host before the render, so the pool is sized from an
    // estimate and from the totals of earlier renders on this tape (grow-only);
    // lists that do not fit are streamed (every kernel, exact tests, no early
    // exit) and counted (gvr_tape_list_stats); host-synchronous renders grow
    // the pool and re-render instead.
    {
        tape->pool_hint = std::max<long long>(tape->pool_hint, tape->h_flags[kListStats]);
        const long long est = std::max<long long>(1 << 18, (4LL * K + 64LL * tiles) / nshards);
        const long long want = std::max(est, tape->pool_hint + tape->pool_hint / 4);
        if (!ctx->capturing || tape->pool.cap == 0)
            CUDA_TRY(ctx, tape->pool.ensure(sizeof(unsigned long long) * (size_t)want));
        if (!ctx->capturing || tape->sorted_pool.cap == 0)
            CUDA_TRY(ctx, tape->sorted_pool.ensure(sizeof(unsigned long long) * (size_t)want));
    }
    // (2 entries of slack at the end: the selection's bulk copies read 16-byte aligned spans)
    const long long pool_cap = std::min<long long>(
        {(long long)(tape->pool.cap / sizeof(unsigned long long)) - 2, (long long)(tape->sorted_pool.cap / sizeof(unsigned long long)),
         0x7fffffffLL, ctx->pool_override > 0 ? ctx->pool_override : 0x7fffffffLL});
    // mask rectangles of the deterministic backward: one 8-byte pixel mask per
    // (kernel, tile of its box), sized like the pool (estimate / earlier totals)
    {
        tape->mask_hint = std::max<long long>(tape->mask_hint, tape->h_flags[kMaskTotal]);
        const long long est = std::max<long long>(1 << 18, 4LL * K + 64LL * tiles);
        const long long want = std::max(est, tape->mask_hint + tape->mask_hint / 4);
        if (!ctx->capturing || tape->masks.cap == 0) {
            CUDA_TRY(ctx, tape->masks.ensure(sizeof(unsigned long long) * (size_t)want));
        }
        CUDA_TRY(ctx, tape->kinfo.ensure(sizeof(int4) * (size_t)(K > 0 ? K : 1)));
        CUDA_TRY(ctx, tape->kcount.ensure(sizeof(int) * ((size_t)(K > 0 ? K : 1) + (K + kScanThreads - 1) / kScanThreads + 1)));
    }
    const long long mask_cap = std::min<long long>({(long long)(tape->masks.cap / sizeof(unsigned long long)), 0x7fffffffLL,
                                                    ctx->pool_override > 0 ? ctx->pool_override : 0x7fffffffLL});
    CUDA_TRY(ctx, tape->tile_count.ensure(sizeof(int) * 2 * (size_t)tiles));
    CUDA_TRY(ctx, tape->tile_off.ensure(sizeof(int) * (size_t)tiles));
    CUDA_TRY(ctx, tape->sched.ensure(sizeof(int) * (2 + 2 * (size_t)tiles)));
    CUDA_TRY(ctx, tape->topk.ensure(sizeof(int) * (size_t)P * kp));
    CUDA_TRY(ctx, tape->count.ensure(sizeof(int) * (size_t)P));
    CUDA_TRY(ctx, tape->tape_t.ensure(sizeof(double) * (size_t)P * kp));
    CUDA_TRY(ctx, tape->ent.ensure(sizeof(EntryRec) * (size_t)P * kp));
    CUDA_TRY(ctx, tape->ent_a.ensure(sizeof(double) * (size_t)P * kp));
    CUDA_TRY(ctx, tape->image.ensure(sizeof(double) * (size_t)P * Dc));
    CUDA_TRY(ctx, tape->alpha.ensure(sizeof(double) * (size_t)P));
    CUDA_TRY(ctx, tape->depth.ensure(sizeof(double) * (size_t)P));
    const bool want_w = out && out->topk_w;
    if (want_w) CUDA_TRY(ctx, tape->topk_w.ensure(sizeof(double) * (size_t)P * kp));

    int* dflags = tape->flags.as<int>();
    int* tile_count = tape->tile_count.as<int>();
    int* sched = tape->sched.as<int>();
    int* order_f = sched + 2;
    int* tile_fill = tile_count + tiles;  // emit cursors, contiguous with the counts
    // flags, tile counts + emit cursors, the per-tile selection hand-off flags:
    // cleared by one launch (instead of memset nodes). (Clearing the outputs here
    // too, so that the blend visits only the selected tiles: C2 +4 µs, C4 -4 µs.)
    {
        ClearList cl{};
        long long words = 0;
        auto add = [&](void* ptr, long long n) {
            cl.ptr[cl.m] = static_cast<int*>(ptr);
            cl.n[cl.m++] = n;
            words += n;
        };
        add(dflags, 16);
        add(tile_count, 2LL * tiles);
        add(sched + 2 + (size_t)tiles, tiles);
        clear_kernel<<<std::min<unsigned>(blocks_for(words, 256), 148 * 8), 256, 0, ctx->stream>>>(cl);
    }
    LAUNCH_CHECK(ctx);

    if (K > 0) {
        // K1 projection + culling + binning into per-tile lists
        ProjectParams pp{};
        pp.K = K;
        pp.centers = scene->centers.as<double>();
        pp.inv_cov = scene->inv_cov.as<double>();
        pp.cam = cp;
        pp.sel = sp;
        pp.tile = tile;
        pp.tiles_x = tiles_x;
        pp.tiles_y = tiles_y;
        pp.rec32 = tape->rec32.as<Rec32>();
        pp.rec64 = tape->rec64.as<Rec64>();
        pp.tile_count = tile_count;
        pp.shard = shard;
        pp.nshards = nshards;
        pp.kinfo = tape->kinfo.as<int4>();
        pp.masks = tape->masks.as<unsigned long long>();
        pp.mask_total = dflags + kMaskTotal;
        pp.mask_cap = (int)mask_cap;
        pp.dropped_behind = dflags;
        {
            StageTimer st(ctx, ST_PROJECT);
            project_kernel<<<blocks_for(K, 128), 128, 0, ctx->stream>>>(pp);
        }
        LAUNCH_CHECK(ctx);
    }

    // K3 over the non-empty tiles, longest first: by the last render's selection
    // cycles when this tape rendered the same view before, else by list length
    const bool use_hint = tape->hint_valid && tape->hint_tiles == tiles && tape->hint_shard == shard &&
                          tape->hint_nshards == nshards && std::memcmp(&tape->hint_cam, &cp, sizeof cp) == 0;
    const bool want_hint = kp <= 32;  // the warp selection measures it
    if (want_hint) CUDA_TRY(ctx, tape->tile_hint.ensure(sizeof(unsigned) * (size_t)tiles));
    {
        StageTimer st(ctx, ST_RANGES);
        const size_t osmem = tiles <= kOrderSmemTiles ? 6ull * (size_t)tiles : 0;
        CUDA_TRY(ctx, cudaFuncSetAttribute(order_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(6ull * kOrderSmemTiles)));
        order_tiles_kernel<<<1, 1024, osmem, ctx->stream>>>(tiles, tile_count, order_f, sched, shard, nshards,
                                                        sched + 1, tape->tile_off.as<int>(),
                                                        (int)pool_cap, ctx->list_smem, dflags + kListStats,
                                                        use_hint ? tape->tile_hint.as<unsigned>() : nullptr);
    }
    LAUNCH_CHECK(ctx);
    if (K > 0) {
        // K2 emit: fill the laid-out tile lists
        EmitParams ep;
        ep.K = K;
        ep.rec32 = tape->rec32.as<Rec32>();
        ep.H = H;
        ep.W = W;
        ep.tile = tile;
        ep.tiles_x = tiles_x;
        ep.tile_off = tape->tile_off.as<int>();
        ep.tile_fill = tile_fill;
        ep.pool = tape->pool.as<unsigned long long>();
        {
            StageTimer st(ctx, ST_EMIT);
            emit_kernel<<<blocks_for(K, 128), 128, 0, ctx->stream>>>(ep);
        }
        LAUNCH_CHECK(ctx);
    }
    FwdParams fp{};
    fp.cam = cp;
    fp.sel = sp;
    fp.D = D;
    fp.Dc = Dc;
    fp.tau = scene->tau;
    fp.guard_abs = (float)ctx->guard;
    fp.prefilter_c1 = 1.0f - 1e-4f;
    {
        const float neg_log_eta = -(float)sp.log_eta;
        fp.qc.c_rej = 2.0f * (neg_log_eta + fp.guard_abs);
        fp.qc.c_acc = 2.0f * (neg_log_eta - fp.guard_abs);
        fp.qc.slack_lo = fp.prefilter_c1;
        fp.qc.slack_hi = 2.0f - fp.prefilter_c1;
        fp.qc.f = (float)cp.focal;
        fp.qc.inv_f = (float)(1.0 / cp.focal);
    }
    fp.exact_only = ctx->guard > 1e3 ? 1 : 0;
    fp.tiles_x = tiles_x;
    fp.tile_order = order_f;
    fp.n_order = sched;
    fp.tile_order_blend = order_f;
    fp.n_order_blend = sched + 1;  // all tiles: selected first, then cleared ones
    fp.tile_count = tile_count;
    fp.tile_off = tape->tile_off.as<int>();
    fp.pool = tape->pool.as<unsigned long long>();
    fp.sorted_pool = tape->sorted_pool.as<unsigned long long>();
    fp.list_smem = ctx->list_smem;
    fp.K = K;
    fp.rec32 = tape->rec32.as<Rec32>();
    fp.rec64 = tape->rec64.as<Rec64>();
    fp.attr = scene->attr.as<double>();
    fp.image = tape->image.as<double>();
    fp.alpha = tape->alpha.as<double>();
    fp.depth = tape->depth.as<double>();
    fp.topk = tape->topk.as<int>();
    fp.count = tape->count.as<int>();
    fp.topk_w = want_w ? tape->topk_w.as<double>() : nullptr;
    fp.tape_t = tape->tape_t.as<double>();
    fp.ent = tape->ent.as<EntryRec>();
    fp.ent_a = tape->ent_a.as<double>();
    fp.nonfinite = dflags + 1;
    fp.kinfo = tape->kinfo.as<int4>();
    fp.masks = tape->masks.as<unsigned long long>();
    fp.presorted = kp <= 32 ? 1 : 0;  // select_warp_kernel emits the exact (l, idx) order
    fp.precise = ctx->precise ? 1 : 0;
    fp.tile_cycles = nullptr;
    fp.tile_done = GVR_PDL ? reinterpret_cast<unsigned*>(sched + 2 + (size_t)tiles) : nullptr;
    fp.tile_hint = want_hint ? tape->tile_hint.as<unsigned>() : nullptr;
    tape->hint_valid = want_hint;
    tape->hint_cam = cp;
    tape->hint_tiles = tiles;
    tape->hint_shard = shard;
    tape->hint_nshards = nshards;
    tape->profiled = ctx->tile_profile;
    if (ctx->tile_profile) {
        CUDA_TRY(ctx, tape->tile_cycles.ensure(sizeof(long long) * (size_t)tiles));
        CUDA_TRY(ctx, cudaMemsetAsync(tape->tile_cycles.p, 0, sizeof(long long) * (size_t)tiles, ctx->stream));
        fp.tile_cycles = tape->tile_cycles.as<long long>();
    }
    int rc = GVR_OK;
    if (kp <= 8) rc = launch_forward<8>(ctx, fp, tiles);
    else if (kp <= 16) rc = launch_forward<16>(ctx, fp, tiles);
    else if (kp <= 20) rc = launch_forward<20>(ctx, fp, tiles);
    else if (kp <= 24) rc = launch_forward<24>(ctx, fp, tiles);
    else if (kp <= 32) rc = launch_forward<32>(ctx, fp, tiles);
    else if (kp <= 48) rc = launch_forward<48>(ctx, fp, tiles);
    else if (kp <= 64) rc = launch_forward<64>(ctx, fp, tiles);
    else if (kp <= 96) rc = launch_forward<96>(ctx, fp, tiles);
    else rc = launch_forward<128>(ctx, fp, tiles);
    if (rc) return rc;

    tape->valid = true;
    if (!ctx->capturing)  // sizing hint for the next render (read without a sync: a stale value is harmless)
        CUDA_TRY(ctx, cudaMemcpyAsync(tape->h_flags + kListStats, dflags + kListStats, 5 * sizeof(int),
                                      cudaMemcpyDeviceToHost, ctx->stream));

    if (out) {
        bool host = false;
        cudaStream_t hs;
        if ((rc = out_begin(ctx, &hs))) return rc;
        if ((rc = copy_out(ctx, out->image, tape->image.p, sizeof(double) * P * Dc, &host, hs))) return rc;
        if ((rc = copy_out(ctx, out->alpha, tape->alpha.p, sizeof(double) * P, &host, hs))) return rc;
        if ((rc = copy_out(ctx, out->depth, tape->depth.p, sizeof(double) * P, &host, hs))) return rc;
        if (out->topk_idx || out->topk_w) {
            const bool dev_i = !out->topk_idx || is_device_ptr(out->topk_idx);
            const bool dev_w = !out->topk_w || is_device_ptr(out->topk_w);
            int* oi = out->topk_idx;
            double* ow = out->topk_w;
            if (!dev_i) {
                CUDA_TRY(ctx, tape->stage_i.ensure(sizeof(int) * (size_t)P * kp));
                oi = tape->stage_i.as<int>();
            }
            if (!dev_w) {
                CUDA_TRY(ctx, tape->stage_w.ensure(sizeof(double) * (size_t)P * kp));
                ow = tape->stage_w.as<double>();
            }
            expand_topk_kernel<<<blocks_for(P * kp, 256), 256, 0, ctx->stream>>>(
                P, kp, tape->topk.as<int>(), tape->count.as<int>(), tape->topk_w.as<double>(), oi, ow);
            LAUNCH_CHECK(ctx);
            if (!dev_i) CUDA_TRY(ctx, cudaMemcpyAsync(out->topk_idx, oi, sizeof(int) * (size_t)P * kp,
                                                      cudaMemcpyDeviceToHost, ctx->stream));
            if (!dev_w) CUDA_TRY(ctx, cudaMemcpyAsync(out->topk_w, ow, sizeof(double) * (size_t)P * kp,
                                                      cudaMemcpyDeviceToHost, ctx->stream));
            host = host || !dev_i || !dev_w;
        }
        if ((rc = out_end(ctx, tape, 0, hs))) return rc;
        if (host) {
            CUDA_TRY(ctx, cudaMemcpyAsync(tape->h_flags + 1, dflags + 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
            *host_out = true;
        }
    }
    return GVR_OK;
}

// validate_finite (blender.cpp:132-134) after the host copy-out has completed.
static int check_finite(gvr_context* ctx, gvr_tape* tape) {
    if (tape->h_flags[1]) {
        tape->valid = false;
        return set_err(ctx, GVR_ERR_VALIDATION, "image contains non-finite values");
    }
    return GVR_OK;
}

extern "C" int gvr_render_shard(gvr_context* ctx, const gvr_scene* scene, const gvr_camera* camera,
                                const gvr_selection* cfg, gvr_tape* tape, const gvr_render_outputs* out, int32_t shard,
                                int32_t nshards) {
    bool host = false;
    if (int rc = render_impl(ctx, scene, camera, cfg, tape, out, shard, nshards, &host)) return rc;
    if (!host || ctx->async) return GVR_OK;  // async: gvr_context_synchronize + gvr_tape_check_finite
    if (int rc = sync_and_check(ctx)) return rc;
    if ((tape->h_flags[kListStats + 2] > 0 && ctx->pool_override == 0) ||
        ((long long)tape->h_flags[kMaskTotal] > (long long)(tape->masks.cap / sizeof(unsigned long long)) &&
         ctx->pool_override == 0)) {
        // some tile lists / mask rectangles did not fit: size them from this render's totals and render again
        tape->pool_hint = std::max<long long>(tape->pool_hint, tape->h_flags[kListStats]);
        tape->mask_hint = std::max<long long>(tape->mask_hint, tape->h_flags[kMaskTotal]);
        if (int rc = render_impl(ctx, scene, camera, cfg, tape, out, shard, nshards, &host)) return rc;
        if (int rc = sync_and_check(ctx)) return rc;
    }
    return check_finite(ctx, tape);
}

extern "C" {

int gvr_tape_traced(gvr_context* ctx, const gvr_tape* t, int32_t* idx, double* l, double* q, double* sigma) {
    if (!ctx || !t || !t->valid) return set_err(ctx, GVR_ERR_RUNTIME, "tape is not valid");
    if (t->ctx != ctx) return set_err(ctx, GVR_ERR_RUNTIME, "objects belong to another context");
    const long long P = (long long)t->H * t->W;
    const int kp = t->cfg.k_prime;
    const size_t n = (size_t)P * kp;
    // stage everything on device, then copy out
    Buf si, sl, sq, ss;
    CUDA_TRY(ctx, si.ensure(sizeof(int) * n));
    CUDA_TRY(ctx, sl.ensure(sizeof(double) * n));
    CUDA_TRY(ctx, sq.ensure(sizeof(double) * n));
    CUDA_TRY(ctx, ss.ensure(sizeof(double) * n));
    traced_kernel<<<blocks_for((long long)n, 256), 256, 0, ctx->stream>>>(
        t->camp, kp, t->topk.as<int>(), t->count.as<int>(), t->rec64.as<Rec64>(), si.as<int>(), sl.as<double>(),
        sq.as<double>(), ss.as<double>());
    LAUNCH_CHECK(ctx);
    bool host = false;
    int rc;
    if ((rc = copy_out(ctx, idx, si.p, sizeof(int) * n, &host))) return rc;
    if ((rc = copy_out(ctx, l, sl.p, sizeof(double) * n, &host))) return rc;
    if ((rc = copy_out(ctx, q, sq.p, sizeof(double) * n, &host))) return rc;
    if ((rc = copy_out(ctx, sigma, ss.p, sizeof(double) * n, &host))) return rc;
    rc = sync_and_check(ctx);
    si.release();
    sl.release();
    sq.release();
    ss.release();
    return rc;
}

// ---------------------------------------------------------------- loss / backward

}  // extern "C"

// ScalarLoss on ctx->stream; the loss lands in the tape (flags + 8 B) and, when
// loss_dev is given, is also added into *loss_dev (zeroed first). *host_out
// set when host copies are pending (caller synchronises).
static int scalar_loss_impl(gvr_context* ctx, gvr_tape* t, const double* target_image, const double* target_alpha,
                            double w_image, double w_alpha, double* loss_out, double* d_image_out, double* d_alpha_out,
                            bool* host_out) {
    *host_out = false;
    if (!ctx || !t || !t->valid) return set_err(ctx, GVR_ERR_RUNTIME, "tape is not valid");
    if (t->ctx != ctx) return set_err(ctx, GVR_ERR_RUNTIME, "objects belong to another context");
    if (!target_image || !target_alpha) return set_err(ctx, GVR_ERR_RUNTIME, "targets must not be null");
    if (int rc = out_wait(ctx, t, 1)) return rc;  // the last loss's host copies read d_image / d_alpha
    const long long P = (long long)t->H * t->W;
    const int Dc = t->D > 1 ? t->D : 1;
    const long long n_img = P * Dc;
    CUDA_TRY(ctx, t->d_image.ensure(sizeof(double) * (size_t)(n_img + P) * 2));
    CUDA_TRY(ctx, t->d_alpha.ensure(sizeof(double) * (size_t)P));
    double* timg = t->d_image.as<double>() + n_img;  // target staging after the gradient
    double* talpha = timg + 0;                       // alpha target staged after the image target
    const double* ti = target_image;
    const double* ta = target_alpha;
    if (!is_device_ptr(target_image)) {
        CUDA_TRY(ctx, cudaMemcpyAsync(timg, target_image, sizeof(double) * n_img, cudaMemcpyHostToDevice, ctx->stream));
        ti = timg;
    }
    talpha = timg + n_img;
    if (!is_device_ptr(target_alpha)) {
        CUDA_TRY(ctx, cudaMemcpyAsync(talpha, target_alpha, sizeof(double) * P, cudaMemcpyHostToDevice, ctx->stream));
        ta = talpha;
    }
    double* dloss = reinterpret_cast<double*>(t->flags.as<int>() + 2);
    // block partials (<= kLossBlocks) + the last-block ticket (zero between launches)
    if (int rc = ensure_zeroed(ctx, t->loss_part, sizeof(double) * kLossBlocks + 16)) return rc;
    // (*dloss is written by the loss kernel's last block: no clearing needed)
    const int threads = 256;
    const unsigned blocks = std::min<unsigned>(blocks_for(n_img + P, threads), kLossBlocks);
    {
        StageTimer st(ctx, ST_LOSS);
        scalar_loss_kernel<<<blocks, threads, 0, ctx->stream>>>(n_img, P, t->image.as<double>(), ti,
                                                                t->alpha.as<double>(), ta, w_image, w_alpha,
                                                                t->d_image.as<double>(), t->d_alpha.as<double>(),
                                                                dloss, t->loss_part.as<double>(),
                                                                t->loss_part.as<unsigned>() + 2 * kLossBlocks);
    }
    LAUNCH_CHECK(ctx);
    t->has_upstream = true;
    bool host = false;
    int rc;
    cudaStream_t hs;
    if ((rc = out_begin(ctx, &hs))) return rc;
    if ((rc = copy_out(ctx, d_image_out, t->d_image.p, sizeof(double) * n_img, &host, hs))) return rc;
    if ((rc = copy_out(ctx, d_alpha_out, t->d_alpha.p, sizeof(double) * P, &host, hs))) return rc;
    if ((rc = copy_out(ctx, loss_out, dloss, sizeof(double), &host, hs))) return rc;
    if ((rc = out_end(ctx, t, 1, hs))) return rc;
    *host_out = host;
    return GVR_OK;
}

extern "C" int gvr_scalar_loss(gvr_context* ctx, gvr_tape* t, const double* target_image, const double* target_alpha,
                               double w_image, double w_alpha, double* loss_out, double* d_image_out,
                               double* d_alpha_out) {
    bool host = false;
    if (int rc = scalar_loss_impl(ctx, t, target_image, target_alpha, w_image, w_alpha, loss_out, d_image_out,
                                  d_alpha_out, &host))
        return rc;
    return host && !ctx->async ? sync_and_check(ctx) : GVR_OK;
}

extern "C" {

int gvr_backward(gvr_context* ctx, gvr_tape* t, const double* d_image, const double* d_alpha,
                 const gvr_grad_flags* flags, const gvr_gradients* out) {
    return backward_impl(ctx, t, d_image, d_alpha, flags, out, false);
}

int gvr_backward_accumulate(gvr_context* ctx, gvr_tape* t, const double* d_image, const double* d_alpha,
                            const gvr_grad_flags* flags, const gvr_gradients* out) {
    return backward_impl(ctx, t, d_image, d_alpha, flags, out, true);
}

int gvr_backward_packed(gvr_context* ctx, gvr_tape* t, const double* d_image, const double* d_alpha,
                        const gvr_grad_flags* flags, double* packed, double* d_rt) {
    if (!ctx || !t) return GVR_ERR_RUNTIME;
    if (!packed || !d_rt || !is_device_ptr(packed) || !is_device_ptr(d_rt))
        return set_err(ctx, GVR_ERR_RUNTIME, "gvr_backward_packed needs device outputs");
    return backward_impl(ctx, t, d_image, d_alpha, flags, nullptr, false, packed, d_rt);
}

}  // extern "C"

static int backward_impl(gvr_context* ctx, gvr_tape* t, const double* d_image, const double* d_alpha,
                         const gvr_grad_flags* flags, const gvr_gradients* out, bool accumulate, double* packed,
                         double* packed_rt) {
    if (!ctx || !t || !t->valid) return set_err(ctx, GVR_ERR_RUNTIME, "tape is not valid");
    if (t->ctx != ctx) return set_err(ctx, GVR_ERR_RUNTIME, "objects belong to another context");
    if (!t->scene || t->scene->version != t->scene_version || !t->scene->valid)
        return set_err(ctx, GVR_ERR_RUNTIME, "the scene changed after the forward render");
    if (int rc = out_wait(ctx, t, 2)) return rc;  // the last backward's host copies read the gradients
    if (d_image || d_alpha)
        if (int rc = out_wait(ctx, t, 1)) return rc;  // the upstream is staged into d_image / d_alpha
    const gvr_scene* scene = t->scene;
    const int K = t->K, D = t->D;
    const long long P = (long long)t->H * t->W;
    const double* di;
    const double* da;
    if (!d_image && !d_alpha) {
        if (!t->has_upstream) return set_err(ctx, GVR_ERR_RUNTIME, "no upstream gradient stored in the tape");
        // gvr_scalar_loss stores H*W*max(D,1); backward reads H*W*D (identical layout when D >= 1)
        di = t->d_image.as<double>();
        da = t->d_alpha.as<double>();
    } else {
        if (!d_alpha || (D > 0 && !d_image))
            return set_err(ctx, GVR_ERR_VALIDATION, "backward: d_image shape does not match the forward render");
        CUDA_TRY(ctx, t->d_image.ensure(sizeof(double) * (size_t)(P * (D > 0 ? D : 1) + P) * 2));
        CUDA_TRY(ctx, t->d_alpha.ensure(sizeof(double) * (size_t)P));
        di = d_image;
        da = d_alpha;
        int rc;
        if (D > 0 && !is_device_ptr(d_image)) {
            if ((rc = copy_in(ctx, t->d_image.p, d_image, sizeof(double) * P * D))) return rc;
            di = t->d_image.as<double>();
        }
        if (!is_device_ptr(d_alpha)) {
            if ((rc = copy_in(ctx, t->d_alpha.p, d_alpha, sizeof(double) * P))) return rc;
            da = t->d_alpha.as<double>();
        }
    }
    const int through_t = flags ? flags->through_transmittance : 1;
    const int through_rho = flags ? flags->through_density : 1;

    const long long P_kp = P * t->cfg.k_prime;
    const unsigned finish_grid = (unsigned)std::max<long long>(1, (K + kFinishThreads - 1) / kFinishThreads);
    const unsigned rt_groups = (finish_grid + kRtGroup - 1) / kRtGroup;
    const long long scan_ctas = std::max<long long>(1, (K + kScanThreads - 1) / kScanThreads);
    const long long windows = (P_kp + 31) / 32;
    // fallback accumulators and tickets are zero between backwards (the gather
    // re-zeroes what it consumed): cleared only when (re)allocated
    if (int rc = ensure_zeroed(ctx, t->acc, sizeof(double) * 9 * (size_t)(K > 0 ? K : 1))) return rc;
    if (int rc = ensure_zeroed(ctx, t->attr_fb, sizeof(double) * (size_t)(D > 0 ? D : 1) * (K > 0 ? K : 1))) return rc;
    if (int rc = ensure_zeroed(ctx, t->tickets, sizeof(unsigned) * (2 + (size_t)rt_groups))) return rc;
    CUDA_TRY(ctx, t->rt_part.ensure(sizeof(double) * 12 * ((size_t)finish_grid + rt_groups)));
    CUDA_TRY(ctx, t->pieces.ensure(sizeof(double) * (10 + (size_t)D) * ((size_t)K + windows + 1)));

    CUDA_TRY(ctx, t->bent.ensure(sizeof(double4) * (size_t)(P_kp > 0 ? P_kp : 1)));
    CUDA_TRY(ctx, t->bkey.ensure(sizeof(int2) * (size_t)(P_kp > 0 ? P_kp : 1)));
    CUDA_TRY(ctx, t->rays.ensure(sizeof(double4) * (size_t)(P > 0 ? P : 1)));
    CUDA_TRY(ctx, t->app.ensure(sizeof(int2) * (size_t)(K > 0 ? K : 1)));
    CUDA_TRY(ctx, t->slot_off.ensure(sizeof(int) * (t->masks.cap / sizeof(unsigned long long) + 1)));
    CUDA_TRY(ctx, t->d_attr.ensure(sizeof(double) * (size_t)(D > 0 ? D : 1) * (K > 0 ? K : 1)));
    CUDA_TRY(ctx, t->d_center.ensure(sizeof(double) * 3 * (size_t)(K > 0 ? K : 1)));
    CUDA_TRY(ctx, t->d_inv_cov.ensure(sizeof(double) * 9 * (size_t)(K > 0 ? K : 1)));
    CUDA_TRY(ctx, t->d_rt.ensure(sizeof(double) * 12));
    if (K == 0) CUDA_TRY(ctx, cudaMemsetAsync(t->d_rt.p, 0, sizeof(double) * 12, ctx->stream));

    if (K > 0) {
        BwdParams bp{};
        bp.cam = t->camp;
        bp.kp = t->cfg.k_prime;
        bp.D = D;
        bp.Dc = D > 1 ? D : 1;
        bp.tau = scene->tau;
        bp.through_t = through_t;
        bp.through_rho = through_rho;
        const int btx = t->tiles_x, bty = t->tiles_y;
        int* sched = t->sched.as<int>();
        int* order_b = sched + 2;  // the selection's order
        bp.n_order = sched;
        bp.tiles_x = btx;
        bp.tile_order = order_b;
        bp.topk = t->topk.as<int>();
        bp.count = t->count.as<int>();
        bp.tape_t = t->tape_t.as<double>();
        bp.ent = t->ent.as<EntryRec>();
        bp.ent_a = t->ent_a.as<double>();
        bp.rec64 = t->rec64.as<Rec64>();
        bp.attr = scene->attr.as<double>();
        bp.d_image = di;
        bp.d_alpha = da;
        bp.kinfo = t->kinfo.as<int4>();
        bp.masks = t->masks.as<unsigned long long>();
        bp.slot_off = t->slot_off.as<int>();
        bp.bent = t->bent.as<double4>();
        bp.bkey = t->bkey.as<int2>();
        bp.rays = t->rays.as<double4>();
        bp.acc = t->acc.as<double>();
        bp.attr_fb = t->attr_fb.as<double>();
        const int kp = t->cfg.k_prime;
        unsigned* rec_total = t->tickets.as<unsigned>() + 1 + rt_groups;
        AppParams ap{};
        ap.K = K;
        ap.kinfo = t->kinfo.as<int4>();
        ap.masks = t->masks.as<unsigned long long>();
        ap.count = t->kcount.as<int>();
        ap.cta_sum = t->kcount.as<int>() + K;
        ap.slot_off = t->slot_off.as<int>();
        ap.app = t->app.as<int2>();
        ap.total = reinterpret_cast<int*>(rec_total);
        {
            // K4a-c: record layout (per-kernel counts from the blend's masks, scan, offsets)
            StageTimer st(ctx, ST_OBJECT);
            count_kernel<<<(unsigned)scan_ctas, kScanThreads, 0, ctx->stream>>>(ap);
            offsets_kernel<<<(unsigned)scan_ctas, kScanThreads, 0, ctx->stream>>>(ap);
        }
        ctx->launches += 1;
        LAUNCH_CHECK(ctx);
        int rc;
        if (kp <= 8) rc = launch_backward<8>(ctx, bp, btx * bty);
        else if (kp <= 16) rc = launch_backward<16>(ctx, bp, btx * bty);
        else if (kp <= 20) rc = launch_backward<20>(ctx, bp, btx * bty);
        else if (kp <= 24) rc = launch_backward<24>(ctx, bp, btx * bty);
        else if (kp <= 32) rc = launch_backward<32>(ctx, bp, btx * bty);
        else if (kp <= 48) rc = launch_backward<48>(ctx, bp, btx * bty);
        else if (kp <= 64) rc = launch_backward<64>(ctx, bp, btx * bty);
        else if (kp <= 96) rc = launch_backward<96>(ctx, bp, btx * bty);
        else rc = launch_backward<128>(ctx, bp, btx * bty);
        if (rc) return rc;

        GatherParams gp{};
        gp.K = K;
        gp.D = D;
        gp.nv = 10 + D;
        gp.cam = t->camp;
        gp.kinfo = t->kinfo.as<int4>();
        gp.app = t->app.as<int2>();
        gp.total = reinterpret_cast<const int*>(rec_total);
        gp.bent = t->bent.as<double4>();
        gp.bkey = t->bkey.as<int2>();
        gp.rays = t->rays.as<double4>();
        gp.rec64 = t->rec64.as<Rec64>();
        gp.d_image = di;
        gp.pieces = t->pieces.as<double>();
        gp.acc = t->acc.as<double>();
        gp.attr_fb = t->attr_fb.as<double>();
        gp.centers = scene->centers.as<double>();
        gp.inv_cov = scene->inv_cov.as<double>();
        gp.d_center = t->d_center.as<double>();
        gp.d_inv_cov = t->d_inv_cov.as<double>();
        gp.d_attr = t->d_attr.as<double>();
        gp.packed = packed;
        gp.rt_part = t->rt_part.as<double>();
        gp.tickets = t->tickets.as<unsigned>();
        gp.d_rt = packed_rt ? packed_rt : t->d_rt.as<double>();
        {
            StageTimer st(ctx, ST_OBJECT);
            const size_t rsmem = sizeof(double) * kRecThreads * (size_t)gp.nv;
            CUDA_TRY(ctx, cudaFuncSetAttribute(records_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem));
            records_kernel<<<148 * kRecCtasPerSm, kRecThreads, rsmem, ctx->stream>>>(gp);
            // programmatic dependent of the records: stages its object-space rows first
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)finish_grid);
            cfg.blockDim = dim3(kFinishThreads);
            cfg.stream = ctx->stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, finish_kernel, gp));
        }
        ++ctx->launches;
        LAUNCH_CHECK(ctx);
    }
    if (out && accumulate) {
        const double* srcs[5] = {t->d_center.as<double>(), t->d_inv_cov.as<double>(), t->d_attr.as<double>(),
                                 t->d_rt.as<double>(), t->d_rt.as<double>() + 9};
        double* dsts[5] = {out->d_center, out->d_inv_cov, out->d_attr, out->d_rotation, out->d_translation};
        const long long ns[5] = {3ll * K, 9ll * K, (long long)D * K, 9, 3};
        for (int b = 0; b < 5; ++b) {
            if (!dsts[b] || ns[b] == 0) continue;
            if (!is_device_ptr(dsts[b]))
                return set_err(ctx, GVR_ERR_RUNTIME, "gvr_backward_accumulate needs device output pointers");
            axpy_kernel<<<blocks_for(ns[b], 256), 256, 0, ctx->stream>>>(ns[b], srcs[b], dsts[b]);
            LAUNCH_CHECK(ctx);
        }
        return GVR_OK;
    }
    if (out) {
        bool host = false;
        int rc;
        cudaStream_t hs;
        if ((rc = out_begin(ctx, &hs))) return rc;
        if ((rc = copy_out(ctx, out->d_center, t->d_center.p, sizeof(double) * 3 * (size_t)K, &host, hs))) return rc;
        if ((rc = copy_out(ctx, out->d_inv_cov, t->d_inv_cov.p, sizeof(double) * 9 * (size_t)K, &host, hs)))
            return rc;
        if ((rc = copy_out(ctx, out->d_attr, t->d_attr.p, sizeof(double) * (size_t)D * K, &host, hs))) return rc;
        if ((rc = copy_out(ctx, out->d_rotation, t->d_rt.p, sizeof(double) * 9, &host, hs))) return rc;
        if ((rc = copy_out(ctx, out->d_translation, t->d_rt.as<double>() + 9, sizeof(double) * 3, &host, hs)))
            return rc;
        if ((rc = out_end(ctx, t, 2, hs))) return rc;
        if (host && !ctx->async) return sync_and_check(ctx);
    }
    return GVR_OK;
}

namespace {

TapeView tape_view(const gvr_tape* t) {
    TapeView v;
    v.cam = t->camp;
    v.kp = t->cfg.k_prime;
    v.topk = t->topk.as<int>();
    v.count = t->count.as<int>();
    v.tape_t = t->tape_t.as<double>();
    v.ent = t->ent.as<EntryRec>();
    v.rec64 = t->rec64.as<Rec64>();
    return v;
}

// Device view of an input that may live in host memory (staged through `buf`).
int stage_in(gvr_context* ctx, Buf& buf, const void* src, size_t bytes, const void** dev) {
    if (!src || is_device_ptr(src) || bytes == 0) {
        *dev = src;
        return GVR_OK;
    }
    CUDA_TRY(ctx, buf.ensure(bytes));
    CUDA_TRY(ctx, cudaMemcpyAsync(buf.p, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    *dev = buf.p;
    return GVR_OK;
}

// Device target for an output that may live in host memory; *host set when a
// copy back (copy_out of `buf`) is needed.
int stage_out(gvr_context* ctx, Buf& buf, void* dst, size_t bytes, void** dev, bool* host) {
    *host = dst && !is_device_ptr(dst);
    if (!*host) {
        *dev = dst;
        return GVR_OK;
    }
    CUDA_TRY(ctx, buf.ensure(bytes));
    *dev = buf.p;
    return GVR_OK;
}

int tape_ready(gvr_context* ctx, const gvr_tape* t) {
    if (!ctx || !t || !t->valid) return set_err(ctx, GVR_ERR_RUNTIME, "tape is not valid");
    if (t->ctx != ctx) return set_err(ctx, GVR_ERR_RUNTIME, "objects belong to another context");
    if (!t->scene || t->scene->version != t->scene_version || !t->scene->valid)
        return set_err(ctx, GVR_ERR_RUNTIME, "the scene changed after the forward render");
    return GVR_OK;
}

}  // namespace

extern "C" {

int gvr_tape_sample_attributes(gvr_context* ctx, const gvr_tape* t, const double* observed, int32_t channels,
                               int32_t normalized, double* attrs, double* support, uint8_t* masked) {
    if (int rc = tape_ready(ctx, t)) return rc;
    if (channels < 0) return set_err(ctx, GVR_ERR_VALIDATION, "channels must be >= 0");
    const long long P = (long long)t->H * t->W;
    const int K = t->K, C = channels;
    if (P * C > 0 && !observed) return set_err(ctx, GVR_ERR_RUNTIME, "observed image must not be null");
    const void* obs = nullptr;
    if (int rc = stage_in(ctx, ctx->scratch[0], observed, sizeof(double) * P * C, &obs)) return rc;
    void *da, *ds, *dm;
    bool ha, hs, hm;
    if (int rc = stage_out(ctx, ctx->scratch[1], attrs, sizeof(double) * (size_t)K * C + 8, &da, &ha)) return rc;
    if (int rc = stage_out(ctx, ctx->scratch[2], support, sizeof(double) * (size_t)K + 8, &ds, &hs)) return rc;
    if (int rc = stage_out(ctx, ctx->scratch[3], masked, (size_t)K + 8, &dm, &hm)) return rc;
    // support is needed even when the caller does not want it
    if (!ds) {
        CUDA_TRY(ctx, ctx->scratch[2].ensure(sizeof(double) * (size_t)K + 8));
        ds = ctx->scratch[2].p;
    }
    if (!da && C > 0) {
        CUDA_TRY(ctx, ctx->scratch[1].ensure(sizeof(double) * (size_t)K * C + 8));
        da = ctx->scratch[1].p;
    }
    if (!dm) {
        CUDA_TRY(ctx, ctx->scratch[3].ensure((size_t)K + 8));
        dm = ctx->scratch[3].p;
    }
    if (K > 0) {
        CUDA_TRY(ctx, cudaMemsetAsync(ds, 0, sizeof(double) * (size_t)K, ctx->stream));
        if (C > 0) CUDA_TRY(ctx, cudaMemsetAsync(da, 0, sizeof(double) * (size_t)K * C, ctx->stream));
        if (P > 0) {
            sample_scatter_kernel<<<blocks_for(P, 128), 128, 0, ctx->stream>>>(
                tape_view(t), static_cast<const double*>(obs), C, normalized ? 1 : 0, static_cast<double*>(ds),
                static_cast<double*>(da));
            LAUNCH_CHECK(ctx);
        }
        sample_finalize_kernel<<<blocks_for(K, 256), 256, 0, ctx->stream>>>(
            K, C, static_cast<const double*>(ds), static_cast<double*>(da), static_cast<unsigned char*>(dm));
        LAUNCH_CHECK(ctx);
    }
    bool host = false;
    int rc;
    if (ha && (rc = copy_out(ctx, attrs, da, sizeof(double) * (size_t)K * C, &host))) return rc;
    if (hs && (rc = copy_out(ctx, support, ds, sizeof(double) * (size_t)K, &host))) return rc;
    if (hm && (rc = copy_out(ctx, masked, dm, (size_t)K, &host))) return rc;
    if (host) return sync_and_check(ctx);
    return GVR_OK;
}

int gvr_sample_attributes(gvr_context* ctx, const gvr_scene* scene, const gvr_camera* camera,
                          const gvr_selection* cfg, const double* observed, int32_t obs_height, int32_t obs_width,
                          int32_t channels, int32_t normalized, double* attrs, double* support, uint8_t* masked) {
    if (!ctx || !scene || !camera) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (obs_height != camera->height || obs_width != camera->width)
        return set_err(ctx, GVR_ERR_VALIDATION, "observed image size does not match the camera");
    if (!ctx->aux_tape)
        if (int rc = gvr_tape_create(ctx, &ctx->aux_tape)) return rc;
    if (int rc = gvr_render(ctx, scene, camera, cfg, ctx->aux_tape, nullptr)) return rc;
    return gvr_tape_sample_attributes(ctx, ctx->aux_tape, observed, channels, normalized, attrs, support, masked);
}

int gvr_scene_resynthesize(gvr_context* ctx, gvr_scene* dst, const gvr_scene* src, int32_t n_attrs, int32_t channels,
                           const double* attrs, const uint8_t* masked) {
    if (!ctx || !dst || !src) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (!src->valid) return set_err(ctx, GVR_ERR_VALIDATION, "scene has not been validated");
    if (n_attrs != src->K) return set_err(ctx, GVR_ERR_VALIDATION, "sampled attribute count does not match the scene");
    if (channels < 0) return set_err(ctx, GVR_ERR_VALIDATION, "channels must be >= 0");
    const int K = src->K, C = channels;
    if ((size_t)K * C > 0 && !attrs) return set_err(ctx, GVR_ERR_RUNTIME, "attrs must not be null");
    const void* da = nullptr;
    const void* dm = nullptr;
    if (int rc = stage_in(ctx, ctx->scratch[0], attrs, sizeof(double) * (size_t)K * C, &da)) return rc;
    if (int rc = stage_in(ctx, ctx->scratch[1], masked, (size_t)K, &dm)) return rc;
    if (dst != src) {
        dst->valid = false;
        CUDA_TRY(ctx, dst->centers.ensure(sizeof(double) * 3 * (size_t)K));
        CUDA_TRY(ctx, dst->inv_cov.ensure(sizeof(double) * 9 * (size_t)K));
        if (K > 0) {
            CUDA_TRY(ctx, cudaMemcpyAsync(dst->centers.p, src->centers.p, sizeof(double) * 3 * (size_t)K,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
            CUDA_TRY(ctx, cudaMemcpyAsync(dst->inv_cov.p, src->inv_cov.p, sizeof(double) * 9 * (size_t)K,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
        }
    }
    dst->valid = false;
    ++dst->version;
    CUDA_TRY(ctx, dst->attr.ensure(sizeof(double) * (size_t)K * C));
    const long long n = (long long)K * C;
    if (n > 0) {
        resynth_attr_kernel<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(
            n, C, static_cast<const double*>(da), static_cast<const unsigned char*>(dm), dst->attr.as<double>());
        LAUNCH_CHECK(ctx);
    }
    dst->K = K;
    dst->D = C;
    dst->tau = src->tau;
    // render() re-validates the recolored scene (blender.cpp:70): same decisions
    if (int rc = validate_uploaded(ctx, dst)) return rc;
    dst->valid = true;
    return GVR_OK;
}

int gvr_tape_transmittance(gvr_context* ctx, const gvr_tape* t, const double* depth_t, double* out) {
    if (int rc = tape_ready(ctx, t)) return rc;
    const long long P = (long long)t->H * t->W;
    if (!depth_t || !out) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    const void* dt = nullptr;
    void* dout = nullptr;
    bool host = false;
    if (int rc = stage_in(ctx, ctx->scratch[0], depth_t, sizeof(double) * P, &dt)) return rc;
    if (int rc = stage_out(ctx, ctx->scratch[1], out, sizeof(double) * P, &dout, &host)) return rc;
    transmittance_kernel<<<blocks_for(P, 128), 128, 0, ctx->stream>>>(tape_view(t), t->scene->tau,
                                                                       static_cast<const double*>(dt),
                                                                       static_cast<double*>(dout));
    LAUNCH_CHECK(ctx);
    if (host) {
        bool h2 = false;
        if (int rc = copy_out(ctx, out, dout, sizeof(double) * P, &h2)) return rc;
        return sync_and_check(ctx);
    }
    return GVR_OK;
}

int gvr_tape_normalized_weights(gvr_context* ctx, const gvr_tape* t, double eps, double* out) {
    if (int rc = tape_ready(ctx, t)) return rc;
    if (!out) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    const long long P = (long long)t->H * t->W;
    const size_t bytes = sizeof(double) * (size_t)P * t->cfg.k_prime;
    void* dout = nullptr;
    bool host = false;
    if (int rc = stage_out(ctx, ctx->scratch[1], out, bytes, &dout, &host)) return rc;
    normalized_weights_kernel<<<blocks_for(P, 128), 128, 0, ctx->stream>>>(tape_view(t), eps,
                                                                            static_cast<double*>(dout));
    LAUNCH_CHECK(ctx);
    if (host) {
        bool h2 = false;
        if (int rc = copy_out(ctx, out, dout, bytes, &h2)) return rc;
        return sync_and_check(ctx);
    }
    return GVR_OK;
}

int gvr_shade_lambert(gvr_context* ctx, const gvr_camera* camera, const double* normals, const double* alpha,
                      const double* depth, const double* light_pos, const double* light_color, double* out) {
    if (!ctx || !camera || !normals || !alpha || !depth || !light_pos || !light_color || !out)
        return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (camera->height < 0 || camera->width < 0) return set_err(ctx, GVR_ERR_VALIDATION, "bad image size");
    const long long P = (long long)camera->height * camera->width;
    if (P == 0) return GVR_OK;
    CameraP cp;
    std::memcpy(cp.R, camera->rotation, sizeof cp.R);
    std::memcpy(cp.T, camera->translation, sizeof cp.T);
    cp.focal = camera->focal;
    cp.ox = camera->ox;
    cp.oy = camera->oy;
    cp.H = camera->height;
    cp.W = camera->width;
    const void *dn, *da, *dd;
    void* dout;
    bool host = false;
    if (int rc = stage_in(ctx, ctx->scratch[0], normals, sizeof(double) * 3 * P, &dn)) return rc;
    if (int rc = stage_in(ctx, ctx->scratch[1], alpha, sizeof(double) * P, &da)) return rc;
    if (int rc = stage_in(ctx, ctx->scratch[2], depth, sizeof(double) * P, &dd)) return rc;
    if (int rc = stage_out(ctx, ctx->scratch[3], out, sizeof(double) * 3 * P, &dout, &host)) return rc;
    double lp[3], lc[3];
    if (is_device_ptr(light_pos) || is_device_ptr(light_color))
        return set_err(ctx, GVR_ERR_RUNTIME, "light_pos / light_color must be host arrays");
    std::memcpy(lp, light_pos, sizeof lp);
    std::memcpy(lc, light_color, sizeof lc);
    shade_lambert_kernel<<<blocks_for(P, 128), 128, 0, ctx->stream>>>(
        cp, static_cast<const double*>(dn), static_cast<const double*>(da), static_cast<const double*>(dd), lp[0],
        lp[1], lp[2], lc[0], lc[1], lc[2], static_cast<double*>(dout));
    LAUNCH_CHECK(ctx);
    if (host) {
        bool h2 = false;
        if (int rc = copy_out(ctx, out, dout, sizeof(double) * 3 * P, &h2)) return rc;
        return sync_and_check(ctx);
    }
    return GVR_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- multi-view (C3 / C5 batches)
//
// The views of one call are independent renders of the same scene (SURVEY.md
// §8b "batched variants over V cameras"). A single C2 view fills only part of
// the B200 (its per-tile kernels are latency bound at ~1000 tiles), so the
// views are spread round-robin over worker streams forked from the context
// stream and joined back into it: kernels of different views overlap, and the
// whole fork/join pattern is capturable in one CUDA graph.

namespace {

#ifndef GVR_VIEW_STREAMS
#define GVR_VIEW_STREAMS 16
#endif
constexpr int kViewStreams = GVR_VIEW_STREAMS;
constexpr int kSumViews = 64;  // views per gradient-sum launch (kernel parameter space)

struct ViewSumParams {
    int V;
    long long n[5];
    const double* src[kSumViews][5];
    double* dst[5];
};

// sum[b][i] += sum_v src[v][b][i], views in ascending order (deterministic).
__global__ void view_sum_kernel(ViewSumParams p) {
    for (int b = 0; b < 5; ++b) {
        if (!p.dst[b]) continue;
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.n[b];
             i += (long long)gridDim.x * blockDim.x) {
            double acc = p.dst[b][i];
            int v = 0;
            for (; v + 8 <= p.V; v += 8) {  // 8 loads in flight, added in view order
                double a[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) a[u] = p.src[v + u][b][i];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc += a[u];
            }
            for (; v < p.V; ++v) acc += p.src[v][b][i];
            p.dst[b][i] = acc;
        }
    }
}

int ensure_workers(gvr_context* ctx, int n) {
    if (!ctx->fork_ev) CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
    while ((int)ctx->workers.size() < n) {
        cudaStream_t s;
        cudaEvent_t e;
        CUDA_TRY(ctx, cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->workers.push_back(s);
        ctx->join_ev.push_back(e);
    }
    return GVR_OK;
}

int fork_workers(gvr_context* ctx, int n) {
    if (int rc = ensure_workers(ctx, n)) return rc;
    CUDA_TRY(ctx, cudaEventRecord(ctx->fork_ev, ctx->stream));
    for (int w = 0; w < n; ++w) CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->workers[w], ctx->fork_ev, 0));
    return GVR_OK;
}

int join_workers(gvr_context* ctx, cudaStream_t home, int n) {
    ctx->stream = home;
    for (int w = 0; w < n; ++w) {
        CUDA_TRY(ctx, cudaEventRecord(ctx->join_ev[w], ctx->workers[w]));
        CUDA_TRY(ctx, cudaStreamWaitEvent(home, ctx->join_ev[w], 0));
    }
    return GVR_OK;
}

// Runs fn(v) for every view on worker stream v % n, then joins; the first
// error is returned after the join (so a capture is never left forked).
template <typename F>
int for_views(gvr_context* ctx, int V, F&& fn) {
    if (V <= 0) return GVR_OK;
    const int n = V < kViewStreams ? V : kViewStreams;
    cudaStream_t home = ctx->stream;
    if (int rc = fork_workers(ctx, n)) return rc;
    int first = GVR_OK;
    std::string err;
    for (int v = 0; v < V && first == GVR_OK; ++v) {
        ctx->stream = ctx->workers[v % n];
        const int rc = fn(v);
        if (rc != GVR_OK) {
            first = rc;
            err = ctx->err;
        }
    }
    const int jr = join_workers(ctx, home, n);
    if (first != GVR_OK) {
        ctx->err = err;
        return first;
    }
    return jr;
}

}  // namespace

extern "C" {

int gvr_render_views(gvr_context* ctx, const gvr_scene* scene, int32_t n_views, const gvr_camera* cameras,
                     const gvr_selection* cfg, gvr_tape* const* tapes, const gvr_render_outputs* outs) {
    if (!ctx || !scene || !tapes || (n_views > 0 && !cameras)) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (n_views < 0) return set_err(ctx, GVR_ERR_RUNTIME, "n_views must be >= 0");
    for (int v = 0; v < n_views; ++v) {  // host-side checks first: nothing is enqueued for an invalid batch
        if (!tapes[v]) return set_err(ctx, GVR_ERR_RUNTIME, "tape %d is null", v);
        for (int u = 0; u < v; ++u)
            if (tapes[u] == tapes[v]) return set_err(ctx, GVR_ERR_RUNTIME, "views %d and %d share a tape", u, v);
        if (int rc = validate_camera(ctx, cameras + v)) return rc;
    }
    if (int rc = validate_cfg(ctx, cfg)) return rc;
    bool any_host = false;
    const int rc = for_views(ctx, n_views, [&](int v) {
        bool host = false;
        const int r = render_impl(ctx, scene, cameras + v, cfg, tapes[v], outs ? outs + v : nullptr, 0, 1, &host);
        any_host = any_host || host;
        return r;
    });
    if (rc) return rc;
    if (!any_host) return GVR_OK;
    if (int r = sync_and_check(ctx)) return r;
    for (int v = 0; v < n_views; ++v)
        if (int r = check_finite(ctx, tapes[v])) return r;
    return GVR_OK;
}

int gvr_scalar_loss_views(gvr_context* ctx, int32_t n_views, gvr_tape* const* tapes, const double* const* target_images,
                          const double* const* target_alphas, double w_image, double w_alpha, double* losses) {
    if (!ctx || !tapes || (n_views > 0 && (!target_images || !target_alphas)))
        return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    bool any_host = false;
    const int rc = for_views(ctx, n_views, [&](int v) {
        bool host = false;
        const int r = scalar_loss_impl(ctx, tapes[v], target_images[v], target_alphas[v], w_image, w_alpha,
                                       losses ? losses + v : nullptr, nullptr, nullptr, &host);
        any_host = any_host || host;
        return r;
    });
    if (rc) return rc;
    return any_host ? sync_and_check(ctx) : GVR_OK;
}

int gvr_backward_views(gvr_context* ctx, int32_t n_views, gvr_tape* const* tapes, const gvr_grad_flags* flags,
                       const gvr_gradients* outs, const gvr_gradients* sum) {
    if (!ctx || !tapes) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    auto dev_ok = [](const gvr_gradients* g) {
        const void* ps[5] = {g->d_center, g->d_inv_cov, g->d_attr, g->d_rotation, g->d_translation};
        for (const void* q : ps)
            if (q && !is_device_ptr(q)) return false;
        return true;
    };
    for (int v = 0; v < n_views; ++v) {
        if (!tapes[v] || !tapes[v]->valid) return set_err(ctx, GVR_ERR_RUNTIME, "tape %d is not valid", v);
        if (tapes[v]->ctx != ctx) return set_err(ctx, GVR_ERR_RUNTIME, "objects belong to another context");
        if (!tapes[v]->has_upstream)
            return set_err(ctx, GVR_ERR_RUNTIME, "tape %d has no upstream gradient (gvr_scalar_loss_views first)", v);
        if (outs && !dev_ok(outs + v)) return set_err(ctx, GVR_ERR_RUNTIME, "gvr_backward_views needs device outputs");
    }
    if (sum && !dev_ok(sum)) return set_err(ctx, GVR_ERR_RUNTIME, "gvr_backward_views needs device outputs");
    if (sum)
        for (int v = 1; v < n_views; ++v)
            if (tapes[v]->K != tapes[0]->K || tapes[v]->D != tapes[0]->D)
                return set_err(ctx, GVR_ERR_RUNTIME, "summed views must share the scene size");
    int rc = for_views(ctx, n_views, [&](int v) {
        return backward_impl(ctx, tapes[v], nullptr, nullptr, flags, outs ? outs + v : nullptr, false);
    });
    if (rc || !sum || n_views == 0) return rc;
    const int K = tapes[0]->K, D = tapes[0]->D;
    for (int v0 = 0; v0 < n_views; v0 += kSumViews) {
        ViewSumParams sp{};
        sp.V = std::min(kSumViews, n_views - v0);
        sp.n[0] = 3ll * K;
        sp.n[1] = 9ll * K;
        sp.n[2] = (long long)D * K;
        sp.n[3] = 9;
        sp.n[4] = 3;
        sp.dst[0] = sum->d_center;
        sp.dst[1] = sum->d_inv_cov;
        sp.dst[2] = D > 0 ? sum->d_attr : nullptr;
        sp.dst[3] = sum->d_rotation;
        sp.dst[4] = sum->d_translation;
        for (int v = 0; v < sp.V; ++v) {
            const gvr_tape* t = tapes[v0 + v];
            sp.src[v][0] = t->d_center.as<double>();
            sp.src[v][1] = t->d_inv_cov.as<double>();
            sp.src[v][2] = t->d_attr.as<double>();
            sp.src[v][3] = t->d_rt.as<double>();
            sp.src[v][4] = t->d_rt.as<double>() + 9;
        }
        view_sum_kernel<<<148 * 4, 256, 0, ctx->stream>>>(sp);
        LAUNCH_CHECK(ctx);
    }
    return GVR_OK;
}

}  // extern "C"


// ---------------------------------------------------------------- fitting regularizers (fit.cpp:44-115)

struct gvr_regularizer {
    gvr_context* ctx = nullptr;
    int N = 0, E = 0;
    Buf edges, rest_len, adj_start, adj, rest_lap, value;
};

namespace {

RegView reg_view(const gvr_regularizer* r) {
    RegView v;
    v.N = r->N;
    v.E = r->E;
    v.edges = r->edges.as<int>();
    v.rest_len = r->rest_len.as<double>();
    v.adj_start = r->adj_start.as<int>();
    v.adj = r->adj.as<int>();
    v.rest_lap = r->rest_lap.as<double>();
    return v;
}

int reg_term(gvr_context* ctx, const gvr_regularizer* r, const double* centers, double weight, double* value,
             double* grad, int32_t accumulate, bool laplacian) {
    if (!ctx || !r || !centers) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (r->ctx != ctx) return set_err(ctx, GVR_ERR_RUNTIME, "objects belong to another context");
    const void* dc = nullptr;
    if (int rc = stage_in(ctx, ctx->scratch[0], centers, sizeof(double) * 3 * (size_t)r->N, &dc)) return rc;
    void* dg = nullptr;
    bool host_g = false;
    if (grad) {
        if (int rc = stage_out(ctx, ctx->scratch[1], grad, sizeof(double) * 3 * (size_t)r->N, &dg, &host_g)) return rc;
        if (!accumulate || host_g) {
            if (host_g && accumulate)
                CUDA_TRY(ctx, cudaMemcpyAsync(dg, grad, sizeof(double) * 3 * (size_t)r->N, cudaMemcpyHostToDevice,
                                              ctx->stream));
            else
                CUDA_TRY(ctx, cudaMemsetAsync(dg, 0, sizeof(double) * 3 * (size_t)r->N, ctx->stream));
        }
    }
    double* dv = r->value.as<double>();
    CUDA_TRY(ctx, cudaMemsetAsync(dv, 0, sizeof(double), ctx->stream));
    const RegView v = reg_view(r);
    if (laplacian)
        laplacian_reg_kernel<<<blocks_for(r->N, 256), 256, 0, ctx->stream>>>(v, static_cast<const double*>(dc), weight,
                                                                              dv, static_cast<double*>(dg));
    else
        edge_reg_kernel<<<blocks_for(r->E, 256), 256, 0, ctx->stream>>>(v, static_cast<const double*>(dc), weight, dv,
                                                                         static_cast<double*>(dg));
    LAUNCH_CHECK(ctx);
    bool host = false;
    if (value)
        if (int rc = copy_out(ctx, value, dv, sizeof(double), &host)) return rc;
    if (host_g)
        if (int rc = copy_out(ctx, grad, dg, sizeof(double) * 3 * (size_t)r->N, &host)) return rc;
    return host ? sync_and_check(ctx) : GVR_OK;
}

}  // namespace

extern "C" {

int gvr_regularizer_create(gvr_context* ctx, int32_t n_vertices, int32_t n_edges, const int32_t* edges,
                           const double* rest_centers, gvr_regularizer** out) {
    if (!ctx || !out) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    *out = nullptr;
    if (n_edges <= 0 || !edges) return set_err(ctx, GVR_ERR_VALIDATION, "regularizer needs a non-empty neighbor graph");
    if (n_vertices < 0 || (n_vertices > 0 && !rest_centers)) return set_err(ctx, GVR_ERR_RUNTIME, "bad vertex array");
    if (is_device_ptr(edges)) return set_err(ctx, GVR_ERR_RUNTIME, "edges must be a host array");
    // CSR adjacency, each vertex's neighbours in the order the edges list them
    // (adjacency[a].push_back(b); adjacency[b].push_back(a), fit.cpp:53-55)
    std::vector<int> start(n_vertices + 1, 0), fill, adj(2 * (size_t)n_edges);
    for (int e = 0; e < n_edges; ++e) {
        const int a = edges[2 * e], b = edges[2 * e + 1];
        if (a < 0 || b < 0 || a >= n_vertices || b >= n_vertices)
            return set_err(ctx, GVR_ERR_VALIDATION, "regularizer edge index out of range");
        ++start[a + 1];
        ++start[b + 1];
    }
    for (int i = 0; i < n_vertices; ++i) start[i + 1] += start[i];
    fill.assign(start.begin(), start.end() - 1);
    for (int e = 0; e < n_edges; ++e) {
        const int a = edges[2 * e], b = edges[2 * e + 1];
        adj[fill[a]++] = b;
        adj[fill[b]++] = a;
    }
    auto* r = new gvr_regularizer();
    r->ctx = ctx;
    r->N = n_vertices;
    r->E = n_edges;
    auto fail = [&](int rc) {
        delete r;
        return rc;
    };
    const size_t vb = sizeof(double) * 3 * (size_t)std::max(n_vertices, 1);
    if (r->edges.ensure(sizeof(int) * 2 * (size_t)n_edges) != cudaSuccess ||
        r->rest_len.ensure(sizeof(double) * (size_t)n_edges) != cudaSuccess ||
        r->adj_start.ensure(sizeof(int) * (size_t)(n_vertices + 1)) != cudaSuccess ||
        r->adj.ensure(sizeof(int) * adj.size()) != cudaSuccess || r->rest_lap.ensure(vb) != cudaSuccess ||
        r->value.ensure(sizeof(double)) != cudaSuccess)
        return fail(set_err(ctx, GVR_ERR_RUNTIME, "regularizer allocation failed"));
    cudaError_t e1 = cudaMemcpyAsync(r->edges.p, edges, sizeof(int) * 2 * (size_t)n_edges, cudaMemcpyHostToDevice,
                                     ctx->stream);
    cudaError_t e2 = cudaMemcpyAsync(r->adj_start.p, start.data(), sizeof(int) * start.size(), cudaMemcpyHostToDevice,
                                     ctx->stream);
    cudaError_t e3 = cudaMemcpyAsync(r->adj.p, adj.data(), sizeof(int) * adj.size(), cudaMemcpyHostToDevice, ctx->stream);
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
        return fail(set_err(ctx, GVR_ERR_RUNTIME, "regularizer upload failed"));
    const void* dc = nullptr;
    if (int rc = stage_in(ctx, ctx->scratch[0], rest_centers, sizeof(double) * 3 * (size_t)n_vertices, &dc))
        return fail(rc);
    const RegView v = reg_view(r);
    rest_edge_kernel<<<blocks_for(n_edges, 256), 256, 0, ctx->stream>>>(v, static_cast<const double*>(dc),
                                                                         r->rest_len.as<double>());
    if (n_vertices > 0)
        rest_laplacian_kernel<<<blocks_for(n_vertices, 256), 256, 0, ctx->stream>>>(v, static_cast<const double*>(dc),
                                                                                     r->rest_lap.as<double>());
    ctx->launches += 2;
    if (int rc = sync_and_check(ctx)) return fail(rc);  // host vectors above are released on return
    *out = r;
    return GVR_OK;
}

void gvr_regularizer_destroy(gvr_regularizer* r) {
    if (!r) return;
    cudaStreamSynchronize(r->ctx->stream);
    Buf* bufs[] = {&r->edges, &r->rest_len, &r->adj_start, &r->adj, &r->rest_lap, &r->value};
    for (Buf* b : bufs) b->release();
    delete r;
}

int gvr_edge_reg(gvr_context* ctx, const gvr_regularizer* reg, const double* centers, double weight, double* value,
                 double* grad, int32_t accumulate) {
    return reg_term(ctx, reg, centers, weight, value, grad, accumulate, false);
}

int gvr_laplacian_reg(gvr_context* ctx, const gvr_regularizer* reg, const double* centers, double weight, double* value,
                      double* grad, int32_t accumulate) {
    return reg_term(ctx, reg, centers, weight, value, grad, accumulate, true);
}

}  // extern "C"


// ---------------------------------------------------------------- tape extras

extern "C" {

int gvr_tape_cam_scene(gvr_context* ctx, const gvr_tape* t, double* centers, double* inv_cov) {
    if (int rc = tape_ready(ctx, t)) return rc;
    const int K = t->K;
    if (K == 0) return GVR_OK;
    void *dc = nullptr, *ds = nullptr;
    bool hc = false, hs = false;
    if (int rc = stage_out(ctx, ctx->scratch[0], centers, sizeof(double) * 3 * (size_t)K, &dc, &hc)) return rc;
    if (int rc = stage_out(ctx, ctx->scratch[1], inv_cov, sizeof(double) * 9 * (size_t)K, &ds, &hs)) return rc;
    cam_scene_kernel<<<blocks_for(K, 256), 256, 0, ctx->stream>>>(K, t->rec64.as<Rec64>(), static_cast<double*>(dc),
                                                                  static_cast<double*>(ds));
    LAUNCH_CHECK(ctx);
    bool host = false;
    if (hc)
        if (int rc = copy_out(ctx, centers, dc, sizeof(double) * 3 * (size_t)K, &host)) return rc;
    if (hs)
        if (int rc = copy_out(ctx, inv_cov, ds, sizeof(double) * 9 * (size_t)K, &host)) return rc;
    return host ? sync_and_check(ctx) : GVR_OK;
}

int gvr_tape_tile_cycles(gvr_context* ctx, const gvr_tape* t, int64_t* cycles, int64_t n) {
    if (int rc = tape_ready(ctx, t)) return rc;
    const int64_t tiles = (int64_t)t->tiles_x * t->tiles_y;
    if (!cycles || n != tiles || !t->profiled || t->tile_cycles.cap < sizeof(long long) * (size_t)tiles)
        return set_err(ctx, GVR_ERR_RUNTIME, "tile_cycles: render with the tile profile on, n = tiles_x * tiles_y");
    CUDA_TRY(ctx, cudaMemcpyAsync(cycles, t->tile_cycles.p, sizeof(long long) * (size_t)tiles, cudaMemcpyDefault,
                                  ctx->stream));
    return sync_and_check(ctx);
}

int gvr_tape_check_finite(gvr_context* ctx, gvr_tape* t) {
    if (!ctx || !t || !t->valid) return set_err(ctx, GVR_ERR_RUNTIME, "tape is not valid");
    if (t->ctx != ctx) return set_err(ctx, GVR_ERR_RUNTIME, "objects belong to another context");
    CUDA_TRY(ctx, cudaMemcpyAsync(t->h_flags + 1, t->flags.as<int>() + 1, sizeof(int), cudaMemcpyDeviceToHost,
                                  ctx->stream));
    if (int rc = sync_and_check(ctx)) return rc;
    return check_finite(ctx, t);
}

int gvr_tape_list_stats(gvr_context* ctx, const gvr_tape* t, int64_t* stats) {
    if (!ctx || !t || !t->valid || !stats) return set_err(ctx, GVR_ERR_RUNTIME, "tape is not valid");
    if (t->ctx != ctx) return set_err(ctx, GVR_ERR_RUNTIME, "objects belong to another context");
    CUDA_TRY(ctx, cudaMemcpyAsync(t->h_flags + kListStats, t->flags.as<int>() + kListStats, 5 * sizeof(int),
                                  cudaMemcpyDeviceToHost, ctx->stream));
    if (int rc = sync_and_check(ctx)) return rc;
    for (int i = 0; i < 4; ++i) stats[i] = t->h_flags[kListStats + i];
    stats[4] = std::min<long long>((long long)(t->pool.cap / sizeof(unsigned long long)),
                                   ctx->pool_override > 0 ? ctx->pool_override : 0x7fffffffLL);
    stats[5] = t->h_flags[kMaskTotal];
    stats[6] = (long long)(t->masks.cap / sizeof(unsigned long long));
    return GVR_OK;
}

int gvr_tape_dropped_behind_camera(gvr_context* ctx, const gvr_tape* t, int32_t* count) {
    if (!ctx || !t || !t->valid || !count) return set_err(ctx, GVR_ERR_RUNTIME, "tape is not valid");
    CUDA_TRY(ctx, cudaMemcpyAsync(t->h_flags, t->flags.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    if (int rc = sync_and_check(ctx)) return rc;
    *count = t->h_flags[0];
    return GVR_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- building blocks (C++ drop-in)

namespace {

CameraP camera_params(const gvr_camera* camera) {
    CameraP cp;
    std::memcpy(cp.R, camera->rotation, sizeof cp.R);
    std::memcpy(cp.T, camera->translation, sizeof cp.T);
    cp.focal = camera->focal;
    cp.ox = camera->ox;
    cp.oy = camera->oy;
    cp.H = camera->height;
    cp.W = camera->width;
    return cp;
}

// device copies of up to four host-or-device inputs (freed with the guard)
struct Tmp {
    Buf b[8];
    ~Tmp() {
        for (Buf& x : b) x.release();
    }
};

int in_dev(gvr_context* ctx, Buf& buf, const void* src, size_t bytes, const void** dev) {
    return stage_in(ctx, buf, src, bytes, dev);
}

}  // namespace

extern "C" {

int gvr_trace_pairs(gvr_context* ctx, int64_t n, const double* dirs, const double* centers, const double* inv_cov,
                    double* l, double* q, double* sigma) {
    if (!ctx || n < 0 || (n > 0 && (!dirs || !centers || !inv_cov)))
        return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (n == 0) return GVR_OK;
    if (ctx->capturing) return set_err(ctx, GVR_ERR_RUNTIME, "gvr_trace_pairs synchronises; not capturable");
    Tmp t;
    const void *dd, *dc, *ds;
    if (int rc = in_dev(ctx, t.b[0], dirs, sizeof(double) * 3 * (size_t)n, &dd)) return rc;
    if (int rc = in_dev(ctx, t.b[1], centers, sizeof(double) * 3 * (size_t)n, &dc)) return rc;
    if (int rc = in_dev(ctx, t.b[2], inv_cov, sizeof(double) * 9 * (size_t)n, &ds)) return rc;
    CUDA_TRY(ctx, t.b[3].ensure(sizeof(double) * 3 * (size_t)n + sizeof(unsigned long long)));
    double* out = t.b[3].as<double>();
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(out + 3 * n);
    CUDA_TRY(ctx, cudaMemsetAsync(bad, 0xff, sizeof *bad, ctx->stream));
    trace_pairs_kernel<<<blocks_for(n, 128), 128, 0, ctx->stream>>>(
        n, static_cast<const double*>(dd), static_cast<const double*>(dc), static_cast<const double*>(ds), out,
        out + n, out + 2 * n, bad);
    LAUNCH_CHECK(ctx);
    bool host = false;
    int rc;
    if ((rc = copy_out(ctx, l, out, sizeof(double) * n, &host))) return rc;
    if ((rc = copy_out(ctx, q, out + n, sizeof(double) * n, &host))) return rc;
    if ((rc = copy_out(ctx, sigma, out + 2 * n, sizeof(double) * n, &host))) return rc;
    unsigned long long hbad = 0;
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_flags + 2, bad, sizeof hbad, cudaMemcpyDeviceToHost, ctx->stream));
    if ((rc = sync_and_check(ctx))) return rc;
    std::memcpy(&hbad, ctx->h_flags + 2, sizeof hbad);
    if (hbad != ~0ull)
        return set_err(ctx, GVR_ERR_VALIDATION, "trace_kernel: D^T inv_cov D <= 0 (inv_cov not positive-definite)");
    return GVR_OK;
}

int gvr_view_transform(gvr_context* ctx, int32_t K, const double* centers, const double* inv_cov,
                       const gvr_camera* camera, double* out_centers, double* out_inv_cov) {
    if (!ctx || K < 0 || (K > 0 && (!centers || !inv_cov))) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (int rc = validate_camera(ctx, camera)) return rc;  // view_transform validates the camera (scene.cpp:6)
    if (K == 0) return GVR_OK;
    Tmp t;
    const void *dc, *ds;
    if (int rc = in_dev(ctx, t.b[0], centers, sizeof(double) * 3 * (size_t)K, &dc)) return rc;
    if (int rc = in_dev(ctx, t.b[1], inv_cov, sizeof(double) * 9 * (size_t)K, &ds)) return rc;
    CUDA_TRY(ctx, t.b[2].ensure(sizeof(double) * 12 * (size_t)K));
    double* out = t.b[2].as<double>();
    view_transform_kernel<<<blocks_for(K, 128), 128, 0, ctx->stream>>>(K, camera_params(camera),
                                                                        static_cast<const double*>(dc),
                                                                        static_cast<const double*>(ds), out,
                                                                        out + 3 * (size_t)K);
    LAUNCH_CHECK(ctx);
    bool host = false;
    int rc;
    if ((rc = copy_out(ctx, out_centers, out, sizeof(double) * 3 * (size_t)K, &host))) return rc;
    if ((rc = copy_out(ctx, out_inv_cov, out + 3 * (size_t)K, sizeof(double) * 9 * (size_t)K, &host))) return rc;
    return sync_and_check(ctx);
}

int gvr_pixel_rays(gvr_context* ctx, const gvr_camera* camera, int64_t n, const int32_t* rows, const int32_t* cols,
                   double* dirs) {
    if (!ctx || !camera || !dirs || n < 0 || (!rows) != (!cols)) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (!rows && n != (int64_t)camera->height * camera->width)
        return set_err(ctx, GVR_ERR_RUNTIME, "gvr_pixel_rays: n must be height * width without rows / cols");
    if (n == 0) return GVR_OK;
    Tmp t;
    const void *dr = nullptr, *dcl = nullptr;
    if (rows) {
        if (int rc = in_dev(ctx, t.b[0], rows, sizeof(int32_t) * (size_t)n, &dr)) return rc;
        if (int rc = in_dev(ctx, t.b[1], cols, sizeof(int32_t) * (size_t)n, &dcl)) return rc;
    }
    CUDA_TRY(ctx, t.b[2].ensure(sizeof(double) * 3 * (size_t)n));
    pixel_rays_kernel<<<blocks_for(n, 128), 128, 0, ctx->stream>>>(camera_params(camera), n,
                                                                    static_cast<const int*>(dr),
                                                                    static_cast<const int*>(dcl), t.b[2].as<double>());
    LAUNCH_CHECK(ctx);
    bool host = false;
    if (int rc = copy_out(ctx, dirs, t.b[2].p, sizeof(double) * 3 * (size_t)n, &host)) return rc;
    return sync_and_check(ctx);
}

int gvr_coarse_select_boxes(gvr_context* ctx, int32_t K, const double* cam_centers, const double* cam_inv_cov,
                            const gvr_camera* camera, const gvr_selection* cfg, int32_t* boxes, int32_t* dropped) {
    if (!ctx || !camera || K < 0 || (K > 0 && (!cam_centers || !cam_inv_cov || !boxes)))
        return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (int rc = validate_cfg_ref(ctx, cfg)) return rc;  // coarse_select validates the config (tracer.cpp:39)
    if (dropped) *dropped = 0;
    if (K == 0) return GVR_OK;
    Tmp t;
    const void *dc, *ds;
    if (int rc = in_dev(ctx, t.b[0], cam_centers, sizeof(double) * 3 * (size_t)K, &dc)) return rc;
    if (int rc = in_dev(ctx, t.b[1], cam_inv_cov, sizeof(double) * 9 * (size_t)K, &ds)) return rc;
    CUDA_TRY(ctx, t.b[2].ensure(sizeof(Rec32) * (size_t)K));
    CUDA_TRY(ctx, t.b[3].ensure(sizeof(Rec64) * (size_t)K));
    CUDA_TRY(ctx, t.b[4].ensure(sizeof(int4) * (size_t)K + sizeof(int)));
    int* ddrop = reinterpret_cast<int*>(t.b[4].as<int4>() + K);
    CUDA_TRY(ctx, cudaMemsetAsync(ddrop, 0, sizeof(int), ctx->stream));
    gvr_camera ident = *camera;  // the scene is already in camera space: identity extrinsics, exact
    for (int i = 0; i < 9; ++i) ident.rotation[i] = (i % 4 == 0) ? 1.0 : 0.0;
    for (int i = 0; i < 3; ++i) ident.translation[i] = 0.0;
    ProjectParams pp{};
    pp.K = K;
    pp.centers = static_cast<const double*>(dc);
    pp.inv_cov = static_cast<const double*>(ds);
    pp.cam = camera_params(&ident);
    pp.sel.eta = cfg->eta;
    pp.sel.log_eta = std::log(cfg->eta);
    pp.sel.chi = 2.0 * std::log(1.0 / cfg->eta);
    pp.sel.kp = cfg->k_prime;
    pp.sel.coarse = 1;
    pp.sel.ds = cfg->coarse_downsample;
    pp.tile = kFwdTile;
    pp.rec32 = t.b[2].as<Rec32>();
    pp.rec64 = t.b[3].as<Rec64>();
    pp.dropped_behind = ddrop;
    pp.ref_box = t.b[4].as<int4>();
    coarse_box_kernel<<<blocks_for(K, 128), 128, 0, ctx->stream>>>(pp);
    LAUNCH_CHECK(ctx);
    bool host = false;
    if (int rc = copy_out(ctx, boxes, t.b[4].p, sizeof(int4) * (size_t)K, &host)) return rc;
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_flags, ddrop, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    if (int rc = sync_and_check(ctx)) return rc;
    if (dropped) *dropped = ctx->h_flags[0];
    return GVR_OK;
}

int gvr_ray_sort(gvr_context* ctx, int32_t n, const int32_t* idx, const double* l, const double* q, double eta,
                 int32_t* order, int32_t* m_out) {
    if (!ctx || n < 0 || !order || !m_out || (n > 0 && (!idx || !l))) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    const bool filter = eta > 0.0 && eta < 1.0;
    if (filter && n > 0 && !q) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (n > kRaySortMax)
        return set_err(ctx, GVR_ERR_RUNTIME, "gvr_ray_sort: at most %d entries per call", kRaySortMax);
    *m_out = 0;
    if (n == 0) return GVR_OK;
    Tmp t;
    const void *di, *dl, *dq = nullptr;
    if (int rc = in_dev(ctx, t.b[0], idx, sizeof(int32_t) * (size_t)n, &di)) return rc;
    if (int rc = in_dev(ctx, t.b[1], l, sizeof(double) * (size_t)n, &dl)) return rc;
    if (filter)
        if (int rc = in_dev(ctx, t.b[2], q, sizeof(double) * (size_t)n, &dq)) return rc;
    CUDA_TRY(ctx, t.b[3].ensure(sizeof(int32_t) * ((size_t)n + 1)));
    int* dorder = t.b[3].as<int>();
    ray_sort_kernel<<<1, 1024, 0, ctx->stream>>>(n, static_cast<const int*>(di), static_cast<const double*>(dl),
                                                 static_cast<const double*>(dq), filter ? std::log(eta) : 0.0,
                                                 filter ? 1 : 0, dorder, dorder + n);
    LAUNCH_CHECK(ctx);
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_flags, dorder + n, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    if (int rc = sync_and_check(ctx)) return rc;
    const int m = ctx->h_flags[0];
    *m_out = m;
    bool host = false;
    if (int rc = copy_out(ctx, order, dorder, sizeof(int32_t) * (size_t)m, &host)) return rc;
    return sync_and_check(ctx);
}

int gvr_blend_ray(gvr_context* ctx, int32_t n, const int32_t* idx, const double* l, const double* q,
                  const double* sigma, double tau, int32_t* out_idx, double* out_w, double* alpha) {
    if (!ctx || n < 0 || (n > 0 && (!idx || !l || !q || !sigma || !out_idx || !out_w)) || !alpha)
        return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (n > kRaySortMax)
        return set_err(ctx, GVR_ERR_RUNTIME, "gvr_blend_ray: at most %d entries per call", kRaySortMax);
    Tmp t;
    const void *di, *dl, *dq, *dsg;
    if (int rc = in_dev(ctx, t.b[0], idx, sizeof(int32_t) * (size_t)n, &di)) return rc;
    if (int rc = in_dev(ctx, t.b[1], l, sizeof(double) * (size_t)n, &dl)) return rc;
    if (int rc = in_dev(ctx, t.b[2], q, sizeof(double) * (size_t)n, &dq)) return rc;
    if (int rc = in_dev(ctx, t.b[3], sigma, sizeof(double) * (size_t)n, &dsg)) return rc;
    CUDA_TRY(ctx, t.b[4].ensure(sizeof(int32_t) * ((size_t)n + 1)));
    CUDA_TRY(ctx, t.b[5].ensure(sizeof(double) * ((size_t)n + 1)));
    int* dorder = t.b[4].as<int>();
    double* dw = t.b[5].as<double>();
    if (n > 0) {
        ray_sort_kernel<<<1, 1024, 0, ctx->stream>>>(n, static_cast<const int*>(di), static_cast<const double*>(dl),
                                                     nullptr, 0.0, 0, dorder, dorder + n);
        LAUNCH_CHECK(ctx);
    }
    blend_ray_kernel<<<blocks_for(n > 0 ? n : 1, 128), 128, 0, ctx->stream>>>(
        n, dorder, static_cast<const double*>(dl), static_cast<const double*>(dq), static_cast<const double*>(dsg), tau,
        dw, dw + n);
    LAUNCH_CHECK(ctx);
    std::vector<int32_t> ord((size_t)n);
    bool host = false;
    int rc;
    if (n > 0 && (rc = copy_out(ctx, ord.data(), dorder, sizeof(int32_t) * (size_t)n, &host))) return rc;
    if (n > 0 && (rc = copy_out(ctx, out_w, dw, sizeof(double) * (size_t)n, &host))) return rc;
    if ((rc = copy_out(ctx, alpha, dw + n, sizeof(double), &host))) return rc;
    if ((rc = sync_and_check(ctx))) return rc;
    // the sorted kernel indices (host input: re-read; device input: gathered on the host copy)
    std::vector<int32_t> hidx((size_t)n);
    if (n > 0) {
        CUDA_TRY(ctx, cudaMemcpy(hidx.data(), di, sizeof(int32_t) * (size_t)n, cudaMemcpyDefault));
        std::vector<int32_t> sorted_idx((size_t)n);
        for (int k = 0; k < n; ++k) sorted_idx[(size_t)k] = hidx[(size_t)ord[(size_t)k]];
        CUDA_TRY(ctx, cudaMemcpy(out_idx, sorted_idx.data(), sizeof(int32_t) * (size_t)n, cudaMemcpyDefault));
    }
    return GVR_OK;
}

int gvr_transmittance_ray(gvr_context* ctx, int32_t n, const double* l, const double* q, const double* sigma,
                          double tau, int32_t nt, const double* t_in, double* out) {
    if (!ctx || n < 0 || nt < 0 || (n > 0 && (!l || !q || !sigma)) || (nt > 0 && (!t_in || !out)))
        return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (nt == 0) return GVR_OK;
    Tmp t;
    const void *dl = nullptr, *dq = nullptr, *dsg = nullptr, *dt;
    if (n > 0) {
        if (int rc = in_dev(ctx, t.b[0], l, sizeof(double) * (size_t)n, &dl)) return rc;
        if (int rc = in_dev(ctx, t.b[1], q, sizeof(double) * (size_t)n, &dq)) return rc;
        if (int rc = in_dev(ctx, t.b[2], sigma, sizeof(double) * (size_t)n, &dsg)) return rc;
    }
    if (int rc = in_dev(ctx, t.b[3], t_in, sizeof(double) * (size_t)nt, &dt)) return rc;
    CUDA_TRY(ctx, t.b[4].ensure(sizeof(double) * (size_t)nt));
    transmittance_ray_kernel<<<blocks_for(nt, 128), 128, 0, ctx->stream>>>(
        n, static_cast<const double*>(dl), static_cast<const double*>(dq), static_cast<const double*>(dsg), tau, nt,
        static_cast<const double*>(dt), t.b[4].as<double>());
    LAUNCH_CHECK(ctx);
    bool host = false;
    if (int rc = copy_out(ctx, out, t.b[4].p, sizeof(double) * (size_t)nt, &host)) return rc;
    return sync_and_check(ctx);
}

int gvr_normalized_weights_ray(gvr_context* ctx, int32_t n, const double* w, double eps, double* out) {
    if (!ctx || n < 0 || (n > 0 && (!w || !out))) return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    if (n == 0) return GVR_OK;
    Tmp t;
    const void* dw;
    if (int rc = in_dev(ctx, t.b[0], w, sizeof(double) * (size_t)n, &dw)) return rc;
    CUDA_TRY(ctx, t.b[1].ensure(sizeof(double) * (size_t)n));
    normalized_weights_ray_kernel<<<1, 256, 0, ctx->stream>>>(n, static_cast<const double*>(dw), eps,
                                                               t.b[1].as<double>());
    LAUNCH_CHECK(ctx);
    bool host = false;
    if (int rc = copy_out(ctx, out, t.b[1].p, sizeof(double) * (size_t)n, &host)) return rc;
    return sync_and_check(ctx);
}

int gvr_scalar_loss_buffers(gvr_context* ctx, int64_t n_img, const double* image, const double* target_image,
                            int64_t n_alpha, const double* alpha, const double* target_alpha, double w_image,
                            double w_alpha, double* loss, double* d_image, double* d_alpha) {
    if (!ctx || n_img < 0 || n_alpha < 0 || !loss || (n_img > 0 && (!image || !target_image)) ||
        (n_alpha > 0 && (!alpha || !target_alpha)))
        return set_err(ctx, GVR_ERR_RUNTIME, "null argument");
    Tmp t;
    const void *di = nullptr, *dti = nullptr, *da = nullptr, *dta = nullptr;
    if (n_img > 0) {
        if (int rc = in_dev(ctx, t.b[0], image, sizeof(double) * (size_t)n_img, &di)) return rc;
        if (int rc = in_dev(ctx, t.b[1], target_image, sizeof(double) * (size_t)n_img, &dti)) return rc;
    }
    if (n_alpha > 0) {
        if (int rc = in_dev(ctx, t.b[2], alpha, sizeof(double) * (size_t)n_alpha, &da)) return rc;
        if (int rc = in_dev(ctx, t.b[3], target_alpha, sizeof(double) * (size_t)n_alpha, &dta)) return rc;
    }
    CUDA_TRY(ctx, t.b[4].ensure(sizeof(double) * ((size_t)n_img + (size_t)n_alpha + 1)));
    double* dout = t.b[4].as<double>();
    loss_buffers_kernel<<<1, 1024, 0, ctx->stream>>>(
        n_img, static_cast<const double*>(di), static_cast<const double*>(dti), n_alpha, static_cast<const double*>(da),
        static_cast<const double*>(dta), w_image, w_alpha, d_image ? dout : nullptr,
        d_alpha ? dout + n_img : nullptr, dout + n_img + n_alpha);
    LAUNCH_CHECK(ctx);
    bool host = false;
    int rc;
    if (d_image && n_img > 0 && (rc = copy_out(ctx, d_image, dout, sizeof(double) * (size_t)n_img, &host))) return rc;
    if (d_alpha && n_alpha > 0 && (rc = copy_out(ctx, d_alpha, dout + n_img, sizeof(double) * (size_t)n_alpha, &host)))
        return rc;
    if ((rc = copy_out(ctx, loss, dout + n_img + n_alpha, sizeof(double), &host))) return rc;
    return sync_and_check(ctx);
}

}  // extern "C"
