// K3: fused per-pixel trace -> eta filter -> K'-nearest selection -> closed-form blend.
#pragma once

#include "gvr_common.cuh"

namespace gvrk {

struct FwdParams {
    CameraP cam;
    SelP sel;
    int D, Dc;
    double tau;
    float guard_abs;     // FP32 pre-filter guard band on q (absolute)
    float prefilter_c1;  // 1 - relative slack
    int tiles_x;
    int need_predicate;  // coarse cells not aligned to tiles: per-pixel exact cell test
    const int* tile_start;
    const int* tile_end;
    const int* vals;   // sorted kernel ids
    const Rec32* rec32;
    const Rec64* rec64;
    const double* attr;  // [K*D] object attributes (FP64)
    // outputs
    double* image;  // [P*Dc]
    double* alpha;  // [P]
    double* depth;  // [P]
    int* topk;      // [P*kp], first count[p] valid
    int* count;     // [P]
    double* topk_w; // [P*kp] or null
    int* nonfinite; // flag
};

// FP32 centre-relative pre-filter (conservative): true unless q is certainly
// <= ln(eta). With dt = ((i-Oy)/F, (j-Ox)/F, 1), delta = m - z dt =
// (z/F)(c_i - i, c_j - j, 0) is formed without cancellation from the integer
// and fractional parts of the projected centre, and
//   q = -(delta.S.delta - (dt.S.delta)^2 / dt.S.dt) / 2
// (the line minimum is parametrisation independent). Division-free test:
//   dSd*A - B^2 < 2 (g - ln eta) A  (+ relative slack), A = dt.S.dt > 0.
__device__ __forceinline__ bool prefilter_pass(const Rec32& r, int i, int j, float u, float v, float c2,
                                               float c1) {
    if (r.zf < 0.0f) return true;  // unusual geometry: exact path only
    const float di = (float)(r.ci_int - i) + r.ci_frac;
    const float dj = (float)(r.cj_int - j) + r.cj_frac;
    const float dx = r.zf * di, dy = r.zf * dj;
    const float sd0 = fmaf(r.s00, u, fmaf(r.s01, v, r.s02));
    const float sd1 = fmaf(r.s01, u, fmaf(r.s11, v, r.s12));
    const float sd2 = fmaf(r.s02, u, fmaf(r.s12, v, r.s22));
    const float A = fmaf(u, sd0, fmaf(v, sd1, sd2));
    const float B = fmaf(dx, sd0, dy * sd1);
    const float dsd = fmaf(dx, fmaf(r.s00, dx, 2.0f * r.s01 * dy), r.s11 * dy * dy);
    return fmaf(dsd * c1, A, -B * B) < c2 * A;
}

// Sorted (ascending (l, idx)) list with KMAX slots holding K' <= KMAX live
// entries: slots [0, KMAX-K') are dead (-inf, never displaced), the rest start
// empty (+inf); the current K'-th nearest is always slot KMAX-1. The FP64 keys
// live in registers (static indices), the kernel ids in shared memory
// ([slot][thread], read only to break exact ties and written on shifts).
template <int KMAX, int NT>
struct TopK {
    double l[KMAX];
    int* id;  // smem + tid, stride NT

    __device__ __forceinline__ void init(int kp, int* base) {
        id = base;
#pragma unroll
        for (int s = 0; s < KMAX; ++s) l[s] = (s < KMAX - kp) ? -INFINITY : INFINITY;
    }
    __device__ __forceinline__ double worst() const { return l[KMAX - 1]; }
    __device__ __forceinline__ bool less_than_slot(double cl, int ci, int s) const {
        return cl < l[s] || (cl == l[s] && ci < id[s * NT]);
    }
    __device__ __forceinline__ bool accepts(double cl, int ci) const { return less_than_slot(cl, ci, KMAX - 1); }
    // Precondition: accepts(cl, ci). Candidates arrive roughly in ascending l
    // (lists are sorted by the depth bound), so insert from the back; the
    // shifting stops at the first slot that stays put, usually after 1-2 steps.
    __device__ __forceinline__ void insert(double cl, int ci) {
        bool placed = false;
#pragma unroll
        for (int s = KMAX - 1; s > 0; --s) {
            if (!placed) {
                if (less_than_slot(cl, ci, s - 1)) {
                    l[s] = l[s - 1];
                    id[s * NT] = id[(s - 1) * NT];
                } else {
                    l[s] = cl;
                    id[s * NT] = ci;
                    placed = true;
                }
            }
        }
        if (!placed) {
            l[0] = cl;
            id[0] = ci;
        }
    }
};

template <int KMAX, int TILE>
__global__ void __launch_bounds__(TILE* TILE, KMAX <= 24 ? 8 : (KMAX <= 32 ? 5 : 4)) fine_forward_kernel(FwdParams p) {
    constexpr int NT = TILE * TILE;
    extern __shared__ __align__(16) unsigned char smem[];
    // region A: candidate chunk (selection) / blend staging (after selection)
    Rec32* s32 = reinterpret_cast<Rec32*>(smem);
    Rec64* s64 = reinterpret_cast<Rec64*>(s32 + NT);
    int* sidx = reinterpret_cast<int*>(s64 + NT);
    double* b_dl = reinterpret_cast<double*>(smem);  // l relative to the nearest entry (FP64)
    float* b_pk = reinterpret_cast<float*>(b_dl + KMAX * NT);
    float* b_is = b_pk + KMAX * NT;
    // region H: kernel ids of the selection list, [slot][thread]
    constexpr size_t kRegionA = (sizeof(Rec32) + sizeof(Rec64) + sizeof(int)) * NT > 16 * KMAX * NT
                                    ? (sizeof(Rec32) + sizeof(Rec64) + sizeof(int)) * NT
                                    : 16 * KMAX * NT;
    int* h_id = reinterpret_cast<int*>(smem + kRegionA);

    const int tid = threadIdx.x;
    const int tile = blockIdx.x;
    const int i = (tile / p.tiles_x) * TILE + tid / TILE;
    const int j = (tile % p.tiles_x) * TILE + tid % TILE;
    const bool inside = i < p.cam.H && j < p.cam.W;
    const int list = p.sel.coarse ? tile : 0;
    const int start = p.tile_start[list];
    const int end = p.tile_end[list];
    const long long pix = (long long)i * p.cam.W + j;

    double d[3];
    pixel_ray(p.cam, inside ? i : 0, inside ? j : 0, d);
    const float u = (float)xdiv(xsub((double)i, p.cam.oy), p.cam.focal);
    const float v = (float)xdiv(xsub((double)j, p.cam.ox), p.cam.focal);
    const int ci = i / p.sel.ds, cj = j / p.sel.ds;
    const float c2 = 2.0f * (p.guard_abs - (float)p.sel.log_eta);
    const double log_eta = p.sel.log_eta;

    TopK<KMAX, NT> top;
    top.init(p.sel.kp, h_id + tid);
    bool done = !inside;

    for (int base = start; base < end; base += NT) {
        __syncthreads();
        const int e = base + tid;
        if (e < end) {
            const int k = p.vals[e];
            sidx[tid] = k;
            s32[tid] = p.rec32[k];
            s64[tid] = p.rec64[k];
        }
        __syncthreads();
        const int cnt = min(NT, end - base);
        if (!done) {
            for (int c = 0; c < cnt; ++c) {
                const Rec32& r = s32[c];
                // early exit: lists are sorted by the depth bound zmin <= l
                if ((double)r.zmin > top.worst()) {
                    done = true;
                    break;
                }
                if (p.need_predicate && !(ci >= r.cr_lo && ci <= r.cr_hi && cj >= r.cc_lo && cj <= r.cc_hi)) continue;
                if (!prefilter_pass(r, i, j, u, v, c2, p.prefilter_c1)) continue;
                const Traced64 t = trace_exact(d, s64[c]);
                if (!(t.q > log_eta)) continue;  // fine_select threshold (tracer.cpp:117-118)
                const int k = sidx[c];
                if (top.accepts(t.l, k)) top.insert(t.l, k);
            }
        }
        if (!__syncthreads_or(!done)) break;
    }
    __syncthreads();  // chunk buffers are re-used below

    if (!inside) return;

    // The selection (ascending (l, idx)) occupies slots [KMAX-K', KMAX-K'+n).
    int n = 0;
#pragma unroll
    for (int s = 0; s < KMAX; ++s) n += isfinite(top.l[s]) ? 1 : 0;
    const int* b_id = h_id + (KMAX - p.sel.kp) * NT;
    // Stage the selected entries: FP64 re-trace for q and sigma, l relative to
    // the nearest entry so the pairwise differences keep FP64 accuracy.
    double l0 = 0.0, total_peak = 0.0;
    for (int s = 0; s < n; ++s) {
        const int k = b_id[s * NT + tid];
        const Traced64 t = trace_exact(d, p.rec64[k]);
        if (s == 0) l0 = t.l;
        const double pk = exp(t.q);
        total_peak += pk;
        b_dl[s * NT + tid] = t.l - l0;
        b_pk[s * NT + tid] = (float)pk;
        b_is[s * NT + tid] = (float)__dsqrt_rn(t.a);  // 1/sigma
        p.topk[pix * p.sel.kp + s] = k;
    }
    p.count[pix] = n;

    // blend (blender.cpp:27-53): W_k = exp(-tau sum_m e^{q_m} Phi((l_k - l_m)/sigma_m)) e^{q_k}
    const float tau = (float)p.tau;
    double img[4] = {0.0, 0.0, 0.0, 0.0};
    double wsum = 0.0, wl = 0.0;
    for (int k = 0; k < n; ++k) {
        const double dlk = b_dl[k * NT + tid];
        float acc = 0.0f;
        for (int m = 0; m < n; ++m) {
            const float z = (float)((dlk - b_dl[m * NT + tid]) * (double)b_is[m * NT + tid]);
            acc = fmaf(b_pk[m * NT + tid], fast_normal_cdf(z), acc);
        }
        const float w = expf(-tau * acc) * b_pk[k * NT + tid];
        const double wd = (double)w;
        const int kid = b_id[k * NT + tid];
        if (p.D <= 4) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (c < p.D) img[c] = xadd(img[c], xmul(wd, p.attr[(long long)p.D * kid + c]));
        } else {
            for (int c = 0; c < p.D; ++c) {
                const long long o = pix * p.Dc + c;
                p.image[o] = xadd(k == 0 ? 0.0 : p.image[o], xmul(wd, p.attr[(long long)p.D * kid + c]));
            }
        }
        wsum += wd;
        wl += wd * (l0 + dlk);
        if (p.topk_w) p.topk_w[pix * p.sel.kp + k] = wd;
    }
    if (p.D <= 4) {
        for (int c = 0; c < p.Dc; ++c) p.image[pix * p.Dc + c] = img[c];
    } else if (n == 0) {
        for (int c = 0; c < p.Dc; ++c) p.image[pix * p.Dc + c] = 0.0;
    }
    const double alpha = 1.0 - exp(-p.tau * total_peak);
    const double depth = wsum > 1e-12 ? wl / wsum : 0.0;
    p.alpha[pix] = alpha;
    p.depth[pix] = depth;
    if (!isfinite(alpha) || !isfinite(depth) || !isfinite(wsum)) atomicExch(p.nonfinite, 1);
}

}  // namespace gvrk
