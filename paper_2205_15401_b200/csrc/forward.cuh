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
    const int* tile_order;  // tiles by list length, longest first (LPT); first *n_order valid
    const int* n_order;
    const int* tile_order_blend;  // tiles by sum_p n_p^2 (from the selection); first *n_order_blend valid
    const int* n_order_blend;
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
    double* tape_t; // [P*kp] T(l_k) of the selected entries (backward input)
    float* bwd_cost; // [tiles] sum_p n_p^2 of each tile (backward scheduling)
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

// Per-warp candidate chunk entry.
struct __align__(16) Cand {
    Rec32 r;
    int k;
    int pad[3];
};

// Worst (largest (l, idx)) of the n kept entries of this thread.
__device__ __forceinline__ void find_worst(const double* s_l, const int* s_id, int n, int tid, double& wl, int& wid,
                                           int& wslot) {
    wl = s_l[tid];
    wid = s_id[tid];
    wslot = 0;
    for (int s = 1; s < n; ++s) {
        const double ls = s_l[s * 64 + tid];
        const int is = s_id[s * 64 + tid];
        if (traced_less(wl, wid, ls, is)) {
            wl = ls;
            wid = is;
            wslot = s;
        }
    }
}

// K3a selection. CTA = one 8x8 pixel tile = 2 warps that stream the tile's
// list independently (no CTA barriers; a warp stops as soon as its 32 pixels
// are done). Per pixel, the K' nearest (l, idx) are kept UNSORTED in shared
// memory with the current worst tracked in registers; candidates arrive roughly
// in ascending l (lists are sorted by the depth bound), so replacements after
// the list fills are rare. The FP32 pre-filter of 4 consecutive candidates is
// evaluated together (independent work: instruction-level parallelism for the
// latency-bound pixels that scan whole lists). Output: the selection sorted by
// (l, idx) into the tape, and the tile's backward/blend cost sum n_p^2.
template <int KMAX>
__global__ void __launch_bounds__(64) select_kernel(FwdParams p) {
    constexpr int TILE = 8, NT = 64;
    extern __shared__ __align__(16) unsigned char smem[];
    Cand* chunk = reinterpret_cast<Cand*>(smem) + (threadIdx.x & ~31);
    double* s_l = reinterpret_cast<double*>(smem + sizeof(Cand) * NT);
    int* s_id = reinterpret_cast<int*>(s_l + KMAX * NT);

    if ((int)blockIdx.x >= *p.n_order) return;
    const int tid = threadIdx.x, lane = tid & 31;
    const int tile = p.tile_order[blockIdx.x];
    const int i = (tile / p.tiles_x) * TILE + tid / TILE;
    const int j = (tile % p.tiles_x) * TILE + tid % TILE;
    const bool inside = i < p.cam.H && j < p.cam.W;
    const int start = p.tile_start[tile];
    const int end = p.tile_end[tile];
    const long long pix = (long long)i * p.cam.W + j;
    const int kp = p.sel.kp;

    double d[3];
    pixel_ray(p.cam, inside ? i : 0, inside ? j : 0, d);
    const float u = (float)xdiv(xsub((double)i, p.cam.oy), p.cam.focal);
    const float v = (float)xdiv(xsub((double)j, p.cam.ox), p.cam.focal);
    const float fi = (float)i, fj = (float)j;
    const float c2 = 2.0f * (p.guard_abs - (float)p.sel.log_eta);
    const float c1 = p.prefilter_c1;
    const double log_eta = p.sel.log_eta;

    // selection state: n kept; once full, the worst kept (l, idx) and its slot
    int n = 0, wslot = 0, wid = 0x7fffffff;
    double wl = INFINITY;
    bool done = !inside;

    for (int base = start; base < end; base += 32) {
        if (__all_sync(0xffffffffu, done)) break;
        const int e = base + lane;
        if (e < end) {
            const int k = p.vals[e];
            chunk[lane].r = p.rec32[k];
            chunk[lane].k = k;
        }
        __syncwarp();
        const int cnt = min(32, end - base);
        for (int c0 = 0; c0 < cnt && !done; c0 += 4) {
            // early exit: every later candidate has l >= zmin > worst kept
            if ((double)chunk[c0].r.zmin > wl) {
                done = true;
                break;
            }
            bool pass[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const Rec32& r = chunk[min(c0 + q, cnt - 1)].r;
                pass[q] = c0 + q < cnt && fi >= r.top && fi <= r.bottom && fj >= r.left && fj <= r.right &&
                          prefilter_pass(r, i, j, u, v, c2, c1);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!pass[q]) continue;
                const int k = chunk[c0 + q].k;
                const Traced64 t = trace_exact(d, p.rec64[k]);
                if (!(t.q > log_eta)) continue;  // fine_select threshold (tracer.cpp:117-118)
                if (n < kp) {
                    s_l[n * NT + tid] = t.l;
                    s_id[n * NT + tid] = k;
                    if (++n == kp) find_worst(s_l, s_id, n, tid, wl, wid, wslot);
                } else if (traced_less(t.l, k, wl, wid)) {
                    s_l[wslot * NT + tid] = t.l;
                    s_id[wslot * NT + tid] = k;
                    find_worst(s_l, s_id, n, tid, wl, wid, wslot);
                }
            }
        }
        __syncwarp();
    }

    // tile cost for the blend / backward schedulers
    const int n_eff = inside ? n : 0;
    float cost = (float)(n_eff * n_eff);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cost += __shfl_xor_sync(0xffffffffu, cost, o);
    if (lane == 0 && cost > 0.0f) atomicAdd(p.bwd_cost + tile, cost);
    if (!inside) return;

    // sort the selection ascending by (l, idx): insertion sort of nearly sorted input
    for (int s = 1; s < n; ++s) {
        const double ls = s_l[s * NT + tid];
        const int is = s_id[s * NT + tid];
        int t = s - 1;
        while (t >= 0 && traced_less(ls, is, s_l[t * NT + tid], s_id[t * NT + tid])) {
            s_l[(t + 1) * NT + tid] = s_l[t * NT + tid];
            s_id[(t + 1) * NT + tid] = s_id[t * NT + tid];
            --t;
        }
        s_l[(t + 1) * NT + tid] = ls;
        s_id[(t + 1) * NT + tid] = is;
    }
    for (int s = 0; s < n; ++s) p.topk[pix * kp + s] = s_id[s * NT + tid];
    p.count[pix] = n;
}

// K3b closed-form blend (blender.cpp:27-53, 98-128). CTA = one 8x8 tile with
// 4 threads per pixel (256 threads): entries are re-traced (exact FP64) and the
// O(n^2) transmittance sums split 4 ways; the ordered attribute/depth sums are
// then done by one thread per pixel so that image == sum_k W_k attr_k exactly
// in ascending (l, idx) order.
//   W_k = exp(-tau sum_m e^{q_m} Phi((l_k - l_m)/sigma_m)) e^{q_k}
// The sum is accumulated in FP64 and T(l_k) is taped for the backward.
template <int KMAX>
__global__ void __launch_bounds__(256) blend_kernel(FwdParams p) {
    constexpr int TILE = 8, NP = 64;
    extern __shared__ __align__(16) unsigned char smem[];
    double* b_dl = reinterpret_cast<double*>(smem);  // [slot][pixel] l - l0
    double* b_w = b_dl + KMAX * NP;                  // W_k
    float* b_pk = reinterpret_cast<float*>(b_w + KMAX * NP);
    float* b_is = b_pk + KMAX * NP;
    int* b_id = reinterpret_cast<int*>(b_is + KMAX * NP);

    if ((int)blockIdx.x >= *p.n_order_blend) return;
    const int g = threadIdx.x >> 2, sub = threadIdx.x & 3;
    const int tile = p.tile_order_blend[blockIdx.x];
    const int i = (tile / p.tiles_x) * TILE + g / TILE;
    const int j = (tile % p.tiles_x) * TILE + g % TILE;
    const bool inside = i < p.cam.H && j < p.cam.W;
    const long long pix = (long long)i * p.cam.W + j;
    const int kp = p.sel.kp;
    const int n = inside ? p.count[pix] : 0;
    if (n == 0) {
        if (inside && sub == 0) {
            for (int c = 0; c < p.Dc; ++c) p.image[pix * p.Dc + c] = 0.0;
            p.alpha[pix] = 0.0;
            p.depth[pix] = 0.0;
        }
        return;  // the 4 threads of a pixel leave together
    }
    const unsigned grp = 0xfu << (threadIdx.x & 28);  // the pixel's 4 lanes

    double d[3];
    pixel_ray(p.cam, i, j, d);
    const double l0 = trace_exact(d, p.rec64[p.topk[pix * kp]]).l;
    double peak_part = 0.0;
    for (int s = sub; s < n; s += 4) {
        const int k = p.topk[pix * kp + s];
        const Traced64 t = trace_exact(d, p.rec64[k]);
        const double pk = exp(t.q);
        peak_part += pk;
        b_dl[s * NP + g] = t.l - l0;
        b_pk[s * NP + g] = (float)pk;
        b_is[s * NP + g] = (float)__dsqrt_rn(t.a);  // 1/sigma
        b_id[s * NP + g] = k;
    }
    peak_part += __shfl_xor_sync(grp, peak_part, 1, 4);
    peak_part += __shfl_xor_sync(grp, peak_part, 2, 4);
    __syncwarp(grp);

    for (int k = sub; k < n; k += 4) {
        const double dlk = b_dl[k * NP + g];
        double acc = 0.0;
        for (int m = 0; m < n; ++m) {
            const float z = (float)((dlk - b_dl[m * NP + g]) * (double)b_is[m * NP + g]);
            acc = fma((double)b_pk[m * NP + g], (double)fast_normal_cdf(z), acc);
        }
        const double trans = exp(-p.tau * acc);
        const double wd = trans * (double)b_pk[k * NP + g];
        p.tape_t[pix * kp + k] = trans;
        b_w[k * NP + g] = wd;
        if (p.topk_w) p.topk_w[pix * kp + k] = wd;
    }
    __syncwarp(grp);
    if (sub != 0) return;

    double img[4] = {0.0, 0.0, 0.0, 0.0};
    double wsum = 0.0, wld = 0.0;
    for (int k = 0; k < n; ++k) {
        const double wd = b_w[k * NP + g];
        const int kid = b_id[k * NP + g];
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
        wld += wd * (l0 + b_dl[k * NP + g]);
    }
    if (p.D <= 4)
        for (int c = 0; c < p.Dc; ++c) p.image[pix * p.Dc + c] = img[c];
    const double alpha = 1.0 - exp(-p.tau * peak_part);
    const double depth = wsum > 1e-12 ? wld / wsum : 0.0;
    p.alpha[pix] = alpha;
    p.depth[pix] = depth;
    if (!isfinite(alpha) || !isfinite(depth) || !isfinite(wsum)) atomicExch(p.nonfinite, 1);
}

// Tiles whose pixels selected nothing (zero blend cost) are not visited by the
// blend grid: write their empty-render outputs (image 0, alpha 0, depth 0, count 0).
__global__ void clear_empty_tiles_kernel(CameraP cam, int Dc, int tiles_x, const float* __restrict__ tile_cost,
                                         double* __restrict__ image, double* __restrict__ alpha,
                                         double* __restrict__ depth, int* __restrict__ count) {
    const int tile = blockIdx.x;
    if (tile_cost[tile] > 0.0f) return;
    const int i = (tile / tiles_x) * 8 + threadIdx.x / 8;
    const int j = (tile % tiles_x) * 8 + threadIdx.x % 8;
    if (i >= cam.H || j >= cam.W) return;
    const long long pix = (long long)i * cam.W + j;
    for (int c = 0; c < Dc; ++c) image[pix * Dc + c] = 0.0;
    alpha[pix] = 0.0;
    depth[pix] = 0.0;
    count[pix] = 0;
}

// Longest-processing-time-first order of tiles (single-CTA counting sort over
// log-spaced cost buckets, descending). Zero-cost tiles are dropped and
// *n_out receives the number kept. Cost = list length (fcost == null) or fcost[t].
__global__ void __launch_bounds__(1024) order_tiles_kernel(int tiles, int coarse, const int* __restrict__ start,
                                                           const int* __restrict__ end, const float* __restrict__ fcost,
                                                           int* __restrict__ order, int* __restrict__ n_out) {
    __shared__ int hist[256];
    __shared__ int offs[256];
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    auto bucket_of = [&](int t) -> int {
        float c;
        if (fcost) {
            c = fcost[t];
        } else {
            const int l = coarse ? t : 0;
            c = (float)(end[l] - start[l]);
        }
        if (!(c > 0.0f)) return -1;
        const int b = (int)(__log2f(c + 1.0f) * 8.0f);
        return 255 - min(b, 255);  // descending cost
    };
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
        const int b = bucket_of(t);
        if (b >= 0) atomicAdd(&hist[b], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int b = 0; b < 256; ++b) {
            offs[b] = run;
            run += hist[b];
        }
        *n_out = run;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
        const int b = bucket_of(t);
        if (b >= 0) order[atomicAdd(&offs[b], 1)] = t;
    }
}

}  // namespace gvrk
