// Building blocks of the reference API on the device (tracer.hpp:45-54,
// blender.hpp:29-36, scene.hpp:10-19, grad.hpp:68): the per-ray / per-kernel
// functions the C++ drop-in (include/gvr/*.hpp) exposes with the reference's
// signatures. Same formulas and evaluation order as the render path's exact
// FP64 helpers; one launch per call (API convenience, not the render path).
#pragma once

#include "project.cuh"

namespace gvrk {

// trace_kernel (tracer.cpp:20-35) for n (ray, kernel) pairs. *bad receives the
// smallest pair index with d.Sd <= 0 (the reference throws there).
__global__ void trace_pairs_kernel(long long n, const double* __restrict__ dirs, const double* __restrict__ centers,
                                   const double* __restrict__ inv_cov, double* __restrict__ l, double* __restrict__ q,
                                   double* __restrict__ sigma, unsigned long long* bad) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    Rec64 r;
#pragma unroll
    for (int t = 0; t < 3; ++t) r.m[t] = centers[3 * i + t];
#pragma unroll
    for (int t = 0; t < 9; ++t) r.s[t] = inv_cov[9 * i + t];
    xmatvec(r.s, r.m, r.sm);
    const double d[3] = {dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]};
    const Traced64 t = trace_exact(d, r);
    if (!(t.a > 0.0)) atomicMin(bad, (unsigned long long)i);
    l[i] = t.l;
    q[i] = t.q;
    sigma[i] = sigma_of(t.a);
}

// view_transform (scene.cpp:5-17) of K kernels.
__global__ void view_transform_kernel(int K, CameraP cam, const double* __restrict__ centers,
                                      const double* __restrict__ inv_cov, double* __restrict__ out_c,
                                      double* __restrict__ out_s) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    double mo[3], so[9], m[3], s[9];
#pragma unroll
    for (int t = 0; t < 3; ++t) mo[t] = centers[3ll * k + t];
#pragma unroll
    for (int t = 0; t < 9; ++t) so[t] = inv_cov[9ll * k + t];
    view_transform_one(cam, mo, so, m, s);
#pragma unroll
    for (int t = 0; t < 3; ++t) out_c[3ll * k + t] = m[t];
#pragma unroll
    for (int t = 0; t < 9; ++t) out_s[9ll * k + t] = s[t];
}

// pixel_ray (scene.cpp:19-22) for n pixels (rows / cols given, or every pixel
// in row-major order when rows == nullptr: generate_rays, scene.cpp:24-33).
__global__ void pixel_rays_kernel(CameraP cam, long long n, const int* __restrict__ rows, const int* __restrict__ cols,
                                  double* __restrict__ dirs) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = rows ? rows[i] : (int)(i / cam.W), c = cols ? cols[i] : (int)(i % cam.W);
    double d[3];
    pixel_ray(cam, r, c, d);
#pragma unroll
    for (int t = 0; t < 3; ++t) dirs[3 * i + t] = d[t];
}

// coarse_select boxes (tracer.cpp:37-104): the projection of the render path
// (project_one) with the reference's pushed pixel box written per kernel.
__global__ void coarse_box_kernel(ProjectParams p) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < p.K) project_one(p, k);
}

// A traced entry in the (l, kernel index) order of fine_select / blend
// (tracer.cpp:119-122, blender.cpp:29-32); pos = the entry's input position.
struct SortEnt {
    double l;
    int idx, pos;
};

__device__ __forceinline__ bool ent_less(const SortEnt& a, const SortEnt& b) {
    return a.l < b.l || (a.l == b.l && (a.idx < b.idx || (a.idx == b.idx && a.pos < b.pos)));
}

// One CTA: entries with keep (q > log_eta, or all when !filter) compacted in
// input order, then sorted by (l, idx) with a shared-memory bitonic sort
// (n <= kRaySortMax); out_pos[0..m) = input positions in sorted order, *m_out = m.
constexpr int kRaySortMax = 2048;

__global__ void __launch_bounds__(1024) ray_sort_kernel(int n, const int* __restrict__ idx, const double* __restrict__ l,
                                                        const double* __restrict__ q, double log_eta, int filter,
                                                        int* __restrict__ out_pos, int* __restrict__ m_out) {
    __shared__ SortEnt s[kRaySortMax];
    __shared__ int s_count;
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    // order-preserving compaction: one warp-aggregated pass per 1024 entries
    for (int base = 0; base < n; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const bool keep = i < n && (!filter || q[i] > log_eta);
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        __shared__ int s_wsum[32];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) s_wsum[warp] = __popc(b);
        __syncthreads();
        int before = 0;
        for (int w = 0; w < warp; ++w) before += s_wsum[w];
        const int pos = s_count + before + __popc(b & ((1u << lane) - 1u));
        if (keep) s[pos] = SortEnt{l[i], idx[i], i};
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += s_wsum[w];
            s_count += tot;
        }
        __syncthreads();
    }
    const int m = s_count;
    int np2 = 1;
    while (np2 < m) np2 <<= 1;
    for (int i = m + threadIdx.x; i < np2; i += blockDim.x) s[i] = SortEnt{INFINITY, 0x7fffffff, 0x7fffffff};
    __syncthreads();
    for (int size = 2; size <= np2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < np2; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool asc = (i & size) == 0;
                    const SortEnt a = s[i], b = s[j];
                    if (ent_less(b, a) == asc) {
                        s[i] = b;
                        s[j] = a;
                    }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < m; i += blockDim.x) out_pos[i] = s[i].pos;
    if (threadIdx.x == 0) *m_out = m;
}

// Standard normal CDF via erfc (blender.cpp:13-15).
__device__ __forceinline__ double normal_cdf_ref(double x) { return 0.5 * erfc(-x * 0.7071067811865476); }

// blend (blender.cpp:27-53) of one ray whose entries are already in (l, idx)
// order (ray_sort_kernel): W_k = exp(-tau sum_m e^{q_m} Phi((l_k - l_m)/sigma_m)) e^{q_k},
// sums over m in order; alpha = 1 - exp(-tau sum e^q).
__global__ void blend_ray_kernel(int n, const int* __restrict__ order, const double* __restrict__ l,
                                 const double* __restrict__ q, const double* __restrict__ sigma, double tau,
                                 double* __restrict__ w_out, double* __restrict__ alpha) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k == 0) {
        double total = 0.0;
        for (int m = 0; m < n; ++m) total += exp(q[order[m]]);
        *alpha = 1.0 - exp(-tau * total);
    }
    if (k >= n) return;
    const int ik = order[k];
    double acc = 0.0;
    for (int m = 0; m < n; ++m) {
        const int im = order[m];
        acc += exp(q[im]) * normal_cdf_ref((l[ik] - l[im]) / sigma[im]);
    }
    w_out[k] = exp(-tau * acc) * exp(q[ik]);
}

// transmittance_at (blender.cpp:19-25) of one ray at n depths t, entries in input order.
__global__ void transmittance_ray_kernel(int n, const double* __restrict__ l, const double* __restrict__ q,
                                         const double* __restrict__ sigma, double tau, int nt,
                                         const double* __restrict__ t, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nt) return;
    double acc = 0.0;
    for (int k = 0; k < n; ++k) acc += exp(q[k]) * normal_cdf_ref((t[i] - l[k]) / sigma[k]);
    out[i] = exp(-tau * acc);
}

// normalized_weights (blender.cpp:55-62): W / max(sum W, eps), sum in order.
__global__ void normalized_weights_ray_kernel(int n, const double* __restrict__ w, double eps, double* __restrict__ out) {
    __shared__ double s_den;
    if (threadIdx.x == 0) {
        double total = 0.0;
        for (int k = 0; k < n; ++k) total += w[k];
        s_den = fmax(total, eps);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += blockDim.x) out[k] = w[k] / s_den;
}

// ScalarLoss::value (grad.cpp:201-216) on caller buffers (C++ drop-in): one
// CTA, each thread sums a contiguous chunk of (image ++ alpha) in order, the
// chunks are added in order (deterministic).
__global__ void __launch_bounds__(1024) loss_buffers_kernel(long long n_img, const double* __restrict__ img,
                                                            const double* __restrict__ t_img, long long n_alpha,
                                                            const double* __restrict__ alpha,
                                                            const double* __restrict__ t_alpha, double w_image,
                                                            double w_alpha, double* __restrict__ d_img,
                                                            double* __restrict__ d_alpha, double* __restrict__ loss) {
    __shared__ double part[1024];
    const long long n = n_img + n_alpha;
    const long long chunk = (n + blockDim.x - 1) / blockDim.x;
    const long long i0 = (long long)threadIdx.x * chunk, i1 = min(n, i0 + chunk);
    double acc = 0.0;
    for (long long i = i0; i < i1; ++i) {
        if (i < n_img) {
            const double diff = img[i] - t_img[i];
            acc += 0.5 * w_image * diff * diff;
            if (d_img) d_img[i] = w_image * diff;
        } else {
            const double diff = alpha[i - n_img] - t_alpha[i - n_img];
            acc += 0.5 * w_alpha * diff * diff;
            if (d_alpha) d_alpha[i - n_img] = w_alpha * diff;
        }
    }
    part[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int t = 0; t < (int)blockDim.x; ++t) tot += part[t];
        *loss = tot;
    }
}

}  // namespace gvrk
