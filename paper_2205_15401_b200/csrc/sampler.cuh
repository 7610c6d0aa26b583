// Kernels over a taped render: the attribute sampler and the per-pixel API
// helpers of the reference render path.
//
//   sample_scatter_kernel / sample_finalize_kernel  sample_attributes (sampler.cpp:11-51)
//   resynth_attr_kernel                             resynthesize      (sampler.cpp:53-66)
//   transmittance_kernel                            transmittance_at  (blender.cpp:19-25)
//   normalized_weights_kernel                       normalized_weights(blender.cpp:55-62)
//   shade_lambert_kernel                            shade_lambert     (blender.cpp:146-172)
//
// The sampler reads the weights from the tape: W = T(l_k) (taped in FP64 by the
// blend) times the FP32-rounded peak e^{q_k} recomputed with the same
// trace_fast, i.e. exactly the W the forward blended with (blend_kernel), so
// "sampling weights are exactly the rendering weights" (test_sampler.cpp:162)
// holds bit for bit against our own render.
#pragma once

#include "gvr_common.cuh"

namespace gvrk {

struct TapeView {
    CameraP cam;
    int kp;
    const int* topk;       // [P*kp] ascending (l, idx)
    const int* count;      // [P]
    const double* tape_t;  // [P*kp] T(l_k)
    const EntryRec* ent;   // [P*kp] traced entries (e^q as blended)
    const Rec64* rec64;    // [K]
};

// W of the taped entry (pix, s); identical to blend_kernel's wd.
__device__ __forceinline__ double taped_weight(const TapeView& v, const double* d, long long pix, int s) {
    (void)d;
    return v.tape_t[pix * v.kp + s] * (double)v.ent[pix * v.kp + s].pk;
}

// One thread per pixel, row-major pixels; FP64 atomics into the per-kernel sums.
// Support (and with `normalized`, W / max(sum W, 1e-8)) and the weighted
// observation sums (sampler.cpp:29-44).
__global__ void sample_scatter_kernel(TapeView v, const double* __restrict__ observed, int C, int normalized,
                                      double* __restrict__ support, double* __restrict__ attrs) {
    const long long P = (long long)v.cam.H * v.cam.W;
    const long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (pix >= P) return;
    const int n = v.count[pix];
    if (n == 0) return;
    double d[3];
    pixel_ray(v.cam, (int)(pix / v.cam.W), (int)(pix % v.cam.W), d);
    double denom = 1.0;
    if (normalized) {
        double total = 0.0;
        for (int s = 0; s < n; ++s) total += taped_weight(v, d, pix, s);
        denom = total > 1e-8 ? total : 1e-8;  // kSupportEps (sampler.hpp:18)
    }
    for (int s = 0; s < n; ++s) {
        const int k = v.topk[pix * v.kp + s];
        double ww = taped_weight(v, d, pix, s);
        if (normalized) ww = ww / denom;
        atomicAdd(support + k, ww);
        for (int c = 0; c < C; ++c) atomicAdd(attrs + (long long)C * k + c, ww * observed[pix * C + c]);
    }
}

// support < kSupportEps -> zero + masked; else attrs /= support (sampler.cpp:46-54).
__global__ void sample_finalize_kernel(int K, int C, const double* __restrict__ support, double* __restrict__ attrs,
                                       unsigned char* __restrict__ masked) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const double sp = support[k];
    const bool m = sp < 1e-8;
    for (int c = 0; c < C; ++c) {
        const long long o = (long long)C * k + c;
        attrs[o] = m ? 0.0 : attrs[o] / sp;
    }
    masked[k] = m ? 1 : 0;
}

// recolored.attr = masked ? 0 : sampled (sampler.cpp:58-63)
__global__ void resynth_attr_kernel(long long n, int C, const double* __restrict__ sampled,
                                    const unsigned char* __restrict__ masked, double* __restrict__ attr) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o >= n) return;
    attr[o] = masked && masked[o / C] ? 0.0 : sampled[o];
}

// T(t_p) = exp(-tau sum_m e^{q_m} Phi((t_p - l_m)/sigma_m)) over the pixel's
// selected kernels, exact FP64 trace and erfc (blender.cpp:19-25).
__global__ void transmittance_kernel(TapeView v, double tau, const double* __restrict__ t, double* __restrict__ out) {
    const long long P = (long long)v.cam.H * v.cam.W;
    const long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (pix >= P) return;
    const int n = v.count[pix];
    double d[3];
    pixel_ray(v.cam, (int)(pix / v.cam.W), (int)(pix % v.cam.W), d);
    const double tp = t[pix];
    double acc = 0.0;
    for (int s = 0; s < n; ++s) {
        const Traced64 tr = trace_exact(d, v.rec64[v.topk[pix * v.kp + s]]);
        acc += exp(tr.q) * (0.5 * erfc(-((tp - tr.l) / sigma_of(tr.a)) * 0.7071067811865476));
    }
    out[pix] = exp(-tau * acc);
}

// W_k / max(sum W, eps), K'-padded with 0 (blender.cpp:55-62).
__global__ void normalized_weights_kernel(TapeView v, double eps, double* __restrict__ out) {
    const long long P = (long long)v.cam.H * v.cam.W;
    const long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (pix >= P) return;
    const int n = v.count[pix];
    double d[3];
    pixel_ray(v.cam, (int)(pix / v.cam.W), (int)(pix % v.cam.W), d);
    double total = 0.0;
    for (int s = 0; s < n; ++s) total += taped_weight(v, d, pix, s);
    const double denom = total > eps ? total : eps;
    for (int s = 0; s < v.kp; ++s) out[pix * v.kp + s] = s < n ? taped_weight(v, d, pix, s) / denom : 0.0;
}

// Diffuse shading of a normal image (blender.cpp:146-172): surface point from
// depth along the pixel ray, mapped to object space by R^T (p - T).
__global__ void shade_lambert_kernel(CameraP cam, const double* __restrict__ normals, const double* __restrict__ alpha,
                                     const double* __restrict__ depth, double lx, double ly, double lz, double cr,
                                     double cg, double cb, double* __restrict__ out) {
    const long long P = (long long)cam.H * cam.W;
    const long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (pix >= P) return;
    double o0 = 0.0, o1 = 0.0, o2 = 0.0;
    double n0 = normals[3 * pix], n1 = normals[3 * pix + 1], n2 = normals[3 * pix + 2];
    const double len = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
    if (alpha[pix] > 0.0 && len >= 1e-12) {
        n0 /= len;
        n1 /= len;
        n2 /= len;
        double d[3];
        pixel_ray(cam, (int)(pix / cam.W), (int)(pix % cam.W), d);
        const double z = depth[pix];
        const double pc0 = z * d[0] - cam.T[0], pc1 = z * d[1] - cam.T[1], pc2 = z * d[2] - cam.T[2];
        // R^T pc
        const double po0 = cam.R[0] * pc0 + cam.R[3] * pc1 + cam.R[6] * pc2;
        const double po1 = cam.R[1] * pc0 + cam.R[4] * pc1 + cam.R[7] * pc2;
        const double po2 = cam.R[2] * pc0 + cam.R[5] * pc1 + cam.R[8] * pc2;
        double t0 = lx - po0, t1 = ly - po1, t2 = lz - po2;
        const double tn = sqrt(t0 * t0 + t1 * t1 + t2 * t2);
        t0 /= tn;
        t1 /= tn;
        t2 /= tn;
        const double inten = fmax(0.0, n0 * t0 + n1 * t1 + n2 * t2);
        o0 = inten * cr;
        o1 = inten * cg;
        o2 = inten * cb;
    }
    out[3 * pix] = o0;
    out[3 * pix + 1] = o1;
    out[3 * pix + 2] = o2;
}

}  // namespace gvrk
