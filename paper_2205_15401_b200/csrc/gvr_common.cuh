// Shared device definitions of the B200 render path.
//
// Precision contract:
//  * Everything that DECIDES (culling boxes, the eta threshold, the K' nearest by
//    (l, index), early exit) runs on exact FP64 arithmetic that reproduces the
//    reference's evaluation order without FMA contraction (__dmul_rn/__dadd_rn),
//    so index sets, l, q and sigma are bit-identical to the CPU reference
//    (proj/src/tracer.cpp:20-35, scene.cpp:5-22, tracer.cpp:37-113).
//  * The bulk per-candidate work is an FP32 centre-relative pre-filter that
//    only rejects candidates whose q is below ln(eta) by more than a guard band;
//    survivors are re-traced in FP64 and decided exactly.
//  * The O(n^2) closed-form blend and its backward run in FP32 with FP64
//    accumulation where sums cancel (tolerance 1e-4 relative, north star).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

// Minimum resident CTAs per SM of the per-tile kernels (register budget).
#ifndef GVR_SEL_MINB
#define GVR_SEL_MINB 3
#endif
#ifndef GVR_BLEND_MINB
#define GVR_BLEND_MINB 5
#endif
#ifndef GVR_BLEND_SPLIT
#define GVR_BLEND_SPLIT 2
#endif
#ifndef GVR_BWD_SPLIT
#define GVR_BWD_SPLIT 4
#endif
#ifndef GVR_PDL_SLEEP_NS  // back-off of a blend CTA waiting for its tile's selection
#define GVR_PDL_SLEEP_NS 100
#endif
#ifndef GVR_PDL  // select -> blend per-tile hand-off with programmatic dependent launch
#define GVR_PDL 1
#endif
#ifndef GVR_SEL_SPLIT
#define GVR_SEL_SPLIT 1
#endif
#ifndef GVR_BWD_MINB
#define GVR_BWD_MINB 12
#endif

namespace gvrk {

constexpr double kBehindCameraEps = 1e-4;  // include/gvr/tracer.hpp:28

struct CameraP {
    double R[9];
    double T[3];
    double focal, ox, oy;
    int H, W;
};

struct SelP {
    double eta, log_eta, chi;  // chi = 2 ln(1/eta) (tracer.cpp:47), log_eta (tracer.cpp:117)
    int kp, coarse, ds;
};

// Per-kernel FP32 record for the pre-filters (64 B). The screen box comes
// first so a warp can test it with one 16-byte load per candidate.
struct __align__(16) Rec32 {
    // Screen box of the eta-level set (tracer.cpp:61-98, before the +-1 padding
    // and cell rounding), rounded outward: contains every pixel centre whose ray
    // meets the eta-ellipsoid, i.e. every pixel where q > ln(eta) is possible.
    float top, bottom, left, right;
    float zmin, z;             // zmin = conservative lower bound of l; z = camera-space depth
                               // (FP32; < 0: unusual geometry, exact FP64 path only)
    float ci_frac, cj_frac;
    int ci_int, cj_int;        // screen centre (row, col) = int + frac
    float s00, s01, s02, s11, s12, s22;  // S' = R S R^T, off-diagonals symmetrised (S + S^T) / 2
};

// Per-kernel FP64 camera-space record for the exact trace (128 B).
struct __align__(16) Rec64 {
    double m[3];
    double s[9];
    double sm[3];  // S m (tracer.cpp:30, d^T (S m))
    double pad;
};

// ---------------------------------------------------------------- exact FP64 (no contraction)

// select -> blend per-tile hand-off (programmatic dependent launch)
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* a) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}
// TMA bulk copy global -> shared (cp.async.bulk) completing on an mbarrier.
__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(m)), "r"(count) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the async (TMA) proxy
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(m))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_addr(m)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void red_add_release_gpu(unsigned* a, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
// let the next kernel of the stream (launched with programmatic stream
// serialization) start while this grid's last wave runs
__device__ __forceinline__ void launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }

// y = M x, acc = 0.0; acc += m_ik x_k  (oracle mat_vec / Eigen-shim product order)
__device__ __forceinline__ void xmatvec(const double* m, const double* x, double* y) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double acc = xadd(0.0, xmul(m[3 * i], x[0]));
        acc = xadd(acc, xmul(m[3 * i + 1], x[1]));
        acc = xadd(acc, xmul(m[3 * i + 2], x[2]));
        y[i] = acc;
    }
}

__device__ __forceinline__ void xmatmul(const double* a, const double* b, double* c) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double acc = xadd(0.0, xmul(a[3 * i], b[j]));
            acc = xadd(acc, xmul(a[3 * i + 1], b[3 + j]));
            acc = xadd(acc, xmul(a[3 * i + 2], b[6 + j]));
            c[3 * i + j] = acc;
        }
}

// a0 b0 + a1 b1 + a2 b2, left to right (Eigen-shim dot: acc starts at 0.0)
__device__ __forceinline__ double xdot(const double* a, const double* b) {
    double acc = xadd(0.0, xmul(a[0], b[0]));
    acc = xadd(acc, xmul(a[1], b[1]));
    return xadd(acc, xmul(a[2], b[2]));
}

// view_transform (scene.cpp:5-17) of one kernel, in Eigen's evaluation order:
// M' = R M + T ; S' = (R S) R^T.
__device__ __forceinline__ void view_transform_one(const CameraP& c, const double* mo, const double* so, double* m,
                                                   double* s) {
    xmatvec(c.R, mo, m);
#pragma unroll
    for (int i = 0; i < 3; ++i) m[i] = xadd(m[i], c.T[i]);
    double rt[9], rs[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) rt[3 * j + i] = c.R[3 * i + j];
    xmatmul(c.R, so, rs);
    xmatmul(rs, rt, s);
}

// pixel_ray (scene.cpp:19-22): normalize(((i - Oy)/F, (j - Ox)/F, 1))
__device__ __forceinline__ void pixel_ray(const CameraP& c, int row, int col, double* d) {
    d[0] = xdiv(xsub((double)row, c.oy), c.focal);
    d[1] = xdiv(xsub((double)col, c.ox), c.focal);
    d[2] = 1.0;
    const double n = xadd(xadd(xadd(0.0, xmul(d[0], d[0])), xmul(d[1], d[1])), xmul(d[2], d[2]));
    if (n > 0.0) {
        const double s = __dsqrt_rn(n);
        d[0] = xdiv(d[0], s);
        d[1] = xdiv(d[1], s);
        d[2] = xdiv(d[2], s);
    }
}

struct Traced64 {
    double l, q, a;
};

// Per selected entry, taped by the selection for the blend, the backward and
// the sampler: l (FP64), e^q and 1/sigma (FP32, as blended). 16 bytes.
struct __align__(16) EntryRec {
    double l;
    float pk, is;
};

// trace_kernel (tracer.cpp:20-35), bit-exact: a = d.Sd, b = (m.Sd + d.Sm)/2,
// l = b/a, v = m - l d, q = min(0, -v.Sv/2), sigma = 1/sqrt(a).
__device__ __forceinline__ Traced64 trace_exact(const double* d, const Rec64& r) {
    double sd[3], v[3], sv[3];
    xmatvec(r.s, d, sd);
    const double a = xdot(d, sd);
    const double b = xmul(0.5, xadd(xdot(r.m, sd), xdot(d, r.sm)));
    const double l = xdiv(b, a);
#pragma unroll
    for (int i = 0; i < 3; ++i) v[i] = xsub(r.m[i], xmul(l, d[i]));
    xmatvec(r.s, v, sv);
    double q = xmul(-0.5, xdot(v, sv));
    if (q > 0.0) q = 0.0;
    return Traced64{l, q, a};
}

__device__ __forceinline__ double sigma_of(double a) { return xdiv(1.0, __dsqrt_rn(a)); }

// The same trace with contracted FMAs (same formulas as the reference: a = d.Sd,
// b = (m.Sd + d.Sm) / 2 with the full S, so asymmetric S within the validation
// tolerance is treated like the reference does): ~1e-15 relative of trace_exact
// (q: ~1e-13, cancellation in v). Used where values feed tolerance-checked
// arithmetic (blend, backward), never decisions.
__device__ __forceinline__ Traced64 trace_fast(const double* d, const Rec64& r) {
    const double* s = r.s;
    const double sd0 = fma(s[0], d[0], fma(s[1], d[1], s[2] * d[2]));
    const double sd1 = fma(s[3], d[0], fma(s[4], d[1], s[5] * d[2]));
    const double sd2 = fma(s[6], d[0], fma(s[7], d[1], s[8] * d[2]));
    const double a = fma(d[0], sd0, fma(d[1], sd1, d[2] * sd2));
    const double b = 0.5 * (fma(r.m[0], sd0, fma(r.m[1], sd1, r.m[2] * sd2)) +
                            fma(d[0], r.sm[0], fma(d[1], r.sm[1], d[2] * r.sm[2])));
    const double l = b / a;
    const double v0 = fma(-l, d[0], r.m[0]), v1 = fma(-l, d[1], r.m[1]), v2 = fma(-l, d[2], r.m[2]);
    const double sv0 = fma(s[0], v0, fma(s[1], v1, s[2] * v2));
    const double sv1 = fma(s[3], v0, fma(s[4], v1, s[5] * v2));
    const double sv2 = fma(s[6], v0, fma(s[7], v1, s[8] * v2));
    double q = -0.5 * fma(v0, sv0, fma(v1, sv1, v2 * sv2));
    if (q > 0.0) q = 0.0;
    return Traced64{l, q, a};
}

// ---------------------------------------------------------------- FP32 closed-form pieces

// Phi(x) = 0.5 erfc(-x / sqrt 2)  (blender.cpp:13-15)
__device__ __forceinline__ float normal_cdf_f(float x) { return 0.5f * erfcf(-x * 0.70710678118654752f); }
// phi(x) = exp(-x^2/2) / sqrt(2 pi)  (grad.cpp:16)
__device__ __forceinline__ float normal_pdf_f(float x) { return 0.398942280401432678f * expf(-0.5f * x * x); }

// Branch-free Phi for the forward blend: erfc(x) = t exp(-x^2 + P(t)),
// t = 1 / (1 + x/2) (Chebyshev-fitted erfc, fractional error < 1.2e-7 for all
// x >= 0), so |Phi - Phi_exact| < 6e-8 absolute: one reciprocal, one exp2, 10 FMA.
// The SFU instructions without the denormal-range fix-ups of exp2f / __fdividef
// (equal results outside that range: the reciprocal's argument is >= 1 here,
// and exp2 results below 2^-126 flush to zero).
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float fast_normal_cdf(float z) {
    const float x = fabsf(z) * 0.70710678118654752f;
    const float t = rcp_ftz(fmaf(0.5f, x, 1.0f));
    float p = 0.17087277f;
    p = fmaf(p, t, -0.82215223f);
    p = fmaf(p, t, 1.48851587f);
    p = fmaf(p, t, -1.13520398f);
    p = fmaf(p, t, 0.27886807f);
    p = fmaf(p, t, -0.18628806f);
    p = fmaf(p, t, 0.09678418f);
    p = fmaf(p, t, 0.37409196f);
    p = fmaf(p, t, 1.00002368f);
    p = fmaf(p, t, -1.26551223f);
    const float e = ex2_ftz(fmaf(-x, x, p) * 1.4426950408889634f);
    const float half_erfc = 0.5f * t * e;
    return z >= 0.0f ? 1.0f - half_erfc : half_erfc;
}

// phi(z) with the hardware exp2 (relative error ~2^-22 + |z^2/2| 2^-24).
__device__ __forceinline__ float normal_pdf_fast(float z) {
    return 0.398942280401432678f * ex2_ftz(-0.72134752044448170f * z * z);
}

// Order-preserving float <-> uint32 map (sort keys of the depth bound).
__device__ __forceinline__ uint32_t float_order_bits(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float float_from_order_bits(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// (l, idx) lexicographic order of fine_select (tracer.cpp:119-122)
__device__ __forceinline__ bool traced_less(double la, int ia, double lb, int ib) {
    return la < lb || (la == lb && ia < ib);
}

}  // namespace gvrk
