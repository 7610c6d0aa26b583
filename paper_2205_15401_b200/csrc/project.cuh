// K0 scene validation and K1 per-kernel projection / culling.
#pragma once

#include "gvr_common.cuh"

#include <float.h>
#include <limits.h>

namespace gvrk {

// Smallest eigenvalue of the symmetric matrix read from the lower triangle
// (Eigen's SelfAdjointEigenSolver reads the lower triangle), cyclic Jacobi —
// same iteration as the oracle so boundary decisions agree.
__device__ inline double min_eigenvalue_lower(const double* m) {
    double a[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) a[3 * i + j] = i >= j ? m[3 * i + j] : m[3 * j + i];
    for (int sweep = 0; sweep < 100; ++sweep) {
        const double off = a[1] * a[1] + a[2] * a[2] + a[5] * a[5];
        if (off <= DBL_MIN) break;
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int q = p + 1; q < 3; ++q) {
                const double apq = a[3 * p + q];
                if (apq == 0.0) continue;
                const double theta = (a[3 * q + q] - a[3 * p + p]) / (2 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1));
                const double c = 1 / sqrt(t * t + 1), s = t * c;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const double akp = a[3 * k + p], akq = a[3 * k + q];
                    a[3 * k + p] = c * akp - s * akq;
                    a[3 * k + q] = s * akp + c * akq;
                }
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const double apk = a[3 * p + k], aqk = a[3 * q + k];
                    a[3 * p + k] = c * apk - s * aqk;
                    a[3 * q + k] = s * apk + c * aqk;
                }
            }
    }
    return fmin(a[0], fmin(a[4], a[8]));
}

// K0: GaussianKernel::validate (types.cpp:17-29) for every kernel; the first
// failing kernel (lowest index) wins, encoded as (k << 2) | code with
// code 1 = non-finite, 2 = not symmetric, 3 = not positive-definite.
__global__ void validate_scene_kernel(int K, int D, const double* __restrict__ centers,
                                      const double* __restrict__ inv_cov, const double* __restrict__ attr,
                                      unsigned long long* __restrict__ first_error) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    double s[9];
    bool finite = true;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        s[i] = inv_cov[9ll * k + i];
        finite &= isfinite(s[i]);
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) finite &= isfinite(centers[3ll * k + i]);
    for (int c = 0; c < D; ++c) finite &= isfinite(attr[(long long)D * k + c]);
    unsigned code = 0;
    if (!finite) {
        code = 1;
    } else {
        double scale = 0.0, asym = 0.0;
#pragma unroll
        for (int i = 0; i < 9; ++i) scale = fmax(scale, fabs(s[i]));
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) asym = fmax(asym, fabs(s[3 * i + j] - s[3 * j + i]));
        if (scale != 0.0 && !(asym <= 1e-6 * scale)) {
            code = 2;
        } else if (min_eigenvalue_lower(s) <= 0.0) {
            code = 3;
        }
    }
    if (code) atomicMin(first_error, ((unsigned long long)k << 2) | code);
}

// 3x3 inverse by cofactors, exact emulation of the oracle / Eigen-shim order.
__device__ __forceinline__ void xinverse3(const double* m, double* inv) {
#define M(i, j) m[3 * (i) + (j)]
    const double c00 = xsub(xmul(M(1, 1), M(2, 2)), xmul(M(1, 2), M(2, 1)));
    const double c10 = xsub(xmul(M(1, 2), M(2, 0)), xmul(M(1, 0), M(2, 2)));
    const double c20 = xsub(xmul(M(1, 0), M(2, 1)), xmul(M(1, 1), M(2, 0)));
    const double det = xadd(xadd(xmul(M(0, 0), c00), xmul(M(0, 1), c10)), xmul(M(0, 2), c20));
    const double id = xdiv(1.0, det);
    inv[0] = xmul(c00, id);
    inv[3] = xmul(c10, id);
    inv[6] = xmul(c20, id);
    inv[1] = xmul(xsub(xmul(M(0, 2), M(2, 1)), xmul(M(0, 1), M(2, 2))), id);
    inv[4] = xmul(xsub(xmul(M(0, 0), M(2, 2)), xmul(M(0, 2), M(2, 0))), id);
    inv[7] = xmul(xsub(xmul(M(0, 1), M(2, 0)), xmul(M(0, 0), M(2, 1))), id);
    inv[2] = xmul(xsub(xmul(M(0, 1), M(1, 2)), xmul(M(0, 2), M(1, 1))), id);
    inv[5] = xmul(xsub(xmul(M(0, 2), M(1, 0)), xmul(M(0, 0), M(1, 2))), id);
    inv[8] = xmul(xsub(xmul(M(0, 0), M(1, 1)), xmul(M(0, 1), M(1, 0))), id);
#undef M
}

// static_cast<int>(double) as compiled for x86-64 (cvttsd2si): out-of-range and
// NaN give INT_MIN; the reference's box clamps depend on it for extreme boxes.
__device__ __forceinline__ int x86_int(double v) {
    if (!(v > -2147483649.0 && v < 2147483648.0)) return INT_MIN;
    return (int)v;
}


// Tile rectangle of the pixel centres inside a kernel's screen box.
__device__ __forceinline__ bool box_tiles(const Rec32& q, int H, int W, int tile, int& tr0, int& tr1, int& tc0,
                                          int& tc1) {
    const float r0 = fmaxf(0.0f, ceilf(q.top)), r1 = fminf((float)(H - 1), floorf(q.bottom));
    const float c0 = fmaxf(0.0f, ceilf(q.left)), c1 = fminf((float)(W - 1), floorf(q.right));
    if (!(r0 <= r1 && c0 <= c1)) return false;
    tr0 = (int)r0 / tile;
    tr1 = (int)r1 / tile;
    tc0 = (int)c0 / tile;
    tc1 = (int)c1 / tile;
    return true;
}

struct ProjectParams {
    int K;
    const double* centers;  // object space [K*3]
    const double* inv_cov;  // object space [K*9]
    CameraP cam;
    SelP sel;
    int tile;           // pixels per tile edge
    int tiles_x, tiles_y;
    Rec32* rec32;
    Rec64* rec64;
    int* tile_count;  // [tiles] list lengths (zeroed before the launch)
    int shard, nshards;  // only tiles t with t % nshards == shard are binned (C4 tile sharding)
    int* dropped_behind;
    // backward bookkeeping: one 64-bit pixel mask per (kernel, tile of its box rectangle)
    int4* kinfo;                 // [K] {mask base (-1: no room), tr0 << 16 | tc0, tiles per row, tiles}
    unsigned long long* masks;   // [mask_cap], zeroed here for every allocated rectangle
    int* mask_total;             // rectangle tiles requested (bump allocator, zeroed before the launch)
    int4* ref_box;               // nullable: the reference's pushed pixel box {row_lo, row_hi, col_lo, col_hi}
                                 // (tracer.cpp:100-103), {1, 0, 1, 0} when not pushed (coarse_select API)
    int mask_cap;
};

// K1: view transform (scene.cpp:5-17), coarse screen box (tracer.cpp:37-113) in
// exact FP64, the FP32 pre-filter record and the depth key for early exit.
struct BinJob {
    int nt = 0;  // tiles to append to (row-major rectangle from (tr0, tc0), ntc per row)
    int tr0 = 0, tc0 = 0, ntc = 1;
    unsigned long long key = 0;
};

// Tile rectangle of kernel k's box as a binning job (emit pass: from its record).
__device__ __forceinline__ BinJob job_from_record(const Rec32& q, int k, int H, int W, int tile) {
    BinJob job;
    int tr0, tr1, tc0, tc1;
    if (box_tiles(q, H, W, tile, tr0, tr1, tc0, tc1)) {
        job.key = ((unsigned long long)float_order_bits(q.zmin) << 32) | (unsigned)k;
        job.tr0 = tr0;
        job.tc0 = tc0;
        job.ntc = tc1 - tc0 + 1;
        job.nt = (tr1 - tr0 + 1) * job.ntc;
    }
    return job;
}

__device__ __forceinline__ BinJob project_one(const ProjectParams& p, int k) {
    BinJob job;
    const CameraP& c = p.cam;

    double mo[3], so[9];
#pragma unroll
    for (int i = 0; i < 3; ++i) mo[i] = p.centers[3ll * k + i];
#pragma unroll
    for (int i = 0; i < 9; ++i) so[i] = p.inv_cov[9ll * k + i];

    Rec64 r;
    view_transform_one(c, mo, so, r.m, r.s);
    xmatvec(r.s, r.m, r.sm);
    r.pad = 0.0;
    p.rec64[k] = r;

    const double f = c.focal;
    const double z = r.m[2];
    Rec32 q;
    // quadratic forms (and so l and q) depend only on the symmetric part of S'
    q.s00 = (float)r.s[0];
    q.s01 = (float)(0.5 * (r.s[1] + r.s[3]));
    q.s02 = (float)(0.5 * (r.s[2] + r.s[6]));
    q.s11 = (float)r.s[4];
    q.s12 = (float)(0.5 * (r.s[5] + r.s[7]));
    q.s22 = (float)r.s[8];
    q.top = q.left = 1.0f;
    q.bottom = q.right = 0.0f;  // empty box
    q.zmin = -FLT_MAX;

    if (p.ref_box) p.ref_box[k] = make_int4(1, 0, 1, 0);
    if (z <= kBehindCameraEps) {
        // behind the camera: dropped (tracer.cpp:52-56, blender.cpp:86)
        atomicAdd(p.dropped_behind, 1);
        q.z = -1.0f;
        q.ci_int = q.cj_int = 0;
        q.ci_frac = q.cj_frac = 0.0f;
        p.rec32[k] = q;
        return job;
    }

    double cov[9];
    xinverse3(r.s, cov);
    const double chi = p.sel.chi;
    const double ci = xadd(c.oy, xdiv(xmul(f, r.m[0]), z));
    const double cj = xadd(c.ox, xdiv(xmul(f, r.m[1]), z));
    const double ext[3] = {__dsqrt_rn(fmax(0.0, xmul(chi, cov[0]))), __dsqrt_rn(fmax(0.0, xmul(chi, cov[4]))),
                           __dsqrt_rn(fmax(0.0, xmul(chi, cov[8])))};
    const double zmin = xsub(z, ext[2]);
    const bool straddles = zmin <= kBehindCameraEps;

    // Depth key: every selected kernel has l >= z - ext_z (its peak lies inside
    // the eta-ellipsoid, whose camera-space z-extent is +-ext_z); conservative
    // rounding keeps the bound strict under FP64/FP32 rounding.
    if (zmin > 0.0) q.zmin = __double2float_rd(zmin - 1e-12 * zmin);

    // Centre-relative FP32 pre-filter data; unusual geometry (near-plane
    // straddlers, far off-axis centres) bypasses the pre-filter (z < 0).
    q.z = (float)z;
    if (straddles || fabs(ci) > 1e7 || fabs(cj) > 1e7) {
        q.z = -1.0f;
        q.ci_int = q.cj_int = 0;
        q.ci_frac = q.cj_frac = 0.0f;
    } else {
        const double fi = floor(ci), fj = floor(cj);
        q.ci_int = (int)fi;
        q.cj_int = (int)fj;
        q.ci_frac = (float)(ci - fi);
        q.cj_frac = (float)(cj - fj);
    }

    // Screen box of the eta-level set exactly as coarse_select computes it
    // (tracer.cpp:61-98): the linearised ellipse box widened by the projected
    // corners of the camera-space AABB, full screen when that AABB reaches the
    // near plane. jac = [[f/z, 0, -f x/z^2], [0, f/z, -f y/z^2]], cov2 = jac cov jac^T.
    const double zz = xmul(z, z);
    const double jac[6] = {xdiv(f, z), 0.0, xdiv(xmul(-f, r.m[0]), zz), 0.0, xdiv(f, z), xdiv(xmul(-f, r.m[1]), zz)};
    double jc[6];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double acc = xadd(0.0, xmul(jac[3 * i], cov[j]));
            acc = xadd(acc, xmul(jac[3 * i + 1], cov[3 + j]));
            jc[3 * i + j] = xadd(acc, xmul(jac[3 * i + 2], cov[6 + j]));
        }
    double cov2[4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            double acc = xadd(0.0, xmul(jc[3 * i], jac[3 * j]));
            acc = xadd(acc, xmul(jc[3 * i + 1], jac[3 * j + 1]));
            cov2[2 * i + j] = xadd(acc, xmul(jc[3 * i + 2], jac[3 * j + 2]));
        }
    const double rh = __dsqrt_rn(fmax(0.0, xmul(chi, cov2[0])));
    const double rw = __dsqrt_rn(fmax(0.0, xmul(chi, cov2[3])));
    double top = xsub(ci, rh), bottom = xadd(ci, rh), left = xsub(cj, rw), right = xadd(cj, rw);
    if (straddles) {
        top = 0;
        bottom = c.H - 1;
        left = 0;
        right = c.W - 1;
    } else {
#pragma unroll
        for (int corner = 0; corner < 8; ++corner) {
            const double px = xadd(r.m[0], (corner & 1) ? ext[0] : -ext[0]);
            const double py = xadd(r.m[1], (corner & 2) ? ext[1] : -ext[1]);
            const double pz = xadd(r.m[2], (corner & 4) ? ext[2] : -ext[2]);
            const double pi = xadd(c.oy, xdiv(xmul(f, px), pz));
            const double pj = xadd(c.ox, xdiv(xmul(f, py), pz));
            top = pi < top ? pi : top;
            bottom = pi > bottom ? pi : bottom;
            left = pj < left ? pj : left;
            right = pj > right ? pj : right;
        }
    }
    bool candidate = true;
    if (p.sel.coarse) {
        // pushed into the coarse map at all? (tracer.cpp:100-104, reference int semantics)
        const int lo_r = max(0, x86_int(floor(xsub(top, 1.0))));
        const int hi_r = min(c.H - 1, x86_int(ceil(xadd(bottom, 1.0))));
        const int lo_c = max(0, x86_int(floor(xsub(left, 1.0))));
        const int hi_c = min(c.W - 1, x86_int(ceil(xadd(right, 1.0))));
        candidate = lo_r <= hi_r && lo_c <= hi_c;
        if (p.ref_box && candidate) p.ref_box[k] = make_int4(lo_r, hi_r, lo_c, hi_c);
    }
    // Every pushed kernel is in the candidate list of every pixel of its padded
    // box; among those it can only pass the eta test where the pixel centre lies
    // in the unpadded box (the ray must cross the eta-ellipsoid, whose
    // projection the box contains). So binning and testing by the unpadded box
    // reproduces the reference's selection exactly, with far fewer traces.
    if (candidate) {
        const double mt = 1e-6 * (1.0 + fabs(top)), mb = 1e-6 * (1.0 + fabs(bottom));
        const double ml = 1e-6 * (1.0 + fabs(left)), mr = 1e-6 * (1.0 + fabs(right));
        q.top = __double2float_rd(fmax(top - mt, -1.0e30));
        q.bottom = __double2float_ru(fmin(bottom + mb, 1.0e30));
        q.left = __double2float_rd(fmax(left - ml, -1.0e30));
        q.right = __double2float_ru(fmin(right + mr, 1.0e30));
        job = job_from_record(q, k, c.H, c.W, p.tile);  // the emit pass recomputes the same rectangle
    }
    p.rec32[k] = q;
    return job;
}

// K1. Projection + binning count pass: every kernel adds one to the counter of
// every tile (of this shard) its box overlaps. The adds are warp-aggregated:
// lanes that hit the same tile in the same round (neighbouring kernels usually
// do) share one reduction on the tile's counter. The counts size the tile lists
// (exclusive scan in order_tiles_kernel), which emit_kernel then fills.
__global__ void project_kernel(ProjectParams p) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    BinJob job;
    if (k < p.K) job = project_one(p, k);
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    {
        // mask rectangle of the kernel (deterministic backward): one warp-aggregated
        // bump allocation, then the kernel zeroes its own masks
        int incl = job.nt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        int base = 0;
        if (lane == 31 && incl > 0) base = atomicAdd(p.mask_total, incl);
        base = __shfl_sync(FULL, base, 31) + incl - job.nt;
        if (k < p.K) {
            const bool fits = base >= 0 && (long long)base + job.nt <= (long long)p.mask_cap;
            p.kinfo[k] = make_int4(job.nt > 0 && fits ? base : -1, (job.tr0 << 16) | job.tc0, job.ntc, job.nt);
            if (fits)
                for (int t = 0; t < job.nt; ++t) p.masks[base + t] = 0ull;
        }
    }
    for (int it0 = 0; __any_sync(FULL, it0 < job.nt); it0 += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int it = it0 + u;
            int t = it < job.nt ? (job.tr0 + it / job.ntc) * p.tiles_x + job.tc0 + it % job.ntc : -1;
            if (t >= 0 && t % p.nshards != p.shard) t = -1;
            const unsigned mk = __match_any_sync(FULL, t);
            if (t >= 0 && (mk & lt) == 0) atomicAdd(p.tile_count + t, __popc(mk));
        }
    }
}

// Zero up to 8 arrays of 32-bit words in one launch (the render's per-call
// counters and flags, and the outputs of the tiles the blend does not visit).
struct ClearList {
    int* ptr[8];
    long long n[8];  // words
    int m;
};
__global__ void clear_kernel(ClearList c) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (int a = 0; a < c.m; ++a) {
        for (; i < c.n[a]; i += stride) c.ptr[a][i] = 0;
        i -= c.n[a];
    }
}

struct EmitParams {
    int K;
    const Rec32* rec32;
    int H, W, tile, tiles_x;
    const int* tile_off;        // [tiles] list offsets in the pool; -1: not listed (other shard / overflow)
    int* tile_fill;             // [tiles] append cursors (zeroed before the launch)
    unsigned long long* pool;   // tile lists, (order(zmin) << 32 | id), unsorted within a list
};

// K2. Binning emit pass: appends (depth key, id) to the list of every tile the
// kernel's box overlaps (same rectangle as the count pass, recomputed from the
// record), warp-aggregated returned atomics, four rounds in flight.
__global__ void emit_kernel(EmitParams p) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    BinJob job;
    if (k < p.K) job = job_from_record(p.rec32[k], k, p.H, p.W, p.tile);
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    for (int it0 = 0; __any_sync(FULL, it0 < job.nt); it0 += 4) {
        int t[4], off[4], base[4];
        unsigned mk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int it = it0 + u;
            t[u] = it < job.nt ? (job.tr0 + it / job.ntc) * p.tiles_x + job.tc0 + it % job.ntc : -1;
            off[u] = t[u] >= 0 ? p.tile_off[t[u]] : -1;
            if (off[u] < 0) t[u] = -1;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) mk[u] = __match_any_sync(FULL, t[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            base[u] = 0;
            if (t[u] >= 0 && (mk[u] & lt) == 0) base[u] = atomicAdd(p.tile_fill + t[u], __popc(mk[u]));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int pos = __shfl_sync(FULL, base[u], __ffs(mk[u]) - 1) + __popc(mk[u] & lt);
            if (t[u] >= 0) p.pool[(size_t)off[u] + pos] = job.key;
        }
    }
}


}  // namespace gvrk
