// K4 per-pixel backward and K5 per-kernel object-space chain.
#pragma once

#include "gvr_common.cuh"

namespace gvrk {

struct BwdParams {
    CameraP cam;
    int kp, D, Dc;
    double tau;
    int through_t, through_rho;
    int tiles_x;
    const int* tile_order;  // tiles by descending sum_p n_p^2 (LPT); first *n_order valid
    const int* n_order;
    const int* topk;   // [P*kp]
    const int* count;  // [P]
    const double* tape_t;  // [P*kp] T(l_k) from the forward
    const EntryRec* ent;   // [P*kp] traced entries (l, e^q, 1/sigma) from the forward
    const double* ent_a;   // [P*kp] a = d.Sd of the traced entries (FP64)
    const Rec64* rec64;
    const double* attr;     // [K*D]
    const double* d_image;  // [P*D]
    const double* d_alpha;  // [P]
    const int4* kinfo;           // [K] mask rectangle of each kernel (project_kernel)
    const unsigned long long* masks;  // per (kernel, tile): pixels of the tile that selected the kernel
    const int* slot_off;              // per (kernel, tile): first record of its pixels (appearance_kernel)
    double4* bent;                    // records {alpha, d_q, beta, W} (entry_coeffs)
    int2* bkey;                       // records' {pixel, kernel}
    double4* rays;                    // [P] the pixel's ray (pixel_ray), for the record pass
    // fallback for kernels without a mask rectangle (mask pool full): FP64 atomics
    double* acc;            // [K*9] camera space: dm(3), dS upper (00 01 02 11 12 22)
    double* attr_fb;        // [K*D]
};

// Chain of one selected entry to camera space (grad.cpp:150-170): with a = d.Sd,
// l = d.Sm / a, v = m - l d, sigma = a^-1/2:
//   dm = (d_l / a) S d - d_q S v
//   dS = (d_l / a)(0.5 (m d^T + d m^T) - l d d^T) - 0.5 d_q v v^T - 0.5 sigma^3 d_sigma d d^T
// dS as its upper triangle (00 01 02 11 12 22).
__device__ __forceinline__ void chain_entry(const Rec64& r, const double* d, double dl, double dq, double dsg,
                                            double* dm, double* ds) {
    double sd[3], v[3], sv[3];
    const double s00 = r.s[0], s01 = r.s[1], s02 = r.s[2], s11 = r.s[4], s12 = r.s[5], s22 = r.s[8];
    sd[0] = fma(s00, d[0], fma(s01, d[1], s02 * d[2]));
    sd[1] = fma(s01, d[0], fma(s11, d[1], s12 * d[2]));
    sd[2] = fma(s02, d[0], fma(s12, d[1], s22 * d[2]));
    const double a = fma(d[0], sd[0], fma(d[1], sd[1], d[2] * sd[2]));
    const double ia = 1.0 / a;
    const double l = fma(d[0], r.sm[0], fma(d[1], r.sm[1], d[2] * r.sm[2])) * ia;
#pragma unroll
    for (int t = 0; t < 3; ++t) v[t] = fma(-l, d[t], r.m[t]);
    sv[0] = fma(s00, v[0], fma(s01, v[1], s02 * v[2]));
    sv[1] = fma(s01, v[0], fma(s11, v[1], s12 * v[2]));
    sv[2] = fma(s02, v[0], fma(s12, v[1], s22 * v[2]));
    const double scale = dl * ia;
    const double d_a = -0.5 * ia * sqrt(ia) * dsg;  // -0.5 sigma^3 d_sigma, sigma = a^-1/2
#pragma unroll
    for (int t = 0; t < 3; ++t) dm[t] = scale * sd[t] - dq * sv[t];
    const int rr[6] = {0, 0, 0, 1, 1, 2};
    const int cc[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int t = 0; t < 6; ++t) {
        const int a0 = rr[t], a1 = cc[t];
        const double ddt = d[a0] * d[a1];
        ds[t] = scale * (0.5 * (r.m[a0] * d[a1] + d[a0] * r.m[a1]) - l * ddt) - 0.5 * dq * (v[a0] * v[a1]) + d_a * ddt;
    }
}

// The chain of grad.cpp:140-170 regrouped so that the kernel's camera-space
// centre m and inverse covariance S enter only through per-kernel sums: with
// s = d_l / a, v = m - l d and d_a = -0.5 sigma^3 d_sigma,
//   dm = S (s d - d_q v)                  = S (alpha d - d_q m)
//   dS = s sym(v d^T) - d_q/2 v v^T + d_a d d^T
//      = alpha sym(m d^T) + beta d d^T - d_q/2 m m^T,
//   alpha = s + d_q l,   beta = -s l - d_q l^2 / 2 + d_a,
// so a kernel needs A = sum alpha d, Q = sum d_q, B = sum beta d d^T over its
// entries (finish_kernel then applies m and S once). Every entry input is the
// traced (l, a) of the forward and the pixel's ray; the sums cancel at most
// (|m| / sigma)^2 in FP64.
__device__ __forceinline__ void entry_coeffs(double l, double a, double dl, double dq, double dsg, double* alpha,
                                             double* beta) {
    const double ia = 1.0 / a;
    const double sc = dl * ia;
    const double d_a = -0.5 * ia * sqrt(ia) * dsg;  // -0.5 sigma^3 d_sigma, sigma = a^-1/2
    *alpha = fma(dq, l, sc);
    *beta = fma(-0.5 * dq * l, l, fma(-sc, l, d_a));
}

// Entry of a kernel without a mask rectangle (the mask pool was full): FP64
// atomics into camera-space accumulators, consumed by the gather (rare; kept
// out of line so it costs the hot loop no registers).
__device__ __noinline__ void backward_fallback(const Rec64* rec, double* acc, double* attr_fb, const double* dimg, int D,
                                               const double* d, double dl, double dq, double dsg, double w);

// Per pixel (grad.cpp:75-174). CTA = one 8x8 tile, 4 threads per pixel (256
// threads): the pixel's entries are split 4 ways in every pass, which cuts the
// per-pixel serial chain (the latency limit of this kernel) by 4x.
// T(l_k) comes from the forward's tape, so only the pair terms are O(n^2).
// They are evaluated "entry-major": for entry e every contribution to
// d_peak_e, d_l_e and d_sigma_e is gathered in FP64 registers (the reference
// scatters them pair by pair; the sums are the same), so there are no
// per-entry accumulator arrays. Phi / phi are FP32 (~1e-7) from an
// FP64-accurate argument; products and sums are FP64 (the gradient bar is
// 1e-4 of a class-scaled floor, ~1e-7 of the largest gradient).
template <int KMAX>
__global__ void __launch_bounds__(256 / GVR_BWD_SPLIT, GVR_BWD_MINB) backward_pixels_kernel(BwdParams p) {
    constexpr int TILE = 8, NP = 64 / GVR_BWD_SPLIT, PER = (KMAX + 3) / 4;
    extern __shared__ __align__(16) unsigned char smem[];
    // per-entry staging, [slot][pixel]
    // pairs read together are packed: one 16-byte and one 8-byte load per pair
    // {hi, lo of l_k - l_0, d_acc_k = -tau T_k d_w_k e^{q_k}, e^{q_k}} as floats, 1 / sigma_k
    float4* b_q = reinterpret_cast<float4*>(smem);
    double* b_dt = reinterpret_cast<double*>(b_q + KMAX * NP);  // density path d_w_k T_k (grad.cpp:120)
    float* b_is = reinterpret_cast<float*>(b_dt + KMAX * NP);
    int* b_id = reinterpret_cast<int*>(b_is + KMAX * NP);

    if ((int)(blockIdx.x / GVR_BWD_SPLIT) >= *p.n_order) return;
    const int g = threadIdx.x >> 2, sub = threadIdx.x & 3;
    const int tile = p.tile_order[blockIdx.x / GVR_BWD_SPLIT];
    const int gp = (blockIdx.x % GVR_BWD_SPLIT) * NP + g;  // pixel within the tile
    const int i = (tile / p.tiles_x) * TILE + gp / TILE;
    const int j = (tile % p.tiles_x) * TILE + gp % TILE;
    if (i >= p.cam.H || j >= p.cam.W) return;
    const long long pix = (long long)i * p.cam.W + j;
    const int n = p.count[pix];
    if (n == 0) return;  // the pixel's 4 threads leave together
    const unsigned grp = 0xfu << (threadIdx.x & 28);

    double d[3];
    pixel_ray(p.cam, i, j, d);
    if (sub == 0) p.rays[pix] = make_double4(d[0], d[1], d[2], 0.0);
    const double tau = p.tau;
    // d_image of the pixel in registers for D <= 4 (unrolled with constant
    // indices: a runtime-indexed array would live in local memory)
    double dimg[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 4; ++c)
        if (c < p.D) dimg[c] = p.d_image[pix * p.D + c];
    const double l0 = p.ent[pix * p.kp].l;

    // re-trace the taped selection in exact FP64 (bit-identical to the forward),
    // d_weight, attribute gradient, d_acc (grad.cpp:79-120)
    double peak_part = 0.0;
    // ids first: the thread's id loads are independent, the record loads behind them overlap
    int kq[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) kq[q] = sub + 4 * q < n ? p.topk[pix * p.kp + sub + 4 * q] : 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int s = sub + 4 * q;
        if (s >= n) break;
        const int k = kq[q];
        const EntryRec er = p.ent[pix * p.kp + s];  // traced by the forward
        const float pkf = er.pk;
        const double pk = (double)pkf;
        peak_part += pk;
        const double trans = p.tape_t[pix * p.kp + s];
        double dw = 0.0;
        if (p.D <= 4) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (c < p.D) dw += dimg[c] * p.attr[(long long)p.D * k + c];
        } else {
            for (int c = 0; c < p.D; ++c) dw += p.d_image[pix * p.D + c] * p.attr[(long long)p.D * k + c];
        }
        const double dacc = (p.through_t && dw != 0.0) ? -tau * trans * (dw * pk) : 0.0;
        const double dl0 = er.l - l0;
        const float hi = (float)dl0;
        b_q[s * NP + g] = make_float4(hi, (float)(dl0 - (double)hi), (float)dacc, pkf);
        b_is[s * NP + g] = er.is;
        b_dt[s * NP + g] = (p.through_rho && dw != 0.0) ? dw * trans : 0.0;
        b_id[s * NP + g] = k;
    }
    peak_part += __shfl_xor_sync(grp, peak_part, 1, 4);
    peak_part += __shfl_xor_sync(grp, peak_part, 2, 4);
    __syncwarp(grp);
    const double galpha = p.d_alpha[pix];
    const double d_total = (p.through_t && galpha != 0.0) ? galpha * tau * exp(-tau * peak_part) : 0.0;

    // entry-major pair terms + chain to camera space (grad.cpp:121-173)
    for (int e = sub; e < n; e += 4) {
        // FP32 pair terms with Kahan-compensated FP32 sums: no FP64 conversions
        // in the loop (those share the XU pipe with the exp2 / reciprocal)
        const float4 qe = b_q[e * NP + g];
        const float ise = b_is[e * NP + g];
        const float pkef = qe.w;
        const double pke = (double)pkef;
        const int kid = b_id[e * NP + g];
        double dpk = d_total + b_dt[e * NP + g];  // density path (grad.cpp:120)
        float s_pk = 0.0f, c_pk = 0.0f, s_l = 0.0f, c_l = 0.0f, s_sg = 0.0f, c_sg = 0.0f;
        auto kahan = [](float& sum, float& comp, float term) {
            const float y = term - comp;
            const float t = sum + y;
            comp = (t - sum) - y;
            sum = t;
        };
#pragma unroll 2
        for (int k = 0; k < n; ++k) {
            const float4 qk = b_q[k * NP + g];
            const float isk = b_is[k * NP + g];
            // pair (k, m = e): z1 = (l_k - l_e) / sigma_e ; pair (k = e, m = k): z2 = (l_e - l_k) / sigma_k
            const float dlf = (qk.x - qe.x) + (qk.y - qe.y);
            const float z1 = dlf * ise;
            const float phi1 = normal_pdf_fast(z1);
            const float phi2 = normal_pdf_fast(-dlf * isk);  // branch-free (equals phi1 when sigma_k == sigma_e)
            kahan(s_pk, c_pk, qk.z * fast_normal_cdf(z1));
            const float gg = k != e ? qk.z * (phi1 * ise) * pkef : 0.0f;
            kahan(s_sg, c_sg, -gg * z1);
            kahan(s_l, c_l, k != e ? fmaf(qe.z, qk.w * phi2 * isk, -gg) : 0.0f);
        }
        dpk += (double)s_pk - (double)c_pk;
        const double dl = (double)s_l - (double)c_l;
        const double dsg = (double)s_sg - (double)c_sg;
        const double dq = dpk * pke;
        const double w = p.tape_t[pix * p.kp + e] * pke;  // W_e (the forward's weight)
        // (programmatic dependent of offsets_kernel: the record offsets are complete from here)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const int4 ki = p.kinfo[kid];
        if (ki.x >= 0) {
            // deterministic path: the entry's adjoints go to its record in the
            // kernel's block: the slot's first record + the pixel's rank in the mask
            const int slot = ki.x + (i / TILE - (ki.y >> 16)) * ki.z + (j / TILE - (ki.y & 0xffff));
            const int bit = (i % TILE) * TILE + j % TILE;
            const int rec = p.slot_off[slot] + __popcll(p.masks[slot] & ((1ull << bit) - 1ull));
            double alpha, beta;
            entry_coeffs(p.ent[pix * p.kp + e].l, p.ent_a[pix * p.kp + e], dl, dq, dsg, &alpha, &beta);
            p.bent[rec] = make_double4(alpha, dq, beta, w);
            p.bkey[rec] = make_int2((int)pix, kid);
            continue;
        }
        backward_fallback(p.rec64 + kid, p.acc + 9ll * kid, p.attr_fb + (long long)p.D * kid,
                          p.d_image + pix * p.D, p.D, d, dl, dq, dsg, w);
    }
}

__device__ __noinline__ void backward_fallback(const Rec64* rec, double* acc, double* attr_fb, const double* dimg, int D,
                                               const double* d, double dl, double dq, double dsg, double w) {
    if (w != 0.0)
        for (int c = 0; c < D; ++c) atomicAdd(attr_fb + c, w * dimg[c]);
    if (dl == 0.0 && dq == 0.0 && dsg == 0.0) return;
    double dmv[3], dsv[6];
    chain_entry(*rec, d, dl, dq, dsg, dmv, dsv);
    for (int t = 0; t < 3; ++t) atomicAdd(acc + t, dmv[t]);
    for (int t = 0; t < 6; ++t) atomicAdd(acc + 3 + t, dsv[t]);
}

// Block-contiguous rows of `width` doubles staged through shared memory so the
// global side is coalesced 16-byte traffic (rows are 24 / 72 bytes apart).
__device__ __forceinline__ void stage_rows_in(double* dst, const double* __restrict__ src, int k0, int count,
                                              int width) {
    const long long n = (long long)count * width, off = (long long)k0 * width;
    if (((off & 1) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
        const double2* s2 = reinterpret_cast<const double2*>(src + off);
        for (long long i = threadIdx.x; i < n / 2; i += blockDim.x) reinterpret_cast<double2*>(dst)[i] = __ldg(s2 + i);
        if ((n & 1) && threadIdx.x == 0) dst[n - 1] = src[off + n - 1];
    } else {
        for (long long i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[off + i];
    }
}

__device__ __forceinline__ void stage_rows_out(double* __restrict__ dst, const double* src, int k0, int count,
                                               int width) {
    const long long n = (long long)count * width, off = (long long)k0 * width;
    if (((off & 1) == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        double2* d2 = reinterpret_cast<double2*>(dst + off);
        for (long long i = threadIdx.x; i < n / 2; i += blockDim.x) d2[i] = reinterpret_cast<const double2*>(src)[i];
        if ((n & 1) && threadIdx.x == 0) dst[off + n - 1] = src[n - 1];
    } else {
        for (long long i = threadIdx.x; i < n; i += blockDim.x) dst[off + i] = src[i];
    }
}

// ---------------------------------------------------------------- deterministic backward layout
// Kernel k's selected (pixel, entry) pairs are the set bits of its mask
// rectangle (set by the blend). Records are laid out in kernel order, and
// inside a kernel in (tile row-major, pixel) order: an exclusive scan of the
// per-kernel counts (K4a/b: counts + CTA sums, offsets), so
// the layout is a pure function of the selection.
constexpr int kScanThreads = 256;

struct AppParams {
    int K;
    const int4* kinfo;
    const unsigned long long* masks;
    int* count;      // [K] records of each kernel (count_kernel)
    int* cta_sum;    // [ceil(K / kScanThreads)] record totals of each count_kernel CTA
    int* slot_off;   // [mask slots] first record of each (kernel, tile)
    int2* app;       // [K] {first record, count}
    int* total;      // records of the render
};

__device__ __forceinline__ int block_exclusive_scan(int v, int* total) {
    __shared__ int s_warp[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        int w = lane < nw ? s_warp[lane] : 0, wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < nw) s_warp[lane] = wi - w;
        if (lane == nw - 1) s_warp[31] = wi;  // nw <= 31 for blocks <= 992 threads
    }
    __syncthreads();
    const int out = s_warp[warp] + incl - v;
    if (total) *total = s_warp[31];
    __syncthreads();
    return out;
}

__global__ void __launch_bounds__(kScanThreads) count_kernel(AppParams p) {
    const int k = blockIdx.x * kScanThreads + threadIdx.x;
    int c = 0;  // the kernel's selected pixels: the bits of its masks (set by the blend)
    if (k < p.K) {
        const int4 ki = p.kinfo[k];
        if (ki.x >= 0)
            for (int t = 0; t < ki.w; ++t) c += __popcll(p.masks[ki.x + t]);
        p.count[k] = c;
    }
    int tot;
    block_exclusive_scan(c, &tot);
    if (threadIdx.x == 0) p.cta_sum[blockIdx.x] = tot;
}

// Record offsets: this CTA's prefix = the sum of the earlier CTAs' totals (read
// and reduced by the CTA itself: no separate scan launch), then the exclusive
// scan of its kernels' counts. The last CTA writes the render's record total.
__global__ void __launch_bounds__(kScanThreads) offsets_kernel(AppParams p) {
    launch_dependents();  // K4 may start its pair terms while the offsets are written
    const int k = blockIdx.x * kScanThreads + threadIdx.x;
    const int c = k < p.K ? p.count[k] : 0;
    int before = 0;
    for (int b = threadIdx.x; b < (int)blockIdx.x; b += blockDim.x) before += p.cta_sum[b];
    int prefix;
    block_exclusive_scan(before, &prefix);  // (the block total of the partial sums)
    int tot;
    const int off = prefix + block_exclusive_scan(c, &tot);
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *p.total = prefix + tot;
    if (k >= p.K) return;
    p.app[k] = make_int2(off, c);
    if (c > 0) {
        const int4 ki = p.kinfo[k];
        int run = off;
        for (int t = 0; t < ki.w; ++t) {
            p.slot_off[ki.x + t] = run;
            run += __popcll(p.masks[ki.x + t]);
        }
    }
}

constexpr int kRecThreads = 128;
#ifndef GVR_REC_CTAS_PER_SM
#define GVR_REC_CTAS_PER_SM 8
#endif
constexpr int kRecCtasPerSm = GVR_REC_CTAS_PER_SM;  // records grid: CTAs per SM walking the windows (16: slower)

// K5a: one thread per record (grid-stride over 32-record windows, one warp per
// window): the entry's terms of the regrouped chain (entry_coeffs: alpha d,
// d_q, beta d d^T) and its attribute term as a row in shared memory, then the
// window's rows summed per kernel piece, (piece, value) tasks over the lanes,
// each in record order (a fixed order given the layout). Piece j of the window
// goes to pieces[k + window] -- injective, because records are in kernel order,
// so a kernel's pieces are consecutive in window order.
struct GatherParams {
    int K, D, nv;           // nv = 10 + D values per piece: A (3), Q, B upper (6), d_attr (D)
    CameraP cam;
    const int4* kinfo;
    const int2* app;        // [K] {first record, count}
    const int* total;       // records of the render
    const double4* bent;    // records {alpha, d_q, beta, W}
    const int2* bkey;       // records' {pixel, kernel}
    const double4* rays;    // [P] pixel rays (K4)
    const Rec64* rec64;
    const double* d_image;  // [P*D]
    double* pieces;         // [(K + windows) * nv]
    double* acc;            // fallback accumulators (consumed and re-zeroed by K5b)
    double* attr_fb;
    const double* centers;  // object space
    const double* inv_cov;
    double* d_center;       // [K*3]
    double* d_inv_cov;      // [K*9]
    double* d_attr;         // [K*D]
    double* packed;         // nullable: instead of d_center / d_inv_cov / d_attr, rows of 9 + D values
                            // [d_center(3) | d_inv_cov upper (00 01 02 11 12 22) | d_attr(D)] (multi-GPU)
    double* rt_part;        // [gridDim.x * 12] then [groups * 12]
    unsigned* tickets;      // [1 + groups], zero between launches (reset by the last CTAs)
    double* d_rt;           // [12] d_rotation (9), d_translation (3)
};


__global__ void __launch_bounds__(kRecThreads) records_kernel(GatherParams p) {
    launch_dependents();  // the finish may stage its object-space rows meanwhile
    // per warp: the window's record values [32][nv], summed per kernel piece by
    // one lane each, rows in record order
    extern __shared__ __align__(16) double s_rows[];
    const int lane = threadIdx.x & 31;
    double* rows = s_rows + (threadIdx.x >> 5) * 32 * p.nv;
    __shared__ int s_keys[kRecThreads / 32][32];
    __shared__ int s_start[kRecThreads / 32][33];  // first record of each piece of the window, then the end
    int* keys = s_keys[threadIdx.x >> 5];
    int* starts = s_start[threadIdx.x >> 5];
    const int n_rec = *p.total;
    const int windows = (n_rec + 31) >> 5;
    const int wstride = (gridDim.x * blockDim.x) >> 5;
    const float inv_nv = 1.0f / (float)p.nv;
    int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    // the next window's record and key loaded under the current window's work
    int2 key_n = make_int2(0, -1);
    double4 b_n = make_double4(0, 0, 0, 0);
    if (32 * w + lane < n_rec) {
        key_n = p.bkey[32 * w + lane];
        b_n = p.bent[32 * w + lane];
    }
    for (; w < windows; w += wstride) {
        const int r = 32 * w + lane;
        const bool valid = r < n_rec;
        int k = -1;
        const int2 key = key_n;
        const double4 b = b_n;
        if (r + 32 * wstride < n_rec) {
            key_n = p.bkey[r + 32 * wstride];
            b_n = p.bent[r + 32 * wstride];
        }
        if (valid) {
            k = key.y;
            const long long pix = key.x;
            const double4 ray = p.rays[pix];
            double* row = rows + lane * p.nv;
            // upstream image gradient loads issued before the chain (D <= 4 unrolled)
            double di[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) di[c] = c < p.D ? p.d_image[pix * p.D + c] : 0.0;
            // the entry's terms of A = sum alpha d, Q = sum d_q, B = sum beta d d^T (entry_coeffs)
            row[0] = b.x * ray.x;
            row[1] = b.x * ray.y;
            row[2] = b.x * ray.z;
            row[3] = b.y;
            row[4] = b.z * (ray.x * ray.x);
            row[5] = b.z * (ray.x * ray.y);
            row[6] = b.z * (ray.x * ray.z);
            row[7] = b.z * (ray.y * ray.y);
            row[8] = b.z * (ray.y * ray.z);
            row[9] = b.z * (ray.z * ray.z);
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (c < p.D) row[10 + c] = b.w * di[c];
            for (int c = 4; c < p.D; ++c) row[10 + c] = b.w * p.d_image[pix * p.D + c];
        }
        keys[lane] = k;
        const int kprev = __shfl_up_sync(0xffffffffu, k, 1);
        const bool head = valid && (lane == 0 || kprev != k);
        const unsigned heads = __ballot_sync(0xffffffffu, head);
        const int npieces = __popc(heads);
        if (head) starts[__popc(heads & ((1u << lane) - 1u))] = lane;
        if (lane == 0) starts[npieces] = min(32, n_rec - 32 * w);
        __syncwarp();
        // piece sums: (piece, value) tasks over the lanes, each summing its rows
        // in record order
        for (int task = lane; task < npieces * p.nv; task += 32) {
            const int j = __float2int_rd(((float)task + 0.5f) * inv_nv);  // task / nv (exact: task < 2^20)
            const int u = task - j * p.nv;
            const int start = starts[j], end = starts[j + 1];
            // four interleaved partial sums (records q = start + 4i + r), combined in a fixed order
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int q = start;
            for (; q + 4 <= end; q += 4) {
                a0 += rows[q * p.nv + u];
                a1 += rows[(q + 1) * p.nv + u];
                a2 += rows[(q + 2) * p.nv + u];
                a3 += rows[(q + 3) * p.nv + u];
            }
            if (q < end) a0 += rows[q * p.nv + u];
            if (q + 1 < end) a1 += rows[(q + 1) * p.nv + u];
            if (q + 2 < end) a2 += rows[(q + 2) * p.nv + u];
            p.pieces[(long long)(keys[start] + w) * p.nv + u] = (a0 + a1) + (a2 + a3);
        }
        __syncwarp();
    }
}

// K5b: per kernel, its pieces summed in window order, then camera -> object
// space (grad.cpp:184-197):
//   d_center = R^T dm, d_inv_cov = R^T dS R, d_T = sum dm, d_R = sum dm m^T + 2 dS R S.
// d_R, d_T: CTA partial in kernel order -> group of kRtGroup CTAs -> total,
// each in a fixed order (tickets: the last CTA of a level reduces it).
#ifndef GVR_FINISH_THREADS
#define GVR_FINISH_THREADS 128
#endif
constexpr int kFinishThreads = GVR_FINISH_THREADS, kRtGroup = 32;

__global__ void __launch_bounds__(kFinishThreads) finish_kernel(GatherParams p) {
    __shared__ double s_part[kFinishThreads / 32][12];
    __shared__ bool s_last;
    // object-space rows staged through shared memory (coalesced 16-byte traffic)
    __shared__ __align__(16) double s_cov[kFinishThreads * 9];
    __shared__ __align__(16) double s_ctr[kFinishThreads * 3];
    const int k0 = blockIdx.x * kFinishThreads;
    const int count = min(kFinishThreads, p.K - k0);
    stage_rows_in(s_cov, p.inv_cov, k0, count, 9);
    stage_rows_in(s_ctr, p.centers, k0, count, 3);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the records' pieces are complete from here
    __syncthreads();
    const int k = k0 + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double part[12];
#pragma unroll
    for (int t = 0; t < 12; ++t) part[t] = 0.0;
    if (k < p.K) {
        const int2 ap = p.app[k];
        const int4 ki = p.kinfo[k];
        double c9[9];
#pragma unroll
        for (int u = 0; u < 9; ++u) c9[u] = 0.0;
        if (ap.y > 0) {
            const int w0 = ap.x >> 5, w1 = (ap.x + ap.y - 1) >> 5;
            double c10[10], ca[4] = {0.0, 0.0, 0.0, 0.0};  // A (3), Q, B upper (00 01 02 11 12 22); d_attr
#pragma unroll
            for (int u = 0; u < 10; ++u) c10[u] = 0.0;
            for (int w = w0; w <= w1; ++w) {
                const double* src = p.pieces + (long long)(k + w) * p.nv;
#pragma unroll
                for (int u = 0; u < 10; ++u) c10[u] += src[u];
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c < p.D) ca[c] += src[10 + c];
            }
            for (int c = 0; c < p.D; ++c) {
                double a = 0.0;
                if (c < 4) {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (q == c) a = ca[q];
                } else {
                    for (int w = w0; w <= w1; ++w) a += p.pieces[(long long)(k + w) * p.nv + 10 + c];
                }
                if (p.packed) p.packed[(long long)k * (9 + p.D) + 9 + c] = a;
                else p.d_attr[(long long)p.D * k + c] = a;
            }
            // camera-space chain (entry_coeffs): dm = S (A - Q m),
            // dS = sym(m A^T) + B - Q/2 m m^T (upper triangle), with the kernel's
            // camera-space m, S from its staged object-space rows (project_kernel's arithmetic)
            double mm[3], ss[9];
            {
                double mo[3], so[9];
#pragma unroll
                for (int t = 0; t < 3; ++t) mo[t] = s_ctr[3 * threadIdx.x + t];
#pragma unroll
                for (int t = 0; t < 9; ++t) so[t] = s_cov[9 * threadIdx.x + t];
                view_transform_one(p.cam, mo, so, mm, ss);
            }
            const double Q = c10[3];
            const double u0 = fma(-Q, mm[0], c10[0]), u1 = fma(-Q, mm[1], c10[1]), u2 = fma(-Q, mm[2], c10[2]);
#pragma unroll
            for (int t = 0; t < 3; ++t) c9[t] = fma(ss[3 * t], u0, fma(ss[3 * t + 1], u1, ss[3 * t + 2] * u2));
            const int rr[6] = {0, 0, 0, 1, 1, 2};
            const int cc[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
            for (int t = 0; t < 6; ++t) {
                const int a0 = rr[t], a1 = cc[t];
                c9[3 + t] = 0.5 * (mm[a0] * c10[a1] + c10[a0] * mm[a1]) + c10[4 + t] - 0.5 * Q * (mm[a0] * mm[a1]);
            }
        } else if (ki.x < 0 && ki.w > 0) {  // fallback accumulators (no mask rectangle): consume, re-zero
#pragma unroll
            for (int u = 0; u < 9; ++u) {
                c9[u] = p.acc[9ll * k + u];
                p.acc[9ll * k + u] = 0.0;
            }
            for (int c = 0; c < p.D; ++c) {
                const double a = p.attr_fb[(long long)p.D * k + c];
                if (p.packed) p.packed[(long long)k * (9 + p.D) + 9 + c] = a;
                else p.d_attr[(long long)p.D * k + c] = a;
                p.attr_fb[(long long)p.D * k + c] = 0.0;
            }
        } else {
            for (int c = 0; c < p.D; ++c) {
                if (p.packed) p.packed[(long long)k * (9 + p.D) + 9 + c] = 0.0;
                else p.d_attr[(long long)p.D * k + c] = 0.0;
            }
        }
        const double* R = p.cam.R;
        const double dsf[9] = {c9[3], c9[4], c9[5], c9[4], c9[6], c9[7], c9[5], c9[7], c9[8]};
        double dc[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) dc[r] = R[r] * c9[0] + R[3 + r] * c9[1] + R[6 + r] * c9[2];
        double t1[9];  // dS R
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                t1[3 * r + c] = dsf[3 * r] * R[c] + dsf[3 * r + 1] * R[3 + c] + dsf[3 * r + 2] * R[6 + c];
        double dcov[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int rr = r < c ? r : c, cc = r < c ? c : r;  // symmetric: the upper value, mirrored
                dcov[3 * r + c] = R[rr] * t1[cc] + R[3 + rr] * t1[3 + cc] + R[6 + rr] * t1[6 + cc];
            }
        double mo[3], so[9];
#pragma unroll
        for (int t = 0; t < 3; ++t) mo[t] = s_ctr[3 * threadIdx.x + t];
#pragma unroll
        for (int t = 0; t < 9; ++t) so[t] = s_cov[9 * threadIdx.x + t];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                part[3 * r + c] = c9[r] * mo[c] + 2.0 * (t1[3 * r] * so[c] + t1[3 * r + 1] * so[3 + c] +
                                                         t1[3 * r + 2] * so[6 + c]);
#pragma unroll
        for (int t = 0; t < 3; ++t) part[9 + t] = c9[t];
#pragma unroll
        for (int t = 0; t < 3; ++t) s_ctr[3 * threadIdx.x + t] = dc[t];
#pragma unroll
        for (int t = 0; t < 9; ++t) s_cov[9 * threadIdx.x + t] = dcov[t];
        if (p.packed) {
            double* row = p.packed + (long long)k * (9 + p.D);
#pragma unroll
            for (int t = 0; t < 3; ++t) row[t] = dc[t];
            row[3] = dcov[0];
            row[4] = dcov[1];
            row[5] = dcov[2];
            row[6] = dcov[4];
            row[7] = dcov[5];
            row[8] = dcov[8];
        }
    }
    __syncthreads();
    if (!p.packed) {
        stage_rows_out(p.d_center, s_ctr, k0, count, 3);
        stage_rows_out(p.d_inv_cov, s_cov, k0, count, 9);
    }
    // fixed-order block reduction: shfl_down tree per warp, warps in order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int t = 0; t < 12; ++t) part[t] += __shfl_down_sync(0xffffffffu, part[t], o);
    if (lane == 0)
#pragma unroll
        for (int t = 0; t < 12; ++t) s_part[warp][t] = part[t];
    __syncthreads();
    if (threadIdx.x < 12) {
        double v = 0.0;
        for (int w2 = 0; w2 < kFinishThreads / 32; ++w2) v += s_part[w2][threadIdx.x];
        p.rt_part[12ll * blockIdx.x + threadIdx.x] = v;
    }
    __threadfence();
    __syncthreads();
    const int ngroups = (gridDim.x + kRtGroup - 1) / kRtGroup;
    const int group = blockIdx.x / kRtGroup;
    const int gsize = min(kRtGroup, (int)gridDim.x - group * kRtGroup);
    if (threadIdx.x == 0) s_last = atomicAdd(p.tickets + 1 + group, 1u) == (unsigned)gsize - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double* gpart = p.rt_part + 12ll * gridDim.x;
    if (threadIdx.x < 12) {
        double v = 0.0;
        for (int c = group * kRtGroup; c < group * kRtGroup + gsize; ++c) v += __ldcg(p.rt_part + 12ll * c + threadIdx.x);
        gpart[12 * group + threadIdx.x] = v;
    }
    if (threadIdx.x == 0) p.tickets[1 + group] = 0u;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(p.tickets, 1u) == (unsigned)ngroups - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x < 12) {
        double v = 0.0;
        for (int g2 = 0; g2 < ngroups; ++g2) v += __ldcg(gpart + 12 * g2 + threadIdx.x);
        p.d_rt[threadIdx.x] = v;
    }
    if (threadIdx.x == 0) p.tickets[0] = 0u;
}

// ScalarLoss::value (grad.cpp:201-216) on device: d = w (x - target), loss = sum w d^2 / 2.
// Deterministic: a fixed grid-stride partition, per-block partials in a fixed
// tree, and the last block (ticket) sums the partials in block order.
__global__ void scalar_loss_kernel(long long n_img, long long n_alpha, const double* __restrict__ image,
                                   const double* __restrict__ t_image, const double* __restrict__ alpha,
                                   const double* __restrict__ t_alpha, double w_image, double w_alpha,
                                   double* __restrict__ d_image, double* __restrict__ d_alpha,
                                   double* __restrict__ loss, double* __restrict__ part_out, unsigned* ticket) {
    double part = 0.0;
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
    // 16-byte accesses where the buffers allow (pairs of values), two pairs in flight per thread
    const bool vec = ((reinterpret_cast<uintptr_t>(image) | reinterpret_cast<uintptr_t>(t_image) |
                       reinterpret_cast<uintptr_t>(d_image)) & 15) == 0;
    const long long n2 = vec ? n_img / 2 : 0;
    const double2* im2 = reinterpret_cast<const double2*>(image);
    const double2* ti2 = reinterpret_cast<const double2*>(t_image);
    double2* di2 = reinterpret_cast<double2*>(d_image);
#ifndef GVR_LOSS_BATCH
#define GVR_LOSS_BATCH 1
#endif
#if GVR_LOSS_BATCH
    // the thread's first 3 image pairs and 2 alpha values are loaded before any
    // is used (one memory round trip for the common grid; the rest below)
    double2 ia[3], ib[3];
    double aa[2], ab[2];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
        const long long i = tid + u * nt;
        if (i < n2) {
            ia[u] = im2[i];
            ib[u] = ti2[i];
        }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const long long a = tid + u * nt;
        if (a < n_alpha) {
            aa[u] = alpha[a];
            ab[u] = t_alpha[a];
        }
    }
#pragma unroll
    for (int u = 0; u < 3; ++u) {
        const long long i = tid + u * nt;
        if (i < n2) {
            const double x = ia[u].x - ib[u].x, y = ia[u].y - ib[u].y;
            part += 0.5 * w_image * x * x;
            part += 0.5 * w_image * y * y;
            di2[i] = make_double2(w_image * x, w_image * y);
        }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const long long a = tid + u * nt;
        if (a < n_alpha) {
            const double diff = aa[u] - ab[u];
            part += 0.5 * w_alpha * diff * diff;
            d_alpha[a] = w_alpha * diff;
        }
    }
    const long long i0 = tid + 3 * nt, a0 = tid + 2 * nt;
#else
    const long long i0 = tid, a0 = tid;
#endif
#pragma unroll 2
    for (long long i = i0; i < n2; i += nt) {
        const double2 a = im2[i], b = ti2[i];
        const double x = a.x - b.x, y = a.y - b.y;
        part += 0.5 * w_image * x * x;
        part += 0.5 * w_image * y * y;
        di2[i] = make_double2(w_image * x, w_image * y);
    }
    for (long long idx = 2 * n2 + tid; idx < n_img; idx += nt) {
        const double diff = image[idx] - t_image[idx];
        part += 0.5 * w_image * diff * diff;
        d_image[idx] = w_image * diff;
    }
#pragma unroll 2
    for (long long a = a0; a < n_alpha; a += nt) {
        const double diff = alpha[a] - t_alpha[a];
        part += 0.5 * w_alpha * diff * diff;
        d_alpha[a] = w_alpha * diff;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    __shared__ double red[32];
    __shared__ bool s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) v += red[w];
        part_out[blockIdx.x] = v;
        __threadfence();
        s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // last block: partials in block order (lane-strided, then a fixed tree)
    double v = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v += __ldcg(part_out + b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) tot += red[w];
        *loss = tot;
        *ticket = 0u;
    }
}

// dst += src (gradient accumulation across views, fit.cpp:153).
__global__ void axpy_kernel(long long n, const double* __restrict__ src, double* __restrict__ dst) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) dst[i] += src[i];
}

// AdamState::update (fit.cpp:20-42), bias corrections from the host in FP64.
__global__ void adam_kernel(long long n, double* __restrict__ params, const double* __restrict__ grads,
                            double* __restrict__ m, double* __restrict__ v, double lr, double beta1, double beta2,
                            double eps, double bc1, double bc2, const double* __restrict__ loss = nullptr,
                            int* __restrict__ diverged = nullptr) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    // fit_shape (fit.cpp:246-250): a non-finite loss ends the fit before the update;
    // the device flag latches, so every later update is skipped as well
    if (diverged && (*diverged || !isfinite(*loss))) {
        if (i == 0) *diverged = 1;
        return;
    }
    const double g = grads[i];
    const double mi = beta1 * m[i] + (1.0 - beta1) * g;
    const double vi = beta2 * v[i] + (1.0 - beta2) * g * g;
    m[i] = mi;
    v[i] = vi;
    params[i] -= lr * (mi / bc1) / (sqrt(vi / bc2) + eps);
}

// weight_store / traced copy-out: expand the compact per-pixel lists to K'-padded arrays.
__global__ void expand_topk_kernel(long long P, int kp, const int* __restrict__ topk, const int* __restrict__ count,
                                   const double* __restrict__ topk_w, int* __restrict__ out_idx,
                                   double* __restrict__ out_w) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (o >= P * kp) return;
    const long long p = o / kp;
    const int s = (int)(o % kp);
    const bool ok = s < count[p];
    if (out_idx) out_idx[o] = ok ? topk[o] : -1;
    if (out_w) out_w[o] = ok ? topk_w[o] : 0.0;
}

// Tape::cam_scene copy-out: the view-transformed centres and inverse
// covariances (scene.cpp:5-17) exactly as the projection computed them.
__global__ void cam_scene_kernel(int K, const Rec64* __restrict__ rec64, double* __restrict__ centers,
                                 double* __restrict__ inv_cov) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const Rec64& r = rec64[k];
    if (centers)
        for (int t = 0; t < 3; ++t) centers[3ll * k + t] = r.m[t];
    if (inv_cov)
        for (int t = 0; t < 9; ++t) inv_cov[9ll * k + t] = r.s[t];
}

// Tape::traced copy-out: exact FP64 (l, q, sigma) of the taped selection.
__global__ void traced_kernel(CameraP cam, int kp, const int* __restrict__ topk, const int* __restrict__ count,
                              const Rec64* __restrict__ rec64, int* __restrict__ out_idx, double* __restrict__ out_l,
                              double* __restrict__ out_q, double* __restrict__ out_sigma) {
    const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long P = (long long)cam.H * cam.W;
    if (o >= P * kp) return;
    const long long p = o / kp;
    const int s = (int)(o % kp);
    const bool ok = s < count[p];
    double l = 0.0, q = 0.0, sg = 0.0;
    int id = -1;
    if (ok) {
        double d[3];
        pixel_ray(cam, (int)(p / cam.W), (int)(p % cam.W), d);
        id = topk[o];
        const Traced64 t = trace_exact(d, rec64[id]);
        l = t.l;
        q = t.q;
        sg = sigma_of(t.a);
    }
    if (out_idx) out_idx[o] = id;
    if (out_l) out_l[o] = l;
    if (out_q) out_q[o] = q;
    if (out_sigma) out_sigma[o] = sg;
}

}  // namespace gvrk
