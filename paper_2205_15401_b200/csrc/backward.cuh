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
    const Rec64* rec64;
    const double* attr;     // [K*D]
    const double* d_image;  // [P*D]
    const double* d_alpha;  // [P]
    double* acc;            // [K*9] camera space: dm(3), dS upper (00 01 02 11 12 22)
    double* d_attr;         // [K*D]
};

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
    double2* b_lda = reinterpret_cast<double2*>(smem);  // {l_k - l_0, d_acc_k = -tau T_k d_w_k e^{q_k}}
    double* b_dt = reinterpret_cast<double*>(b_lda + KMAX * NP);  // density path d_w_k T_k (grad.cpp:120)
    float2* b_pi = reinterpret_cast<float2*>(b_dt + KMAX * NP);   // {e^{q_k}, 1 / sigma_k}
    int* b_id = reinterpret_cast<int*>(b_pi + KMAX * NP);

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
#if GVR_BWD_IDS_FIRST
    // ids first: the thread's id loads are independent, the record loads behind them overlap
    int kq[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) kq[q] = sub + 4 * q < n ? p.topk[pix * p.kp + sub + 4 * q] : 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int s = sub + 4 * q;
        if (s >= n) break;
        const int k = kq[q];
#else
    for (int s = sub; s < n; s += 4) {
        const int k = p.topk[pix * p.kp + s];
#endif
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
        const double w = trans * pk;
        if (w != 0.0 || dw != 0.0) {
            if (p.D <= 4) {
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c < p.D) atomicAdd(&p.d_attr[(long long)p.D * k + c], w * dimg[c]);
            } else {
                for (int c = 0; c < p.D; ++c) atomicAdd(&p.d_attr[(long long)p.D * k + c], w * p.d_image[pix * p.D + c]);
            }
        }
        b_lda[s * NP + g] = make_double2(er.l - l0, (p.through_t && dw != 0.0) ? -tau * trans * (dw * pk) : 0.0);
        b_dt[s * NP + g] = (p.through_rho && dw != 0.0) ? dw * trans : 0.0;
        b_pi[s * NP + g] = make_float2(pkf, er.is);
        b_id[s * NP + g] = k;
    }
    peak_part += __shfl_xor_sync(grp, peak_part, 1, 4);
    peak_part += __shfl_xor_sync(grp, peak_part, 2, 4);
    __syncwarp(grp);
    const double galpha = p.d_alpha[pix];
    const double d_total = (p.through_t && galpha != 0.0) ? galpha * tau * exp(-tau * peak_part) : 0.0;

    // entry-major pair terms + chain to camera space (grad.cpp:121-173)
    for (int e = sub; e < n; e += 4) {
        const double2 lde = b_lda[e * NP + g];
        const double dle = lde.x, dae = lde.y;
        const float2 pie = b_pi[e * NP + g];
        const float ise = pie.y;
        const double pke = (double)pie.x;
        const int kid = b_id[e * NP + g];
        double dpk = d_total + b_dt[e * NP + g];  // density path (grad.cpp:120)
        // branch-free pair terms, two independent accumulator sets (even / odd k)
        // so that consecutive pairs overlap instead of serialising on one chain
        double dpk2 = 0.0, dl = 0.0, dl2 = 0.0, dsg = 0.0, dsg2 = 0.0;
        auto pair = [&](int k, double& a_pk, double& a_l, double& a_sg) {
            const double2 ldk = b_lda[k * NP + g];
            const double dak = ldk.y, dlk = ldk.x;
            const float2 pik = b_pi[k * NP + g];
            const float isk = pik.y;
            // pair (k, m = e): z1 = (l_k - l_e) / sigma_e ; pair (k = e, m = k): z2 = (l_e - l_k) / sigma_k
            const float dlf = (float)(dlk - dle);
            const float z1 = dlf * ise;
            const float phi1 = normal_pdf_fast(z1);
            // sigma_k == sigma_e (exactly): z2 = -z1 and phi(z2) = phi(z1)
            const float phi2 = isk == ise ? phi1 : normal_pdf_fast(-dlf * isk);
            a_pk = fma(dak, (double)fast_normal_cdf(z1), a_pk);
            const double gg = k != e ? dak * (double)(phi1 * ise) * pke : 0.0;
            a_l -= gg;
            a_sg -= gg * (double)z1;
            if (k != e) a_l = fma(dae, (double)(pik.x * phi2 * isk), a_l);
        };
        int k = 0;
#if GVR_BWD_WAYS == 4
        double dpk3 = 0.0, dpk4 = 0.0, dl3 = 0.0, dl4 = 0.0, dsg3 = 0.0, dsg4 = 0.0;
        for (; k + 4 <= n; k += 4) {
            pair(k, dpk, dl, dsg);
            pair(k + 1, dpk2, dl2, dsg2);
            pair(k + 2, dpk3, dl3, dsg3);
            pair(k + 3, dpk4, dl4, dsg4);
        }
        dpk2 += dpk4;
        dpk += dpk3;
        dl += dl3;
        dl2 += dl4;
        dsg += dsg3;
        dsg2 += dsg4;
#endif
        for (; k + 2 <= n; k += 2) {
            pair(k, dpk, dl, dsg);
            pair(k + 1, dpk2, dl2, dsg2);
        }
        if (k < n) pair(k, dpk, dl, dsg);
        dpk += dpk2;
        dl += dl2;
        dsg += dsg2;
        const double dq = dpk * pke;
        if (dl == 0.0 && dq == 0.0 && dsg == 0.0) continue;

        const Rec64 r = p.rec64[kid];
        double sd[3], v[3], sv[3];
        const double s00 = r.s[0], s01 = r.s[1], s02 = r.s[2], s11 = r.s[4], s12 = r.s[5], s22 = r.s[8];
        sd[0] = fma(s00, d[0], fma(s01, d[1], s02 * d[2]));
        sd[1] = fma(s01, d[0], fma(s11, d[1], s12 * d[2]));
        sd[2] = fma(s02, d[0], fma(s12, d[1], s22 * d[2]));
        const double a = fma(d[0], sd[0], fma(d[1], sd[1], d[2] * sd[2]));
        const double l = fma(d[0], r.sm[0], fma(d[1], r.sm[1], d[2] * r.sm[2])) / a;
#pragma unroll
        for (int t = 0; t < 3; ++t) v[t] = fma(-l, d[t], r.m[t]);
        sv[0] = fma(s00, v[0], fma(s01, v[1], s02 * v[2]));
        sv[1] = fma(s01, v[0], fma(s11, v[1], s12 * v[2]));
        sv[2] = fma(s02, v[0], fma(s12, v[1], s22 * v[2]));
        const double scale = dl / a;
        const double sigma = 1.0 / sqrt(a);
        const double d_a = -0.5 * sigma * sigma * sigma * dsg;
        double* acc = p.acc + 9ll * kid;
        // dm = (d_l/a) S d - d_q S v
#pragma unroll
        for (int t = 0; t < 3; ++t) atomicAdd(acc + t, scale * sd[t] - dq * sv[t]);
        // dS = (d_l/a)(0.5 (m d^T + d m^T) - l d d^T) - 0.5 d_q v v^T + d_a d d^T  (upper triangle)
        const int rr[6] = {0, 0, 0, 1, 1, 2};
        const int cc[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
        for (int t = 0; t < 6; ++t) {
            const int a0 = rr[t], a1 = cc[t];
            const double ddt = d[a0] * d[a1];
            const double val = scale * (0.5 * (r.m[a0] * d[a1] + d[a0] * r.m[a1]) - l * ddt) -
                               0.5 * dq * (v[a0] * v[a1]) + d_a * ddt;
            atomicAdd(acc + 3 + t, val);
        }
    }
}

struct ObjParams {
    int K;
    CameraP cam;
    const double* acc;      // [K*9]
    const double* centers;  // object space
    const double* inv_cov;  // object space
    double* d_center;       // [K*3]
    double* d_inv_cov;      // [K*9]
    double* d_rt;           // [12] = d_rotation(9) d_translation(3), accumulated
};

// K5: camera -> object space once per kernel (grad.cpp:184-197):
// d_center = R^T dm, d_inv_cov = R^T dS R, d_T = sum dm, d_R = sum dm m^T + 2 dS R S.
constexpr int kObjThreads = 128;

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

__global__ void __launch_bounds__(kObjThreads) object_space_kernel(ObjParams p) {
    __shared__ __align__(16) double s_acc[kObjThreads * 9];
    __shared__ __align__(16) double s_cov[kObjThreads * 9];
    __shared__ __align__(16) double s_ctr[kObjThreads * 3];
    const int k0 = blockIdx.x * kObjThreads;
    const int count = min(kObjThreads, p.K - k0);
    stage_rows_in(s_acc, p.acc, k0, count, 9);
    stage_rows_in(s_cov, p.inv_cov, k0, count, 9);
    stage_rows_in(s_ctr, p.centers, k0, count, 3);
    __syncthreads();
    const int t0 = threadIdx.x;
    const int k = k0 + t0;
    double part[12], dc[3] = {0.0, 0.0, 0.0}, dcov[9];
#pragma unroll
    for (int t = 0; t < 12; ++t) part[t] = 0.0;
#pragma unroll
    for (int t = 0; t < 9; ++t) dcov[t] = 0.0;
    if (k < p.K) {
        const double* a = s_acc + 9 * t0;
        const double dm[3] = {a[0], a[1], a[2]};
        const double ds[9] = {a[3], a[4], a[5], a[4], a[6], a[7], a[5], a[7], a[8]};
        const double* R = p.cam.R;
#pragma unroll
        for (int r = 0; r < 3; ++r) dc[r] = R[r] * dm[0] + R[3 + r] * dm[1] + R[6 + r] * dm[2];
        // T1 = dS R; out = R^T T1 (symmetric: compute upper, mirror)
        double t1[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) t1[3 * r + c] = ds[3 * r] * R[c] + ds[3 * r + 1] * R[3 + c] + ds[3 * r + 2] * R[6 + c];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = r; c < 3; ++c) {
                const double val = R[r] * t1[c] + R[3 + r] * t1[3 + c] + R[6 + r] * t1[6 + c];
                dcov[3 * r + c] = val;
                dcov[3 * c + r] = val;
            }
        // d_R += dm m_obj^T + 2 (dS R) S_obj
        const double* mo = s_ctr + 3 * t0;
        const double* so = s_cov + 9 * t0;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                part[3 * r + c] = dm[r] * mo[c] +
                                  2.0 * (t1[3 * r] * so[c] + t1[3 * r + 1] * so[3 + c] + t1[3 * r + 2] * so[6 + c]);
#pragma unroll
        for (int t = 0; t < 3; ++t) part[9 + t] = dm[t];
    }
    __syncthreads();  // the staging rows are reused for the outputs
#pragma unroll
    for (int t = 0; t < 9; ++t) s_acc[9 * t0 + t] = dcov[t];
#pragma unroll
    for (int t = 0; t < 3; ++t) s_ctr[3 * t0 + t] = dc[t];
    __syncthreads();
    stage_rows_out(p.d_inv_cov, s_acc, k0, count, 9);
    stage_rows_out(p.d_center, s_ctr, k0, count, 3);
    // block reduction of the 12 camera-gradient components: a 16-value
    // butterfly (each step halves the values a lane carries), then lane 2v
    // holds the warp total of value v
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double a[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) a[t] = t < 12 ? part[t] : 0.0;
#pragma unroll
    for (int half = 8, bit = 16; half >= 1; half >>= 1, bit >>= 1) {
        const bool hi = lane & bit;
#pragma unroll
        for (int t = 0; t < half; ++t) {
            const double send = hi ? a[t] : a[t + half];
            const double keep = hi ? a[t + half] : a[t];
            a[t] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
        }
    }
    a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
    __shared__ double red[32][12];
    const int v = lane >> 1;
    if (!(lane & 1) && v < 12) red[warp][v] = a[0];
    __syncthreads();
    if (threadIdx.x < 12) {
        double acc = 0.0;
        const int nw = (blockDim.x + 31) / 32;
        for (int w = 0; w < nw; ++w) acc += red[w][threadIdx.x];
        if (acc != 0.0) atomicAdd(p.d_rt + threadIdx.x, acc);
    }
}

// ScalarLoss::value (grad.cpp:201-216) on device: d = w (x - target), loss += w d^2 / 2.
__global__ void scalar_loss_kernel(long long n_img, long long n_alpha, const double* __restrict__ image,
                                   const double* __restrict__ t_image, const double* __restrict__ alpha,
                                   const double* __restrict__ t_alpha, double w_image, double w_alpha,
                                   double* __restrict__ d_image, double* __restrict__ d_alpha,
                                   double* __restrict__ loss) {
    double part = 0.0;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n_img + n_alpha;
         idx += (long long)gridDim.x * blockDim.x) {
        if (idx < n_img) {
            const double diff = image[idx] - t_image[idx];
            part += 0.5 * w_image * diff * diff;
            d_image[idx] = w_image * diff;
        } else {
            const long long a = idx - n_img;
            const double diff = alpha[a] - t_alpha[a];
            part += 0.5 * w_alpha * diff * diff;
            d_alpha[a] = w_alpha * diff;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    __shared__ double red[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) v += red[w];
        atomicAdd(loss, v);
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
