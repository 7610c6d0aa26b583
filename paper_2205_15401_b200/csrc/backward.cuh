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
    const int* topk;   // [P*kp]
    const int* count;  // [P]
    const Rec64* rec64;
    const double* attr;     // [K*D]
    const double* d_image;  // [P*D]
    const double* d_alpha;  // [P]
    double* acc;            // [K*9] camera space: dm(3), dS upper (00 01 02 11 12 22)
    double* d_attr;         // [K*D]
};

// Per pixel (grad.cpp:75-174), one thread per pixel, TILE x TILE pixels per CTA.
// Pair terms are evaluated "entry-major": for entry e all contributions to
// d_peak_e, d_l_e, d_sigma_e are gathered in FP64 registers (the reference
// scatters them pair by pair; the sums are the same), so no per-entry
// accumulator arrays. Arithmetic is FP64; only Phi / phi are evaluated in FP32
// from an FP64-accurate argument (the gradient bar is 1e-4 of a class-scaled
// floor, i.e. ~1e-7 of the largest gradient, which FP32 products would miss).
template <int KMAX, int TILE>
__global__ void __launch_bounds__(TILE* TILE) backward_pixels_kernel(BwdParams p) {
    constexpr int NT = TILE * TILE;
    extern __shared__ __align__(16) unsigned char smem[];
    // per-entry staging, [slot][thread]: FP64 except the kernel id
    double* b_dl = reinterpret_cast<double*>(smem);  // l_k - l_0
    double* b_pk = b_dl + KMAX * NT;                 // e^{q_k}
    double* b_is = b_pk + KMAX * NT;                 // 1 / sigma_k
    double* b_da = b_is + KMAX * NT;                 // d_acc_k = -tau T_k d_w_k e^{q_k}
    double* b_dn = b_da + KMAX * NT;                 // density term d_w_k T_k (or 0)
    int* b_id = reinterpret_cast<int*>(b_dn + KMAX * NT);

    const int tid = threadIdx.x;
    const int tile = blockIdx.x;
    const int i = (tile / p.tiles_x) * TILE + tid / TILE;
    const int j = (tile % p.tiles_x) * TILE + tid % TILE;
    if (i >= p.cam.H || j >= p.cam.W) return;
    const long long pix = (long long)i * p.cam.W + j;
    const int n = p.count[pix];
    if (n == 0) return;

    double d[3];
    pixel_ray(p.cam, i, j, d);

    // re-trace the taped selection in exact FP64 (bit-identical to the forward)
    double l0 = 0.0, total_peak = 0.0;
    for (int s = 0; s < n; ++s) {
        const int k = p.topk[pix * p.kp + s];
        const Traced64 t = trace_exact(d, p.rec64[k]);
        if (s == 0) l0 = t.l;
        const double pk = exp(t.q);
        total_peak += pk;
        b_dl[s * NT + tid] = t.l - l0;
        b_pk[s * NT + tid] = pk;
        b_is[s * NT + tid] = __dsqrt_rn(t.a);
        b_id[s * NT + tid] = k;
    }

    const double tau = p.tau;
    const double galpha = p.d_alpha[pix];
    const double d_total = (p.through_t && galpha != 0.0) ? galpha * tau * exp(-tau * total_peak) : 0.0;
    double dimg[4] = {0, 0, 0, 0};
    for (int c = 0; c < p.D && c < 4; ++c) dimg[c] = p.d_image[pix * p.D + c];

    // transmittance, d_weight, attribute gradient, d_acc (grad.cpp:81-120)
    for (int k = 0; k < n; ++k) {
        const double dlk = b_dl[k * NT + tid];
        double a = 0.0;
        for (int m = 0; m < n; ++m) {
            const float z = (float)((dlk - b_dl[m * NT + tid]) * b_is[m * NT + tid]);
            a += b_pk[m * NT + tid] * (double)normal_cdf_f(z);
        }
        const double trans = exp(-tau * a);
        const double pk = b_pk[k * NT + tid];
        const int kid = b_id[k * NT + tid];
        double dw = 0.0;
        if (p.D <= 4) {
            for (int c = 0; c < p.D; ++c) dw += dimg[c] * p.attr[(long long)p.D * kid + c];
        } else {
            for (int c = 0; c < p.D; ++c) dw += p.d_image[pix * p.D + c] * p.attr[(long long)p.D * kid + c];
        }
        const double w = trans * pk;
        if (w != 0.0 || dw != 0.0) {
            for (int c = 0; c < p.D; ++c)
                atomicAdd(&p.d_attr[(long long)p.D * kid + c], w * (p.D <= 4 ? dimg[c] : p.d_image[pix * p.D + c]));
        }
        double dacc = 0.0, dens = 0.0;
        if (dw != 0.0) {
            if (p.through_rho) dens = dw * trans;
            if (p.through_t) dacc = -tau * trans * (dw * pk);
        }
        b_da[k * NT + tid] = dacc;
        b_dn[k * NT + tid] = dens;
    }

    // entry-major pair terms + chain to camera space (grad.cpp:121-173)
    for (int e = 0; e < n; ++e) {
        const double dle = b_dl[e * NT + tid];
        const double ise = b_is[e * NT + tid];
        const double pke = b_pk[e * NT + tid];
        const double dae = b_da[e * NT + tid];
        double dpk = d_total + b_dn[e * NT + tid];
        double dl = 0.0, dsg = 0.0;
        for (int k = 0; k < n; ++k) {
            const double dak = b_da[k * NT + tid];
            const double dlk = b_dl[k * NT + tid];
            if (dak != 0.0) {
                // pair (k, m = e): z = (l_k - l_e) / sigma_e
                const double z = (dlk - dle) * ise;
                const float zf = (float)z;
                dpk += dak * (double)normal_cdf_f(zf);
                if (k != e) {
                    const double g = dak * pke * (double)normal_pdf_f(zf) * ise;
                    dl -= g;
                    dsg -= g * z;
                }
            }
            if (dae != 0.0 && k != e) {
                // pair (k = e, m = k): z = (l_e - l_k) / sigma_k
                const double isk = b_is[k * NT + tid];
                const float zf = (float)((dle - dlk) * isk);
                dl += dae * b_pk[k * NT + tid] * (double)normal_pdf_f(zf) * isk;
            }
        }
        const double dq = dpk * pke;
        if (dl == 0.0 && dq == 0.0 && dsg == 0.0) continue;

        const int kid = b_id[e * NT + tid];
        const Rec64 r = p.rec64[kid];
        double sd[3], v[3], sv[3];
        xmatvec(r.s, d, sd);
        const double a = xdot(d, sd);
        const double l = xdiv(xmul(0.5, xadd(xdot(r.m, sd), xdot(d, r.sm))), a);
#pragma unroll
        for (int t = 0; t < 3; ++t) v[t] = r.m[t] - l * d[t];
        xmatvec(r.s, v, sv);
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
__global__ void object_space_kernel(ObjParams p) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    double part[12];
#pragma unroll
    for (int t = 0; t < 12; ++t) part[t] = 0.0;
    if (k < p.K) {
        const double* a = p.acc + 9ll * k;
        const double dm[3] = {a[0], a[1], a[2]};
        const double ds[9] = {a[3], a[4], a[5], a[4], a[6], a[7], a[5], a[7], a[8]};
        const double* R = p.cam.R;
        // d_center = R^T dm
#pragma unroll
        for (int r = 0; r < 3; ++r) p.d_center[3ll * k + r] = R[r] * dm[0] + R[3 + r] * dm[1] + R[6 + r] * dm[2];
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
                p.d_inv_cov[9ll * k + 3 * r + c] = val;
                p.d_inv_cov[9ll * k + 3 * c + r] = val;
            }
        // d_R += dm m_obj^T + 2 (dS R) S_obj
        const double* mo = p.centers + 3ll * k;
        const double* so = p.inv_cov + 9ll * k;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                part[3 * r + c] = dm[r] * mo[c] +
                                  2.0 * (t1[3 * r] * so[c] + t1[3 * r + 1] * so[3 + c] + t1[3 * r + 2] * so[6 + c]);
#pragma unroll
        for (int t = 0; t < 3; ++t) part[9 + t] = dm[t];
    }
    // block reduction of the 12 camera-gradient components
#pragma unroll
    for (int t = 0; t < 12; ++t) {
        double v = part[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        part[t] = v;
    }
    __shared__ double red[32][12];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int t = 0; t < 12; ++t) red[warp][t] = part[t];
    __syncthreads();
    if (threadIdx.x < 12) {
        double v = 0.0;
        const int nw = (blockDim.x + 31) / 32;
        for (int w = 0; w < nw; ++w) v += red[w][threadIdx.x];
        if (v != 0.0) atomicAdd(p.d_rt + threadIdx.x, v);
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
