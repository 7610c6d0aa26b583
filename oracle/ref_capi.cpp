// C ABI over the REFERENCE implementation compiled unmodified from
// /root/reference/proj/src (TEST INFRASTRUCTURE ONLY — oracle/_ref).
//
// This file is ours; it only marshals flat FP64 arrays into the reference's
// own types and calls its public API:
//   gvr::render / render_with_tape   (proj/src/blender.cpp:141, proj/src/grad.cpp:38)
//   gvr::backward                    (proj/src/grad.cpp:49)
//   gvr::ScalarLoss::value           (proj/src/grad.cpp:201)
//   gvr::coarse_select               (proj/src/tracer.cpp:37)
//   gvr::make_bench_scene / camera   (proj/src/bench.cpp:9-24)
//   gvr::make_orbit_camera           (proj/src/shapes.cpp:118)
//   gvr::sample_attributes / resynthesize (proj/src/sampler.cpp:11-66)
//   gvr::ShapeRegularizer::make / edge_reg / laplacian_reg (proj/src/fit.cpp:44-113)
//   gvr::transmittance_at / normalized_weights / shade_lambert
//                                    (proj/src/blender.cpp:19-25, 55-62, 146-172)
// Per-pixel variable-length lists come back padded to k_prime (index -1).
// Errors: return 1 for gvr::ValidationError, 2 for anything else; the message
// is available from gvr_ref_last_error().
#include "gvr/bench.hpp"
#include "gvr/blender.hpp"
#include "gvr/grad.hpp"
#include "gvr/fit.hpp"
#include "gvr/sampler.hpp"
#include "gvr/scene.hpp"
#include "gvr/shapes.hpp"
#include "gvr/tracer.hpp"

#include <cstring>
#include <string>

namespace {

thread_local std::string g_err;

gvr::GaussianScene make_scene(int k, int d, double tau, const double* centers, const double* inv_cov,
                              const double* attr) {
    gvr::GaussianScene s;
    s.tau = tau;
    s.kernels.resize(k);
    for (int i = 0; i < k; ++i) {
        auto& g = s.kernels[i];
        g.center = gvr::Vec3(centers[3 * i], centers[3 * i + 1], centers[3 * i + 2]);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) g.inv_cov(r, c) = inv_cov[9 * i + 3 * r + c];
        g.attr = gvr::VecX(d);
        for (int c = 0; c < d; ++c) g.attr[c] = attr[static_cast<size_t>(d) * i + c];
    }
    return s;
}

// cam[17] = R(9, row-major) T(3) focal ox oy height width
gvr::Camera make_camera(const double* cam) {
    gvr::Camera c;
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) c.rotation(r, k) = cam[3 * r + k];
    c.translation = gvr::Vec3(cam[9], cam[10], cam[11]);
    c.focal = cam[12];
    c.ox = cam[13];
    c.oy = cam[14];
    c.height = static_cast<int>(cam[15]);
    c.width = static_cast<int>(cam[16]);
    return c;
}

void export_camera(const gvr::Camera& c, double* cam) {
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) cam[3 * r + k] = c.rotation(r, k);
    cam[9] = c.translation.x();
    cam[10] = c.translation.y();
    cam[11] = c.translation.z();
    cam[12] = c.focal;
    cam[13] = c.ox;
    cam[14] = c.oy;
    cam[15] = c.height;
    cam[16] = c.width;
}

gvr::SelectionConfig make_cfg(double eta, int k_prime, int coarse, int ds) {
    gvr::SelectionConfig c;
    c.eta = eta;
    c.k_prime = k_prime;
    c.coarse_enabled = coarse != 0;
    c.coarse_downsample = ds;
    return c;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const gvr::ValidationError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

void export_buffers(const gvr::RenderBuffers& b, double* image, double* alpha, double* depth) {
    if (image) std::memcpy(image, b.image.data.data(), b.image.data.size() * sizeof(double));
    if (alpha) std::memcpy(alpha, b.alpha.data.data(), b.alpha.data.size() * sizeof(double));
    if (depth) std::memcpy(depth, b.depth.data.data(), b.depth.data.size() * sizeof(double));
}

}  // namespace

extern "C" {

const char* gvr_ref_last_error() { return g_err.c_str(); }

// Forward render. Outputs (nullable): image[H*W*max(D,1)], alpha[H*W], depth[H*W],
// topk_idx[H*W*kp] (int32, -1 pad), topk_w[H*W*kp], topk_l/q/sigma[H*W*kp]
// (the tape: selected traced kernels, ascending (l, idx)).
int gvr_ref_render(int k, int d, double tau, const double* centers, const double* inv_cov,
                   const double* attr, const double* cam, double eta, int k_prime, int coarse,
                   int ds, int threads, double* image, double* alpha, double* depth, int* topk_idx,
                   double* topk_w, double* topk_l, double* topk_q, double* topk_sigma) {
    return guarded([&] {
        const auto scene = make_scene(k, d, tau, centers, inv_cov, attr);
        const auto camera = make_camera(cam);
        const auto cfg = make_cfg(eta, k_prime, coarse, ds);
        const gvr::ForwardResult fr = gvr::render_with_tape(scene, camera, cfg, threads);
        export_buffers(fr.buffers, image, alpha, depth);
        const size_t p_count = static_cast<size_t>(camera.height) * camera.width;
        for (size_t p = 0; p < p_count; ++p) {
            const auto& ws = fr.buffers.weight_store[p];
            const auto& tr = fr.tape.traced[p];
            for (int s = 0; s < k_prime; ++s) {
                const size_t o = p * k_prime + s;
                const bool ok = s < static_cast<int>(ws.size());
                if (topk_idx) topk_idx[o] = ok ? ws[s].first : -1;
                if (topk_w) topk_w[o] = ok ? ws[s].second : 0.0;
                if (topk_l) topk_l[o] = ok ? tr[s].l : 0.0;
                if (topk_q) topk_q[o] = ok ? tr[s].q : 0.0;
                if (topk_sigma) topk_sigma[o] = ok ? tr[s].sigma : 0.0;
            }
        }
    });
}

// render_with_tape + backward for a given upstream gradient. Outputs (nullable):
// d_center[K*3], d_inv_cov[K*9] (row-major), d_attr[K*D], d_rotation[9], d_translation[3].
int gvr_ref_backward(int k, int d, double tau, const double* centers, const double* inv_cov,
                     const double* attr, const double* cam, double eta, int k_prime, int coarse,
                     int ds, int threads, const double* d_image, const double* d_alpha,
                     int through_transmittance, int through_density, double* d_center,
                     double* d_inv_cov, double* d_attr, double* d_rotation, double* d_translation) {
    return guarded([&] {
        const auto scene = make_scene(k, d, tau, centers, inv_cov, attr);
        const auto camera = make_camera(cam);
        const auto cfg = make_cfg(eta, k_prime, coarse, ds);
        const gvr::ForwardResult fr = gvr::render_with_tape(scene, camera, cfg, threads);
        gvr::Image di(camera.height, camera.width, d);
        gvr::Image da(camera.height, camera.width, 1, gvr::ChannelSemantics::Alpha);
        if (d_image) std::memcpy(di.data.data(), d_image, di.data.size() * sizeof(double));
        if (d_alpha) std::memcpy(da.data.data(), d_alpha, da.data.size() * sizeof(double));
        gvr::GradFlags flags;
        flags.through_transmittance = through_transmittance != 0;
        flags.through_density = through_density != 0;
        const gvr::GradientBundle g = gvr::backward(fr.tape, di, da, flags);
        for (int i = 0; i < k; ++i) {
            for (int c = 0; c < 3; ++c)
                if (d_center) d_center[3 * i + c] = g.d_center[i][c];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c)
                    if (d_inv_cov) d_inv_cov[9 * i + 3 * r + c] = g.d_inv_cov[i](r, c);
            for (int c = 0; c < d; ++c)
                if (d_attr) d_attr[static_cast<size_t>(d) * i + c] = g.d_attr[i][c];
        }
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                if (d_rotation) d_rotation[3 * r + c] = g.d_rotation(r, c);
        for (int c = 0; c < 3; ++c)
            if (d_translation) d_translation[c] = g.d_translation[c];
    });
}

// One full fwd+bwd step exactly as the reference's gradcheck / fit loop runs it:
// render_with_tape -> ScalarLoss::value -> backward (proj/src/grad.cpp:38-216).
// Used as the CPU baseline arm. Returns the loss in *loss_out.
int gvr_ref_fwd_bwd_step(int k, int d, double tau, const double* centers, const double* inv_cov,
                         const double* attr, const double* cam, double eta, int k_prime, int coarse,
                         int ds, int threads, const double* target_image, const double* target_alpha,
                         double* loss_out, double* d_center, double* d_attr) {
    return guarded([&] {
        const auto scene = make_scene(k, d, tau, centers, inv_cov, attr);
        const auto camera = make_camera(cam);
        const auto cfg = make_cfg(eta, k_prime, coarse, ds);
        const gvr::ForwardResult fr = gvr::render_with_tape(scene, camera, cfg, threads);
        gvr::ScalarLoss loss;
        loss.target_image = gvr::Image(camera.height, camera.width, std::max(d, 1));
        loss.target_alpha = gvr::Image(camera.height, camera.width, 1, gvr::ChannelSemantics::Alpha);
        std::memcpy(loss.target_image.data.data(), target_image,
                    loss.target_image.data.size() * sizeof(double));
        std::memcpy(loss.target_alpha.data.data(), target_alpha,
                    loss.target_alpha.data.size() * sizeof(double));
        gvr::Image di, da;
        const double l = loss.value(fr.buffers, &di, &da);
        const gvr::GradientBundle g = gvr::backward(fr.tape, di, da);
        if (loss_out) *loss_out = l;
        for (int i = 0; i < k; ++i) {
            for (int c = 0; c < 3; ++c)
                if (d_center) d_center[3 * i + c] = g.d_center[i][c];
            for (int c = 0; c < d; ++c)
                if (d_attr) d_attr[static_cast<size_t>(d) * i + c] = g.d_attr[i][c];
        }
    });
}

// Coarse map statistics and the per-kernel cell boxes actually pushed.
// cell_box[K*4] = (cr_lo, cr_hi, cc_lo, cc_hi) in coarse-cell units, -1 if not pushed.
int gvr_ref_coarse_boxes(int k, int d, double tau, const double* centers, const double* inv_cov,
                         const double* attr, const double* cam, double eta, int k_prime, int ds,
                         int* cell_box, int* dropped_behind) {
    return guarded([&] {
        const auto scene = make_scene(k, d, tau, centers, inv_cov, attr);
        const auto camera = make_camera(cam);
        const auto cfg = make_cfg(eta, k_prime, 1, ds);
        const auto cam_scene = gvr::view_transform(scene, camera);
        const gvr::PixelKernelMap map = gvr::coarse_select(cam_scene, camera, cfg);
        for (int i = 0; i < 4 * k; ++i) cell_box[i] = -1;
        for (int cr = 0; cr < map.grid_rows; ++cr) {
            for (int cc = 0; cc < map.grid_cols; ++cc) {
                for (int kk : map.cells[static_cast<size_t>(cr) * map.grid_cols + cc]) {
                    int* b = cell_box + 4 * kk;
                    if (b[0] < 0 || cr < b[0]) b[0] = cr;
                    if (cr > b[1]) b[1] = cr;
                    if (b[2] < 0 || cc < b[2]) b[2] = cc;
                    if (cc > b[3]) b[3] = cc;
                }
            }
        }
        if (dropped_behind) *dropped_behind = map.dropped_behind_camera;
    });
}

// Work counters on the same inputs (implementation independent):
// counts[0] = C = sum_p |candidates(p)|, counts[1] = N1 = sum_p n_p, counts[2] = N2 = sum_p n_p^2.
int gvr_ref_work_counts(int k, int d, double tau, const double* centers, const double* inv_cov,
                        const double* attr, const double* cam, double eta, int k_prime, int coarse,
                        int ds, int threads, double* counts) {
    return guarded([&] {
        const auto scene = make_scene(k, d, tau, centers, inv_cov, attr);
        const auto camera = make_camera(cam);
        const auto cfg = make_cfg(eta, k_prime, coarse, ds);
        const auto cam_scene = gvr::view_transform(scene, camera);
        double c = 0.0;
        if (coarse) {
            const gvr::PixelKernelMap map = gvr::coarse_select(cam_scene, camera, cfg);
            for (int i = 0; i < camera.height; ++i)
                for (int j = 0; j < camera.width; ++j) c += map.candidates(i, j).size();
        } else {
            int front = 0;
            for (const auto& kk : cam_scene.kernels) front += kk.center.z() > gvr::kBehindCameraEps;
            c = static_cast<double>(front) * camera.height * camera.width;
        }
        const gvr::RenderBuffers b = gvr::render(scene, camera, cfg, threads);
        double n1 = 0.0, n2 = 0.0;
        for (const auto& ws : b.weight_store) {
            n1 += ws.size();
            n2 += static_cast<double>(ws.size()) * ws.size();
        }
        counts[0] = c;
        counts[1] = n1;
        counts[2] = n2;
    });
}

// Synthetic benchmark inputs (proj/src/bench.cpp:9-24, proj/src/shapes.cpp:118-141).
// Call with centers == nullptr to get the kernel count in *k_out.
int gvr_ref_make_bench_scene(int n, int* k_out, int* d_out, double* tau_out, double* centers,
                             double* inv_cov, double* attr) {
    return guarded([&] {
        const gvr::GaussianScene s = gvr::make_bench_scene(n);
        *k_out = s.size();
        *d_out = s.attr_dim();
        *tau_out = s.tau;
        if (!centers) return;
        for (int i = 0; i < s.size(); ++i) {
            const auto& g = s.kernels[i];
            for (int c = 0; c < 3; ++c) centers[3 * i + c] = g.center[c];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) inv_cov[9 * i + 3 * r + c] = g.inv_cov(r, c);
            for (int c = 0; c < s.attr_dim(); ++c) attr[static_cast<size_t>(s.attr_dim()) * i + c] = g.attr[c];
        }
    });
}

int gvr_ref_make_bench_camera(int size, double* cam) {
    return guarded([&] { export_camera(gvr::make_bench_camera(size), cam); });
}

int gvr_ref_make_orbit_camera(double azimuth, double elevation, double distance, const double* target,
                              int height, int width, double focal, double* cam) {
    return guarded([&] {
        export_camera(gvr::make_orbit_camera(azimuth, elevation, distance,
                                             gvr::Vec3(target[0], target[1], target[2]), height,
                                             width, focal),
                      cam);
    });
}

// gvr::sample_attributes (proj/src/sampler.cpp:11-51). observed[H*W*C] with the
// camera's H, W. Outputs: attrs[K*C], support[K], masked[K] (0/1).
int gvr_ref_sample_attributes(int k, int d, double tau, const double* centers, const double* inv_cov,
                              const double* attr, const double* cam, double eta, int k_prime, int coarse,
                              int ds, int threads, const double* observed, int obs_h, int obs_w,
                              int channels, int normalized, double* attrs, double* support,
                              unsigned char* masked) {
    return guarded([&] {
        const auto scene = make_scene(k, d, tau, centers, inv_cov, attr);
        const auto camera = make_camera(cam);
        const auto cfg = make_cfg(eta, k_prime, coarse, ds);
        gvr::Image obs(obs_h, obs_w, channels);
        std::memcpy(obs.data.data(), observed, obs.data.size() * sizeof(double));
        const gvr::SampledAttributes sa =
            gvr::sample_attributes(obs, scene, camera, cfg, normalized != 0, threads);
        for (int i = 0; i < k; ++i) {
            for (int c = 0; c < channels; ++c) attrs[static_cast<size_t>(channels) * i + c] = sa.attrs[i][c];
            support[i] = sa.support[i];
            masked[i] = sa.masked[i] ? 1 : 0;
        }
    });
}

// gvr::resynthesize (proj/src/sampler.cpp:53-66): render with attributes
// replaced (masked -> zero). n_attrs = number of sampled rows (checked).
int gvr_ref_resynthesize(int k, int d, double tau, const double* centers, const double* inv_cov,
                         const double* attr, const double* cam, double eta, int k_prime, int coarse,
                         int ds, int threads, int n_attrs, int channels, const double* attrs,
                         const unsigned char* masked, double* image, double* alpha, double* depth) {
    return guarded([&] {
        const auto scene = make_scene(k, d, tau, centers, inv_cov, attr);
        const auto camera = make_camera(cam);
        const auto cfg = make_cfg(eta, k_prime, coarse, ds);
        gvr::SampledAttributes sa;
        for (int i = 0; i < n_attrs; ++i) {
            gvr::VecX a(channels);
            for (int c = 0; c < channels; ++c) a[c] = attrs[static_cast<size_t>(channels) * i + c];
            sa.attrs.push_back(a);
            sa.support.push_back(1.0);
            sa.masked.push_back(masked[i] != 0);
        }
        export_buffers(gvr::resynthesize(sa, scene, camera, cfg, threads), image, alpha, depth);
    });
}

// Per-pixel gvr::transmittance_at over the pixel's selected traced kernels
// (Tape::traced of render_with_tape) at depth t[p], and gvr::normalized_weights
// of the pixel's RayBlend (weight_store + alpha). Outputs nullable.
int gvr_ref_pixel_helpers(int k, int d, double tau, const double* centers, const double* inv_cov,
                          const double* attr, const double* cam, double eta, int k_prime, int coarse,
                          int ds, int threads, const double* t, double* trans_out, double eps,
                          double* norm_w) {
    return guarded([&] {
        const auto scene = make_scene(k, d, tau, centers, inv_cov, attr);
        const auto camera = make_camera(cam);
        const auto cfg = make_cfg(eta, k_prime, coarse, ds);
        const gvr::ForwardResult fr = gvr::render_with_tape(scene, camera, cfg, threads);
        const size_t p_count = static_cast<size_t>(camera.height) * camera.width;
        for (size_t p = 0; p < p_count; ++p) {
            if (trans_out) trans_out[p] = gvr::transmittance_at(fr.tape.traced[p], tau, t[p]);
            if (norm_w) {
                gvr::RayBlend rb;
                rb.weights = fr.buffers.weight_store[p];
                rb.alpha = fr.buffers.alpha.data[p];
                const auto nw = gvr::normalized_weights(rb, eps);
                for (int s = 0; s < k_prime; ++s)
                    norm_w[p * k_prime + s] = s < static_cast<int>(nw.size()) ? nw[s].second : 0.0;
            }
        }
    });
}

// gvr::shade_lambert (proj/src/blender.cpp:146-172); normals[H*W*3], alpha/depth[H*W].
int gvr_ref_shade_lambert(const double* cam, const double* normals, const double* alpha,
                          const double* depth, const double* light_pos, const double* light_color,
                          double* out) {
    return guarded([&] {
        const auto camera = make_camera(cam);
        const int h = camera.height, w = camera.width;
        gvr::Image n(h, w, 3), a(h, w, 1, gvr::ChannelSemantics::Alpha), z(h, w, 1);
        std::memcpy(n.data.data(), normals, n.data.size() * sizeof(double));
        std::memcpy(a.data.data(), alpha, a.data.size() * sizeof(double));
        std::memcpy(z.data.data(), depth, z.data.size() * sizeof(double));
        const gvr::Image o = gvr::shade_lambert(
            n, a, z, camera, gvr::Vec3(light_pos[0], light_pos[1], light_pos[2]),
            gvr::Vec3(light_color[0], light_color[1], light_color[2]));
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(double));
    });
}

// ShapeRegularizer::make(edges, rest) then edge_reg / laplacian_reg at centers
// (proj/src/fit.cpp:44-113). Outputs: values[2] = (edge, laplacian), grads
// [N*3] each (nullable).
int gvr_ref_shape_reg(int n_vertices, int n_edges, const int* edges, const double* rest, const double* centers,
                      double* values, double* edge_grad, double* lap_grad) {
    return guarded([&] {
        std::vector<std::pair<int, int>> e;
        for (int i = 0; i < n_edges; ++i) e.emplace_back(edges[2 * i], edges[2 * i + 1]);
        std::vector<gvr::Vec3> r(n_vertices), c(n_vertices);
        for (int i = 0; i < n_vertices; ++i) {
            r[i] = gvr::Vec3(rest[3 * i], rest[3 * i + 1], rest[3 * i + 2]);
            c[i] = gvr::Vec3(centers[3 * i], centers[3 * i + 1], centers[3 * i + 2]);
        }
        const gvr::ShapeRegularizer reg = gvr::ShapeRegularizer::make(e, r);
        std::vector<gvr::Vec3> g;
        values[0] = gvr::edge_reg(c, reg, &g);
        if (edge_grad)
            for (int i = 0; i < n_vertices; ++i)
                for (int d = 0; d < 3; ++d) edge_grad[3 * i + d] = g[i][d];
        values[1] = gvr::laplacian_reg(c, reg, &g);
        if (lap_grad)
            for (int i = 0; i < n_vertices; ++i)
                for (int d = 0; d < 3; ++d) lap_grad[3 * i + d] = g[i][d];
    });
}

// gvr::view_transform (proj/src/scene.cpp:5-17): camera-space centers / inv_cov.
int gvr_ref_view_transform(int k, int d, double tau, const double* centers, const double* inv_cov,
                           const double* attr, const double* cam, double* out_centers, double* out_inv_cov) {
    return guarded([&] {
        const auto scene = make_scene(k, d, tau, centers, inv_cov, attr);
        const auto cs = gvr::view_transform(scene, make_camera(cam));
        for (int i = 0; i < k; ++i) {
            for (int t = 0; t < 3; ++t) out_centers[3 * i + t] = cs.kernels[i].center[t];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) out_inv_cov[9 * i + 3 * r + c] = cs.kernels[i].inv_cov(r, c);
        }
    });
}

}  // extern "C"
