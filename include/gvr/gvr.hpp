// gvr/gvr.hpp — C++ drop-in for the reference render API (namespace gvr) on top
// of the C ABI in gvr_cuda.h. Header-only; link against libgvr_cuda.so.
//
// Mirrors /root/reference/proj/include/gvr/{types,tracer,blender,grad}.hpp:
//   GaussianKernel / GaussianScene / Camera / Image / ValidationError   types.hpp:19-93
//   SelectionConfig / TracedKernel                                      tracer.hpp:11-25
//   RenderBuffers (weight_store) / render                               blender.hpp:18-41
//   Tape / ForwardResult / GradFlags / GradientBundle / ScalarLoss /
//   render_with_tape / backward                                         grad.hpp:13-70
// Same field names, argument meaning and error behaviour (ValidationError with
// the reference's message text). `threads` is accepted and ignored.
//
// Linear-algebra types: the reference uses Eigen (Vector3d / Matrix3d /
// VectorXd). Define GVR_WITH_EIGEN (and put Eigen on the include path) to get
// exactly those types; otherwise small value types with the same accessors
// (x(), y(), z(), operator()(r, c), operator[], size()) are used.
#pragma once

#include "../gvr_cuda.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#ifdef GVR_WITH_EIGEN
#include <Eigen/Dense>
#endif

namespace gvr {

#ifdef GVR_WITH_EIGEN
using Vec3 = Eigen::Vector3d;
using Mat3 = Eigen::Matrix3d;
using VecX = Eigen::VectorXd;
#else
struct Vec3 {
    double v[3] = {0.0, 0.0, 0.0};
    Vec3() = default;
    Vec3(double x, double y, double z) : v{x, y, z} {}
    static Vec3 Zero() { return Vec3(); }
    static Vec3 UnitZ() { return Vec3(0, 0, 1); }
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
    double& operator()(int i) { return v[i]; }
    double operator()(int i) const { return v[i]; }
    double x() const { return v[0]; }
    double y() const { return v[1]; }
    double z() const { return v[2]; }
    int size() const { return 3; }
};
struct Mat3 {
    double m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};  // row-major
    static Mat3 Identity() { return Mat3(); }
    static Mat3 Zero() {
        Mat3 z;
        std::memset(z.m, 0, sizeof z.m);
        return z;
    }
    double& operator()(int r, int c) { return m[3 * r + c]; }
    double operator()(int r, int c) const { return m[3 * r + c]; }
};
struct VecX {
    std::vector<double> v;
    VecX() = default;
    explicit VecX(int n) : v(static_cast<size_t>(n), 0.0) {}
    VecX(std::initializer_list<double> l) : v(l) {}
    static VecX Zero(int n) { return VecX(n); }
    double& operator[](int i) { return v[static_cast<size_t>(i)]; }
    double operator[](int i) const { return v[static_cast<size_t>(i)]; }
    double& operator()(int i) { return v[static_cast<size_t>(i)]; }
    double operator()(int i) const { return v[static_cast<size_t>(i)]; }
    int size() const { return static_cast<int>(v.size()); }
};
#endif

// types.hpp:19-22
class ValidationError : public std::runtime_error {
public:
    explicit ValidationError(const std::string& msg) : std::runtime_error(msg) {}
};

// types.hpp:26-33
struct GaussianKernel {
    Vec3 center = Vec3::Zero();
    Mat3 inv_cov = Mat3::Identity();
    VecX attr;
};

// types.hpp:35-42
struct GaussianScene {
    std::vector<GaussianKernel> kernels;
    double tau = 1.0;
    int attr_dim() const { return kernels.empty() ? 0 : static_cast<int>(kernels.front().attr.size()); }
    int size() const { return static_cast<int>(kernels.size()); }
};

// types.hpp:46-56
struct Camera {
    Mat3 rotation = Mat3::Identity();
    Vec3 translation = Vec3::Zero();
    double focal = 1.0;
    double ox = 0.0;
    double oy = 0.0;
    int height = 1;
    int width = 1;

    void validate() const;  // types.cpp:44-63 (gvr_camera_validate: no device needed)
};

enum class ChannelSemantics : std::uint8_t { Color, Alpha, Normal, Feature };

// types.hpp:71-93
struct Image {
    int height = 0;
    int width = 0;
    int channels = 0;
    ChannelSemantics semantics = ChannelSemantics::Color;
    std::vector<double> data;

    Image() = default;
    Image(int h, int w, int c, ChannelSemantics sem = ChannelSemantics::Color)
        : height(h), width(w), channels(c), semantics(sem), data(static_cast<size_t>(h) * w * c, 0.0) {}
    double& at(int r, int c, int ch) { return data[(static_cast<size_t>(r) * width + c) * channels + ch]; }
    double at(int r, int c, int ch) const { return data[(static_cast<size_t>(r) * width + c) * channels + ch]; }
    size_t pixel_count() const { return static_cast<size_t>(height) * width; }
};

// tracer.hpp:11-25
struct TracedKernel {
    int kernel_index = 0;
    double l = 0.0;
    double q = 0.0;
    double sigma = 1.0;
};

struct SelectionConfig {
    double eta = 0.01;
    int k_prime = 20;
    bool coarse_enabled = true;
    int coarse_downsample = 8;
};

// blender.hpp:18-25
struct RenderBuffers {
    Image image;
    Image alpha;
    Image depth;
    std::vector<std::vector<std::pair<int, double>>> weight_store;
};

// grad.hpp:13-22
struct GradientBundle {
    std::vector<Vec3> d_center;
    std::vector<Mat3> d_inv_cov;
    std::vector<VecX> d_attr;
    Mat3 d_rotation = Mat3::Zero();
    Vec3 d_translation = Vec3::Zero();
};

// grad.hpp:46-49
struct GradFlags {
    bool through_transmittance = true;
    bool through_density = true;
};

namespace detail {

// One device context per host thread (the reference's API is free functions).
struct Ctx {
    gvr_context* ctx = nullptr;
    Ctx() {
        int dev = 0;
        if (const char* e = std::getenv("GVR_DEVICE")) dev = std::atoi(e);
        if (gvr_context_create(dev, &ctx) != GVR_OK) throw std::runtime_error("gvr: no usable sm_100 CUDA device");
    }
    ~Ctx() { gvr_context_destroy(ctx); }
};

inline gvr_context* context() {
    thread_local Ctx c;
    return c.ctx;
}

inline void check(int rc) {
    if (rc == GVR_OK) return;
    const std::string msg = gvr_last_error(context());
    if (rc == GVR_ERR_VALIDATION) throw ValidationError(msg);
    throw std::runtime_error(msg);
}

struct SceneHandle {
    gvr_scene* s = nullptr;
    SceneHandle() { check(gvr_scene_create(context(), &s)); }
    ~SceneHandle() { gvr_scene_destroy(s); }
};

struct TapeHandle {
    gvr_tape* t = nullptr;
    TapeHandle() { check(gvr_tape_create(context(), &t)); }
    ~TapeHandle() { gvr_tape_destroy(t); }
};

// GaussianScene (AoS) -> flat FP64 arrays -> gvr_scene_set (validates once).
inline std::shared_ptr<SceneHandle> upload(const GaussianScene& scene) {
    const int k = scene.size(), d = scene.attr_dim();
    if (scene.tau < 0.0 || !std::isfinite(scene.tau)) throw ValidationError("tau must be finite and >= 0");
    std::vector<double> c(3 * static_cast<size_t>(k)), s(9 * static_cast<size_t>(k)), a(static_cast<size_t>(d) * k);
    for (int i = 0; i < k; ++i) {
        const auto& g = scene.kernels[i];
        if (g.attr.size() != d)
            throw ValidationError("attribute dimension is not uniform (kernel " + std::to_string(i) + ")");
        for (int t = 0; t < 3; ++t) c[3 * i + t] = g.center[t];
        for (int r = 0; r < 3; ++r)
            for (int t = 0; t < 3; ++t) s[9 * i + 3 * r + t] = g.inv_cov(r, t);
        for (int t = 0; t < d; ++t) a[static_cast<size_t>(d) * i + t] = g.attr[t];
    }
    auto h = std::make_shared<SceneHandle>();
    check(gvr_scene_set(context(), h->s, k, d, scene.tau, c.data(), s.data(), a.data()));
    return h;
}

inline gvr_camera to_c(const Camera& cam) {
    gvr_camera c;
    for (int r = 0; r < 3; ++r)
        for (int t = 0; t < 3; ++t) c.rotation[3 * r + t] = cam.rotation(r, t);
    for (int t = 0; t < 3; ++t) c.translation[t] = cam.translation[t];
    c.focal = cam.focal;
    c.ox = cam.ox;
    c.oy = cam.oy;
    c.height = cam.height;
    c.width = cam.width;
    return c;
}

}  // namespace detail

inline void Camera::validate() const {
    const gvr_camera c = detail::to_c(*this);
    char msg[256] = {0};
    if (gvr_camera_validate(&c, msg, static_cast<int32_t>(sizeof msg)) != GVR_OK) throw ValidationError(msg);
}

namespace detail {

inline gvr_selection to_c(const SelectionConfig& s) {
    return gvr_selection{s.eta, s.k_prime, s.coarse_enabled ? 1 : 0, s.coarse_downsample};
}

}  // namespace detail

// grad.hpp:26-33. The device record of the forward; `traced` (Tape::traced) and
// the camera-space scene (`cam_scene()`, Tape::cam_scene) are materialised on request.
struct Tape {
    GaussianScene scene;
    Camera camera;
    SelectionConfig cfg;
    int threads = 0;
    std::shared_ptr<detail::SceneHandle> device_scene;
    std::shared_ptr<detail::TapeHandle> device_tape;

    GaussianScene cam_scene() const {  // view_transform (scene.cpp:5-17) as the device computed it
        const size_t k = scene.kernels.size();
        std::vector<double> c(3 * k), s(9 * k);
        detail::check(gvr_tape_cam_scene(detail::context(), device_tape->t, c.data(), s.data()));
        GaussianScene out = scene;
        for (size_t i = 0; i < k; ++i) {
            out.kernels[i].center = Vec3(c[3 * i], c[3 * i + 1], c[3 * i + 2]);
            for (int r = 0; r < 3; ++r)
                for (int t = 0; t < 3; ++t) out.kernels[i].inv_cov(r, t) = s[9 * i + 3 * r + t];
        }
        return out;
    }

    std::vector<std::vector<TracedKernel>> traced() const {
        const size_t p = static_cast<size_t>(camera.height) * camera.width, kp = cfg.k_prime;
        std::vector<int32_t> idx(p * kp);
        std::vector<double> l(p * kp), q(p * kp), s(p * kp);
        detail::check(gvr_tape_traced(detail::context(), device_tape->t, idx.data(), l.data(), q.data(), s.data()));
        std::vector<std::vector<TracedKernel>> out(p);
        for (size_t i = 0; i < p; ++i)
            for (size_t k = 0; k < kp && idx[i * kp + k] >= 0; ++k)
                out[i].push_back({idx[i * kp + k], l[i * kp + k], q[i * kp + k], s[i * kp + k]});
        return out;
    }
};

// grad.hpp:35-38
struct ForwardResult {
    RenderBuffers buffers;
    Tape tape;
};

// grad.hpp:41-42 / grad.cpp:38-47
inline ForwardResult render_with_tape(const GaussianScene& scene, const Camera& camera, const SelectionConfig& cfg,
                                      int threads = 0) {
    ForwardResult fr;
    fr.tape.scene = scene;
    fr.tape.camera = camera;
    fr.tape.cfg = cfg;
    fr.tape.threads = threads;
    fr.tape.device_scene = detail::upload(scene);
    fr.tape.device_tape = std::make_shared<detail::TapeHandle>();
    const int h = camera.height, w = camera.width, dc = std::max(scene.attr_dim(), 1);
    const size_t p = static_cast<size_t>(std::max(h, 0)) * std::max(w, 0), kp = std::max(cfg.k_prime, 0);
    RenderBuffers& b = fr.buffers;
    b.image = Image(h, w, dc, ChannelSemantics::Color);
    b.alpha = Image(h, w, 1, ChannelSemantics::Alpha);
    b.depth = Image(h, w, 1, ChannelSemantics::Feature);
    std::vector<int32_t> idx(p * kp);
    std::vector<double> wts(p * kp);
    const gvr_camera cc = detail::to_c(camera);
    const gvr_selection sc = detail::to_c(cfg);
    const gvr_render_outputs out{b.image.data.data(), b.alpha.data.data(), b.depth.data.data(), idx.data(),
                                 wts.data()};
    detail::check(gvr_render(detail::context(), fr.tape.device_scene->s, &cc, &sc, fr.tape.device_tape->t, &out));
    b.weight_store.assign(p, {});
    for (size_t i = 0; i < p; ++i)
        for (size_t k = 0; k < kp && idx[i * kp + k] >= 0; ++k) b.weight_store[i].emplace_back(idx[i * kp + k], wts[i * kp + k]);
    return fr;
}

// blender.hpp:40-41
inline RenderBuffers render(const GaussianScene& scene, const Camera& camera, const SelectionConfig& cfg,
                            int threads = 0) {
    return render_with_tape(scene, camera, cfg, threads).buffers;
}

// grad.hpp:53-54 / grad.cpp:49-199
inline GradientBundle backward(const Tape& tape, const Image& d_image, const Image& d_alpha,
                               const GradFlags& flags = {}) {
    const int h = tape.camera.height, w = tape.camera.width, dim = tape.scene.attr_dim(), k = tape.scene.size();
    if (d_image.height != h || d_image.width != w || d_image.channels != dim)
        throw ValidationError("backward: d_image shape does not match the forward render");
    if (d_alpha.height != h || d_alpha.width != w || d_alpha.channels != 1)
        throw ValidationError("backward: d_alpha shape does not match the forward render");
    std::vector<double> dc(3 * static_cast<size_t>(k)), ds(9 * static_cast<size_t>(k)),
        da(static_cast<size_t>(dim) * k), dr(9), dt(3);
    const gvr_grad_flags f{flags.through_transmittance ? 1 : 0, flags.through_density ? 1 : 0};
    const gvr_gradients out{dc.data(), ds.data(), dim > 0 ? da.data() : nullptr, dr.data(), dt.data()};
    detail::check(gvr_backward(detail::context(), tape.device_tape->t, dim > 0 ? d_image.data.data() : nullptr,
                               d_alpha.data.data(), &f, &out));
    GradientBundle g;
    g.d_center.resize(k);
    g.d_inv_cov.resize(k);
    g.d_attr.assign(k, VecX::Zero(dim));
    for (int i = 0; i < k; ++i) {
        g.d_center[i] = Vec3(dc[3 * i], dc[3 * i + 1], dc[3 * i + 2]);
        for (int r = 0; r < 3; ++r)
            for (int t = 0; t < 3; ++t) g.d_inv_cov[i](r, t) = ds[9 * i + 3 * r + t];
        for (int t = 0; t < dim; ++t) g.d_attr[i][t] = da[static_cast<size_t>(dim) * i + t];
    }
    for (int r = 0; r < 3; ++r)
        for (int t = 0; t < 3; ++t) g.d_rotation(r, t) = dr[3 * r + t];
    g.d_translation = Vec3(dt[0], dt[1], dt[2]);
    return g;
}

// grad.hpp:62-70 / grad.cpp:201-216 (the reference's host-side loss functional).
struct ScalarLoss {
    Image target_image;
    Image target_alpha;
    double w_image = 1.0;
    double w_alpha = 1.0;

    double value(const RenderBuffers& buf, Image* d_image, Image* d_alpha) const {
        double loss = 0.0;
        if (d_image) *d_image = Image(buf.image.height, buf.image.width, buf.image.channels);
        if (d_alpha) *d_alpha = Image(buf.alpha.height, buf.alpha.width, 1, ChannelSemantics::Alpha);
        for (size_t i = 0; i < buf.image.data.size(); ++i) {
            const double diff = buf.image.data[i] - target_image.data[i];
            loss += 0.5 * w_image * diff * diff;
            if (d_image) d_image->data[i] = w_image * diff;
        }
        for (size_t i = 0; i < buf.alpha.data.size(); ++i) {
            const double diff = buf.alpha.data[i] - target_alpha.data[i];
            loss += 0.5 * w_alpha * diff * diff;
            if (d_alpha) d_alpha->data[i] = w_alpha * diff;
        }
        return loss;
    }
};

// ---------------------------------------------------------------- sampler (sampler.hpp)

// sampler.hpp:8-15
struct SampledAttributes {
    std::vector<VecX> attrs;      // K x D
    std::vector<double> support;  // sum of observed weights per kernel
    std::vector<bool> masked;     // true where support fell below the threshold
    int masked_count() const {
        int n = 0;
        for (bool m : masked) n += m ? 1 : 0;
        return n;
    }
};

inline constexpr double kSupportEps = 1e-8;  // sampler.hpp:18

// sampler.hpp:23-25 / sampler.cpp:11-51 (gvr_sample_attributes: render + device scatter).
inline SampledAttributes sample_attributes(const Image& observed, const GaussianScene& scene, const Camera& camera,
                                           const SelectionConfig& cfg, bool normalized = false, int threads = 0) {
    (void)threads;
    if (observed.height != camera.height || observed.width != camera.width)
        throw ValidationError("observed image size does not match the camera");
    const auto dscene = detail::upload(scene);
    const int k = scene.size(), dim = observed.channels;
    std::vector<double> a(static_cast<size_t>(k) * dim), sp(k);
    std::vector<uint8_t> m(k);
    const gvr_camera cc = detail::to_c(camera);
    const gvr_selection sc = detail::to_c(cfg);
    detail::check(gvr_sample_attributes(detail::context(), dscene->s, &cc, &sc, observed.data.data(), observed.height,
                                        observed.width, dim, normalized ? 1 : 0, a.data(), sp.data(), m.data()));
    SampledAttributes out;
    out.attrs.assign(k, VecX::Zero(dim));
    out.support = sp;
    out.masked.assign(k, false);
    for (int i = 0; i < k; ++i) {
        for (int c = 0; c < dim; ++c) out.attrs[i][c] = a[static_cast<size_t>(dim) * i + c];
        out.masked[i] = m[i] != 0;
    }
    return out;
}

// sampler.hpp:29-30 / sampler.cpp:53-66 (gvr_scene_resynthesize + gvr_render).
inline RenderBuffers resynthesize(const SampledAttributes& attrs, const GaussianScene& scene, const Camera& camera,
                                  const SelectionConfig& cfg, int threads = 0) {
    if (attrs.attrs.size() != static_cast<size_t>(scene.size()))
        throw ValidationError("sampled attribute count does not match the scene");
    GaussianScene recolored = scene;
    for (int k = 0; k < scene.size(); ++k)
        recolored.kernels[k].attr = attrs.masked[k] ? VecX::Zero(attrs.attrs[k].size()) : attrs.attrs[k];
    return render(recolored, camera, cfg, threads);
}

// ---------------------------------------------------------------- helpers (blender.hpp)

// transmittance_at (blender.hpp:29) for every pixel of a taped render: T(t(i,j))
// over that pixel's selected kernels (the reference's per-ray span form, batched).
inline Image transmittance_at(const Tape& tape, const Image& t) {
    if (t.height != tape.camera.height || t.width != tape.camera.width || t.channels != 1)
        throw ValidationError("transmittance_at: depth image shape does not match the forward render");
    Image out(t.height, t.width, 1, ChannelSemantics::Feature);
    detail::check(gvr_tape_transmittance(detail::context(), tape.device_tape->t, t.data.data(), out.data.data()));
    return out;
}

// normalized_weights (blender.hpp:36) of every pixel's weight_store, same layout.
inline std::vector<std::vector<std::pair<int, double>>> normalized_weights(const ForwardResult& fr,
                                                                           double eps = 1e-8) {
    const size_t p = fr.buffers.weight_store.size(), kp = static_cast<size_t>(fr.tape.cfg.k_prime);
    std::vector<double> nw(p * kp);
    detail::check(gvr_tape_normalized_weights(detail::context(), fr.tape.device_tape->t, eps, nw.data()));
    std::vector<std::vector<std::pair<int, double>>> out(p);
    for (size_t i = 0; i < p; ++i)
        for (size_t k = 0; k < fr.buffers.weight_store[i].size(); ++k)
            out[i].emplace_back(fr.buffers.weight_store[i][k].first, nw[i * kp + k]);
    return out;
}

// blender.hpp:46-47 / blender.cpp:146-172 (gvr_shade_lambert).
inline Image shade_lambert(const Image& normals, const Image& alpha, const Image& depth, const Camera& camera,
                           const Vec3& light_pos, const Vec3& light_color) {
    if (normals.channels != 3) throw ValidationError("shade_lambert expects a 3-channel normal image");
    if (normals.height != alpha.height || normals.width != alpha.width || normals.height != depth.height ||
        normals.width != depth.width)
        throw ValidationError("shade_lambert: buffer sizes do not match");
    Image out(normals.height, normals.width, 3, ChannelSemantics::Color);
    Camera cam = camera;
    cam.height = normals.height;
    cam.width = normals.width;
    const gvr_camera cc = detail::to_c(cam);
    const double lp[3] = {light_pos[0], light_pos[1], light_pos[2]};
    const double lc[3] = {light_color[0], light_color[1], light_color[2]};
    if (out.pixel_count() == 0) return out;
    detail::check(gvr_shade_lambert(detail::context(), &cc, normals.data.data(), alpha.data.data(), depth.data.data(),
                                    lp, lc, out.data.data()));
    return out;
}

// ---------------------------------------------------------------- gradcheck (grad.hpp:67-88)

// so3.cpp:7-65 on row-major double[9] (usable with either Vec3 / Mat3 flavour).
namespace detail {
inline void so3_exp_raw(const double w[3], double r[9]) {
    const double th = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    const double k[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
    double kk[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) kk[3 * i + j] = k[3 * i] * k[j] + k[3 * i + 1] * k[3 + j] + k[3 * i + 2] * k[6 + j];
    const double s = th < 1e-12 ? 1.0 : std::sin(th) / th;
    const double c = th < 1e-12 ? 0.5 : (1.0 - std::cos(th)) / (th * th);
    for (int i = 0; i < 9; ++i) r[i] = (i % 4 == 0 ? 1.0 : 0.0) + s * k[i] + c * kk[i];
}
inline void so3_log_raw(const double r[9], double w[3]) {
    const double ct = std::clamp((r[0] + r[4] + r[8] - 1.0) * 0.5, -1.0, 1.0);
    const double th = std::acos(ct);
    if (th < 1e-9) {
        w[0] = 0.5 * (r[7] - r[5]);
        w[1] = 0.5 * (r[2] - r[6]);
        w[2] = 0.5 * (r[3] - r[1]);
        return;
    }
    if (th > M_PI - 1e-6) {
        double a[9];
        for (int i = 0; i < 9; ++i) a[i] = 0.5 * (r[i] + (i % 4 == 0 ? 1.0 : 0.0));
        double ax[3] = {std::sqrt(std::max(0.0, a[0])), std::sqrt(std::max(0.0, a[4])), std::sqrt(std::max(0.0, a[8]))};
        int major = 0;
        for (int i = 1; i < 3; ++i)
            if (a[4 * i] > a[4 * major]) major = i;
        for (int i = 0; i < 3; ++i)
            if (i != major && a[3 * major + i] < 0.0) ax[i] = -ax[i];
        const double n = std::sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
        for (int i = 0; i < 3; ++i) w[i] = n < 1e-12 ? 0.0 : th * ax[i] / n;
        return;
    }
    const double f = th / (2.0 * std::sin(th));
    w[0] = (r[7] - r[5]) * f;
    w[1] = (r[2] - r[6]) * f;
    w[2] = (r[3] - r[1]) * f;
}
inline void so3_exp_gradient_raw(const double w[3], const double dr[9], double g[3]) {
    const double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
    double r[9];
    so3_exp_raw(w, r);
    auto hat = [](const double v[3], double h[9]) {
        const double t[9] = {0, -v[2], v[1], v[2], 0, -v[0], -v[1], v[0], 0};
        std::memcpy(h, t, sizeof t);
    };
    for (int i = 0; i < 3; ++i) {
        double e[3] = {0, 0, 0};
        e[i] = 1.0;
        double d[9];
        if (th2 < 1e-16) {
            hat(e, d);
        } else {
            double ire[3];  // (I - R) e
            for (int a = 0; a < 3; ++a) ire[a] = e[a] - r[3 * a + i];
            const double v[3] = {w[1] * ire[2] - w[2] * ire[1], w[2] * ire[0] - w[0] * ire[2], w[0] * ire[1] - w[1] * ire[0]};
            double hw[9], hv[9], m[9];
            hat(w, hw);
            hat(v, hv);
            for (int a = 0; a < 9; ++a) m[a] = (w[i] * hw[a] + hv[a]) / th2;
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) d[3 * a + b] = m[3 * a] * r[b] + m[3 * a + 1] * r[3 + b] + m[3 * a + 2] * r[6 + b];
        }
        double acc = 0.0;
        for (int a = 0; a < 9; ++a) acc += dr[a] * d[a];
        g[i] = acc;
    }
}
}  // namespace detail

struct GradCheckEntry {
    double max_rel_err = 0.0;
    int checked = 0;
    int skipped_boundary = 0;
    double worst_analytic = 0.0;
    double worst_numeric = 0.0;
};

struct GradCheckReport {
    std::map<std::string, GradCheckEntry> per_class;
    double max_rel_err = 0.0;
    int total_checked = 0;
    int total_skipped = 0;
    bool passed(double tol) const { return max_rel_err < tol; }
};

// grad.cpp:242-350: central differences of the loss over center / inv_cov /
// attr / pose against backward(); directions whose selection sets change
// within +-h are skipped. Forward evaluations run in the library's
// verification mode (exact FP64 pair terms, gvr_context_set_precise).
inline GradCheckReport gradcheck(const GaussianScene& scene, const Camera& camera, const SelectionConfig& cfg,
                                 const ScalarLoss& loss, double h = 1e-4, double tol = 1e-3, int threads = 0) {
    (void)tol;
    struct Precise {
        Precise() { detail::check(gvr_context_set_precise(detail::context(), 1)); }
        ~Precise() { gvr_context_set_precise(detail::context(), 0); }
    } precise;
    double rr[9], w0[3];
    for (int i = 0; i < 9; ++i) rr[i] = camera.rotation(i / 3, i % 3);
    detail::so3_log_raw(rr, w0);
    Camera cam = camera;
    detail::so3_exp_raw(w0, rr);
    for (int i = 0; i < 9; ++i) cam.rotation(i / 3, i % 3) = rr[i];

    ForwardResult base = render_with_tape(scene, cam, cfg, threads);
    Image d_image, d_alpha;
    loss.value(base.buffers, &d_image, &d_alpha);
    const GradientBundle bundle = backward(base.tape, d_image, d_alpha);
    auto sets_of = [](const RenderBuffers& b) {
        std::vector<std::vector<int>> s(b.weight_store.size());
        for (size_t p = 0; p < s.size(); ++p)
            for (const auto& e : b.weight_store[p]) s[p].push_back(e.first);
        return s;
    };
    const auto base_sets = sets_of(base.buffers);
    struct Eval {
        double loss = 0.0;
        bool valid = false;
        std::vector<std::vector<int>> sets;
    };
    auto evaluate = [&](const GaussianScene& s, const Camera& c) {
        Eval e;
        try {
            const RenderBuffers b = render(s, c, cfg, threads);
            e.loss = loss.value(b, nullptr, nullptr);
            e.sets = sets_of(b);
            e.valid = true;
        } catch (const ValidationError&) {
            e.valid = false;
        }
        return e;
    };
    GradCheckReport report;
    auto rel_err = [](double a, double n) {
        if (std::abs(a) < 1e-7 && std::abs(n) < 1e-7) return 0.0;
        return std::abs(a - n) / std::max(std::abs(a) + std::abs(n), 1e-6);
    };
    auto check = [&](const std::string& cls, double analytic, auto apply, double step) {
        auto& entry = report.per_class[cls];
        GaussianScene sp = scene, sm = scene;
        Camera cp = cam, cm = cam;
        apply(sp, cp, step);
        apply(sm, cm, -step);
        const Eval plus = evaluate(sp, cp), minus = evaluate(sm, cm);
        if (!plus.valid || !minus.valid || plus.sets != base_sets || minus.sets != base_sets) {
            ++entry.skipped_boundary;
            ++report.total_skipped;
            return;
        }
        const double numeric = (plus.loss - minus.loss) / (2.0 * step);
        const double rel = rel_err(analytic, numeric);
        ++entry.checked;
        ++report.total_checked;
        if (rel > entry.max_rel_err) {
            entry.max_rel_err = rel;
            entry.worst_analytic = analytic;
            entry.worst_numeric = numeric;
        }
        report.max_rel_err = std::max(report.max_rel_err, rel);
    };
    for (int k = 0; k < scene.size(); ++k) {
        for (int d = 0; d < 3; ++d)
            check("center", bundle.d_center[k][d],
                  [k, d](GaussianScene& s, Camera&, double e) { s.kernels[k].center[d] += e; },
                  h * std::max(1.0, std::abs(scene.kernels[k].center[d])));
        for (int i = 0; i < 3; ++i)
            for (int j = i; j < 3; ++j)
                check("inv_cov", i == j ? bundle.d_inv_cov[k](i, i) : 2.0 * bundle.d_inv_cov[k](i, j),
                      [k, i, j](GaussianScene& s, Camera&, double e) {
                          s.kernels[k].inv_cov(i, j) += e;
                          if (i != j) s.kernels[k].inv_cov(j, i) += e;
                      },
                      h * std::max(1.0, std::abs(scene.kernels[k].inv_cov(i, j))));
        for (int d = 0; d < scene.attr_dim(); ++d)
            check("attr", bundle.d_attr[k][d], [k, d](GaussianScene& s, Camera&, double e) { s.kernels[k].attr[d] += e; },
                  h);
    }
    double dr[9], dw[3];
    for (int i = 0; i < 9; ++i) dr[i] = bundle.d_rotation(i / 3, i % 3);
    detail::so3_exp_gradient_raw(w0, dr, dw);
    for (int d = 0; d < 3; ++d)
        check("pose", dw[d],
              [&w0, d](GaussianScene&, Camera& c, double e) {
                  double w[3] = {w0[0], w0[1], w0[2]}, r[9];
                  w[d] += e;
                  detail::so3_exp_raw(w, r);
                  for (int i = 0; i < 9; ++i) c.rotation(i / 3, i % 3) = r[i];
              },
              h);
    for (int d = 0; d < 3; ++d)
        check("pose", bundle.d_translation[d], [d](GaussianScene&, Camera& c, double e) { c.translation[d] += e; },
              h * std::max(1.0, std::abs(cam.translation[d])));
    return report;
}

}  // namespace gvr
