// gvr/gvr.hpp — C++ drop-in for the reference render API (namespace gvr) on top
// of the C ABI in gvr_cuda.h. Header-only; link against libgvr_cuda.so.
//
// Mirrors /root/reference/proj/include/gvr/{types,tracer,blender,grad,scene,so3,
// parallel,sampler}.hpp, which are re-exported by the same-named headers next to
// this one, so code written against the reference compiles unchanged:
//   GaussianKernel / GaussianScene / Camera / Ray / Image / ValidationError  types.hpp:19-93
//   TracedKernel / SelectionConfig / PixelKernelMap / trace_kernel /
//   coarse_select / fine_select                                            tracer.hpp:11-54
//   RayBlend / RenderBuffers / transmittance_at / blend / normalized_weights /
//   render / shade_lambert / detail::render_core                           blender.hpp:13-56
//   GradientBundle / Tape / ForwardResult / GradFlags / ScalarLoss /
//   render_with_tape / backward / gradcheck                                grad.hpp:13-88
//   view_transform / pixel_ray / generate_rays / compose_extrinsics        scene.hpp:10-19
//   so3_hat / so3_exp / so3_log / so3_exp_gradient / so3_tangent_gradient so3.hpp:7-21
//   resolve_threads / parallel_for_partitions                              parallel.hpp:12-43
//   SampledAttributes / sample_attributes / resynthesize                   sampler.hpp:8-30
// Same field names, argument meaning and error behaviour (ValidationError with
// the reference's message text). Every numerical step runs on the GPU through the
// C ABI (no CPU fallback); the host only marshals containers. `threads` is
// accepted and ignored (results never depend on it).
//
// Deviations a caller can observe: Tape::traced is materialised from the device
// on first access (read-only container view); per-ray building blocks (blend,
// fine_select's sort) accept at most 2048 entries per call on the GPU backend.
//
// Linear-algebra types: the reference uses Eigen (Vector3d / Matrix3d /
// VectorXd). Define GVR_WITH_EIGEN (and put Eigen on the include path) to get
// exactly those types; otherwise small value types with the same accessors
// (x(), y(), z(), operator()(r, c), operator[], size()) are used.
//
// Threading: one device context per host thread; objects (tapes, scenes) share
// ownership of the context that made them, so they may outlive that thread,
// but a context must not be used by two threads at once.
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
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>
#if __cplusplus >= 202002L
#include <span>
#endif

#ifdef GVR_WITH_EIGEN
#include <Eigen/Dense>
#endif

namespace gvr {

#ifdef GVR_WITH_EIGEN
using Vec2 = Eigen::Vector2d;
using Vec3 = Eigen::Vector3d;
using VecX = Eigen::VectorXd;
using Mat2 = Eigen::Matrix2d;
using Mat3 = Eigen::Matrix3d;
#else
struct Vec3 {
    double v[3] = {0.0, 0.0, 0.0};
    Vec3() = default;
    Vec3(double x, double y, double z) : v{x, y, z} {}
    static Vec3 Zero() { return Vec3(); }
    static Vec3 UnitZ() { return Vec3(0, 0, 1); }
    static Vec3 Unit(int i) {
        Vec3 e;
        e.v[i] = 1.0;
        return e;
    }
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
    double& operator()(int i) { return v[i]; }
    double operator()(int i) const { return v[i]; }
    double x() const { return v[0]; }
    double y() const { return v[1]; }
    double z() const { return v[2]; }
    int size() const { return 3; }
    void setZero() { v[0] = v[1] = v[2] = 0.0; }
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
    void setZero() { std::memset(m, 0, sizeof m); }
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
    void validate(int index = -1) const;  // types.cpp:17-29 (on the device)
};

// types.hpp:35-42
struct GaussianScene {
    std::vector<GaussianKernel> kernels;
    double tau = 1.0;
    int attr_dim() const { return kernels.empty() ? 0 : static_cast<int>(kernels.front().attr.size()); }
    int size() const { return static_cast<int>(kernels.size()); }
    void validate() const;  // types.cpp:31-42 (on the device)
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
    void validate() const;  // types.cpp:44-63 (gvr_camera_validate)
};

// types.hpp:60-64
struct Ray {
    Vec3 dir = Vec3::UnitZ();
    int row = 0;
    int col = 0;
};

enum class ChannelSemantics : std::uint8_t { Color, Alpha, Normal, Feature };

// types.cpp:65-73
inline const char* to_string(ChannelSemantics s) {
    switch (s) {
        case ChannelSemantics::Color: return "color";
        case ChannelSemantics::Alpha: return "alpha";
        case ChannelSemantics::Normal: return "normal";
        case ChannelSemantics::Feature: return "feature";
    }
    return "unknown";
}

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
    // types.cpp:75-81 (a check of the caller's host container)
    void validate_finite() const {
        for (double v : data)
            if (!std::isfinite(v)) throw ValidationError("image contains non-finite values");
    }
};

// tracer.hpp:11-16
struct TracedKernel {
    int kernel_index = 0;
    double l = 0.0;
    double q = 0.0;
    double sigma = 1.0;
};

// tracer.hpp:18-25
struct SelectionConfig {
    double eta = 0.01;
    int k_prime = 20;
    bool coarse_enabled = true;
    int coarse_downsample = 8;
    // tracer.cpp:8-18 (parameter checks, same messages)
    void validate() const {
        if (!(eta > 0.0 && eta < 1.0)) throw ValidationError("selection eta must be in (0, 1)");
        if (k_prime < 1) throw ValidationError("selection k_prime must be >= 1");
        if (coarse_downsample < 1) throw ValidationError("coarse downsample must be >= 1");
    }
};

// tracer.hpp:27
inline constexpr double kBehindCameraEps = 1e-4;

// tracer.hpp:31-41
struct PixelKernelMap {
    int grid_rows = 0;
    int grid_cols = 0;
    int downsample = 8;
    std::vector<std::vector<int>> cells;
    int dropped_behind_camera = 0;
    const std::vector<int>& candidates(int row, int col) const {
        return cells[static_cast<size_t>(row / downsample) * grid_cols + col / downsample];
    }
};

// blender.hpp:13-16
struct RayBlend {
    std::vector<std::pair<int, double>> weights;  // (kernel_index, W), ascending (l, idx)
    double alpha = 0.0;
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

    // grad.cpp:20-26
    void init(int kernel_count, int attr_dim) {
        d_center.assign(kernel_count, Vec3::Zero());
        d_inv_cov.assign(kernel_count, Mat3::Zero());
        d_attr.assign(kernel_count, VecX::Zero(attr_dim));
        d_rotation = Mat3::Zero();
        d_translation = Vec3::Zero();
    }
    // grad.cpp:28-36 (parameter bookkeeping of the caller's host bundles)
    void add(const GradientBundle& other) {
        for (size_t k = 0; k < d_center.size(); ++k) {
            for (int i = 0; i < 3; ++i) d_center[k][i] += other.d_center[k][i];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) d_inv_cov[k](r, c) += other.d_inv_cov[k](r, c);
            for (int i = 0; i < static_cast<int>(d_attr[k].size()); ++i) d_attr[k][i] += other.d_attr[k][i];
        }
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) d_rotation(r, c) += other.d_rotation(r, c);
        for (int i = 0; i < 3; ++i) d_translation[i] += other.d_translation[i];
    }
};

// grad.hpp:46-49
struct GradFlags {
    bool through_transmittance = true;
    bool through_density = true;
};

namespace detail {

// One device context per host thread, shared by every object made with it.
struct Ctx {
    gvr_context* ctx = nullptr;
    Ctx() {
        int dev = 0;
        if (const char* e = std::getenv("GVR_DEVICE")) dev = std::atoi(e);
        if (gvr_context_create(dev, &ctx) != GVR_OK) throw std::runtime_error("gvr: no usable sm_100 CUDA device");
    }
    ~Ctx() { gvr_context_destroy(ctx); }
    Ctx(const Ctx&) = delete;
    Ctx& operator=(const Ctx&) = delete;
};

inline const std::shared_ptr<Ctx>& context_ptr() {
    thread_local const std::shared_ptr<Ctx> c = std::make_shared<Ctx>();
    return c;
}

inline gvr_context* context() { return context_ptr()->ctx; }

inline void check(int rc, gvr_context* c) {
    if (rc == GVR_OK) return;
    const std::string msg = gvr_last_error(c);
    if (rc == GVR_ERR_VALIDATION) throw ValidationError(msg);
    throw std::runtime_error(msg);
}

inline void check(int rc) { check(rc, context()); }

struct SceneHandle {
    std::shared_ptr<Ctx> owner = context_ptr();
    gvr_scene* s = nullptr;
    SceneHandle() { check(gvr_scene_create(owner->ctx, &s), owner->ctx); }
    ~SceneHandle() { gvr_scene_destroy(s); }  // before `owner` releases the context
    SceneHandle(const SceneHandle&) = delete;
    SceneHandle& operator=(const SceneHandle&) = delete;
};

struct TapeHandle {
    std::shared_ptr<Ctx> owner = context_ptr();
    gvr_tape* t = nullptr;
    TapeHandle() { check(gvr_tape_create(owner->ctx, &t), owner->ctx); }
    ~TapeHandle() { gvr_tape_destroy(t); }
    TapeHandle(const TapeHandle&) = delete;
    TapeHandle& operator=(const TapeHandle&) = delete;
};

inline void flatten(const std::vector<GaussianKernel>& ks, size_t begin, size_t end, int d, std::vector<double>& c,
                    std::vector<double>& s, std::vector<double>& a) {
    const size_t n = end - begin;
    c.assign(3 * n, 0.0);
    s.assign(9 * n, 0.0);
    a.assign(static_cast<size_t>(d) * n, 0.0);
    for (size_t i = 0; i < n; ++i) {
        const auto& g = ks[begin + i];
        for (int t = 0; t < 3; ++t) c[3 * i + t] = g.center[t];
        for (int r = 0; r < 3; ++r)
            for (int t = 0; t < 3; ++t) s[9 * i + 3 * r + t] = g.inv_cov(r, t);
        for (int t = 0; t < d; ++t) a[static_cast<size_t>(d) * i + t] = g.attr[t];
    }
}

// Uploads kernels [begin, end) (uniform attribute dimension d) and validates them
// on the device (GaussianKernel::validate of each, types.cpp:17-29); a failure
// message names kernel begin + local index.
inline std::shared_ptr<SceneHandle> upload_range(const std::vector<GaussianKernel>& ks, size_t begin, size_t end, int d,
                                                 double tau) {
    std::vector<double> c, s, a;
    flatten(ks, begin, end, d, c, s, a);
    auto h = std::make_shared<SceneHandle>();
    const int rc = gvr_scene_set(h->owner->ctx, h->s, static_cast<int32_t>(end - begin), d, tau, c.data(), s.data(),
                                 a.data());
    if (rc == GVR_ERR_VALIDATION && begin > 0) {
        std::string msg = gvr_last_error(h->owner->ctx);
        const size_t at = msg.rfind("(kernel ");
        if (at != std::string::npos) {
            const long long local = std::atoll(msg.c_str() + at + 8);
            msg = msg.substr(0, at) + "(kernel " + std::to_string(begin + static_cast<size_t>(local)) + ")";
        }
        throw ValidationError(msg);
    }
    check(rc, h->owner->ctx);
    return h;
}

// GaussianScene::validate (types.cpp:31-42) + upload: kernels validated in index
// order on the device, the uniform-dimension rule at the first kernel that breaks it.
inline std::shared_ptr<SceneHandle> upload(const GaussianScene& scene) {
    if (scene.tau < 0.0 || !std::isfinite(scene.tau)) throw ValidationError("tau must be finite and >= 0");
    const int d = scene.attr_dim();
    size_t bad = scene.kernels.size();
    for (size_t i = 0; i < scene.kernels.size(); ++i)
        if (scene.kernels[i].attr.size() != d) {
            bad = i;
            break;
        }
    if (bad == scene.kernels.size()) return upload_range(scene.kernels, 0, bad, d, scene.tau);
    upload_range(scene.kernels, 0, bad, d, scene.tau);  // kernels before the first mismatch
    upload_range(scene.kernels, bad, bad + 1, static_cast<int>(scene.kernels[bad].attr.size()), scene.tau);
    throw ValidationError("attribute dimension is not uniform (kernel " + std::to_string(bad) + ")");
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

inline gvr_selection to_c(const SelectionConfig& s) {
    return gvr_selection{s.eta, s.k_prime, s.coarse_enabled ? 1 : 0, s.coarse_downsample};
}

// The per-pixel selection of a taped render (Tape::traced), copied from the
// device on first access.
struct TracedStore {
    std::shared_ptr<TapeHandle> tape;
    size_t pixels = 0;
    size_t k_prime = 0;
    std::once_flag once;
    std::vector<std::vector<TracedKernel>> data;
    const std::vector<std::vector<TracedKernel>>& get() {
        std::call_once(once, [this] {
            std::vector<int32_t> idx(pixels * k_prime);
            std::vector<double> l(pixels * k_prime), q(pixels * k_prime), s(pixels * k_prime);
            if (pixels * k_prime > 0)
                check(gvr_tape_traced(tape->owner->ctx, tape->t, idx.data(), l.data(), q.data(), s.data()),
                      tape->owner->ctx);
            data.assign(pixels, {});
            for (size_t i = 0; i < pixels; ++i)
                for (size_t k = 0; k < k_prime && idx[i * k_prime + k] >= 0; ++k)
                    data[i].push_back({idx[i * k_prime + k], l[i * k_prime + k], q[i * k_prime + k], s[i * k_prime + k]});
        });
        return data;
    }
};

}  // namespace detail

inline void Camera::validate() const {
    const gvr_camera c = detail::to_c(*this);
    char msg[256] = {0};
    if (gvr_camera_validate(&c, msg, static_cast<int32_t>(sizeof msg)) != GVR_OK) throw ValidationError(msg);
}

inline void GaussianKernel::validate(int index) const {
    std::vector<GaussianKernel> one{*this};
    try {
        detail::upload_range(one, 0, 1, static_cast<int>(attr.size()), 1.0);
    } catch (const ValidationError& e) {
        std::string msg = e.what();
        const size_t at = msg.rfind(" (kernel ");
        if (at != std::string::npos) msg = msg.substr(0, at);
        throw ValidationError(index >= 0 ? msg + " (kernel " + std::to_string(index) + ")" : msg);
    }
}

inline void GaussianScene::validate() const { detail::upload(*this); }

// Read-only view of Tape::traced (grad.hpp:32): a vector of per-pixel lists.
class TracedView {
public:
    using value_type = std::vector<TracedKernel>;
    const std::vector<value_type>& get() const {
        static const std::vector<value_type> empty;
        return store_ ? store_->get() : empty;
    }
    operator const std::vector<value_type>&() const { return get(); }
    const value_type& operator[](size_t i) const { return get()[i]; }
    const value_type& at(size_t i) const { return get().at(i); }
    size_t size() const { return get().size(); }
    bool empty() const { return get().empty(); }
    auto begin() const { return get().begin(); }
    auto end() const { return get().end(); }
    std::shared_ptr<detail::TracedStore> store_;
};

// grad.hpp:26-33. The device record of the forward (device_scene / device_tape)
// plus the reference's fields; `traced` is materialised on first access.
struct Tape {
    GaussianScene scene;      // object space, as passed to the forward
    GaussianScene cam_scene;  // after view_transform (from the device)
    Camera camera;
    SelectionConfig cfg;
    int threads = 0;
    TracedView traced;        // per pixel, ascending (l, idx)
    std::shared_ptr<detail::SceneHandle> device_scene;
    std::shared_ptr<detail::TapeHandle> device_tape;
};

// grad.hpp:35-38
struct ForwardResult {
    RenderBuffers buffers;
    Tape tape;
};

// ---------------------------------------------------------------- scene.hpp

// scene.cpp:5-17 (gvr_view_transform, camera validated first)
inline GaussianScene view_transform(const GaussianScene& scene, const Camera& camera) {
    const size_t k = scene.kernels.size();
    std::vector<double> c, s, a, oc(3 * k), os(9 * k);
    detail::flatten(scene.kernels, 0, k, 0, c, s, a);
    const gvr_camera cc = detail::to_c(camera);
    detail::check(gvr_view_transform(detail::context(), static_cast<int32_t>(k), c.data(), s.data(), &cc, oc.data(),
                                     os.data()));
    GaussianScene out = scene;
    for (size_t i = 0; i < k; ++i) {
        out.kernels[i].center = Vec3(oc[3 * i], oc[3 * i + 1], oc[3 * i + 2]);
        for (int r = 0; r < 3; ++r)
            for (int t = 0; t < 3; ++t) out.kernels[i].inv_cov(r, t) = os[9 * i + 3 * r + t];
    }
    return out;
}

// scene.cpp:19-22
inline Ray pixel_ray(const Camera& camera, int row, int col) {
    const gvr_camera cc = detail::to_c(camera);
    double d[3];
    detail::check(gvr_pixel_rays(detail::context(), &cc, 1, &row, &col, d));
    return Ray{Vec3(d[0], d[1], d[2]), row, col};
}

// scene.cpp:24-33
inline std::vector<Ray> generate_rays(const Camera& camera) {
    camera.validate();
    const size_t n = static_cast<size_t>(camera.height) * camera.width;
    std::vector<double> d(3 * n);
    const gvr_camera cc = detail::to_c(camera);
    detail::check(gvr_pixel_rays(detail::context(), &cc, static_cast<int64_t>(n), nullptr, nullptr, d.data()));
    std::vector<Ray> rays(n);
    for (size_t i = 0; i < n; ++i)
        rays[i] = Ray{Vec3(d[3 * i], d[3 * i + 1], d[3 * i + 2]), static_cast<int>(i / camera.width),
                      static_cast<int>(i % camera.width)};
    return rays;
}

// scene.cpp:35-40 (camera parameter composition: R2 R1, R2 T1 + T2)
inline Camera compose_extrinsics(const Camera& first, const Camera& second) {
    Camera out = second;
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += second.rotation(r, k) * first.rotation(k, c);
            out.rotation(r, c) = acc;
        }
        double t = 0.0;
        for (int k = 0; k < 3; ++k) t += second.rotation(r, k) * first.translation[k];
        out.translation[r] = t + second.translation[r];
    }
    return out;
}

// ---------------------------------------------------------------- tracer.hpp

// tracer.cpp:20-35 (gvr_trace_pairs, bit-exact)
inline TracedKernel trace_kernel(const Ray& ray, const GaussianKernel& kernel, int kernel_index = 0) {
    double d[3], c[3], s[9], out[3];
    for (int t = 0; t < 3; ++t) {
        d[t] = ray.dir[t];
        c[t] = kernel.center[t];
    }
    for (int r = 0; r < 3; ++r)
        for (int t = 0; t < 3; ++t) s[3 * r + t] = kernel.inv_cov(r, t);
    detail::check(gvr_trace_pairs(detail::context(), 1, d, c, s, out, out + 1, out + 2));
    return TracedKernel{kernel_index, out[0], out[1], out[2]};
}

// tracer.cpp:37-113 (gvr_coarse_select_boxes; the cells are filled in kernel order)
inline PixelKernelMap coarse_select(const GaussianScene& cam_scene, const Camera& camera, const SelectionConfig& cfg) {
    const int ds = cfg.coarse_downsample;
    const size_t k = cam_scene.kernels.size();
    std::vector<double> c, s, a;
    detail::flatten(cam_scene.kernels, 0, k, 0, c, s, a);
    std::vector<int32_t> boxes(4 * k + 4);
    int32_t dropped = 0;
    const gvr_camera cc = detail::to_c(camera);
    const gvr_selection sc = detail::to_c(cfg);
    detail::check(gvr_coarse_select_boxes(detail::context(), static_cast<int32_t>(k), c.data(), s.data(), &cc, &sc,
                                          boxes.data(), &dropped));
    PixelKernelMap map;
    map.downsample = ds;
    map.grid_rows = (camera.height + ds - 1) / ds;
    map.grid_cols = (camera.width + ds - 1) / ds;
    map.cells.assign(static_cast<size_t>(map.grid_rows) * map.grid_cols, {});
    map.dropped_behind_camera = dropped;
    for (size_t i = 0; i < k; ++i) {
        const int32_t* b = &boxes[4 * i];
        if (b[0] > b[1] || b[2] > b[3]) continue;
        for (int cr = b[0] / ds; cr <= b[1] / ds; ++cr)
            for (int ccol = b[2] / ds; ccol <= b[3] / ds; ++ccol)
                map.cells[static_cast<size_t>(cr) * map.grid_cols + ccol].push_back(static_cast<int>(i));
    }
    return map;
}

namespace detail {

constexpr int kRayMax = 2048;  // entries per device sort call (gvr_ray_sort / gvr_blend_ray)

// (l, idx)-sorted subset of `traced` with q > ln(eta) (eta outside (0, 1): all),
// truncated to `keep`; longer lists are merged chunk by chunk on the device.
inline std::vector<TracedKernel> device_select(const std::vector<TracedKernel>& traced, double eta, size_t keep) {
    std::vector<TracedKernel> best;
    size_t pos = 0;
    const size_t room = keep < static_cast<size_t>(kRayMax) ? kRayMax - keep : 0;
    if (traced.size() > static_cast<size_t>(kRayMax) && room == 0)
        throw std::runtime_error("gvr: fine_select of more than 2048 entries needs k_prime < 2048 on the GPU backend");
    do {
        std::vector<TracedKernel> cand = best;
        const size_t take = traced.size() <= static_cast<size_t>(kRayMax) ? traced.size()
                                                                          : std::min(room, traced.size() - pos);
        cand.insert(cand.end(), traced.begin() + static_cast<long>(pos), traced.begin() + static_cast<long>(pos + take));
        pos += take;
        const size_t n = cand.size();
        std::vector<int32_t> idx(n), order(n + 1);
        std::vector<double> l(n), q(n);
        for (size_t i = 0; i < n; ++i) {
            idx[i] = cand[i].kernel_index;
            l[i] = cand[i].l;
            q[i] = cand[i].q;
        }
        int32_t m = 0;
        check(gvr_ray_sort(context(), static_cast<int32_t>(n), idx.data(), l.data(), q.data(), eta, order.data(), &m));
        best.clear();
        for (int32_t i = 0; i < m && best.size() < keep; ++i) best.push_back(cand[static_cast<size_t>(order[i])]);
        eta = -1.0;  // entries kept from earlier rounds already passed the threshold
        if (traced.size() <= static_cast<size_t>(kRayMax)) break;
    } while (pos < traced.size());
    return best;
}

}  // namespace detail

// tracer.cpp:115-127
inline std::vector<TracedKernel> fine_select(std::vector<TracedKernel> traced, const SelectionConfig& cfg) {
    cfg.validate();
    return detail::device_select(traced, cfg.eta, static_cast<size_t>(cfg.k_prime));
}

// ---------------------------------------------------------------- blender.hpp

namespace detail {

inline void split(const TracedKernel* t, size_t n, std::vector<int32_t>& idx, std::vector<double>& l,
                  std::vector<double>& q, std::vector<double>& s) {
    idx.resize(n);
    l.resize(n);
    q.resize(n);
    s.resize(n);
    for (size_t i = 0; i < n; ++i) {
        idx[i] = t[i].kernel_index;
        l[i] = t[i].l;
        q[i] = t[i].q;
        s[i] = t[i].sigma;
    }
}

inline double transmittance_at(const TracedKernel* traced, size_t n, double tau, double t) {
    std::vector<int32_t> idx;
    std::vector<double> l, q, s;
    split(traced, n, idx, l, q, s);
    double out = 0.0;
    check(gvr_transmittance_ray(context(), static_cast<int32_t>(n), l.data(), q.data(), s.data(), tau, 1, &t, &out));
    return out;
}

inline RayBlend blend(const TracedKernel* traced, size_t n, double tau) {
    std::vector<int32_t> idx, oidx(n + 1);
    std::vector<double> l, q, s, w(n + 1);
    split(traced, n, idx, l, q, s);
    RayBlend out;
    check(gvr_blend_ray(context(), static_cast<int32_t>(n), idx.data(), l.data(), q.data(), s.data(), tau, oidx.data(),
                        w.data(), &out.alpha));
    for (size_t k = 0; k < n; ++k) out.weights.emplace_back(oidx[k], w[k]);
    return out;
}

}  // namespace detail

#if __cplusplus >= 202002L
// blender.cpp:19-25
inline double transmittance_at(std::span<const TracedKernel> traced, double tau, double t) {
    return detail::transmittance_at(traced.data(), traced.size(), tau, t);
}
// blender.cpp:27-53
inline RayBlend blend(std::span<const TracedKernel> traced, double tau) {
    return detail::blend(traced.data(), traced.size(), tau);
}
#else
inline double transmittance_at(const std::vector<TracedKernel>& traced, double tau, double t) {
    return detail::transmittance_at(traced.data(), traced.size(), tau, t);
}
inline RayBlend blend(const std::vector<TracedKernel>& traced, double tau) {
    return detail::blend(traced.data(), traced.size(), tau);
}
#endif

// blender.cpp:55-62
inline std::vector<std::pair<int, double>> normalized_weights(const RayBlend& b, double eps = 1e-8) {
    const size_t n = b.weights.size();
    std::vector<double> w(n), out(n);
    for (size_t i = 0; i < n; ++i) w[i] = b.weights[i].second;
    detail::check(gvr_normalized_weights_ray(detail::context(), static_cast<int32_t>(n), w.data(), eps, out.data()));
    auto res = b.weights;
    for (size_t i = 0; i < n; ++i) res[i].second = out[i];
    return res;
}

namespace detail {

// blender.cpp:66-137: the whole render on the device (gvr_render); weight_store,
// the taped selection and the camera-space scene are copied out on request.
inline RenderBuffers render_device(const GaussianScene& scene, const Camera& camera, const SelectionConfig& cfg,
                                   std::shared_ptr<SceneHandle>* scene_out, std::shared_ptr<TapeHandle>* tape_out) {
    auto dscene = upload(scene);  // scene.validate() (render_core validates it first)
    auto dtape = std::make_shared<TapeHandle>();
    gvr_context* c = dtape->owner->ctx;
    const int h = camera.height, w = camera.width, dc = std::max(scene.attr_dim(), 1);
    const size_t p = static_cast<size_t>(std::max(h, 0)) * std::max(w, 0), kp = std::max(cfg.k_prime, 0);
    RenderBuffers b;
    b.image = Image(h, w, dc, ChannelSemantics::Color);
    b.alpha = Image(h, w, 1, ChannelSemantics::Alpha);
    b.depth = Image(h, w, 1, ChannelSemantics::Feature);
    std::vector<int32_t> idx(p * kp);
    std::vector<double> wts(p * kp);
    const gvr_camera cc = to_c(camera);
    const gvr_selection sc = to_c(cfg);
    const gvr_render_outputs out{b.image.data.data(), b.alpha.data.data(), b.depth.data.data(), idx.data(), wts.data()};
    check(gvr_render(c, dscene->s, &cc, &sc, dtape->t, &out), c);
    b.weight_store.assign(p, {});
    for (size_t i = 0; i < p; ++i)
        for (size_t k = 0; k < kp && idx[i * kp + k] >= 0; ++k) b.weight_store[i].emplace_back(idx[i * kp + k], wts[i * kp + k]);
    if (scene_out) *scene_out = dscene;
    if (tape_out) *tape_out = dtape;
    return b;
}

inline GaussianScene cam_scene_of(const GaussianScene& scene, const std::shared_ptr<TapeHandle>& tape) {
    const size_t k = scene.kernels.size();
    std::vector<double> c(3 * k + 3), s(9 * k + 9);
    check(gvr_tape_cam_scene(tape->owner->ctx, tape->t, c.data(), s.data()), tape->owner->ctx);
    GaussianScene out = scene;
    for (size_t i = 0; i < k; ++i) {
        out.kernels[i].center = Vec3(c[3 * i], c[3 * i + 1], c[3 * i + 2]);
        for (int r = 0; r < 3; ++r)
            for (int t = 0; t < 3; ++t) out.kernels[i].inv_cov(r, t) = s[9 * i + 3 * r + t];
    }
    return out;
}

// blender.hpp:53-56
inline RenderBuffers render_core(const GaussianScene& scene, const Camera& camera, const SelectionConfig& cfg,
                                 int threads, std::vector<std::vector<TracedKernel>>* traced_out,
                                 GaussianScene* cam_scene_out) {
    (void)threads;
    std::shared_ptr<TapeHandle> tape;
    RenderBuffers b = render_device(scene, camera, cfg, nullptr, &tape);
    if (traced_out) {
        TracedStore st;
        st.tape = tape;
        st.pixels = static_cast<size_t>(camera.height) * camera.width;
        st.k_prime = static_cast<size_t>(cfg.k_prime);
        *traced_out = st.get();
    }
    if (cam_scene_out) *cam_scene_out = cam_scene_of(scene, tape);
    return b;
}

}  // namespace detail

// grad.hpp:41-42 / grad.cpp:38-47
inline ForwardResult render_with_tape(const GaussianScene& scene, const Camera& camera, const SelectionConfig& cfg,
                                      int threads = 0) {
    ForwardResult fr;
    fr.tape.scene = scene;
    fr.tape.camera = camera;
    fr.tape.cfg = cfg;
    fr.tape.threads = threads;
    fr.buffers = detail::render_device(scene, camera, cfg, &fr.tape.device_scene, &fr.tape.device_tape);
    fr.tape.cam_scene = detail::cam_scene_of(scene, fr.tape.device_tape);
    auto st = std::make_shared<detail::TracedStore>();
    st->tape = fr.tape.device_tape;
    st->pixels = static_cast<size_t>(camera.height) * camera.width;
    st->k_prime = static_cast<size_t>(cfg.k_prime);
    fr.tape.traced.store_ = st;
    return fr;
}

// blender.hpp:40-41
inline RenderBuffers render(const GaussianScene& scene, const Camera& camera, const SelectionConfig& cfg,
                            int threads = 0) {
    (void)threads;
    return detail::render_device(scene, camera, cfg, nullptr, nullptr);
}

// grad.hpp:53-54 / grad.cpp:49-199 (gvr_backward; bit-deterministic)
inline GradientBundle backward(const Tape& tape, const Image& d_image, const Image& d_alpha,
                               const GradFlags& flags = {}) {
    const int h = tape.camera.height, w = tape.camera.width, dim = tape.scene.attr_dim(), k = tape.scene.size();
    if (d_image.height != h || d_image.width != w || d_image.channels != dim || d_alpha.height != h ||
        d_alpha.width != w || d_alpha.channels != 1)
        throw ValidationError("backward: d_image shape does not match the forward render");
    if (!tape.device_tape) throw std::runtime_error("gvr: backward needs a tape made by render_with_tape");
    gvr_context* c = tape.device_tape->owner->ctx;
    std::vector<double> dc(3 * static_cast<size_t>(k)), ds(9 * static_cast<size_t>(k)),
        da(static_cast<size_t>(dim) * k), dr(9), dt(3);
    const gvr_grad_flags f{flags.through_transmittance ? 1 : 0, flags.through_density ? 1 : 0};
    const gvr_gradients out{dc.data(), ds.data(), dim > 0 ? da.data() : nullptr, dr.data(), dt.data()};
    detail::check(gvr_backward(c, tape.device_tape->t, dim > 0 ? d_image.data.data() : nullptr, d_alpha.data.data(), &f,
                               &out),
                  c);
    GradientBundle g;
    g.init(k, dim);
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

// grad.hpp:62-70 / grad.cpp:201-216 (gvr_scalar_loss_buffers on the device)
struct ScalarLoss {
    Image target_image;
    Image target_alpha;
    double w_image = 1.0;
    double w_alpha = 1.0;

    double value(const RenderBuffers& buf, Image* d_image, Image* d_alpha) const {
        if (target_image.data.size() < buf.image.data.size() || target_alpha.data.size() < buf.alpha.data.size())
            throw ValidationError("ScalarLoss: target size does not match the render");
        if (d_image) *d_image = Image(buf.image.height, buf.image.width, buf.image.channels);
        if (d_alpha) *d_alpha = Image(buf.alpha.height, buf.alpha.width, 1, ChannelSemantics::Alpha);
        double loss = 0.0;
        detail::check(gvr_scalar_loss_buffers(
            detail::context(), static_cast<int64_t>(buf.image.data.size()), buf.image.data.data(),
            target_image.data.data(), static_cast<int64_t>(buf.alpha.data.size()), buf.alpha.data.data(),
            target_alpha.data.data(), w_image, w_alpha, &loss, d_image ? d_image->data.data() : nullptr,
            d_alpha ? d_alpha->data.data() : nullptr));
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
    gvr_context* c = dscene->owner->ctx;
    const int k = scene.size(), dim = observed.channels;
    std::vector<double> a(static_cast<size_t>(k) * dim), sp(k);
    std::vector<uint8_t> m(k);
    const gvr_camera cc = detail::to_c(camera);
    const gvr_selection sc = detail::to_c(cfg);
    detail::check(gvr_sample_attributes(c, dscene->s, &cc, &sc, observed.data.data(), observed.height, observed.width,
                                        dim, normalized ? 1 : 0, a.data(), sp.data(), m.data()),
                  c);
    SampledAttributes out;
    out.attrs.assign(k, VecX::Zero(dim));
    out.support = sp;
    out.masked.assign(k, false);
    for (int i = 0; i < k; ++i) {
        for (int ch = 0; ch < dim; ++ch) out.attrs[i][ch] = a[static_cast<size_t>(dim) * i + ch];
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

// ---------------------------------------------------------------- per-pixel helpers over a tape

// transmittance_at (blender.hpp:29) for every pixel of a taped render: T(t(i,j))
// over that pixel's selected kernels (the per-ray form, batched on the device).
inline Image transmittance_at(const Tape& tape, const Image& t) {
    if (t.height != tape.camera.height || t.width != tape.camera.width || t.channels != 1)
        throw ValidationError("transmittance_at: depth image shape does not match the forward render");
    Image out(t.height, t.width, 1, ChannelSemantics::Feature);
    gvr_context* c = tape.device_tape->owner->ctx;
    detail::check(gvr_tape_transmittance(c, tape.device_tape->t, t.data.data(), out.data.data()), c);
    return out;
}

// normalized_weights (blender.hpp:36) of every pixel's weight_store, same layout.
inline std::vector<std::vector<std::pair<int, double>>> normalized_weights(const ForwardResult& fr,
                                                                           double eps = 1e-8) {
    const size_t p = fr.buffers.weight_store.size(), kp = static_cast<size_t>(fr.tape.cfg.k_prime);
    std::vector<double> nw(p * kp);
    gvr_context* c = fr.tape.device_tape->owner->ctx;
    detail::check(gvr_tape_normalized_weights(c, fr.tape.device_tape->t, eps, nw.data()), c);
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

// ---------------------------------------------------------------- so3.hpp (pose parameter maps)

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
inline void hat_raw(const double v[3], double h[9]) {
    const double t[9] = {0, -v[2], v[1], v[2], 0, -v[0], -v[1], v[0], 0};
    std::memcpy(h, t, sizeof t);
}
inline void so3_exp_gradient_raw(const double w[3], const double dr[9], double g[3]) {
    const double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
    double r[9];
    so3_exp_raw(w, r);
    for (int i = 0; i < 3; ++i) {
        double e[3] = {0, 0, 0};
        e[i] = 1.0;
        double d[9];
        if (th2 < 1e-16) {
            hat_raw(e, d);
        } else {
            double ire[3];  // (I - R) e
            for (int a = 0; a < 3; ++a) ire[a] = e[a] - r[3 * a + i];
            const double v[3] = {w[1] * ire[2] - w[2] * ire[1], w[2] * ire[0] - w[0] * ire[2], w[0] * ire[1] - w[1] * ire[0]};
            double hw[9], hv[9], m[9];
            hat_raw(w, hw);
            hat_raw(v, hv);
            for (int a = 0; a < 9; ++a) m[a] = (w[i] * hw[a] + hv[a]) / th2;
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) d[3 * a + b] = m[3 * a] * r[b] + m[3 * a + 1] * r[3 + b] + m[3 * a + 2] * r[6 + b];
        }
        double acc = 0.0;
        for (int a = 0; a < 9; ++a) acc += dr[a] * d[a];
        g[i] = acc;
    }
}
inline void vec_raw(const Vec3& v, double o[3]) {
    for (int i = 0; i < 3; ++i) o[i] = v[i];
}
inline void mat_raw(const Mat3& m, double o[9]) {
    for (int i = 0; i < 9; ++i) o[i] = m(i / 3, i % 3);
}
inline Mat3 mat_of(const double r[9]) {
    Mat3 m = Mat3::Identity();
    for (int i = 0; i < 9; ++i) m(i / 3, i % 3) = r[i];
    return m;
}
}  // namespace detail

// so3.cpp:7-13
inline Mat3 so3_hat(const Vec3& w) {
    double v[3], h[9];
    detail::vec_raw(w, v);
    detail::hat_raw(v, h);
    return detail::mat_of(h);
}
// so3.cpp:15-24
inline Mat3 so3_exp(const Vec3& w) {
    double v[3], r[9];
    detail::vec_raw(w, v);
    detail::so3_exp_raw(v, r);
    return detail::mat_of(r);
}
// so3.cpp:26-47
inline Vec3 so3_log(const Mat3& r) {
    double m[9], w[3];
    detail::mat_raw(r, m);
    detail::so3_log_raw(m, w);
    return Vec3(w[0], w[1], w[2]);
}
// so3.cpp:49-65
inline Vec3 so3_exp_gradient(const Vec3& w, const Mat3& d_rotation) {
    double v[3], dr[9], g[3];
    detail::vec_raw(w, v);
    detail::mat_raw(d_rotation, dr);
    detail::so3_exp_gradient_raw(v, dr, g);
    return Vec3(g[0], g[1], g[2]);
}
// so3.cpp:67-73: grad_i = sum(d_rotation .* (hat(e_i) R))
inline Vec3 so3_tangent_gradient(const Mat3& d_rotation, const Mat3& r) {
    double g[3];
    for (int i = 0; i < 3; ++i) {
        double e[3] = {0, 0, 0}, h[9];
        e[i] = 1.0;
        detail::hat_raw(e, h);
        double acc = 0.0;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double hr = 0.0;
                for (int t = 0; t < 3; ++t) hr += h[3 * a + t] * r(t, b);
                acc += d_rotation(a, b) * hr;
            }
        g[i] = acc;
    }
    return Vec3(g[0], g[1], g[2]);
}

// ---------------------------------------------------------------- parallel.hpp

// parallel.hpp:12-20: GVR_THREADS > requested > hardware threads.
inline int resolve_threads(int requested) {
    if (const char* env = std::getenv("GVR_THREADS")) {
        const int n = std::atoi(env);
        if (n > 0) return n;
    }
    if (requested > 0) return requested;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw > 0 ? static_cast<int>(hw) : 1;
}

// parallel.hpp:22-43: fn(worker, begin, end) over contiguous partitions of
// [0, count); the render path itself runs on the GPU and never calls it.
template <typename Fn>
void parallel_for_partitions(int count, int workers, const Fn& fn) {
    workers = std::max(1, std::min(workers, count));
    if (workers <= 1) {
        if (count > 0) fn(0, 0, count);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(static_cast<size_t>(workers));
    const int base = count / workers, extra = count % workers;
    for (int w = 0, begin = 0; w < workers; ++w) {
        const int len = base + (w < extra ? 1 : 0);
        pool.emplace_back(fn, w, begin, begin + len);
        begin += len;
    }
    for (auto& t : pool) t.join();
}

// ---------------------------------------------------------------- gradcheck (grad.hpp:67-88)

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
