// The reference's hot-path test cases, ported onto the C++ drop-in
// (include/gvr/gvr.hpp -> libgvr_cuda.so). Each case cites the reference test
// it follows; assertions keep the reference's form (exact equalities stay exact).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include "gvr/gvr.hpp"

#include <cmath>
#include <random>

using namespace gvr;

namespace {

Camera default_camera(int size = 32, double focal = 16.0) {  // tests/oracles.hpp:153-161
    Camera c;
    c.height = c.width = size;
    c.focal = focal;
    c.oy = c.ox = (size - 1) / 2.0;
    return c;
}

GaussianKernel isotropic(double x, double y, double z, double sigma, VecX attr) {
    GaussianKernel k;
    k.center = Vec3(x, y, z);
    k.inv_cov = Mat3::Identity();
    for (int i = 0; i < 3; ++i) k.inv_cov(i, i) = 1.0 / (sigma * sigma);
    k.attr = attr;
    return k;
}

GaussianScene random_scene(std::mt19937_64& rng, int count) {  // analogue of oracle::random_scene
    std::uniform_real_distribution<double> xy(-1.0, 1.0), zd(3.0, 6.0), ch(0.0, 1.0), ev(2.0, 30.0);
    GaussianScene s;
    for (int k = 0; k < count; ++k) {
        GaussianKernel g;
        g.center = Vec3(xy(rng), xy(rng), zd(rng));
        g.inv_cov = Mat3::Zero();
        for (int i = 0; i < 3; ++i) g.inv_cov(i, i) = ev(rng);  // axis-aligned SPD
        g.attr = VecX{ch(rng), ch(rng), ch(rng)};
        s.kernels.push_back(g);
    }
    return s;
}

}  // namespace

TEST_CASE("single on-axis kernel blends to exp(-1/2)") {  // test_blender.cpp:52-58
    GaussianScene scene;
    scene.kernels.push_back(isotropic(0, 0, 5, 0.05, VecX{1, 1, 1}));
    Camera cam = default_camera(1, 10.0);
    cam.ox = cam.oy = 0.0;
    const RenderBuffers buf = render(scene, cam, SelectionConfig{}, 1);
    REQUIRE(buf.weight_store[0].size() == 1);
    CHECK(buf.weight_store[0][0].second == doctest::Approx(std::exp(-0.5)));
    CHECK(buf.alpha.at(0, 0, 0) == doctest::Approx(1.0 - std::exp(-1.0)));
}

TEST_CASE("kernel on the ray axis peaks at its depth") {  // test_tracer.cpp:24-31
    GaussianScene scene;
    scene.kernels.push_back(isotropic(0, 0, 5, 0.7, VecX{0, 0, 0}));
    Camera cam = default_camera(1, 10.0);
    cam.ox = cam.oy = 0.0;
    const ForwardResult fr = render_with_tape(scene, cam, SelectionConfig{}, 1);
    const auto& traced = fr.tape.traced.get();
    REQUIRE(traced[0].size() == 1);
    CHECK(traced[0][0].l == doctest::Approx(5.0));
    CHECK(traced[0][0].q == doctest::Approx(0.0));
    CHECK(traced[0][0].sigma == doctest::Approx(0.7));
}

TEST_CASE("empty scene renders to zeros") {  // test_blender.cpp:213-219
    GaussianScene scene;
    const RenderBuffers buf = render(scene, default_camera(), SelectionConfig{}, 1);
    for (double v : buf.image.data) CHECK(v == 0.0);
    for (double v : buf.alpha.data) CHECK(v == 0.0);
}

TEST_CASE("the image is exactly the weight_store blended with attributes") {  // test_blender.cpp:247-261
    std::mt19937_64 rng(55);
    const GaussianScene scene = random_scene(rng, 20);
    const Camera cam = default_camera();
    const RenderBuffers buf = render(scene, cam, SelectionConfig{}, 1);
    for (int i = 0; i < cam.height; ++i)
        for (int j = 0; j < cam.width; ++j) {
            double acc[3] = {0, 0, 0};
            for (const auto& [k, w] : buf.weight_store[static_cast<size_t>(i) * cam.width + j])
                for (int c = 0; c < 3; ++c) acc[c] = acc[c] + w * scene.kernels[k].attr[c];
            for (int c = 0; c < 3; ++c) CHECK(buf.image.at(i, j, c) == acc[c]);
        }
}

TEST_CASE("renders are identical across calls") {  // test_blender.cpp:284-292 (thread counts)
    std::mt19937_64 rng(57);
    const GaussianScene scene = random_scene(rng, 30);
    const Camera cam = default_camera(40, 20.0);
    const RenderBuffers a = render(scene, cam, SelectionConfig{}, 1);
    const RenderBuffers b = render(scene, cam, SelectionConfig{}, 4);
    CHECK(a.image.data == b.image.data);
    CHECK(a.alpha.data == b.alpha.data);
}

TEST_CASE("zero upstream gradient gives a zero bundle") {  // test_grad.cpp:24-39
    std::mt19937_64 rng(61);
    const GaussianScene scene = random_scene(rng, 4);
    const Camera cam = default_camera();
    const ForwardResult fr = render_with_tape(scene, cam, SelectionConfig{}, 1);
    const Image d_image(cam.height, cam.width, 3);
    const Image d_alpha(cam.height, cam.width, 1, ChannelSemantics::Alpha);
    const GradientBundle g = backward(fr.tape, d_image, d_alpha);
    for (int k = 0; k < scene.size(); ++k)
        for (int t = 0; t < 3; ++t) {
            CHECK(g.d_center[k][t] == 0.0);
            CHECK(g.d_attr[k][t] == 0.0);
        }
    CHECK(g.d_translation[0] == 0.0);
}

TEST_CASE("backward rejects mismatched shapes") {  // test_grad.cpp:41-49
    std::mt19937_64 rng(62);
    const GaussianScene scene = random_scene(rng, 2);
    const Camera cam = default_camera();
    const ForwardResult fr = render_with_tape(scene, cam, SelectionConfig{}, 1);
    const Image wrong(cam.height + 1, cam.width, 3);
    const Image d_alpha(cam.height, cam.width, 1, ChannelSemantics::Alpha);
    CHECK_THROWS_AS(backward(fr.tape, wrong, d_alpha), ValidationError);
}

TEST_CASE("attribute gradients equal weights summed against the upstream image") {  // test_grad.cpp:133-156
    std::mt19937_64 rng(66);
    const GaussianScene scene = random_scene(rng, 6);
    const Camera cam = default_camera();
    const ForwardResult fr = render_with_tape(scene, cam, SelectionConfig{}, 1);
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    ScalarLoss loss;
    loss.target_image = Image(cam.height, cam.width, 3);
    loss.target_alpha = Image(cam.height, cam.width, 1, ChannelSemantics::Alpha);
    for (auto& v : loss.target_image.data) v = uni(rng);
    for (auto& v : loss.target_alpha.data) v = uni(rng);
    Image d_image, d_alpha;
    loss.value(fr.buffers, &d_image, &d_alpha);
    d_alpha.data.assign(d_alpha.data.size(), 0.0);
    const GradientBundle g = backward(fr.tape, d_image, d_alpha);
    std::vector<double> expected(scene.size() * 3, 0.0);
    for (int i = 0; i < cam.height; ++i)
        for (int j = 0; j < cam.width; ++j)
            for (const auto& [k, w] : fr.buffers.weight_store[static_cast<size_t>(i) * cam.width + j])
                for (int c = 0; c < 3; ++c) expected[3 * k + c] += w * d_image.at(i, j, c);
    for (int k = 0; k < scene.size(); ++k)
        for (int c = 0; c < 3; ++c) CHECK(std::abs(g.d_attr[k][c] - expected[3 * k + c]) < 1e-12);
}

TEST_CASE("scene validation catches broken kernels") {  // test_scene.cpp:156-183
    GaussianScene scene;
    scene.kernels.push_back(isotropic(0, 0, 4, 1.0, VecX{0, 0, 0}));
    SUBCASE("asymmetric inv_cov") {
        scene.kernels[0].inv_cov(0, 1) = 0.5;
        CHECK_THROWS_AS(render(scene, default_camera(), SelectionConfig{}), ValidationError);
    }
    SUBCASE("non positive-definite inv_cov") {
        scene.kernels[0].inv_cov(2, 2) = -1.0;
        CHECK_THROWS_AS(render(scene, default_camera(), SelectionConfig{}), ValidationError);
    }
    SUBCASE("mixed attribute dimensions") {
        GaussianKernel other = scene.kernels[0];
        other.attr = VecX{0, 0};
        scene.kernels.push_back(other);
        CHECK_THROWS_AS(render(scene, default_camera(), SelectionConfig{}), ValidationError);
    }
    SUBCASE("negative tau") {
        scene.tau = -0.5;
        CHECK_THROWS_AS(render(scene, default_camera(), SelectionConfig{}), ValidationError);
    }
}

TEST_CASE("camera validation") {  // test_scene.cpp:83-89 (non-orthonormal rotation), types.cpp:44-63
    Camera cam = default_camera();
    CHECK_NOTHROW(cam.validate());
    cam.rotation(0, 0) = 2.0;
    CHECK_THROWS_WITH_AS(cam.validate(), "camera rotation is not orthonormal", ValidationError);
    cam = default_camera();
    cam.rotation(0, 0) = -1.0;  // reflection: orthonormal, det = -1
    CHECK_THROWS_WITH_AS(cam.validate(), "camera rotation determinant is not +1", ValidationError);
    cam = default_camera();
    cam.focal = 0.0;
    CHECK_THROWS_AS(cam.validate(), ValidationError);
    cam = default_camera();
    cam.height = 0;
    CHECK_THROWS_AS(cam.validate(), ValidationError);
    cam = default_camera();
    cam.translation[1] = std::nan("");
    CHECK_THROWS_AS(cam.validate(), ValidationError);
}

TEST_CASE("selection config validation") {  // test_tracer.cpp:252-259
    GaussianScene scene;
    scene.kernels.push_back(isotropic(0, 0, 4, 1.0, VecX{0, 0, 0}));
    SelectionConfig cfg;
    cfg.eta = 1.0;
    CHECK_THROWS_AS(render(scene, default_camera(), cfg), ValidationError);
    cfg.eta = 0.01;
    cfg.k_prime = 0;
    CHECK_THROWS_AS(render(scene, default_camera(), cfg), ValidationError);
}

TEST_CASE("sampling a constant image recovers the constant") {  // test_sampler.cpp:71-82
    std::mt19937_64 rng(5);
    const GaussianScene scene = random_scene(rng, 150);
    const Camera cam = default_camera(48, 48.0);
    Image observed(48, 48, 3);
    for (auto& v : observed.data) v = 0.7;
    const SampledAttributes attrs = sample_attributes(observed, scene, cam, SelectionConfig{});
    int tested = 0;
    for (size_t k = 0; k < attrs.attrs.size(); ++k) {
        if (attrs.masked[k]) continue;
        ++tested;
        for (int c = 0; c < 3; ++c) CHECK(attrs.attrs[k][c] == doctest::Approx(0.7).epsilon(1e-9));
    }
    CHECK(tested > 20);
}

TEST_CASE("sampling weights are exactly the rendering weights") {  // test_sampler.cpp:162-176
    std::mt19937_64 rng(6);
    const GaussianScene scene = random_scene(rng, 120);
    const Camera cam = default_camera(40, 40.0);
    const RenderBuffers buf = render(scene, cam, SelectionConfig{}, 1);
    std::vector<double> support(scene.size(), 0.0);
    for (const auto& ws : buf.weight_store)
        for (const auto& [k, w] : ws) support[k] += w;
    Image observed(cam.height, cam.width, 3);
    const SampledAttributes attrs = sample_attributes(observed, scene, cam, SelectionConfig{});
    for (int k = 0; k < scene.size(); ++k) CHECK(attrs.support[k] == doctest::Approx(support[k]).epsilon(1e-12));
}

TEST_CASE("zeroed attributes render black") {  // test_sampler.cpp:131-143
    std::mt19937_64 rng(7);
    const GaussianScene scene = random_scene(rng, 100);
    SampledAttributes attrs;
    attrs.attrs.assign(scene.size(), VecX::Zero(3));
    attrs.support.assign(scene.size(), 1.0);
    attrs.masked.assign(scene.size(), false);
    const RenderBuffers buf = resynthesize(attrs, scene, default_camera(32, 32.0), SelectionConfig{}, 1);
    for (double v : buf.image.data) CHECK(v == 0.0);
}

TEST_CASE("sampler size checks") {  // test_sampler.cpp:190-205
    std::mt19937_64 rng(8);
    const GaussianScene scene = random_scene(rng, 50);
    const Camera cam = default_camera(32, 32.0);
    Image observed(16, 16, 3);
    CHECK_THROWS_AS(sample_attributes(observed, scene, cam, SelectionConfig{}), ValidationError);
    SampledAttributes attrs;
    attrs.attrs.assign(10, VecX::Zero(3));
    attrs.support.assign(10, 1.0);
    attrs.masked.assign(10, false);
    CHECK_THROWS_AS(resynthesize(attrs, scene, cam, SelectionConfig{}), ValidationError);
}

TEST_CASE("normalized weights and transmittance of a taped render") {  // test_blender.cpp:11-21, 197-211
    GaussianScene scene;
    scene.kernels.push_back(isotropic(0, 0, 5, 0.8, VecX{1, 1, 1}));
    Camera cam = default_camera(1, 10.0);
    cam.ox = cam.oy = 0.0;
    const ForwardResult fr = render_with_tape(scene, cam, SelectionConfig{}, 1);
    Image t(1, 1, 1);
    t.data[0] = -100.0;
    CHECK(transmittance_at(fr.tape, t).data[0] == doctest::Approx(1.0));
    t.data[0] = 5.0 + 60 * 0.8;
    CHECK(transmittance_at(fr.tape, t).data[0] == doctest::Approx(std::exp(-1.0)));
    const auto nw = normalized_weights(fr);
    REQUIRE(nw[0].size() == 1);
    CHECK(nw[0][0].second == doctest::Approx(1.0));
}

TEST_CASE("lambert shading basics") {  // test_blender.cpp:294-320
    Image normals(1, 2, 3, ChannelSemantics::Normal);
    Image alpha(1, 2, 1, ChannelSemantics::Alpha);
    Image depth(1, 2, 1, ChannelSemantics::Feature);
    normals.at(0, 0, 2) = -1.0;
    normals.at(0, 1, 0) = 1.0;
    alpha.at(0, 0, 0) = 1.0;
    alpha.at(0, 1, 0) = 1.0;
    depth.at(0, 0, 0) = 4.0;
    depth.at(0, 1, 0) = 4.0;
    Camera cam = default_camera(1, 8.0);
    cam.width = 2;
    cam.ox = 0.0;
    cam.oy = 0.0;
    const Image lit = shade_lambert(normals, alpha, depth, cam, Vec3(0, 0, -10), Vec3(1, 1, 1));
    CHECK(lit.at(0, 0, 0) == doctest::Approx(1.0).epsilon(1e-3));
    CHECK(lit.at(0, 1, 0) == doctest::Approx(0.0).epsilon(1e-2));
    alpha.at(0, 0, 0) = 0.0;
    const Image masked = shade_lambert(normals, alpha, depth, cam, Vec3(0, 0, -10), Vec3(1, 1, 1));
    CHECK(masked.at(0, 0, 0) == 0.0);
    Image bad(1, 2, 2);
    CHECK_THROWS_AS(shade_lambert(bad, alpha, depth, cam, Vec3(0, 0, -10), Vec3(1, 1, 1)), ValidationError);
}

TEST_CASE("gradcheck passes on random five-kernel scenes") {  // test_grad.cpp:95-110
    std::mt19937_64 rng(64);
    std::uniform_real_distribution<double> u01(0.0, 1.0);
    for (int trial = 0; trial < 2; ++trial) {
        const GaussianScene scene = random_scene(rng, 5);
        Camera cam = default_camera(24, 12.0);
        cam.translation = Vec3(0.02, 0.01, 0.1);
        ScalarLoss loss;
        loss.target_image = Image(24, 24, 3);
        loss.target_alpha = Image(24, 24, 1, ChannelSemantics::Alpha);
        for (auto& v : loss.target_image.data) v = u01(rng);
        for (auto& v : loss.target_alpha.data) v = u01(rng);
        const GradCheckReport report = gradcheck(scene, cam, SelectionConfig{}, loss, 1e-4, 1e-3, 1);
        CHECK(report.max_rel_err < 1e-3);
        CHECK(report.total_checked > 0);
    }
}
