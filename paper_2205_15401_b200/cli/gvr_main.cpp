// gvr — command-line front end of the GPU backend (the reference's tools/gvr_main.cpp
// interface: subcommands, flags, output files, messages and exit codes), built on the
// C++ drop-in (include/gvr/*.hpp -> libgvr_cuda.so). Every render, loss, backward
// and sampling step runs on the GPU.
//
//   render           gvr_main.cpp:111-137    extract-texture  gvr_main.cpp:434-449
//   bench            gvr_main.cpp:154-186    rerender         gvr_main.cpp:451-466
//   gradcheck        gvr_main.cpp:188-223    fit-translation  gvr_main.cpp:271-352
//                                            fit-pose         gvr_main.cpp:354-432
// The converters (convert: OBJ/PLY -> scene) and fit-shape (whose initial scene is
// an icosphere through the mesh converter) are not part of this backend's CLI: they
// exit 1 with a message (the device shape-fitting loop is the Python Fitter,
// paper_2205_15401_b200/fit.py, and gvr::fit_shape in include/gvr/fit.hpp).
//
// Exit codes: 0 ok, 1 runtime error, 2 usage / validation error (gvr_main.cpp:19-21, 612-621).
#include "gvr/fit.hpp"
#include "gvr/image_io.hpp"
#include "gvr/scene_io.hpp"

#include <chrono>
#include <cstdio>
#include <filesystem>
#include <iostream>
#include <map>
#include <random>
#include <set>
#include <string>
#include <vector>

namespace fs = std::filesystem;

namespace {

constexpr int kExitOk = 0;
constexpr int kExitRuntime = 1;
constexpr int kExitUsage = 2;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void require_file(const fs::path& path, const std::string& what) {
    if (!fs::exists(path)) throw UsageError(what + " file does not exist: " + path.string());
}

nlohmann::json load_config(const fs::path& path) {
    require_file(path, "config");
    std::ifstream in(path);
    nlohmann::json j;
    try {
        in >> j;
    } catch (const nlohmann::json::exception& e) {
        throw UsageError("invalid JSON in " + path.string() + ": " + e.what());
    }
    return j;
}

// gvr_main.cpp:46-66
gvr::SelectionConfig selection_from_json(const nlohmann::json& j) {
    gvr::SelectionConfig sel;
    if (j.contains("selection")) {
        const auto& s = j.at("selection");
        sel.eta = s.value("eta", sel.eta);
        sel.k_prime = s.value("k_prime", sel.k_prime);
        sel.coarse_enabled = s.value("coarse", sel.coarse_enabled);
    }
    return sel;
}

gvr::LossSpec loss_from_json(const nlohmann::json& j) {
    gvr::LossSpec spec;
    if (j.contains("loss")) {
        const auto& l = j.at("loss");
        spec.rgb_weight = l.value("rgb", spec.rgb_weight);
        spec.silhouette_weight = l.value("silhouette", spec.silhouette_weight);
        spec.edge_weight = l.value("edge", spec.edge_weight);
        spec.laplacian_weight = l.value("laplacian", spec.laplacian_weight);
    }
    return spec;
}

// gvr_main.cpp:74-92
void write_report_json(const gvr::FitReport& report, const nlohmann::json& extra, const fs::path& path) {
    nlohmann::json j = extra;
    j["iterations"] = report.iterations;
    j["diverged"] = report.diverged;
    j["loss_trace"] = report.loss_trace;
    for (const auto& [key, value] : report.metrics) j["metrics"][key] = value;
    gvr::atomic_write_text(path, j.dump(2) + "\n");
}

void write_loss_csv(const gvr::FitReport& report, const fs::path& path) {
    std::string csv = "iteration,loss\n";
    for (size_t i = 0; i < report.loss_trace.size(); ++i)
        csv += std::to_string(i) + "," + std::to_string(report.loss_trace[i]) + "\n";
    gvr::atomic_write_text(path, csv);
}

// ---------------------------------------------------------------- flags

struct Args {
    std::string cmd;
    std::map<std::string, std::vector<std::string>> opt;
    std::set<std::string> flags;
    bool has(const std::string& k) const { return opt.count(k) > 0; }
    std::string str(const std::string& k, const std::string& def = "") const {
        auto it = opt.find(k);
        return it == opt.end() || it->second.empty() ? def : it->second.front();
    }
    double num(const std::string& k, double def) const {
        if (!has(k)) return def;
        try {
            return std::stod(str(k));
        } catch (const std::exception&) {
            throw UsageError("--" + k + ": not a number: " + str(k));
        }
    }
    std::vector<int> ints(const std::string& k) const {
        std::vector<int> out;
        if (has(k))
            for (const auto& v : opt.at(k)) {
                try {
                    out.push_back(std::stoi(v));
                } catch (const std::exception&) {
                    throw UsageError("--" + k + ": not an integer: " + v);
                }
            }
        return out;
    }
};

// Per subcommand: options taking values (multi-valued ones take every following
// non-flag token) and boolean flags; --threads and --seed are accepted anywhere.
Args parse(int argc, char** argv) {
    static const std::map<std::string, std::pair<std::set<std::string>, std::set<std::string>>> spec = {
        {"render", {{"scene", "camera", "out", "out-pfm", "alpha-pfm", "weights-pfm", "tau", "eta", "k-prime"},
                    {"no-coarse"}}},
        {"bench", {{"kernels", "sizes", "repeats", "out"}, {"no-coarse"}}},
        {"gradcheck", {{"scene", "camera", "fd-step", "tol", "out", "eta", "k-prime"}, {"no-coarse"}}},
        {"extract-texture", {{"image", "scene", "camera", "out", "eta", "k-prime"}, {"normalized", "no-coarse"}}},
        {"rerender", {{"attrs", "scene", "camera", "out", "out-pfm", "eta", "k-prime"}, {"no-coarse"}}},
        {"convert", {{"in", "out", "zeta", "flatten", "neighbors", "tau"}, {}}},
        {"fit-shape", {{"config", "out", "out-scene"}, {}}},
        {"fit-translation", {{"config", "out"}, {}}},
        {"fit-pose", {{"config", "out"}, {}}},
    };
    static const std::set<std::string> multi = {"kernels", "sizes"};
    Args a;
    if (argc < 2) throw UsageError("a subcommand is required: render, bench, gradcheck, extract-texture, rerender");
    a.cmd = argv[1];
    auto it = spec.find(a.cmd);
    if (it == spec.end()) throw UsageError("unknown subcommand: " + a.cmd);
    for (int i = 2; i < argc; ++i) {
        std::string tok = argv[i];
        if (tok.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + tok);
        std::string key = tok.substr(2), val;
        const size_t eq = key.find('=');
        const bool inline_val = eq != std::string::npos;
        if (inline_val) {
            val = key.substr(eq + 1);
            key = key.substr(0, eq);
        }
        const bool is_opt = it->second.first.count(key) || key == "threads" || key == "seed";
        const bool is_flag = it->second.second.count(key) > 0;
        if (!is_opt && !is_flag) throw UsageError("unknown option: --" + key);
        if (is_flag) {
            a.flags.insert(key);
            continue;
        }
        auto& vals = a.opt[key];
        if (inline_val) {
            vals.push_back(val);
            continue;
        }
        if (i + 1 >= argc) throw UsageError("--" + key + " needs a value");
        vals.push_back(argv[++i]);
        while (multi.count(key) && i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) vals.push_back(argv[++i]);
    }
    return a;
}

void require_opts(const Args& a, std::initializer_list<const char*> keys) {
    for (const char* k : keys)
        if (!a.has(k)) throw UsageError("--" + std::string(k) + " is required");
}

gvr::SelectionConfig selection(const Args& a) {
    gvr::SelectionConfig sel;
    sel.eta = a.num("eta", sel.eta);
    sel.k_prime = static_cast<int>(a.num("k-prime", sel.k_prime));
    sel.coarse_enabled = !a.flags.count("no-coarse");
    return sel;
}

// ---------------------------------------------------------------- bench scene (bench.cpp:9-24)

// make_bench_scene: the reference's unit cube surface grid at (0, 0, 4) (shapes.cpp:57-116,
// convert.cpp:90-130), restated from paper_2205_15401_b200/synthetic.py: welded lattice
// vertices in creation order, two triangles per cell, one isotropic kernel per vertex with
// sigma = mean_edge^2 / (4 ln 2).
gvr::GaussianScene make_bench_scene(int min_kernels) {
    int n = 1;
    while (6 * n * n + 2 < min_kernels) ++n;
    std::map<long long, int> id;
    std::vector<std::array<int, 3>> ijk;
    std::vector<std::array<int, 3>> faces;
    auto vertex = [&](int x, int y, int z) {
        const long long key = (static_cast<long long>(x) * (n + 1) + y) * (n + 1) + z;
        auto f = id.find(key);
        if (f != id.end()) return f->second;
        const int v = static_cast<int>(ijk.size());
        id.emplace(key, v);
        ijk.push_back({x, y, z});
        return v;
    };
    const int dudv[4][2] = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
    for (int axis = 0; axis < 3; ++axis) {
        const int u = (axis + 1) % 3, w = (axis + 2) % 3;
        for (int side = 0; side < 2; ++side)
            for (int p = 0; p < n; ++p)
                for (int q = 0; q < n; ++q) {
                    int v[4];
                    for (int c = 0; c < 4; ++c) {
                        int xyz[3];
                        xyz[axis] = side * n;
                        xyz[u] = p + dudv[c][0];
                        xyz[w] = q + dudv[c][1];
                        v[c] = vertex(xyz[0], xyz[1], xyz[2]);
                    }
                    if (side == 1) {
                        faces.push_back({v[0], v[1], v[2]});
                        faces.push_back({v[0], v[2], v[3]});
                    } else {
                        faces.push_back({v[0], v[2], v[1]});
                        faces.push_back({v[0], v[3], v[2]});
                    }
                }
    }
    const int nv = static_cast<int>(ijk.size());
    std::vector<double> pos(3 * static_cast<size_t>(nv));
    for (int i = 0; i < nv; ++i)
        for (int d = 0; d < 3; ++d) pos[3 * i + d] = (d == 2 ? 4.0 : 0.0) + (static_cast<double>(ijk[i][d]) / n - 0.5);
    std::set<std::pair<int, int>> edges;
    for (const auto& f : faces)
        for (int e = 0; e < 3; ++e) {
            const int a = f[e], b = f[(e + 1) % 3];
            if (a != b) edges.insert({std::min(a, b), std::max(a, b)});
        }
    std::vector<double> sum(nv, 0.0);
    std::vector<int> cnt(nv, 0);
    for (const auto& [a, b] : edges) {
        double sq[3];
        for (int d = 0; d < 3; ++d) {
            const double t = pos[3 * a + d] - pos[3 * b + d];
            sq[d] = t * t;
        }
        const double len = std::sqrt((sq[0] + sq[1]) + sq[2]);
        sum[a] += len;
        sum[b] += len;
        ++cnt[a];
        ++cnt[b];
    }
    gvr::GaussianScene scene;
    for (int i = 0; i < nv; ++i) {
        const double me = sum[i] / cnt[i];
        const double sigma = me * me / (4.0 * std::log(1.0 / 0.5));
        gvr::GaussianKernel k;
        k.center = gvr::Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]);
        k.inv_cov = gvr::Mat3::Identity();
        for (int d = 0; d < 3; ++d) k.inv_cov(d, d) = 1.0 / sigma;
        k.attr = gvr::VecX(3);
        k.attr[0] = 0.8;
        k.attr[1] = 0.3;
        k.attr[2] = 0.2;
        scene.kernels.push_back(k);
    }
    return scene;
}

gvr::Camera make_bench_camera(int s) {
    gvr::Camera c;
    c.focal = 1.6 * s;
    c.ox = c.oy = (s - 1) / 2.0;
    c.height = c.width = s;
    return c;
}

// ---------------------------------------------------------------- commands

int cmd_render(const Args& a) {
    require_opts(a, {"scene", "camera"});
    const fs::path scene_path = a.str("scene"), camera_path = a.str("camera");
    require_file(scene_path, "scene");
    require_file(camera_path, "camera");
    gvr::GaussianScene scene = gvr::load_scene_json(scene_path);
    const gvr::Camera camera = gvr::load_camera_json(camera_path);
    if (a.has("tau") && a.num("tau", -1.0) >= 0.0) scene.tau = a.num("tau", -1.0);
    const gvr::RenderBuffers buf = gvr::render(scene, camera, selection(a));
    if (a.has("out")) gvr::write_png(buf.image, a.str("out"));
    if (a.has("out-pfm")) gvr::write_pfm(buf.image, a.str("out-pfm"));
    if (a.has("alpha-pfm")) gvr::write_pfm(buf.alpha, a.str("alpha-pfm"));
    if (a.has("weights-pfm")) {
        gvr::Image wsum(camera.height, camera.width, 1, gvr::ChannelSemantics::Feature);
        for (size_t p = 0; p < buf.weight_store.size(); ++p) {
            double total = 0.0;
            for (const auto& kw : buf.weight_store[p]) total += kw.second;
            wsum.data[p] = total;
        }
        gvr::write_pfm(wsum, a.str("weights-pfm"));
    }
    return kExitOk;
}

int cmd_bench(const Args& a) {
    std::vector<int> kernels = a.ints("kernels"), sizes = a.ints("sizes");
    if (kernels.empty()) kernels = {1000, 4000, 16000};
    if (sizes.empty()) sizes = {128, 256, 512};
    const int repeats = static_cast<int>(a.num("repeats", 3));
    gvr::SelectionConfig sel;
    sel.coarse_enabled = !a.flags.count("no-coarse");
    nlohmann::json j;
    j["version"] = 1;
    j["coarse"] = sel.coarse_enabled;
    j["results"] = nlohmann::json::array();
    for (int kc : kernels) {
        const gvr::GaussianScene scene = make_bench_scene(kc);
        for (int s : sizes) {
            const gvr::Camera cam = make_bench_camera(s);
            const gvr::RenderBuffers warm = gvr::render(scene, cam, sel);
            size_t total = 0, peak = 0;
            for (const auto& ws : warm.weight_store) {
                total += ws.size();
                peak = std::max(peak, ws.size());
            }
            const auto t0 = std::chrono::steady_clock::now();
            for (int r = 0; r < repeats; ++r) (void)gvr::render(scene, cam, sel);
            const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            nlohmann::json jr;
            jr["kernel_count"] = scene.size();
            jr["image_size"] = s;
            jr["kernels_per_pixel_mean"] = static_cast<double>(total) / std::max<size_t>(warm.weight_store.size(), 1);
            jr["kernels_per_pixel_max"] = static_cast<double>(peak);
            jr["images_per_second"] = repeats / std::max(wall, 1e-12);
            jr["wall_seconds"] = wall;
            jr["repeats"] = repeats;
            j["results"].push_back(jr);
            std::cout << scene.size() << " kernels @ " << s << "x" << s << ": " << jr["images_per_second"].get<double>()
                      << " images/s (mean " << jr["kernels_per_pixel_mean"].get<double>() << " kernels/px)\n";
        }
    }
    if (a.has("out")) gvr::atomic_write_text(a.str("out"), j.dump(2) + "\n");
    return kExitOk;
}

int cmd_gradcheck(const Args& a) {
    require_opts(a, {"scene", "camera"});
    const fs::path scene_path = a.str("scene"), camera_path = a.str("camera");
    require_file(scene_path, "scene");
    require_file(camera_path, "camera");
    const gvr::GaussianScene scene = gvr::load_scene_json(scene_path);
    const gvr::Camera camera = gvr::load_camera_json(camera_path);
    const double h = a.num("fd-step", 1e-4), tol = a.num("tol", 1e-3);
    std::mt19937_64 rng(static_cast<uint64_t>(a.num("seed", 0)));
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    gvr::ScalarLoss loss;
    loss.target_image = gvr::Image(camera.height, camera.width, scene.attr_dim());
    loss.target_alpha = gvr::Image(camera.height, camera.width, 1, gvr::ChannelSemantics::Alpha);
    for (auto& v : loss.target_image.data) v = uni(rng);
    for (auto& v : loss.target_alpha.data) v = uni(rng);
    const gvr::GradCheckReport report = gvr::gradcheck(scene, camera, selection(a), loss, h, tol);
    nlohmann::json j;
    j["version"] = 1;
    j["h"] = h;
    j["tol"] = tol;
    j["max_rel_err"] = report.max_rel_err;
    j["total_checked"] = report.total_checked;
    j["total_skipped"] = report.total_skipped;
    for (const auto& [name, e] : report.per_class) {
        j["classes"][name] = {{"max_rel_err", e.max_rel_err}, {"checked", e.checked},
                              {"skipped_boundary", e.skipped_boundary}};
        std::cout << name << ": max rel err " << e.max_rel_err << " over " << e.checked << " params ("
                  << e.skipped_boundary << " skipped)\n";
    }
    if (a.has("out")) gvr::atomic_write_text(a.str("out"), j.dump(2) + "\n");
    const bool pass = report.passed(tol);
    std::cout << (pass ? "PASS" : "FAIL") << " max rel err " << report.max_rel_err << " (tol " << tol << ")\n";
    return pass ? kExitOk : kExitRuntime;
}

gvr::Image load_image_any(const fs::path& path) {
    require_file(path, "image");
    if (path.extension() == ".pfm") return gvr::read_pfm(path);
    return gvr::read_png(path);
}

int cmd_extract_texture(const Args& a) {
    require_opts(a, {"image", "scene", "camera"});
    const fs::path scene_path = a.str("scene"), camera_path = a.str("camera");
    require_file(scene_path, "scene");
    require_file(camera_path, "camera");
    const gvr::Image observed = load_image_any(a.str("image"));
    const gvr::GaussianScene scene = gvr::load_scene_json(scene_path);
    const gvr::Camera camera = gvr::load_camera_json(camera_path);
    const auto attrs = gvr::sample_attributes(observed, scene, camera, selection(a), a.flags.count("normalized") > 0);
    if (a.has("out")) gvr::save_attrs_json(attrs, a.str("out"));
    std::cout << "sampled " << attrs.attrs.size() << " kernels, " << attrs.masked_count() << " masked (support < "
              << gvr::kSupportEps << ")\n";
    return kExitOk;
}

int cmd_fit_translation(const Args& a) {
    require_opts(a, {"config"});
    const nlohmann::json cfg = load_config(a.str("config"));
    const auto sel = selection_from_json(cfg);
    const auto spec = loss_from_json(cfg);
    std::vector<gvr::GaussianScene> parts;
    for (const auto& jp : cfg.at("parts")) {
        const fs::path p = jp.get<std::string>();
        require_file(p, "part scene");
        parts.push_back(gvr::load_scene_json(p));
    }
    if (parts.empty()) throw UsageError("fit-translation needs at least one part");
    gvr::GaussianScene scene;
    scene.tau = parts.front().tau;
    std::vector<std::vector<int>> groups;
    for (const auto& part : parts) {
        std::vector<int> group;
        for (const auto& k : part.kernels) {
            group.push_back(scene.size());
            scene.kernels.push_back(k);
        }
        groups.push_back(std::move(group));
    }
    const fs::path camera_path = cfg.at("camera").get<std::string>();
    require_file(camera_path, "camera");
    gvr::FitView target;
    target.camera = gvr::load_camera_json(camera_path);
    std::vector<gvr::Vec3> gt(groups.size(), gvr::Vec3::Zero());
    if (cfg.contains("gt_offsets")) {
        const auto& jg = cfg.at("gt_offsets");
        for (size_t g = 0; g < groups.size() && g < jg.size(); ++g) {
            const auto v = jg[g].get<std::vector<double>>();
            gt[g] = gvr::Vec3(v[0], v[1], v[2]);
        }
    }
    if (cfg.contains("target_image")) {
        target.image = load_image_any(cfg.at("target_image").get<std::string>());
        target.alpha = gvr::Image(target.camera.height, target.camera.width, 1, gvr::ChannelSemantics::Alpha);
    } else {  // synthesised from the ground-truth offsets
        gvr::GaussianScene gts = scene;
        for (size_t g = 0; g < groups.size(); ++g)
            for (int k : groups[g])
                for (int d = 0; d < 3; ++d) gts.kernels[k].center[d] += gt[g][d];
        gvr::RenderBuffers buf = gvr::render(gts, target.camera, sel);
        target.image = std::move(buf.image);
        target.alpha = std::move(buf.alpha);
    }
    if (cfg.contains("init_offsets")) {
        const auto& jo = cfg.at("init_offsets");
        for (size_t g = 0; g < groups.size() && g < jo.size(); ++g) {
            const auto v = jo[g].get<std::vector<double>>();
            for (int k : groups[g])
                for (int d = 0; d < 3; ++d) scene.kernels[k].center[d] += v[d];
        }
    }
    gvr::AdamConfig adam;
    adam.lr = cfg.value("lr", 0.05);
    const auto result = gvr::fit_translation(scene, groups, target, spec, cfg.value("iters", 300), adam, sel);
    nlohmann::json extra;
    extra["task"] = "fit-translation";
    extra["translations"] = nlohmann::json::array();
    for (size_t g = 0; g < result.translations.size(); ++g) {
        const gvr::Vec3& t = result.translations[g];
        extra["translations"].push_back({t[0], t[1], t[2]});
        if (cfg.contains("init_offsets")) {
            const auto jo = cfg.at("init_offsets")[g].get<std::vector<double>>();
            double e2 = 0.0;
            for (int d = 0; d < 3; ++d) e2 += (jo[d] + t[d] - gt[g][d]) * (jo[d] + t[d] - gt[g][d]);
            extra["residual_error"].push_back(std::sqrt(e2));
        }
    }
    const fs::path out = a.str("out", "fit_translation.json");
    write_report_json(result.report, extra, out);
    write_loss_csv(result.report, fs::path(out).replace_extension(".csv"));
    std::cout << "fit-translation finished: iters=" << result.report.iterations
              << " final loss=" << (result.report.loss_trace.empty() ? 0.0 : result.report.loss_trace.back()) << "\n";
    return result.report.diverged ? kExitRuntime : kExitOk;
}

int cmd_fit_pose(const Args& a) {
    require_opts(a, {"config"});
    const nlohmann::json cfg = load_config(a.str("config"));
    const auto sel = selection_from_json(cfg);
    gvr::LossSpec spec = loss_from_json(cfg);
    const fs::path scene_path = cfg.at("scene").get<std::string>();
    require_file(scene_path, "scene");
    const gvr::GaussianScene scene = gvr::load_scene_json(scene_path);
    const fs::path camera_path = cfg.at("camera").get<std::string>();
    require_file(camera_path, "camera");
    const gvr::Camera model = gvr::load_camera_json(camera_path);
    gvr::Image target_image, target_alpha;
    if (cfg.contains("target_image")) {
        target_image = load_image_any(cfg.at("target_image").get<std::string>());
        spec.silhouette_weight = 0.0;
    } else {  // the camera file carries the ground-truth extrinsics: synthesise
        gvr::RenderBuffers buf = gvr::render(scene, model, sel);
        target_image = std::move(buf.image);
        target_alpha = std::move(buf.alpha);
    }
    std::vector<gvr::PoseStart> starts;
    if (cfg.contains("starts")) {
        for (const auto& js : cfg.at("starts")) {
            const auto w = js.at("omega").get<std::vector<double>>();
            const auto t = js.at("translation").get<std::vector<double>>();
            gvr::PoseStart st;
            st.omega = gvr::Vec3(w[0], w[1], w[2]);
            st.translation = gvr::Vec3(t[0], t[1], t[2]);
            starts.push_back(st);
        }
    } else {  // ring of azimuth starts around the ground-truth pose
        const int n = cfg.value("azimuth_starts", 8);
        const gvr::Mat3 r_gt = gvr::so3_exp(gvr::so3_log(model.rotation));
        for (int i = 0; i < n; ++i) {
            const gvr::Mat3 ry = gvr::so3_exp(gvr::Vec3(0, 2.0 * M_PI * i / n, 0));
            gvr::Mat3 prod = gvr::Mat3::Identity();
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) {
                    double acc = 0.0;
                    for (int k = 0; k < 3; ++k) acc += ry(r, k) * r_gt(k, c);
                    prod(r, c) = acc;
                }
            gvr::PoseStart st;
            st.omega = gvr::so3_log(prod);
            st.translation = model.translation;
            starts.push_back(st);
        }
    }
    gvr::AdamConfig adam;
    adam.lr = cfg.value("lr", 0.05);
    const auto result =
        gvr::fit_pose(scene, target_image, target_alpha, model, starts, spec, cfg.value("iters", 300), adam, sel);
    nlohmann::json extra;
    extra["task"] = "fit-pose";
    extra["best_start"] = result.best_start;
    extra["best_omega"] = {result.best_pose.omega[0], result.best_pose.omega[1], result.best_pose.omega[2]};
    extra["best_translation"] = {result.best_pose.translation[0], result.best_pose.translation[1],
                                 result.best_pose.translation[2]};
    if (!cfg.contains("target_image"))
        extra["rotation_error_rad"] = gvr::rotation_error(result.best_camera.rotation, model.rotation);
    const fs::path out = a.str("out", "fit_pose.json");
    write_report_json(result.report, extra, out);
    write_loss_csv(result.report, fs::path(out).replace_extension(".csv"));
    std::cout << "fit-pose finished: best start " << result.best_start << " loss "
              << result.report.metrics.at("best_loss") << "\n";
    return result.report.diverged ? kExitRuntime : kExitOk;
}

int cmd_rerender(const Args& a) {
    require_opts(a, {"attrs", "scene", "camera"});
    const fs::path attrs_path = a.str("attrs"), scene_path = a.str("scene"), camera_path = a.str("camera");
    require_file(attrs_path, "attrs");
    require_file(scene_path, "scene");
    require_file(camera_path, "camera");
    const auto attrs = gvr::load_attrs_json(attrs_path);
    const gvr::GaussianScene scene = gvr::load_scene_json(scene_path);
    const gvr::Camera camera = gvr::load_camera_json(camera_path);
    const gvr::RenderBuffers buf = gvr::resynthesize(attrs, scene, camera, selection(a));
    if (a.has("out")) gvr::write_png(buf.image, a.str("out"));
    if (a.has("out-pfm")) gvr::write_pfm(buf.image, a.str("out-pfm"));
    return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Args a = parse(argc, argv);
        if (a.cmd == "render") return cmd_render(a);
        if (a.cmd == "bench") return cmd_bench(a);
        if (a.cmd == "gradcheck") return cmd_gradcheck(a);
        if (a.cmd == "extract-texture") return cmd_extract_texture(a);
        if (a.cmd == "rerender") return cmd_rerender(a);
        if (a.cmd == "fit-translation") return cmd_fit_translation(a);
        if (a.cmd == "fit-pose") return cmd_fit_pose(a);
        std::cerr << "error: " << a.cmd
                  << " is not part of the GPU backend (converters and fitting drivers: see INTEGRATION.md)\n";
        return kExitRuntime;
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitUsage;
    } catch (const gvr::ValidationError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitUsage;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitRuntime;
    }
}
