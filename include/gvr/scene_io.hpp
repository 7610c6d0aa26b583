// gvr/scene_io.hpp — the reference's data formats (proj/include/gvr/scene_io.hpp,
// src/scene_io.cpp) for the C++ drop-in. Host file I/O over nlohmann::json
// (`#include <json.hpp>`, as the reference builds it); loaders validate like the
// reference's (scene on the device, camera via gvr_camera_validate). Same
// formats as paper_2205_15401_b200/scene_io.py:
//   scene  {"version": 1, "tau", "kernels": [{"center": [3], "inv_cov": [9], "attr": [D]}]}
//   camera {"version": 1, "R": [9], "T": [3], "F", "Ox", "Oy", "H", "W"}
//   attrs  {"version": 1, "attrs": [[D]...], "support": [K], "masked": [bool...]}
// The mesh / point-cloud loaders (load_obj / load_ply) belong to the converters,
// which are outside the render path and not part of this backend.
#pragma once

#include "gvr.hpp"
#include "image_io.hpp"

#include <json.hpp>

#include <filesystem>
#include <fstream>
#include <string>

namespace gvr {

namespace detail {

inline nlohmann::json load_json_file(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw ValidationError("cannot open file: " + path.string());
    nlohmann::json j;
    try {
        in >> j;
    } catch (const nlohmann::json::exception& e) {
        throw ValidationError("invalid JSON in " + path.string() + ": " + e.what());
    }
    if (j.contains("version") && j.at("version").get<int>() != 1)
        throw ValidationError("unsupported format version in " + path.string());
    return j;
}

}  // namespace detail

// scene_io.hpp:36
inline void atomic_write_text(const std::filesystem::path& path, const std::string& content) {
    detail::write_file_atomic(path, content);
}

// scene_io.cpp:53-74
inline GaussianScene load_scene_json(const std::filesystem::path& path) {
    const nlohmann::json j = detail::load_json_file(path);
    GaussianScene scene;
    scene.tau = j.value("tau", 1.0);
    for (const auto& jk : j.at("kernels")) {
        const auto c = jk.at("center").get<std::vector<double>>();
        const auto s = jk.at("inv_cov").get<std::vector<double>>();
        const auto a = jk.at("attr").get<std::vector<double>>();
        if (c.size() != 3 || s.size() != 9) throw ValidationError("bad kernel entry in " + path.string());
        GaussianKernel k;
        k.center = Vec3(c[0], c[1], c[2]);
        for (int r = 0; r < 3; ++r)
            for (int t = 0; t < 3; ++t) k.inv_cov(r, t) = s[3 * r + t];
        k.attr = VecX(static_cast<int>(a.size()));
        for (size_t i = 0; i < a.size(); ++i) k.attr[static_cast<int>(i)] = a[i];
        scene.kernels.push_back(std::move(k));
    }
    scene.validate();
    return scene;
}

// scene_io.cpp:76-92
inline void save_scene_json(const GaussianScene& scene, const std::filesystem::path& path) {
    nlohmann::json j;
    j["version"] = 1;
    j["tau"] = scene.tau;
    j["kernels"] = nlohmann::json::array();
    for (const auto& k : scene.kernels) {
        std::vector<double> c(3), s(9), a(static_cast<size_t>(k.attr.size()));
        for (int t = 0; t < 3; ++t) c[t] = k.center[t];
        for (int r = 0; r < 3; ++r)
            for (int t = 0; t < 3; ++t) s[3 * r + t] = k.inv_cov(r, t);
        for (size_t i = 0; i < a.size(); ++i) a[i] = k.attr[static_cast<int>(i)];
        j["kernels"].push_back({{"center", c}, {"inv_cov", s}, {"attr", a}});
    }
    atomic_write_text(path, j.dump(2) + "\n");
}

// scene_io.cpp:94-113
inline Camera load_camera_json(const std::filesystem::path& path) {
    const nlohmann::json j = detail::load_json_file(path);
    const auto r = j.at("R").get<std::vector<double>>();
    const auto t = j.at("T").get<std::vector<double>>();
    if (r.size() != 9 || t.size() != 3) throw ValidationError("bad camera extrinsics in " + path.string());
    Camera cam;
    for (int i = 0; i < 3; ++i)
        for (int c = 0; c < 3; ++c) cam.rotation(i, c) = r[3 * i + c];
    cam.translation = Vec3(t[0], t[1], t[2]);
    cam.focal = j.at("F").get<double>();
    cam.ox = j.at("Ox").get<double>();
    cam.oy = j.at("Oy").get<double>();
    cam.height = j.at("H").get<int>();
    cam.width = j.at("W").get<int>();
    cam.validate();
    return cam;
}

// scene_io.cpp:115-129
inline void save_camera_json(const Camera& camera, const std::filesystem::path& path) {
    std::vector<double> r(9), t(3);
    for (int i = 0; i < 3; ++i) {
        for (int c = 0; c < 3; ++c) r[3 * i + c] = camera.rotation(i, c);
        t[i] = camera.translation[i];
    }
    const nlohmann::json j = {{"version", 1}, {"R", r},       {"T", t},           {"F", camera.focal},
                              {"Ox", camera.ox}, {"Oy", camera.oy}, {"H", camera.height}, {"W", camera.width}};
    atomic_write_text(path, j.dump(2) + "\n");
}

// scene_io.cpp:131-145
inline SampledAttributes load_attrs_json(const std::filesystem::path& path) {
    const nlohmann::json j = detail::load_json_file(path);
    SampledAttributes out;
    for (const auto& ja : j.at("attrs")) {
        const auto a = ja.get<std::vector<double>>();
        VecX v(static_cast<int>(a.size()));
        for (size_t i = 0; i < a.size(); ++i) v[static_cast<int>(i)] = a[i];
        out.attrs.push_back(v);
    }
    out.support = j.at("support").get<std::vector<double>>();
    for (const auto& m : j.at("masked")) out.masked.push_back(m.get<bool>());
    if (out.support.size() != out.attrs.size() || out.masked.size() != out.attrs.size())
        throw ValidationError("inconsistent attrs file: " + path.string());
    return out;
}

// scene_io.cpp:147-158
inline void save_attrs_json(const SampledAttributes& attrs, const std::filesystem::path& path) {
    nlohmann::json j;
    j["version"] = 1;
    j["attrs"] = nlohmann::json::array();
    for (const auto& a : attrs.attrs) {
        std::vector<double> v(static_cast<size_t>(a.size()));
        for (size_t i = 0; i < v.size(); ++i) v[i] = a[static_cast<int>(i)];
        j["attrs"].push_back(v);
    }
    j["support"] = attrs.support;
    j["masked"] = nlohmann::json::array();
    for (bool m : attrs.masked) j["masked"].push_back(m);
    atomic_write_text(path, j.dump(2) + "\n");
}

}  // namespace gvr
