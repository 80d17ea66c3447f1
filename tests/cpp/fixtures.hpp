// Port of the reference's test fixtures (proj/tests/support/fixtures.hpp:15-45,
// :102-121) over the drop-in stand-in types: the same std::mt19937_64 streams
// and libstdc++ distributions, drawn in the same call order (argument lists of
// three draws go through a function call, as the reference's Vec3f(...)
// constructor call does), so the reference tests' random inputs are reproduced
// with this toolchain's libstdc++.  The float arithmetic of look_at_camera
// follows Eigen 3.4's fixed-size orders (3-term sums x0 + (x1 + x2)).
#pragma once
#include <hsplat/gpu.hpp>

#include <cmath>
#include <random>

namespace fixtures {

using Rng = std::mt19937_64;
using hsplat::Gaussian;
using hsplat::Quatf;
using hsplat::Vec3f;

inline float uniform(Rng& rng, float lo, float hi) { return std::uniform_real_distribution<float>(lo, hi)(rng); }

inline Vec3f uniform_vec3(Rng& rng, float lo, float hi) {
    return hsplat::make_vec3(uniform(rng, lo, hi), uniform(rng, lo, hi), uniform(rng, lo, hi));
}

inline Quatf make_quat(float w, float x, float y, float z) { return Quatf{w, x, y, z}; }

// Eigen Quaternion::normalize over coeffs (x, y, z, w): SSE reduction (x^2 + z^2) + (y^2 + w^2)
inline Quatf normalized(const Quatf& q) {
    const float n = std::sqrt((q.x() * q.x() + q.z() * q.z()) + (q.y() * q.y() + q.w() * q.w()));
    return Quatf{q.w() / n, q.x() / n, q.y() / n, q.z() / n};
}

inline Quatf random_quat(Rng& rng) {
    std::normal_distribution<float> n(0.0f, 1.0f);
    return normalized(make_quat(n(rng), n(rng), n(rng), n(rng)));
}

inline Gaussian random_gaussian(Rng& rng, float mean_spread = 2.0f, float scale_min = 0.3f, float scale_max = 1.5f,
                                float falloff_min = 0.1f, float falloff_max = 1.0f) {
    Gaussian g;
    g.mean = uniform_vec3(rng, -mean_spread, mean_spread);
    g.scale = uniform_vec3(rng, scale_min, scale_max);
    g.rotation = random_quat(rng);
    g.falloff = uniform(rng, falloff_min, falloff_max);
    for (auto& v : g.sh) v = uniform(rng, -0.5f, 0.5f);
    return g;
}

inline float dot3(const Vec3f& a, const Vec3f& b) { return a[0] * b[0] + (a[1] * b[1] + a[2] * b[2]); }
inline Vec3f cross(const Vec3f& a, const Vec3f& b) {
    return hsplat::make_vec3(a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]);
}
inline Vec3f normalize(const Vec3f& v) {
    const float n = std::sqrt(dot3(v, v));
    return n > 0.0f ? hsplat::make_vec3(v[0] / n, v[1] / n, v[2] / n) : v;
}

// Proper-rotation look-at camera: +z forward, +x right, +y = z cross x.
inline hsplat::CameraModel look_at_camera(const Vec3f& pos, const Vec3f& target, int width, int height, float focal,
                                          const Vec3f& up = hsplat::make_vec3(0.0f, 1.0f, 0.0f)) {
    const Vec3f zc = normalize(hsplat::make_vec3(target[0] - pos[0], target[1] - pos[1], target[2] - pos[2]));
    Vec3f xc = cross(up, zc);
    if (std::sqrt(dot3(xc, xc)) < 1e-5f) xc = hsplat::make_vec3(1.0f, 0.0f, 0.0f);
    xc = normalize(xc);
    const Vec3f yc = cross(zc, xc);
    hsplat::CameraModel cam;
    cam.width = width;
    cam.height = height;
    cam.focal.x() = cam.focal.y() = focal;
    cam.principal.x() = width * 0.5f;
    cam.principal.y() = height * 0.5f;
    const Vec3f rows[3] = {xc, yc, zc};
    for (int r = 0; r < 3; ++r) {
        for (int k = 0; k < 3; ++k) cam.world_to_camera(r, k) = rows[r][k];
        cam.world_to_camera(r, 3) = -dot3(rows[r], pos);
    }
    return cam;
}

// build_bvh (build.hpp:73-149) over the leaves, through the library's host tool
inline hsplat::Hierarchy build_bvh(const std::vector<Gaussian>& leaves) {
    const std::size_t n = leaves.size();
    const hsplat::gpu::GaussianArrays a{std::span<const Gaussian>(leaves)};
    hsplat::gpu::NodeArrays out(2 * n - 1);
    hs_node_soa_out o = out.out();
    if (hs_build_bvh(a.mean.data(), a.scale.data(), a.rot.data(), a.fall.data(), a.sh.data(), n, 1, &o) != HS_OK)
        throw std::runtime_error("build_bvh failed");
    return out.hierarchy(3);
}

}  // namespace fixtures
