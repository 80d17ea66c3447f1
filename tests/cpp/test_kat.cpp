// The reference's hot-path known-answer tests, run through the drop-in C++ API
// (include/hsplat/gpu.hpp -> C ABI -> CUDA) on the reference's own fixture
// streams (tests/cpp/fixtures.hpp = proj/tests/support/fixtures.hpp).  Each
// case names the reference test it ports (proj/tests/test_lod.cpp,
// proj/tests/test_render.cpp) and keeps its tolerances.  Needs a GPU; run by
// tests/test_dropin_cpp.py.  Exit code = number of failed checks.
#include "fixtures.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <set>
#include <vector>

using namespace hsplat;
using fixtures::Rng;

static int failures = 0, checks = 0;
#define CHECK(cond)                                                     \
    do {                                                                \
        ++checks;                                                       \
        if (!(cond)) {                                                  \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                 \
        }                                                               \
    } while (0)
#define CHECK_REL(a, b, rel) CHECK(std::fabs(double(a) - double(b)) <= (rel) * std::fabs(double(b)))
#define CHECK_ABS(a, b, tol) CHECK(std::fabs(double(a) - double(b)) <= (tol))
#define CHECK_THROWS(expr, errc)                     \
    do {                                             \
        bool threw__ = false;                        \
        try {                                        \
            (void)(expr);                            \
        } catch (const Error& e__) {                 \
            threw__ = e__.code() == (errc);          \
        }                                            \
        CHECK(threw__);                              \
    } while (0)

static void run(const char* name, const std::function<void()>& body) {
    const int before = failures;
    body();
    std::printf("%s %s\n", failures == before ? "ok  " : "FAIL", name);
}

namespace {

Vec3f V(float x, float y, float z) { return make_vec3(x, y, z); }

// test_lod.cpp:18-27: recursive descent from the root, nothing but granularity()
void descend(const Hierarchy& h, const CameraModel& cam, float tau, std::uint32_t i, std::vector<std::uint32_t>& out) {
    const auto& n = h.nodes[i];
    if (granularity(n.bounds, cam) <= tau || n.is_leaf()) {
        out.push_back(i);
        return;
    }
    for (std::uint32_t c = 0; c < n.child_count; ++c) descend(h, cam, tau, n.first_child + c, out);
}

std::vector<std::uint32_t> cut_nodes(const std::vector<CutEntry>& cut) {
    std::vector<std::uint32_t> ids;
    for (const auto& e : cut) ids.push_back(e.node);
    std::sort(ids.begin(), ids.end());
    return ids;
}

Hierarchy random_hierarchy(Rng& rng, int n, float spread = 5.0f) {  // test_lod.cpp:36-42
    std::vector<Gaussian> leaves;
    for (int i = 0; i < n; ++i) leaves.push_back(fixtures::random_gaussian(rng, spread, 0.05f, 0.5f, 0.2f, 1.0f));
    return fixtures::build_bvh(leaves);
}

CameraModel random_camera(Rng& rng, float spread) {  // test_lod.cpp:44-52
    float r = fixtures::uniform(rng, 0.5f * spread, 6.0f * spread);
    float az = fixtures::uniform(rng, 0.0f, 6.2831853f);
    float el = fixtures::uniform(rng, -1.2f, 1.2f);
    Vec3f pos = V(r * std::cos(el) * std::cos(az), r * std::sin(el), r * std::cos(el) * std::sin(az));
    Vec3f target = fixtures::uniform_vec3(rng, -0.3f * spread, 0.3f * spread);
    int w = 64 << (rng() % 4), hgt = 64 << (rng() % 4);
    return fixtures::look_at_camera(pos, target, w, hgt, fixtures::uniform(rng, 100.0f, 600.0f));
}

CameraModel axis_camera(int w, int h, float focal) {  // test_render.cpp:19-21
    return fixtures::look_at_camera(V(0, 0, 0), V(0, 0, 1), w, h, focal);
}

RenderSplat gray_splat(const Vec3f& mean, float sigma, float falloff) {  // test_render.cpp:36-42
    Gaussian g;
    g.mean = mean;
    g.scale = V(sigma, sigma, sigma);
    g.falloff = falloff;
    return RenderSplat::plain(g);
}

std::vector<RenderSplat> random_scene(Rng& rng, int n, bool with_transitions) {  // test_render.cpp:44-56
    std::vector<RenderSplat> splats;
    for (int i = 0; i < n; ++i) {
        RenderSplat s = RenderSplat::plain(fixtures::random_gaussian(rng, 2.0f, 0.05f, 0.6f));
        if (with_transitions && rng() % 3 == 0) {
            s.t = fixtures::uniform(rng, 0.05f, 0.95f);
            s.parent_falloff = fixtures::uniform(rng, 0.1f, 1.0f);
            s.transition_siblings = 2 + static_cast<int>(rng() % 3);
        }
        splats.push_back(s);
    }
    return splats;
}

CameraModel random_scene_camera(Rng& rng) {  // test_render.cpp:58-67
    float az = fixtures::uniform(rng, 0.0f, 6.2831853f);
    float el = fixtures::uniform(rng, -0.9f, 0.9f);
    float r = fixtures::uniform(rng, 6.0f, 14.0f);
    Vec3f pos = V(r * std::cos(el) * std::cos(az), r * std::sin(el), r * std::cos(el) * std::sin(az));
    int w = 48 + 16 * static_cast<int>(rng() % 4);
    int h = 40 + 8 * static_cast<int>(rng() % 5);
    return fixtures::look_at_camera(pos, fixtures::uniform_vec3(rng, -0.5f, 0.5f), w, h,
                                    fixtures::uniform(rng, 40.0f, 120.0f));
}

template <class T>
bool bitwise_equal(const Image<T>& a, const Image<T>& b) {
    return a.width == b.width && a.height == b.height && a.channels == b.channels &&
           std::memcmp(a.data.data(), b.data.data(), a.data.size() * sizeof(T)) == 0;
}

}  // namespace

int main() {
    // ---------------------------------------------------------------- test_lod.cpp
    run("granularity: pinhole size of a box at known depth (test_lod.cpp:55-72)", [] {
        CameraModel cam = fixtures::look_at_camera(V(0, 0, 0), V(0, 0, 1), 640, 480, 500.0f);
        Aabb thin;
        thin.min = V(-0.5f, -0.1f, 10.0f);
        thin.max = V(0.5f, 0.1f, 10.0f);
        CHECK_REL(granularity(thin, cam), 50.0f, 1e-5f);
        thin.min.z() = thin.max.z() = 20.0f;
        CHECK_REL(granularity(thin, cam), 25.0f, 1e-5f);
        Aabb cube;
        cube.min = V(-0.5f, -0.5f, 9.5f);
        cube.max = V(0.5f, 0.5f, 10.5f);
        CHECK_REL(granularity(cube, cam), 500.0f / 9.5f, 1e-5f);
    });
    run("granularity: nearest corner under arbitrary pose, 200 cameras (test_lod.cpp:74-100)", [] {
        Rng rng(60);
        for (int c = 0; c < 200; ++c) {
            CameraModel cam = random_camera(rng, 4.0f);
            Aabb box;
            Vec3f a = fixtures::uniform_vec3(rng, -5.0f, 5.0f);
            Vec3f b = fixtures::uniform_vec3(rng, -5.0f, 5.0f);
            for (int k = 0; k < 3; ++k) box.min[k] = std::min(a[k], b[k]), box.max[k] = std::max(a[k], b[k]);
            float z_near = kInf;
            for (int k = 0; k < 8; ++k) {
                Vec3f corner = V((k & 1) ? box.max.x() : box.min.x(), (k & 2) ? box.max.y() : box.min.y(),
                                 (k & 4) ? box.max.z() : box.min.z());
                z_near = std::min(z_near, cam.to_camera(corner).z());
            }
            const bool inside = box.contains(cam.position());
            const float got = granularity(box, cam);
            if (inside || z_near <= kNearPlane) {
                CHECK(got == kInf);
            } else {
                const float expect = cam.max_focal() * box.largest_dim() / z_near;
                CHECK_REL(got, expect, 1e-4f);
            }
        }
    });
    run("granularity: camera inside or behind the box (test_lod.cpp:102-113)", [] {
        CameraModel cam = fixtures::look_at_camera(V(0, 0, 0), V(0, 0, 1), 640, 480, 500.0f);
        Aabb around;
        around.min = V(-1, -1, -1);
        around.max = V(1, 1, 1);
        CHECK(granularity(around, cam) == kInf);
        Aabb behind;
        behind.min = V(-1, -1, -5);
        behind.max = V(1, 1, -4);
        CHECK(granularity(behind, cam) == kInf);
    });
    run("granularity never increases from parent to child (test_lod.cpp:115-128)", [] {
        Rng rng(61);
        for (int trial = 0; trial < 8; ++trial) {
            Hierarchy h = random_hierarchy(rng, 64);
            for (int c = 0; c < 12; ++c) {
                CameraModel cam = random_camera(rng, 5.0f);
                for (std::size_t i = 1; i < h.nodes.size(); ++i) {
                    const float child = granularity(h.nodes[i].bounds, cam);
                    const float parent = granularity(h.nodes[h.nodes[i].parent].bounds, cam);
                    CHECK(parent >= child);
                }
            }
        }
    });
    run("interpolation weight across the granularity interval (test_lod.cpp:130-141)", [] {
        CHECK(interp_weight(4.0f, 8.0f, 4.0f) == 1.0f);
        CHECK(interp_weight(4.0f, 8.0f, 8.0f) == 0.0f);
        CHECK(interp_weight(4.0f, 8.0f, 6.0f) == 0.5f);
        CHECK(interp_weight(4.0f, 8.0f, 2.0f) == 1.0f);
        CHECK(interp_weight(4.0f, 8.0f, 99.0f) == 0.0f);
        CHECK(interp_weight(5.0f, 5.0f, 3.0f) == 1.0f);
        CHECK(interp_weight(3.0f, kInf, 7.0f) == 1.0f);
    });
    run("sibling-split opacity composes back to the parent (test_lod.cpp:143-158)", [] {
        CHECK_ABS(transition_alpha(0.75f, 2), 0.5f, 1e-6f);
        CHECK_ABS(transition_alpha(0.36f, 1), 0.36f, 1e-6f);
        Rng rng(62);
        for (int i = 0; i < 100; ++i) {
            const float a = fixtures::uniform(rng, 0.0f, 0.99f);
            const int k = 1 + static_cast<int>(rng() % 6);
            const float ap = transition_alpha(a, k);
            CHECK_ABS(1.0f - std::pow(1.0f - ap, static_cast<float>(k)), a, 1e-5f);
        }
        CHECK(transition_alpha(5.0f, 2) == transition_alpha(0.99f, 2));
        CHECK_THROWS(transition_alpha(0.5f, 0), Errc::InvalidArgument);
    });
    run("cut selection matches recursive descent from the root, 60 trees (test_lod.cpp:160-174)", [] {
        Rng rng(63);
        for (int trial = 0; trial < 60; ++trial) {
            Hierarchy h = random_hierarchy(rng, 1 + static_cast<int>(rng() % 128));
            CameraModel cam = random_camera(rng, 5.0f);
            const float tau = fixtures::uniform(rng, 0.5f, 400.0f);
            std::vector<std::uint32_t> expect;
            descend(h, cam, tau, 0, expect);
            std::sort(expect.begin(), expect.end());
            CHECK(cut_nodes(select_cut(h, cam, tau)) == expect);
        }
    });
    run("cut is a partition of the leaves (test_lod.cpp:176-199)", [] {
        Rng rng(64);
        Hierarchy h = random_hierarchy(rng, 200);
        for (int c = 0; c < 10; ++c) {
            CameraModel cam = random_camera(rng, 5.0f);
            auto cut = select_cut(h, cam, fixtures::uniform(rng, 1.0f, 300.0f));
            std::vector<int> covered(h.nodes.size(), 0);
            for (const auto& e : cut) {
                std::vector<std::uint32_t> walk{e.node};
                while (!walk.empty()) {
                    const std::uint32_t i = walk.back();
                    walk.pop_back();
                    const auto& n = h.nodes[i];
                    if (n.is_leaf()) covered[i]++;
                    for (std::uint32_t k = 0; k < n.child_count; ++k) walk.push_back(n.first_child + k);
                }
            }
            for (std::size_t i = 0; i < h.nodes.size(); ++i)
                if (h.nodes[i].is_leaf()) CHECK(covered[i] == 1);
        }
    });
    run("zero threshold selects exactly the leaves at full weight (test_lod.cpp:201-212)", [] {
        Rng rng(65);
        Hierarchy h = random_hierarchy(rng, 75);
        CameraModel cam = random_camera(rng, 5.0f);
        auto cut = select_cut(h, cam, 0.0f);
        std::vector<std::uint32_t> leaves;
        for (std::uint32_t i = 0; i < h.nodes.size(); ++i)
            if (h.nodes[i].is_leaf()) leaves.push_back(i);
        CHECK(cut_nodes(cut) == leaves);
        for (const auto& e : cut) CHECK(e.t == 1.0f);
    });
    run("huge threshold selects only the root (test_lod.cpp:214-222)", [] {
        Rng rng(66);
        Hierarchy h = random_hierarchy(rng, 75);
        CameraModel cam = fixtures::look_at_camera(V(0, 0, -400), V(0, 0, 0), 64, 64, 100.0f);
        auto cut = select_cut(h, cam, 1e9f);
        CHECK(cut.size() == 1);
        if (!cut.empty()) CHECK(cut[0].node == 0 && cut[0].t == 1.0f);
    });
    run("cut entries carry the sibling-split opacity of their parent (test_lod.cpp:224-241)", [] {
        Rng rng(67);
        Hierarchy h = random_hierarchy(rng, 90);
        CameraModel cam = random_camera(rng, 5.0f);
        auto cut = select_cut(h, cam, 24.0f);
        for (const auto& e : cut) {
            const auto& n = h.nodes[e.node];
            CHECK(e.t >= 0.0f);
            CHECK(e.t <= 1.0f);
            if (e.node == 0) {
                CHECK(e.t == 1.0f);
                continue;
            }
            const auto& p = h.nodes[n.parent];
            CHECK_ABS(e.alpha_prime, transition_alpha(p.g.falloff, static_cast<int>(p.child_count)), 1e-6f);
        }
    });
    run("blended node matches child at t=1 and parent shape at t=0 (test_lod.cpp:243-265)", [] {
        Rng rng(68);
        Gaussian child = fixtures::random_gaussian(rng);
        Gaussian parent = fixtures::random_gaussian(rng);
        Gaussian at1 = interpolated_gaussian(child, parent, 1.0f, 2);
        CHECK(at1.mean == child.mean);
        CHECK(at1.scale == child.scale);
        CHECK(at1.falloff == child.falloff);
        CHECK(at1.sh == child.sh);
        const Vec4f a = quat_coeffs_wxyz(at1.rotation), b = quat_coeffs_wxyz(child.rotation);
        CHECK(std::fabs(a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + a[3] * b[3]) > 1.0f - 1e-6f);
        Gaussian at0 = interpolated_gaussian(child, parent, 0.0f, 3);
        CHECK(at0.mean == parent.mean);
        CHECK(at0.scale == parent.scale);
        CHECK(at0.sh == parent.sh);
        CHECK_ABS(at0.falloff, transition_alpha(parent.falloff, 3), 1e-6f);
        Gaussian mid = interpolated_gaussian(child, parent, 0.5f, 2);
        for (int k = 0; k < 3; ++k) CHECK_ABS(mid.mean[k], 0.5f * (child.mean[k] + parent.mean[k]), 1e-6f);
    });
    run("assembled splats expose blend inputs for the renderer (test_lod.cpp:267-292)", [] {
        Rng rng(69);
        Hierarchy h = random_hierarchy(rng, 120);
        CameraModel cam = random_camera(rng, 5.0f);
        auto cut = select_cut(h, cam, 16.0f);
        auto splats = cut_render_splats(h, cut);
        CHECK(splats.size() == cut.size());
        // the generic assembly over caller attribute arrays gives the same splats (lod.hpp:148-153)
        std::vector<Gaussian> attrs;
        for (const auto& n : h.nodes) attrs.push_back(n.g);
        auto generic = assemble_cut_splats<float>(h, attrs, cut);
        CHECK(generic.size() == splats.size());
        for (std::size_t i = 0; i < cut.size() && i < generic.size(); ++i) {
            CHECK(generic[i].mean == splats[i].mean && generic[i].sh == splats[i].sh &&
                  generic[i].rotation == splats[i].rotation && generic[i].t == splats[i].t);
            const auto& e = cut[i];
            const auto& s = splats[i];
            const auto& n = h.nodes[e.node];
            CHECK(s.t == e.t);
            if (e.node == 0 || e.t >= 1.0f) {
                CHECK(s.mean == n.g.mean);
                CHECK(s.falloff == n.g.falloff);
                CHECK(s.transition_siblings == 1);
            } else {
                const auto& p = h.nodes[n.parent];
                CHECK(s.transition_siblings == static_cast<int>(p.child_count));
                CHECK(s.parent_falloff == p.g.falloff);
                CHECK(s.falloff == n.g.falloff);
                for (int k = 0; k < 3; ++k)
                    CHECK_ABS(s.mean[k], e.t * n.g.mean[k] + (1.0f - e.t) * p.g.mean[k],
                              1e-5f * (1.0f + std::fabs(n.g.mean[k])));
            }
        }
    });
    run("assembled splats reject mismatched attribute arrays (test_lod.cpp:294-301)", [] {
        Rng rng(70);
        Hierarchy h = random_hierarchy(rng, 10);
        CameraModel cam = random_camera(rng, 5.0f);
        auto cut = select_cut(h, cam, 8.0f);
        std::vector<Gaussian> attrs(h.nodes.size() - 1);
        CHECK_THROWS(assemble_cut_splats<float>(h, attrs, cut), Errc::DimensionMismatch);
    });

    // ---------------------------------------------------------------- test_render.cpp
    run("projection of an on-axis isotropic splat has closed form (test_render.cpp:71-87)", [] {
        const float f = 80.0f, z = 5.0f, sigma = 0.3f;
        CameraModel cam = axis_camera(64, 64, f);
        ProjectedSplat p = project(gray_splat(V(0, 0, z), sigma, 0.7f), cam);
        CHECK(!p.culled);
        const float s2 = (f * sigma / z) * (f * sigma / z);
        CHECK_REL(p.cov2d(0, 0), s2 + kDilation2d, 1e-5f);
        CHECK_REL(p.cov2d(1, 1), s2 + kDilation2d, 1e-5f);
        CHECK_ABS(p.cov2d(0, 1), 0.0f, 1e-4f);
        CHECK_REL(p.det_pre, s2 * s2, 1e-4f);
        CHECK_REL(p.alpha_scale, s2 / (s2 + kDilation2d), 1e-5f);
        CHECK_ABS(p.mean2d.x(), 32.0f, 1e-4f);
        CHECK_ABS(p.mean2d.y(), 32.0f, 1e-4f);
        CHECK_REL(p.inv_depth, 1.0f / z, 1e-6f);
        CHECK(p.radius == static_cast<int>(std::ceil(3.0f * std::sqrt(s2 + kDilation2d))));
    });
    run("projection of a small off-axis splat is near the pinhole scaling (test_render.cpp:89-101)", [] {
        const float f = 300.0f, z = 20.0f, sigma = 0.02f;
        CameraModel cam = axis_camera(128, 128, f);
        ProjectedSplat p = project(gray_splat(V(0.4f, -0.3f, z), sigma, 0.7f), cam);
        CHECK(!p.culled);
        const float s2 = (f * sigma / z) * (f * sigma / z);
        CHECK_REL(p.cov2d(0, 0) - kDilation2d, s2, 1e-2f);
        CHECK_REL(p.cov2d(1, 1) - kDilation2d, s2, 1e-2f);
        CHECK(std::fabs(p.cov2d(0, 1)) < 1e-2f * s2);
    });
    run("band-0 radiance is view independent and clamped at zero (test_render.cpp:103-122)", [] {
        Gaussian g;
        g.mean = V(0.5f, -0.2f, 6.0f);
        g.scale = V(0.2f, 0.2f, 0.2f);
        g.sh[0] = 1.1f;
        g.sh[1] = -0.4f;
        g.sh[2] = -2.5f;
        const float c0 = 0.28209479177387814f;
        const float expect[3] = {0.5f + c0 * 1.1f, 0.5f + c0 * -0.4f, 0.0f};
        for (Vec3f pos : {V(0, 0, 0), V(3, 1, 0), V(-2, -4, 1)}) {
            CameraModel cam = fixtures::look_at_camera(pos, g.mean, 64, 64, 90.0f);
            ProjectedSplat p = project(RenderSplat::plain(g), cam);
            CHECK(!p.culled);
            for (int ch = 0; ch < 3; ++ch) CHECK_ABS(p.color[ch], expect[ch], 1e-5f);
            CHECK(!p.color_clamped[0]);
            CHECK(p.color_clamped[2]);
        }
    });
    run("screen-space dilation barely dampens an already huge splat (test_render.cpp:124-133)", [] {
        CameraModel cam = axis_camera(64, 64, 100.0f);
        ProjectedSplat p = project(gray_splat(V(0, 0, 2), 4.0f, 0.5f), cam);
        CHECK(!p.culled);
        CHECK(p.alpha_scale > 0.999f);
        ProjectedSplat tiny = project(gray_splat(V(0, 0, 40), 0.01f, 0.5f), cam);
        CHECK(!tiny.culled);
        CHECK(tiny.alpha_scale < 0.1f);
    });
    run("projection culls degenerate and invisible splats (test_render.cpp:135-144)", [] {
        CameraModel cam = axis_camera(64, 64, 100.0f);
        CHECK(project(gray_splat(V(0, 0, -3), 0.3f, 0.7f), cam).culled);
        CHECK(project(gray_splat(V(0, 0, 0.005f), 0.3f, 0.7f), cam).culled);
        CHECK(project(gray_splat(V(50, 0, 5), 0.1f, 0.7f), cam).culled);
        RenderSplat bad = gray_splat(V(0, 0, 5), 0.3f, 0.7f);
        bad.rotation = {0, 0, 0, 0};
        CHECK(project(bad, cam).culled);
        // the Gaussian overload (render.hpp:176) projects RenderSplat::plain(g)
        Gaussian g;
        g.mean = V(0, 0, 5);
        g.scale = V(0.3f, 0.3f, 0.3f);
        const ProjectedSplat a = project(g, cam), b = project(RenderSplat::plain(g), cam);
        CHECK(a.mean2d == b.mean2d && a.radius == b.radius && a.alpha_scale == b.alpha_scale);
    });
    run("single splat render matches a hand-computed pixel oracle (test_render.cpp:146-183)", [] {
        const float f = 80.0f, z = 5.0f, sigma = 0.3f, falloff = 0.6f;
        CameraModel cam = axis_camera(64, 64, f);
        std::vector<RenderSplat> splats{gray_splat(V(0, 0, z), sigma, falloff)};
        RenderOutput out = render_forward<float>(splats, cam);
        const double s2 = std::pow(double(f) * sigma / z, 2.0);
        const double var = s2 + kDilation2d;
        const double ascale = s2 / var;
        const int radius = static_cast<int>(std::ceil(3.0 * std::sqrt(var)));
        const int tx0 = (32 - radius) / 16, tx1 = (32 + radius) / 16 + 1;
        int contributing = 0;
        for (int y = 0; y < 64; ++y)
            for (int x = 0; x < 64; ++x) {
                const bool in_tiles = x / 16 >= tx0 && x / 16 < tx1 && y / 16 >= tx0 && y / 16 < tx1;
                double alpha = 0.0;
                if (in_tiles) {
                    const double dx = x + 0.5 - 32.0, dy = y + 0.5 - 32.0;
                    const double gx = std::exp(-0.5 * (dx * dx + dy * dy) / var);
                    const double a = std::min(0.99, falloff * ascale * gx);
                    if (a >= 1.0 / 255.0) {
                        alpha = a;
                        contributing++;
                    }
                }
                CHECK_ABS(out.color.at(x, y, 0), float(0.5 * alpha), 2e-6f);
                CHECK_ABS(out.color.at(x, y, 1), float(0.5 * alpha), 2e-6f);
                CHECK_ABS(out.depth.at(x, y, 0), float(alpha / z), 2e-6f);
                CHECK_ABS(out.transmittance.at(x, y, 0), float(1.0 - alpha), 2e-6f);
            }
        CHECK(contributing > 200);
        CHECK(out.rendered_count == 1);
    });
    run("depth map of one splat is blend weight times inverse depth (test_render.cpp:185-196)", [] {
        const float z = 7.0f;
        CameraModel cam = axis_camera(48, 48, 70.0f);
        std::vector<RenderSplat> splats{gray_splat(V(0, 0, z), 0.4f, 0.8f)};
        RenderOutput out = render_forward<float>(splats, cam);
        for (int y = 0; y < 48; ++y)
            for (int x = 0; x < 48; ++x) CHECK_ABS(out.depth.at(x, y, 0), (1.0f - out.transmittance.at(x, y, 0)) / z, 1e-6f);
    });
    run("input order does not affect the image (test_render.cpp:198-218)", [] {
        Rng rng(70);
        CameraModel cam = axis_camera(64, 48, 90.0f);
        std::vector<RenderSplat> a;
        for (int i = 0; i < 20; ++i) {
            Vec3f mean = fixtures::uniform_vec3(rng, -1.0f, 1.0f);
            mean.z() = fixtures::uniform(rng, 4.0f, 9.0f);
            const float sigma = fixtures::uniform(rng, 0.1f, 0.4f);
            a.push_back(gray_splat(mean, sigma, fixtures::uniform(rng, 0.3f, 0.9f)));
        }
        std::vector<RenderSplat> b(a.rbegin(), a.rend());
        RenderOutput ra = render_forward<float>(a, cam), rb = render_forward<float>(b, cam),
                     ra2 = render_forward<float>(a, cam);
        CHECK(bitwise_equal(ra.color, rb.color));
        CHECK(bitwise_equal(ra.depth, rb.depth));
        CHECK(bitwise_equal(ra.transmittance, rb.transmittance));
        CHECK(ra.rendered_count == rb.rendered_count);
        CHECK(bitwise_equal(ra.color, ra2.color));
    });
    run("tiled renderer equals the naive reference bit for bit (test_render.cpp:220-232)", [] {
        Rng rng(71);
        for (int trial = 0; trial < 4; ++trial) {
            auto splats = random_scene(rng, 150, true);
            CameraModel cam = random_scene_camera(rng);
            RenderOutput tiled = render_forward<float>(splats, cam);
            RenderOutput naive = render_reference<float>(splats, cam);
            CHECK(bitwise_equal(tiled.color, naive.color));
            CHECK(bitwise_equal(tiled.depth, naive.depth));
            CHECK(bitwise_equal(tiled.transmittance, naive.transmittance));
            CHECK(tiled.rendered_count == naive.rendered_count);
        }
    });
    run("empty splat list renders black with full transmittance (test_render.cpp:234-241)", [] {
        CameraModel cam = axis_camera(40, 24, 60.0f);
        RenderOutput out = render_forward<float>(std::span<const RenderSplat>(), cam);
        CHECK(out.rendered_count == 0);
        for (float v : out.color.data) CHECK(v == 0.0f);
        for (float v : out.depth.data) CHECK(v == 0.0f);
        for (float v : out.transmittance.data) CHECK(v == 1.0f);
    });
    run("falloff beyond one only saturates the blend alpha (test_render.cpp:243-261)", [] {
        CameraModel cam = axis_camera(64, 64, 80.0f);
        for (float big : {4.0f, 1e8f}) {
            std::vector<RenderSplat> splats{gray_splat(V(0, 0, 5), 0.3f, big)};
            RenderOutput out = render_forward<float>(splats, cam);
            for (float v : out.color.data) CHECK(std::isfinite(v));
            for (float v : out.transmittance.data) CHECK(std::isfinite(v));
            CHECK_ABS(out.transmittance.at(32, 32, 0), 1.0f - kAlphaMax, 1e-6f);
        }
        std::vector<RenderSplat> neg{gray_splat(V(0, 0, 5), 0.3f, -0.5f)};
        RenderOutput out = render_forward<float>(neg, cam);
        CHECK(out.rendered_count == 0);
        for (float v : out.transmittance.data) CHECK(v == 1.0f);
    });
    run("blended coverage never exceeds one (test_render.cpp:263-283)", [] {
        Rng rng(72);
        auto splats = random_scene(rng, 120, true);
        const float white = 0.5f / 0.28209479177387814f;
        for (auto& s : splats) {
            s.sh.fill(0.0f);
            for (int ch = 0; ch < 3; ++ch) s.sh[ch] = white;
        }
        CameraModel cam = random_scene_camera(rng);
        RenderOutput out = render_forward<float>(splats, cam);
        for (int y = 0; y < cam.height; ++y)
            for (int x = 0; x < cam.width; ++x) {
                const float t = out.transmittance.at(x, y, 0);
                CHECK(t >= 0.0f && t <= 1.0f);
                CHECK_ABS(out.color.at(x, y, 0), 1.0f - t, 1e-5f);
                CHECK(out.color.at(x, y, 0) <= 1.0f + 1e-6f);
            }
    });
    run("transition splat blends the two falloff laws per pixel (test_render.cpp:285-309)", [] {
        CameraModel cam = axis_camera(48, 48, 70.0f);
        RenderSplat s = gray_splat(V(0, 0, 6), 0.5f, 0.8f);
        s.t = 0.4f;
        s.parent_falloff = 0.6f;
        s.transition_siblings = 3;
        std::vector<RenderSplat> splats{s};
        RenderOutput out = render_forward<float>(splats, cam);
        ProjectedSplat p = project(s, cam);
        CHECK(!p.culled);
        for (int y = 0; y < 48; ++y)
            for (int x = 0; x < 48; ++x) {
                const double dx = x + 0.5 - p.mean2d.x(), dy = y + 0.5 - p.mean2d.y();
                const double g = std::exp(-0.5 * (p.conic[0] * dx * dx + p.conic[2] * dy * dy) - p.conic[1] * dx * dy);
                double self = std::min(double(kAlphaMax), 0.8 * p.alpha_scale * g);
                const double par = std::min(double(kAlphaMax), 0.6 * p.alpha_scale * g);
                if (self < kAlphaMin) self = 0.0;
                const double split = par >= kAlphaMin ? 1.0 - std::pow(1.0 - par, 1.0 / 3.0) : 0.0;
                CHECK_ABS(1.0f - out.transmittance.at(x, y, 0), float(0.4 * self + 0.6 * split), 1e-5f);
            }
    });
    run("render_backward from an older ForwardContext (render.hpp:478) re-renders its splats", [] {
        Rng rng(75);
        auto splats = random_scene(rng, 60, true);
        CameraModel cam = random_scene_camera(rng);
        ForwardContext ctx;
        (void)render_forward<float>(splats, cam, &ctx);
        CHECK(ctx.valid && ctx.splats.size() == splats.size() && ctx.projected.size() == splats.size());
        CHECK(ctx.tile_start.back() == ctx.tile_entries.size());
        std::size_t visible = 0;
        for (const auto& p : ctx.projected) visible += !p.culled;
        CHECK(ctx.order.size() == visible);
        for (std::size_t i = 1; i < ctx.order.size(); ++i)
            CHECK(ctx.projected[ctx.order[i - 1]].cam_point.z() <= ctx.projected[ctx.order[i]].cam_point.z());
        Image<float> lg(cam.width, cam.height, 3, 0.01f);
        const RenderGrads now = render_backward<float>(ctx, lg);
        (void)render_forward<float>(random_scene(rng, 30, false), cam);  // the device state moves on
        const RenderGrads later = render_backward<float>(ctx, lg);
        CHECK(now.mean.size() == later.mean.size());
        for (std::size_t i = 0; i < now.mean.size() && i < later.mean.size(); ++i)
            CHECK(now.mean[i] == later.mean[i] && now.sh[i] == later.sh[i]);
    });

    std::printf("%s: %d failure(s) in %d checks\n", failures ? "FAIL" : "PASS", failures, checks);
    return failures;
}
