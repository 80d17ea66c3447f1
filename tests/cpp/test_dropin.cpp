// C++ drop-in check: the reference-shaped API of include/hsplat/gpu.hpp, used
// exactly like the reference's own tests use hsplat:: (tests/test_lod.cpp,
// tests/test_render.cpp, tests/test_bench.cpp).  Needs a GPU; run by
// tests/test_dropin_cpp.py.  Exit code = number of failed checks.
#include <hsplat/gpu.hpp>

#include <cmath>
#include <cstdio>
#include <thread>
#include <vector>

static int failures = 0;
#define CHECK(cond)                                                       \
    do {                                                                  \
        if (!(cond)) {                                                    \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
            ++failures;                                                   \
        }                                                                 \
    } while (0)

static hsplat::CameraModel look_at(float px, float py, float pz, float tx, float ty, float tz, int w, int h, float f) {
    auto norm = [](float v[3]) {
        const float n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        for (int k = 0; k < 3; ++k) v[k] /= n;
    };
    float z[3] = {tx - px, ty - py, tz - pz};
    norm(z);
    float x[3] = {1.0f * z[2] - 0.0f * z[1], 0.0f * z[0] - 0.0f * z[2], 0.0f * z[1] - 1.0f * z[0]};  // up x z
    norm(x);
    const float y[3] = {z[1] * x[2] - z[2] * x[1], z[2] * x[0] - z[0] * x[2], z[0] * x[1] - z[1] * x[0]};
    hsplat::CameraModel c;
    c.width = w;
    c.height = h;
    c.focal.x() = c.focal.y() = f;
    c.principal.x() = w * 0.5f;
    c.principal.y() = h * 0.5f;
    const float p[3] = {px, py, pz};
    for (int k = 0; k < 3; ++k) {
        c.world_to_camera(0, k) = x[k];
        c.world_to_camera(1, k) = y[k];
        c.world_to_camera(2, k) = z[k];
    }
    for (int r = 0; r < 3; ++r)
        c.world_to_camera(r, 3) = -(c.world_to_camera(r, 0) * p[0] + c.world_to_camera(r, 1) * p[1] +
                                    c.world_to_camera(r, 2) * p[2]);
    return c;
}

static hsplat::Hierarchy synth(std::uint64_t leaves) {
    const std::uint64_t n = hs_synth_node_count(leaves);
    std::vector<std::uint32_t> parent(n), fc(n), cc(n);
    std::vector<float> bmin(3 * n), bmax(3 * n), mean(3 * n), scale(3 * n), rot(4 * n), fall(n), sh(48 * n);
    hs_node_soa_out o{parent.data(), fc.data(), cc.data(), bmin.data(), bmax.data(),
                      mean.data(),   scale.data(), rot.data(), fall.data(), sh.data()};
    if (hs_synth_city(leaves, 7, 0, &o) != HS_OK) std::abort();
    hs_node_soa in{parent.data(), fc.data(), cc.data(), bmin.data(), bmax.data(),
                   mean.data(),   scale.data(), rot.data(), fall.data(), sh.data()};
    hs_h3dg_write("/tmp/hs_dropin.h3dg", &in, n, 3);
    return hsplat::read_hierarchy("/tmp/hs_dropin.h3dg");
}

int main() {
    using namespace hsplat;
    const Hierarchy h = synth(20000);
    CHECK(h.leaf_count() == 20000);
    const float side = hs_synth_scene_side(20000);
    const CameraModel cam = look_at(0, 12, -0.5f * side - 8, 0, 0, -0.5f * side + 40, 160, 120, 120.0f);

    // select_cut: ascending node order, partition sanity, t in [0,1] (test_lod.cpp:160-241)
    const auto cut = select_cut(h, cam, 3.0f);
    CHECK(!cut.empty());
    for (std::size_t i = 1; i < cut.size(); ++i) CHECK(cut[i - 1].node < cut[i].node);
    for (const auto& e : cut) CHECK(e.t >= 0.0f && e.t <= 1.0f);
    const auto leaves = select_cut(h, cam, 0.0f);
    CHECK(leaves.size() == h.leaf_count());
    bool threw = false;
    try {
        select_cut(h, cam, -1.0f);
    } catch (const Error& e) {
        threw = e.code() == Errc::InvalidArgument;
    }
    CHECK(threw);

    // cut_render_splats: plain entries copy the node (test_lod.cpp:267-292)
    const auto splats = cut_render_splats(h, cut);
    CHECK(splats.size() == cut.size());
    for (std::size_t i = 0; i < cut.size(); ++i)
        if (cut[i].t >= 1.0f) CHECK(splats[i].falloff == h.nodes[cut[i].node].g.falloff);

    // render_hierarchy == render_forward(cut_render_splats(select_cut)) (render.hpp:706-720)
    StageTimes st;
    ForwardContext fctx;
    const RenderOutput a = render_hierarchy(h, cam, 3.0f, &fctx, &st);
    const RenderOutput b = render_forward<float>(std::span<const RenderSplat>(splats), cam);
    CHECK(a.rendered_count > 0 && a.rendered_count == b.rendered_count);
    CHECK(a.color.data == b.color.data);
    CHECK(a.transmittance.data == b.transmittance.data);
    CHECK(fctx.valid && fctx.tile_start.back() == fctx.tile_entries.size());
    CHECK(st.alpha_blend > 0.0 && st.cut_expand > 0.0);
    for (float v : a.transmittance.data) CHECK(v >= 0.0f && v <= 1.0f);

    // empty scene (test_render.cpp:234-241)
    const RenderOutput e = render_forward<float>(std::span<const RenderSplat>(), cam);
    CHECK(e.rendered_count == 0);
    for (float v : e.transmittance.data) CHECK(v == 1.0f);

    // bench_path: static path uploads once (test_bench.cpp:91-113)
    CameraPath path;
    for (int i = 0; i < 6; ++i) path.cameras.push_back(cam);
    const BenchReport rep = bench_path(h, path, 3.0f);
    CHECK(rep.frames.size() == 6);
    CHECK(rep.frames[0].transferred == rep.frames[0].rendered);
    for (std::size_t i = 1; i < 6; ++i) CHECK(rep.frames[i].transferred == 0);
    for (std::size_t i = 1; i < 6; i += 2) CHECK(rep.frames[i].stages.cut_expand == 0.0);

    // render_backward (render.hpp:427-702): band-0 closed form (test_render.cpp:556-576)
    {
        CameraModel bc;
        bc.width = bc.height = 48;
        bc.focal.x() = bc.focal.y() = 70.0f;
        bc.principal.x() = bc.principal.y() = 24.0f;
        for (int r = 0; r < 3; ++r) bc.world_to_camera(r, r) = 1.0f;
        RenderSplat s;
        s.mean[2] = 6.0f;
        s.scale = Vec3f{{0.4f, 0.4f, 0.4f}};
        s.falloff = 0.5f;
        s.sh[0] = s.sh[1] = s.sh[2] = 1.0f;
        std::vector<RenderSplat> one{s};
        ForwardContext bctx;
        const RenderOutput bo = render_forward<float>(std::span<const RenderSplat>(one), bc, &bctx);
        const double n = 48.0 * 48.0 * 3.0;
        Image<float> lg(48, 48, 3, static_cast<float>(1.0 / n));
        const RenderGrads g = render_backward<float>(bctx, lg);
        double mass = 0.0;
        for (float t : bo.transmittance.data) mass += 1.0 - t;
        const double want = 0.28209479177387814 * mass / n;
        CHECK(std::abs(g.sh[0][0] - want) <= 1e-4 * std::abs(want));
        // a context from an older render still differentiates its own forward pass
        (void)render_forward<float>(std::span<const RenderSplat>(one), bc, nullptr);
        const RenderGrads g2 = render_backward<float>(bctx, lg);
        CHECK(g2.sh[0][0] == g.sh[0][0]);
        // an invalid context has no forward state (render.hpp:432-433)
        ForwardContext empty;
        threw = false;
        try {
            render_backward<float>(empty, lg);
        } catch (const Error& err) {
            threw = err.code() == Errc::MissingForwardState;
        }
        CHECK(threw);
    }
    // compact (build.hpp:168-272): leaves kept, every interior node has >= 2 children
    {
        std::vector<CameraModel> cams{cam};
        const Hierarchy c = compact(h, cams, 3.0f);
        CHECK(c.nodes.size() <= h.nodes.size());
        CHECK(c.leaf_count() == h.leaf_count());
        for (const auto& nd : c.nodes) CHECK(nd.is_leaf() || nd.child_count >= 2);
        threw = false;
        try {
            compact(h, std::span<const CameraModel>{}, 3.0f);
        } catch (const Error& err) {
            threw = err.code() == Errc::InvalidArgument;
        }
        CHECK(threw);
    }
    // assemble (consolidate's BFS layout): two parts under one root
    {
        const Hierarchy parts[2] = {h, h};
        const Hierarchy a = gpu::assemble(parts);
        CHECK(a.nodes.size() == 2 * h.nodes.size() + 1);
        CHECK(a.nodes[0].child_count == 2 && a.nodes[0].first_child == 1);
        CHECK(a.leaf_count() == 2 * h.leaf_count());
    }

    // explicit device residency: the DeviceHierarchy overloads agree with the cached ones
    {
        const gpu::DeviceHierarchy dh(h);
        CHECK(dh.size() == h.nodes.size() && dh.leaf_count() == h.leaf_count());
        const auto a = select_cut(h, cam, 3.0f);
        const auto b = select_cut(dh, cam, 3.0f);
        CHECK(a.size() == b.size());
        for (std::size_t i = 0; i < a.size() && i < b.size(); ++i) CHECK(a[i].node == b[i].node && a[i].t == b[i].t);
        const RenderOutput ra = render_hierarchy(h, cam, 3.0f);
        const RenderOutput rb = render_hierarchy(dh, cam, 3.0f);
        CHECK(ra.color.data == rb.color.data);
        const Hierarchy back = dh.download();
        CHECK(back.nodes.size() == h.nodes.size() && back.nodes[1].g.mean[0] == h.nodes[1].g.mean[0]);
        CameraPath p2;
        for (int i = 0; i < 4; ++i) p2.cameras.push_back(cam);
        CHECK(bench_path(dh, p2, 3.0f).frames.size() == 4);
    }

    // write_hierarchy / read_hierarchy round trip (io.hpp:350-408); camera text IO (io.hpp:410-511)
    {
        write_hierarchy("/tmp/hs_dropin_rt.h3dg", h);
        const Hierarchy back = read_hierarchy("/tmp/hs_dropin_rt.h3dg");
        CHECK(back.nodes.size() == h.nodes.size() && back.nodes.back().g.sh[7] == h.nodes.back().g.sh[7]);
        const CameraModel cams[2] = {cam, look_at(3, 9, -40, 0, 0, 0, 320, 200, 250.0f)};
        write_cameras("/tmp/hs_dropin_cams.txt", cams);
        const auto rc = read_cameras("/tmp/hs_dropin_cams.txt");
        CHECK(rc.size() == 2 && rc[1].width == 320 && rc[1].world_to_camera(2, 3) == cams[1].world_to_camera(2, 3));
        CameraPath cp;
        cp.cameras = {cams[0], cams[1]};
        cp.timestamps = {0.0, 1.0 / 30.0};
        write_camera_path("/tmp/hs_dropin_path.txt", cp);
        const CameraPath rp = read_camera_path("/tmp/hs_dropin_path.txt");
        CHECK(rp.cameras.size() == 2 && rp.timestamps[1] == cp.timestamps[1]);
        cp.timestamps = {1.0, 1.0};
        threw = false;
        try {
            write_camera_path("/tmp/hs_dropin_path.txt", cp);
        } catch (const Error& err) {
            threw = err.code() == Errc::InvalidArgument;
        }
        CHECK(threw);
        // bench_path CSV schema (bench.hpp:33-48, test_bench.cpp:141-158) and metrics (bench.hpp:105-112)
        const std::string csv = rep.csv();
        CHECK(csv.rfind("frame,rendered,rendered_pct,transferred,cut_expand_s", 0) == 0);
        CHECK(csv.find("\ntotal,") != std::string::npos);
        const Metrics m = metrics(a.color, b.color);
        CHECK(m.psnr_db == 99.0 && std::abs(m.ssim - 1.0) < 1e-6);
        set_thread_count(3);
        CHECK(thread_count() == 3);
        set_thread_count(0);
    }

    // reentrant across host threads: every thread its own device context
    {
        std::vector<float> got(4, 0.0f);
        std::vector<std::thread> pool;
        for (int k = 0; k < 4; ++k)
            pool.emplace_back([&, k] {
                const RenderOutput r = render_hierarchy(h, cam, 3.0f);
                got[k] = r.color.data[r.color.data.size() / 2] + float(r.rendered_count == a.rendered_count);
            });
        for (auto& t : pool) t.join();
        for (int k = 1; k < 4; ++k) CHECK(got[k] == got[0]);
    }

    // photometric_loss (image.hpp:193-206) and refine_hierarchy (refine.hpp:253-402) through the shim
    {
        Imagef img = a.color, g;
        CHECK(photometric_loss(img, img, &g) == 0.0f);
        for (float v : g.data) CHECK(v == 0.0f);
        std::vector<CameraModel> cams = {cam};
        std::vector<Imagef> targets = {a.color};
        for (float& v : targets[0].data) v = std::min(1.0f, v * 0.9f + 0.05f);
        RefineConfig rc;
        rc.steps = 3;
        rc.tau_min = 3.0f;
        rc.tau_max = 12.0f;
        RefineStats rs;
        const Hierarchy out = refine_hierarchy(h, cams, targets, rc, &rs);
        CHECK(out.nodes.size() == h.nodes.size());
        CHECK(rs.loss.size() == 3 && rs.loss[0] > 0.0);
        CHECK(rs.max_screen_grad.size() == h.nodes.size());
        std::size_t frozen = 0, leaves = 0;
        for (std::size_t i = 0; i < h.nodes.size(); ++i)
            if (h.nodes[i].is_leaf()) {
                ++leaves;
                frozen += std::memcmp(&out.nodes[i].g, &h.nodes[i].g, sizeof(Gaussian)) == 0;
            }
        CHECK(frozen == leaves);
    }

    // read_hierarchy error code (io.hpp:375-387)
    threw = false;
    try {
        read_hierarchy("/nonexistent/x.h3dg");
    } catch (const Error& err) {
        threw = err.code() == Errc::IoFailure;
    }
    CHECK(threw);

    std::printf("%s: %d failure(s)\n", failures ? "FAIL" : "PASS", failures);
    return failures;
}
