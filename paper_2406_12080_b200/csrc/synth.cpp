// synth.cpp — deterministic synthetic Gaussian hierarchies (host tool).
//
// Produces the inputs the benchmark configurations name (BASELINE.json: 100K /
// 10M / 100M-leaf hierarchies) in the reference's own node layout:
//   * leaves: clustered city-like scene with the statistics of the reference's
//     acceptance toy scene (proj/tests/acceptance.cpp:62-94: 21 leaves per
//     cluster, offsets U(-0.55,0.55) m, scales U(0.06,0.2) m, falloff
//     U(0.4,0.9), two-tone SH DC U(-1.2,1.5), higher bands U(-0.08,0.08)),
//     cluster centres spread at constant areal density over a square of side
//     28 m * sqrt(clusters / 240);
//   * tree: build_bvh (proj/include/hsplat/build.hpp:73-149) — top-down median
//     split on the longest axis of the group box, 2N-1 nodes, sibling pairs
//     contiguous, parent < child, identical stack-order index allocation;
//     leaf boxes are leaf_aabb (build.hpp:20-29), parent boxes the union of
//     child boxes (build.hpp:130-136);
//   * interior Gaussians: moment-matched merge (merge.hpp:86-118) with an
//     Eigen-free Jacobi eigensolver in double, then the root-down 24-way
//     axis-convention match (merge.hpp:123-173).
// The output only has to be a valid hierarchy that both the GPU path and the
// CPU oracle consume bit-identically; it is not compared against Eigen.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

#include "hsplat_b200_internal.h"

namespace {

struct Rng {  // splitmix64 stream
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    float u01() { return static_cast<float>(next() >> 40) * (1.0f / 16777216.0f); }
    float uniform(float lo, float hi) { return lo + (hi - lo) * u01(); }
    float normal() {
        double u1 = (static_cast<double>(next() >> 11) + 0.5) * (1.0 / 9007199254740992.0);
        double u2 = static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0);
        return static_cast<float>(std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2));
    }
};

struct G {  // Gaussian, quaternion wxyz
    float mean[3], scale[3], q[4], falloff, sh[48];
};

void quat_to_mat(const float q[4], float r[3][3]) {  // Eigen toRotationMatrix, q = (w,x,y,z)
    const float w = q[0], x = q[1], y = q[2], z = q[3];
    const float tx = 2 * x, ty = 2 * y, tz = 2 * z;
    const float twx = tx * w, twy = ty * w, twz = tz * w, txx = tx * x, txy = ty * x, txz = tz * x;
    const float tyy = ty * y, tyz = tz * y, tzz = tz * z;
    r[0][0] = 1 - (tyy + tzz), r[0][1] = txy - twz, r[0][2] = txz + twy;
    r[1][0] = txy + twz, r[1][1] = 1 - (txx + tzz), r[1][2] = tyz - twx;
    r[2][0] = txz - twy, r[2][1] = tyz + twx, r[2][2] = 1 - (txx + tyy);
}

void mat_to_quat(const double m[3][3], double q[4]) {  // Shepperd (Eigen Quaternion(Mat3))
    const double tr = m[0][0] + m[1][1] + m[2][2];
    if (tr > 0) {
        double t = std::sqrt(tr + 1.0);
        q[0] = 0.5 * t;
        t = 0.5 / t;
        q[1] = (m[2][1] - m[1][2]) * t;
        q[2] = (m[0][2] - m[2][0]) * t;
        q[3] = (m[1][0] - m[0][1]) * t;
    } else {
        int i = 0;
        if (m[1][1] > m[0][0]) i = 1;
        if (m[2][2] > m[i][i]) i = 2;
        const int j = (i + 1) % 3, k = (j + 1) % 3;
        double t = std::sqrt(m[i][i] - m[j][j] - m[k][k] + 1.0);
        double v[3];
        v[i] = 0.5 * t;
        t = 0.5 / t;
        q[0] = (m[k][j] - m[j][k]) * t;
        v[j] = (m[j][i] + m[i][j]) * t;
        v[k] = (m[k][i] + m[i][k]) * t;
        q[1] = v[0], q[2] = v[1], q[3] = v[2];
    }
    const double n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    for (int k = 0; k < 4; ++k) q[k] /= n;
}

// Symmetric 3x3 eigen-decomposition by cyclic Jacobi (double).
void jacobi3(double a[3][3], double evals[3], double evecs[3][3]) {
    double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    for (int sweep = 0; sweep < 50; ++sweep) {
        const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
        if (off < 1e-30 * (a[0][0] * a[0][0] + a[1][1] * a[1][1] + a[2][2] * a[2][2]) || off == 0.0) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                if (a[p][q] == 0.0) continue;
                const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 3; ++k) {  // A = J^T A J
                    const double akp = a[k][p], akq = a[k][q];
                    a[k][p] = c * akp - s * akq;
                    a[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) {
                    const double apk = a[p][k], aqk = a[q][k];
                    a[p][k] = c * apk - s * aqk;
                    a[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 3; ++k) {
                    const double vkp = v[k][p], vkq = v[k][q];
                    v[k][p] = c * vkp - s * vkq;
                    v[k][q] = s * vkp + c * vkq;
                }
            }
    }
    for (int k = 0; k < 3; ++k) evals[k] = a[k][k];
    std::memcpy(evecs, v, sizeof(v));
}

double ellipsoid_surface(const float s[3]) {  // merge.hpp:20-26 (Thomsen)
    constexpr double p = 1.6075;
    const double a = std::pow((double)s[0], p), b = std::pow((double)s[1], p), c = std::pow((double)s[2], p);
    return 4.0 * M_PI * std::pow((a * b + a * c + b * c) / 3.0, 1.0 / p);
}

void covariance(const G& g, double cov[3][3]) {
    float r[3][3];
    quat_to_mat(g.q, r);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0;
            for (int k = 0; k < 3; ++k) acc += (double)r[i][k] * r[j][k] * (double)g.scale[k] * g.scale[k];
            cov[i][j] = acc;
        }
}

G merge(const G* kids, int n) {  // merge.hpp:86-118
    double w[64], raw_sum = 0;
    for (int i = 0; i < n; ++i) raw_sum += (w[i] = (double)kids[i].falloff * ellipsoid_surface(kids[i].scale));
    for (int i = 0; i < n; ++i) w[i] = raw_sum > 0 ? w[i] / raw_sum : 1.0 / n;
    double mean[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) mean[k] += w[i] * kids[i].mean[k];
    double cov[3][3] = {};
    for (int i = 0; i < n; ++i) {
        double c[3][3];
        covariance(kids[i], c);
        double d[3];
        for (int k = 0; k < 3; ++k) d[k] = kids[i].mean[k] - mean[k];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) cov[a][b] += w[i] * (c[a][b] + d[a] * d[b]);
    }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < a; ++b) cov[a][b] = cov[b][a] = 0.5 * (cov[a][b] + cov[b][a]);
    double ev[3], V[3][3];
    jacobi3(cov, ev, V);
    int idx[3] = {0, 1, 2};
    std::sort(idx, idx + 3, [&](int a, int b) { return ev[a] > ev[b]; });
    double R[3][3];
    G out{};
    for (int c = 0; c < 3; ++c) {
        out.scale[c] = static_cast<float>(std::sqrt(std::max(ev[idx[c]], 1e-12)));
        for (int r = 0; r < 3; ++r) R[r][c] = V[r][idx[c]];
    }
    const double det = R[0][0] * (R[1][1] * R[2][2] - R[1][2] * R[2][1]) -
                       R[0][1] * (R[1][0] * R[2][2] - R[1][2] * R[2][0]) +
                       R[0][2] * (R[1][0] * R[2][1] - R[1][1] * R[2][0]);
    if (det < 0)
        for (int r = 0; r < 3; ++r) R[r][2] = -R[r][2];
    double q[4];
    mat_to_quat(R, q);
    for (int k = 0; k < 4; ++k) out.q[k] = static_cast<float>(q[k]);
    for (int k = 0; k < 3; ++k) out.mean[k] = static_cast<float>(mean[k]);
    for (int k = 0; k < 48; ++k) {
        double acc = 0;
        for (int i = 0; i < n; ++i) acc += w[i] * kids[i].sh[k];
        out.sh[k] = static_cast<float>(acc);
    }
    out.falloff = static_cast<float>(raw_sum / ellipsoid_surface(out.scale));
    return out;
}

// match_orientation (merge.hpp:123-173) over the 24 proper signed permutations.
void match_orientation(G& child, const float pq[4]) {
    static const std::vector<std::array<int, 6>> table = [] {
        std::vector<std::array<int, 6>> t;  // perm[3], sign[3]
        int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
        for (auto& pm : perms)
            for (int sx = -1; sx <= 1; sx += 2)
                for (int sy = -1; sy <= 1; sy += 2)
                    for (int sz = -1; sz <= 1; sz += 2) {
                        int sign[3] = {sx, sy, sz};
                        double m[3][3] = {};
                        for (int col = 0; col < 3; ++col) m[pm[col]][col] = sign[col];
                        double det = m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
                                     m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
                                     m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
                        if (det > 0.5) t.push_back({pm[0], pm[1], pm[2], sx, sy, sz});
                    }
        return t;
    }();
    float r[3][3];
    quat_to_mat(child.q, r);
    float best_score = -1.0f;
    double best_q[4] = {child.q[0], child.q[1], child.q[2], child.q[3]};
    float best_s[3] = {child.scale[0], child.scale[1], child.scale[2]};
    for (const auto& e : table) {
        double rp[3][3];  // r * P, P(perm[col], col) = sign[col]
        for (int row = 0; row < 3; ++row)
            for (int col = 0; col < 3; ++col) rp[row][col] = (double)r[row][e[col]] * e[3 + col];
        double q[4];
        mat_to_quat(rp, q);
        const float score = static_cast<float>(std::fabs(q[0] * pq[0] + q[1] * pq[1] + q[2] * pq[2] + q[3] * pq[3]));
        if (score > best_score) {
            best_score = score;
            std::memcpy(best_q, q, sizeof(q));
            for (int col = 0; col < 3; ++col) best_s[col] = child.scale[e[col]];
        }
    }
    if (best_q[0] * pq[0] + best_q[1] * pq[1] + best_q[2] * pq[2] + best_q[3] * pq[3] < 0)
        for (int k = 0; k < 4; ++k) best_q[k] = -best_q[k];
    for (int k = 0; k < 4; ++k) child.q[k] = static_cast<float>(best_q[k]);
    std::memcpy(child.scale, best_s, sizeof(best_s));
}

struct Box {
    float mn[3], mx[3];
};

Box leaf_aabb(const G& g) {  // build.hpp:20-29
    float r[3][3];
    quat_to_mat(g.q, r);
    Box b;
    for (int k = 0; k < 3; ++k) {
        float var = 0.0f;
        for (int j = 0; j < 3; ++j) var += r[k][j] * r[k][j] * g.scale[j] * g.scale[j];
        const float h = 3.0f * std::sqrt(var);
        b.mn[k] = g.mean[k] - h;
        b.mx[k] = g.mean[k] + h;
    }
    return b;
}

struct Shape {  // binary split tree over ranges of `order`
    uint32_t begin, end;
    int32_t left = -1, right = -1;
};

struct Builder {
    const std::vector<Box>& boxes;
    const std::vector<G>& leaves;
    std::vector<uint32_t>& order;
    Builder(const std::vector<Box>& b, const std::vector<G>& l, std::vector<uint32_t>& o)
        : boxes(b), leaves(l), order(o) {}

    // detail::partition_group (build.hpp:42-65)
    uint32_t partition(uint32_t begin, uint32_t end) {
        const uint32_t n = end - begin;
        Box gb{{INFINITY, INFINITY, INFINITY}, {-INFINITY, -INFINITY, -INFINITY}};
        for (uint32_t i = begin; i < end; ++i) {
            const Box& b = boxes[order[i]];
            for (int k = 0; k < 3; ++k) gb.mn[k] = std::min(gb.mn[k], b.mn[k]), gb.mx[k] = std::max(gb.mx[k], b.mx[k]);
        }
        int axis = 0;
        float best = gb.mx[0] - gb.mn[0];
        for (int k = 1; k < 3; ++k)
            if (gb.mx[k] - gb.mn[k] > best) best = gb.mx[k] - gb.mn[k], axis = k;
        std::vector<float> proj(n);
        for (uint32_t i = 0; i < n; ++i) proj[i] = leaves[order[begin + i]].mean[axis];
        std::vector<float> sorted = proj;
        std::nth_element(sorted.begin(), sorted.begin() + n / 2, sorted.end());
        const float median = sorted[n / 2];
        std::vector<uint32_t> lower, upper;
        lower.reserve(n);
        upper.reserve(n);
        for (uint32_t i = 0; i < n; ++i) (proj[i] < median ? lower : upper).push_back(order[begin + i]);
        if (lower.empty() || upper.empty()) return n / 2;
        std::copy(lower.begin(), lower.end(), order.begin() + begin);
        std::copy(upper.begin(), upper.end(), order.begin() + begin + lower.size());
        return static_cast<uint32_t>(lower.size());
    }

    // Recursive split into a private shape arena (parallel at the top levels).
    int32_t build(std::vector<Shape>& arena, uint32_t begin, uint32_t end, int par_depth) {
        const int32_t me = static_cast<int32_t>(arena.size());
        arena.push_back(Shape{begin, end});
        if (end - begin == 1) return me;
        const uint32_t split = begin + partition(begin, end);
        if (par_depth > 0 && end - begin > 65536) {
            std::vector<Shape> la, ra;
            int32_t lr = -1, rr = -1;
            std::thread tl([&] { lr = build(la, begin, split, par_depth - 1); });
            rr = build(ra, split, end, par_depth - 1);
            tl.join();
            // splice: offset indices
            const int32_t lo = static_cast<int32_t>(arena.size());
            for (auto& s : la) {
                if (s.left >= 0) s.left += lo, s.right += lo;
                arena.push_back(s);
            }
            const int32_t ro = static_cast<int32_t>(arena.size());
            for (auto& s : ra) {
                if (s.left >= 0) s.left += ro, s.right += ro;
                arena.push_back(s);
            }
            arena[me].left = lr + lo;
            arena[me].right = rr + ro;
        } else {
            const int32_t l = build(arena, begin, split, 0);
            const int32_t r = build(arena, split, end, 0);
            arena[me].left = l;
            arena[me].right = r;
        }
        return me;
    }
};

}  // namespace

extern "C" {

uint64_t hs_synth_node_count(uint64_t leaves) { return leaves ? 2 * leaves - 1 : 0; }

float hs_synth_scene_side(uint64_t leaves) {
    const double clusters = std::ceil(static_cast<double>(leaves) / 21.0);
    return static_cast<float>(28.0 * std::sqrt(clusters / 240.0));
}

// City-like leaves: `leaves` Gaussians in 21-leaf clusters over a square of
// side hs_synth_scene_side(leaves) centred at (cx, 0, cz).
static void city_leaves(std::vector<G>& lv, uint64_t leaves, uint64_t seed, float cx, float cz, int nthreads) {
    const uint64_t clusters = (leaves + 20) / 21;
    const float side = hs_synth_scene_side(leaves);
    lv.resize(leaves);
    std::vector<std::thread> pool;
    for (int w = 0; w < nthreads; ++w)
        pool.emplace_back([&, w] {
            for (uint64_t c = w; c < clusters; c += nthreads) {
                Rng rng(seed * 0x632BE59BD9B4E019ull + c * 0x9E3779B97F4A7C15ull + 1);
                float center[3] = {cx + rng.uniform(-0.5f * side, 0.5f * side), rng.uniform(-4.2f, 4.2f),
                                   cz + rng.uniform(-0.5f * side, 0.5f * side)};
                float tone[2][3];
                for (auto& t : tone)
                    for (float& v : t) v = rng.uniform(-1.2f, 1.5f);
                for (uint64_t i = c * 21; i < std::min<uint64_t>(leaves, c * 21 + 21); ++i) {
                    G& g = lv[i];
                    for (int k = 0; k < 3; ++k) g.mean[k] = center[k] + rng.uniform(-0.55f, 0.55f);
                    for (int k = 0; k < 3; ++k) g.scale[k] = rng.uniform(0.06f, 0.2f);
                    float q[4];
                    for (float& v : q) v = rng.normal();
                    const float qn = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
                    for (int k = 0; k < 4; ++k) g.q[k] = q[k] / qn;
                    g.falloff = rng.uniform(0.4f, 0.9f);
                    const float* tn = tone[(i - c * 21) % 2];
                    for (int ch = 0; ch < 3; ++ch) {
                        g.sh[ch] = tn[ch];
                        for (int k = 1; k < 16; ++k) g.sh[k * 3 + ch] = rng.uniform(-0.08f, 0.08f);
                    }
                }
            }
        });
    for (auto& t : pool) t.join();
}

static int thread_count(int threads) {
    return threads > 0 ? threads : std::max(1u, std::thread::hardware_concurrency());
}

hs_status hs_synth_city(uint64_t leaves, uint64_t seed, int threads, const hs_node_soa_out* out) {
    return hs_synth_city_chunk(leaves, seed, 0.0f, 0.0f, threads, out);
}

hs_status hs_synth_city_chunk(uint64_t leaves, uint64_t seed, float cx, float cz, int threads,
                              const hs_node_soa_out* out) {
    if (leaves < 1 || leaves > 0x7fffffffull || !out) return HS_INVALID_ARGUMENT;
    const int nthreads = thread_count(threads);
    std::vector<G> lv;
    city_leaves(lv, leaves, seed, cx, cz, nthreads);
    return hs_synth_build_bvh_internal(lv.data(), leaves, nthreads, out);
}

// make_skybox (scene.hpp:111-137): a shell of mid-gray splats (SH zero) 5 scene
// diameters out, scale = circumference / sqrt(count), falloff 0.7, identity
// rotation; then build_bvh over it, as consolidate does (scene.hpp:256-258).
hs_status hs_synth_skybox(uint64_t count, float scene_diameter, uint64_t seed, const float centroid[3], int threads,
                          const hs_node_soa_out* out) {
    if (!(scene_diameter > 0.0f)) return HS_INVALID_ARGUMENT;  // scene.hpp:115
    if (count < 1 || count > 0x7fffffffull || !out) return HS_INVALID_ARGUMENT;
    const float radius = 5.0f * scene_diameter;
    const float spacing = 2.0f * 3.14159265358979323846f * radius / std::sqrt(static_cast<float>(count));
    Rng rng(seed * 0xD1B54A32D192ED03ull + 7);
    std::vector<G> lv(count);
    for (uint64_t i = 0; i < count; ++i) {
        const float z = 1.0f - 2.0f * rng.u01();
        const float phi = 2.0f * 3.14159265358979323846f * rng.u01();
        const float r = std::sqrt(std::max(0.0f, 1.0f - z * z));
        G& g = lv[i];
        g.mean[0] = centroid[0] + radius * (r * std::cos(phi));
        g.mean[1] = centroid[1] + radius * z;
        g.mean[2] = centroid[2] + radius * (r * std::sin(phi));
        for (float& v : g.scale) v = spacing;
        g.q[0] = 1.0f, g.q[1] = g.q[2] = g.q[3] = 0.0f;
        g.falloff = 0.7f;
        std::fill(std::begin(g.sh), std::end(g.sh), 0.0f);
    }
    return hs_synth_build_bvh_internal(lv.data(), count, thread_count(threads), out);
}

}  // extern "C"

// build_bvh over `leaves` Gaussians (quaternion wxyz) into the caller's SoA.
hs_status hs_synth_build_bvh_internal(const void* leaves_v, uint64_t n, int nthreads, const hs_node_soa_out* out) {
    const G* leaves_p = static_cast<const G*>(leaves_v);
    std::vector<G> leaves(leaves_p, leaves_p + n);
    std::vector<Box> boxes(n);
    for (uint64_t i = 0; i < n; ++i) boxes[i] = leaf_aabb(leaves[i]);
    std::vector<uint32_t> order(n);
    std::iota(order.begin(), order.end(), 0u);
    Builder b(boxes, leaves, order);
    std::vector<Shape> arena;
    arena.reserve(2 * n);
    int par_depth = 0;
    while ((1 << par_depth) < nthreads && par_depth < 6) ++par_depth;
    const int32_t root = b.build(arena, 0, static_cast<uint32_t>(n), par_depth);

    // Stack-order index allocation exactly as build.hpp:101-123.
    const uint64_t nn = 2 * n - 1;
    std::vector<int32_t> shape_of(nn, -1);
    std::vector<uint32_t> parent(nn, 0xFFFFFFFFu), first_child(nn, 0xFFFFFFFFu), child_count(nn, 0);
    std::vector<std::pair<int32_t, uint32_t>> stack{{root, 0u}};
    uint32_t next_free = 1;
    while (!stack.empty()) {
        auto [s, node] = stack.back();
        stack.pop_back();
        shape_of[node] = s;
        if (arena[s].left < 0) continue;
        const uint32_t fc = next_free;
        next_free += 2;
        first_child[node] = fc;
        child_count[node] = 2;
        parent[fc] = node;
        parent[fc + 1] = node;
        stack.push_back({arena[s].right, fc + 1});
        stack.push_back({arena[s].left, fc});
    }

    std::vector<G> g(nn);
    std::vector<Box> bx(nn);
    for (uint64_t i = 0; i < nn; ++i)
        if (child_count[i] == 0) {
            const uint32_t leaf = order[arena[shape_of[i]].begin];
            g[i] = leaves[leaf];
            bx[i] = boxes[leaf];
        }
    // Bottom-up merges: children always have larger indices (build.hpp:125-137).
    // Parallelised per depth level (nodes of one level are independent).
    std::vector<uint32_t> depth(nn, 0);
    uint32_t max_depth = 0;
    for (uint64_t i = 1; i < nn; ++i) max_depth = std::max(max_depth, depth[i] = depth[parent[i]] + 1);
    std::vector<std::vector<uint32_t>> levels(max_depth + 1);
    for (uint64_t i = 0; i < nn; ++i)
        if (child_count[i]) levels[depth[i]].push_back(static_cast<uint32_t>(i));
    auto par = [&](const std::vector<uint32_t>& items, auto&& fn) {
        const std::size_t m = items.size();
        if (m < 4096 || nthreads <= 1) {
            for (uint32_t i : items) fn(i);
            return;
        }
        std::vector<std::thread> pool;
        const std::size_t chunk = (m + nthreads - 1) / nthreads;
        for (int w = 0; w < nthreads; ++w)
            pool.emplace_back([&, w] {
                for (std::size_t k = w * chunk; k < std::min(m, (w + 1) * chunk); ++k) fn(items[k]);
            });
        for (auto& t : pool) t.join();
    };
    for (int d = static_cast<int>(max_depth); d >= 0; --d)
        par(levels[d], [&](uint32_t i) {
            const uint32_t fc = first_child[i], cc = child_count[i];
            g[i] = merge(&g[fc], static_cast<int>(cc));
            Box u = bx[fc];
            for (uint32_t c = 1; c < cc; ++c)
                for (int k = 0; k < 3; ++k)
                    u.mn[k] = std::min(u.mn[k], bx[fc + c].mn[k]), u.mx[k] = std::max(u.mx[k], bx[fc + c].mx[k]);
            bx[i] = u;
        });
    // Root-down orientation matching (build.hpp:139-147).
    for (uint32_t d = 0; d <= max_depth; ++d)
        par(levels[d], [&](uint32_t i) {
            for (uint32_t c = 0; c < child_count[i]; ++c) match_orientation(g[first_child[i] + c], g[i].q);
        });

    for (uint64_t i = 0; i < nn; ++i) {
        out->parent[i] = parent[i];
        out->first_child[i] = first_child[i];
        out->child_count[i] = child_count[i];
        for (int k = 0; k < 3; ++k) {
            out->bmin[3 * i + k] = bx[i].mn[k];
            out->bmax[3 * i + k] = bx[i].mx[k];
            out->mean[3 * i + k] = g[i].mean[k];
            out->scale[3 * i + k] = g[i].scale[k];
        }
        for (int k = 0; k < 4; ++k) out->rot_wxyz[4 * i + k] = g[i].q[k];
        out->falloff[i] = g[i].falloff;
        std::memcpy(out->sh + 48 * i, g[i].sh, 48 * sizeof(float));
    }
    return HS_OK;
}

// consolidate's global root (scene.hpp:264-279, 307-313): the moment-matched merge
// of the k forest roots, their bounds' union, then each forest root re-matched to
// the new root's axis convention.  gin/gout: k records of 59 floats
// {mean3, scale3, quat wxyz 4, falloff, sh48}; root: one record + bounds.
void hs_merge_root_internal(const float* gin, uint32_t k, const float* bmin, const float* bmax, float* root,
                            float* root_bmin, float* root_bmax, float* gout) {
    std::vector<G> kids(k);
    for (uint32_t i = 0; i < k; ++i) std::memcpy(&kids[i], gin + 59 * i, sizeof(G));
    G r = merge(kids.data(), static_cast<int>(k));
    std::memcpy(root, &r, sizeof(G));
    for (int a = 0; a < 3; ++a) {
        root_bmin[a] = INFINITY;
        root_bmax[a] = -INFINITY;
        for (uint32_t i = 0; i < k; ++i) {
            root_bmin[a] = std::min(root_bmin[a], bmin[3 * i + a]);
            root_bmax[a] = std::max(root_bmax[a], bmax[3 * i + a]);
        }
    }
    for (uint32_t i = 0; i < k; ++i) {
        match_orientation(kids[i], r.q);
        std::memcpy(gout + 59 * i, &kids[i], sizeof(G));
    }
}

extern "C" hs_status hs_build_bvh(const float* mean, const float* scale, const float* rot_wxyz, const float* falloff,
                                  const float* sh, uint64_t n, int threads, const hs_node_soa_out* out) {
    // build_bvh (build.hpp:73-79) input checks: non-empty, valid Gaussians, leaf falloff in (0, 1]
    if (n == 0) return HS_EMPTY_SCENE;
    if (n > 0x7fffffffull || !out) return HS_INVALID_ARGUMENT;
    std::vector<G> lv(n);
    for (uint64_t i = 0; i < n; ++i) {
        G& g = lv[i];
        for (int k = 0; k < 3; ++k) g.mean[k] = mean[3 * i + k], g.scale[k] = scale[3 * i + k];
        for (int k = 0; k < 4; ++k) g.q[k] = rot_wxyz[4 * i + k];
        g.falloff = falloff[i];
        std::memcpy(g.sh, sh + 48 * i, sizeof(g.sh));
        if (!(g.falloff > 0.0f && g.falloff <= 1.0f)) return HS_INVALID_ARGUMENT;
        if (!(g.scale[0] > 0.0f && g.scale[1] > 0.0f && g.scale[2] > 0.0f)) return HS_INVALID_ARGUMENT;
    }
    const int nthreads = threads > 0 ? threads : std::max(1u, std::thread::hardware_concurrency());
    return hs_synth_build_bvh_internal(lv.data(), n, nthreads, out);
}
