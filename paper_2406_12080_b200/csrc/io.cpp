// io.cpp — hierarchy binary IO and structural validation on host arrays.
//   .h3dg format (io.hpp:342-408): "H3DG", version u32 = 1, node count u64,
//   SH degree u32, then 272 bytes per node: parent u32, first-child u32,
//   child-count u32, AABB 6f (min xyz, max xyz), mean 3f, scale 3f,
//   rotation wxyz 4f, falloff f, SH 48f.  Little-endian.
//   validate_hierarchy (model.hpp:118-139) + validate_gaussian (model.hpp:52-59).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <sstream>
#include <string>
#include <vector>

#include "hsplat_b200_internal.h"

namespace {

void put_msg(char* msg, size_t len, const std::string& s) {
    if (msg && len) {
        std::strncpy(msg, s.c_str(), len - 1);
        msg[len - 1] = 0;
    }
}

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

// ---- camera text (io.hpp:410-511)
struct CamErr {
    hs_status s;
    std::string what;
};

bool read_text(const std::string& path, std::string& out) {  // detail::read_file (io.hpp:37-46)
    std::ifstream f(path, std::ios::binary);
    if (!f.good()) return false;
    std::ostringstream ss;
    ss << f.rdbuf();
    out = ss.str();
    return true;
}

std::vector<std::string> data_lines(const std::string& text) {  // io.hpp:445-456
    std::vector<std::string> out;
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        const std::size_t ns = line.find_first_not_of(" \t");
        if (ns == std::string::npos || line[ns] == '#') continue;
        out.push_back(line);
    }
    return out;
}

// validate_camera (model.hpp:84-91)
bool camera_ok(const hs_camera& c, CamErr& e) {
    auto bad = [&](const char* m) {
        e = {HS_INVALID_ARGUMENT, std::string("InvalidArgument: ") + m};
        return false;
    };
    if (!(c.width > 0 && c.height > 0)) return bad("camera resolution must be positive");
    if (!(c.fx > 0.0f && c.fy > 0.0f)) return bad("camera focal must be positive");
    for (float v : c.w2c)
        if (!std::isfinite(v)) return bad("camera pose must be finite");
    float acc = 0.0f;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            float v = c.w2c[4 * i] * c.w2c[4 * j] + (c.w2c[4 * i + 1] * c.w2c[4 * j + 1] + c.w2c[4 * i + 2] * c.w2c[4 * j + 2]);
            v -= (i == j) ? 1.0f : 0.0f;
            acc += v * v;
        }
    if (!(std::sqrt(acc) < 1e-3f)) return bad("world_to_camera rotation block must be orthonormal");
    return true;
}

// detail::get_camera (io.hpp:431-442): 18 numbers, nothing trailing, then validated
bool get_camera(std::istringstream& ls, const std::string& line, hs_camera& c, CamErr& e) {
    ls >> c.width >> c.height >> c.fx >> c.fy >> c.cx >> c.cy;
    for (int k = 0; k < 12; ++k) ls >> c.w2c[k];
    std::string trailing;
    if (ls.fail() || (ls >> trailing)) {
        e = {HS_MALFORMED_HEADER, "MalformedHeader: expected 18 numbers per camera: " + line};
        return false;
    }
    return camera_ok(c, e);
}

void put_camera(std::ostream& os, const hs_camera& c) {  // io.hpp:423-429
    os << c.width << ' ' << c.height << ' ' << c.fx << ' ' << c.fy << ' ' << c.cx << ' ' << c.cy;
    for (int k = 0; k < 12; ++k) os << ' ' << c.w2c[k];
    os << '\n';
}

bool write_text(const std::string& path, const std::string& bytes, CamErr& e) {  // io.hpp:48-54
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f.good()) {
        e = {HS_IO_FAILURE, "IoFailure: cannot open " + path + " for writing"};
        return false;
    }
    f.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
    f.flush();
    if (!f.good()) {
        e = {HS_IO_FAILURE, "IoFailure: cannot write " + path};
        return false;
    }
    return true;
}

hs_status report(const CamErr& e, char* msg, size_t len) {
    put_msg(msg, len, e.what);
    return e.s;
}

}  // namespace

extern "C" {

hs_status hs_read_cameras(const char* path, hs_camera* out, uint64_t cap, uint64_t* n, char* msg, size_t msg_len) {
    if (!path || !n) return HS_INVALID_ARGUMENT;
    std::string text;
    if (!read_text(path, text)) return report({HS_IO_FAILURE, std::string("IoFailure: cannot open ") + path}, msg, msg_len);
    uint64_t k = 0;
    CamErr e{HS_OK, ""};
    for (const std::string& line : data_lines(text)) {
        std::istringstream ls(line);
        hs_camera c{};
        if (!get_camera(ls, line, c, e)) return report(e, msg, msg_len);
        if (out && k < cap) out[k] = c;
        ++k;
    }
    *n = k;
    return HS_OK;
}

hs_status hs_read_camera_path(const char* path, double* ts, hs_camera* out, uint64_t cap, uint64_t* n, char* msg,
                              size_t msg_len) {
    if (!path || !n) return HS_INVALID_ARGUMENT;
    std::string text;
    if (!read_text(path, text)) return report({HS_IO_FAILURE, std::string("IoFailure: cannot open ") + path}, msg, msg_len);
    uint64_t k = 0;
    double prev = 0.0;
    CamErr e{HS_OK, ""};
    for (const std::string& line : data_lines(text)) {  // io.hpp:498-511
        std::istringstream ls(line);
        double t;
        ls >> t;
        if (ls.fail()) return report({HS_MALFORMED_HEADER, "MalformedHeader: expected a leading timestamp: " + line}, msg, msg_len);
        hs_camera c{};
        if (!get_camera(ls, line, c, e)) return report(e, msg, msg_len);
        if (k > 0 && !(t > prev))
            return report({HS_INVALID_ARGUMENT, "InvalidArgument: timestamps must be strictly increasing"}, msg, msg_len);
        if (k < cap) {
            if (out) out[k] = c;
            if (ts) ts[k] = t;
        }
        prev = t;
        ++k;
    }
    *n = k;
    return HS_OK;
}

hs_status hs_write_cameras(const char* path, const hs_camera* cams, uint64_t n, char* msg, size_t msg_len) {
    if (!path || (n && !cams)) return HS_INVALID_ARGUMENT;
    std::ostringstream os;  // io.hpp:461-467
    os << std::setprecision(9);
    os << "# width height fx fy cx cy  world-to-camera 3x4 row-major\n";
    for (uint64_t i = 0; i < n; ++i) put_camera(os, cams[i]);
    CamErr e{HS_OK, ""};
    if (!write_text(path, os.str(), e)) return report(e, msg, msg_len);
    return HS_OK;
}

hs_status hs_write_camera_path(const char* path, const double* ts, const hs_camera* cams, uint64_t n, char* msg,
                               size_t msg_len) {
    if (!path || (n && (!cams || !ts))) return HS_INVALID_ARGUMENT;
    for (uint64_t i = 1; i < n; ++i)  // io.hpp:478-481
        if (!(ts[i] > ts[i - 1]))
            return report({HS_INVALID_ARGUMENT, "InvalidArgument: timestamps must be strictly increasing"}, msg, msg_len);
    std::ostringstream os;
    os << std::setprecision(17);
    os << "# timestamp  width height fx fy cx cy  world-to-camera 3x4 row-major\n";
    for (uint64_t i = 0; i < n; ++i) {
        os << ts[i] << ' ';
        put_camera(os, cams[i]);
    }
    CamErr e{HS_OK, ""};
    if (!write_text(path, os.str(), e)) return report(e, msg, msg_len);
    return HS_OK;
}

hs_status hs_validate_hierarchy(const hs_node_soa* s, uint64_t n, char* msg, size_t msg_len) {
    auto fail = [&](const char* m) {
        put_msg(msg, msg_len, m);
        return HS_INVALID_ARGUMENT;
    };
    if (n == 0) return fail("hierarchy has no nodes");
    if (s->parent[0] != HS_NO_NODE) return fail("node 0 must be the root");
    for (uint64_t i = 0; i < n; ++i) {
        if (i != 0 && !(s->parent[i] != HS_NO_NODE && s->parent[i] < n))
            return fail("non-root node must have a valid parent");
        const float* mn = s->bmin + 3 * i;
        const float* mx = s->bmax + 3 * i;
        if (!(mn[0] <= mx[0] && mn[1] <= mx[1] && mn[2] <= mx[2])) return fail("node bounds must be a valid box");
        // validate_gaussian (model.hpp:52-59)
        const float* m = s->mean + 3 * i;
        const float* sc = s->scale + 3 * i;
        const float* q = s->rot_wxyz + 4 * i;
        const float f = s->falloff[i];
        if (!(std::isfinite(m[0]) && std::isfinite(m[1]) && std::isfinite(m[2]) && std::isfinite(sc[0]) &&
              std::isfinite(sc[1]) && std::isfinite(sc[2]) && std::isfinite(f)))
            return fail("gaussian has non-finite fields");
        if (!(sc[0] > 0.0f && sc[1] > 0.0f && sc[2] > 0.0f)) return fail("gaussian scale must be > 0");
        // Quaternion::norm over coeffs (x, y, z, w): SSE predux (x*x + z*z) + (y*y + w*w)
        const float qn = std::sqrt((q[1] * q[1] + q[3] * q[3]) + (q[2] * q[2] + q[0] * q[0]));
        if (!(std::fabs(qn - 1.0f) < 1e-3f)) return fail("gaussian rotation must be a unit quaternion");
        if (!(f >= 0.0f)) return fail("gaussian falloff must be >= 0");
        const uint32_t cc = s->child_count[i];
        if (cc == 0) continue;
        const uint32_t fc = s->first_child[i];
        if (!(fc != HS_NO_NODE && (uint64_t)fc + cc <= n)) return fail("child range out of bounds");
        for (uint32_t c = 0; c < cc; ++c) {
            const uint64_t k = (uint64_t)fc + c;
            if (s->parent[k] != (uint32_t)i) return fail("child parent back-pointer mismatch");
            const float* cmn = s->bmin + 3 * k;
            const float* cmx = s->bmax + 3 * k;
            if (!(cmn[0] >= mn[0] && cmn[1] >= mn[1] && cmn[2] >= mn[2] && cmx[0] <= mx[0] && cmx[1] <= mx[1] &&
                  cmx[2] <= mx[2]))
                return fail("parent bounds must contain child bounds");
        }
    }
    return HS_OK;
}

hs_status hs_h3dg_read_header(const char* path, uint64_t* n_nodes, uint32_t* sh_degree) {
    File fh;
    fh.f = std::fopen(path, "rb");
    if (!fh.f) return HS_IO_FAILURE;
    unsigned char hdr[20];
    std::fseek(fh.f, 0, SEEK_END);
    const long size = std::ftell(fh.f);
    std::fseek(fh.f, 0, SEEK_SET);
    if (size < 20 || std::fread(hdr, 1, 20, fh.f) != 20 || std::memcmp(hdr, "H3DG", 4) != 0)
        return HS_MALFORMED_HEADER;
    uint32_t version, degree;
    uint64_t count;
    std::memcpy(&version, hdr + 4, 4);
    std::memcpy(&count, hdr + 8, 8);
    std::memcpy(&degree, hdr + 16, 4);
    if (version != 1) return HS_MALFORMED_HEADER;
    if ((uint64_t)(size - 20) != count * 272) return HS_TRUNCATED_RECORD;
    if (degree > 3) return HS_UNSUPPORTED_SH_DEGREE;
    *n_nodes = count;
    *sh_degree = degree;
    return HS_OK;
}

hs_status hs_h3dg_read(const char* path, const hs_node_soa_out* o, uint64_t n) {
    uint64_t count;
    uint32_t degree;
    hs_status st = hs_h3dg_read_header(path, &count, &degree);
    if (st != HS_OK) return st;
    if (count != n) return HS_DIMENSION_MISMATCH;
    File fh;
    fh.f = std::fopen(path, "rb");
    if (!fh.f) return HS_IO_FAILURE;
    std::fseek(fh.f, 20, SEEK_SET);
    std::vector<unsigned char> rec(272 * 4096);
    for (uint64_t lo = 0; lo < n; lo += 4096) {
        const uint64_t m = std::min<uint64_t>(4096, n - lo);
        if (std::fread(rec.data(), 272, m, fh.f) != m) return HS_TRUNCATED_RECORD;
        for (uint64_t k = 0; k < m; ++k) {
            const unsigned char* r = rec.data() + 272 * k;
            const uint64_t i = lo + k;
            std::memcpy(&o->parent[i], r, 4);
            std::memcpy(&o->first_child[i], r + 4, 4);
            std::memcpy(&o->child_count[i], r + 8, 4);
            std::memcpy(o->bmin + 3 * i, r + 12, 12);
            std::memcpy(o->bmax + 3 * i, r + 24, 12);
            std::memcpy(o->mean + 3 * i, r + 36, 12);
            std::memcpy(o->scale + 3 * i, r + 48, 12);
            std::memcpy(o->rot_wxyz + 4 * i, r + 60, 16);
            std::memcpy(o->falloff + i, r + 76, 4);
            std::memcpy(o->sh + 48 * i, r + 80, 192);
        }
    }
    return HS_OK;
}

hs_status hs_h3dg_write(const char* path, const hs_node_soa* s, uint64_t n, uint32_t sh_degree) {
    File fh;
    fh.f = std::fopen(path, "wb");
    if (!fh.f) return HS_IO_FAILURE;
    unsigned char hdr[20];
    std::memcpy(hdr, "H3DG", 4);
    const uint32_t version = 1;
    std::memcpy(hdr + 4, &version, 4);
    std::memcpy(hdr + 8, &n, 8);
    std::memcpy(hdr + 16, &sh_degree, 4);
    if (std::fwrite(hdr, 1, 20, fh.f) != 20) return HS_IO_FAILURE;
    std::vector<unsigned char> rec(272 * 4096);
    for (uint64_t lo = 0; lo < n; lo += 4096) {
        const uint64_t m = std::min<uint64_t>(4096, n - lo);
        for (uint64_t k = 0; k < m; ++k) {
            unsigned char* r = rec.data() + 272 * k;
            const uint64_t i = lo + k;
            std::memcpy(r, &s->parent[i], 4);
            std::memcpy(r + 4, &s->first_child[i], 4);
            std::memcpy(r + 8, &s->child_count[i], 4);
            std::memcpy(r + 12, s->bmin + 3 * i, 12);
            std::memcpy(r + 24, s->bmax + 3 * i, 12);
            std::memcpy(r + 36, s->mean + 3 * i, 12);
            std::memcpy(r + 48, s->scale + 3 * i, 12);
            std::memcpy(r + 60, s->rot_wxyz + 4 * i, 16);
            std::memcpy(r + 76, s->falloff + i, 4);
            std::memcpy(r + 80, s->sh + 48 * i, 192);
        }
        if (std::fwrite(rec.data(), 272, m, fh.f) != m) return HS_IO_FAILURE;
    }
    if (std::fflush(fh.f) != 0) return HS_IO_FAILURE;
    return HS_OK;
}

}  // extern "C"
