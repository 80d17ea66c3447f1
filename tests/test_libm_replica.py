"""The device's expf / powf replicas (paper_2406_12080_b200/csrc/hs_libm.cuh)
compiled for the host and compared bit for bit with this host's glibc —
which is what the reference's std::exp / std::pow call.  expf: every float in
[-104, 0.5] (the blend's argument range) plus a sample of the rest; powf: every
x in [1e-2, 1] for the exponents 1/K, K = 1..17 (the split law and
transition_alpha), plus random (x, y) pairs.  CPU only, ~20 s."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SRC = r"""
#include "hs_libm.cuh"
#include <cmath>
#include <cstdio>
#include <thread>
#include <vector>
#include <atomic>
static const uint64_t ET[32] = HS_EXP2F_TAB_INIT;
static const uint64_t LT[32] = HS_POWF_LOG2_TAB_INIT;
static bool same(float a, float b) { return hs_libm::as_u32(a) == hs_libm::as_u32(b) || (a != a && b != b); }
int main() {
    const int T = std::max(1u, std::thread::hardware_concurrency());
    std::atomic<unsigned long long> bad{0}, n{0};
    std::vector<std::thread> th;
    // expf over [-104, 0.5]: negative floats from -0 to -104 and positives up to 0.5
    const uint32_t neg_hi = hs_libm::as_u32(-104.0f), pos_hi = hs_libm::as_u32(0.5f);
    for (int w = 0; w < T; ++w) th.emplace_back([&, w] {
        unsigned long long b = 0, c = 0;
        for (uint32_t u = 0x80000000u + w; u <= neg_hi; u += T) { float x = hs_libm::as_float(u); c++; b += !same(expf(x), hs_libm::expf_glibc(x, ET)); }
        for (uint32_t u = w; u <= pos_hi; u += T) { float x = hs_libm::as_float(u); c++; b += !same(expf(x), hs_libm::expf_glibc(x, ET)); }
        for (uint64_t u = w; u < (1ull << 32); u += 4099ull * T) { float x = hs_libm::as_float((uint32_t)u); c++; b += !same(expf(x), hs_libm::expf_glibc(x, ET)); }
        bad += b; n += c; });
    for (auto& t : th) t.join();
    printf("expf %llu %llu\n", (unsigned long long)n.load(), (unsigned long long)bad.load());
    bad = 0; n = 0; th.clear();
    const uint32_t lo = hs_libm::as_u32(1e-2f), hi = hs_libm::as_u32(1.0f);
    for (int w = 0; w < T; ++w) th.emplace_back([&, w] {
        unsigned long long b = 0, c = 0;
        for (int K = 1; K <= 17; ++K) { float y = 1.0f / (float)K;
            for (uint32_t u = lo + w; u <= hi; u += T) { float x = hs_libm::as_float(u); c++; const float ref = powf(x, y);
                b += !same(ref, hs_libm::powf_glibc(x, y, LT, ET)); b += !same(ref, hs_libm::powf_glibc_normal(x, y, LT, ET)); } }
        uint64_t s = 0x9E3779B97F4A7C15ull * (w + 1);
        for (int i = 0; i < 2000000; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            float x = hs_libm::as_float((uint32_t)s), y = hs_libm::as_float((uint32_t)(s >> 32)); c++;
            b += !same(powf(x, y), hs_libm::powf_glibc(x, y, LT, ET)); }
        bad += b; n += c; });
    for (auto& t : th) t.join();
    printf("powf %llu %llu\n", (unsigned long long)n.load(), (unsigned long long)bad.load());
    return 0;
}
"""


def test_libm_replicas_match_host_glibc(tmp_path):
    src = tmp_path / "chk.cpp"
    src.write_text(SRC)
    exe = tmp_path / "chk"
    inc = os.path.join(ROOT, "paper_2406_12080_b200", "csrc")
    # -mfma: fma() inlines to vfmadd (any correctly rounded fma is valid); no contraction elsewhere
    flags = ["-O2", "-std=c++17", "-ffp-contract=off", "-pthread"]
    try:
        subprocess.run(["g++", *flags, "-mfma", f"-I{inc}", str(src), "-o", str(exe), "-lm"], check=True)
    except subprocess.CalledProcessError:
        subprocess.run(["g++", *flags, f"-I{inc}", str(src), "-o", str(exe), "-lm"], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True, timeout=600).stdout.split("\n")
    res = {ln.split()[0]: (int(ln.split()[1]), int(ln.split()[2])) for ln in out if ln.strip()}
    assert res["expf"][0] > 1_100_000_000 and res["expf"][1] == 0
    assert res["powf"][0] > 900_000_000 and res["powf"][1] == 0
