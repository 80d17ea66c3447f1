"""Golden vectors for the third-party libm the reference path calls (glibc 2.39 expf /
powf behind std::exp(float) / std::pow(float, float): render.hpp:209, :223, lod.hpp:44),
taken from THIS image's host glibc through ctypes.  The reference itself cannot be built
here (Eigen3 is absent), so these are the one set of reference-side
outputs that can be pinned as files: tests/test_golden.py checks the host glibc still
produces them, the oracle's transition_alpha against them, and (GPU) the device's
transition_alpha (the powf replica of csrc/hs_libm.cuh) bit for bit.

    python tests/golden/make_golden.py   ->  tests/golden/glibc_libm.npz
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def libm():
    m = ctypes.CDLL("libm.so.6")
    m.expf.argtypes = [ctypes.c_float]
    m.expf.restype = ctypes.c_float
    m.powf.argtypes = [ctypes.c_float, ctypes.c_float]
    m.powf.restype = ctypes.c_float
    return m


def glibc_version():
    c = ctypes.CDLL("libc.so.6")
    c.gnu_get_libc_version.restype = ctypes.c_char_p
    return c.gnu_get_libc_version().decode()


def expf_inputs():
    rng = np.random.default_rng(2406)
    # the blend's power range [-104, 0.5] (dense), its ends, and special values
    x = np.concatenate([rng.uniform(-104.0, 0.5, 3000), rng.uniform(-6.0, 0.0, 1000),
                        [0.0, -0.0, -1e-30, -87.3, -103.97, -103.28, -104.0, 0.5, 88.0, 88.8, -np.inf]])
    return x.astype(np.float32)


def transition_inputs():
    rng = np.random.default_rng(12080)
    a = np.concatenate([rng.uniform(0.0, 0.99, 2000), rng.uniform(0.98, 0.99, 200),
                        [0.0, 1.0 / 255.0, 0.5, 0.99, 0.999, 1.0, -0.5]]).astype(np.float32)
    k = rng.integers(1, 18, a.size).astype(np.int32)
    k[-7:] = [1, 2, 3, 8, 16, 17, 4]
    return a, k


def transition_alpha_host(m, a, k):
    """lod.hpp:41-45: 1 - pow(1 - clamp(a, 0, 0.99), 1 / K), float arithmetic."""
    out = np.empty(a.size, np.float32)
    for i, (ai, ki) in enumerate(zip(a, k)):
        ac = np.float32(min(max(float(ai), 0.0), float(np.float32(0.99))))
        base = np.float32(np.float32(1.0) - ac)
        e = np.float32(np.float32(1.0) / np.float32(ki))
        out[i] = np.float32(1.0) - np.float32(m.powf(base, e))
    return out


def make():
    m = libm()
    x = expf_inputs()
    ex = np.array([m.expf(float(v)) for v in x], np.float32)
    a, k = transition_inputs()
    ta = transition_alpha_host(m, a, k)
    return dict(expf_x=x, expf_y=ex, ta_alpha=a, ta_k=k, ta_out=ta, glibc=np.array(glibc_version()))


if __name__ == "__main__":
    np.savez_compressed(os.path.join(HERE, "glibc_libm.npz"), **make())
    print("wrote", os.path.join(HERE, "glibc_libm.npz"))
