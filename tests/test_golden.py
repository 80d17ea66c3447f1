"""Golden vectors of the reference's third-party libm (tests/golden/glibc_libm.npz,
made by tests/golden/make_golden.py from this image's glibc 2.39): the host still
produces them, the oracle's transition_alpha (lod.hpp:41-45) reproduces them, and the
device's transition_alpha -- the glibc powf replica the split law shares -- matches
them bit for bit."""
import os

import numpy as np
import pytest

from oracle import oracle as orc
from tests.golden import make_golden as mg

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "glibc_libm.npz"))


def bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


def test_host_glibc_reproduces_golden():
    m = mg.libm()
    assert mg.glibc_version() == str(GOLD["glibc"])
    ex = np.array([m.expf(float(v)) for v in GOLD["expf_x"]], np.float32)
    assert np.array_equal(bits(ex), bits(GOLD["expf_y"]))
    ta = mg.transition_alpha_host(m, GOLD["ta_alpha"], GOLD["ta_k"])
    assert np.array_equal(bits(ta), bits(GOLD["ta_out"]))


def test_oracle_transition_alpha_matches_golden():
    out = np.array([orc.transition_alpha(float(a), int(k)) for a, k in zip(GOLD["ta_alpha"], GOLD["ta_k"])],
                   np.float32)
    assert np.array_equal(bits(out), bits(GOLD["ta_out"]))


@pytest.mark.gpu
def test_device_transition_alpha_matches_golden(renderer):
    out = renderer.transition_alpha(GOLD["ta_alpha"], GOLD["ta_k"])
    assert np.array_equal(bits(out), bits(GOLD["ta_out"]))
