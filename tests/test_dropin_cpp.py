"""The C++ drop-in header (include/hsplat/gpu.hpp) used like the reference's
hsplat:: API; the binary is built by __graft_entry__.build()."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")
KAT = os.path.join(ROOT, "tests", "cpp", "test_kat")


@pytest.mark.parametrize("src", ["test_dropin.cpp", "test_kat.cpp"])
def test_dropin_header_compiles(src):
    # compile-only check on CPU (no device calls)
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror", f"-I{os.path.join(ROOT, 'include')}",
                    os.path.join(ROOT, "tests", "cpp", src)], check=True)


@pytest.mark.gpu
def test_dropin_cpp_api_on_gpu():
    assert os.path.exists(BIN), "build() compiles tests/cpp/test_dropin"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


@pytest.mark.gpu
def test_reference_kats_through_dropin_on_gpu():
    """The reference's test_lod.cpp / test_render.cpp known-answer tests, on its own
    mt19937_64 fixture streams, through include/hsplat/gpu.hpp on the device."""
    assert os.path.exists(KAT), "build() compiles tests/cpp/test_kat"
    r = subprocess.run([KAT], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "PASS" in r.stdout
