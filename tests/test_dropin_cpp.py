"""The C++ drop-in header (include/hsplat/gpu.hpp) used like the reference's
hsplat:: API; the binary is built by __graft_entry__.build()."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def test_dropin_header_compiles():
    # compile-only check on CPU (no device calls)
    out = os.path.join(ROOT, "tests", "cpp", "_syntax_check.o")
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{os.path.join(ROOT, 'include')}",
                    os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")], check=True)
    assert not os.path.exists(out)


@pytest.mark.gpu
def test_dropin_cpp_api_on_gpu():
    assert os.path.exists(BIN), "build() compiles tests/cpp/test_dropin"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
