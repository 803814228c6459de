"""The shared-reciprocal quotient of the 3-D projection (ff_div2 and its packed pair form
ff_div2_pair, csrc/device/ff_exact.cuh) equals
div.rn.f32 bit for bit (reading R18: px = (c_x / c_w + 1) * W/2 with a correctly rounded quotient),
on sampled operands inside its fast box, over all float bit patterns, at the box edges and over
the projection's own range. The kernel is compiled here with nvcc from tests/cuda/div_check.cu."""
import ctypes
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    out = tmp_path_factory.mktemp("divchk") / "div_check.so"
    subprocess.run(["nvcc", "-O2", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-o", str(out), os.path.join(HERE, "cuda", "div_check.cu")], check=True)
    return ctypes.CDLL(str(out))


@pytest.mark.gpu
@pytest.mark.parametrize("mode,n", [(0, 1 << 26), (1, 1 << 26), (2, 1 << 22), (3, 1 << 26)])
def test_shared_reciprocal_division_is_div_rn(lib, mode, n):
    out = (ctypes.c_ulonglong * 6)()
    assert lib.div_check(mode, ctypes.c_ulonglong(n), ctypes.c_ulonglong(0x5EED + mode), out) == 0
    bad, fast = out[0], out[1]
    assert bad == 0, f"{bad} mismatches, first (nx, ny, d) bits = {[hex(v) for v in out[2:5]]}"
    if mode in (0, 3):
        assert fast > 0.9 * n and out[5] > 0.8 * n   # the scalar and the packed fast paths really ran
