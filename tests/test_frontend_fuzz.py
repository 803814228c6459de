"""Front-end fuzzing: random systems from the expression grammar parse, emit deterministic
straight-line CUDA C and (a few) compile to sm_100a CUBINs -- CPU only. The GPU half
(`test_gpu_frontend_fuzz`) integrates them and compares with an independent float64 evaluation."""
import re

import numpy as np
import pytest

import paper_1505_00344_b200 as FF
from fuzz_exprs import gen_system, rk4_numpy
from paper_1505_00344_b200.systems import SystemDef


@pytest.mark.parametrize("seed", range(60))
def test_random_systems_emit(seed):
    vars_, texts, _, params, pvals = gen_system(seed)
    s = SystemDef("fuzz", vars_, texts, [(p, v, None, None) for p, v in pvals.items()])
    a = FF.ff_emit_source(s)
    assert a == FF.ff_emit_source(s)
    body = a[a.index("void ff_rhs_v0(const V* __restrict__"):]
    body = body[:body.index("\n}\n")]
    assert not re.search(r"(^|\W)(if|for|while|switch|goto)(\W|$)", body.split("\n", 1)[1])
    for i in range(len(vars_)):
        assert f"dx[{i}] =" in body


@pytest.mark.parametrize("seed", [0, 7, 21])
def test_random_systems_compile(seed):
    vars_, texts, _, params, pvals = gen_system(seed)
    s = SystemDef("fuzz", vars_, texts, [(p, v, None, None) for p, v in pvals.items()])
    assert FF.ff_compile_cubin(s)[:4] == b"\x7fELF"


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8))
def test_gpu_frontend_fuzz(seed):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    vars_, texts, fns, params, pvals = gen_system(seed)
    s = SystemDef("fuzz", vars_, texts, [(p, v, None, None) for p, v in pvals.items()])
    n, dim = 700, len(vars_)
    ctx = FF.Context(s, [n])
    g = ctx.init_group([-1.0] * dim, [1.0] * dim, n, 1, 0, seed=seed)
    x0 = ctx.read_state(g)
    ctx.step(5, 0.01)
    got = ctx.read_state(g).astype(np.float64)
    h = float(np.float32(0.01))
    for i in range(0, n, 35):
        want = rk4_numpy(fns, vars_, pvals, x0[:, i].astype(np.float64), h, 5)
        err = np.abs(got[:, i] - want) / np.maximum(np.abs(want), 1.0)
        assert err.max() <= 2e-5, (texts, i, got[:, i], want)


# ---------------------------------------------------------------- structured systems (rewrites)
from fuzz_exprs import gen_structured  # noqa: E402


@pytest.mark.parametrize("seed", range(12))
def test_structured_systems_emit_with_rewrites(seed):
    """Systems built from the rewritten forms (gating, driving forces, parameter-only factors): the
    emission is deterministic, splits the factors into slots and stays branch-free."""
    vars_, texts, _, params, pvals = gen_structured(seed)
    s = SystemDef("structured", vars_, texts, [(p, v, None, None) for p, v in pvals.items()])
    a = FF.ff_emit_source(s)
    assert a == FF.ff_emit_source(s)
    slots = [int(v) for v in re.search(r"FF_SSLOT\[FF_DIM\] = \{([^}]*)\}", a).group(1).split(",")]
    assert max(slots) >= 0 and max(slots) < 4
    body = a[a.index("void ff_rhs_v0(const V* __restrict__"):]
    body = body[:body.index("\n}\n")]
    assert not re.search(r"(^|\W)(if|for|while|switch|goto)(\W|$)", body.split("\n", 1)[1])


@pytest.mark.gpu
@pytest.mark.parametrize("balance", ["auto", "0"])
@pytest.mark.parametrize("seed", range(12))
def test_gpu_structured_systems(seed, balance, monkeypatch):
    """The rewritten forms integrate like their plain definitions: GPU vs an independent float64
    RK4 of the expressions as written (with and without exponentials moved to the FMA pipe)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if balance != "auto":
        monkeypatch.setenv("FF_TUNE_EXP2P", balance)
    vars_, texts, fns, params, pvals = gen_structured(seed)
    s = SystemDef("structured", vars_, texts, [(p, v, None, None) for p, v in pvals.items()])
    n, dim = 64 * 1024, len(vars_)   # enough tiles for the pipe-balanced (throughput) variant
    ctx = FF.Context(s, [n])
    g = ctx.init_group([-1.0] * dim, [1.0] * dim, n, 1, 0, seed=seed)
    x0 = ctx.read_state(g)
    ctx.step(5, 0.01)
    got = ctx.read_state(g).astype(np.float64)
    h = float(np.float32(0.01))
    for i in range(0, n, 1111):
        want = rk4_numpy(fns, vars_, pvals, x0[:, i].astype(np.float64), h, 5)
        err = np.abs(got[:, i] - want) / np.maximum(np.abs(want), 1.0)
        assert err.max() <= 2e-5, (texts, i, got[:, i], want)
