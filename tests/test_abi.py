"""CPU tests of the C-ABI library: it loads, exports every symbol include/fireflies.h declares, and
its front end (parse / validate / emit / NVRTC) works without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1505_00344_b200 as FF
from paper_1505_00344_b200 import _abi, systems

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "fireflies.h")).read()
    return sorted(set(re.findall(r"^(?:const char\*|int|ff_status)\s+(ff_\w+)\(", text, re.M)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(_abi.EXPORTS)


def test_library_exports_every_symbol():
    L = _abi.lib()
    for name in header_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True).stdout
    for name in header_functions():
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_abi_version():
    assert FF.ff_abi_version() == 1


@pytest.mark.parametrize("mk", [systems.lorenz, systems.stn_gpe, lambda: systems.hh_ring(3)])
def test_emit_is_deterministic_and_branch_free(mk):
    s = mk()
    a, b = FF.ff_emit_source(s), FF.ff_emit_source(s)
    assert a == b
    body = a[a.index("__device__ __forceinline__ void ff_rhs"):]
    body = body[:body.index("\n}\n")]
    # the generated derivative is straight-line code (no data-dependent branches)
    for kw in ("if", "for", "while", "switch", "?", "goto"):
        assert not re.search(rf"(^|\W){re.escape(kw)}(\W|$)", body.split("\n", 1)[1]), kw
    for i, v in enumerate(s.var_names):
        assert f"dx[{i}] =" in body


def test_emit_contains_equations_and_sweep_variant():
    s = systems.lorenz()
    src = FF.ff_emit_source(s, sweep_param=1)
    assert "(swept: the per-particle value sw is used instead)" in src
    assert "sw" in src[src.index("void ff_rhs_v0(const V* __restrict__"):]
    assert "a.p[1]" not in src[src.index("void ff_rhs_v0(const V* __restrict__"):src.index("per-slot helpers")]


def test_nvrtc_compiles_sm100a_cubin():
    c = FF.ff_compile_cubin(systems.lorenz())
    assert c[:4] == b"\x7fELF"
    # the ELF e_flags carry the SM version; cuobjdump lists the kernels
    path = "/tmp/ff_test_lorenz.cubin"
    open(path, "wb").write(c)
    out = subprocess.run(["cuobjdump", "-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper() or "arch = sm_100" in out
    names = subprocess.run(["cuobjdump", "-symbols", path], capture_output=True, text=True).stdout
    for k in ("ff_init", "ff_step_p1_t256", "ff_step_p2_t256"):
        assert k in names


def status_of(fn, *a):
    with pytest.raises(_abi.FFError) as e:
        fn(*a)
    return e.value.status


def test_parse_errors_have_positions():
    s = systems.SystemDef("t", ["x"], ["x +"], [])
    with pytest.raises(_abi.FFError) as e:
        FF.ff_emit_source(s)
    assert e.value.status == _abi.FF_ERR_PARSE and "end of input" in str(e.value)
    s = systems.SystemDef("t", ["x"], ["sigma*(y-q)"], [("sigma", 1.0, None, None)])
    assert status_of(FF.ff_emit_source, s) == _abi.FF_ERR_UNKNOWN_SYMBOL
    s = systems.SystemDef("t", ["x"], ["foo(x)"], [])
    assert status_of(FF.ff_emit_source, s) == _abi.FF_ERR_PARSE
    s = systems.SystemDef("t", ["x"], ["pow(x)"], [])
    assert status_of(FF.ff_emit_source, s) == _abi.FF_ERR_PARSE
    s = systems.SystemDef("t", ["x"], ["x * (2"], [])
    assert status_of(FF.ff_emit_source, s) == _abi.FF_ERR_PARSE
    s = systems.SystemDef("t", ["x"], ["1.5e"], [])
    assert status_of(FF.ff_emit_source, s) == _abi.FF_ERR_PARSE


def test_validation_errors():
    mk = systems.SystemDef
    assert status_of(FF.ff_emit_source, mk("t", ["x", "x"], ["1", "2"], [])) == _abi.FF_ERR_INVALID_ARG
    assert status_of(FF.ff_emit_source, mk("t", ["x"], ["1"], [("x", 1.0, None, None)])) == _abi.FF_ERR_INVALID_ARG
    assert status_of(FF.ff_emit_source, mk("t", ["pi"], ["1"], [])) == _abi.FF_ERR_INVALID_ARG
    assert status_of(FF.ff_emit_source, mk("t", ["exp"], ["1"], [])) == _abi.FF_ERR_INVALID_ARG
    assert status_of(FF.ff_emit_source, mk("t", ["1x"], ["1"], [])) == _abi.FF_ERR_INVALID_ARG
    assert status_of(FF.ff_emit_source, mk("t", ["x"], ["k"], [("k", 5.0, 0.0, 1.0)])) == _abi.FF_ERR_INVALID_ARG
    assert status_of(FF.ff_emit_source, mk("t", [], [], [])) == _abi.FF_ERR_INVALID_ARG


def test_precedence_and_folding():
    # "-x^2" is -(x^2); integer powers expand to products; exp folds log2(e)
    src = FF.ff_emit_source(systems.SystemDef("t", ["x"], ["-x^2 + exp(-x/2)"], []))
    body = src[src.index("void ff_rhs_v0(const V* __restrict__"):src.index("per-slot helpers")]
    assert "x[0] * x[0]" in body
    assert "-0.721347511f * x[0]" in body and "ff_exp2(t" in body
    src = FF.ff_emit_source(systems.SystemDef("t", ["x"], ["2^3 + x*0 + 2*(3 - x)"], []))
    body = src[src.index("void ff_rhs_v0(const V* __restrict__"):src.index("per-slot helpers")]
    assert "8.0f" in body and "6.0f" in body


def test_create_without_gpu_reports_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_abi.FFError) as e:
        FF.ff_create(systems.lorenz(), 0)
    assert e.value.status == _abi.FF_ERR_CUDA


def test_null_context_rejected():
    L = _abi.lib()
    assert L.ff_step(None, 1, ctypes.c_float(0.01)) == _abi.FF_ERR_INVALID_ARG
    assert L.ff_sync(None) == _abi.FF_ERR_INVALID_ARG
    assert b"ctx is NULL" in L.ff_last_error()
    # the exchange setters (no device needed to reject them)
    assert L.ff_set_exchange(None, 0, 0, None, None, 1.0) == _abi.FF_ERR_INVALID_ARG
    assert L.ff_set_exchange_multicast(None, None) == _abi.FF_ERR_INVALID_ARG
    assert L.ff_set_exchange_push(None, 1, None) == _abi.FF_ERR_INVALID_ARG
    assert L.ff_set_grid_limit(None, 0) == _abi.FF_ERR_INVALID_ARG
    assert L.ff_destroy(None) == _abi.FF_OK


def test_uniform_values_beyond_the_parameter_block_table_still_compile():
    """More loop-invariant values than FFStepArgs::q holds (FF_MAX_DERIVED = 192): the rest are
    computed in the kernel as before; the source still compiles to an sm_100a CUBIN."""
    from paper_1505_00344_b200.systems import SystemDef
    n = 100
    params = [(f"p{k}", 1.0 + k * 1e-3, None, None) for k in range(n)]
    terms = " + ".join(f"p{k}*p{(k + 1) % n}*x + p{k}*p{(k + 2) % n}*x*x" for k in range(n))   # 200 products
    s = SystemDef("many", ["x"], [terms], params)
    src = FF.ff_emit_source(s)
    assert "a.q[191]" in src and "a.q[192]" not in src
    assert "const float u" in src                  # the overflow values, computed per thread
    cub = FF.ff_compile_cubin(s)
    assert cub[:4] == b"\x7fELF"


def test_uniform_factor_slots_and_sweep():
    """Components with a parameter-only factor are split (at most 4 slots); a factor that is the
    swept parameter stays in the RHS (it is per particle)."""
    src = FF.ff_emit_source(systems.lorenz())
    assert "FF_SSLOT[FF_DIM] = {0, -1, -1}" in src          # sigma (y - x)
    src = FF.ff_emit_source(systems.lorenz(), sweep_param=0)
    assert "FF_SSLOT[FF_DIM] = {-1, -1, -1}" in src         # sigma swept: not factored
    src = FF.ff_emit_source(systems.hh_ring(3))
    m = re.search(r"FF_SSLOT\[FF_DIM\] = \{([^}]*)\}", src)
    slots = [int(v) for v in m.group(1).split(",")]
    assert [slots[i] for i in (0, 5, 10)] == [0, 0, 0]       # dV/dt = (...)/C: one shared slot
    assert all(v == -1 for i, v in enumerate(slots) if i not in (0, 5, 10))


def test_multi_line_rhs_text_stays_in_its_comment():
    """A right-hand side written over several lines (newlines are whitespace to the tokenizer) compiles:
    the text echoed into the generated source's comments has its control characters blanked."""
    s = systems.SystemDef("ml", ["x", "y"], ["-x\n  + 0.5*y", "x\r\n\t- y\n"], [])
    src = FF.ff_emit_source(s)
    head = src[:src.index("template <class V>")]
    for ln in head.splitlines():
        if "dx/dt" in ln or "dy/dt" in ln:
            assert ln.lstrip().startswith("//")
    assert FF.ff_compile_cubin(s)[:4] == b"\x7fELF"
