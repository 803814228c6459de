"""CPU oracle for the Fireflies hot path (arXiv:1505.00344) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package. The product (paper_1505_00344_b200/) never imports it, and this package
imports nothing from the product: it is a plain, slow C implementation (fireflies_oracle.c,
oracle_impl.h) with its own right-hand sides, RK4, Philox, IC formula and binning, wrapped
here with ctypes + numpy (argument marshalling only).

Pins and the unpinned parts are listed in fireflies_oracle.c's header and DESIGN.md.
"""
import ctypes as C
import os

import numpy as np

from . import build as _build

LINEAR, HARMONIC, LORENZ, STN, HH, FUNCS = 0, 1, 2, 3, 4, 5

# Parameter vector layouts (fireflies_oracle.c header).
PARAMS = {
    HARMONIC: ["omega"],
    LORENZ: ["sigma", "r", "beta"],
    STN: ["w_ss", "w_gs", "w_sg", "w_gg", "I", "tau_s", "tau_g", "a_s", "theta_s", "a_g", "theta_g"],
}


def hh_param_names(n_neurons: int):
    return ["C", "g_na", "g_k", "g_lk", "e_na", "e_k", "e_lk", "g_syn", "e_syn", "tau_r", "tau_d",
            "sigma", "theta"] + [f"I{i + 1}" for i in range(n_neurons)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        # FF_ORACLE_LIB: a timing build of the same source (oracle/build.py build_timing; bench.py only)
        path = os.environ.get("FF_ORACLE_LIB") or _build.build()
        L = C.CDLL(path)
        P = C.c_void_p
        i64 = C.c_int64
        for sfx in ("_f32", "_f64"):
            f = getattr(L, "orc_rhs" + sfx)
            f.argtypes = [C.c_int, C.c_int, P, P, P]
            f.restype = C.c_int
            f = getattr(L, "orc_rk4" + sfx)
            f.argtypes = [C.c_int, C.c_int, P, i64, i64, P, C.c_int, C.c_int, P,
                          C.c_float if sfx == "_f32" else C.c_double, i64]
            f.restype = C.c_int
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_philox4x32_10.restype = None
        L.orc_ic_uniform_f32.argtypes = [P, P, C.c_int, C.c_uint64, i64, i64, P, i64]
        L.orc_ic_uniform_f32.restype = C.c_int
        L.orc_sweep_values_f32.argtypes = [C.c_float, C.c_float, C.c_int, C.c_uint64, i64, i64, i64, P]
        L.orc_sweep_values_f32.restype = C.c_int
        L.orc_bin_f32.argtypes = [P, i64, i64, C.c_int, P, P, C.c_int, P, C.c_int, C.c_int, P]
        L.orc_bin_f32.restype = C.c_int
        L.orc_histogram_f32.argtypes = [P, i64, i64, C.c_int, P, P, C.c_int, P, C.c_int, C.c_int,
                                        C.c_int, C.c_int, P]
        L.orc_histogram_f32.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _suffix(dtype):
    dtype = np.dtype(dtype)
    if dtype == np.float32:
        return "_f32"
    if dtype == np.float64:
        return "_f64"
    raise TypeError(dtype)


def rhs(model: int, x, p, dtype=np.float64):
    """f(x; p) for one point (model ids above)."""
    x = np.ascontiguousarray(x, dtype=dtype)
    p = np.ascontiguousarray(p, dtype=dtype)
    dx = np.empty_like(x)
    rc = getattr(lib(), "orc_rhs" + _suffix(dtype))(model, x.size, _ptr(x), _ptr(p), _ptr(dx))
    if rc != 0:
        raise ValueError("orc_rhs rejected its arguments")
    return dx


def rk4(model: int, x_soa, p, h: float, nsteps: int, sweep_idx: int = -1, sweep_vals=None, dtype=None):
    """Return x after nsteps RK4 steps of signed size h. x_soa: (dim, n) array (not modified).

    dtype defaults to x_soa's dtype (float32 or float64)."""
    x = np.array(x_soa, dtype=dtype if dtype is not None else np.asarray(x_soa).dtype, order="C", copy=True)
    if x.ndim == 1:
        x = x[:, None]
    dim, n = x.shape
    p = np.ascontiguousarray(p, dtype=x.dtype)
    sv = None if sweep_vals is None else np.ascontiguousarray(sweep_vals, dtype=x.dtype)
    if sv is not None and sv.size != n:
        raise ValueError("sweep_vals must have one value per particle")
    rc = getattr(lib(), "orc_rk4" + _suffix(x.dtype))(model, dim, _ptr(x), n, n, _ptr(p), p.size,
                                                     sweep_idx, _ptr(sv), h, nsteps)
    if rc != 0:
        raise ValueError("orc_rk4 rejected its arguments")
    return x


def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.empty(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def ic_uniform(lo, hi, seed: int, first: int, count: int):
    """(dim, count) float32 initial conditions of particles first..first+count-1 of a group."""
    lo = np.ascontiguousarray(lo, dtype=np.float32)
    hi = np.ascontiguousarray(hi, dtype=np.float32)
    out = np.empty((lo.size, count), dtype=np.float32)
    rc = lib().orc_ic_uniform_f32(_ptr(lo), _ptr(hi), lo.size, seed, first, count, _ptr(out), count)
    if rc != 0:
        raise ValueError("orc_ic_uniform_f32 rejected its arguments")
    return out


def sweep_values(lo: float, hi: float, mode: int, seed: int, first: int, count: int, n_group: int):
    out = np.empty(count, dtype=np.float32)
    rc = lib().orc_sweep_values_f32(lo, hi, mode, seed, first, count, n_group, _ptr(out))
    if rc != 0:
        raise ValueError("orc_sweep_values_f32 rejected its arguments")
    return out


def bins(x_soa, axes, view, W: int, H: int, sweep_vals=None):
    """Per-particle bin index iy*W+ix (int64), -1 if dropped. x_soa: (dim, n) float32."""
    x = np.ascontiguousarray(x_soa, dtype=np.float32)
    dim, n = x.shape
    ax = np.ascontiguousarray(axes, dtype=np.int32)
    vw = np.ascontiguousarray(view, dtype=np.float32)
    sv = None if sweep_vals is None else np.ascontiguousarray(sweep_vals, dtype=np.float32)
    out = np.empty(n, dtype=np.int64)
    rc = lib().orc_bin_f32(_ptr(x), n, n, dim, _ptr(sv), _ptr(ax), ax.size, _ptr(vw), W, H, _ptr(out))
    if rc != 0:
        raise ValueError("orc_bin_f32 rejected its arguments")
    return out


def histogram(x_soa, axes, view, W: int, H: int, C_: int, colour: int, image=None, sweep_vals=None):
    """Add one count per kept particle into image (C, H, W) uint32 (allocated if None)."""
    x = np.ascontiguousarray(x_soa, dtype=np.float32)
    dim, n = x.shape
    if image is None:
        image = np.zeros((C_, H, W), dtype=np.uint32)
    assert image.dtype == np.uint32 and image.flags.c_contiguous and image.shape == (C_, H, W)
    ax = np.ascontiguousarray(axes, dtype=np.int32)
    vw = np.ascontiguousarray(view, dtype=np.float32)
    sv = None if sweep_vals is None else np.ascontiguousarray(sweep_vals, dtype=np.float32)
    rc = lib().orc_histogram_f32(_ptr(x), n, n, dim, _ptr(sv), _ptr(ax), ax.size, _ptr(vw), W, H, C_,
                                 colour, _ptr(image))
    if rc != 0:
        raise ValueError("orc_histogram_f32 rejected its arguments")
    return image


def reset(x_soa, bound_lo, bound_hi, t_max, t_now, birth, epoch, ic_lo, ic_hi, seed, first_global=0, sweep=None):
    """Apply the reset rule (fireflies_oracle.c) in place to float32 x_soa (dim, n),
    float32 birth (n) and uint32 epoch (n). bound_lo/hi None = non-finite check only.
    sweep = None, or dict(vals=float32 (n) lifted-parameter values (updated in place), lo, hi, mode,
    seed=sweep seed, n_group=particles in the whole group) -- reset particles redraw the lifted
    parameter too (reading R16)."""
    L = lib()
    if not hasattr(L, "_reset_sig"):
        L.orc_reset_f32.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_float,
                                    C.c_float, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int64,
                                    C.c_void_p, C.c_float, C.c_float, C.c_int, C.c_uint64, C.c_int64]
        L.orc_reset_f32.restype = C.c_int
        L._reset_sig = True
    assert x_soa.dtype == np.float32 and x_soa.flags.c_contiguous
    assert birth.dtype == np.float32 and epoch.dtype == np.uint32
    dim, n = x_soa.shape
    blo = None if bound_lo is None else np.ascontiguousarray(bound_lo, dtype=np.float32)
    bhi = None if bound_hi is None else np.ascontiguousarray(bound_hi, dtype=np.float32)
    lo = np.ascontiguousarray(ic_lo, dtype=np.float32)
    hi = np.ascontiguousarray(ic_hi, dtype=np.float32)
    sv, slo, shi, smode, sseed, ngroup = None, 0.0, 0.0, -1, 0, 0
    if sweep is not None:
        sv = sweep["vals"]
        assert sv.dtype == np.float32 and sv.flags.c_contiguous and sv.shape == (n,)
        slo, shi, smode, sseed = sweep["lo"], sweep["hi"], sweep["mode"], sweep.get("seed", 0)
        ngroup = sweep.get("n_group", first_global + n)
    rc = L.orc_reset_f32(_ptr(x_soa), n, n, dim, _ptr(blo), _ptr(bhi), t_max, t_now, _ptr(birth), _ptr(epoch),
                         _ptr(lo), _ptr(hi), seed, first_global, _ptr(sv), slo, shi, smode, sseed, ngroup)
    if rc != 0:
        raise ValueError("orc_reset_f32 rejected its arguments")
    return x_soa


def lifted_values(lo: float, hi: float, mode: int, sweep_seed: int, ic_seed: int, dim: int, first: int, count: int,
                  n_group: int, epoch=None):
    """Lifted (swept) parameter of particles first..first+count-1 of a group after epoch[j] resets
    (fireflies_oracle.c orc_lifted_values_f32; readings R13, R16)."""
    L = lib()
    L.orc_lifted_values_f32.argtypes = [C.c_float, C.c_float, C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_int64,
                                        C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
    L.orc_lifted_values_f32.restype = C.c_int
    ep = None if epoch is None else np.ascontiguousarray(epoch, dtype=np.uint32)
    assert ep is None or ep.shape == (count,)
    out = np.empty(count, np.float32)
    if L.orc_lifted_values_f32(lo, hi, mode, sweep_seed, ic_seed, dim, first, count, n_group, _ptr(ep),
                               _ptr(out)) != 0:
        raise ValueError("orc_lifted_values_f32 rejected its arguments")
    return out


def render(image, colours, intensity, radius):
    """RGB float32 (3, H, W) of a uint32 count image (C, H, W) (fireflies_oracle.c orc_render_f32)."""
    L = lib()
    L.orc_render_f32.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_float, C.c_float,
                                 C.c_void_p]
    L.orc_render_f32.restype = C.c_int
    img = np.ascontiguousarray(image, dtype=np.uint32)
    C_, H, W = img.shape
    col = np.ascontiguousarray(colours, dtype=np.float32)
    out = np.empty((3, H, W), np.float32)
    if L.orc_render_f32(_ptr(img), W, H, C_, _ptr(col), intensity, radius, _ptr(out)) != 0:
        raise ValueError("orc_render_f32 rejected its arguments")
    return out


def colour_histogram(x_soa, axes, view, W, H, lo, hi, colour=None, sweep_vals=None):
    """Add position-colour sums into colour (3, H, W) uint32 (fireflies_oracle.c)."""
    L = lib()
    L.orc_colour_histogram_f32.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                           C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                           C.c_void_p]
    L.orc_colour_histogram_f32.restype = C.c_int
    x = np.ascontiguousarray(x_soa, dtype=np.float32)
    dim, n = x.shape
    if colour is None:
        colour = np.zeros((3, H, W), np.uint32)
    ax = np.ascontiguousarray(axes, dtype=np.int32)
    vw = np.ascontiguousarray(view, dtype=np.float32)
    lo_a = np.ascontiguousarray(lo, dtype=np.float32)
    hi_a = np.ascontiguousarray(hi, dtype=np.float32)
    sv = None if sweep_vals is None else np.ascontiguousarray(sweep_vals, dtype=np.float32)
    rc = L.orc_colour_histogram_f32(_ptr(x), n, n, dim, _ptr(sv), _ptr(ax), ax.size, _ptr(vw), W, H, _ptr(lo_a),
                                    _ptr(hi_a), _ptr(colour))
    if rc != 0:
        raise ValueError("orc_colour_histogram_f32 rejected its arguments")
    return colour


def render_colour(colour, intensity, radius):
    L = lib()
    L.orc_render_colour_f32.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_float, C.c_float, C.c_void_p]
    L.orc_render_colour_f32.restype = C.c_int
    col = np.ascontiguousarray(colour, dtype=np.uint32)
    _, H, W = col.shape
    out = np.empty((3, H, W), np.float32)
    if L.orc_render_colour_f32(_ptr(col), W, H, intensity, radius, _ptr(out)) != 0:
        raise ValueError("orc_render_colour_f32 rejected its arguments")
    return out
