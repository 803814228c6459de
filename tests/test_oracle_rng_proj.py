"""Pins of the oracle's Philox, initial-condition sampling, sweep values, projection and binning
(no GPU). Readings R5 (IC recipe), R13 (sweep), R17-R19 (projection / bins) of DESIGN.md."""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def h2u(s):
    return int(s, 16)


def test_philox_known_answers():
    g = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for v in g["vectors"]:
        out = O.philox4x32_10([h2u(c) for c in v["ctr"]], [h2u(k) for k in v["key"]])
        assert [int(o) for o in out] == [h2u(o) for o in v["out"]]


def test_ic_golden_bits():
    g = json.load(open(os.path.join(GOLD, "ic_golden.json")))
    for c in g["ic"]:
        x = O.ic_uniform(c["lo"], c["hi"], c["seed"], c["index"], 1)[:, 0]
        assert [int(b) for b in x.view(np.uint32)] == [h2u(b) for b in c["bits"]]
        if "words" in c:
            w = O.philox4x32_10([c["index"] & 0xffffffff, c["index"] >> 32, 0, 0], [c["seed"], 0])
            assert [int(v) for v in w[:3]] == [h2u(s) for s in c["words"]]
    for c in g["sweep"]:
        v = O.sweep_values(c["lo"], c["hi"], c["mode"], c["seed"], c["index"], 1, c["index"] + 1)
        assert v[0] == pytest.approx(c["value"], rel=1e-7)


def test_ic_inside_half_open_box_and_uniform():
    lo, hi = [-10.0, -30.0, 0.0, 0.25], [10.0, 30.0, 50.0, 0.25000006]
    x = O.ic_uniform(lo, hi, 9, 0, 200000)
    for d in range(4):
        assert np.all(x[d] >= np.float32(lo[d])) and np.all(x[d] < np.float32(hi[d]))
    # uniformity (KS-style bound on the empirical CDF) for the wide dims
    for d in range(3):
        u = np.sort((x[d].astype(np.float64) - lo[d]) / (hi[d] - lo[d]))
        ecdf = np.arange(1, u.size + 1) / u.size
        assert np.max(np.abs(ecdf - u)) < 0.005
    # dims 0..3 use words 0..3 of one Philox block; dims are not all equal
    assert not np.array_equal(x[0], x[1])


def test_ic_offset_consistency_sharding():
    # Sharding invariant: particles [a, b) of a group are the same whether
    # generated in one call or in pieces.
    lo, hi = [0.0, 0.0], [1.0, 1.0]
    whole = O.ic_uniform(lo, hi, 77, 0, 1000)
    parts = np.hstack([O.ic_uniform(lo, hi, 77, a, b - a) for a, b in ((0, 333), (333, 700), (700, 1000))])
    assert np.array_equal(whole, parts)


def test_ic_high_dim_uses_more_blocks():
    lo, hi = [0.0] * 15, [1.0] * 15
    x = O.ic_uniform(lo, hi, 4, 0, 4)
    w = O.philox4x32_10([0, 0, 3, 0], [4, 0])  # dims 12..14 of particle 0 use block 3
    want = ((w[:3] >> 8).astype(np.float32) * np.float32(2 ** -24))
    assert np.array_equal(x[12:15, 0], want)


def test_ic_rejects_empty_box():
    with pytest.raises(ValueError):
        O.ic_uniform([0.5], [0.2], 1, 0, 10)


def test_sweep_linspace_exact():
    v = O.sweep_values(0.0, 200.0, 1, 0, 0, 4, 4)
    # (i + 0.5)/4 = 0.125, 0.375, 0.625, 0.875 exactly; * 200 exact.
    assert list(v) == [25.0, 75.0, 125.0, 175.0]


def test_sweep_uniform_range():
    v = O.sweep_values(0.0, 200.0, 0, 5, 0, 100000, 100000)
    assert v.min() >= 0 and v.max() < 200 and abs(v.mean() - 100) < 1.0


# ----------------------------------------------------------------------------- binning
def test_2d_bin_centres_land_in_their_bins():
    W, H = 7, 5
    view = [-1.0, 2.5, 10.0, 20.0]
    ix, iy = np.meshgrid(np.arange(W), np.arange(H))
    ix, iy = ix.ravel(), iy.ravel()
    cx = -1.0 + (ix + 0.5) * (3.5 / W)
    cy = 10.0 + (iy + 0.5) * (10.0 / H)
    x = np.vstack([cx, cy]).astype(np.float32)
    b = O.bins(x, [0, 1], view, W, H)
    assert np.array_equal(b, iy * W + ix)
    img = O.histogram(x, [0, 1], view, W, H, 2, 1)
    assert img[0].sum() == 0 and np.all(img[1] == 1)


def test_2d_edges_and_non_finite():
    W, H = 4, 4
    view = [0.0, 1.0, 0.0, 1.0]
    pts = np.array([
        [0.0, 0.0],                 # lo edge kept -> bin 0
        [1.0, 0.5],                 # v == hi dropped
        [np.nextafter(np.float32(1), np.float32(0)), 0.5],   # just below hi -> last column
        [-1e-30, 0.5],              # below lo dropped
        [np.nan, 0.5], [np.inf, 0.5], [0.5, -np.inf],
    ], dtype=np.float32).T
    b = O.bins(pts, [0, 1], view, W, H)
    assert list(b) == [0, -1, 2 * W + 3, -1, -1, -1, -1]


def test_histogram_brute_force_small():
    rng = np.random.default_rng(40)
    x = rng.uniform(-1.2, 1.2, (3, 3000)).astype(np.float32)
    x[0, ::97] = np.nan
    W, H = 9, 6
    view = [-1.0, 1.0, -0.5, 1.0]
    img = O.histogram(x, [2, 0], view, W, H, 1, 0)
    brute = np.zeros((H, W), np.uint32)
    for i in range(x.shape[1]):
        a, b = float(x[2, i]), float(x[0, i])
        if not (-1.0 <= a < 1.0 and -0.5 <= b < 1.0):
            continue
        # exact-rational bin: floor((a - lo) / width * W) is the true bin unless rounding puts the
        # value within one float ulp of an edge; those are skipped in the comparison below.
        ia = int(np.floor((a + 1.0) / 2.0 * W))
        ib = int(np.floor((b + 0.5) / 1.5 * H))
        brute[min(ib, H - 1), min(ia, W - 1)] += 1
    assert img.sum() == brute.sum()
    assert np.abs(img[0].astype(int) - brute.astype(int)).sum() <= 2


def test_histogram_count_conservation_and_sweep_axis():
    rng = np.random.default_rng(41)
    x = rng.uniform(-160, 160, (3, 5000)).astype(np.float32)
    sv = rng.uniform(0, 200, 5000).astype(np.float32)
    view = [0.0, 200.0, -160.0, 160.0]
    img = O.histogram(x, [3, 1], view, 64, 32, 1, 0, sweep_vals=sv)
    inside = (sv >= 0) & (sv < 200) & (x[1] >= -160) & (x[1] < 160)
    assert img.sum() == inside.sum()
    b = O.bins(x, [3, 1], view, 64, 32, sweep_vals=sv)
    assert np.array_equal(b >= 0, inside)
    assert np.array_equal(np.bincount(b[b >= 0], minlength=64 * 32).reshape(32, 64), img[0])


def test_3d_projection_golden_pixels():
    g = json.load(open(os.path.join(GOLD, "projection_golden.json")))
    M = np.array(g["pv"], np.float32).ravel()
    pts = np.array([p["x"] for p in g["points"]], np.float32).T
    b = O.bins(pts, [0, 1, 2], M, g["W"], g["H"])
    for k, p in enumerate(g["points"]):
        ix, iy = p["pixel"]
        assert b[k] == iy * g["W"] + ix, p["name"]


def test_3d_behind_camera_dropped():
    g = json.load(open(os.path.join(GOLD, "projection_golden.json")))
    M = np.array(g["pv"], np.float32).ravel()
    # y = -130 is behind the eye at y = -120 (w = y + 120 < 0); y = -120 gives w = 0.
    pts = np.array([[0.0, -130.0, 25.0], [0.0, -120.0, 25.0], [np.nan, 0.0, 0.0]], np.float32).T
    assert list(O.bins(pts, [0, 1, 2], M, 64, 64)) == [-1, -1, -1]


def test_3d_identity_matrix_is_2d_window():
    # With M = identity (w = 1) the 3-D rule is the 2-D rule on the window [-1, 1)^2.
    rng = np.random.default_rng(42)
    x = rng.uniform(-1.5, 1.5, (3, 4000)).astype(np.float32)
    M = np.eye(4, dtype=np.float32).ravel()
    b3 = O.bins(x, [0, 1, 2], M, 32, 16)
    b2 = O.bins(x[:2], [0, 1], [-1.0, 1.0, -1.0, 1.0], 32, 16)
    # both: ix = floor((v+1) * W/2); the 2-D form computes (v+1) * (W/2) the same way
    assert np.array_equal(b3, b2)
