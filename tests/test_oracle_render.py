"""Pins of the oracle's render post-process (SPEC.md:388 falloff) -- no GPU."""
import numpy as np

import oracle as O


def test_single_particle_is_the_sprite():
    img = np.zeros((1, 15, 15), np.uint32)
    img[0, 7, 7] = 1
    rgb = O.render(img, [[1.0, 0.5, 0.25]], 1.0, 3.0)
    yy, xx = np.mgrid[0:15, 0:15]
    r = np.hypot(xx - 7, yy - 7) / 3.0
    sprite = ((1 - np.minimum(r, 1)) ** 2).astype(np.float32)   # (1 - d)^2
    np.testing.assert_allclose(rgb[0], sprite, rtol=1e-7, atol=0)
    np.testing.assert_allclose(rgb[1], 0.5 * sprite.astype(np.float64), rtol=1e-7, atol=1e-12)
    assert rgb[0, 7, 7] == 1.0 and rgb[0, 7, 10] == 0.0 and rgb[0, 7, 9] > 0


def test_additive_blending_and_saturation():
    # "current colour plus the colour contributed": two channels add; 1 caps
    img = np.zeros((2, 9, 9), np.uint32)
    img[0, 4, 4] = 1
    img[1, 4, 4] = 2
    rgb = O.render(img, [[0.1, 0.0, 0.0], [0.2, 0.3, 0.0]], 1.0, 2.0)
    assert rgb[0, 4, 4] == np.float32(0.1 + 0.4) and rgb[1, 4, 4] == np.float32(0.6)
    img[1, 4, 4] = 100
    rgb = O.render(img, [[0.1, 0.0, 0.0], [0.2, 0.3, 0.0]], 1.0, 2.0)
    assert rgb[0, 4, 4] == 1.0 and rgb[1, 4, 4] == 1.0 and rgb[2].max() == 0.0


def test_position_colour_hand_values():
    # colour linear in position: q = min(255, floor(256 clamp((v - lo)/(hi - lo), 0, 1)))
    x = np.array([[0.0, 0.25, 0.999, 1.0, -0.5], [0.5, 0.5, 0.5, 0.5, 0.5]], np.float32)
    c = O.colour_histogram(x, [0, 1], [-1.0, 2.0, 0.0, 1.0], 3, 1, [0.0, 0.0], [1.0, 1.0])
    # bins (window [-1, 2), W = 3): -0.5 -> 0; 0, 0.25, 0.999 -> 1; 1.0 -> 2
    assert list(c[0, 0]) == [0, 0 + 64 + 255, 255]
    assert list(c[1, 0]) == [128, 384, 128] and list(c[2, 0]) == [128, 384, 128]   # 2-D: blue = 128
    rgb = O.render_colour(c, 1.0, 1.0)           # radius 1: centre tap only
    assert rgb[0, 0, 2] == 1.0 and rgb[1, 0, 0] == np.float32(128 / 255)


def test_linearity_below_saturation_and_borders():
    rng = np.random.default_rng(3)
    img = rng.integers(0, 3, (1, 20, 30)).astype(np.uint32)
    a = O.render(img, [[1e-3, 0, 0]], 1.0, 2.5)
    b = O.render(2 * img, [[1e-3, 0, 0]], 1.0, 2.5)
    np.testing.assert_allclose(b, 2 * a, rtol=1e-6, atol=1e-9)
    # brute force with an explicit kernel, edges included
    yy, xx = np.mgrid[-3:4, -3:4]
    k = ((1 - np.minimum(np.hypot(xx, yy) / 2.5, 1)) ** 2).astype(np.float32).astype(np.float64)
    pad = np.pad(img[0].astype(np.float64), 3)
    want = np.zeros((20, 30))
    for dy in range(7):
        for dx in range(7):
            want += k[dy, dx] * pad[dy:dy + 20, dx:dx + 30]
    np.testing.assert_allclose(a[0], np.float32(1e-3) * want, rtol=1e-6)
