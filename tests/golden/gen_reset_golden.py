"""Writes reset_golden.json: the reset redraws of DESIGN.md reading R16,
computed by THIS script's own pure-Python Philox4x32-10 -- independent of oracle/ and of the CUDA path.

The Philox below is checked against the Random123 known-answer vectors (philox_kat.json) before any
value is written. Recipe (readings R5, R16):
  reset number e (0-based) of particle i of a group with IC seed s redraws every state component d
  from word d % 4 of Philox(ctr = {i lo, i hi, d / 4, 2 + e}, key = {s lo, s hi}), and the lifted
  (swept, mode 0) parameter as component dim of the same draw (word dim % 4 of block dim / 4);
  u = (r >> 8) * 2^-24, x = lo + (hi - lo) * u in float32 round-to-nearest, capped at the largest
  float below hi.

Run: python tests/golden/gen_reset_golden.py   (rewrites reset_golden.json next to it)
"""
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
M32 = 0xFFFFFFFF


def philox(ctr, key):
    c = list(ctr)
    k0, k1 = key
    for rnd in range(10):
        if rnd:
            k0 = (k0 + 0x9E3779B9) & M32
            k1 = (k1 + 0xBB67AE85) & M32
        p0 = 0xD2511F53 * c[0]
        p1 = 0xCD9E8D57 * c[2]
        c = [((p1 >> 32) ^ c[1] ^ k0) & M32, p1 & M32, ((p0 >> 32) ^ c[3] ^ k1) & M32, p0 & M32]
    return c


def check_kat():
    kat = json.load(open(os.path.join(HERE, "philox_kat.json")))
    for v in kat["vectors"]:
        out = philox([int(h, 16) for h in v["ctr"]], [int(h, 16) for h in v["key"]])
        assert ["%08x" % o for o in out] == v["out"], v


def in_box(lo, hi, r):
    lo, hi = np.float32(lo), np.float32(hi)
    u = np.float32(r >> 8) * np.float32(2.0 ** -24)
    x = np.float32(lo + np.float32(np.float32(hi - lo) * u))
    top = np.nextafter(hi, np.float32(-np.inf))
    return min(x, top)


def redraw(seed, i, e, lo, hi, sw):
    dim = len(lo)
    key = [seed & M32, seed >> 32]
    words = {}
    for b in range((dim + 1 + 3) // 4):
        words[b] = philox([i & M32, i >> 32, b, 2 + e], key)
    x = [in_box(lo[d], hi[d], words[d // 4][d % 4]) for d in range(dim)]
    out = {"seed": seed, "index": i, "reset": e, "lo": lo, "hi": hi,
           "words": ["%08x" % words[d // 4][d % 4] for d in range(dim)],
           "bits": ["%08x" % int(np.float32(v).view(np.uint32)) for v in x]}
    if sw is not None:
        r = words[dim // 4][dim % 4]
        v = in_box(sw[0], sw[1], r)
        out.update(sweep=list(sw), lifted_word="%08x" % r, lifted_bits="%08x" % int(np.float32(v).view(np.uint32)))
    return out


def main():
    check_kat()
    cases = []
    # STN-GPe 3-D bifurcation (NEXT 4: w_ss swept over [0, 12), IC box (0,1)^2 of PAPER.md:42; bench seed 22)
    for i, e in ((0, 0), (1, 0), (12345, 1), (4194303, 7)):
        cases.append(redraw(22, i, e, [0.0, 0.0], [1.0, 1.0], (0.0, 12.0)))
    # Lorenz r swept over [0, 200) (configs[3]), Fig. 3A box, seed 5
    for i, e in ((0, 0), (7, 2), (16777215, 0)):
        cases.append(redraw(5, i, e, [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0], (0.0, 200.0)))
    # 4 state variables: the lifted component is word 0 of block 1 (a second Philox block)
    cases.append(redraw(0x123456789, 3, 4, [-1.0, -1.0, -1.0, -1.0], [1.0, 1.0, 1.0, 1.0], (2.0, 3.0)))
    # 15-D HH ring box (reading R11): state words span blocks 0-3; the lifted one is word 3 of block 3
    cases.append(redraw(4, 99, 1, [-20.0, 0, 0, 0, 0] * 3, [100.0, 1, 1, 1, 1] * 3, (0.0, 20.0)))
    # no sweep: state redraw only
    cases.append(redraw(3, 4194304 + 17, 0, [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0], None))
    doc = {"source": "tests/golden/gen_reset_golden.py: its own pure-Python Philox4x32-10 (checked against "
                     "philox_kat.json), not oracle/ and not the CUDA path. Recipe: DESIGN.md readings R5 and R16 "
                     "(PAPER.md:42 reset to new random initial conditions; :54, :95 the lifted parameter is a "
                     "state variable whose IC range is the swept range; :207 a position is chosen when the "
                     "particle is first initialized or reset).",
           "cases": cases}
    with open(os.path.join(HERE, "reset_golden.json"), "w") as f:
        json.dump(doc, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
