"""Random expression systems for front-end fuzzing (test logic: a tiny generator and a numpy
evaluator of the grammar in include/fireflies.h, independent of the library's parser)."""
import math

import numpy as np

UNARY = ["exp", "sin", "cos", "tanh", "sqrt", "abs", "sigmoid", "log"]
BINARY = ["min", "max", "pow"]


def gen_expr(rng, vars_, params, depth=0):
    """Returns (text, python-evaluable function of dict env). Domains kept safe: sqrt/log/pow get
    positive arguments, exp a bounded one."""
    r = rng.random()
    if depth >= 3 or r < 0.25:
        c = rng.random()
        if c < 0.45:
            v = vars_[rng.integers(len(vars_))]
            return v, (lambda e, v=v: e[v])
        if c < 0.7 and params:
            p = params[rng.integers(len(params))]
            return p, (lambda e, p=p: e[p])
        k = float(np.round(rng.uniform(-3, 3), 3))
        return f"({k})", (lambda e, k=k: k)
    if r < 0.6:
        op = "+-*/"[rng.integers(4)]
        a, fa = gen_expr(rng, vars_, params, depth + 1)
        b, fb = gen_expr(rng, vars_, params, depth + 1)
        if op == "/":
            return f"({a})/(1.5 + ({b})^2)", (lambda e: fa(e) / (1.5 + fb(e) ** 2))
        return f"({a}) {op} ({b})", {"+": lambda e: fa(e) + fb(e), "-": lambda e: fa(e) - fb(e),
                                     "*": lambda e: fa(e) * fb(e)}[op]
    if r < 0.7:
        a, fa = gen_expr(rng, vars_, params, depth + 1)
        n = int(rng.integers(2, 4))
        return f"({a})^{n}", (lambda e: fa(e) ** n)
    if r < 0.9:
        f = UNARY[rng.integers(len(UNARY))]
        a, fa = gen_expr(rng, vars_, params, depth + 1)
        if f == "exp":
            return f"exp(0.3*tanh({a}))", (lambda e: math.exp(0.3 * math.tanh(fa(e))))
        if f in ("sqrt", "log"):
            g = math.sqrt if f == "sqrt" else math.log
            return f"{f}(1 + ({a})^2)", (lambda e: g(1 + fa(e) ** 2))
        g = {"sin": math.sin, "cos": math.cos, "tanh": math.tanh, "abs": abs,
             "sigmoid": lambda u: 1 / (1 + math.exp(-u))}[f]
        return f"{f}({a})", (lambda e: g(fa(e)))
    f = BINARY[rng.integers(len(BINARY))]
    a, fa = gen_expr(rng, vars_, params, depth + 1)
    b, fb = gen_expr(rng, vars_, params, depth + 1)
    if f == "pow":
        return f"pow(1 + ({a})^2, 0.5*tanh({b}))", (lambda e: (1 + fa(e) ** 2) ** (0.5 * math.tanh(fb(e))))
    g = min if f == "min" else max
    return f"{f}({a}, {b})", (lambda e: g(fa(e), fb(e)))


def gen_system(seed, dim=None):
    rng = np.random.default_rng(seed)
    dim = dim or int(rng.integers(1, 5))
    vars_ = [f"x{i}" for i in range(dim)]
    params = [f"p{k}" for k in range(int(rng.integers(0, 3)))]
    texts, fns = [], []
    for _ in range(dim):
        t, f = gen_expr(rng, vars_, params)
        texts.append(t)
        fns.append(f)
    pvals = {p: float(np.round(rng.uniform(-2, 2), 3)) for p in params}
    return vars_, texts, fns, params, pvals


def rk4_numpy(fns, vars_, pvals, x0, h, n):
    """Plain float64 RK4 (the classical tableau) of one particle with the generated functions."""
    x = np.array(x0, np.float64)

    def f(y):
        env = dict(pvals)
        env.update({v: y[i] for i, v in enumerate(vars_)})
        return np.array([g(env) for g in fns])

    for _ in range(n):
        k1 = f(x)
        k2 = f(x + h / 2 * k1)
        k3 = f(x + h / 2 * k2)
        k4 = f(x + h * k3)
        x = x + h / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
    return x


def gen_structured(seed):
    """Random systems built from the forms the front end rewrites: kinetic gating
    a (1 - x) - b x, driving-force sums sum c_i (E_i - V) in either orientation, parameter-only
    factors (products, divisions by parameters, negation). Returns the gen_system tuple."""
    rng = np.random.default_rng(1000 + seed)
    dim = int(rng.integers(3, 6))
    vars_ = [f"x{i}" for i in range(dim)]
    params = [f"p{k}" for k in range(4)]
    pvals = {p: float(np.round(rng.uniform(0.5, 2.0), 3)) for p in params}
    texts, fns = [], []

    def var():
        v = vars_[rng.integers(dim)]
        return v, (lambda e, v=v: e[v])

    def pos_term():   # a positive-ish varying coefficient
        v, fv = var()
        k = int(rng.integers(3))
        if k == 0:
            return f"sigmoid({v})", (lambda e: 1 / (1 + math.exp(-fv(e))))
        if k == 1:
            return f"exp(0.2*tanh({v}))", (lambda e: math.exp(0.2 * math.tanh(fv(e))))
        return f"({v})^2", (lambda e: fv(e) ** 2)

    def uni():        # a parameter-only factor
        p = params[rng.integers(4)]
        k = int(rng.integers(3))
        if k == 0:
            return p, (lambda e, p=p: e[p])
        if k == 1:
            q = params[rng.integers(4)]
            return f"{p}*{q}", (lambda e, p=p, q=q: e[p] * e[q])
        return f"(1.5 - {p})", (lambda e, p=p: 1.5 - e[p])

    for i in range(dim):
        form = int(rng.integers(3))
        x = vars_[i]
        if form == 0:     # gating: a (1 - x) - b x  (either order)
            (a, fa), (b, fb) = pos_term(), pos_term()
            if rng.random() < 0.5:
                t, f = f"({a})*(1 - {x}) - ({b})*{x}", (lambda e, fa=fa, fb=fb, x=x: fa(e) * (1 - e[x]) - fb(e) * e[x])
            else:
                t, f = f"-{x}*({b}) + (1 - {x})*({a})", (lambda e, fa=fa, fb=fb, x=x: -e[x] * fb(e) + (1 - e[x]) * fa(e))
        elif form == 1:   # driving forces on one variable V, 2-4 terms, both orientations
            V = vars_[rng.integers(dim)]
            parts, fs = [], []
            for _ in range(int(rng.integers(2, 5))):
                (c, fc), (u, fu) = pos_term(), uni()
                if rng.random() < 0.5:
                    parts.append(f"({c})*({u} - {V})")
                    fs.append(lambda e, fc=fc, fu=fu, V=V: fc(e) * (fu(e) - e[V]))
                else:
                    parts.append(f"- ({V} - {u})*({c})")
                    fs.append(lambda e, fc=fc, fu=fu, V=V: -(e[V] - fu(e)) * fc(e))
            t = " + ".join(parts) + " + p0"
            f = (lambda e, fs=tuple(fs): sum(g(e) for g in fs) + e["p0"])
        else:             # a plain nonlinear term
            (a, fa), (b, fb) = pos_term(), var()
            t, f = f"({a}) - {b}*{x}", (lambda e, fa=fa, fb=fb, x=x: fa(e) - fb(e) * e[x])
        k = int(rng.integers(4))          # parameter-only factor of the whole component
        if k == 1:
            t, f = f"({t})/{params[1]}", (lambda e, f=f: f(e) / e["p1"])
        elif k == 2:
            (u, fu) = uni()
            t, f = f"{u}*({t})", (lambda e, f=f, fu=fu: fu(e) * f(e))
        elif k == 3:
            t, f = f"-({t})*p2", (lambda e, f=f: -f(e) * e["p2"])
        texts.append(t)
        fns.append(f)
    return vars_, texts, fns, params, pvals
