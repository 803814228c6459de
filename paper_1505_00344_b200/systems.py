"""The paper's three example systems as user-level definitions (expression text + parameters).

These go through the same front end as any user system (state variables with a
right-hand side, parameters with a default and an allowed range). Constants the paper does not
publish are the readings of DESIGN.md (R6 STN-GPe sigmoids, R7/R8 Hodgkin-Huxley).
"""
from dataclasses import dataclass, field
from typing import List, Optional, Tuple


@dataclass
class SystemDef:
    name: str
    var_names: List[str]
    rhs: List[str]
    # (name, default, min, max); None = unbounded
    params: List[Tuple[str, float, Optional[float], Optional[float]]] = field(default_factory=list)

    @property
    def dim(self):
        return len(self.var_names)

    def param_default(self, name):
        for p in self.params:
            if p[0] == name:
                return p[1]
        raise KeyError(name)


def lorenz() -> SystemDef:
    """Lorenz system, PAPER.md:66-77 (Eqs. 3-5); sigma = 10, beta = 8/3."""
    return SystemDef(
        "lorenz", ["x", "y", "z"],
        ["sigma*(y - x)", "x*(r - z) - y", "x*y - beta*z"],
        [("sigma", 10.0, 0.0, 50.0), ("r", 28.0, 0.0, 350.0), ("beta", 8.0 / 3.0, 0.0, 10.0)])


# Reading R6: logistic sigmoids and constants chosen so that the w_ss sweep of
# PAPER.md:47 shows a stable focus (0, 4.9), an oscillation (7.8) and a node pair (11).
STN_DEFAULTS = dict(w_ss=0.0, w_gs=8.971, w_sg=15.168, w_gg=8.502, I=2.216, tau_s=1.0, tau_g=2.77,
                    a_s=2.891, theta_s=2.049, a_g=1.826, theta_g=2.032)


def stn_gpe() -> SystemDef:
    """STN-GPe Wilson-Cowan model, PAPER.md:31-38 (Eqs. 1-2):
    tau_s x' = -x + Z_s(w_ss x - w_gs y + I),  tau_g y' = -y + Z_g(-w_gg y + w_sg x),
    with Z(u) = sigmoid(a (u - theta)) (reading R6)."""
    d = STN_DEFAULTS
    params = [("w_ss", d["w_ss"], 0.0, 15.0)] + [(k, d[k], None, None) for k in
                                                ("w_gs", "w_sg", "w_gg", "I", "tau_s", "tau_g", "a_s", "theta_s",
                                                 "a_g", "theta_g")]
    return SystemDef(
        "stn_gpe", ["x", "y"],
        ["(-x + sigmoid(a_s*(w_ss*x - w_gs*y + I - theta_s)))/tau_s",
         "(-y + sigmoid(a_g*(-w_gg*y + w_sg*x - theta_g)))/tau_g"],
        params)


HH_DEFAULTS = dict(C=1.0, g_na=120.0, g_k=36.0, g_lk=0.3, e_na=115.0, e_k=-12.0, e_lk=10.613,
                   g_syn=0.5, e_syn=10.0, tau_r=0.5, tau_d=3.0, sigma=5.0, theta=20.0)


def hh_ring(n: int = 3, current: float = 10.0) -> SystemDef:
    """Ring of n Hodgkin-Huxley neurons, PAPER.md:109-138 (Eqs. 6-10), 5n state variables
    [V_i, h_i, m_i, n_i, s_i] (reading R11); neuron i receives s of neuron i-1, neuron 1 of neuron n
    (reading R9). Rate functions: shifted Hodgkin-Huxley 1952 set (readings R7, R10); synapse
    constants reading R8; g_syn = 0.5, e_syn = 10, I_j = 10 from PAPER.md:156."""
    names, rhs = [], []
    for i in range(1, n + 1):
        pre = n if i == 1 else i - 1
        V, h, m, nn, s = f"V{i}", f"h{i}", f"m{i}", f"n{i}", f"s{i}"
        names += [V, h, m, nn, s]
        rhs += [
            f"(g_lk*(e_lk - {V}) + {h}*{m}^3*g_na*(e_na - {V}) + {nn}^4*g_k*(e_k - {V})"
            f" + g_syn*(e_syn - {V})*s{pre} + I{i})/C",
            f"0.07*exp(-{V}/20)*(1 - {h}) - {h}/(exp((30 - {V})/10) + 1)",
            f"0.1*vtrap(25 - {V}, 10)*(1 - {m}) - 4*exp(-{V}/18)*{m}",
            f"0.01*vtrap(10 - {V}, 10)*(1 - {nn}) - 0.125*exp(-{V}/80)*{nn}",
            f"sigmoid(sigma*({V} - theta))*(1 - {s})/tau_r - {s}/tau_d",
        ]
    d = HH_DEFAULTS
    params = [(k, d[k], None, None) for k in ("C", "g_na", "g_k", "g_lk", "e_na", "e_k", "e_lk")]
    params += [("g_syn", d["g_syn"], 0.0, 10.0), ("e_syn", d["e_syn"], None, None),
               ("tau_r", d["tau_r"], None, None), ("tau_d", d["tau_d"], None, None),
               ("sigma", d["sigma"], None, None), ("theta", d["theta"], None, None)]
    params += [(f"I{i}", current, -50.0, 100.0) for i in range(1, n + 1)]
    return SystemDef(f"hh_ring{n}", names, rhs, params)


def linear(A) -> SystemDef:
    """x' = A x (closed-form test system)."""
    n = len(A)
    names = [f"x{i}" for i in range(n)]
    rhs = [" + ".join(f"a{i}_{j}*x{j}" for j in range(n)) for i in range(n)]
    params = [(f"a{i}_{j}", float(A[i][j]), None, None) for i in range(n) for j in range(n)]
    return SystemDef("linear", names, rhs, params)


def harmonic(omega: float = 1.0) -> SystemDef:
    """x' = v, v' = -omega^2 x."""
    return SystemDef("harmonic", ["x", "v"], ["v", "-omega^2*x"], [("omega", omega, None, None)])
