/* oracle_impl.h -- REAL-generic body of the CPU oracle. TEST INFRASTRUCTURE ONLY.
 *
 * Included twice by fireflies_oracle.c, once with REAL=float (SFX=_f32) and once with
 * REAL=double (SFX=_f64). Nothing in here is shared with the CUDA path (see the header
 * comment of fireflies_oracle.c for the independence rules).
 *
 * Every routine is the plain definition, written in the order the paper / DESIGN.md
 * readings state it, with no blocking, fusion or reordering.
 */

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define F(name) CAT(name, SFX)

/* ---------------------------------------------------------------------------------
 * Right-hand sides f(x; p). One function per model of the paper (+ two textbook
 * systems used for closed-form pins). x and dx have length dim, p has the model's
 * parameter vector in the order documented in fireflies_oracle.c.
 * --------------------------------------------------------------------------------- */

/* linear: dx/dt = A x, A row-major dim x dim (closed-form pin system). */
static void F(rhs_linear)(int dim, const REAL* x, const REAL* p, REAL* dx) {
  for (int i = 0; i < dim; ++i) {
    REAL s = 0;
    for (int j = 0; j < dim; ++j) s = s + p[i * dim + j] * x[j];
    dx[i] = s;
  }
}

/* harmonic oscillator: dx/dt = v, dv/dt = -omega^2 x. p = {omega}. */
static void F(rhs_harmonic)(int dim, const REAL* x, const REAL* p, REAL* dx) {
  (void)dim;
  dx[0] = x[1];
  dx[1] = -(p[0] * p[0]) * x[0];
}

/* Lorenz, PAPER.md:66-77 (Eqs. 3-5): x' = sigma (y - x); y' = x (r - z) - y; z' = x y - beta z.
 * p = {sigma, r, beta}. */
static void F(rhs_lorenz)(int dim, const REAL* x, const REAL* p, REAL* dx) {
  (void)dim;
  const REAL sigma = p[0], r = p[1], beta = p[2];
  dx[0] = sigma * (x[1] - x[0]);
  dx[1] = x[0] * (r - x[2]) - x[1];
  dx[2] = x[0] * x[1] - beta * x[2];
}

/* Logistic sigmoid Z(u) = 1 / (1 + exp(-a (u - theta)))  -- reading S6 of DESIGN.md
 * (PAPER.md:40 says only "monotonically increasing sigmoid curves"). */
static REAL F(sigmoid_z)(REAL u, REAL a, REAL theta) {
  return (REAL)1 / ((REAL)1 + EXP(-(a * (u - theta))));
}

/* STN-GPe Wilson-Cowan model, PAPER.md:31-38 (Eqs. 1-2):
 *   tau_s x' = -x + Z_s(w_ss x - w_gs y + I)
 *   tau_g y' = -y + Z_g(-w_gg y + w_sg x)
 * p = {w_ss, w_gs, w_sg, w_gg, I, tau_s, tau_g, a_s, theta_s, a_g, theta_g}. */
static void F(rhs_stn)(int dim, const REAL* x, const REAL* p, REAL* dx) {
  (void)dim;
  const REAL w_ss = p[0], w_gs = p[1], w_sg = p[2], w_gg = p[3], I = p[4];
  const REAL tau_s = p[5], tau_g = p[6], a_s = p[7], th_s = p[8], a_g = p[9], th_g = p[10];
  const REAL zs = F(sigmoid_z)(w_ss * x[0] - w_gs * x[1] + I, a_s, th_s);
  const REAL zg = F(sigmoid_z)(-(w_gg * x[1]) + w_sg * x[0], a_g, th_g);
  dx[0] = (-x[0] + zs) / tau_s;
  dx[1] = (-x[1] + zg) / tau_g;
}

/* vtrap(x, y) = x / (exp(x / y) - 1), the removable-singularity form of the HH alpha_m and
 * alpha_n rates (reading R10). For |x/y| < 0.1 the Taylor series
 * y (1 - u/2 + u^2/12 - u^4/720), u = x/y, is used instead (truncation error < 4e-11 rel). */
static REAL F(vtrap)(REAL x, REAL y) {
  const REAL u = x / y;
  if (FABS(u) < (REAL)0.1) {
    const REAL u2 = u * u;
    return y * ((REAL)1 - u / (REAL)2 + u2 / (REAL)12 - (u2 * u2) / (REAL)720);
  }
  return x / (EXP(u) - (REAL)1);
}

/* Hodgkin-Huxley rate functions, "values given in [Hodgkin1952]" in the
 * shifted (rest = 0 mV) convention; exact forms from SPEC.md:492 (reading R7). */
static REAL F(hh_am)(REAL V) { return (REAL)0.1 * F(vtrap)((REAL)25 - V, (REAL)10); }
static REAL F(hh_bm)(REAL V) { return (REAL)4 * EXP(-V / (REAL)18); }
static REAL F(hh_ah)(REAL V) { return (REAL)0.07 * EXP(-V / (REAL)20); }
static REAL F(hh_bh)(REAL V) { return (REAL)1 / (EXP(((REAL)30 - V) / (REAL)10) + (REAL)1); }
static REAL F(hh_an)(REAL V) { return (REAL)0.01 * F(vtrap)((REAL)10 - V, (REAL)10); }
static REAL F(hh_bn)(REAL V) { return (REAL)0.125 * EXP(-V / (REAL)80); }

/* HH ring of N neurons, PAPER.md:109-138 (Eqs. 6-10). State per neuron i (0-based):
 * x[5i+0..4] = V_i, h_i, m_i, n_i, s_i (reading R11).
 *   C V_i' = g_lk (e_lk - V_i) + h_i m_i^3 g_na (e_na - V_i) + n_i^4 g_k (e_k - V_i) + I_syn^i + I_i
 *   h_i' = a_h(V_i)(1 - h_i) - b_h(V_i) h_i      (same for m, n)
 *   I_syn^i = g_syn (e_syn - V_i) s_{(i-1) mod N}  (neuron 0 reads neuron N-1; reading R9)
 *   s_i' = tau_r^-1 (1 + exp(-sigma (V_i - theta)))^-1 (1 - s_i) - tau_d^-1 s_i
 * p = {C, g_na, g_k, g_lk, e_na, e_k, e_lk, g_syn, e_syn, tau_r, tau_d, sigma, theta, I_0..I_{N-1}}. */
static void F(rhs_hh)(int dim, const REAL* x, const REAL* p, REAL* dx) {
  const int N = dim / 5;
  const REAL C = p[0], g_na = p[1], g_k = p[2], g_lk = p[3], e_na = p[4], e_k = p[5], e_lk = p[6];
  const REAL g_syn = p[7], e_syn = p[8], tau_r = p[9], tau_d = p[10], sig = p[11], theta = p[12];
  for (int i = 0; i < N; ++i) {
    const REAL V = x[5 * i + 0], h = x[5 * i + 1], m = x[5 * i + 2], n = x[5 * i + 3], s = x[5 * i + 4];
    const int pre = (i - 1 + N) % N;
    const REAL s_pre = x[5 * pre + 4];
    const REAL I_syn = g_syn * (e_syn - V) * s_pre;
    const REAL I_inj = p[13 + i];
    const REAL i_lk = g_lk * (e_lk - V);
    const REAL i_na = h * (m * m * m) * g_na * (e_na - V);
    const REAL i_k = (n * n * n * n) * g_k * (e_k - V);
    dx[5 * i + 0] = (i_lk + i_na + i_k + I_syn + I_inj) / C;
    dx[5 * i + 1] = F(hh_ah)(V) * ((REAL)1 - h) - F(hh_bh)(V) * h;
    dx[5 * i + 2] = F(hh_am)(V) * ((REAL)1 - m) - F(hh_bm)(V) * m;
    dx[5 * i + 3] = F(hh_an)(V) * ((REAL)1 - n) - F(hh_bn)(V) * n;
    dx[5 * i + 4] = ((REAL)1 / tau_r) * ((REAL)1 / ((REAL)1 + EXP(-(sig * (V - theta))))) * ((REAL)1 - s)
                    - ((REAL)1 / tau_d) * s;
  }
}

/* Front-end coverage system (not from the paper; exercises every builtin function of the
 * expression grammar in include/fireflies.h). p = {a, b}. Pinned by closed-form values at the
 * origin and at three points where every term is non-zero (tests/test_oracle_models.py, Python's
 * math module in double) and by the RK4 pins. */
static void F(rhs_funcs)(int dim, const REAL* v, const REAL* p, REAL* dx) {
  (void)dim;
  const REAL x = v[0], y = v[1], z = v[2], a = p[0], b = p[1];
  const REAL pi = (REAL)3.14159265358979323846, e = (REAL)2.71828182845904523536;
  dx[0] = SIN(a * x) * COS(y) + TANH(z) - POW((REAL)1 + x * x, (REAL)0.75) + pi * (REAL)0.1;
  dx[1] = SQRT((REAL)1 + y * y) - LOG((REAL)2 + SIN(x)) + EXP(-(b * (x * x))) + FABS(z - x) - (y * y * y) / (REAL)10;
  dx[2] = FMIN(x, y) - FMAX(y, z) * ((REAL)1 / ((REAL)1 + EXP(-(x - z)))) + (x + y) / ((REAL)1 + z * z) +
          TAN((REAL)0.3 * z) - e * (REAL)0.05 * z;
}

static int F(rhs_dispatch)(int model, int dim, const REAL* x, const REAL* p, REAL* dx) {
  switch (model) {
    case ORC_LINEAR: F(rhs_linear)(dim, x, p, dx); return 0;
    case ORC_HARMONIC: if (dim != 2) return -1; F(rhs_harmonic)(dim, x, p, dx); return 0;
    case ORC_LORENZ: if (dim != 3) return -1; F(rhs_lorenz)(dim, x, p, dx); return 0;
    case ORC_STN: if (dim != 2) return -1; F(rhs_stn)(dim, x, p, dx); return 0;
    case ORC_HH: if (dim < 5 || dim % 5 != 0) return -1; F(rhs_hh)(dim, x, p, dx); return 0;
    case ORC_FUNCS: if (dim != 3) return -1; F(rhs_funcs)(dim, x, p, dx); return 0;
    default: return -1;
  }
}

/* Public: evaluate f(x; p) once. */
int F(orc_rhs)(int model, int dim, const REAL* x, const REAL* p, REAL* dx) {
  if (dim < 1 || dim > ORC_MAX_DIM) return -1;
  return F(rhs_dispatch)(model, dim, x, p, dx);
}

/* ---------------------------------------------------------------------------------
 * Classical RK4 step ("4th order Runge-Kutta"; tableau):
 *   k1 = f(x), k2 = f(x + h/2 k1), k3 = f(x + h/2 k2), k4 = f(x + h k3)
 *   x' = x + h/6 (k1 + 2 k2 + 2 k3 + k4)
 * --------------------------------------------------------------------------------- */
static void F(rk4_step)(int model, int dim, REAL* x, const REAL* p, REAL h) {
  REAL k1[ORC_MAX_DIM], k2[ORC_MAX_DIM], k3[ORC_MAX_DIM], k4[ORC_MAX_DIM], t[ORC_MAX_DIM];
  const REAL h2 = h / (REAL)2, h6 = h / (REAL)6;
  F(rhs_dispatch)(model, dim, x, p, k1);
  for (int d = 0; d < dim; ++d) t[d] = x[d] + h2 * k1[d];
  F(rhs_dispatch)(model, dim, t, p, k2);
  for (int d = 0; d < dim; ++d) t[d] = x[d] + h2 * k2[d];
  F(rhs_dispatch)(model, dim, t, p, k3);
  for (int d = 0; d < dim; ++d) t[d] = x[d] + h * k3[d];
  F(rhs_dispatch)(model, dim, t, p, k4);
  for (int d = 0; d < dim; ++d) x[d] = x[d] + h6 * (k1[d] + (REAL)2 * k2[d] + (REAL)2 * k3[d] + k4[d]);
}

/* Public: advance n particles (SoA, x[d*pitch + i]) by nsteps RK4 steps of signed size h.
 * The parameter vector p (np entries) is shared; if sweep_idx >= 0, particle i uses
 * p[sweep_idx] = sweep_vals[i] instead (the lifted parameter of PAPER.md:54, :95 -- held
 * fixed, never integrated). Particles are independent, so the OpenMP loop over particles
 * does not change any result. */
int F(orc_rk4)(int model, int dim, REAL* x_soa, int64_t n, int64_t pitch, const REAL* p, int np,
               int sweep_idx, const REAL* sweep_vals, REAL h, int64_t nsteps) {
  if (dim < 1 || dim > ORC_MAX_DIM || np < 0 || np > ORC_MAX_PARAMS || n < 0 || pitch < n) return -1;
  if (sweep_idx >= np || (sweep_idx >= 0 && !sweep_vals)) return -1;
  REAL probe[ORC_MAX_DIM] = {0}, dprobe[ORC_MAX_DIM];
  if (F(rhs_dispatch)(model, dim, probe, p, dprobe) != 0) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    REAL x[ORC_MAX_DIM], pl[ORC_MAX_PARAMS];
    for (int k = 0; k < np; ++k) pl[k] = p[k];
    if (sweep_idx >= 0) pl[sweep_idx] = sweep_vals[i];
    for (int d = 0; d < dim; ++d) x[d] = x_soa[(int64_t)d * pitch + i];
    for (int64_t s = 0; s < nsteps; ++s) F(rk4_step)(model, dim, x, pl, h);
    for (int d = 0; d < dim; ++d) x_soa[(int64_t)d * pitch + i] = x[d];
  }
  return 0;
}

#undef F
