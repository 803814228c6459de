/* fireflies_oracle.c -- the CPU oracle for the Fireflies hot path (arXiv:1505.00344).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_1505_00344_b200/) never imports, links or calls anything under oracle/.
 *
 * Independence: this file shares no code, header, table or constant generator with the
 * CUDA path. It has its own hand-coded right-hand sides (oracle_impl.h), its own
 * Philox4x32-10, its own initial-condition formula and its own projection / binning.
 *
 * Build (see oracle/build.py): gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp
 * -shared -fPIC. FP contraction is off and fast-math is off, so every float operation is one
 * IEEE-754 round-to-nearest operation in program order (x86-64 SSE, no x87 excess precision).
 *
 * What is pinned (tests/test_oracle_*.py) and what is not -- see DESIGN.md "Oracle":
 *   rk4 (all models)       pinned: closed forms (linear, harmonic), order-4 convergence,
 *                          round trip, fixed points
 *   rhs_lorenz             pinned: PAPER.md:87-93 landmarks, analytic fixed points, rhs(1,1,1),
 *                          the homoclinic crossing at r ~ 13.926, chaos at r = 28 and
 *                          the regular window at r ~ 92 by Lyapunov exponents
 *   rhs_hh                 pinned: textbook m,h,n steady states, rest 0 mV,
 *                          onset of repetitive firing ~6.25, the vtrap series
 *                          branch (alpha_m(25) = 1, alpha_n(10) = 0.1, series vs expm1 within its
 *                          truncation term, continuity at |u| = 0.1; reading R10); the synapse
 *                          constants tau_r, tau_d, sigma, theta are unpublished,
 *                          pinned only against PAPER.md:156-158's synchrony and two-spiking cycles
 *                          (the 1-3-2 sequence cycle of :160 is not reproduced) -> "parity
 *                          unpinned" for their values (reading R8)
 *   rhs_funcs              pinned: closed forms at the origin and at 3 points where every term
 *                          is non-zero (Python math, double)
 *   reset / lifted values  pinned: an independent Python Philox4x32-10 golden
 *                          (tests/golden/reset_golden.json), inclusive bounds, epochs, uniformity
 *   rhs_stn                pinned by special cases (w = 0 closed form, forward invariance of
 *                          (0,1)^2 per PAPER.md:40); the sigmoid constants themselves are
 *                          unpublished (reading R6), their values pinned only against the phase
 *                          portraits the paper prints (w_ss = 0 / 7.8 / 11 and the
 *                          Hopf / SNIC order) -- the w_ss = 4.9 limit-cycle pair is not reproduced,
 *                          so "parity unpinned" for the exact values
 *   philox4x32_10          pinned: Random123 known-answer vectors
 *   ic / sweep / project   pinned: bin-centre placement, edge rules, brute force, golden pixels
 *
 * Model ids and parameter vectors:
 *   ORC_LINEAR   (0) dim d, p = A (d*d, row-major)
 *   ORC_HARMONIC (1) dim 2, p = {omega}
 *   ORC_LORENZ   (2) dim 3, p = {sigma, r, beta}
 *   ORC_STN      (3) dim 2, p = {w_ss, w_gs, w_sg, w_gg, I, tau_s, tau_g,
 *                               a_s, theta_s, a_g, theta_g}
 *   ORC_HH       (4) dim 5N, p = {C, g_na, g_k, g_lk, e_na, e_k, e_lk, g_syn, e_syn,
 *                                 tau_r, tau_d, sigma, theta, I_1..I_N}
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define ORC_LINEAR 0
#define ORC_HARMONIC 1
#define ORC_LORENZ 2
#define ORC_STN 3
#define ORC_HH 4
#define ORC_FUNCS 5
#define ORC_MAX_DIM 64
#define ORC_MAX_PARAMS 1024

/* ---- float instantiation (libm single-precision functions) ---- */
#define REAL float
#define SFX _f32
#define EXP expf
#define FABS fabsf
#define SIN sinf
#define COS cosf
#define TAN tanf
#define TANH tanhf
#define POW powf
#define SQRT sqrtf
#define LOG logf
#define FMIN fminf
#define FMAX fmaxf
#include "oracle_impl.h"
#undef REAL
#undef SFX
#undef EXP
#undef FABS
#undef SIN
#undef COS
#undef TAN
#undef TANH
#undef POW
#undef SQRT
#undef LOG
#undef FMIN
#undef FMAX

/* ---- double instantiation ---- */
#define REAL double
#define SFX _f64
#define EXP exp
#define FABS fabs
#define SIN sin
#define COS cos
#define TAN tan
#define TANH tanh
#define POW pow
#define SQRT sqrt
#define LOG log
#define FMIN fmin
#define FMAX fmax
#include "oracle_impl.h"
#undef REAL
#undef SFX
#undef EXP
#undef FABS
#undef SIN
#undef COS
#undef TAN
#undef TANH
#undef POW
#undef SQRT
#undef LOG
#undef FMIN
#undef FMAX

/* =====================================================================================
 * Philox4x32-10 (Salmon et al., SC'11, "Parallel random numbers: as easy as 1, 2, 3";
 * the Random123 reference definition). The paper names no generator (PAPER.md:42 says only
 * "uniform random distribution"); reading R5 fixes Philox4x32-10.
 *   round: (L0, R0, L1, R1) = (c0, c1, c2, c3)
 *     hi0:lo0 = M0 * c0,  hi1:lo1 = M1 * c2
 *     c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
 *   key bump after each of the first 9 rounds: k0 += W0, k1 += W1.
 * ===================================================================================== */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
    const uint64_t p0 = (uint64_t)PHILOX_M0 * c[0];
    const uint64_t p1 = (uint64_t)PHILOX_M1 * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
  }
  out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* Uniform float in [0,1) from one 32-bit word: u = (r >> 8) * 2^-24 (exact in float). */
static float u01_from_word(uint32_t r) { return (float)(r >> 8) * 0x1p-24f; }

/* The largest float strictly below hi (hi finite). */
static float float_below(float hi) { return nextafterf(hi, -INFINITY); }

/* One uniform sample in [lo, hi) per DESIGN.md reading R5:
 *   x = lo + (hi - lo) * u   (three IEEE float ops, in this order)
 *   x = min(x, largest float below hi)   (rounding can otherwise reach hi). */
static float uniform_in_box(float lo, float hi, float u) {
  const float w = hi - lo;
  const float t = w * u;
  float x = lo + t;
  const float top = float_below(hi);
  if (x > top) x = top;
  return x;
}

/* Philox counter layout of DESIGN.md reading R5 (initial conditions of PAPER.md:42, :207):
 *   key = {seed lo32, seed hi32}
 *   ctr = {i lo32, i hi32, d / 4, stream}   i = particle index inside its group
 *   word = d % 4                             stream 0 = IC, 1 = swept parameter */
static uint32_t philox_word(uint64_t seed, uint64_t i, uint32_t block, uint32_t stream, int word) {
  const uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), block, stream};
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t out[4];
  orc_philox4x32_10(ctr, key, out);
  return out[word];
}

/* Public: initial conditions for particles first .. first+count-1 of one group whose IC cube
 * is [lo_d, hi_d) per dimension. Output SoA: out[d*pitch + j] for the j-th particle. */
int orc_ic_uniform_f32(const float* lo, const float* hi, int dim, uint64_t seed, int64_t first,
                       int64_t count, float* out, int64_t pitch) {
  if (dim < 1 || count < 0 || first < 0 || pitch < count) return -1;
  for (int d = 0; d < dim; ++d)
    if (!(lo[d] < hi[d]) || !isfinite(lo[d]) || !isfinite(hi[d])) return -1;
  for (int64_t j = 0; j < count; ++j) {
    const uint64_t i = (uint64_t)(first + j);
    for (int d = 0; d < dim; ++d) {
      const uint32_t r = philox_word(seed, i, (uint32_t)(d / 4), 0u, d % 4);
      out[(int64_t)d * pitch + j] = uniform_in_box(lo[d], hi[d], u01_from_word(r));
    }
  }
  return 0;
}

/* Public: swept-parameter values (each particle has its own fixed value).
 * mode 0: Philox-uniform in [lo, hi) (stream 1, block 0, word 0);
 * mode 1: linspace, v_i = lo + (hi - lo) * u with u = (float)(((double)i + 0.5) / n_group), one
 *         double division rounded once to float (reading R13). */
int orc_sweep_values_f32(float lo, float hi, int mode, uint64_t seed, int64_t first, int64_t count,
                         int64_t n_group, float* out) {
  if (!(lo < hi) || count < 0 || first < 0 || n_group < 1 || first + count > n_group) return -1;
  for (int64_t j = 0; j < count; ++j) {
    const uint64_t i = (uint64_t)(first + j);
    if (mode == 0) {
      out[j] = uniform_in_box(lo, hi, u01_from_word(philox_word(seed, i, 0u, 1u, 0)));
    } else if (mode == 1) {
      /* (i + 0.5) / n in double (exact numerator for i < 2^52), rounded once to float. */
      const float u = (float)(((double)i + 0.5) / (double)n_group);
      out[j] = uniform_in_box(lo, hi, u);
    } else {
      return -1;
    }
  }
  return 0;
}

/* =====================================================================================
 * Projection + density histogram (readings R17-R19).
 * Axis values v_k are picked from the "extended state" = the dim state components followed
 * by the swept value (index dim). Each particle adds 1 to image[colour][iy][ix] if it lands
 * in the window; everything else (non-finite, outside, behind the camera) is dropped.
 *
 * 2-D (n_axes = 2), view = {lo_0, hi_0, lo_1, hi_1}:
 *   keep iff lo_k <= v_k < hi_k for k = 0, 1
 *   s_0 = (float)W / (hi_0 - lo_0), s_1 = (float)H / (hi_1 - lo_1)     (IEEE float ops)
 *   ix = min(floor((v_0 - lo_0) * s_0), W - 1), iy likewise with H
 * 3-D (n_axes = 3), view = row-major 4x4 M (view-projection):
 *   c_r = ((M[r][0] a + M[r][1] b) + M[r][2] c) + M[r][3]   for r = 0 (x), 1 (y), 3 (w);
 *   every product and sum rounded separately, in that order
 *   keep iff c_w > 0;  px = (c_0 / c_w + 1) * (W * 0.5),  py = (c_1 / c_w + 1) * (H * 0.5)
 *   keep iff 0 <= px < W and 0 <= py < H;  ix = floor(px), iy = floor(py)
 * ===================================================================================== */
static int64_t bin_2d(const float* v, const float* view, int W, int H) {
  const float lo0 = view[0], hi0 = view[1], lo1 = view[2], hi1 = view[3];
  if (!(v[0] >= lo0 && v[0] < hi0)) return -1;
  if (!(v[1] >= lo1 && v[1] < hi1)) return -1;
  const float s0 = (float)W / (hi0 - lo0);
  const float s1 = (float)H / (hi1 - lo1);
  const float px = (v[0] - lo0) * s0;
  const float py = (v[1] - lo1) * s1;
  int64_t ix = (int64_t)floorf(px), iy = (int64_t)floorf(py);
  if (ix > W - 1) ix = W - 1;
  if (iy > H - 1) iy = H - 1;
  return iy * (int64_t)W + ix;
}

static float mat_row(const float* M, int r, float a, float b, float c) {
  float acc = M[4 * r + 0] * a;
  const float t1 = M[4 * r + 1] * b;
  acc = acc + t1;
  const float t2 = M[4 * r + 2] * c;
  acc = acc + t2;
  acc = acc + M[4 * r + 3];
  return acc;
}

static int64_t bin_3d(const float* v, const float* M, int W, int H) {
  const float cx = mat_row(M, 0, v[0], v[1], v[2]);
  const float cy = mat_row(M, 1, v[0], v[1], v[2]);
  const float cw = mat_row(M, 3, v[0], v[1], v[2]);
  if (!(cw > 0.0f)) return -1;
  const float nx = cx / cw, ny = cy / cw;
  const float px = (nx + 1.0f) * ((float)W * 0.5f);
  const float py = (ny + 1.0f) * ((float)H * 0.5f);
  if (!(px >= 0.0f && px < (float)W)) return -1;
  if (!(py >= 0.0f && py < (float)H)) return -1;
  const int64_t ix = (int64_t)floorf(px), iy = (int64_t)floorf(py);
  return iy * (int64_t)W + ix;
}

/* Public: bin index (iy*W + ix, within one channel) of each particle, or -1 if dropped. */
int orc_bin_f32(const float* x_soa, int64_t n, int64_t pitch, int dim, const float* sweep_vals,
                const int* axes, int n_axes, const float* view, int W, int H, int64_t* bins) {
  if (n_axes != 2 && n_axes != 3) return -1;
  if (W < 1 || H < 1 || n < 0) return -1;
  for (int k = 0; k < n_axes; ++k) {
    if (axes[k] < 0 || axes[k] > dim) return -1;
    if (axes[k] == dim && !sweep_vals) return -1;
  }
  for (int64_t i = 0; i < n; ++i) {
    float v[3];
    for (int k = 0; k < n_axes; ++k)
      v[k] = (axes[k] == dim) ? sweep_vals[i] : x_soa[(int64_t)axes[k] * pitch + i];
    bins[i] = (n_axes == 2) ? bin_2d(v, view, W, H) : bin_3d(v, view, W, H);
  }
  return 0;
}

/* Public: add 1 to image[colour][bin] for every kept particle (image is C*H*W uint32,
 * caller-initialised; additive blending analogue of PAPER.md:236). */
int orc_histogram_f32(const float* x_soa, int64_t n, int64_t pitch, int dim, const float* sweep_vals,
                      const int* axes, int n_axes, const float* view, int W, int H, int C, int colour,
                      uint32_t* image) {
  if (colour < 0 || colour >= C) return -1;
  for (int64_t i = 0; i < n; ++i) {
    int64_t b;
    float v[3];
    if (n_axes != 2 && n_axes != 3) return -1;
    for (int k = 0; k < n_axes; ++k) {
      if (axes[k] < 0 || axes[k] > dim || (axes[k] == dim && !sweep_vals)) return -1;
      v[k] = (axes[k] == dim) ? sweep_vals[i] : x_soa[(int64_t)axes[k] * pitch + i];
    }
    b = (n_axes == 2) ? bin_2d(v, view, W, H) : bin_3d(v, view, W, H);
    if (b >= 0) image[(int64_t)colour * H * W + b] += 1u;
  }
  return 0;
}

/* =====================================================================================
 * Lifted parameter ("we redefine the system so that the bifurcation parameter (w_ss)
 * is a new state variable, subject to dw_ss/dt = 0. The initial condition range for this new state
 * variable is set to be the range of parameter values that are of interest"; PAPER.md:95 the same
 * for Lorenz r; a particle's position "is chosen when the particle is first
 * initialized (or reset as a result of going out of bounds)"). DESIGN.md readings R13 and R16:
 * the lifted parameter is component number dim of the particle's extended state. Its value after
 * e resets of the particle is
 *   e = 0:            the sweep draw of orc_sweep_values_f32 (mode 0: Philox stream 1 of the
 *                     sweep seed; mode 1: linspace)
 *   e >= 1, mode 0:   the lifted component of the e-th reset draw -- word dim % 4 of
 *                     Philox(ctr {i lo, i hi, dim / 4, 2 + (e - 1)}, key = the group's IC seed),
 *                     u = (r >> 8) 2^-24, v = uniform_in_box(sw_lo, sw_hi, u)  (as every other
 *                     component of that draw, see orc_reset_f32)
 *   e >= 1, mode 1:   unchanged (a linspace sweep is a deterministic grid, not a random initial
 *                     condition: kept fixed as a deliberate extension of the paper)
 * ===================================================================================== */
static float lifted_value(float sw_lo, float sw_hi, int mode, uint64_t sweep_seed, uint64_t ic_seed, int dim,
                          uint64_t i, int64_t n_group, uint32_t epoch) {
  if (mode == 0 && epoch > 0) {
    const uint32_t r = philox_word(ic_seed, i, (uint32_t)(dim / 4), 2u + (epoch - 1u), dim % 4);
    return uniform_in_box(sw_lo, sw_hi, u01_from_word(r));
  }
  if (mode == 0) return uniform_in_box(sw_lo, sw_hi, u01_from_word(philox_word(sweep_seed, i, 0u, 1u, 0)));
  return uniform_in_box(sw_lo, sw_hi, (float)(((double)i + 0.5) / (double)n_group));
}

/* Public: lifted-parameter values of particles first .. first+count-1 of a group whose epochs (resets
 * so far) are epoch[0 .. count-1] (NULL = all 0). */
int orc_lifted_values_f32(float lo, float hi, int mode, uint64_t sweep_seed, uint64_t ic_seed, int dim, int64_t first,
                          int64_t count, int64_t n_group, const uint32_t* epoch, float* out) {
  if (!(lo < hi) || (mode != 0 && mode != 1) || dim < 1 || count < 0 || first < 0 || n_group < 1 ||
      first + count > n_group)
    return -1;
  for (int64_t j = 0; j < count; ++j)
    out[j] = lifted_value(lo, hi, mode, sweep_seed, ic_seed, dim, (uint64_t)(first + j), n_group, epoch ? epoch[j] : 0u);
  return 0;
}

/* =====================================================================================
 * Reset ("Any trajectories that leave this square region, or which have not been reset for
 * more than time T_max, are reset to a new random set of initial conditions";
 * per-variable bounds; reading R16). Applied to particles
 * first_global .. first_global + n - 1 of one group (SoA x[d*pitch + j]):
 *   bad = (bounds given ? some component outside [lo_d, hi_d] (NaN counts as outside)
 *                       : some component non-finite)
 *         or (age on: (t_now - birth[j]) > t_max)      (t_max > 0 and finite = age on)
 *   if bad: e = epoch[j]; epoch[j] = e + 1; birth[j] = t_now;
 *           x_d = uniform_in_box(ic_lo_d, ic_hi_d, u) with u from Philox word d%4 of
 *                 ctr {i lo, i hi, d/4, 2 + e}, key = seed   (stream 2 + e; reading R5)
 *           and, if the group sweeps a parameter (sweep_vals != NULL), the lifted component
 *           sweep_vals[j] = lifted_value(..., epoch e + 1) -- component dim of the same draw in
 *           mode 0, unchanged in mode 1.
 * ===================================================================================== */
int orc_reset_f32(float* x, int64_t n, int64_t pitch, int dim, const float* bound_lo, const float* bound_hi,
                  float t_max, float t_now, float* birth, uint32_t* epoch, const float* ic_lo, const float* ic_hi,
                  uint64_t seed, int64_t first_global, float* sweep_vals, float sw_lo, float sw_hi, int sweep_mode,
                  uint64_t sweep_seed, int64_t n_group) {
  if (dim < 1 || n < 0 || pitch < n || (bound_lo == NULL) != (bound_hi == NULL)) return -1;
  if (sweep_vals && (!(sw_lo < sw_hi) || (sweep_mode != 0 && sweep_mode != 1) || n_group < first_global + n))
    return -1;
  const int age_on = t_max > 0.0f && isfinite(t_max);
  for (int64_t j = 0; j < n; ++j) {
    int bad = 0;
    for (int d = 0; d < dim; ++d) {
      const float v = x[(int64_t)d * pitch + j];
      if (bound_lo) {
        if (!(v >= bound_lo[d] && v <= bound_hi[d])) bad = 1;
      } else {
        if (!isfinite(v)) bad = 1;
      }
    }
    if (age_on && (t_now - birth[j]) > t_max) bad = 1;
    if (!bad) continue;
    const uint32_t e = epoch[j];
    epoch[j] = e + 1u;
    birth[j] = t_now;
    const uint64_t i = (uint64_t)(first_global + j);
    for (int d = 0; d < dim; ++d) {
      const uint32_t r = philox_word(seed, i, (uint32_t)(d / 4), 2u + e, d % 4);
      x[(int64_t)d * pitch + j] = uniform_in_box(ic_lo[d], ic_hi[d], u01_from_word(r));
    }
    if (sweep_vals) sweep_vals[j] = lifted_value(sw_lo, sw_hi, sweep_mode, sweep_seed, seed, dim, i, n_group, e + 1u);
  }
  return 0;
}

/* =====================================================================================
 * Render post-process (reading R24): sprites of radius R pixels
 * centred on their pixel, falloff w(q) = (1 - min(|q|/R, 1))^2 rounded to float,
 * additive blending saturating at 1:
 *   rgb[k][y][x] = min(1, sum_c colour[c][k] * (intensity * sum_{dy,dx} count_c[y+dy][x+dx] w(dx,dy)))
 * taps |dx|, |dy| <= ceil(R) inside the image, dy outer / dx inner, sums in double in this order.
 * ===================================================================================== */
int orc_render_f32(const uint32_t* image, int W, int H, int C, const float* colour, float intensity, float radius,
                   float* rgb) {
  if (W < 1 || H < 1 || C < 1 || !(radius > 0.0f) || radius > 8.0f) return -1;
  const int hw = (int)ceil((double)radius);
  for (int y = 0; y < H; ++y) {
    for (int x = 0; x < W; ++x) {
      double v[3] = {0.0, 0.0, 0.0};
      for (int c = 0; c < C; ++c) {
        double acc = 0.0;
        for (int dy = -hw; dy <= hw; ++dy) {
          for (int dx = -hw; dx <= hw; ++dx) {
            const int yy = y + dy, xx = x + dx;
            if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
            const double r = sqrt((double)(dx * dx + dy * dy)) / (double)radius;
            const double f = 1.0 - (r < 1.0 ? r : 1.0);
            const float w = (float)(f * f);
            acc = acc + (double)image[((int64_t)c * H + yy) * W + xx] * (double)w;
          }
        }
        const double s = (double)intensity * acc;
        for (int k = 0; k < 3; ++k) v[k] = v[k] + (double)colour[3 * c + k] * s;
      }
      for (int k = 0; k < 3; ++k) rgb[((int64_t)k * H + y) * W + x] = (float)(v[k] < 1.0 ? v[k] : 1.0);
    }
  }
  return 0;
}

/* Position-linear colour ("varies linearly as a function of the particle's
 * position"; reading R26): for every particle kept by the binning rule, add
 *   q_k = min(255, floor(256 * clamp((v_k - lo_k) * s_k, 0, 1))),  s_k = 1 / (hi_k - lo_k) (float)
 * to colour[k][bin] for the n_axes projected axes (2-D: q_2 = 128). */
int orc_colour_histogram_f32(const float* x_soa, int64_t n, int64_t pitch, int dim, const float* sweep_vals,
                             const int* axes, int n_axes, const float* view, int W, int H, const float* lo,
                             const float* hi, uint32_t* colour) {
  if (n_axes != 2 && n_axes != 3) return -1;
  float s[3] = {0, 0, 0};
  for (int k = 0; k < n_axes; ++k) {
    if (!(lo[k] < hi[k])) return -1;
    s[k] = 1.0f / (hi[k] - lo[k]);
  }
  for (int64_t i = 0; i < n; ++i) {
    float v[3];
    for (int k = 0; k < n_axes; ++k) {
      if (axes[k] < 0 || axes[k] > dim || (axes[k] == dim && !sweep_vals)) return -1;
      v[k] = (axes[k] == dim) ? sweep_vals[i] : x_soa[(int64_t)axes[k] * pitch + i];
    }
    const int64_t b = (n_axes == 2) ? bin_2d(v, view, W, H) : bin_3d(v, view, W, H);
    if (b < 0) continue;
    for (int k = 0; k < 3; ++k) {
      uint32_t q = 128u;
      if (k < n_axes) {
        float t = (v[k] - lo[k]) * s[k];
        if (!(t > 0.0f)) t = 0.0f;
        if (!(t < 1.0f)) t = 1.0f;
        const float f = floorf(t * 256.0f);
        q = f > 255.0f ? 255u : (uint32_t)f;
      }
      colour[(int64_t)k * H * W + b] += q;
    }
  }
  return 0;
}

/* Render of position-colour sums: rgb_k = min(1, intensity * sum_taps colour_k w / 255) (taps, order
 * and weights as orc_render_f32). */
int orc_render_colour_f32(const uint32_t* colour, int W, int H, float intensity, float radius, float* rgb) {
  if (W < 1 || H < 1 || !(radius > 0.0f) || radius > 8.0f) return -1;
  const int hw = (int)ceil((double)radius);
  for (int k = 0; k < 3; ++k) {
    for (int y = 0; y < H; ++y) {
      for (int x = 0; x < W; ++x) {
        double acc = 0.0;
        for (int dy = -hw; dy <= hw; ++dy) {
          for (int dx = -hw; dx <= hw; ++dx) {
            const int yy = y + dy, xx = x + dx;
            if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
            const double r = sqrt((double)(dx * dx + dy * dy)) / (double)radius;
            const double f = 1.0 - (r < 1.0 ? r : 1.0);
            const float w = (float)(f * f);
            acc = acc + (double)colour[((int64_t)k * H + yy) * W + xx] * (double)w;
          }
        }
        const double v = ((double)intensity * acc) / 255.0;
        rgb[((int64_t)k * H + y) * W + x] = (float)(v < 1.0 ? v : 1.0);
      }
    }
  }
  return 0;
}

int orc_version(void) { return 1; }
