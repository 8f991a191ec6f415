/*
 * fabf_oracle.c -- CPU ORACLE for the fast adaptive bilateral filter of
 * Gavaskar & Chaudhury, "Fast Adaptive Bilateral Filtering", arXiv 1811.02308.
 *
 * THIS FILE IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *   Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
 *   `--impl reference`) may load, call or execute it.  It shares no code, no
 *   header, no table and no constant generator with the CUDA path under
 *   paper_1811_02308_b200/csrc; neither side includes or links the other.
 *
 * Citations: "P:<n>" is a line of /root/reference/PAPER.md (the paper's LaTeX);
 * equation numbers are the paper's as compiled.
 *
 * What it computes (plain, slow, obviously correct):
 *   fabfo_bounds   alpha_i = min, beta_i = max over the window   eq.(8)
 *   fabfo_brute    the adaptive bilateral filter g by brute force eq.(1)-(3)
 *                  P:54-67, with a box spatial kernel (reading R1)
 *   fabfo_fast     the paper's approximation g-hat of eq.(29), per
 *                  pixel, evaluated in __float128:
 *                    mu_k  = sum_{t in Gamma_i} t^k H_i(t)      eq.(22)
 *                            (the stretched moments, summed over the distinct
 *                            values of the window weighted by their counts --
 *                            the histogram h_i of eq.(5) P:184-189 -- and
 *                            cross-checked against the sample-by-sample sum;
 *                            Prop.3 / eq.(24) is checked against this in tests,
 *                            it is not needed to *define* mu)
 *                    c     = A^{-1} mu, A^{-1} by Theorem 1     eq.(19)
 *                    lambda, theta_0                           eq.(25)
 *                    I_0..I_{N+1}                              eq.(28)
 *                            by eq.(31) (two erf), eq.(32), and the recursion
 *                            eq.(30); where eq.(30) is numerically
 *                            unusable (small lambda, reading R9) the
 *                            integral of eq.(28) is evaluated by 64-node
 *                            Gauss-Legendre quadrature instead (its definition).
 *                    g-hat = alpha + (beta-alpha) (sum c_k I_{k+1})/(sum c_k I_k)
 *                                                                eq.(29)
 *                  plus the guard of DESIGN.md reading R7 (T2 <= 0 or kappa > 1e3
 *                  -> the paper's own N=0 value alpha+(beta-alpha) I_1/I_0).
 *
 * Border handling (the paper is silent): half-sample symmetric reflection,
 * DESIGN.md reading R2.  Window: box of half-width rho, (2rho+1)^2 samples,
 * omega == 1 (reading R1; the paper allows any kernel).
 *
 * Precision: every step of fabfo_fast is carried in __float128 (113-bit
 * mantissa) and rounded once to double at the end (reading R6).  fabfo_brute
 * is fp64 with the exponent shifted by the window's smallest (f-theta)^2 so no
 * weight underflows; the ratio eq.(1)/(2) is unchanged by that common factor.
 *
 * Pins (tests/test_oracle_*.py, marker "not gpu"): Hilbert inverse against the
 * exact rational inverse; moment matching residuals; eq.(24) against direct
 * stretched moments; integrals against mpmath quadrature and closed forms;
 * g-hat against an independent projection-identity evaluation; limits
 * (constant window, sigma -> inf, rho = 0); brute force against an independent
 * numpy implementation and its limits.  Nothing here is "parity unpinned".
 */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __float128 qd;

#define FABFO_MAX_N 16
#define FABFO_GL_NODES 64
#define FABFO_KAPPA_MAX 1000.0

/* output code bits (mirrors the meaning documented in DESIGN.md) */
#define FABFO_CODE_IDENTITY 1u /* alpha == beta -> g-hat = f(i) */
#define FABFO_CODE_GUARD 2u    /* guard of reading R7 fired                      */
#define FABFO_CODE_QUAD 4u     /* I_k by quadrature (small lambda), not eq.(30)  */

/* ------------------------------------------------------------------------- */
/* borders: half-sample symmetric reflection (reading R2); one fold suffices   */
/* because the caller guarantees 2*rho+1 <= min(H, W).                         */
static long reflect_index(long i, long n) {
  if (i < 0) return -i - 1;
  if (i >= n) return 2 * n - 1 - i;
  return i;
}

/* gather the (2rho+1)^2 window of pixel (b, y, x) into vals[] */
static int gather_window(const float* img, int H, int W, int rho, long b, long y,
                         long x, float* vals) {
  const float* base = img + b * (long)H * (long)W;
  int n = 0;
  for (long dy = -rho; dy <= rho; ++dy) {
    long yy = reflect_index(y + dy, H);
    for (long dx = -rho; dx <= rho; ++dx) {
      long xx = reflect_index(x + dx, W);
      vals[n++] = base[yy * W + xx];
    }
  }
  return n;
}

/* ------------------------------------------------------------------------- */
/* eq.(8): alpha_i = min Lambda_i, beta_i = max Lambda_i, by scan    */
int fabfo_bounds(const float* img, int B, int H, int W, int rho, long p0, long p1,
                 float* alpha, float* beta) {
  if (!img || !alpha || !beta || B < 1 || H < 1 || W < 1 || rho < 0) return 1;
  if (2 * rho + 1 > H || 2 * rho + 1 > W) return 1;
  long HW = (long)H * W;
  for (long p = p0; p < p1; ++p) {
    long b = p / HW, r = p % HW, y = r / W, x = r % W;
    const float* base = img + b * HW;
    float mn = INFINITY, mx = -INFINITY;
    for (long dy = -rho; dy <= rho; ++dy) {
      long yy = reflect_index(y + dy, H);
      for (long dx = -rho; dx <= rho; ++dx) {
        float v = base[yy * W + reflect_index(x + dx, W)];
        if (v < mn) mn = v;
        if (v > mx) mx = v;
      }
    }
    alpha[p] = mn;
    beta[p] = mx;
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* eq.(1)-(3) P:54-67: brute-force adaptive bilateral filter, box omega.       */
/* phi_i(t) = exp(-t^2 / (2 sigma(i)^2)); weights shifted by the smallest      */
/* exponent in the window (common factor, cancels in the ratio).               */
static int gauss_weights(int rho, double** w);
static int brute_impl(const float* img, const float* theta, const float* sigma, int B,
                      int H, int W, int rho, int gauss, long p0, long p1, double* g) {
  if (!img || !theta || !sigma || !g || B < 1 || H < 1 || W < 1 || rho < 0) return 1;
  double* wts = NULL;
  const int R = gauss ? gauss_weights(rho, &wts) : rho;
  if (R < 0) return 2;
  if (2 * R + 1 > H || 2 * R + 1 > W) {
    free(wts);
    return 1;
  }
  long HW = (long)H * W;
  int n = (2 * R + 1) * (2 * R + 1);
  float* vals = (float*)malloc(sizeof(float) * (size_t)n);
  if (!vals) {
    free(wts);
    return 2;
  }
  for (long p = p0; p < p1; ++p) {
    long b = p / HW, r = p % HW, y = r / W, x = r % W;
    gather_window(img, H, W, R, b, y, x, vals);
    double th = theta[p], s = sigma[p];
    double inv2s2 = 1.0 / (2.0 * s * s);
    double emin = INFINITY;
    for (int j = 0; j < n; ++j) {
      double e = ((double)vals[j] - th) * ((double)vals[j] - th) * inv2s2;
      if (e < emin) emin = e;
    }
    double num = 0.0, den = 0.0;
    for (int j = 0; j < n; ++j) {
      double e = ((double)vals[j] - th) * ((double)vals[j] - th) * inv2s2;
      double w = exp(-(e - emin)) * (wts ? wts[j] : 1.0); /* omega(j): 1 (box) or eq.(4) */
      num += w * (double)vals[j];
      den += w;
    }
    g[p] = num / den;
  }
  free(vals);
  free(wts);
  return 0;
}

int fabfo_brute(const float* img, const float* theta, const float* sigma, int B,
                int H, int W, int rho, long p0, long p1, double* g) {
  return brute_impl(img, theta, sigma, B, H, W, rho, 0, p0, p1, g);
}

/* eq.(1)-(3) with the Gaussian omega of eq.(4) on [-3 rho, 3 rho]^2 (NEXT-1)  */
int fabfo_brute_gauss(const float* img, const float* theta, const float* sigma, int B,
                      int H, int W, int rho, long p0, long p1, double* g) {
  return brute_impl(img, theta, sigma, B, H, W, rho, 1, p0, p1, g);
}

/* ------------------------------------------------------------------------- */
/* exact integer binomial coefficient (small arguments only)                   */
static qd binom_q(int n, int k) {
  if (k < 0 || k > n) return 0;
  unsigned __int128 c = 1;
  for (int i = 1; i <= k; ++i) c = c * (unsigned)(n - k + i) / (unsigned)i;
  return (qd)c;
}

/* Theorem 1, eq.(19) P:290-299, 1-based indices m, n = 1..N+1:                */
/* (A^{-1})_{mn} = (-1)^{m+n} (m+n-1) C(N+m, N+1-n) C(N+n, N+1-m) C(m+n-2,m-1)^2 */
static qd hilbert_inv_entry_formula(int N, int m, int n) {
  qd b3 = binom_q(m + n - 2, m - 1);
  qd v = (qd)(m + n - 1) * binom_q(N + m, N + 1 - n) * binom_q(N + n, N + 1 - m) * b3 * b3;
  return ((m + n) % 2) ? -v : v;
}

/* eq.(19)'s entries for every N <= FABFO_MAX_N, evaluated once at load time
 * (the same exact integers, looked up instead of re-multiplied per pixel)    */
static qd hinv_tab[FABFO_MAX_N + 1][FABFO_MAX_N + 1][FABFO_MAX_N + 1];
__attribute__((constructor)) static void hinv_init(void) {
  for (int N = 0; N <= FABFO_MAX_N; ++N)
    for (int m = 1; m <= N + 1; ++m)
      for (int n = 1; n <= N + 1; ++n) hinv_tab[N][m - 1][n - 1] = hilbert_inv_entry_formula(N, m, n);
}
static qd hilbert_inv_entry(int N, int m, int n) { return hinv_tab[N][m - 1][n - 1]; }

int fabfo_hilbert_inverse(int N, double* out) {
  if (N < 0 || N > FABFO_MAX_N || !out) return 1;
  for (int m = 1; m <= N + 1; ++m)
    for (int n = 1; n <= N + 1; ++n)
      out[(m - 1) * (N + 1) + (n - 1)] = (double)hilbert_inv_entry(N, m, n);
  return 0;
}

/* c = A^{-1} mu (Algorithm 1 line 11), in __float128 */
static void fit_q(const qd* mu, int N, qd* c) {
  for (int m = 1; m <= N + 1; ++m) {
    qd s = 0;
    for (int n = 1; n <= N + 1; ++n) s += hilbert_inv_entry(N, m, n) * mu[n - 1];
    c[m - 1] = s;
  }
}

int fabfo_fit(const double* mu, int N, double* c) {
  if (N < 0 || N > FABFO_MAX_N || !mu || !c) return 1;
  qd muq[FABFO_MAX_N + 1], cq[FABFO_MAX_N + 1];
  for (int k = 0; k <= N; ++k) muq[k] = mu[k];
  fit_q(muq, N, cq);
  for (int k = 0; k <= N; ++k) c[k] = (double)cq[k];
  return 0;
}

/* Prop.3, eq.(24): mu_k = (beta-alpha)^{-k} sum_r C(k,r)(-alpha)^{k-r} m_r */
int fabfo_stretch(const double* m, int N, double alpha, double beta, double* mu) {
  if (N < 0 || N > FABFO_MAX_N || !m || !mu || !(beta > alpha)) return 1;
  qd a = alpha, d = (qd)beta - (qd)alpha;
  for (int k = 0; k <= N; ++k) {
    qd s = 0;
    for (int r = 0; r <= k; ++r) {
      qd pw = 1;
      for (int e = 0; e < k - r; ++e) pw *= -a;
      s += binom_q(k, r) * pw * (qd)m[r];
    }
    qd dk = 1;
    for (int e = 0; e < k; ++e) dk *= d;
    mu[k] = (double)(s / dk);
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* 64-node Gauss-Legendre rule on [0,1] in __float128 (library-primitive use:  */
/* numerical quadrature of the integral that eq.(28) defines).                 */
static qd gl_x[FABFO_GL_NODES], gl_w[FABFO_GL_NODES];

__attribute__((constructor)) static void gl_init(void) {
  const int n = FABFO_GL_NODES;
  for (int i = 0; i < n; ++i) {
    qd x = cosq(M_PIq * ((qd)i + 0.75Q) / ((qd)n + 0.5Q));
    qd dp = 0;
    for (int it = 0; it < 100; ++it) {
      qd p0 = 1, p1 = x;
      for (int k = 2; k <= n; ++k) {
        qd p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1);
      qd dx = p1 / dp;
      x -= dx;
      if (fabsq(dx) < 1e-40Q) break;
    }
    /* recompute derivative at the converged node */
    {
      qd p0 = 1, p1 = x;
      for (int k = 2; k <= n; ++k) {
        qd p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1);
    }
    gl_x[i] = (x + 1) / 2;                       /* map [-1,1] -> [0,1] */
    gl_w[i] = (2 / ((1 - x * x) * dp * dp)) / 2; /* Jacobian 1/2        */
  }
}

/* I_k = int_0^1 t^k exp(-lambda (t - t0)^2) dt, k = 0..K   (eq.(28))
 * method 1: eq.(31) P:432-435 for I_0 (two erf; written with erfc where both
 *           arguments share a sign so the difference does not cancel), eq.(32)
 *           P:436-440 for I_1, recursion eq.(30) P:423-426 for k >= 2.
 * method 2: 64-node Gauss-Legendre quadrature of the eq.(28) integrand.
 * method 0: automatic -- method 2 where eq.(30)'s forward recursion loses
 *           precision (lambda <= 1 and a slowly varying integrand, reading R9),
 *           method 1 otherwise.                                                */
static int integrals_q(qd lam, qd t0, int K, qd* I, int method) {
  qd far = fmaxq(fabsq(t0), fabsq(1 - t0));
  if (method == 0) method = (lam <= 1 && 2 * lam * far <= 24) ? 2 : 1;
  if (method == 2) {
    for (int k = 0; k <= K; ++k) I[k] = 0;
    for (int q = 0; q < FABFO_GL_NODES; ++q) {
      qd x = gl_x[q];
      qd e = gl_w[q] * expq(-lam * (x - t0) * (x - t0));
      qd xp = 1;
      for (int k = 0; k <= K; ++k) {
        I[k] += e * xp;
        xp *= x;
      }
    }
    return 2;
  }
  qd sl = sqrtq(lam);
  qd a = sl * (1 - t0), b = -sl * t0; /* I_0 = 1/2 sqrt(pi/lam) [erf(a) - erf(b)] */
  qd diff;
  if (a > 0 && b > 0)
    diff = erfcq(b) - erfcq(a);
  else if (a < 0 && b < 0)
    diff = erfcq(-a) - erfcq(-b);
  else
    diff = erfq(a) - erfq(b);
  qd E0 = expq(-lam * t0 * t0);
  qd E1 = expq(-lam * (1 - t0) * (1 - t0));
  I[0] = 0.5Q * sqrtq(M_PIq / lam) * diff;
  if (K >= 1) I[1] = t0 * I[0] + (E0 - E1) / (2 * lam);
  for (int k = 2; k <= K; ++k) I[k] = t0 * I[k - 1] + (qd)(k - 1) / (2 * lam) * I[k - 2] - E1 / (2 * lam);
  return 1;
}

int fabfo_integrals(double lam, double t0, int K, double* I, int method) {
  if (!(lam > 0) || K < 0 || K > FABFO_MAX_N + 1 || !I || method < 0 || method > 2) return -1;
  qd Iq[FABFO_MAX_N + 2];
  int used = integrals_q(lam, t0, K, Iq, method);
  for (int k = 0; k <= K; ++k) I[k] = (double)Iq[k];
  return used;
}

/* shifted Legendre polynomial coefficients: P~_k(t) = P_k(2t-1)
 * = sum_r (-1)^{k+r} C(k,r) C(k+r,r) t^r  (used only for the diagnostic kappa
 * of reading R7 -- the guard's condition number is stated in this basis).      */
static qd shifted_legendre_coef_formula(int k, int r) {
  qd v = binom_q(k, r) * binom_q(k + r, r);
  return ((k + r) % 2) ? -v : v;
}
static qd sleg_tab[FABFO_MAX_N + 1][FABFO_MAX_N + 1];
__attribute__((constructor)) static void sleg_init(void) {
  for (int k = 0; k <= FABFO_MAX_N; ++k)
    for (int r = 0; r <= k; ++r) sleg_tab[k][r] = shifted_legendre_coef_formula(k, r);
}
static qd shifted_legendre_coef(int k, int r) { return sleg_tab[k][r]; }

/* ------------------------------------------------------------------------- */
/* eq.(22): the stretched moments mu_k = sum_{t in Gamma_i} t^k H_i(t)
 * of the window whose samples are vals[0..n-1] (alpha, beta = their min, max).
 * H_i is the histogram of eq.(5) P:184-189 moved to Gamma_i by eq.(20)-(21)
 * P:301-310; with omega == 1 (reading R1) h_i(t) is the number of samples equal
 * to t.  route 0 follows eq.(22) as printed: the distinct values t of the
 * window with their counts (a counting table when the samples are integers
 * spanning at most 4096 levels -- every workload image -- else a sorted copy,
 * qsort being a library primitive); route 1 sums t_j^k over the n samples one by
 * one (the same sum, term by term; kept as the cross-check of route 0).  Both
 * in __float128; they differ only in the order of additions.                 */
static int cmp_float(const void* a, const void* b) {
  const float x = *(const float*)a, y = *(const float*)b;
  return (x > y) - (x < y);
}

#define FABFO_HIST_SPAN 4096

static void add_powers(qd t, qd count, int N, qd* mu) {
  qd tp = count;
  for (int k = 0; k <= N; ++k) {
    mu[k] += tp;
    tp *= t;
  }
}

static void stretched_moments(const float* vals, const double* wts, int n, float amin, float bmax, int N,
                              int route, qd* mu) {
  const qd alpha = amin, d = (qd)bmax - (qd)amin;
  for (int k = 0; k <= N; ++k) mu[k] = 0;
  if (wts) { /* weighted histogram h_i of eq.(5) with omega(j) = wts[j] (Gaussian omega, eq.(4)) */
    if (route == 1) {
      for (int j = 0; j < n; ++j) add_powers(((qd)vals[j] - alpha) / d, wts[j], N, mu);
      return;
    }
    int integral = (double)bmax - (double)amin <= FABFO_HIST_SPAN;
    for (int j = 0; j < n && integral; ++j) integral = vals[j] == floorf(vals[j]);
    if (!integral) {
      for (int j = 0; j < n; ++j) add_powers(((qd)vals[j] - alpha) / d, wts[j], N, mu);
      return;
    }
    static __thread qd hw[FABFO_HIST_SPAN + 1];
    const int span = (int)((double)bmax - (double)amin);
    for (int v = 0; v <= span; ++v) hw[v] = 0;
    for (int j = 0; j < n; ++j) hw[(int)((double)vals[j] - (double)amin)] += wts[j];
    for (int v = 0; v <= span; ++v)
      if (hw[v] != 0) add_powers((qd)v / d, hw[v], N, mu);
    return;
  }
  if (route == 1) {
    for (int j = 0; j < n; ++j) add_powers(((qd)vals[j] - alpha) / d, 1, N, mu);
    return;
  }
  int integral = (double)bmax - (double)amin <= FABFO_HIST_SPAN;
  for (int j = 0; j < n && integral; ++j) integral = vals[j] == floorf(vals[j]);
  if (integral) { /* counts of the levels amin .. bmax */
    static __thread int cnt[FABFO_HIST_SPAN + 1];
    const int span = (int)((double)bmax - (double)amin);
    memset(cnt, 0, sizeof(int) * (size_t)(span + 1));
    for (int j = 0; j < n; ++j) cnt[(int)((double)vals[j] - (double)amin)]++;
    for (int v = 0; v <= span; ++v)
      if (cnt[v]) add_powers((qd)v / d, (qd)cnt[v], N, mu);
    return;
  }
  float* s = (float*)malloc(sizeof(float) * (size_t)n);
  if (!s) { /* out of memory: the term-by-term sum is the same quantity */
    for (int j = 0; j < n; ++j) add_powers(((qd)vals[j] - alpha) / d, 1, N, mu);
    return;
  }
  memcpy(s, vals, sizeof(float) * (size_t)n);
  qsort(s, (size_t)n, sizeof(float), cmp_float);
  for (int j = 0; j < n;) {
    int e = j + 1;
    while (e < n && s[e] == s[j]) ++e;
    add_powers(((qd)s[j] - alpha) / d, (qd)(e - j), N, mu);
    j = e;
  }
  free(s);
}

/* ------------------------------------------------------------------------- */
/* the per-pixel result                                                        */
typedef struct {
  double g_lit;   /* eq.(29) as printed                                  */
  double g_guard; /* with the guard of reading R7                        */
  double kappa;   /* sum_k |(2k+1) nu_k J_k| / T2 (Legendre basis)       */
  double t2n;     /* T2 / n  (n = window size)                           */
  double lam;     /* lambda_i, eq.(25)                                   */
  double t0;      /* theta_0(i)                                          */
  int code;
} fabfo_px;

/* Algorithm 1 P:446-477 for one pixel whose window samples are vals[0..n-1]  */
static void fast_window(const float* vals, const double* wts, int n, float f_center, float theta,
                        float sigma, int N, int route, fabfo_px* out) {
  memset(out, 0, sizeof(*out));
  float amin = vals[0], bmax = vals[0];
  for (int j = 1; j < n; ++j) {
    if (vals[j] < amin) amin = vals[j];
    if (vals[j] > bmax) bmax = vals[j];
  }
  if (amin == bmax) { /* lines 4-5 P:454-455: g-hat(i) = f(i) */
    out->g_lit = out->g_guard = f_center;
    out->kappa = 1.0;
    out->t2n = 1.0;
    out->code = FABFO_CODE_IDENTITY;
    return;
  }
  qd alpha = amin, beta = bmax, d = beta - alpha;

  /* eq.(22): mu_k = sum_{t in Gamma_i} t^k H_i(t) */
  qd mu[FABFO_MAX_N + 1];
  stretched_moments(vals, wts, n, amin, bmax, N, route, mu);
  /* line 11: c = A^{-1} mu */
  qd c[FABFO_MAX_N + 1];
  fit_q(mu, N, c);
  /* lines 12-13: t0, lambda (eq.(25)) */
  qd t0 = ((qd)theta - alpha) / d;
  qd lam = d * d / (2 * (qd)sigma * (qd)sigma);
  /* line 14 + 18: I_0 .. I_{N+1} */
  qd I[FABFO_MAX_N + 2];
  int used = integrals_q(lam, t0, N + 1, I, 0);
  /* lines 15-20: T1, T2 */
  qd T1 = 0, T2 = 0;
  for (int k = 0; k <= N; ++k) {
    T1 += c[k] * I[k + 1];
    T2 += c[k] * I[k];
  }
  qd g_lit = alpha + d * (T1 / T2); /* line 21, eq.(29) */

  /* diagnostic condition number in the Legendre basis (reading R7) */
  qd absum = 0;
  for (int k = 0; k <= N; ++k) {
    qd nu = 0, J = 0;
    for (int r = 0; r <= k; ++r) {
      qd L = shifted_legendre_coef(k, r);
      nu += L * mu[r];
      J += L * I[r];
    }
    absum += fabsq((qd)(2 * k + 1) * nu * J);
  }
  qd kappa = (T2 > 0) ? absum / T2 : (qd)INFINITY;
  qd g_guard = g_lit;
  int code = (used == 2) ? FABFO_CODE_QUAD : 0;
  if (!(T2 > 0) || kappa > (qd)FABFO_KAPPA_MAX) {
    g_guard = alpha + d * (I[1] / I[0]); /* the paper's N = 0 value */
    code |= FABFO_CODE_GUARD;
  }
  out->g_lit = (double)g_lit;
  out->g_guard = (double)g_guard;
  out->kappa = (double)kappa;
  out->t2n = (double)(T2 / mu[0]); /* T2 / (sum of the weights) */
  out->lam = (double)lam;
  out->t0 = (double)t0;
  out->code = code;
}

/* one window given explicitly: out6 = {g_lit, g_guard, kappa, t2n, lam, t0};
 * route: how eq.(22) is summed (0 distinct values with counts, 1 sample by sample) */
int fabfo_window(const float* vals, int n, float f_center, float theta, float sigma, int N,
                 int route, double* out6, int* code) {
  if (!vals || n < 1 || N < 0 || N > FABFO_MAX_N || !out6 || route < 0 || route > 1) return 1;
  fabfo_px px;
  fast_window(vals, NULL, n, f_center, theta, sigma, N, route, &px);
  out6[0] = px.g_lit;
  out6[1] = px.g_guard;
  out6[2] = px.kappa;
  out6[3] = px.t2n;
  out6[4] = px.lam;
  out6[5] = px.t0;
  if (code) *code = px.code;
  return 0;
}

/* whole-image (or pixel-list) driver.  Pixels are flat indices into B*H*W.
 * If idx is NULL the pixels are p0..p1-1, else idx[p0..p1-1].  Any output
 * pointer may be NULL.  Output arrays are indexed like the pixel list.        */
/* NEXT-1: the paper's default spatial kernel, eq.(4): omega(j) =
 * exp(-|j|^2 / 2 rho^2) on Omega = [-3 rho, 3 rho]^2 (the window "typically
 * set").  Returns the window half-width R and fills w[(2R+1)^2] in the
 * order gather_window produces the samples (dy outer, dx inner), or -1.      */
static int gauss_weights(int rho, double** w) {
  const int R = 3 * rho, side = 2 * R + 1;
  *w = (double*)malloc(sizeof(double) * (size_t)side * side);
  if (!*w) return -1;
  for (int dy = -R; dy <= R; ++dy)
    for (int dx = -R; dx <= R; ++dx)
      (*w)[(dy + R) * side + dx + R] = rho > 0 ? exp(-(double)(dy * dy + dx * dx) / (2.0 * rho * rho)) : 1.0;
  return R;
}

static int fast_impl(const float* img, const float* theta, const float* sigma, int B, int H, int W,
                     int rho, int N, int gauss, const long* idx, long p0, long p1, double* g_lit,
                     double* g_guard, double* kappa, double* t2n, unsigned char* code) {
  if (!img || !theta || !sigma || B < 1 || H < 1 || W < 1 || rho < 0) return 1;
  double* wts = NULL;
  const int R = gauss ? gauss_weights(rho, &wts) : rho;
  if (R < 0) return 2;
  if (2 * R + 1 > H || 2 * R + 1 > W || N < 0 || N > FABFO_MAX_N) {
    free(wts);
    return 1;
  }
  long HW = (long)H * W;
  int n = (2 * R + 1) * (2 * R + 1);
  float* vals = (float*)malloc(sizeof(float) * (size_t)n);
  if (!vals) {
    free(wts);
    return 2;
  }
  for (long q = p0; q < p1; ++q) {
    long p = idx ? idx[q] : q;
    if (p < 0 || p >= (long)B * HW) {
      free(vals);
      free(wts);
      return 1;
    }
    long b = p / HW, r = p % HW, y = r / W, x = r % W;
    gather_window(img, H, W, R, b, y, x, vals);
    fabfo_px px;
    fast_window(vals, wts, n, img[p], theta[p], sigma[p], N, 0, &px);
    if (g_lit) g_lit[q] = px.g_lit;
    if (g_guard) g_guard[q] = px.g_guard;
    if (kappa) kappa[q] = px.kappa;
    if (t2n) t2n[q] = px.t2n;
    if (code) code[q] = (unsigned char)px.code;
  }
  free(vals);
  free(wts);
  return 0;
}

int fabfo_fast(const float* img, const float* theta, const float* sigma, int B, int H, int W,
               int rho, int N, const long* idx, long p0, long p1, double* g_lit,
               double* g_guard, double* kappa, double* t2n, unsigned char* code) {
  return fast_impl(img, theta, sigma, B, H, W, rho, N, 0, idx, p0, p1, g_lit, g_guard, kappa, t2n, code);
}

/* Algorithm 1 with the Gaussian omega of eq.(4) on [-3 rho, 3 rho]^2 (NEXT-1):
 * the weighted histogram of eq.(5), everything else as fabfo_fast.            */
int fabfo_fast_gauss(const float* img, const float* theta, const float* sigma, int B, int H, int W,
                     int rho, int N, const long* idx, long p0, long p1, double* g_lit,
                     double* g_guard, double* kappa, double* t2n, unsigned char* code) {
  return fast_impl(img, theta, sigma, B, H, W, rho, N, 1, idx, p0, p1, g_lit, g_guard, kappa, t2n, code);
}

/* one explicitly weighted window (pins of the Gaussian route): omega(j) = wts[j] */
int fabfo_window_w(const float* vals, const double* wts, int n, float f_center, float theta, float sigma,
                   int N, int route, double* out6, int* code) {
  if (!vals || !wts || n < 1 || N < 0 || N > FABFO_MAX_N || !out6 || route < 0 || route > 1) return 1;
  fabfo_px px;
  fast_window(vals, wts, n, f_center, theta, sigma, N, route, &px);
  out6[0] = px.g_lit;
  out6[1] = px.g_guard;
  out6[2] = px.kappa;
  out6[3] = px.t2n;
  out6[4] = px.lam;
  out6[5] = px.t0;
  if (code) *code = px.code;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* O3 "literal": Algorithm 1 as printed, in plain fp64, with the   */
/* paper's own scaling (f, theta, sigma divided by 255 before, g-hat times 255 */
/* after).  CONTEXT ONLY -- it is not a parity target: it shows how */
/* far the paper's own numerics drift from the __float128 reference above.     */
/*   line 2  alpha, beta: window min / max (eq.(8); exhaustive scan -- the same  */
/*           values the O(1) MAX-FILTER gives);                                 */
/*   line 6  gamma_k = omega * f^k, k = 0..N, omega = 1/n on the box (gamma_0 =  */
/*           1), by O(1) separable running sums in fp64 (the paper's      */
/*           recursive-filter route);                                    */
/*   line 9  mu from m = gamma by eq.(24);                            */
/*   line 11 c = A^{-1} mu with eq.(19) in fp64;                         */
/*   lines 12-14 t0, lambda, I_0 by eq.(31) (C99 erf), I_1 by eq.(32);          */
/*   lines 17-20 I_k by the forward recursion eq.(30) for every lambda;          */
/*   line 21 g-hat = alpha + (beta - alpha) T1/T2 (no guard, eq.(29)).           */
/* Identity (alpha == beta) pixels copy f (lines 4-5).  Whole images only (the  */
/* running sums need every row).                                               */
int fabfo_literal(const float* img, const float* theta, const float* sigma, int B, int H, int W,
                  int rho, int N, double* g) {
  if (!img || !theta || !sigma || !g || B < 1 || H < 1 || W < 1 || rho < 0) return 1;
  if (2 * rho + 1 > H || 2 * rho + 1 > W || N < 0 || N > FABFO_MAX_N) return 1;
  const long HW = (long)H * W;
  const int w = 2 * rho + 1;
  const double inv_n = 1.0 / ((double)w * w);
  double* rowsum = (double*)malloc(sizeof(double) * (size_t)HW * (N + 1));
  double* gam = (double*)malloc(sizeof(double) * (size_t)HW * (N + 1));
  float* amin = (float*)malloc(sizeof(float) * (size_t)HW);
  float* bmax = (float*)malloc(sizeof(float) * (size_t)HW);
  if (!rowsum || !gam || !amin || !bmax) {
    free(rowsum), free(gam), free(amin), free(bmax);
    return 2;
  }
  double Ainv[(FABFO_MAX_N + 1) * (FABFO_MAX_N + 1)];
  fabfo_hilbert_inverse(N, Ainv);
  for (long b = 0; b < B; ++b) {
    const float* f = img + b * HW;
    fabfo_bounds(f, 1, H, W, rho, 0, HW, amin, bmax);
    /* horizontal running sums of (f/255)^k (reflected borders, reading R2) */
    for (long y = 0; y < H; ++y)
      for (int k = 0; k <= N; ++k) {
        double s = 0;
        for (long dx = -rho; dx <= rho; ++dx) s += pow((double)f[y * W + reflect_index(dx, W)] / 255.0, k);
        rowsum[((size_t)k * H + y) * W + 0] = s;
        for (long x = 1; x < W; ++x) {
          s += pow((double)f[y * W + reflect_index(x + rho, W)] / 255.0, k) -
               pow((double)f[y * W + reflect_index(x - rho - 1, W)] / 255.0, k);
          rowsum[((size_t)k * H + y) * W + x] = s;
        }
      }
    /* vertical running sums, times omega = 1/n */
    for (int k = 0; k <= N; ++k)
      for (long x = 0; x < W; ++x) {
        const double* R = rowsum + (size_t)k * HW;
        double s = 0;
        for (long dy = -rho; dy <= rho; ++dy) s += R[reflect_index(dy, H) * W + x];
        gam[(size_t)k * HW + x] = s * inv_n;
        for (long y = 1; y < H; ++y) {
          s += R[reflect_index(y + rho, H) * W + x] - R[reflect_index(y - rho - 1, H) * W + x];
          gam[(size_t)k * HW + y * W + x] = s * inv_n;
        }
      }
    for (long p = 0; p < HW; ++p) {
      const double al = amin[p] / 255.0, be = bmax[p] / 255.0;
      if (amin[p] == bmax[p]) { /* lines 4-5 */
        g[b * HW + p] = f[p];
        continue;
      }
      const double d = be - al;
      double mu[FABFO_MAX_N + 1], c[FABFO_MAX_N + 1];
      for (int k = 0; k <= N; ++k) { /* eq.(24) */
        double s = 0;
        for (int r = 0; r <= k; ++r) s += (double)binom_q(k, r) * pow(-al, k - r) * gam[(size_t)r * HW + p];
        mu[k] = s / pow(d, k);
      }
      for (int m = 0; m <= N; ++m) { /* c = A^{-1} mu */
        double s = 0;
        for (int n2 = 0; n2 <= N; ++n2) s += Ainv[m * (N + 1) + n2] * mu[n2];
        c[m] = s;
      }
      const double t0 = (theta[b * HW + p] / 255.0 - al) / d;
      const double sg = sigma[b * HW + p] / 255.0;
      const double lam = 0.5 * d * d / (sg * sg);
      const double sl = sqrt(lam);
      const double E1 = exp(-lam * (1 - t0) * (1 - t0));
      double I0 = 0.5 * sqrt(M_PI / lam) * (erf(sl * (1 - t0)) - erf(-sl * t0)); /* eq.(31) */
      double I1 = t0 * I0 + (exp(-lam * t0 * t0) - E1) / (2 * lam);            /* eq.(32) */
      double T1 = c[0] * I1, T2 = c[0] * I0;
      double Ikm2 = I0, Ikm1 = I1;
      for (int k = 2; k <= N + 1; ++k) { /* eq.(30) */
        const double Ik = t0 * Ikm1 + (k - 1) / (2 * lam) * Ikm2 - E1 / (2 * lam);
        T1 += c[k - 1] * Ik;
        T2 += c[k - 1] * Ikm1;
        Ikm2 = Ikm1;
        Ikm1 = Ik;
      }
      g[b * HW + p] = 255.0 * (al + d * (T1 / T2));
    }
  }
  free(rowsum), free(gam), free(amin), free(bmax);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Mozerov & van de Weijer's uniform-prior filter as the paper compares it    */
/* (Fig.3): a constant (degree-0) fit of the local histogram */
/* on [f(i), 2 fbar(i) - f(i)] (Delta = 0, the narrowest valid uniform         */
/* distribution; fbar = the Omega-mean, omega = 1 on the box, reading R1)      */
/* instead of [alpha_i, beta_i]:  with [a, b] that interval in increasing      */
/* order, t0 = (theta - a)/(b - a), lambda = (b - a)^2 / (2 sigma^2),          */
/*   g_moz = a + (b - a) I_1 / I_0                          (eq.(29) at N = 0) */
/* and g_moz = f(i) when a = b.  __float128 throughout (the window mean is a   */
/* direct sum); integrals as for fabfo_fast.                                   */
int fabfo_mozerov(const float* img, const float* theta, const float* sigma, int B, int H, int W,
                  int rho, long p0, long p1, double* g) {
  if (!img || !theta || !sigma || !g || B < 1 || H < 1 || W < 1 || rho < 0) return 1;
  if (2 * rho + 1 > H || 2 * rho + 1 > W) return 1;
  const long HW = (long)H * W;
  const int n = (2 * rho + 1) * (2 * rho + 1);
  float* vals = (float*)malloc(sizeof(float) * (size_t)n);
  if (!vals) return 2;
  for (long p = p0; p < p1; ++p) {
    const long b = p / HW, r = p % HW, y = r / W, x = r % W;
    gather_window(img, H, W, rho, b, y, x, vals);
    qd s = 0;
    for (int j = 0; j < n; ++j) s += vals[j];
    const qd fb = s / n, f = img[p], e = 2 * fb - f;
    const qd a = f < e ? f : e, bb = f < e ? e : f;
    if (!(bb > a)) {
      g[p] = img[p];
      continue;
    }
    const qd d = bb - a, t0 = ((qd)theta[p] - a) / d, lam = d * d / (2 * (qd)sigma[p] * (qd)sigma[p]);
    qd I[2];
    integrals_q(lam, t0, 1, I, 0);
    g[p] = (double)(a + d * (I[1] / I[0]));
  }
  free(vals);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* NEXT-2: the sharpening / denoising application's range-kernel maps,        */
/* P:620-630 (after Zhang & Allebach):                                         */
/*   theta(i) = f(i) + zeta(i),  zeta(i) = f(i) - fbar(i)                      */
/*              (fbar = average over the Omega neighbourhood: the box of       */
/*              half-width rho, reading R1);                                   */
/*   sigma(i) = an affine map of |LoG f|(i) that maps low values to high sigma:*/
/*              sigma = s_hi - (s_hi - s_lo) min(|L(i)| / l_sat, 1)            */
/*              (the paper gives neither the LoG scale nor the map; reading    */
/*              R15: these four parameters are inputs);                        */
/*   L = Laplacian of Gaussian at scale s: the sampled, normalised Gaussian    */
/*       g(x) ~ exp(-x^2 / 2s^2) on |x| <= ceil(4 s) and its second derivative */
/*       g''(x) = (x^2 - s^2) / s^4 g(x); L(i) = sum_{dy,dx} [g''(dx) g(dy) +  */
/*       g(dx) g''(dy)] f(i - (dy, dx)), borders reflected (reading R2).        */
/* Direct sums in fp64 (__float128 for fbar), pixel by pixel.                 */
int fabfo_sharpen_maps(const float* img, int B, int H, int W, int rho, double s, double s_lo, double s_hi,
                       double l_sat, long p0, long p1, double* theta, double* sigma) {
  if (!img || !theta || !sigma || B < 1 || H < 1 || W < 1 || rho < 0 || !(s > 0) || !(l_sat > 0)) return 1;
  const int r = (int)ceil(4.0 * s);
  if (2 * rho + 1 > H || 2 * rho + 1 > W || 2 * r + 1 > H || 2 * r + 1 > W || r > 64) return 1;
  const long HW = (long)H * W;
  double g[129], g2[129], gs = 0;
  for (int k = -r; k <= r; ++k) gs += (g[k + r] = exp(-0.5 * k * k / (s * s)));
  for (int k = -r; k <= r; ++k) {
    g[k + r] /= gs;
    g2[k + r] = ((double)k * k - s * s) / (s * s * s * s) * g[k + r];
  }
  const int n = (2 * rho + 1) * (2 * rho + 1);
  for (long p = p0; p < p1; ++p) {
    const long b = p / HW, rr = p % HW, y = rr / W, x = rr % W;
    const float* base = img + b * HW;
    qd acc = 0;
    for (long dy = -rho; dy <= rho; ++dy)
      for (long dx = -rho; dx <= rho; ++dx) acc += base[reflect_index(y + dy, H) * W + reflect_index(x + dx, W)];
    const double fbar = (double)(acc / n), f = base[y * W + x];
    theta[p] = f + (f - fbar);
    double L = 0;
    for (int dy = -r; dy <= r; ++dy)
      for (int dx = -r; dx <= r; ++dx)
        L += (g2[dx + r] * g[dy + r] + g[dx + r] * g2[dy + r]) *
             base[reflect_index(y - dy, H) * W + reflect_index(x - dx, W)];
    const double u = fabs(L) / l_sat;
    sigma[p] = s_hi - (s_hi - s_lo) * (u < 1.0 ? u : 1.0);
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* NEXT-2, second application: texture filtering.                   */
/*   mRTV(i) = Delta(i) max_{j in W_i} |grad f(j)| / (sum_{j in W_i} |grad f(j)| + eps)   */
/*   Delta(i) = max_{j in W_i} f(j) - min_{j in W_i} f(j) */
/*   sigma(i) = an affine map of mRTV(i), high where mRTV is low    */
/* The paper fixes neither W_i, the gradient stencil, eps nor the map; reading */
/* R19: W_i = the box of half-width `patch` around i; grad f(j) =   */
/* forward differences (f(y, x+1) - f(y, x), f(y+1, x) - f(y, x)) with the      */
/* image reflected at its borders (reading R2: the difference across the last  */
/* column / row is 0), |.| the Euclidean norm; a window position j outside the */
/* image takes the value of the pixel it reflects to;                          */
/*   sigma = s_hi - (s_hi - s_lo) min(mRTV / m_sat, 1).                        */
/* Direct window scans per pixel, fp64 (the sum in __float128).               */
static double grad_mag(const float* base, long H, long W, long y, long x) {
  const double f = base[y * W + x];
  const double gx = (double)base[y * W + reflect_index(x + 1, W)] - f;
  const double gy = (double)base[reflect_index(y + 1, H) * W + x] - f;
  return sqrt(gx * gx + gy * gy);
}

int fabfo_texture_maps(const float* img, int B, int H, int W, int patch, double s_lo, double s_hi, double m_sat,
                       double eps, long p0, long p1, double* mrtv, double* sigma) {
  if (!img || !mrtv || !sigma || B < 1 || H < 1 || W < 1 || patch < 0 || !(m_sat > 0) || !(eps > 0)) return 1;
  if (2 * patch + 1 > H || 2 * patch + 1 > W) return 1;
  const long HW = (long)H * W;
  for (long p = p0; p < p1; ++p) {
    const long b = p / HW, rr = p % HW, y = rr / W, x = rr % W;
    const float* base = img + b * HW;
    double fmin_ = INFINITY, fmax_ = -INFINITY, gmax = 0.0;
    qd gsum = 0;
    for (long dy = -patch; dy <= patch; ++dy)
      for (long dx = -patch; dx <= patch; ++dx) {
        const long yy = reflect_index(y + dy, H), xx = reflect_index(x + dx, W);
        const double f = base[yy * W + xx], g = grad_mag(base, H, W, yy, xx);
        if (f < fmin_) fmin_ = f;
        if (f > fmax_) fmax_ = f;
        if (g > gmax) gmax = g;
        gsum += g;
      }
    const double m = (fmax_ - fmin_) * gmax / ((double)gsum + eps);
    mrtv[p] = m;
    const double u = m / m_sat;
    sigma[p] = s_hi - (s_hi - s_lo) * (u < 1.0 ? u : 1.0);
  }
  return 0;
}
