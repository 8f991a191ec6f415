// fabf_device.cuh -- per-pixel device math of the fast adaptive bilateral
// filter (arXiv 1811.02308) for sm_100a.  Included by fabf.cu only.
//
// P:<n> = line of /root/reference/PAPER.md.  The stage names follow SURVEY.md
// section 8(a) (a4 stretch, a5 fit, a6 range parameters, a7 integrals, a8 ratio).
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>


namespace fabf {

constexpr int kMaxN = 10;
constexpr int kGlB = 16;  // fixed-node Gauss-Legendre rule on [0,1], small lambda
constexpr int kGlC = 24;  // Gauss-Legendre rule on the effective support, far theta_0
constexpr float kKappaMax = 1000.0f;
#ifndef FABF_LAMBDA_B
#define FABF_LAMBDA_B 2.0
#endif
constexpr double kLambdaSmall = FABF_LAMBDA_B;  // below: fixed-node quadrature (regime B)

// code bits (mirror FABF_CODE_* in include/fabf.h)
constexpr unsigned kCodeIdentity = 0x1u;
constexpr unsigned kCodeGuard = 0x2u;
constexpr unsigned kCodeSmallLambda = 0x4u;
constexpr unsigned kCodeFallback = 0x8u;
constexpr unsigned kCodeFarTheta = 0x10u;

// plan flags (mirror FABF_FLAG_*)
constexpr unsigned kFlagLiteral = 0x1u;
constexpr unsigned kFlagClamp = 0x2u;

// Regime B: W[k][q] = w_q * P~_k(x_q), 16-node Gauss-Legendre on [0,1].
__constant__ float c_glB_x[kGlB];
__constant__ float c_glB_W[kMaxN + 2][kGlB];
// Regime C: 24-node Gauss-Legendre nodes / weights on [0,1] (fp64).
__constant__ double c_glC_x[kGlC];
__constant__ double c_glC_w[kGlC];

// Horner evaluation of sum_j c[j] x^j with the coefficients in constant
// memory: every DFMA takes its coefficient as a c[bank][offset] operand (no
// LDC, no extra registers); the independent seed polynomials of a pixel give
// the scheduler its ILP.
template <int DEG>
__device__ __forceinline__ double poly_horner(const double* c, double x) {
  double p = c[DEG];
#pragma unroll
  for (int j = DEG - 1; j >= 0; --j) p = fma(p, x, c[j]);
  return p;
}

// The same polynomial as WAYS interleaved Horner chains in x^WAYS:
// p(x) = sum_r x^r E_r(x^WAYS), r < WAYS.  Same operation count (+ the powers),
// 1/WAYS of the dependent depth: C2 is bound by the fp64 pipe's latency at the
// occupancy its registers allow, not by its throughput.
#ifndef FABF_ERFCX_WAYS
#define FABF_ERFCX_WAYS 1
#endif
template <int DEG, int WAYS>
__device__ __forceinline__ double poly_split(const double* c, double x) {
  if constexpr (WAYS == 1) {
    return poly_horner<DEG>(c, x);
  } else {
    double xp[WAYS + 1];
    xp[0] = 1.0;
    xp[1] = x;
#pragma unroll
    for (int r = 2; r <= WAYS; ++r) xp[r] = xp[r / 2] * xp[r - r / 2];
    double acc = 0.0;
#pragma unroll
    for (int r = WAYS - 1; r >= 0; --r) {
      const int top = r + ((DEG - r) / WAYS) * WAYS;  // highest index = r mod WAYS
      double e = c[top];
#pragma unroll
      for (int j = top - WAYS; j >= 0; j -= WAYS) e = fma(e, xp[WAYS], c[j]);
      acc = (r == 0) ? acc + e : fma(e, xp[r], acc);
    }
    return acc;
  }
}

// 1/d for normal positive d: MUFU.RCP64H seed + two Newton steps (relative
// error ~1e-16, no special-case branches: d is in [1, 1e4] here).
__device__ __forceinline__ double rcp64(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// exp(z) for z <= 0 in fp64 (z < -708 gives 0): k = rint(z / ln2) by the
// 1.5 * 2^52 shifter (k lands in the low word, no F2I / FRND), Cody-Waite
// reduction with a hi/lo ln2, degree-12 Taylor polynomial on |r| <= ln2/2
// (truncation < 2e-16), 2^k assembled in the exponent field.
__constant__ double c_exp_poly[13] = {
    1.0, 1.0, 1.0 / 2, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040, 1.0 / 40320,
    1.0 / 362880, 1.0 / 3628800, 1.0 / 39916800, 1.0 / 479001600};
__device__ __forceinline__ double exp_nonpos(double z) {
  const double kShift = 6755399441055744.0;  // 1.5 * 2^52
  const double zc = fmax(z, -708.0);  // (z is never NaN here)
  const double ks = fma(zc, 1.4426950408889634074, kShift);
  const double kd = ks - kShift;
  double r = fma(kd, -6.93147180369123816490e-01, zc);
  r = fma(kd, -1.90821492927058770002e-10, r);
  const double p = poly_horner<12>(c_exp_poly, r);
  const int k = __double2loint(ks);
  const double scale = __hiloint2double((k + 1023) << 20, 0);
  return (z < -708.0) ? 0.0 : p * scale;
}

// The same with a 64-entry table T[j] = 2^(j/64) (correctly rounded, host
// computed, staged in shared memory by the caller): K = rint(z 64/ln2),
// z = K ln2/64 + r with |r| <= ln2/128, exp(z) = 2^(K>>6) T[K&63] exp(r) and a
// degree-5 Taylor polynomial for exp(r) (truncation r^6/720 < 4e-17): 5 DFMA
// instead of 12 for one LDS.  z is clamped at -708 (the result is then
// ~e^-708, not 0: every use here scales a term that is negligible there).
__constant__ double c_exp2_64[64];
__device__ __forceinline__ double exp_nonpos_tab(double z, const double* __restrict__ tab) {
  const double kShift = 6755399441055744.0;  // 1.5 * 2^52
  const double zc = z < -708.0 ? -708.0 : z;  // (a select: fmax's NaN handling costs 4 more)
  const double ks = fma(zc, 92.33248261689366, kShift);
  const double kd = ks - kShift;
  double r = fma(kd, -0.01083042469326756, zc);  // ln2/64, 32 significant bits: kd * hi exact
  r = fma(kd, -2.9815858269852933e-12, r);
  const double p = poly_horner<5>(c_exp_poly, r);
  const int K = __double2loint(ks);
  const double scale = __hiloint2double(((K >> 6) + 1023) << 20, 0);
  return (p * tab[K & 63]) * scale;
}

#include "fabf_erfcx.cuh"

struct PixelResult {
  float g;
  float kappa;
  float t2n;
  unsigned code;
};

// ---------------------------------------------------------------------------
// a7: the integrals of eq.(28) in the Legendre basis.  With s = 2t - 1,
// kappa = lambda/4, s0 = 2 t0 - 1 and g(s) = exp(-kappa (s - s0)^2):
//   A_k = int_{-1}^{1} P_k(s) g(s) ds   ( = 2 J_k,  J_k = int_0^1 P~_k psi dt )
//   X_k = int_{-1}^{1} s P_k(s) g(s) ds = ((k+1) A_{k+1} + k A_{k-1}) / (2k+1)
// for k = 0..N, up to one common positive factor per pixel (eq.(29) and the
// guard are invariant to it).  X is what the ratio needs: with the fit
// p = sum_k (2k+1) nu_k P~_k (a5), T2 = sum_k (2k+1) nu_k A_k and
// 2 T1 - T2 = sum_k (2k+1) nu_k X_k.
//
// Regime A (lambda >= 2, t0 in [-1,2]): the integration-by-parts idea of
// P:411-426 applied in the Legendre basis:
//   X_k     = s0 A_k - (g(1) - (-1)^k g(-1) - D_k) / (2 kappa)
//   A_{k+1} = ((2k+1) X_k - k A_{k-1}) / (k+1)
//   D_k     = sum_{j<k, j = k-1 mod 2} (2j+1) A_j
// (from int P_k g' = [P_k g] - int P_k' g, s P_k = ((k+1)P_{k+1} + k P_{k-1})/(2k+1)
// and P_k' = sum (2j+1) P_j), so X_k is the recurrence's own intermediate.
// Seeds: A_0 by two erf (eq.(31)) written as erfc = erfcx * exp so
// that the two boundary exponentials g(+-1) (as in eq.(32)) are
// reused -- 2 erfcx + 2 exp, branch-free; when t0 is outside [0,1]
// everything is scaled by exp(kappa (nearer boundary distance)^2).  fp64
// throughout: the recurrence amplifies seed error by up to ~4e7 at lambda = 2
// ("Kernels").  The range parameters come straight from the fp32 inputs in fp64 (their
// rounding to fp32 would be amplified by kappa up to 1e3):
//   sk = sqrt(kappa) = (beta-alpha) / (2 sqrt2 sigma), s0 = (2 theta - alpha - beta)/(beta - alpha),
//   csk = sqrt(pi)/2 / sk, inv2k = 1/(2 kappa).
// (2k+1)/(k+1) and -k/(k+1), k = 0..kMaxN: c[] operands instead of rebuilt immediates
__constant__ double c_rec[2 * (kMaxN + 1)] = {
    1.0, -0.0, 3.0 / 2, -1.0 / 2, 5.0 / 3, -2.0 / 3, 7.0 / 4, -3.0 / 4, 9.0 / 5, -4.0 / 5, 11.0 / 6,
    -5.0 / 6, 13.0 / 7, -6.0 / 7, 15.0 / 8, -7.0 / 8, 17.0 / 9, -8.0 / 9, 19.0 / 10, -9.0 / 10,
    21.0 / 11, -10.0 / 11};

template <int N, bool TAB = false>
__device__ __forceinline__ void integrals_regime_a(double sk, double s0, double csk, double inv2k,
                                                   const double* nup, int ns, double nu0, double& T2,
                                                   double& U, double& ab, double& A0, double& X0,
                                                   const double* etab = nullptr) {
  const double xa = sk * (1.0 - s0), xb = sk * (1.0 + s0);  // s = +1 and s = -1 ends
  // near / far end first (xa + xb = 2 sk > 0: the far end is never negative)
  const bool a_near = fabs(xa) < fabs(xb);
  const double xn = a_near ? xa : xb, xf = a_near ? xb : xa;
  const double qn = xn * xn, qf = xf * xf;
  const bool inside = xn >= 0.0;
  double E, Gn;
  if constexpr (TAB) {
    E = exp_nonpos_tab(qn - qf, etab);               // <= 1
    Gn = exp_nonpos_tab(inside ? -qn : 0.0, etab);   // scale 1 inside, exp(qn) outside
  } else {
    E = exp_nonpos(qn - qf);
    Gn = exp_nonpos(inside ? -qn : 0.0);
  }
  double cn, cf;
  erfcx_pos2(fabs(xn), xf, cn, cf);
  const double gn = Gn, gf = Gn * E;
  // erf(xa) + erf(xb): inside 2 - erfc(xa) - erfc(xb); outside erfc(|x_near|) - erfc(x_far)
  const double a0 = csk * (inside ? (2.0 - cn * gn - cf * gf) : fma(cn, gn, -cf * gf));
  // boundary values g(+1) - g(-1) = +-(gn - gf) (+ when the s = +1 end is the near one)
  const double bnd_even = (gn - gf) * (a_near ? inv2k : -inv2k), bnd_odd = (gn + gf) * inv2k;
  double a_prev = 0.0, a_cur = a0, d_even = 0.0, d_odd = 0.0;
  // a8 sums consumed on the fly (no A / X arrays): T2 = sum nup_k A_k,
  // U = sum nup_k X_k, ab = sum |nup_k A_k|
  // nup_k = nup[(k - 1) * ns], k >= 1: read where used, not held across the
  // seeds; nup_0 = nu0 = n (the window size) is never stored
  T2 = nu0 * a0;
  ab = fabs(T2);
  U = 0.0;
  A0 = a0;
#pragma unroll
  for (int k = 0; k <= N; ++k) {
    const double dk = (k & 1) ? d_even : d_odd;
    const double bk = (k & 1) ? bnd_odd : bnd_even;
    const double x = fma(s0, a_cur, fma(dk, inv2k, -bk));
    if (k == 0) X0 = x;
    U = fma(k == 0 ? nu0 : nup[(k - 1) * ns], x, U);
    if (k < N) {
      const double a_next = fma(c_rec[2 * k], x, c_rec[2 * k + 1] * a_prev);
      if (k & 1)
        d_odd = fma((double)(2 * k + 1), a_cur, d_odd);
      else
        d_even = fma((double)(2 * k + 1), a_cur, d_even);
      a_prev = a_cur;
      a_cur = a_next;
      const double nk = nup[k * ns];
      T2 = fma(nk, a_next, T2);
      ab = fma(fabs(nk), fabs(a_next), ab);
    }
  }
}

// Regime B (lambda < 2, t0 in [-1,2]): the integrand is smooth on [0,1]; a
// 16-node Gauss-Legendre rule with a constant (N+2) x 16 table, fp32 (J_k =
// A_k / 2: one common factor).
template <int N>
__device__ __forceinline__ void integrals_regime_b(float lam, float t0, float A[N + 1],
                                                   float X[N + 1]) {
  float J[N + 2];
#pragma unroll
  for (int k = 0; k <= N + 1; ++k) J[k] = 0.0f;
#pragma unroll
  for (int q = 0; q < kGlB; ++q) {
    const float z = c_glB_x[q] - t0;
    const float e = __expf(-lam * z * z);
#pragma unroll
    for (int k = 0; k <= N + 1; ++k) J[k] = fmaf(c_glB_W[k][q], e, J[k]);
  }
#pragma unroll
  for (int k = 0; k <= N; ++k) {
    A[k] = J[k];
    const float jm = (k > 0) ? (float)k * J[k - 1] : 0.0f;
    X[k] = fmaf((float)(k + 1), J[k + 1], jm) * (1.0f / (float)(2 * k + 1));
  }
}

// Regime C (t0 outside [-1,2]): 24-node Gauss-Legendre on the effective
// support [a,b] of the integrand (truncated where it has decayed by e^-24 from
// its value at the nearer end of [0,1]), fp64, scaled by exp(lambda d^2).
template <int N>
__device__ __forceinline__ void integrals_regime_c(double lam, double t0, double A[N + 1],
                                                double X[N + 1]) {
  double a, b, d;
  if (t0 < 0.0) {
    d = -t0;
    a = 0.0;
    b = fmin(1.0, -d + sqrt(d * d + 24.0 / lam));
  } else {
    d = t0 - 1.0;
    b = 1.0;
    a = fmax(0.0, 1.0 - (-d + sqrt(d * d + 24.0 / lam)));
  }
  const double len = b - a;
  double acc[N + 2];
#pragma unroll
  for (int k = 0; k <= N + 1; ++k) acc[k] = 0.0;
  for (int q = 0; q < kGlC; ++q) {
    const double x = fma(len, c_glC_x[q], a);
    const double z = x - t0;
    const double e = c_glC_w[q] * len * exp(-lam * (z - d) * (z + d));
    const double s = 2.0 * x - 1.0;
    double p0 = 1.0, p1 = s;
    acc[0] += e;
    acc[1] += e * s;
#pragma unroll
    for (int k = 1; k <= N; ++k) {
      const double p2 = fma((double)(2 * k + 1) / (double)(k + 1) * s, p1,
                            -((double)k / (double)(k + 1)) * p0);
      acc[k + 1] += e * p2;
      p0 = p1;
      p1 = p2;
    }
  }
#pragma unroll
  for (int k = 0; k <= N; ++k) {
    A[k] = acc[k];
    const double jm = (k > 0) ? (double)k * acc[k - 1] : 0.0;
    X[k] = fma((double)(k + 1), acc[k + 1], jm) * (1.0 / (double)(2 * k + 1));
  }
}

// ---------------------------------------------------------------------------
// a6 + a7 + a8: from the scaled Legendre moments nup_k = (2k+1) sum_j P_k(w_j)
// of the window (w = stretched intensity in [-1,1], eq.(20)-(22)) to g-hat.
//   T2 = sum_k nup_k A_k          (= sum_k c_k I_k of eq.(29), Legendre form of c = A^{-1} mu)
//   U  = sum_k nup_k X_k          (= 2 T1 - T2)
//   g-hat = alpha + (beta-alpha) T1/T2 = mid + half * U/T2      eq.(29)
// The sums are fp64 (kappa up to 1e3 multiplies their rounding into the
// ratio); the ratio itself is rounded to fp32 (its error is 6e-8 * |U/T2|).
// Guard (reading R7): T2 <= 0 or kappa = sum_k |nup_k A_k| / T2 >
// 1e3 -> the N = 0 value alpha + (beta-alpha) I_1/I_0, i.e. U/T2 -> X_0/A_0.
enum Regime : int { kRegA = 0, kRegB = 1, kRegC = 2 };

// a6: lambda = (beta-alpha)^2 / (2 sigma^2) (eq.(25)) and
// theta_0 = (theta-alpha)/(beta-alpha), both rounded to fp32 (the
// output's sensitivity to them is ~1e-5 grey), and the regime.
// The regime alone, without the divisions (d > 0, sigma > 0): t0 < -1 <=> theta - alpha < -d,
// t0 > 2 <=> theta - alpha > 2 d, lambda < kLambdaSmall <=> d^2 < 2 kLambdaSmall sigma^2.
__device__ __forceinline__ int regime_of(float alpha, float beta, float theta, float sigma) {
  const float d = beta - alpha, x = theta - alpha;
  if (x < -d || x > 2.0f * d) return 2;  // kRegC
  return (d * d < (float)(2.0 * kLambdaSmall) * (sigma * sigma)) ? 1 : 0;  // kRegB : kRegA
}

__device__ __forceinline__ int range_params(float alpha, float beta, float theta, float sigma,
                                            float& lam, float& t0) {
  const float d = beta - alpha;  // exact unless the range spans >2^24 ulps
  t0 = __fdividef(theta - alpha, d);
  const float r = __fdividef(d, sigma);
  lam = 0.5f * r * r;
  if (t0 < -1.0f || t0 > 2.0f) return kRegC;
  return (lam < (float)kLambdaSmall) ? kRegB : kRegA;
}

// the fp64 sums of a8 (see above), rounded to fp32 once formed
template <int N>
__device__ __forceinline__ void contract(const double* nup, int ns, double nu0, const double A[N + 1],
                                         const double X[N + 1], float& T2f, float& Uf, float& abf,
                                         float& A0f, float& X0f) {
  double T2 = 0.0, U = 0.0, ab = 0.0;
#pragma unroll
  for (int k = 0; k <= N; ++k) {
    const double nk = k == 0 ? nu0 : nup[(k - 1) * ns];
    T2 = fma(nk, A[k], T2);
    ab = fma(fabs(nk), fabs(A[k]), ab);
    U = fma(nk, X[k], U);
  }
  T2f = (float)T2, Uf = (float)U, abf = (float)ab, A0f = (float)A[0], X0f = (float)X[0];
}

template <int N, bool TAB = false>
__device__ __forceinline__ PixelResult ghat_from_record(const double* nup, int ns, float theta,
                                                        float sigma, float alpha, float beta,
                                                        int regime, unsigned flags, bool want_t2n,
                                                        double n, const double* etab = nullptr,
                                                        bool want_kappa = true) {
  PixelResult res;
  res.code = 0u;
  double scale_log = 0.0;  // log of the common factor applied to A (diagnostics only)
  float T2f, Uf, abf, A0f, X0f;
  if (regime == kRegB) {
    float lam, t0;
    range_params(alpha, beta, theta, sigma, lam, t0);
    float A[N + 1], X[N + 1];
    integrals_regime_b<N>(lam, t0, A, X);
    float T2 = 0.0f, U = 0.0f, ab = 0.0f;
#pragma unroll
    for (int k = 0; k <= N; ++k) {
      const float v = k == 0 ? (float)n : (float)nup[(k - 1) * ns];
      const float t = v * A[k];
      T2 += t;
      ab += fabsf(t);
      U = fmaf(v, X[k], U);
    }
    T2f = T2, Uf = U, abf = ab, A0f = A[0], X0f = X[0];
    res.code |= kCodeSmallLambda;
    scale_log = -0.69314718055994530942;  // A = J here
  } else if (regime == kRegA) {
    const double da = (double)alpha, db = (double)beta, d = db - da;
    const double sg = (double)sigma;
    const double rds = rcp64(d * sg);  // one reciprocal for 1/d and 1/sigma
    const double rd = sg * rds;
    const double s0 = fma(2.0, (double)theta, -(da + db)) * rd;
    const double sk = 0.35355339059327376220 * d * (d * rds);  // d / (2 sqrt2 sigma)
    const double csk = 2.50662827463100050242 * sg * rd;         // sqrt(pi)/2 / sk
    const double sr = sg * rd, inv2k = 4.0 * sr * sr;             // 1/(2 kappa)
    double T2, U, ab, A0, X0;
    integrals_regime_a<N, TAB>(sk, s0, csk, inv2k, nup, ns, n, T2, U, ab, A0, X0, etab);
    T2f = (float)T2, Uf = (float)U, abf = (float)ab, A0f = (float)A0, X0f = (float)X0;
    if (want_t2n) {
      const double xa = sk * (1.0 - s0), xb = sk * (1.0 + s0);
      scale_log = (xa >= 0.0 && xb >= 0.0) ? 0.0 : fmin(xa * xa, xb * xb);
    }
  } else {
    double A[N + 1], X[N + 1];
    const double da = (double)alpha, db = (double)beta, d = db - da;
    const double t0 = ((double)theta - da) / d;
    const double r = d / (double)sigma, lam = 0.5 * r * r;
    integrals_regime_c<N>(lam, t0, A, X);
    res.code |= kCodeFarTheta;
    const double dist = t0 < 0.0 ? -t0 : t0 - 1.0;
    scale_log = lam * dist * dist - 0.69314718055994530942;  // A = J here
    contract<N>(nup, ns, n, A, X, T2f, Uf, abf, A0f, X0f);
  }
  // one division on the selected operands (2 ulp: the sums carry the cancellation, not the ratio)
  const bool guard = !(flags & kFlagLiteral) && (!(T2f > 0.0f) || abf > kKappaMax * T2f);
  if (guard) res.code |= kCodeGuard;
  const float ratio = __fdividef(guard ? X0f : Uf, guard ? A0f : T2f);
  res.kappa = !want_kappa ? 0.0f : (T2f > 0.0f) ? abf / T2f : CUDART_INF_F;
  // T2 / n in the units of eq.(29) (J = A/2, unscaled)
  res.t2n = want_t2n ? (float)(0.5 * (double)T2f / n * exp(-scale_log)) : 0.0f;
  const float mid = 0.5f * (alpha + beta), half = 0.5f * (beta - alpha);
  float g = fmaf(half, ratio, mid);
  if (flags & kFlagClamp) g = fminf(fmaxf(g, alpha), beta);
  res.g = g;
  return res;
}

// Legendre polynomial coefficients on [-1,1] as compile-time constants
// (dyadic rationals, exact in fp64 and encodable as instruction immediates):
// P_k(w) = 2^-k sum_m (-1)^m C(k,m) C(2k-2m,k) w^{k-2m}.
__host__ __device__ constexpr double binom_c(int n, int k) {
  double c = 1.0;
  for (int i = 1; i <= k; ++i) c = c * (double)(n - k + i) / (double)i;
  return c;
}
__host__ __device__ constexpr double leg_coef(int k, int r) {
  if (r > k || ((k - r) & 1)) return 0.0;
  const int m = (k - r) / 2;
  double v = binom_c(k, m) * binom_c(2 * k - 2 * m, k);
  for (int i = 0; i < k; ++i) v *= 0.5;
  return (m & 1) ? -v : v;
}

// a4 + a5: from window power sums in tile units to Legendre moments.
//   S[q] = sum_j u_j^q, q = 0..N (S[0] = n), u = (f - c_T) / s_T.
//   au, bu = alpha, beta in the same units (exact: s_T is a power of two).
// Taylor shift to the pixel midrange m, scaling by its half-range h gives the
// moments of w = (u - m)/h in [-1,1] (eq.(24) P:341-345 up to the affine map
// w = 2t - 1); the fixed Legendre table then gives nu_k = sum_j P_k(w_j).
// Returns false (flag) when the fp64 centring amplification
// ((1 + |m|)/h)^N exceeds 2^flag_bits ("Numerical envelope"), tested
// as 1 + |m| > flag_root * h with flag_root = 2^(flag_bits/N) from the host.
__device__ __forceinline__ bool stretch_flagged(double au, double bu, double flag_root) {
  const double m = 0.5 * (au + bu), h = 0.5 * (bu - au);
  return 1.0 + fabs(m) > flag_root * h;
}
// (m, h = the pixel's midrange and half-range in tile units, as stretch_flagged forms them)
template <int N>
__device__ __forceinline__ void nu_from_sums_mh(double S[N + 1], double m, double h, double* nup, int ns) {
#pragma unroll
  for (int i = 1; i <= N; ++i) {
#pragma unroll
    for (int k = N; k >= i; --k) S[k] = fma(-m, S[k - 1], S[k]);
  }
  const double ih = rcp64(h);
  double p = ih;
#pragma unroll
  for (int k = 1; k <= N; ++k) {
    S[k] *= p;
    p *= ih;
  }
#pragma unroll
  for (int k = 1; k <= N; ++k) {  // nup_k = (2k+1) nu_k: the fit's coefficients (a5); nup_0 = n
    double v = 0.0;
#pragma unroll
    for (int r = k & 1; r <= k; r += 2) v = fma((double)(2 * k + 1) * leg_coef(k, r), S[r], v);
    nup[(k - 1) * ns] = v;
  }
}
template <int N>
__device__ __forceinline__ void nu_from_sums(double S[N + 1], double au, double bu, double* nup,
                                             int ns) {
  nu_from_sums_mh<N>(S, 0.5 * (au + bu), 0.5 * (bu - au), nup, ns);
}

__device__ __forceinline__ int reflect_hi(int i, int n) { return i < n ? i : 2 * n - 1 - i; }
__device__ __forceinline__ int reflect_lo(int i) { return i >= 0 ? i : -i - 1; }
__device__ __forceinline__ int reflect_index(int i, int n) {
  // half-sample symmetric (reading R2); one fold: -n <= i < 2n
  return i < 0 ? -i - 1 : (i >= n ? 2 * n - 1 - i : i);
}

}  // namespace fabf
