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
constexpr double kLambdaSmall = 2.0;  // below: fixed-node quadrature (regime B)

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

// Estrin evaluation of sum_{j=LO}^{HI} c[j] x^(j-LO), pw[l] = x^(2^l): the
// dependency depth is ~log2(terms) instead of Horner's (terms - 1), which is
// what matters in this latency-bound kernel.
__host__ __device__ constexpr int estrin_split(int n) {
  int h = 1;
  while (2 * h < n) h *= 2;
  return h;
}
__host__ __device__ constexpr int ilog2c(int n) {
  int l = 0;
  while ((1 << (l + 1)) <= n) ++l;
  return l;
}
template <int LO, int HI>
__device__ __forceinline__ double estrin(const double* c, const double* pw) {
  constexpr int n = HI - LO + 1;
  if constexpr (n == 1) {
    return c[LO];
  } else {
    constexpr int h = estrin_split(n);
    return fma(estrin<LO + h, HI>(c, pw), pw[ilog2c(h)], estrin<LO, LO + h - 1>(c, pw));
  }
}
template <int DEG>
__device__ __forceinline__ double poly_estrin(const double* c, double x) {
  double pw[5];
  pw[0] = x;
#pragma unroll
  for (int l = 1; l < 5; ++l) pw[l] = pw[l - 1] * pw[l - 1];
  return estrin<0, DEG>(c, pw);
}

// exp(z) for z <= 0 in fp64 (z < -708 gives 0): Cody-Waite reduction by ln 2
// (hi/lo split), degree-12 Taylor polynomial on |r| <= ln2/2 (truncation
// < 2e-16), 2^k built in the exponent field.  Branch-free; coefficients in
// constant memory so DFMA reads them as c[] operands.
__constant__ double c_exp_poly[13] = {
    1.0, 1.0, 1.0 / 2, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040, 1.0 / 40320,
    1.0 / 362880, 1.0 / 3628800, 1.0 / 39916800, 1.0 / 479001600};
__device__ __forceinline__ double exp_nonpos(double z) {
  const double kd = rint(z * 1.4426950408889634074);
  double r = fma(kd, -6.93147180369123816490e-01, z);
  r = fma(kd, -1.90821492927058770002e-10, r);
  const double p = poly_estrin<12>(c_exp_poly, r);
  const long long k = (long long)kd;
  const double scale = __longlong_as_double((k + 1023) << 52);
  return (z < -708.0) ? 0.0 : p * scale;
}

#include "fabf_erfcx.cuh"

struct PixelResult {
  float g;
  float kappa;
  float t2n;
  unsigned code;
};

// ---------------------------------------------------------------------------
// a7: Legendre-Gauss integrals J_k = int_0^1 P~_k(t) exp(-lambda (t-t0)^2) dt,
// k = 0..N+1, up to one common positive factor per pixel (the ratio eq.(29) and
// the guard are invariant to it).  P~_k(t) = P_k(2t-1).
//
// Regime A (lambda >= 2, t0 in [-1,2]): the integration-by-parts idea of
// P:411-426 applied in the Legendre basis.  With s = 2t-1, kappa = lambda/4,
// s0 = 2t0-1, g(s) = exp(-kappa (s-s0)^2), a_k = int_{-1}^{1} P_k g ds = 2 J_k:
//   a_{k+1} = [(2k+1)(s0 a_k - (g(1) - (-1)^k g(-1) - D_k)/(2 kappa)) - k a_{k-1}]/(k+1)
//   D_k     = sum_{j<k, j = k-1 mod 2} (2j+1) a_j
// (from int P_k g' = [P_k g] - int P_k' g, s P_k = ((k+1)P_{k+1} + k P_{k-1})/(2k+1)
// and P_k' = sum (2j+1) P_j).  Seeds: a_0 by two erf (eq.(31)) written
// as erfc = erfcx * exp so that the two boundary exponentials g(+-1) (as in
// eq.(32)) are reused -- 2 erfcx + 2 exp, branch-free; when t0 is
// outside [0,1] everything is scaled by exp(kappa (nearer boundary distance)^2).
// fp64 throughout: the recurrence amplifies seed error ("Kernels").
// lam and t0 arrive rounded to fp32; kappa is re-derived from the fp32 sqrt so
// that the seeds and the recurrence describe one and the same problem.
template <int N>
__device__ __forceinline__ void integrals_regime_a(float lam, float t0, float J[N + 2]) {
  const double sk = (double)sqrtf(0.25f * lam);
  const double kap = sk * sk;
  const double s0 = 2.0 * (double)t0 - 1.0;
  const double xa = sk * (1.0 - s0), xb = sk * (1.0 + s0);  // s = +1 and s = -1 ends
  const double qa = xa * xa, qb = xb * xb;
  const bool a_near = qa < qb;
  const double qn = a_near ? qa : qb, qf = a_near ? qb : qa;
  const double E = exp_nonpos(qn - qf);        // <= 1
  const bool inside = (xa >= 0.0) && (xb >= 0.0);
  const double Gn = inside ? exp_nonpos(-qn) : 1.0;  // scale 1 inside, exp(qn) outside
  const double ca = erfcx_pos(fabs(xa)), cb = erfcx_pos(fabs(xb));
  const double cn = a_near ? ca : cb, cf = a_near ? cb : ca;
  const double gn = Gn, gf = Gn * E;
  const double c = 0.88622692545275801365 / sk;  // sqrt(pi)/2 / sqrt(kappa)
  // erf(xa) + erf(xb): inside 2 - erfc(xa) - erfc(xb); outside erfc(|x_near|) - erfc(x_far)
  const double a0 = c * (inside ? (2.0 - cn * gn - cf * gf) : (cn * gn - cf * gf));
  const double gp = a_near ? gn : gf, gm = a_near ? gf : gn;
  const double inv2k = 0.5 / kap;  // 1/(2 kappa)
  const double bnd_even = (gp - gm) * inv2k, bnd_odd = (gp + gm) * inv2k;
  double a_prev = 0.0, a_cur = a0, d_even = 0.0, d_odd = 0.0;
  J[0] = (float)a0;
#pragma unroll
  for (int k = 0; k <= N; ++k) {
    const double dk = (k & 1) ? d_even : d_odd;
    const double bk = (k & 1) ? bnd_odd : bnd_even;
    const double x = fma(s0, a_cur, fma(dk, inv2k, -bk));
    const double a_next = fma((double)(2 * k + 1) / (double)(k + 1), x,
                              -((double)k / (double)(k + 1)) * a_prev);
    if (k & 1)
      d_odd = fma((double)(2 * k + 1), a_cur, d_odd);
    else
      d_even = fma((double)(2 * k + 1), a_cur, d_even);
    a_prev = a_cur;
    a_cur = a_next;
    J[k + 1] = (float)a_next;
  }
}

// Regime B (lambda < 2, t0 in [-1,2]): the integrand is smooth on [0,1]; a
// 16-node Gauss-Legendre rule with a constant (N+2) x 16 table, fp32.
template <int N>
__device__ __forceinline__ void integrals_regime_b(float lam, float t0, float J[N + 2]) {
  float E[kGlB];
#pragma unroll
  for (int q = 0; q < kGlB; ++q) {
    const float z = c_glB_x[q] - t0;
    E[q] = __expf(-lam * z * z);
  }
#pragma unroll
  for (int k = 0; k <= N + 1; ++k) {
    float s = 0.0f;
#pragma unroll
    for (int q = 0; q < kGlB; ++q) s = fmaf(c_glB_W[k][q], E[q], s);
    J[k] = s;
  }
}

// Regime C (t0 outside [-1,2]): 24-node Gauss-Legendre on the effective
// support [a,b] of the integrand (truncated where it has decayed by e^-24 from
// its value at the nearer end of [0,1]), fp64, scaled by exp(lambda d^2).
template <int N>
__device__ __noinline__ void integrals_regime_c(double lam, double t0, float J[N + 2]) {
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
    if (N + 1 >= 1) acc[1] += e * s;
#pragma unroll
    for (int k = 1; k <= N; ++k) {
      const double p2 = ((double)(2 * k + 1) * s * p1 - (double)k * p0) / (double)(k + 1);
      acc[k + 1] += e * p2;
      p0 = p1;
      p1 = p2;
    }
  }
#pragma unroll
  for (int k = 0; k <= N + 1; ++k) J[k] = (float)acc[k];
}

// ---------------------------------------------------------------------------
// a6 + a7 + a8: from the Legendre moments nu_k = sum_j P_k(w_j) of the window
// (w = stretched intensity in [-1,1], eq.(20)-(22)) to g-hat.
//   T2 = sum_k (2k+1) nu_k J_k  (= sum_k c_k I_k of eq.(29), Legendre form of c = A^{-1} mu)
//   T1/T2 = 1/2 + 1/2 sum_k nu_k [(k+1) J_{k+1} + k J_{k-1}] / T2
//   g-hat = alpha + (beta-alpha) T1/T2                     eq.(29)
// Guard (reading R7): T2 <= 0 or kappa > 1e3 -> the N = 0 value
// alpha + (beta-alpha) I_1/I_0.
enum Regime : int { kRegA = 0, kRegB = 1, kRegC = 2 };

// a6: lambda = (beta-alpha)^2 / (2 sigma^2) (eq.(25)) and
// theta_0 = (theta-alpha)/(beta-alpha), both rounded to fp32 (the
// output's sensitivity to them is ~1e-5 grey), and the regime.
__device__ __forceinline__ int range_params(float alpha, float beta, float theta, float sigma,
                                            float& lam, float& t0) {
  const float d = (float)((double)beta - (double)alpha);
  t0 = __fdividef((float)((double)theta - (double)alpha), d);
  const float r = __fdividef(d, sigma);
  lam = 0.5f * r * r;
  if (t0 < -1.0f || t0 > 2.0f) return kRegC;
  return (lam < (float)kLambdaSmall) ? kRegB : kRegA;
}

template <int N>
__device__ __forceinline__ PixelResult ghat_from_record(const float nu[N + 1], float lam, float t0,
                                                        float alpha, float beta, int regime,
                                                        unsigned flags, bool want_t2n, float n) {
  PixelResult res;
  res.code = 0u;
  float J[N + 2];
  double scale_log = 0.0;  // log of the common factor applied to J (diagnostics only)
  if (regime == kRegA) {
    integrals_regime_a<N>(lam, t0, J);
    if (want_t2n) {
      const double sk = (double)sqrtf(0.25f * lam), s0 = 2.0 * (double)t0 - 1.0;
      const double xa = sk * (1.0 - s0), xb = sk * (1.0 + s0);
      scale_log = (xa >= 0.0 && xb >= 0.0) ? 0.0 : fmin(xa * xa, xb * xb);
      scale_log += 0.69314718055994530942;  // a_k = 2 J_k
    }
  } else if (regime == kRegB) {
    integrals_regime_b<N>(lam, t0, J);
    res.code |= kCodeSmallLambda;
  } else {
    integrals_regime_c<N>((double)lam, (double)t0, J);
    res.code |= kCodeFarTheta;
    const double dist = t0 < 0.0f ? -(double)t0 : (double)t0 - 1.0;
    scale_log = (double)lam * dist * dist;
  }
  float T2 = 0.0f, U = 0.0f, ab = 0.0f;
#pragma unroll
  for (int k = 0; k <= N; ++k) {
    const float t = (float)(2 * k + 1) * nu[k] * J[k];
    T2 += t;
    ab += fabsf(t);
    const float jm = (k > 0) ? (float)k * J[k - 1] : 0.0f;
    U = fmaf(nu[k], fmaf((float)(k + 1), J[k + 1], jm), U);
  }
  float ratio;
  if (!(flags & kFlagLiteral) && (!(T2 > 0.0f) || ab > kKappaMax * T2)) {
    ratio = J[1] / J[0];
    res.code |= kCodeGuard;
  } else {
    ratio = U / T2;
  }
  res.kappa = (T2 > 0.0f) ? ab / T2 : CUDART_INF_F;
  res.t2n = want_t2n ? (float)((double)T2 / (double)n * exp(-scale_log)) : 0.0f;
  const double da = (double)alpha, db = (double)beta;
  const double mid = 0.5 * (da + db), half = 0.5 * (db - da);
  float g = (float)fma(half, (double)ratio, mid);
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
// ((1 + |m|)/h)^N exceeds 2^flag_bits ("Numerical envelope").
template <int N>
__device__ __forceinline__ bool nu_from_sums(double S[N + 1], double au, double bu, float nu[N + 1],
                                             float flag_bits) {
  const double m = 0.5 * (au + bu), h = 0.5 * (bu - au);
  const float ratio = (float)(1.0 + fabs(m)) / (float)h;
  if ((float)N * __log2f(ratio) > flag_bits) return false;
#pragma unroll
  for (int i = 1; i <= N; ++i) {
#pragma unroll
    for (int k = N; k >= i; --k) S[k] = fma(-m, S[k - 1], S[k]);
  }
  const double ih = 1.0 / h;
  double p = ih;
#pragma unroll
  for (int k = 1; k <= N; ++k) {
    S[k] *= p;
    p *= ih;
  }
#pragma unroll
  for (int k = 0; k <= N; ++k) {
    double v = 0.0;
#pragma unroll
    for (int r = k & 1; r <= k; r += 2) v = fma(leg_coef(k, r), S[r], v);
    nu[k] = (float)v;
  }
  return true;
}

__device__ __forceinline__ int reflect_index(int i, int n) {
  // half-sample symmetric (reading R2); one fold: -n <= i < 2n
  return i < 0 ? -i - 1 : (i >= n ? 2 * n - 1 - i : i);
}

}  // namespace fabf
