// fabf.cu -- B200 (sm_100a) implementation of the C ABI in include/fabf.h:
// the fast adaptive bilateral filter of Gavaskar & Chaudhury, arXiv 1811.02308,
// Algorithm 1 (P:446-477 of /root/reference/PAPER.md) with a box spatial kernel.
//
// Kernels ("Kernels"):
//   k_bounds_rows / k_bounds_cols  -- step a1, eq.(8): separable sliding min/max
//       by van Herk / Gil-Werman (the O(1) MAX-FILTER of Prop.1).
//   k_filter<N>  -- steps a3-a8: a CTA walks down a strip of TW output columns,
//       keeping fp64 vertical running power sums per input column (Prop.2,
//       P:274-282), horizontal window sums by warp prefix scans in shared
//       memory, then the per-pixel stretch / fit / integrals / ratio in
//       registers (fabf_device.cuh).
//   k_fallback<N> -- pixels whose centring amplification is too large get
//       exact direct window Legendre moments (one warp per pixel).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/fabf.h"
#include "fabf_device.cuh"

using namespace fabf;

// the opaque plan handle of include/fabf.h
struct fabf_plan_s {
  int B = 0, H = 0, W = 0;
  unsigned flags = 0;
  int device = 0;
  float* alpha = nullptr;  // workspace: bounds
  float* beta = nullptr;
  float* hmin = nullptr;   // workspace: row-pass min/max
  float* hmax = nullptr;
  int* fb_count = nullptr;  // exact-moment fallback list
  int* fb_list = nullptr;
  float* h_in = nullptr;  // device staging for fabf_filter_host
  float* h_out = nullptr;
  void* last_stream = nullptr;
};

namespace {

constexpr int kThreads = 256;
constexpr int kBoundsTX = 256;  // outputs per CTA row task (rows pass)
constexpr int kBoundsCX = 32;   // columns per CTA (columns pass)
constexpr int kMaxRho = 96;     // L = TW + 2 rho <= 256 input columns per strip
constexpr float kFlagBits = 26.0f;
constexpr int kMaxDynSmem = 227 * 1024 - 1024;  // opt-in limit minus static shared memory

using Plan = fabf_plan_s;

thread_local std::string g_last_error;

fabf_status_t fail(fabf_status_t s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

fabf_status_t cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? FABF_ERR_OUT_OF_MEMORY : FABF_ERR_CUDA;
}

#define FABF_CUDA(call, what)                       \
  do {                                              \
    cudaError_t e_ = (call);                        \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

// ----------------------------------------------------------------------------
// constant tables (computed on the host, copied once per device)
std::mutex g_tables_mu;
bool g_tables_ready[64] = {};

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  // nodes/weights on [0,1] by Newton iteration on P_n (long double)
  x.resize(n);
  w.resize(n);
  for (int i = 0; i < n; ++i) {
    long double z = cosl(3.14159265358979323846264338327950288L * (i + 0.75L) / (n + 0.5L));
    long double dp = 0;
    for (int it = 0; it < 100; ++it) {
      long double p0 = 1, p1 = z;
      for (int k = 2; k <= n; ++k) {
        long double p2 = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1);
      long double dz = p1 / dp;
      z -= dz;
      if (fabsl(dz) < 1e-19L) break;
    }
    long double p0 = 1, p1 = z;
    for (int k = 2; k <= n; ++k) {
      long double p2 = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    dp = n * (z * p1 - p0) / (z * z - 1);
    x[i] = (double)((z + 1) / 2);
    w[i] = (double)(1.0L / ((1 - z * z) * dp * dp));  // 2/(...) * 1/2 for [0,1]
  }
}

fabf_status_t ensure_tables(int dev) {
  std::lock_guard<std::mutex> lk(g_tables_mu);
  if (dev >= 0 && dev < 64 && g_tables_ready[dev]) return FABF_OK;
  // Legendre coefficients, (k+1) P_{k+1} = (2k+1) w P_k - k P_{k-1}
  double leg[kMaxN + 1][kMaxN + 1] = {};
  leg[0][0] = 1.0;
  leg[1][1] = 1.0;
  for (int k = 1; k < kMaxN; ++k)
    for (int r = 0; r <= k + 1; ++r) {
      double v = 0.0;
      if (r >= 1) v += (2 * k + 1) * leg[k][r - 1];
      v -= k * leg[k - 1][r];
      leg[k + 1][r] = v / (k + 1);
    }
  std::vector<double> xb, wb, xc, wc;
  gauss_legendre(kGlB, xb, wb);
  gauss_legendre(kGlC, xc, wc);
  float bx[kGlB], bW[kMaxN + 2][kGlB];
  for (int q = 0; q < kGlB; ++q) {
    bx[q] = (float)xb[q];
    long double s = 2.0L * xb[q] - 1.0L, p0 = 1, p1 = s;
    bW[0][q] = (float)(wb[q]);
    bW[1][q] = (float)(wb[q] * s);
    for (int k = 1; k <= kMaxN; ++k) {
      long double p2 = ((2 * k + 1) * s * p1 - k * p0) / (k + 1);
      bW[k + 1][q] = (float)(wb[q] * p2);
      p0 = p1;
      p1 = p2;
    }
  }
  FABF_CUDA(cudaMemcpyToSymbol(c_leg, leg, sizeof(leg)), "cudaMemcpyToSymbol(c_leg)");
  FABF_CUDA(cudaMemcpyToSymbol(c_glB_x, bx, sizeof(bx)), "cudaMemcpyToSymbol(c_glB_x)");
  FABF_CUDA(cudaMemcpyToSymbol(c_glB_W, bW, sizeof(bW)), "cudaMemcpyToSymbol(c_glB_W)");
  FABF_CUDA(cudaMemcpyToSymbol(c_glC_x, xc.data(), sizeof(double) * kGlC), "cudaMemcpyToSymbol(c_glC_x)");
  FABF_CUDA(cudaMemcpyToSymbol(c_glC_w, wc.data(), sizeof(double) * kGlC), "cudaMemcpyToSymbol(c_glC_w)");
  if (dev >= 0 && dev < 64) g_tables_ready[dev] = true;
  return FABF_OK;
}

}  // namespace

// ============================================================================
// step a1: bounds.  Rows pass: grid (ceil(W/TX), H, B).  Each CTA stages the
// row segment [x0-rho, x0+TX+rho) (reflected) and computes, per block of
// w = 2rho+1 staged samples, the prefix and suffix min/max (one thread per
// block and direction); output x takes min(S[x], P[x+2rho]) (van Herk /
// Gil-Werman: 3 comparisons per sample and pass, independent of rho).
__global__ void __launch_bounds__(kThreads) k_bounds_rows(const float* __restrict__ img, int H,
                                                           int W, int rho,
                                                           float* __restrict__ hmin,
                                                           float* __restrict__ hmax) {
  extern __shared__ float sm[];
  const int w = 2 * rho + 1;
  const int x0 = blockIdx.x * kBoundsTX;
  const int y = blockIdx.y;
  const size_t plane = (size_t)blockIdx.z * H * W;
  const int nout = min(kBoundsTX, W - x0);
  const int L = nout + 2 * rho;
  float* f = sm;
  float* Pmin = f + (kBoundsTX + 2 * kMaxRho);
  float* Pmax = Pmin + (kBoundsTX + 2 * kMaxRho);
  float* Smin = Pmax + (kBoundsTX + 2 * kMaxRho);
  float* Smax = Smin + (kBoundsTX + 2 * kMaxRho);
  const float* row = img + plane + (size_t)y * W;
  for (int c = threadIdx.x; c < L; c += blockDim.x) f[c] = row[reflect_index(x0 - rho + c, W)];
  __syncthreads();
  const int nb = (L + w - 1) / w;
  for (int t = threadIdx.x; t < 2 * nb; t += blockDim.x) {
    const int blk = t >> 1;
    const int s = blk * w, e = min(L, s + w);
    if ((t & 1) == 0) {
      float mn = f[s], mx = f[s];
      Pmin[s] = mn;
      Pmax[s] = mx;
      for (int c = s + 1; c < e; ++c) {
        const float v = f[c];
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
        Pmin[c] = mn;
        Pmax[c] = mx;
      }
    } else {
      float mn = f[e - 1], mx = f[e - 1];
      Smin[e - 1] = mn;
      Smax[e - 1] = mx;
      for (int c = e - 2; c >= s; --c) {
        const float v = f[c];
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
        Smin[c] = mn;
        Smax[c] = mx;
      }
    }
  }
  __syncthreads();
  float* omin = hmin + plane + (size_t)y * W + x0;
  float* omax = hmax + plane + (size_t)y * W + x0;
  for (int x = threadIdx.x; x < nout; x += blockDim.x) {
    omin[x] = fminf(Smin[x], Pmin[x + 2 * rho]);
    omax[x] = fmaxf(Smax[x], Pmax[x + 2 * rho]);
  }
}

// Columns pass: grid (ceil(W/32), ceil(H/TY), B), block (32, 8).  Same van
// Herk / Gil-Werman scheme along y on the row-pass output.
__global__ void __launch_bounds__(kThreads) k_bounds_cols(const float* __restrict__ hmin,
                                                           const float* __restrict__ hmax, int H,
                                                           int W, int rho, int TY,
                                                           float* __restrict__ amin,
                                                           float* __restrict__ bmax) {
  extern __shared__ float sm[];
  const int w = 2 * rho + 1;
  const int x0 = blockIdx.x * kBoundsCX;
  const int y0 = blockIdx.y * TY;
  const size_t plane = (size_t)blockIdx.z * H * W;
  const int nrow = min(TY, H - y0);
  const int L = nrow + 2 * rho;
  const int LS = TY + 2 * rho;
  const int tx = threadIdx.x, ty = threadIdx.y;
  float* vmin = sm;
  float* vmax = vmin + LS * kBoundsCX;
  float* Pmin = vmax + LS * kBoundsCX;
  float* Pmax = Pmin + LS * kBoundsCX;
  float* Smin = Pmax + LS * kBoundsCX;
  float* Smax = Smin + LS * kBoundsCX;
  const int x = x0 + tx;
  const bool colok = x < W;
  for (int r = ty; r < L; r += blockDim.y) {
    const int yy = reflect_index(y0 - rho + r, H);
    const size_t o = plane + (size_t)yy * W + (colok ? x : 0);
    vmin[r * kBoundsCX + tx] = colok ? hmin[o] : 0.0f;
    vmax[r * kBoundsCX + tx] = colok ? hmax[o] : 0.0f;
  }
  __syncthreads();
  const int nb = (L + w - 1) / w;
  // task = (block, direction), tx = column
  for (int t = ty; t < 2 * nb; t += blockDim.y) {
    const int blk = t >> 1;
    const int s = blk * w, e = min(L, s + w);
    if ((t & 1) == 0) {
      float mn = vmin[s * kBoundsCX + tx], mx = vmax[s * kBoundsCX + tx];
      Pmin[s * kBoundsCX + tx] = mn;
      Pmax[s * kBoundsCX + tx] = mx;
      for (int r = s + 1; r < e; ++r) {
        mn = fminf(mn, vmin[r * kBoundsCX + tx]);
        mx = fmaxf(mx, vmax[r * kBoundsCX + tx]);
        Pmin[r * kBoundsCX + tx] = mn;
        Pmax[r * kBoundsCX + tx] = mx;
      }
    } else {
      float mn = vmin[(e - 1) * kBoundsCX + tx], mx = vmax[(e - 1) * kBoundsCX + tx];
      Smin[(e - 1) * kBoundsCX + tx] = mn;
      Smax[(e - 1) * kBoundsCX + tx] = mx;
      for (int r = e - 2; r >= s; --r) {
        mn = fminf(mn, vmin[r * kBoundsCX + tx]);
        mx = fmaxf(mx, vmax[r * kBoundsCX + tx]);
        Smin[r * kBoundsCX + tx] = mn;
        Smax[r * kBoundsCX + tx] = mx;
      }
    }
  }
  __syncthreads();
  if (!colok) return;
  for (int r = ty; r < nrow; r += blockDim.y) {
    const size_t o = plane + (size_t)(y0 + r) * W + x;
    amin[o] = fminf(Smin[r * kBoundsCX + tx], Pmin[(r + 2 * rho) * kBoundsCX + tx]);
    bmax[o] = fmaxf(Smax[r * kBoundsCX + tx], Pmax[(r + 2 * rho) * kBoundsCX + tx]);
  }
}

// ============================================================================
// steps a3-a8.  Grid (ceil(W/TW), ceil(H/SH), B), 256 threads, RB = 256/TW
// output rows per step.  Shared memory: f ring [w][L] (fp32) and the per-step
// prefix-sum buffer [RB][N][L] (fp64).  L = TW + 2 rho <= 256.
struct FilterArgs {
  const float* img;
  const float* theta;
  const float* sigma;
  const float* alpha;
  const float* beta;
  float* out;
  int H, W, rho, TW, SH;
  unsigned flags;
  float flag_bits;
  int* fb_count;
  int* fb_list;
  float* d_kappa;
  float* d_t2n;
  unsigned char* d_code;
};

template <int N>
__global__ void __launch_bounds__(kThreads, 2) k_filter(FilterArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int rho = a.rho, w = 2 * rho + 1, TW = a.TW;
  const int RB = kThreads / TW;
  const int x0 = blockIdx.x * TW;
  const int Y0 = blockIdx.y * a.SH;
  const int H = a.H, W = a.W;
  const int Y1 = min(H, Y0 + a.SH);  // output rows [Y0, Y1)
  const int L = TW + 2 * rho;
  const size_t plane = (size_t)blockIdx.z * H * W;
  const int tid = threadIdx.x;
  double* Ps = reinterpret_cast<double*>(smraw);            // [RB][N][L]
  float* fring = reinterpret_cast<float*>(Ps + (size_t)RB * (N > 0 ? N : 1) * L);  // [w][L]
  __shared__ float red_min[kThreads / 32], red_max[kThreads / 32];

  // ---- tile-local centre c_T and power-of-two scale s_T from the bounds of
  // ---- the tile's outputs (their windows cover exactly the tile footprint)
  float lmin = CUDART_INF_F, lmax = -CUDART_INF_F;
  {
    const int ox = x0 + (tid % TW);
    for (int yy = Y0 + tid / TW; yy < Y1; yy += RB) {
      if (ox < W) {
        const size_t o = plane + (size_t)yy * W + ox;
        lmin = fminf(lmin, a.alpha[o]);
        lmax = fmaxf(lmax, a.beta[o]);
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      lmin = fminf(lmin, __shfl_xor_sync(0xffffffffu, lmin, off));
      lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, off));
    }
    if ((tid & 31) == 0) {
      red_min[tid >> 5] = lmin;
      red_max[tid >> 5] = lmax;
    }
    __syncthreads();
    lmin = red_min[0];
    lmax = red_max[0];
    for (int i = 1; i < kThreads / 32; ++i) {
      lmin = fminf(lmin, red_min[i]);
      lmax = fmaxf(lmax, red_max[i]);
    }
  }
  const double cT = 0.5 * ((double)lmin + (double)lmax);
  double halfr = 0.5 * ((double)lmax - (double)lmin);
  int e2 = 0;
  if (halfr > 0.0) frexp(halfr, &e2);
  const double invS = ldexp(1.0, -e2);  // 1/s_T, s_T = 2^e2 >= half range: exact scaling

  // ---- column-owner state (thread c owns input column c of the strip)
  const int c = tid;
  const bool owner = c < L;
  const int xin = reflect_index(min(x0 - rho + c, W - 1 + rho), W);
  double V[N + 1];
#pragma unroll
  for (int q = 0; q <= N; ++q) V[q] = 0.0;
  const int ystart = Y0 - rho;
  int slot = 0, loaded = 0;

  auto enter_row = [&](int yin) {
    // one entering row for this column: ring update + running power sums
    if (!owner) return;
    const float fv = a.img[plane + (size_t)reflect_index(yin, H) * W + xin];
    float* cell = fring + (size_t)slot * L + c;
    const float fo = *cell;
    *cell = fv;
    const double u = ((double)fv - cT) * invS;
    if (loaded >= w) {
      const double uo = ((double)fo - cT) * invS;
      double pu = u, po = uo;
#pragma unroll
      for (int q = 1; q <= N; ++q) {
        V[q] += pu - po;
        pu *= u;
        po *= uo;
      }
    } else {
      double pu = u;
#pragma unroll
      for (int q = 1; q <= N; ++q) {
        V[q] += pu;
        pu *= u;
      }
    }
    slot = (slot + 1 == w) ? 0 : slot + 1;
    ++loaded;
  };

  // prologue: rows ystart .. Y0 + rho - 1 (no outputs yet)
  for (int yin = ystart; yin < Y0 + rho; ++yin) enter_row(yin);
  if (!owner) loaded += 2 * rho;  // keep counters consistent (unused)

  const float n = (float)(w * w);
  const int lane = tid & 31, warp = tid >> 5;
  const int E = (L + 31) / 32;

  for (int Yb = Y0; Yb < Y1; Yb += RB) {
    const int nr = min(RB, Y1 - Yb);
    // ---- phase A: entering rows Yb+r+rho, write V into the prefix buffer
    for (int r = 0; r < nr; ++r) {
      enter_row(Yb + r + rho);
      if (owner) {
#pragma unroll
        for (int q = 1; q <= N; ++q) Ps[((size_t)r * N + (q - 1)) * L + c] = V[q];
      }
    }
    __syncthreads();
    // ---- phase B: inclusive prefix sums over c for each (r, q), one warp per scan
    if (N > 0) {
      for (int s = warp; s < nr * N; s += kThreads / 32) {
        double* row = Ps + (size_t)s * L;
        double loc[8];
        double tot = 0.0;
        const int cb = lane * E;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (e < E && cb + e < L) tot += row[cb + e];
          loc[e] = tot;
        }
        double inc = tot;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const double v = __shfl_up_sync(0xffffffffu, inc, off);
          if (lane >= off) inc += v;
        }
        const double excl = inc - tot;
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (e < E && cb + e < L) row[cb + e] = loc[e] + excl;
      }
    }
    __syncthreads();
    // ---- phase C: one output pixel per thread
    {
      const int r = tid / TW, x = tid % TW;
      const int Y = Yb + r, X = x0 + x;
      if (r < nr && X < W) {
        const size_t o = plane + (size_t)Y * W + X;
        const float al = a.alpha[o], be = a.beta[o];
        PixelResult res;
        bool done = true;
        if (al == be) {  // P:204, Algorithm 1 lines 4-5
          res.g = a.img[o];
          res.kappa = 1.0f;
          res.t2n = 1.0f;
          res.code = kCodeIdentity;
        } else {
          double S[N + 1];
          S[0] = (double)n;
#pragma unroll
          for (int q = 1; q <= N; ++q) {
            const double* row = Ps + ((size_t)r * N + (q - 1)) * L;
            S[q] = row[x + 2 * rho] - (x > 0 ? row[x - 1] : 0.0);
          }
          float nu[N + 1];
          const double au = ((double)al - cT) * invS, bu = ((double)be - cT) * invS;
          if (nu_from_sums<N>(S, au, bu, nu, a.flag_bits)) {
            res = ghat_from_nu<N>(nu, al, be, a.theta[o], a.sigma[o], n, a.flags);
          } else {
            done = false;  // exact-moment fallback pass writes this pixel
            const int slotfb = atomicAdd(a.fb_count, 1);
            a.fb_list[slotfb] = (int)(o);
          }
        }
        if (done) {
          a.out[o] = res.g;
          if (a.d_kappa) a.d_kappa[o] = res.kappa;
          if (a.d_t2n) a.d_t2n[o] = res.t2n;
          if (a.d_code) a.d_code[o] = (unsigned char)res.code;
        }
      }
    }
    __syncthreads();
  }
}

// ============================================================================
// exact-moment fallback: one warp per listed pixel; lanes split the window,
// nu_k = sum_j P_k(w_j) directly in fp64, warp reduction, then the same
// per-pixel integrals / ratio as k_filter.
template <int N>
__global__ void __launch_bounds__(kThreads) k_fallback(FilterArgs a) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int count = *a.fb_count;
  const int rho = a.rho, w = 2 * rho + 1, n = w * w;
  const int H = a.H, W = a.W;
  for (int i = gw; i < count; i += nw) {
    const int o = a.fb_list[i];
    const int b = o / (H * W), rem = o - b * H * W, y = rem / W, x = rem - y * W;
    const float* img = a.img + (size_t)b * H * W;
    const double al = a.alpha[o], be = a.beta[o];
    const double mid = 0.5 * (al + be), ih = 2.0 / (be - al);
    double acc[N + 1];
#pragma unroll
    for (int k = 0; k <= N; ++k) acc[k] = 0.0;
    for (int j = lane; j < n; j += 32) {
      const int dy = j / w - rho, dx = j % w - rho;
      const float fv = img[(size_t)reflect_index(y + dy, H) * W + reflect_index(x + dx, W)];
      const double s = ((double)fv - mid) * ih;
      double p0 = 1.0, p1 = s;
      acc[0] += 1.0;
      if (N >= 1) acc[1] += s;
#pragma unroll
      for (int k = 1; k < N; ++k) {
        const double p2 = ((double)(2 * k + 1) * s * p1 - (double)k * p0) / (double)(k + 1);
        acc[k + 1] += p2;
        p0 = p1;
        p1 = p2;
      }
    }
#pragma unroll
    for (int k = 0; k <= N; ++k)
      for (int off = 16; off > 0; off >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
    if (lane == 0) {
      float nu[N + 1];
#pragma unroll
      for (int k = 0; k <= N; ++k) nu[k] = (float)acc[k];
      PixelResult res = ghat_from_nu<N>(nu, (float)al, (float)be, a.theta[o], a.sigma[o],
                                        (float)n, a.flags);
      a.out[o] = res.g;
      if (a.d_kappa) a.d_kappa[o] = res.kappa;
      if (a.d_t2n) a.d_t2n[o] = res.t2n;
      if (a.d_code) a.d_code[o] = (unsigned char)(res.code | kCodeFallback);
    }
  }
}

// ============================================================================
// host side
namespace {

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const char* pa = (const char*)a;
  const char* pb = (const char*)b;
  return pa < pb + nb && pb < pa + na;
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

fabf_status_t check_device(int* dev_out) {
  int dev = 0;
  FABF_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  cudaDeviceProp prop;
  FABF_CUDA(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(FABF_ERR_UNSUPPORTED, "device is sm_" + std::to_string(prop.major) +
                                          std::to_string(prop.minor) +
                                          "; this library is built for sm_100a (B200) only");
  *dev_out = dev;
  return FABF_OK;
}

// optional stage events (fabf_filter_profile): ev[0..4] recorded between kernels
thread_local cudaEvent_t* g_prof_ev = nullptr;

inline void prof_mark(int i, cudaStream_t st) {
  if (g_prof_ev) cudaEventRecord(g_prof_ev[i], st);
}

fabf_status_t launch_bounds(Plan* p, const float* img, int rho, float* alpha, float* beta,
                            cudaStream_t st) {
  const size_t smem_rows = sizeof(float) * 5 * (kBoundsTX + 2 * kMaxRho);
  dim3 g1((p->W + kBoundsTX - 1) / kBoundsTX, p->H, p->B);
  prof_mark(0, st);
  k_bounds_rows<<<g1, kThreads, smem_rows, st>>>(img, p->H, p->W, rho, p->hmin, p->hmax);
  FABF_CUDA(cudaGetLastError(), "k_bounds_rows launch");
  prof_mark(1, st);
  int TY = 64;
  while (TY > 8 && sizeof(float) * 6 * (TY + 2 * rho) * kBoundsCX > 160 * 1024) TY >>= 1;
  const size_t smem_cols = sizeof(float) * 6 * (TY + 2 * rho) * kBoundsCX;
  static bool attr_set = false;
  if (!attr_set) {
    FABF_CUDA(cudaFuncSetAttribute(k_bounds_cols, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   200 * 1024),
              "cudaFuncSetAttribute(k_bounds_cols)");
    attr_set = true;
  }
  dim3 g2((p->W + kBoundsCX - 1) / kBoundsCX, (p->H + TY - 1) / TY, p->B);
  k_bounds_cols<<<g2, dim3(kBoundsCX, kThreads / kBoundsCX), smem_cols, st>>>(
      p->hmin, p->hmax, p->H, p->W, rho, TY, alpha, beta);
  FABF_CUDA(cudaGetLastError(), "k_bounds_cols launch");
  prof_mark(2, st);
  return FABF_OK;
}

template <int N>
fabf_status_t launch_filter_n(FilterArgs& fa, int B, cudaStream_t st) {
  const int L = fa.TW + 2 * fa.rho, w = 2 * fa.rho + 1, RB = kThreads / fa.TW;
  const size_t smem = sizeof(double) * RB * (N > 0 ? N : 1) * L + sizeof(float) * w * L;
  static bool attr_set = false;
  if (!attr_set) {
    FABF_CUDA(cudaFuncSetAttribute(k_filter<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kMaxDynSmem),
              "cudaFuncSetAttribute(k_filter)");
    attr_set = true;
  }
  if (smem > kMaxDynSmem) return fail(FABF_ERR_INVALID_ARGUMENT, "rho too large for shared memory");
  dim3 grid((fa.W + fa.TW - 1) / fa.TW, (fa.H + fa.SH - 1) / fa.SH, B);
  k_filter<N><<<grid, kThreads, smem, st>>>(fa);
  FABF_CUDA(cudaGetLastError(), "k_filter launch");
  prof_mark(3, st);
  k_fallback<N><<<148 * 2, kThreads, 0, st>>>(fa);
  FABF_CUDA(cudaGetLastError(), "k_fallback launch");
  prof_mark(4, st);
  return FABF_OK;
}

fabf_status_t launch_filter(FilterArgs& fa, int N, int B, cudaStream_t st) {
  switch (N) {
    case 0: return launch_filter_n<0>(fa, B, st);
    case 1: return launch_filter_n<1>(fa, B, st);
    case 2: return launch_filter_n<2>(fa, B, st);
    case 3: return launch_filter_n<3>(fa, B, st);
    case 4: return launch_filter_n<4>(fa, B, st);
    case 5: return launch_filter_n<5>(fa, B, st);
    case 6: return launch_filter_n<6>(fa, B, st);
    case 7: return launch_filter_n<7>(fa, B, st);
    case 8: return launch_filter_n<8>(fa, B, st);
    case 9: return launch_filter_n<9>(fa, B, st);
    case 10: return launch_filter_n<10>(fa, B, st);
    default: return fail(FABF_ERR_UNSUPPORTED, "N > FABF_MAX_N");
  }
}

fabf_status_t validate_common(Plan* p, int rho) {
  if (!p) return fail(FABF_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (rho < 0) return fail(FABF_ERR_INVALID_ARGUMENT, "rho < 0");
  if (2 * rho + 1 > p->H || 2 * rho + 1 > p->W)
    return fail(FABF_ERR_INVALID_ARGUMENT, "2*rho+1 exceeds min(height, width)");
  if (rho > kMaxRho)
    return fail(FABF_ERR_INVALID_ARGUMENT, "rho > " + std::to_string(kMaxRho) + " not supported");
  return FABF_OK;
}

fabf_status_t filter_impl(Plan* p, const float* img, const float* theta, const float* sigma,
                          int rho, int N, float* out, const fabf_diag_t* diag, cudaStream_t st) {
  fabf_status_t s = validate_common(p, rho);
  if (s != FABF_OK) return s;
  if (N < 0) return fail(FABF_ERR_INVALID_ARGUMENT, "N < 0");
  if (N > FABF_MAX_N) return fail(FABF_ERR_UNSUPPORTED, "N > FABF_MAX_N");
  if (!img || !theta || !sigma || !out) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL image pointer");
  if (!aligned16(img) || !aligned16(theta) || !aligned16(sigma) || !aligned16(out))
    return fail(FABF_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  const size_t bytes = sizeof(float) * (size_t)p->B * p->H * p->W;
  if (overlaps(out, bytes, img, bytes) || overlaps(out, bytes, theta, bytes) ||
      overlaps(out, bytes, sigma, bytes))
    return fail(FABF_ERR_INVALID_ARGUMENT, "out overlaps an input");
  FABF_CUDA(cudaMemsetAsync(p->fb_count, 0, sizeof(int), st), "cudaMemsetAsync(fb_count)");
  p->last_stream = st;
  s = launch_bounds(p, img, rho, p->alpha, p->beta, st);
  if (s != FABF_OK) return s;
  if (diag && diag->alpha)
    FABF_CUDA(cudaMemcpyAsync(diag->alpha, p->alpha, bytes, cudaMemcpyDeviceToDevice, st), "copy alpha");
  if (diag && diag->beta)
    FABF_CUDA(cudaMemcpyAsync(diag->beta, p->beta, bytes, cudaMemcpyDeviceToDevice, st), "copy beta");
  FilterArgs fa;
  fa.img = img;
  fa.theta = theta;
  fa.sigma = sigma;
  fa.alpha = p->alpha;
  fa.beta = p->beta;
  fa.out = out;
  fa.H = p->H;
  fa.W = p->W;
  fa.rho = rho;
  fa.TW = (rho <= 64) ? 128 : 64;
  fa.SH = 128;
  fa.flags = p->flags;
  fa.flag_bits = kFlagBits;
  fa.fb_count = p->fb_count;
  fa.fb_list = p->fb_list;
  fa.d_kappa = diag ? diag->kappa : nullptr;
  fa.d_t2n = diag ? diag->t2n : nullptr;
  fa.d_code = diag ? diag->code : nullptr;
  return launch_filter(fa, N, p->B, st);
}

}  // namespace

// ============================================================================
extern "C" {

fabf_status_t fabf_plan(fabf_plan_t* plan, int batch, int height, int width, unsigned flags) {
  if (!plan) return fail(FABF_ERR_INVALID_ARGUMENT, "plan out-pointer is NULL");
  *plan = nullptr;
  if (batch < 1 || height < 1 || width < 1)
    return fail(FABF_ERR_INVALID_ARGUMENT, "batch, height and width must be >= 1");
  if ((size_t)batch * height * width >= (size_t)1 << 31)
    return fail(FABF_ERR_INVALID_ARGUMENT, "more than 2^31-1 pixels per call");
  if (flags & ~(unsigned)(FABF_FLAG_LITERAL | FABF_FLAG_CLAMP))
    return fail(FABF_ERR_INVALID_ARGUMENT, "unknown flag bits");
  int dev = 0;
  fabf_status_t s = check_device(&dev);
  if (s != FABF_OK) return s;
  s = ensure_tables(dev);
  if (s != FABF_OK) return s;
  Plan* p = new (std::nothrow) Plan();
  if (!p) return fail(FABF_ERR_OUT_OF_MEMORY, "host allocation failed");
  p->B = batch;
  p->H = height;
  p->W = width;
  p->flags = flags;
  p->device = dev;
  const size_t px = (size_t)batch * height * width;
  cudaError_t e;
  if ((e = cudaMalloc(&p->alpha, px * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&p->beta, px * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&p->hmin, px * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&p->hmax, px * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&p->fb_count, sizeof(int))) != cudaSuccess ||
      (e = cudaMalloc(&p->fb_list, px * sizeof(int))) != cudaSuccess) {
    fabf_destroy(p);
    return cuda_fail(e, "cudaMalloc(plan workspace)");
  }
  *plan = p;
  return FABF_OK;
}

fabf_status_t fabf_filter(fabf_plan_t plan, const float* img, const float* theta,
                          const float* sigma, int rho, int N, float* out, void* stream) {
  return filter_impl(reinterpret_cast<Plan*>(plan), img, theta, sigma, rho, N, out, nullptr,
                     (cudaStream_t)stream);
}

fabf_status_t fabf_filter_diag(fabf_plan_t plan, const float* img, const float* theta,
                               const float* sigma, int rho, int N, float* out,
                               const fabf_diag_t* diag, void* stream) {
  return filter_impl(reinterpret_cast<Plan*>(plan), img, theta, sigma, rho, N, out, diag,
                     (cudaStream_t)stream);
}

fabf_status_t fabf_bounds(fabf_plan_t plan, const float* img, int rho, float* alpha, float* beta,
                          void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  fabf_status_t s = validate_common(p, rho);
  if (s != FABF_OK) return s;
  if (!img || !alpha || !beta) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!aligned16(img) || !aligned16(alpha) || !aligned16(beta))
    return fail(FABF_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  const size_t bytes = sizeof(float) * (size_t)p->B * p->H * p->W;
  if (overlaps(alpha, bytes, img, bytes) || overlaps(beta, bytes, img, bytes) ||
      overlaps(alpha, bytes, beta, bytes))
    return fail(FABF_ERR_INVALID_ARGUMENT, "outputs overlap");
  return launch_bounds(p, img, rho, alpha, beta, (cudaStream_t)stream);
}

fabf_status_t fabf_filter_host(fabf_plan_t plan, const float* img, const float* theta,
                               const float* sigma, int rho, int N, float* out, void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  if (!p) return fail(FABF_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (!img || !theta || !sigma || !out) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  const size_t px = (size_t)p->B * p->H * p->W, bytes = px * sizeof(float);
  if (!p->h_in) {
    cudaError_t e;
    if ((e = cudaMalloc(&p->h_in, 3 * bytes)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
    if ((e = cudaMalloc(&p->h_out, bytes)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
  }
  cudaStream_t st = (cudaStream_t)stream;
  FABF_CUDA(cudaMemcpyAsync(p->h_in, img, bytes, cudaMemcpyHostToDevice, st), "H2D img");
  FABF_CUDA(cudaMemcpyAsync(p->h_in + px, theta, bytes, cudaMemcpyHostToDevice, st), "H2D theta");
  FABF_CUDA(cudaMemcpyAsync(p->h_in + 2 * px, sigma, bytes, cudaMemcpyHostToDevice, st), "H2D sigma");
  fabf_status_t s = filter_impl(p, p->h_in, p->h_in + px, p->h_in + 2 * px, rho, N, p->h_out,
                                nullptr, st);
  if (s != FABF_OK) return s;
  FABF_CUDA(cudaMemcpyAsync(out, p->h_out, bytes, cudaMemcpyDeviceToHost, st), "D2H out");
  FABF_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  return FABF_OK;
}

fabf_status_t fabf_last_fallback_count(fabf_plan_t plan, long long* count) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  if (!p || !count) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  int c = 0;
  FABF_CUDA(cudaMemcpyAsync(&c, p->fb_count, sizeof(int), cudaMemcpyDeviceToHost,
                            (cudaStream_t)p->last_stream),
            "read fallback count");
  FABF_CUDA(cudaStreamSynchronize((cudaStream_t)p->last_stream), "cudaStreamSynchronize");
  *count = c;
  return FABF_OK;
}

fabf_status_t fabf_filter_profile(fabf_plan_t plan, const float* img, const float* theta,
                                  const float* sigma, int rho, int N, float* out, void* stream,
                                  float stage_ms[4]) {
  if (!stage_ms) return fail(FABF_ERR_INVALID_ARGUMENT, "stage_ms is NULL");
  cudaEvent_t ev[5];
  for (int i = 0; i < 5; ++i) FABF_CUDA(cudaEventCreate(&ev[i]), "cudaEventCreate");
  g_prof_ev = ev;
  fabf_status_t s = filter_impl(reinterpret_cast<Plan*>(plan), img, theta, sigma, rho, N, out,
                                nullptr, (cudaStream_t)stream);
  g_prof_ev = nullptr;
  if (s == FABF_OK) {
    cudaError_t e = cudaEventSynchronize(ev[4]);
    if (e != cudaSuccess) s = cuda_fail(e, "cudaEventSynchronize");
    for (int i = 0; i < 4 && s == FABF_OK; ++i) cudaEventElapsedTime(&stage_ms[i], ev[i], ev[i + 1]);
  }
  for (int i = 0; i < 5; ++i) cudaEventDestroy(ev[i]);
  return s;
}

fabf_status_t fabf_destroy(fabf_plan_t plan) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  if (!p) return FABF_OK;
  cudaFree(p->alpha);
  cudaFree(p->beta);
  cudaFree(p->hmin);
  cudaFree(p->hmax);
  cudaFree(p->fb_count);
  cudaFree(p->fb_list);
  cudaFree(p->h_in);
  cudaFree(p->h_out);
  delete p;
  return FABF_OK;
}

const char* fabf_status_string(fabf_status_t status) {
  switch (status) {
    case FABF_OK: return "FABF_OK";
    case FABF_ERR_INVALID_ARGUMENT: return "FABF_ERR_INVALID_ARGUMENT";
    case FABF_ERR_UNSUPPORTED: return "FABF_ERR_UNSUPPORTED";
    case FABF_ERR_CUDA: return "FABF_ERR_CUDA";
    case FABF_ERR_OUT_OF_MEMORY: return "FABF_ERR_OUT_OF_MEMORY";
  }
  return "unknown fabf_status_t";
}

const char* fabf_last_error_message(void) { return g_last_error.c_str(); }

int fabf_version(void) { return FABF_VERSION; }

}  // extern "C"
