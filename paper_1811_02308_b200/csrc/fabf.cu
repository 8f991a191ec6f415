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
#include <cuda.h>  // CUtensorMap (TMA descriptors; encoded through the runtime's driver entry point)
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
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
  float2* blkmm = nullptr;  // per bounds tile (min alpha, max beta), fabf_bounds only
  float2* hmm = nullptr;    // row-pass (min, max) plane of the separable bounds
  // k_filter's vertical-bounds suffix rings (per resident CTA, sized at plan
  // time for the largest rho the shape allows; L2-resident while in use)
  float2* ring = nullptr;
  long long ring_elems = 0;
  // exact-moment fallback: one counter per band of a call (slot b * kMaxBandsPlan
  // + k for band k of image b in fabf_filter_host, slot 0 otherwise); a band's
  // list is the region of fb_list at its own first pixel, so bands never share
  // entries and the call's total is the sum of its slots
  int* fb_count = nullptr;
  int* fb_list = nullptr;
  unsigned* fb_bits = nullptr;  // one bit per pixel, 32-pixel row words (all zero between calls)
  int* seg_list = nullptr;      // row words holding flagged pixels, per band region
  int* seg_count = nullptr;     // per band slot, like fb_count
  int fb_slots = 0;  // slots the last call used
  int launches = 0;  // kernels the last call launched (fabf_last_launch_count)
  // FABF_FLAG_DEBUG: [0] inputs violating the preconditions, [1] the first one's index
  unsigned long long* dbg = nullptr;
  float* h_in = nullptr;  // device staging for fabf_filter_host
  float* h_out = nullptr;
  void* last_stream = nullptr;
  // TMA descriptor of the last image k_bounds staged (per rho class)
  CUtensorMap tmap;
  const void* tmap_ptr = nullptr;
  int tmap_rc = -1;
  bool tmap_ok = false;
  // fabf_filter_host pipeline: copy streams and per-band events
  static constexpr int kMaxBandsPlan = 16;
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  cudaEvent_t ev_in[kMaxBandsPlan + 1] = {};
  cudaEvent_t ev_done[kMaxBandsPlan + 1] = {};
};

namespace {

constexpr int kThreads = 256;
constexpr int kMaxBands = fabf_plan_s::kMaxBandsPlan;  // fabf_filter_host row bands
// bounds inside k_filter by default for rho <= kFuseRho on calls of at most
// kFusePixels pixels (configs 1-2: one launch less outweighs the dearer
// in-kernel bounds); the separate bounds kernel elsewhere (faster at every rho
// of configs 3-5); FABF_FLAG_FUSED plans always fuse.
constexpr int kFuseRho = 5;
constexpr long long kFusePixels = 1LL << 21;
int g_fuse_rho = getenv("FABF_FUSE_RHO") ? atoi(getenv("FABF_FUSE_RHO")) : kFuseRho;
// segment cap: max(g_seg_min, g_seg_w w) rows (A/B switch FABF_SEG_MIN)
int g_seg_min = getenv("FABF_SEG_MIN") ? std::max(8, atoi(getenv("FABF_SEG_MIN"))) : 64;
// ... and g_seg_w window heights (FABF_SEG_W): long segments save prologues
// where they are dear (2 rho rows each), short ones keep the centring local
// (fewer fallback pixels) where they are cheap
int g_seg_w = getenv("FABF_SEG_W") ? std::max(1, atoi(getenv("FABF_SEG_W"))) : 6;
// fabf_filter_host row bands per frame (A/B switch FABF_HOST_BANDS, 1..16)
int g_host_bands = getenv("FABF_HOST_BANDS") ? std::max(1, std::min(16, atoi(getenv("FABF_HOST_BANDS")))) : 6;
#ifndef FABF_FILTER_MINB
#define FABF_FILTER_MINB 2
#endif
constexpr int kMaxRho = 96;     // L = TW + 2 rho <= 256 input columns per strip
#ifndef FABF_FLAG_BITS
#define FABF_FLAG_BITS 40.0f
#endif
constexpr float kFlagBits = FABF_FLAG_BITS;
constexpr int kMaxDynSmem = 227 * 1024 - 1024;  // opt-in limit minus static shared memory

using Plan = fabf_plan_s;

thread_local std::string g_last_error;
thread_local int g_launches = 0;  // kernels launched by the current entry point

fabf_status_t fail(fabf_status_t s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

// PDL launches of k_filter / k_fallback_seg (FABF_PDL=0 turns them off: A/B)
bool g_pdl = !(getenv("FABF_PDL") && atoi(getenv("FABF_PDL")) == 0);
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
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
constexpr int kMaxDevices = 64;
std::mutex g_tables_mu;
bool g_tables_ready[kMaxDevices] = {};
std::mutex g_launch_mu;  // per-device launch caches (attributes, occupancy, TMA encoder)

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
  if (g_tables_ready[dev]) return FABF_OK;
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
  FABF_CUDA(cudaMemcpyToSymbol(c_glB_x, bx, sizeof(bx)), "cudaMemcpyToSymbol(c_glB_x)");
  FABF_CUDA(cudaMemcpyToSymbol(c_glB_W, bW, sizeof(bW)), "cudaMemcpyToSymbol(c_glB_W)");
  FABF_CUDA(cudaMemcpyToSymbol(c_glC_x, xc.data(), sizeof(double) * kGlC), "cudaMemcpyToSymbol(c_glC_x)");
  FABF_CUDA(cudaMemcpyToSymbol(c_glC_w, wc.data(), sizeof(double) * kGlC), "cudaMemcpyToSymbol(c_glC_w)");
  {
    double e2[64];
    for (int j = 0; j < 64; ++j) e2[j] = (double)exp2l((long double)j / 64.0L);
    FABF_CUDA(cudaMemcpyToSymbol(c_exp2_64, e2, sizeof(e2)), "cudaMemcpyToSymbol(c_exp2_64)");
  }
  g_tables_ready[dev] = true;
  return FABF_OK;
}

}  // namespace

// ============================================================================
// step a1: bounds (eq.(8)) -- one CTA per kBT x kBT output tile,
// separable sliding min/max by van Herk / Gil-Werman (the O(1) MAX-FILTER of
// Prop.1), both passes in one kernel:
//   pass V: walkers = (footprint column, row segment); inputs straight from
//           global memory (lanes = adjacent columns: coalesced), results into
//           shared Vm[kBT][P] (P = kBT + 2 rho, odd pitch);
//   pass H: walkers = (output row, column segment) over Vm, results into
//           shared O[kBT][kBT + 1], then copied out coalesced as alpha, beta,
//           together with the tile's (min alpha, max beta) for k_filter.
// A walker with outputs o = 0..len-1 over inputs in(0 .. len + 2 rho - 1) cuts
// the inputs into blocks of w = 2 rho + 1 aligned at 0; for o in block b
//   out(o) = op(h(o), g(o + w - 1)),
// h = suffix op within block b (backward sweep, stored in the output slot),
// g = prefix op within block b + 1 (running register, empty at o = b w).
// 3 comparisons per sample and pass whatever rho is; comparisons only: exact.
constexpr int kBT = 64;    // bounds tile side (output rows and columns)
#ifndef FABF_BSEGV
#define FABF_BSEGV 32
#endif
#ifndef FABF_BSEGH
#define FABF_BSEGH 16
#endif
constexpr int kBSegV = FABF_BSEGV;  // pass-V segment length (rows)
constexpr int kBSegH = FABF_BSEGH;  // pass-H segment length (columns)

__device__ __forceinline__ float2 mm2(float2 a, float2 b) {
  return make_float2(fminf(a.x, b.x), fmaxf(a.y, b.y));
}

// Programmatic dependent launch (PDL): a kernel of the path lets the next one
// be scheduled as soon as all of its CTAs are running (launch_dependents), and
// the next one waits for the previous grid's completion and memory flush
// before touching anything it produced (wait; a no-op when launched without
// the attribute).  Hides the launch gap and the previous kernel's tail.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Loads are issued kU at a time ahead of the comparison chain (the walk is
// otherwise one dependent load per sample).
constexpr int kU = 8;
template <class Load, class Slot>
__device__ __forceinline__ void vhgw_walk(int len, int w, Load in, Slot slot) {
  for (int b0 = 0; b0 < len; b0 += w) {
    float2 run = make_float2(CUDART_INF_F, -CUDART_INF_F);
    int i = b0 + w - 1;
    for (; i - (kU - 1) >= b0; i -= kU) {  // h: suffix within block b
      float2 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = in(i - u);
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        run = mm2(run, v[u]);
        if (i - u < len) *slot(i - u) = run;
      }
    }
    for (; i >= b0; --i) {
      run = mm2(run, in(i));
      if (i < len) *slot(i) = run;
    }
    const int oe = min(b0 + w, len);
    // o = b0: the window is block b itself, out = h(b0) already in place
    float2 g = make_float2(CUDART_INF_F, -CUDART_INF_F);
    int o = b0 + 1;
    for (; o + kU - 1 < oe; o += kU) {  // g: prefix within block b + 1
      float2 v[kU], h[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        v[u] = in(o + u + w - 1);
        h[u] = *slot(o + u);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        g = mm2(g, v[u]);
        *slot(o + u) = mm2(h[u], g);
      }
    }
    for (; o < oe; ++o) {
      g = mm2(g, in(o + w - 1));
      *slot(o) = mm2(*slot(o), g);
    }
  }
}

// The same walk over shared memory with 32-bit strides and no per-sample
// predicates: in[i * sin] (float: min = max = value, or float2), out[o * sout].
__device__ __forceinline__ float2 mm_in(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 mm_in(float2 v) { return v; }
template <class TIn, int sin, int sout>
__device__ __forceinline__ void vhgw_run(const TIn* __restrict__ in, float2* __restrict__ out, int len,
                                         int w) {
  constexpr int B8 = 8;  // loads issued in batches ahead of the comparison chain
  for (int b0 = 0; b0 < len; b0 += w) {
    float2 run = make_float2(CUDART_INF_F, -CUDART_INF_F);
    const int top = b0 + w - 1, last = min(top, len - 1);
    int i = top;
    for (; i - (B8 - 1) > last; i -= B8) {  // beyond the outputs: no stores
      TIn v[B8];
#pragma unroll
      for (int u = 0; u < B8; ++u) v[u] = in[(i - u) * sin];
#pragma unroll
      for (int u = 0; u < B8; ++u) run = mm2(run, mm_in(v[u]));
    }
    for (; i > last; --i) run = mm2(run, mm_in(in[i * sin]));
    for (; i - (B8 - 1) >= b0; i -= B8) {  // h: suffix within block b
      TIn v[B8];
#pragma unroll
      for (int u = 0; u < B8; ++u) v[u] = in[(i - u) * sin];
#pragma unroll
      for (int u = 0; u < B8; ++u) {
        run = mm2(run, mm_in(v[u]));
        out[(i - u) * sout] = run;
      }
    }
    for (; i >= b0; --i) {
      run = mm2(run, mm_in(in[i * sin]));
      out[i * sout] = run;
    }
    float2 g = make_float2(CUDART_INF_F, -CUDART_INF_F);
    const int oe = min(b0 + w, len);
    int o = b0 + 1;
    for (; o + (B8 - 1) < oe; o += B8) {  // g: prefix within block b + 1
      TIn v[B8];
      float2 h[B8];
#pragma unroll
      for (int u = 0; u < B8; ++u) {
        v[u] = in[(o + u + w - 1) * sin];
        h[u] = out[(o + u) * sout];
      }
#pragma unroll
      for (int u = 0; u < B8; ++u) {
        g = mm2(g, mm_in(v[u]));
        out[(o + u) * sout] = mm2(h[u], g);
      }
    }
    for (; o < oe; ++o) {
      g = mm2(g, mm_in(in[(o + w - 1) * sin]));
      out[o * sout] = mm2(out[o * sout], g);
    }
  }
}

// A full segment of SEG <= w outputs (inputs in[0 .. SEG + w - 2]): every
// window [o, o + w - 1] is the suffix of block 0 (inputs [0, w)) from o joined
// with the prefix of block 1 up to o + w - 1, so the suffix values of the SEG
// output positions stay in registers (compile-time indices) and each output
// is stored once -- no read-back of the output slot.
template <int SEG, class TIn, int sin, int sout>
__device__ __forceinline__ void vhgw_seg(const TIn* __restrict__ in, float2* __restrict__ out, int w) {
  float2 suf[SEG];
  float2 run = make_float2(CUDART_INF_F, -CUDART_INF_F);
  {
    constexpr int B4 = 4;
    int i = w - 1;
    for (; i - (B4 - 1) >= SEG; i -= B4) {  // inputs above the outputs: accumulate only
      TIn v[B4];
#pragma unroll
      for (int u = 0; u < B4; ++u) v[u] = in[(i - u) * sin];
#pragma unroll
      for (int u = 0; u < B4; ++u) run = mm2(run, mm_in(v[u]));
    }
    for (; i >= SEG; --i) run = mm2(run, mm_in(in[i * sin]));
  }
#pragma unroll
  for (int i = SEG - 1; i >= 0; --i) {
    run = mm2(run, mm_in(in[i * sin]));
    suf[i] = run;
  }
  out[0] = suf[0];  // o = 0: the window is block 0 itself
  const TIn* nx = in + (w - 1) * sin;
  float2 g = make_float2(CUDART_INF_F, -CUDART_INF_F);
#pragma unroll
  for (int o = 1; o < SEG; ++o) {
    g = mm2(g, mm_in(nx[o * sin]));
    out[o * sout] = mm2(suf[o], g);
  }
}

// TMA (cp.async.bulk.tensor) staging of an interior footprint: one thread
// issues the 3-D box load, the CTA waits on an mbarrier.
__device__ __forceinline__ void tma_load_box(void* dst, const CUtensorMap* map, int x, int y, int b,
                                             unsigned long long* bar, unsigned bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned mb = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(d),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(b), "r"(mb)
      : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  const unsigned mb = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned mb = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(mb), "r"(parity)
        : "memory");
  }
}

// shared memory: F (staged footprint, fp32, row pitch FP; reused as O after
// pass V) and Vm (row pitch VP, odd).  Pitches are compile-time per rho class
// RC (rho <= RC) so that every walk address is a base plus an immediate.
template <int RC>
struct BoundsGeom {
  static constexpr int FP = kBT + 2 * RC + 4;    // >= footprint columns + TMA start alignment
  static constexpr int FR = kBT + 2 * RC;        // TMA box rows
  static constexpr int VP = (kBT + 2 * RC) | 1;  // odd: pass-H lanes (rows) conflict-free
  static constexpr int OP = kBT + 1;
};
template <int RC>
__host__ __device__ inline size_t bounds_f_bytes(int rho, bool stage) {
  using G = BoundsGeom<RC>;
  // staged: room for the whole TMA box (FR rows x FP) of interior tiles
  const size_t f = stage ? sizeof(float) * (size_t)G::FP * G::FR : 0;
  const size_t o = sizeof(float2) * (size_t)kBT * G::OP;
  return ((f > o ? f : o) + 15) & ~(size_t)15;
}
template <int RC>
__host__ inline size_t bounds_smem(int rho, bool stage) {
  return bounds_f_bytes<RC>(rho, stage) + sizeof(float2) * (size_t)kBT * BoundsGeom<RC>::VP;
}

template <int RC, bool kStage>
__global__ void __launch_bounds__(kThreads) k_bounds(const float* __restrict__ img, int H, int W,
                                                      int rho, float* __restrict__ amin,
                                                      float* __restrict__ bmax,
                                                      float2* __restrict__ blkmm, int b0, int ty0,
                                                      const __grid_constant__ CUtensorMap tmap,
                                                      int use_tma) {
  using G = BoundsGeom<RC>;
  pdl_trigger();
  __shared__ __align__(8) unsigned long long tbar;
  constexpr int FP = G::FP, VP = G::VP, OP = G::OP;
  extern __shared__ __align__(1024) unsigned char smb[];
  __shared__ float2 red[kThreads / 32];
  const int w = 2 * rho + 1;
  float* F = reinterpret_cast<float*>(smb);                                  // [ny + 2 rho][FP]
  float2* O = reinterpret_cast<float2*>(smb);                                // [kBT][OP] (after pass V)
  float2* Vm = reinterpret_cast<float2*>(smb + bounds_f_bytes<RC>(rho, kStage));  // [kBT][VP]
  // tile (blockIdx.x, ty0 + blockIdx.y) of image b0 + blockIdx.z (row bands: fabf_filter_host)
  const int ty = ty0 + blockIdx.y, bimg = b0 + blockIdx.z;
  const int x0 = blockIdx.x * kBT, y0 = ty * kBT;
  const size_t plane = (size_t)bimg * H * W;
  const int nx = min(kBT, W - x0), ny = min(kBT, H - y0);
  const int C = nx + 2 * rho;  // footprint columns
  const int R = ny + 2 * rho;  // footprint rows
  const int tid = threadIdx.x;
  const float* src = img + plane;

  const bool interior_tile = x0 - rho >= 0 && x0 + nx + rho <= W && y0 - rho >= 0 && y0 + ny + rho <= H;
  if (kStage && use_tma && interior_tile) {
    // one TMA box load; the box starts at a 16-byte aligned column (a TMA
    // requirement), the footprint then sits delta columns into each row
    const int xs = (x0 - rho) & ~3, delta = (x0 - rho) - xs;
    if (tid == 0) {
      mbar_init(&tbar, 1);
      tma_load_box(F, &tmap, xs, y0 - rho, bimg, &tbar, sizeof(float) * FP * G::FR);
    }
    __syncthreads();  // mbarrier initialised before anyone polls it
    mbar_wait(&tbar, 0);
    F += delta;
  } else if (kStage) {  // coalesced staging of the footprint, many loads in flight
    // cp.async (LDGSTS): every element in flight at once, no register round trip
    constexpr int kCU = (kBT + 2 * RC + 31) / 32;  // 32-column chunks per row, max
    const int lane = tid & 31;
    const bool interior = x0 - rho >= 0 && x0 + nx + rho <= W && y0 - rho >= 0 && y0 + ny + rho <= H;
    int xs[kCU];
#pragma unroll
    for (int k = 0; k < kCU; ++k)
      xs[k] = interior ? x0 - rho + lane + 32 * k
                       : reflect_index(min(x0 - rho + lane + 32 * k, W - 1 + rho), W);
    const unsigned fbase = (unsigned)__cvta_generic_to_shared(F);
    for (int r = tid / 32; r < R; r += kThreads / 32) {
      const int yr = interior ? y0 - rho + r : reflect_index(y0 - rho + r, H);
      const float* rowp = src + (size_t)yr * W;
#pragma unroll
      for (int k = 0; k < kCU; ++k)
        if (lane + 32 * k < C) {
          const unsigned dst = fbase + 4u * (unsigned)(r * FP + lane + 32 * k);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(rowp + xs[k]) : "memory");
        }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
  }
  // pass V
  const int segV = (ny + kBSegV - 1) / kBSegV;
  for (int t = tid; t < C * segV; t += kThreads) {
    const int c = t % C, s = t / C;
    const int o0 = s * kBSegV, len = min(kBSegV, ny - o0);
    if (kStage) {
      if (len == kBSegV && w >= kBSegV)
        vhgw_seg<kBSegV, float, FP, VP>(F + o0 * FP + c, Vm + o0 * VP + c, w);
      else
        vhgw_run<float, FP, VP>(F + o0 * FP + c, Vm + o0 * VP + c, len, w);
    } else {
      const float* col = src + reflect_index(x0 - rho + c, W);
      const int yb = y0 - rho + o0;
      vhgw_walk(
          len, w,
          [&](int i) {
            const float v = __ldg(col + (size_t)reflect_index(yb + i, H) * W);
            return make_float2(v, v);
          },
          [&](int o) { return Vm + (size_t)(o0 + o) * VP + c; });
    }
  }
  __syncthreads();
  // pass H (O aliases F, which is dead now)
  const int segH = (nx + kBSegH - 1) / kBSegH;
  for (int t = tid; t < ny * segH; t += kThreads) {
    const int r = t % ny, s = t / ny;
    const int o0 = s * kBSegH, len = min(kBSegH, nx - o0);
    if (len == kBSegH && w >= kBSegH)
      vhgw_seg<kBSegH, float2, 1, 1>(Vm + r * VP + o0, O + r * OP + o0, w);
    else
      vhgw_run<float2, 1, 1>(Vm + r * VP + o0, O + r * OP + o0, len, w);
  }
  __syncthreads();
  // copy out (coalesced) + the tile's (min alpha, max beta)
  float2 bm = make_float2(CUDART_INF_F, -CUDART_INF_F);
  for (int t = tid; t < ny * kBT; t += kThreads) {
    const int r = t / kBT, x = t % kBT;
    if (x < nx) {
      const float2 v = O[r * OP + x];
      const size_t o = plane + (size_t)(y0 + r) * W + x0 + x;
      amin[o] = v.x;
      bmax[o] = v.y;
      bm = mm2(bm, v);
    }
  }
  if (blkmm) {
    for (int off = 16; off > 0; off >>= 1)
      bm = mm2(bm, make_float2(__shfl_xor_sync(0xffffffffu, bm.x, off),
                               __shfl_xor_sync(0xffffffffu, bm.y, off)));
    if ((tid & 31) == 0) red[tid >> 5] = bm;
    __syncthreads();
    if (tid == 0) {
      for (int i = 1; i < kThreads / 32; ++i) bm = mm2(bm, red[i]);
      blkmm[((size_t)bimg * ((H + kBT - 1) / kBT) + ty) * gridDim.x + blockIdx.x] = bm;
    }
  }
}

// ============================================================================
// step a1, separable in two streaming passes (default): eq.(8) as a row pass
// and a column pass of the van Herk / Gil-Werman MAX-FILTER (Prop.1,
// P:266-270; min and max are separable over the box, reflection is per axis):
//   k_bounds_h: Hmm(y, x) = (min, max) of f(y, x - rho .. x + rho)  (float2 plane)
//   k_bounds_v: alpha, beta(y, x) = (min, max) of Hmm(y - rho .. y + rho, x),
//               plus the (min alpha, max beta) of each kBT x kBT tile.
// Every output segment of SEG <= w positions is one van Herk block boundary
// (vhgw_regs: suffix in registers, compile-time indices), so each pass reads
// (SEG + w - 1) / SEG inputs and makes 3 comparisons per output whatever rho
// is; the whole pass streams: 4 + 8 B/px (h) and 8 + 8 B/px (v) of DRAM, the
// intermediate plane mostly L2-resident between the two.  Windows narrower
// than 8 (rho < 4) take direct minima (at most 7 inputs per output).
template <int SEG, class LoadF>
__device__ __forceinline__ void vhgw_regs(LoadF in, int w, float2 (&res)[SEG]) {
  float2 run = make_float2(CUDART_INF_F, -CUDART_INF_F);
  int i = w - 1;
  for (; i - 3 >= SEG; i -= 4) {  // inputs above the outputs: accumulate only
    const float2 v0 = in(i), v1 = in(i - 1), v2 = in(i - 2), v3 = in(i - 3);
    run = mm2(mm2(run, v0), mm2(mm2(v1, v2), v3));
  }
  for (; i >= SEG; --i) run = mm2(run, in(i));
#pragma unroll
  for (int j = SEG - 1; j >= 0; --j) {
    run = mm2(run, in(j));
    res[j] = run;  // suffix of block 0 from j
  }
  float2 g = make_float2(CUDART_INF_F, -CUDART_INF_F);
#pragma unroll
  for (int o = 1; o < SEG; ++o) {  // prefix of block 1 up to o + w - 1
    g = mm2(g, in(o + w - 1));
    res[o] = mm2(res[o], g);
  }
}
template <int SEG, class LoadF>
__device__ __forceinline__ void direct_regs(LoadF in, int w, float2 (&res)[SEG]) {
#pragma unroll
  for (int o = 0; o < SEG; ++o) {
    float2 m = in(o);
    for (int d = 1; d < w; ++d) m = mm2(m, in(o + d));
    res[o] = m;
  }
}

constexpr int kHR = 32;   // k_bounds_h: rows per CTA
constexpr int kHW = 256;  // k_bounds_h: output columns per CTA
__host__ __device__ inline int hpass_pitch(int rho) { return (kHW + 2 * rho) | 1; }
__host__ inline size_t hpass_smem(int rho) {
  const size_t f = sizeof(float) * (size_t)kHR * hpass_pitch(rho);
  const size_t o = sizeof(float2) * (size_t)kHR * (kHW + 1);
  return f > o ? f : o;
}

// rows [ry0, ry1) of images [b0, b0 + gridDim.z); threads: lane = row of the
// CTA's 32 (odd pitch: conflict-free), warp = segment group
template <int SEG, bool DIRECT>
__global__ void __launch_bounds__(kThreads) k_bounds_h(const float* __restrict__ img, int H, int W, int rho,
                                                      float2* __restrict__ hmm, int b0, int ry0, int ry1) {
  extern __shared__ __align__(16) unsigned char smh[];
  float* F = reinterpret_cast<float*>(smh);    // [kHR][FP] footprint rows
  float2* O = reinterpret_cast<float2*>(smh);  // [kHR][kHW + 1] results (after the walk)
  constexpr int NSEG = kHW / SEG, WPT = kHR * NSEG / kThreads;  // walkers per thread
  const int w = 2 * rho + 1, FP = hpass_pitch(rho);
  const int x0 = blockIdx.x * kHW, y0 = ry0 + blockIdx.y * kHR, bimg = b0 + blockIdx.z;
  const int nx = min(kHW, W - x0), ny = min(kHR, ry1 - y0), C = nx + 2 * rho;
  const size_t plane = (size_t)bimg * H * W;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_trigger();
  // stage the footprint rows (coalesced, reflected at the left / right edges):
  // cp.async, every element in flight at once, no register round trip
  const bool inner = x0 - rho >= 0 && x0 + nx + rho <= W;
  const unsigned fbase = (unsigned)__cvta_generic_to_shared(F);
  for (int r = warp; r < ny; r += kThreads / 32) {
    const float* row = img + plane + (size_t)(y0 + r) * W;
    for (int c = lane; c < C; c += 32) {
      const float* src = row + (inner ? x0 - rho + c : reflect_index(x0 - rho + c, W));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(fbase + 4u * (unsigned)(r * FP + c)),
                   "l"(src)
                   : "memory");
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  float2 res[WPT][SEG];
#pragma unroll
  for (int k = 0; k < WPT; ++k) {
    const int s = warp + k * (kThreads / 32);  // segment of row `lane`
    const float* in = F + lane * FP + s * SEG;
    auto ld = [&](int i) { const float v = in[i]; return make_float2(v, v); };
    if (DIRECT)
      direct_regs<SEG>(ld, w, res[k]);
    else
      vhgw_regs<SEG>(ld, w, res[k]);
  }
  __syncthreads();  // the footprint is dead: O aliases it
#pragma unroll
  for (int k = 0; k < WPT; ++k) {
    const int s = warp + k * (kThreads / 32);
#pragma unroll
    for (int o = 0; o < SEG; ++o) O[lane * (kHW + 1) + s * SEG + o] = res[k][o];
  }
  __syncthreads();
  for (int t = tid; t < ny * kHW; t += kThreads) {
    const int r = t / kHW, x = t - r * kHW;
    if (x < nx) hmm[plane + (size_t)(y0 + r) * W + x0 + x] = O[r * (kHW + 1) + x];
  }
}

// one CTA per kBT x kBT tile (tile row ty0 + blockIdx.y), kBT * kBT / SEG
// threads: column tid % kBT (coalesced), segment tid / kBT
template <int SEG, bool DIRECT>
__global__ void __launch_bounds__(kBT * kBT / SEG) k_bounds_v(const float2* __restrict__ hmm, int H, int W, int rho,
                                                             float* __restrict__ amin, float* __restrict__ bmax,
                                                             float2* __restrict__ blkmm, int b0, int ty0) {
  constexpr int NT = kBT * kBT / SEG;
  __shared__ float2 red[NT / 32];
  const int w = 2 * rho + 1;
  const int ty = ty0 + blockIdx.y, bimg = b0 + blockIdx.z;
  const int x0 = blockIdx.x * kBT, y0 = ty * kBT;
  const int tid = threadIdx.x, c = tid % kBT, s = tid / kBT;
  const int x = x0 + c, ys = y0 + s * SEG;  // first output row of this thread
  const size_t plane = (size_t)bimg * H * W;
  pdl_trigger();
  pdl_wait();  // k_bounds_h's plane
  float2 bm = make_float2(CUDART_INF_F, -CUDART_INF_F);
  if (x < W && ys < H) {
    const float2* col = hmm + plane + x;
    float2 res[SEG];
    if (ys - rho >= 0 && ys + SEG - 1 + rho <= H - 1) {  // no reflection: fixed row stride
      const float2* base = col + (size_t)(ys - rho) * W;
      auto ld = [&](int i) { return base[(size_t)i * W]; };
      if (DIRECT) direct_regs<SEG>(ld, w, res); else vhgw_regs<SEG>(ld, w, res);
    } else {
      auto ld = [&](int i) { return col[(size_t)reflect_index(min(ys - rho + i, H - 1 + rho), H) * W]; };
      if (DIRECT) direct_regs<SEG>(ld, w, res); else vhgw_regs<SEG>(ld, w, res);
    }
#pragma unroll
    for (int o = 0; o < SEG; ++o) {
      if (ys + o < H) {
        const size_t off = plane + (size_t)(ys + o) * W + x;
        amin[off] = res[o].x;
        bmax[off] = res[o].y;
        bm = mm2(bm, res[o]);
      }
    }
  }
  if (blkmm) {
    for (int off = 16; off > 0; off >>= 1)
      bm = mm2(bm, make_float2(__shfl_xor_sync(0xffffffffu, bm.x, off), __shfl_xor_sync(0xffffffffu, bm.y, off)));
    if ((tid & 31) == 0) red[tid >> 5] = bm;
    __syncthreads();
    if (tid == 0) {
      for (int i = 1; i < NT / 32; ++i) bm = mm2(bm, red[i]);
      blkmm[((size_t)bimg * ((H + kBT - 1) / kBT) + ty) * gridDim.x + blockIdx.x] = bm;
    }
  }
}

// ============================================================================
// step a1, default for 8 <= rho <= 24 on large images: one CTA per 64-column x
// 128-row output tile (two kBT x kBT bounds tiles).  The (128 + 2 rho) x
// (64 + 2 rho) footprint of f is staged with a 512-byte row pitch (cp.async,
// 16-byte copies for interior tiles); the row pass (van Herk / Gil-Werman,
// vhgw_regs: suffix in registers) turns each footprint row into its 64
// horizontal (min, max) pairs IN PLACE (a row of 64 float2 is 512 bytes), and
// the column pass walks those rows down each column and writes alpha, beta
// straight to global memory (lane = column: coalesced) with the two tiles'
// (min alpha, max beta).  Against the 64 x 64 tile kernel: the vertical halo
// is shared by two tiles (footprint rows 1.31x instead of 1.63x the outputs),
// the horizontal halo costs loads only, and no output staging.
constexpr int kB2C = 64, kB2R = 128;  // output columns / rows per CTA
constexpr int kB2P = 130;             // footprint row pitch (floats): one row of 65 float2, 2-way conflicts at most
__host__ inline size_t bounds2_smem(int rho) { return sizeof(float) * (size_t)kB2P * (kB2R + 2 * rho); }

template <int SEGH, int SEGV>
__global__ void __launch_bounds__(kThreads) k_bounds2(const float* __restrict__ img, int H, int W, int rho,
                                                     float* __restrict__ amin, float* __restrict__ bmax,
                                                     float2* __restrict__ blkmm, int b0, int ty0, int ty1) {
  extern __shared__ __align__(16) unsigned char smb2[];
  __shared__ float2 red[2 * kThreads / 32];
  float* F = reinterpret_cast<float*>(smb2);    // [FR][kB2P] footprint rows
  float2* Hm = reinterpret_cast<float2*>(smb2);  // [FR][kB2P / 2] row-pass results, in place
  const int w = 2 * rho + 1;
  const int x0 = blockIdx.x * kB2C, y0 = (ty0 + 2 * blockIdx.y) * kBT, bimg = b0 + blockIdx.z;
  const int yend = min(H, ty1 * kBT);  // rows this launch writes
  const int ny = min(kB2R, yend - y0), FR = ny + 2 * rho, C = kB2C + 2 * rho;
  const size_t plane = (size_t)bimg * H * W;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_trigger();
  // ---- stage the footprint (rows y0 - rho .., columns x0 - rho ..), reflected at the borders
  const unsigned fbase = (unsigned)__cvta_generic_to_shared(F);
  const bool inner = x0 - rho >= 0 && x0 + kB2C + rho <= W && y0 - rho >= 0 && y0 + ny + rho <= H;
  int delta = 0;
  const int xs = (x0 - rho) & ~1, nq = (C + (x0 - rho - xs) + 1) >> 1;  // float2 per row (<= kB2P / 2)
  if (inner && (W & 1) == 0 && xs + 2 * nq <= W) {  // 8-byte copies from the even column below x0 - rho
    delta = (x0 - rho) - xs;
    const float* src = img + plane + (size_t)(y0 - rho + warp) * W + xs + 2 * lane;
    unsigned dst = fbase + 4u * (unsigned)(warp * kB2P + 2 * lane);
    for (int r = warp; r < FR; r += kThreads / 32, src += (kThreads / 32) * (size_t)W, dst += 4u * (kThreads / 32) * kB2P) {
#pragma unroll
      for (int q = 0; q < kB2P / 2; q += 32)
        if (q + lane < nq)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + 8u * q), "l"(src + 2 * q) : "memory");
    }
  } else {
    for (int r = warp; r < FR; r += kThreads / 32) {
      const float* row = img + plane + (size_t)reflect_index(min(y0 - rho + r, H - 1 + rho), H) * W;
      for (int c = lane; c < C; c += 32)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(fbase + 4u * (unsigned)(r * kB2P + c)),
                     "l"(row + reflect_index(min(x0 - rho + c, W - 1 + rho), W))
                     : "memory");
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  // ---- row pass, in place, in rounds of kThreads walkers (a round's rows are
  // read completely before any of them is overwritten)
  constexpr int NSH = kB2C / SEGH;  // segments per row
  constexpr int RPR = kThreads / NSH;  // rows per round
  for (int rr = 0; rr < FR; rr += RPR) {
    // lane = row (32 consecutive rows per warp, one segment): banks 2 r + c
    const int s = (tid >> 5) % NSH, r = rr + lane + 32 * ((tid >> 5) / NSH);
    float2 res[SEGH];
    const bool act = r < FR;
    if (act) {
      const float* in = F + r * kB2P + delta + s * SEGH;
      vhgw_regs<SEGH>([&](int i) { const float v = in[i]; return make_float2(v, v); }, w, res);
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int o = 0; o < SEGH; ++o) Hm[r * (kB2P / 2) + s * SEGH + o] = res[o];
    }
    __syncthreads();
  }
  // ---- column pass: lane = column, warp = segment of SEGV output rows
  constexpr int NSV = kB2R / SEGV;  // segments per column
  float2 bm[2] = {make_float2(CUDART_INF_F, -CUDART_INF_F), make_float2(CUDART_INF_F, -CUDART_INF_F)};
  for (int t = tid; t < kB2C * NSV; t += kThreads) {
    const int c = t % kB2C, s = t / kB2C;
    const int x = x0 + c, ys = s * SEGV;  // first output row (tile-relative)
    if (ys < ny) {
      float2 res[SEGV];
      const float2* in = Hm + ys * (kB2P / 2) + c;
      vhgw_regs<SEGV>([&](int i) { return in[i * (kB2P / 2)]; }, w, res);
      if (x < W) {
        float2 m = make_float2(CUDART_INF_F, -CUDART_INF_F);
        // one base per plane, 32-bit row offsets (a tile's rows span < 2^31 elements)
        float* __restrict__ pa = amin + plane + (size_t)(y0 + ys) * W + x;
        float* __restrict__ pb = bmax + plane + (size_t)(y0 + ys) * W + x;
#pragma unroll
        for (int o = 0; o < SEGV; ++o) {
          if (ys + o < ny) {
            pa[o * W] = res[o].x;
            pb[o * W] = res[o].y;
            m = mm2(m, res[o]);
          }
        }
        if (ys < kBT) bm[0] = mm2(bm[0], m); else bm[1] = mm2(bm[1], m);  // SEGV divides kBT
      }
    }
  }
  if (blkmm) {  // the two kBT x kBT tiles' (min alpha, max beta)
#pragma unroll
    for (int h = 0; h < 2; ++h)
      for (int off = 16; off > 0; off >>= 1)
        bm[h] = mm2(bm[h], make_float2(__shfl_xor_sync(0xffffffffu, bm[h].x, off),
                                       __shfl_xor_sync(0xffffffffu, bm[h].y, off)));
    __syncthreads();  // (Hm reads done before red is written: red is separate anyway)
    if (lane == 0) red[warp] = bm[0], red[kThreads / 32 + warp] = bm[1];
    __syncthreads();
    if (tid < 2) {
      float2 m = make_float2(CUDART_INF_F, -CUDART_INF_F);
      for (int wi = 0; wi < kThreads / 32; ++wi) m = mm2(m, red[tid * (kThreads / 32) + wi]);
      const int ty = ty0 + 2 * blockIdx.y + tid;
      if (ty < ty1 && ty * kBT < H)
        blkmm[((size_t)bimg * ((H + kBT - 1) / kBT) + ty) * ((W + kBT - 1) / kBT) + blockIdx.x] = m;
    }
  }
}

// ============================================================================
// steps a1-a8 in one pass (north_star (e)).  Persistent grid,
// 256 threads; a CTA walks down vertical segments of strips of TW output
// columns, RB = QS/TW output rows per step.  Per step:
//   A  column owners (thread c < L = TW + 2 rho owns input column c):
//      moments (a3): add the entering row's powers to / remove the leaving
//        row's powers from the fp64 vertical sums V_q (shared memory, odd
//        stride) and write them to the prefix rows Ps;
//      bounds (a1), vertical van Herk / Gil-Werman streamed down the column:
//        the segment's input rows are cut into blocks of w = 2 rho + 1 rows;
//        a running prefix min/max of the current block, and the suffix
//        min/max of the previous block from a per-CTA ring in global memory
//        (L2-resident) that a look-ahead sweep fills one block in advance
//        (one extra load per row, 2w rows ahead at most); the window's
//        vertical (min, max) = op(suffix_{b-1}, prefix_b) goes to VX;
//   B  a 16-lane group per (row, q) turns the row into an exclusive prefix
//      P[0] = 0, P[1 + c] = sum_{c' <= c} V(c') in place (lane l owns E
//      odd consecutive entries), 4 shuffle rounds; and, per (row, block of w
//      columns), one thread runs the horizontal van Herk / Gil-Werman sweeps
//      over VX: backward suffix, forward prefix of the next block -> alpha,
//      beta of every output pixel in VY (3 comparisons per sample, any rho);
//   C1 one pixel per thread-iteration: S_q = P[x + w] - P[x], identity test,
//      stretch to the fit's Legendre coefficients (fp64), regime; the record
//      goes to a shared-memory queue, regime-A from the front, B/C from the back;
//   C2 thread j finishes queue record j (integrals, ratio, guard, store).
constexpr int kSL = 16;  // lanes per prefix scan


// FABF_EXP_TIMERS (experiments only): thread 0 of every CTA accumulates clock64
// deltas per phase; fabf_exp_timers() reads them back
#ifdef FABF_EXP_TIMERS
__device__ unsigned long long g_exp_timers[8];
#define EXP_T(slot)                                  \
  do {                                               \
    if (tid == 0) {                                  \
      const long long now_ = clock64();              \
      t_acc[slot] += (unsigned long long)(now_ - t_last); \
      t_last = now_;                                 \
    }                                                \
  } while (0)
#else
#define EXP_T(slot) \
  do {              \
  } while (0)
#endif

struct FilterArgs {
  const float* img;
  const float* theta;
  const float* sigma;
  const float* alpha;   // !FB: the bounds planes k_bounds wrote
  const float* beta;
  const float2* blkmm;  // !FB: per kBT x kBT bounds tile (min alpha, max beta)
  float* out;
  float* alpha_w;  // alpha / beta of fallback pixels (read by k_fallback)
  float* beta_w;
  int fused;        // 1: bounds inside k_filter (FB), 0: from k_bounds' planes
  float2* ring;     // per-CTA vertical suffix rings [grid][2][w][L]
  long long ring_cta;  // float2 elements per CTA
  long long ring_ctas;  // CTAs the plan's ring buffer holds (grid cap)
  int B, H, W, rho;
  int SH;          // segment cap (rows)
  int b0, r0, r1;  // images [b0, b0 + B), rows [r0, r1) of each (row bands)
  unsigned flags;
  double flag_root;         // 2^(flag_bits / N) with the prefix-row magnitude
  double flag_root_direct;  // 2^(flag_bits / N): direct sums (k_fallback_seg)
  int* fb_count;
  int* fb_list;
  // exact-moment fallback by 32-pixel row segments (k_fallback_seg): one bit
  // per flagged pixel, the segments that hold any, and their count
  unsigned* fb_bits;
  int* seg_list;
  int* seg_count;
  int WS;  // 32-pixel words per image row
  float* d_alpha;  // diagnostics (fabf_filter_diag), may be NULL
  float* d_beta;
  float* d_kappa;
  float* d_t2n;
  unsigned char* d_code;
};

template <int N, int E>
struct FilterGeom {
  static constexpr int NN = N > 0 ? N : 1;
  static constexpr int PSQ = kSL * E + 2;  // one (row, q) prefix row: P[0..16E], even length
  static constexpr int VST = NN | 1;       // odd per-column stride of the V state
};

template <int N, int E>
struct FilterSmem {
  // byte offsets into dynamic shared memory
  size_t ps, vs, qnu, qo, q4, vx, vy, vz, total;
  // bounds rows: VX (pitch L; the prefix sweeps read up to 2 rho samples past
  // a row's end -- into the next row or VY -- which only reach outputs
  // x >= TW), VY / VZ (pitch TW)
  __host__ __device__ static int xpitch(int L, int TW, int w) { return L; }
  __host__ __device__ static int ypitch(int TW, int w) { return TW; }
  __host__ __device__ FilterSmem(int L, int RB, int QS, int TW, bool FB) {
    const int w = L - TW + 1, XP = FB ? xpitch(L, TW, w) : 0, YP = FB ? ypitch(TW, w) : 0;
    using G = FilterGeom<N, E>;
    size_t off = 0;
    // the arrays whose size is a compile-time constant come first: their
    // addresses are immediates in the kernel (no per-use pointer arithmetic
    // from the run-time strip width L)
    ps = off;
    off += sizeof(double) * (size_t)RB * G::NN * G::PSQ;
    // the pixel queue: C2 of step s reads it before the barrier after A of
    // step s+1 and C1 of step s+1 writes it after the next one: single
    // buffer; nup_1..nup_N (nup_0 = n is not stored)
    qnu = off;
    off += sizeof(double) * (size_t)G::NN * QS;
    qo = off;  // in-step pixel index of each record
    off += sizeof(int) * QS;
    off = (off + 15) & ~(size_t)15;
    q4 = off;  // !FB: (theta, sigma, alpha, beta) of each record, one 16-byte access
    off += FB ? 0 : sizeof(float4) * QS;
    off = (off + 7) & ~(size_t)7;
    vs = off;
    off += sizeof(double) * (size_t)G::VST * L;
    off = (off + 7) & ~(size_t)7;
    vx = off;  // vertical (min, max) of each input column, per step row
    off += sizeof(float2) * (size_t)RB * XP;
    vy = off;  // (alpha, beta) of each output pixel: suffix within its block
    off += sizeof(float2) * (size_t)RB * YP;
    vz = off;  // ... and prefix within the next block
    off += sizeof(float2) * (size_t)RB * YP;
    total = off;
  }
};

template <int N, int E, int TW, int PPT, int WD, bool FB>
__global__ void __launch_bounds__(kThreads, FABF_FILTER_MINB) k_filter(FilterArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ int cnt[2];  // per step parity: regime-A count (low 16 bits), B/C count (high 16)
  __shared__ float red_min[kThreads / 32], red_max[kThreads / 32];
  __shared__ double s_etab[64];  // 2^(j/64) for exp_nonpos_tab (C2)
  using G = FilterGeom<N, E>;
  constexpr int NN = G::NN, PSQ = G::PSQ, VST = G::VST;
  constexpr int QS = PPT * kThreads;  // pixels (queue records) per step
  constexpr int RB = QS / TW;         // output rows per step
  const int rho = a.rho, w = 2 * rho + 1;
  const int H = a.H, W = a.W;
  const int L = TW + 2 * rho;  // input columns of a strip, <= 16 * E (host picks E)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const FilterSmem<N, E> lay(L, RB, QS, TW, FB);
  double* Ps = reinterpret_cast<double*>(smraw + lay.ps);    // [RB][NN][PSQ]
  double* Vs = reinterpret_cast<double*>(smraw + lay.vs);    // [L][VST]
  double* qnu = reinterpret_cast<double*>(smraw + lay.qnu);  // [N][QS]
  int* qo = reinterpret_cast<int*>(smraw + lay.qo);
  float4* q4 = reinterpret_cast<float4*>(smraw + lay.q4);
  const int XP = FilterSmem<N, E>::xpitch(L, TW, w), YP = FilterSmem<N, E>::ypitch(TW, w);
  float2* VX = reinterpret_cast<float2*>(smraw + lay.vx);    // [RB][XP]
  float2* VY = reinterpret_cast<float2*>(smraw + lay.vy);    // [RB][YP]
  float2* VZ = reinterpret_cast<float2*>(smraw + lay.vz);    // [RB][YP]
  const float n = (float)(w * w);
  const bool want_t2n = a.d_t2n != nullptr, want_kappa = a.d_kappa != nullptr;
  const bool want_diag = want_t2n || want_kappa || a.d_code != nullptr || a.d_alpha != nullptr;  // fabf_filter_diag
  const float2 kEmpty = make_float2(CUDART_INF_F, -CUDART_INF_F);

  for (int i = tid; i < RB * NN * PSQ; i += kThreads) Ps[i] = 0.0;  // P[0] = 0 for good
  if (tid < 64) s_etab[tid] = c_exp2_64[tid];  // read after the first centring barrier
  pdl_trigger();
  pdl_wait();  // k_bounds' planes and tile ranges (PDL launch)
#ifdef FABF_EXP_TIMERS
  unsigned long long t_acc[8] = {};
  long long t_last = clock64();
#endif

  // column-owner identity (thread c owns input column c of the strip)
  const int c = tid;
  const bool owner = c < L;
  double* vsc = Vs + (owner ? c : 0) * VST;
  double* psc = Ps + 1 + c;
  // this CTA's vertical suffix rings: ring[(buf * w + i) * L + c], buf = block
  // parity, i = suffix position (int offsets: a ring is < 2^31 elements)
  float2* ringc = a.ring + (long long)blockIdx.x * a.ring_cta + (owner ? c : 0);
  // pixel identity within a step: pixels tid + i * kThreads, i < PPT
  const int px_r = tid / TW, px_x = tid % TW;  // (row px_r + i * kThreads / TW)
  // phase-B identity
  const int sgrp = tid / kSL, sl = tid % kSL;
  const int nbk = (TW + w - 1) / w;  // horizontal bounds blocks per output row

  // balanced static schedule: the B * nstrips * H strip-rows are split into
  // gridDim.x contiguous chunks (one per resident CTA); a chunk is one or two
  // vertical segments of a strip, each walked top to bottom.
  const int nstrips = (W + TW - 1) / TW;
  const int HR = a.r1 - a.r0;  // rows of the band
  const long long U = (long long)a.B * nstrips * HR;
  const long long u0 = (long long)blockIdx.x * U / gridDim.x;
  const long long u1 = (long long)(blockIdx.x + 1) * U / gridDim.x;
  int step = 0;
  for (long long u = u0; u < u1;) {
    const long long seg = u / HR;
    const int Y0 = a.r0 + (int)(u - seg * HR);
    // a segment is at most a.SH rows: its centring region (and the error of
    // its running sums) stays local ("Numerical envelope")
    const int Y1 = (int)min(min((long long)a.r1, (long long)Y0 + (u1 - u)), (long long)Y0 + a.SH);
    u += Y1 - Y0;
    const int bl = (int)(seg / nstrips), strip = (int)(seg - (long long)bl * nstrips);
    const int bimg = a.b0 + bl;
    const int x0 = strip * TW;
    const size_t plane = (size_t)bimg * H * W;
    const float* colp = a.img + plane + reflect_index(min(x0 - rho + c, W - 1 + rho), W);

    // ---- tile-local centre c_T and power-of-two scale s_T: the range of the
    // ---- segment's input footprint (rows Y0-rho .. Y1+rho-1, the strip's
    // ---- L columns) -- every sample the running sums will ever see
    // ---- (FB: a pass over the footprint; else the bounds tiles of k_bounds,
    // ---- whose windows cover the footprint)
    float lmin = CUDART_INF_F, lmax = -CUDART_INF_F;
    if constexpr (FB) {
      if (owner) {
        if (Y0 - rho >= 0 && Y1 + rho <= H) {  // (uniform) no reflection
          const float* cp = colp + (Y0 - rho) * W;
#pragma unroll 16
          for (int y = 0; y < Y1 - Y0 + 2 * rho; ++y) {
            const float v = __ldg(cp + y * W);
            lmin = fminf(lmin, v);
            lmax = fmaxf(lmax, v);
          }
        } else {
#pragma unroll 8
          for (int y = Y0 - rho; y < Y1 + rho; ++y) {
            const float v = __ldg(colp + reflect_index(y, H) * W);
            lmin = fminf(lmin, v);
            lmax = fmaxf(lmax, v);
          }
        }
      }
    } else {
      const int nby = (H + kBT - 1) / kBT, nbx = (W + kBT - 1) / kBT;
      const int by0 = Y0 / kBT, by1 = (Y1 - 1) / kBT;
      const int bx0 = x0 / kBT, bx1 = min(W - 1, x0 + TW - 1) / kBT;
      const int nbw = bx1 - bx0 + 1, nblk = (by1 - by0 + 1) * nbw;
      for (int i = tid; i < nblk; i += kThreads) {
        const int by = by0 + i / nbw, bx = bx0 + i % nbw;
        const float2 mm = a.blkmm[((size_t)bimg * nby + by) * nbx + bx];
        lmin = fminf(lmin, mm.x);
        lmax = fmaxf(lmax, mm.y);
      }
    }
    {
      for (int off = 16; off > 0; off >>= 1) {
        lmin = fminf(lmin, __shfl_xor_sync(0xffffffffu, lmin, off));
        lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, off));
      }
      __syncthreads();  // previous segment's readers of red_* are done
      if (lane == 0) {
        red_min[warp] = lmin;
        red_max[warp] = lmax;
      }
      __syncthreads();
      lmin = red_min[0];
      lmax = red_max[0];
#pragma unroll
      for (int i = 1; i < kThreads / 32; ++i) {
        lmin = fminf(lmin, red_min[i]);
        lmax = fmaxf(lmax, red_max[i]);
      }
    }
    EXP_T(0);
    const double cT = 0.5 * ((double)lmin + (double)lmax);
    const double halfr = 0.5 * ((double)lmax - (double)lmin);
    int e2 = 0;
    if (halfr > 0.0) frexp(halfr, &e2);
    const double invS = ldexp(1.0, -e2);  // 1/s_T, s_T = 2^e2 >= half range: exact scaling
    const double mcs = -cT * invS;         // u = f * invS + mcs, exact

    // ---- vertical bounds (van Herk / Gil-Werman streamed down each column).
    // Segment-local entering row k = y - (Y0 - rho), block b = k / w, position
    // j = k - b w.  For the entering row k the look-ahead sweep takes row
    // b w + (w-1-j) of the same block and stores suffix_b(w-1-j) in the ring
    // buffer b & 1; the output window [k-w+1, k] is prefix_b(j) (j = w-1) or
    // op(suffix_{b-1}(j+1), prefix_b(j)), suffix_{b-1}(1) from a register (it
    // is written 2 rows before it is read, possibly in the same step).
    // kb, kj: block / position of the next entering row (uniform).  Phase A
    // writes the vertical (min, max) of the step's rows to VX.
    int kb = 0, kj = 2 * rho;
    const int ysweep0 = Y0 - rho;
    float2 pre = kEmpty, suf = kEmpty, s1 = kEmpty, s1n = kEmpty;  // per column
    const bool pro_inside = Y0 - rho >= 0 && Y0 + rho <= H - 1;      // uniform
    // general (row by row) bounds step: entering samples e[0..nr) of the rows
    // whose window ends there; writes VX row r
    auto bounds_rows_general = [&](const float (&e)[RB], int nr) {
      float fs[RB];
      float2 rgv[RB];
      {
        int b = kb, j = kj;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          fs[r] = 0.f;
          rgv[r] = kEmpty;
          if (r < nr) {
            const int y = min(ysweep0 + b * w + (w - 1 - j), H - 1 + rho);
            fs[r] = __ldg(colp + reflect_index(y, H) * W);
            if (j >= 1 && j + 1 < w) rgv[r] = ringc[(((b - 1) & 1) * w + j + 1) * L];
            if (++j == w) j = 0, ++b;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        if (r >= nr) break;
        const float2 vin = mm_in(e[r]);
        pre = (kj == 0) ? vin : mm2(pre, vin);
        suf = (kj == 0) ? mm_in(fs[r]) : mm2(suf, mm_in(fs[r]));
        const int i = w - 1 - kj;
        if (i >= 2) ringc[((kb & 1) * w + i) * L] = suf;
        float2 v = pre;
        if (kj == 0) v = mm2(s1, pre);
        else if (kj + 1 < w) v = mm2(rgv[r], pre);
        if (i == 1) s1n = suf;
        VX[r * XP + c] = v;
        if (++kj == w) {
          kj = 0;
          ++kb;
          s1 = s1n;
        }
      }
    };
    auto advance_counters = [&](int nr) {  // non-owners: the same uniform kb, kj
      for (int r = 0; r < nr; ++r)
        if (++kj == w) kj = 0, ++kb;
    };

    // prologue: entering rows k = 0 .. 2 rho - 1 (rows Y0-rho .. Y0+rho-1), no
    // outputs yet.  Row Y0-rho-1 lies outside every window of the segment and
    // so possibly far outside its centring range: it is never added, and the
    // first step's leaving sample is u = 0.
    if (owner) {
      double V[NN];
#pragma unroll
      for (int q = 0; q < NN; ++q) V[q] = 0.0;
      constexpr int PB = 8;  // loads issued in batches ahead of the arithmetic
      for (int y0 = Y0 - rho; y0 < Y0 + rho; y0 += PB) {
        float fb[PB];
#pragma unroll
        for (int k = 0; k < PB; ++k) {
          const int yin = min(y0 + k, Y0 + rho - 1);
          fb[k] = __ldg(colp + (pro_inside ? yin : reflect_index(yin, H)) * W);
        }
#pragma unroll
        for (int k = 0; k < PB; ++k) {
          if (y0 + k < Y0 + rho) {
            const double uu = fma((double)fb[k], invS, mcs);
            double pu = uu;
#pragma unroll
            for (int q = 0; q < N; ++q) {
              V[q] += pu;
              pu *= uu;
            }
            if constexpr (FB) pre = mm2(pre, mm_in(fb[k]));  // prefix of block 0
          }
        }
      }
#pragma unroll
      for (int q = 0; q < N; ++q) vsc[q] = V[q];
      // block 0's look-ahead suffix: positions i = w-1 .. 1 (rows Y0-rho+i),
      // ring buffer 0; suffix_0(1) kept for the first output of block 1
      if constexpr (FB)
      for (int i0 = w - 1; i0 >= 1; i0 -= PB) {
        float sb[PB];
#pragma unroll
        for (int k = 0; k < PB; ++k) {
          const int y = Y0 - rho + max(i0 - k, 1);
          sb[k] = __ldg(colp + (pro_inside ? y : reflect_index(y, H)) * W);
        }
#pragma unroll
        for (int k = 0; k < PB; ++k) {
          const int i = i0 - k;
          if (i >= 1) {
            suf = mm2(suf, mm_in(sb[k]));
            if (i >= 2) ringc[i * L] = suf;
          }
        }
      }
      s1n = suf;
    }

    EXP_T(1);
    // phase-A input prefetch: entering / leaving samples of the next step's rows
    float pf_in[RB], pf_out[RB];
    auto prefetch = [&](int Yb) {
      const int y0 = Yb + rho;  // entering row of r = 0
      if (y0 + RB <= H && y0 - w >= 0) {  // (uniform) no reflection: one base, fixed row strides
        const float* pin = colp + y0 * W;
        const float* pout = pin - w * W;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          pf_in[r] = __ldg(pin + r * W);
          pf_out[r] = __ldg(pout + r * W);
        }
        return;
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int yin = min(Yb + r + rho, H - 1 + rho), yout = yin - w;
        pf_in[r] = __ldg(colp + reflect_hi(yin, H) * W);   // yin >= 0
        pf_out[r] = __ldg(colp + reflect_lo(yout) * W);    // yout < H
      }
    };
    if (owner) prefetch(Y0);

    for (int Yb = Y0; Yb < Y1; Yb += RB, ++step) {
      const int nr = min(RB, Y1 - Yb);
      const int qb = step & 1;
      // this thread's pixel parameters (latency hidden behind A and B)
      bool pvalid[PPT];
      int po[PPT];
      float p_th[PPT], p_sg[PPT], p_al[PPT], p_be[PPT];
#pragma unroll
      for (int i = 0; i < PPT; ++i) {
        const int pr = px_r + i * (kThreads / TW);
        const int pY = Yb + pr, pX = x0 + px_x;
        pvalid[i] = (pr < nr) && (pX < W);
        po[i] = (int)plane + pY * W + pX;
        p_th[i] = p_al[i] = p_be[i] = 0.f;
        p_sg[i] = 1.f;
        if (pvalid[i]) {
          p_th[i] = __ldg(a.theta + po[i]);
          p_sg[i] = __ldg(a.sigma + po[i]);
          if constexpr (!FB) {
            p_al[i] = __ldg(a.alpha + po[i]);
            p_be[i] = __ldg(a.beta + po[i]);
          }
        }
      }
      if (tid == 0) {
        cnt[qb] = 0;
      }
      // ---- phase A: moments (entering row Yb+r+rho in, leaving row
      // ---- Yb+r-rho-1 out) and vertical bounds of the step's rows
      // the bounds' fast path: a full step with every row at 1 <= j <= w-3
      // (no block edge, no special case), look-ahead rows inside the image
      const int srow0 = ysweep0 + kb * w + (w - 1 - kj);  // look-ahead row of r = 0
      const bool fast = !FB || (nr == RB && kj >= 1 && kj + RB <= w - 2 && srow0 - (RB - 1) >= 0 &&
                                srow0 <= H - 1);  // uniform
      if (owner) {
        float fin[RB], fout[RB], fsw[RB];
        float2 rg[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          fin[r] = pf_in[r];
          fout[r] = pf_out[r];
        }
        // bounds loads first (ring entries were written at least one step
        // ago; look-ahead samples are L2 hits after the centring pass)
        if (FB && fast) {
          const float* sp = colp + srow0 * W;
          const float2* rp = ringc + (((kb - 1) & 1) * w + kj + 1) * L;
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            fsw[r] = __ldg(sp - r * W);
            rg[r] = rp[r * L];
          }
        }
        prefetch(Yb + RB);
        double V[NN];
#pragma unroll
        for (int q = 0; q < N; ++q) V[q] = vsc[q];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          if (r < nr) {
            const double ui = fma((double)fin[r], invS, mcs);
            // (only the segment's first row has no leaving sample: r = 0 of its first step)
            const double uo = (r == 0 && Yb == Y0) ? 0.0 : fma((double)fout[r], invS, mcs);
            // d_q = ui^q - uo^q by its own recurrence d_{q+1} = (ui + uo) d_q
            // - ui uo d_{q-1} (d_0 = 0): one DMUL + one DFMA per power instead
            // of two DMULs and a DADD
            const double sp = ui + uo, pp = ui * uo;
            double dm = ui - uo, d = sp * dm;  // d_1, d_2
            if (N >= 1) V[0] += dm;
#pragma unroll
            for (int q = 1; q < N; ++q) {
              V[q] += d;
              const double dn = fma(sp, d, -pp * dm);
              dm = d;
              d = dn;
            }
#pragma unroll
            for (int q = 0; q < N; ++q) psc[(r * NN + q) * PSQ] = V[q];
          }
        }
#pragma unroll
        for (int q = 0; q < N; ++q) vsc[q] = V[q];
        // vertical bounds of the step's rows
        if constexpr (!FB) {
        } else if (fast) {
          float2* wp = ringc + ((kb & 1) * w + (w - 1 - kj)) * L;
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            pre = mm2(pre, mm_in(fin[r]));
            suf = mm2(suf, mm_in(fsw[r]));
            wp[-r * L] = suf;
            VX[r * XP + c] = mm2(rg[r], pre);
          }
          kj += RB;
        } else {
          bounds_rows_general(fin, nr);
        }
      } else if constexpr (FB) {
        if (fast) kj += RB;
        else advance_counters(nr);
      }
      __syncthreads();
      EXP_T(2);
      // ---- phase B: exclusive prefix rows, 16 lanes per (r, q) (WD > 0: small
      // ---- windows are summed directly in C1 instead, no prefix magnitudes)
      if (N > 0 && WD == 0) {
        // warp-uniform trip count: both half-warps run the shuffles; a half
        // without a row of its own re-scans its partner's and does not store.
        // Two rows per group and pass (s0, s0 + 16): two independent add chains.
        constexpr int G = kThreads / kSL;  // 16 groups
        if (E > 13) {  // wide rows: one scan per pass (two would spill)
          for (int b = 2 * warp; b < nr * N; b += G) {
            const int s0 = b + (sgrp & 1);
            const bool act0 = s0 < nr * N;
            double* row0 = Ps + (act0 ? s0 : b) * PSQ + 1 + sl * E;
            double v0[E];
#pragma unroll
            for (int e = 0; e < E; ++e) v0[e] = row0[e];
            double t0 = 0.0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
              t0 += v0[e];
              v0[e] = t0;
            }
            double i0 = t0;
#pragma unroll
            for (int off = 1; off < kSL; off <<= 1) {
              const double u0 = __shfl_up_sync(0xffffffffu, i0, off, kSL);
              if (sl >= off) i0 += u0;
            }
            double e0 = __shfl_up_sync(0xffffffffu, i0, 1, kSL);
            if (sl == 0) e0 = 0.0;
            if (act0) {
#pragma unroll
              for (int e = 0; e < E; ++e) row0[e] = v0[e] + e0;
            }
          }
        } else {
        // 1.0 where the shuffle has a source lane (sl >= off), else 0.0: one
        // DFMA per round instead of a DADD under two selects
        double fo[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) fo[k] = (sl >= (1 << k)) ? 1.0 : 0.0;
        for (int b = 2 * warp; b < nr * N; b += 2 * G) {
          const int s0 = b + (sgrp & 1), s1r = s0 + G;
          const bool act0 = s0 < nr * N, act1 = s1r < nr * N;
          double* row0 = Ps + (act0 ? s0 : b) * PSQ + 1 + sl * E;
          double* row1 = Ps + (act1 ? s1r : b) * PSQ + 1 + sl * E;
          double v0[E], v1[E];
#pragma unroll
          for (int e = 0; e < E; ++e) {
            v0[e] = row0[e];
            v1[e] = row1[e];
          }
          double t0 = 0.0, t1 = 0.0;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            t0 += v0[e];
            t1 += v1[e];
            v0[e] = t0;
            v1[e] = t1;
          }
          double i0 = t0, i1 = t1;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double u0 = __shfl_up_sync(0xffffffffu, i0, 1 << k, kSL);
            const double u1v = __shfl_up_sync(0xffffffffu, i1, 1 << k, kSL);
            i0 = fma(u0, fo[k], i0);
            i1 = fma(u1v, fo[k], i1);
          }
          // the offset comes straight from the neighbour (never inc - tot: a
          // lane whose chunk runs into the padding carries garbage in tot)
          double e0 = __shfl_up_sync(0xffffffffu, i0, 1, kSL);
          double e1 = __shfl_up_sync(0xffffffffu, i1, 1, kSL);
          if (sl == 0) e0 = e1 = 0.0;
          if (act0) {
#pragma unroll
            for (int e = 0; e < E; ++e) row0[e] = v0[e] + e0;
          }
          if (act1) {
#pragma unroll
            for (int e = 0; e < E; ++e) row1[e] = v1[e] + e1;
          }
        }
        }
      }
      // horizontal bounds over VX, per (row r, block jb of w
      // output columns): one lane runs the suffix within block jb into VY,
      // another the prefix within block jb + 1 into VZ, so that the outputs x
      // in [jb w, (jb+1) w) get alpha, beta = op(VY[x], VZ[x]) -- 3
      // comparisons per sample whatever rho is.  Fixed trip counts (w, w - 1):
      // no divergence except the prefix's one shorter trip; samples past L
      // only reach outputs x >= TW, whose stores are skipped.  The jobs
      // (2 nr nbk) fill the top warps.
#ifndef FABF_EXP_NOHB
      for (int t = kThreads - 1 - tid; FB && t < 2 * nr * nbk; t += kThreads) {
        const int dir = t & 1, rj = t >> 1, r = rj / nbk, jb = rj - r * nbk;
        const float2* __restrict__ X = VX + r * XP;
        const int xlo = jb * w;
        // suffix: positions xlo + w - 1 down to xlo, outputs at the same index;
        // prefix: positions (jb+1) w .. (jb+1) w + w - 2, outputs at p - w + 1
        const int p0 = dir ? xlo + w : xlo + w - 1, dp = dir ? 1 : -1, os = dir ? 1 - w : 0;
        float2* __restrict__ O = (dir ? VZ : VY) + r * YP;
        if (dir) O[xlo] = kEmpty;  // VZ[jb w]: the window is block jb itself
        const int trips = w - dir;
        float2 acc = kEmpty;
        int p = p0, k = 0;
        for (; k + 4 <= trips; k += 4, p += 4 * dp) {
          float2 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = X[p + u * dp];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            acc = mm2(acc, v[u]);
            const int o = p + u * dp + os;
            if (o < TW) O[o] = acc;
          }
        }
        for (; k < trips; ++k, p += dp) {
          acc = mm2(acc, X[p]);
          if (p + os < TW) O[p + os] = acc;
        }
      }
#else
      for (int t = tid; t < RB * TW; t += kThreads) {  // experiment: vertical-only range
        const int r = t / TW, x = t - r * TW;
        VY[r * YP + x] = VX[r * XP + x + rho];
        VZ[r * YP + x] = kEmpty;
      }
#endif
      __syncthreads();
      EXP_T(3);
      // ---- phase C1: window sums, flag, regime, slot in the queue, stretch
      // ---- written straight into the slot
      // (two passes: regimes of this thread's PPT pixels first, so that one
      // shared atomic per warp and step reserves the slots of all of them)
      int regime[PPT];
      double p_m[PPT], p_h[PPT];  // midrange, half-range in tile units (flag test and stretch)
#pragma unroll
      for (int i = 0; i < PPT; ++i) {
        regime[i] = -1;  // -1: no record (invalid, identity or fallback)
        p_m[i] = 0.0, p_h[i] = 1.0;
        if constexpr (FB) {
          const int pix = (px_r + i * (kThreads / TW)) * YP + px_x;
          const float2 ab = mm2(VY[pix], VZ[pix]);
          p_al[i] = ab.x;
          p_be[i] = ab.y;
        }
        if (pvalid[i]) {
          // (diagnostics: alpha, beta of the pixels that get a record are stored
          // by C2's diagnostic copy; the two rare branches store their own)
          if (p_al[i] == p_be[i]) {  // P:204, Algorithm 1 lines 4-5: g-hat = f(i) = alpha
            a.out[po[i]] = p_al[i];
            if (a.d_alpha) {
              a.d_alpha[po[i]] = p_al[i];
              a.d_beta[po[i]] = p_be[i];
            }
            if (a.d_kappa) a.d_kappa[po[i]] = 1.0f;
            if (a.d_t2n) a.d_t2n[po[i]] = 1.0f;
            if (a.d_code) a.d_code[po[i]] = (unsigned char)kCodeIdentity;
          } else if (const double au = fma((double)p_al[i], invS, mcs), bu = fma((double)p_be[i], invS, mcs);
                     (p_m[i] = 0.5 * (au + bu), p_h[i] = 0.5 * (bu - au),
                      1.0 + fabs(p_m[i]) > a.flag_root * p_h[i])) {  // stretch_flagged: exact-moment fallback pass
            const int pX = x0 + px_x, pY = Yb + px_r + i * (kThreads / TW);
            const int sw = (bimg * H + pY) * a.WS + (pX >> 5);
            if (atomicOr(&a.fb_bits[sw], 1u << (pX & 31)) == 0u) a.seg_list[atomicAdd(a.seg_count, 1)] = sw;
            if (a.d_alpha) {
              a.d_alpha[po[i]] = p_al[i];
              a.d_beta[po[i]] = p_be[i];
            }
            if constexpr (FB) {  // the fallback kernel reads alpha, beta from the plan
              a.alpha_w[po[i]] = p_al[i];
              a.beta_w[po[i]] = p_be[i];
            }
          } else {
            regime[i] = regime_of(p_al[i], p_be[i], p_th[i], p_sg[i]);
          }
        }
      }
      unsigned mA[PPT], mB[PPT];
      int inc = 0;
#pragma unroll
      for (int i = 0; i < PPT; ++i) {
        mA[i] = __ballot_sync(0xffffffffu, regime[i] == kRegA);
        mB[i] = __ballot_sync(0xffffffffu, regime[i] > kRegA);
        inc += __popc(mA[i]) | (__popc(mB[i]) << 16);
      }
      int old = 0;  // one atomic for both counters (QS <= 512 < 2^16) and all PPT pixels
      if (lane == 0 && inc) old = atomicAdd(&cnt[qb], inc);
      old = __shfl_sync(0xffffffffu, old, 0);
      int baseA = old & 0xffff, baseB = old >> 16;
      const unsigned lt = (1u << lane) - 1u;
#pragma unroll
      for (int i = 0; i < PPT; ++i) {
        if (regime[i] >= 0) {
          double S[N + 1];
          S[0] = (double)n;
          const double* prow = Ps + (px_r + i * (kThreads / TW)) * NN * PSQ + px_x;
          if (WD == 0) {
#pragma unroll
            for (int q = 1; q <= N; ++q) S[q] = prow[(q - 1) * PSQ + w] - prow[(q - 1) * PSQ];
          } else {
#pragma unroll
            for (int q = 1; q <= N; ++q) {
              double acc = 0.0;
#pragma unroll
              for (int d = 1; d <= WD; ++d) acc += prow[(q - 1) * PSQ + d];
              S[q] = acc;
            }
          }
          const int j = (regime[i] == kRegA) ? baseA + __popc(mA[i] & lt)
                                             : QS - 1 - (baseB + __popc(mB[i] & lt));
          nu_from_sums_mh<N>(S, p_m[i], p_h[i], qnu + j, QS);
          // FB: in-step pixel index (C2 looks alpha, beta up in VY / VZ); else the output index itself
          qo[j] = FB ? (px_r + i * (kThreads / TW)) * TW + px_x : po[i];
          if constexpr (!FB) q4[j] = make_float4(p_th[i], p_sg[i], p_al[i], p_be[i]);
        }
        baseA += __popc(mA[i]);
        baseB += __popc(mB[i]);
      }
      __syncthreads();
      EXP_T(4);
      // ---- phase C2: integrals, ratio, guard, store (one regime per warp).  No
      // ---- barrier after it (the counters are double buffered; the queue is
      // ---- read before the barrier that ends the next step's phase A).
      // (the diagnostics' per-record work is compiled into a second copy of
      // the loop: the product path tests no diagnostic pointer per record)
      auto c2 = [&](auto diag_tag) {
        constexpr bool D = decltype(diag_tag)::value;
        const int nA = cnt[qb] & 0xffff, nBC = cnt[qb] >> 16;
        const int rowbase = (int)plane + Yb * W + x0;
#ifdef FABF_C2_UNROLL1
#pragma unroll 1
#else
#pragma unroll
#endif
        for (int i = 0; i < PPT; ++i) {
          const int j = tid + i * kThreads;
          if (j < nA || j >= QS - nBC) {
            const double* nu = qnu + j;  // nup_k = nu[(k - 1) * QS]
            // the record's pixel within the step: (alpha, beta) still in VY / VZ
            // (rewritten only in the next step's phase A, after C2 of this one)
            const int pix = qo[j];
            int o = pix;
            float th, sg, al, be;
            if constexpr (FB) {
              const int pr = pix / TW, px = pix - pr * TW;
              o = rowbase + pr * W + px;
              const float2 ab = mm2(VY[pr * YP + px], VZ[pr * YP + px]);
              th = __ldg(a.theta + o), sg = __ldg(a.sigma + o), al = ab.x, be = ab.y;
            } else {
              const float4 rec = q4[j];
              th = rec.x, sg = rec.y, al = rec.z, be = rec.w;
            }
            int regime = kRegA;
            if (j >= nA) regime = regime_of(al, be, th, sg);
            PixelResult res = ghat_from_record<N, true>(nu, QS, th, sg, al, be, regime, a.flags, D && want_t2n, n,
                                                        s_etab, D && want_kappa);
            a.out[o] = res.g;
            if constexpr (D) {
              if (a.d_alpha) {
                a.d_alpha[o] = al;
                a.d_beta[o] = be;
              }
              if (a.d_kappa) a.d_kappa[o] = res.kappa;
              if (a.d_t2n) a.d_t2n[o] = res.t2n;
              if (a.d_code) a.d_code[o] = (unsigned char)res.code;
            }
          }
        }
      };
      if (want_diag)
        c2(std::true_type{});
      else
        c2(std::false_type{});
      EXP_T(5);
    }
  }
#ifdef FABF_EXP_TIMERS
  if (tid == 0) {
    t_acc[6] = 1;
    for (int i = 0; i < 7; ++i) atomicAdd(&g_exp_timers[i], t_acc[i]);
  }
#endif
}

// ============================================================================
// exact-moment fallback helpers: nu_k = sum_j P_k(w_j) directly in fp64 over the
// window of a pixel (w_j stretched by the pixel's own alpha, beta: no centring
// error), then the same per-pixel integrals / ratio as k_filter (used by
// k_fallback_seg for the pixels its segment centring cannot serve, and by the
// Gaussian path's k_fallback_gauss with weights).
// The Legendre values come from the monic recurrence
// R_{k+1} = s R_k - k^2 / (4k^2 - 1) R_{k-1}, R_k = P_k / m_k with
// m_k = binom(2k, k) / 2^k (the three-term recurrence of P_k divided by its
// leading coefficient): one DMUL + one DFMA per degree instead of the
// two DMULs + DFMA of the (2k+1) s Q_k - k^2 Q_{k-1} form; P_k = m_k R_k once
// per pixel at the end.
__constant__ double c_monic_scale[kMaxN + 1] = {1.0, 1.0, 1.5, 2.5, 4.375, 7.875, 14.4375,
                                                26.8125, 50.2734375, 94.9609375, 180.42578125};
template <int N>
__device__ __forceinline__ void fb_accumulate(double (&acc)[N + 1], double sv) {
  double r0 = 1.0, r1 = sv;
  acc[0] += 1.0;
  if (N >= 1) acc[1] += sv;
#pragma unroll
  for (int k = 1; k < N; ++k) {
    const double r2 = fma(-(double)(k * k) / (double)(4 * k * k - 1), r0, sv * r1);
    acc[k + 1] += r2;
    r0 = r1;
    r1 = r2;
  }
}
// ============================================================================
// exact-moment fallback by row segments (O(rho) per pixel instead of the
// O(rho^2) direct window sums of k_fallback).  k_filter marks each flagged
// pixel in a bitmap of 32-pixel row segments and lists the segments.  One warp
// per listed segment (lane = pixel): the segment's own centre and power-of-two
// scale come from the union of its flagged pixels' [alpha, beta] (flagged
// pixels sit in flat areas, so that union is narrow: little amplification),
// the lanes build the fp64 power sums of the segment's 32 + 2 rho columns over
// the window rows, each flagged lane sums its w columns (direct sums, no
// prefix magnitudes), re-checks the amplification against the segment centre,
// and finishes like k_filter; a lane that still fails takes the exact direct
// window sums of k_fallback (its own stretch).  The segment's bits are cleared
// for the next call.
template <int N>
__device__ __forceinline__ PixelResult fallback_direct(const FilterArgs& a, const float* img, int x, int y, float al,
                                                       float be, float th, float sg) {
  const int rho = a.rho, H = a.H, W = a.W;
  const double mid = 0.5 * ((double)al + (double)be), ih = 2.0 / ((double)be - (double)al);
  double acc[N + 1];
#pragma unroll
  for (int k = 0; k <= N; ++k) acc[k] = 0.0;
  for (int dy = -rho; dy <= rho; ++dy) {
    const float* row = img + reflect_index(y + dy, H) * W;
    for (int dx = -rho; dx <= rho; ++dx)
      fb_accumulate<N>(acc, ((double)__ldg(row + reflect_index(x + dx, W)) - mid) * ih);
  }
  double nu[N + 1];
#pragma unroll
  for (int k = 0; k <= N; ++k) nu[k] = (double)(2 * k + 1) * c_monic_scale[k] * acc[k];
  float lam, t0;
  const int regime = range_params(al, be, th, sg, lam, t0);
  const int w = 2 * rho + 1;
  return ghat_from_record<N>(nu + 1, 1, th, sg, al, be, regime, a.flags, a.d_t2n != nullptr, (double)(w * w));
}

constexpr int kSegWarps = 4;  // warps per CTA of k_fallback_seg
constexpr int kSegDirectRho = 5;  // rho <= this: per-lane direct window sums (measured crossover)
template <int N>
__global__ void __launch_bounds__(32 * kSegWarps) k_fallback_seg(FilterArgs a) {
  extern __shared__ __align__(16) unsigned char smf[];
  constexpr int NN = N > 0 ? N : 1;
  const int rho = a.rho, w = 2 * rho + 1, H = a.H, W = a.W, Lc = 32 + 2 * rho;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* Vw = reinterpret_cast<double*>(smf) + (size_t)wib * NN * Lc;  // [NN][Lc] this warp's column sums
  pdl_wait();  // k_filter's segment list (PDL launch)
  const int count = *a.seg_count;
  const int nwarps = gridDim.x * kSegWarps;
  for (int si = blockIdx.x * kSegWarps + wib; si < count; si += nwarps) {
    const int sw = a.seg_list[si];
    const unsigned mask = a.fb_bits[sw];
    __syncwarp();
    if (lane == 0) {
      a.fb_bits[sw] = 0u;  // clean for the next call
      atomicAdd(a.fb_count, __popc(mask));
    }
    const int by = sw / a.WS, x0 = (sw - by * a.WS) * 32, b = by / H, y = by - b * H;
    const float* img = a.img + (size_t)b * H * W;
    const int x = x0 + lane;
    const bool flagged = ((mask >> lane) & 1u) && x < W;
    const size_t o = (size_t)b * H * W + (size_t)y * W + x;
    float al = 0.f, be = 0.f;
    if (flagged) al = a.alpha_w[o], be = a.beta_w[o];
    if (rho <= kSegDirectRho) {  // small windows: each lane's direct sums are cheaper than the columns
      if (flagged) {
        const float th = a.theta[o], sg = a.sigma[o];
        const PixelResult res = fallback_direct<N>(a, img, x, y, al, be, th, sg);
        a.out[o] = res.g;
        if (a.d_kappa) a.d_kappa[o] = res.kappa;
        if (a.d_t2n) a.d_t2n[o] = res.t2n;
        if (a.d_code) a.d_code[o] = (unsigned char)(res.code | kCodeFallback);
      }
      continue;
    }
    float th = 0.f, sg = 1.f;
    if (flagged) th = a.theta[o], sg = a.sigma[o];
    // The segment's flagged lanes are served in clusters of compatible ranges
    // (a segment may straddle two flat areas): greedy in lane order from the
    // lowest pending lane, the union of the members' [alpha, beta] may grow
    // while its half-range stays within flag_root / 3 of the narrowest
    // member's (then every member passes the amplification test against the
    // union's centre and power-of-two scale); one pass of column power sums
    // per cluster.  A member that still fails (never the first) waits for a
    // later cluster; the first one failing -- impossible by construction --
    // would take the exact direct sums.
    const float lim = (float)(a.flag_root_direct / 3.0);
    unsigned pending = __ballot_sync(0xffffffffu, flagged);
    // greedy cluster from the lowest lane of `rem`: members and their union
    auto greedy = [&](unsigned rem, float& cl, float& ch) {
      const int r = __ffs(rem) - 1;
      cl = __shfl_sync(0xffffffffu, al, r), ch = __shfl_sync(0xffffffffu, be, r);
      float hmin = 0.5f * (ch - cl);
      unsigned mem = 1u << r;
      for (int j = r + 1; j < 32; ++j) {  // warp-uniform
        const float aj = __shfl_sync(0xffffffffu, al, j), bj = __shfl_sync(0xffffffffu, be, j);
        if (!((rem >> j) & 1u)) continue;
        const float nl = fminf(cl, aj), nh = fmaxf(ch, bj), nhm = fminf(hmin, 0.5f * (bj - aj));
        if (0.5f * (nh - nl) <= lim * nhm) cl = nl, ch = nh, hmin = nhm, mem |= 1u << j;
      }
      return mem;
    };
    bool first = true, counted = false;
    while (pending) {
      const int r0 = __ffs(pending) - 1;
      float cl, ch;
      unsigned members;
      if (first) {  // first pass: the union of every flagged lane (one pass serves most segments)
        float umin = flagged ? al : CUDART_INF_F, umax = flagged ? be : -CUDART_INF_F;
        for (int off = 16; off > 0; off >>= 1) {
          umin = fminf(umin, __shfl_xor_sync(0xffffffffu, umin, off));
          umax = fmaxf(umax, __shfl_xor_sync(0xffffffffu, umax, off));
        }
        cl = umin, ch = umax, members = pending;
      } else {  // then greedy clusters of the lanes that failed it
        members = greedy(pending, cl, ch);
        if (!counted) {
          // as many cluster passes as that takes, or every remaining lane's
          // exact direct window sums in parallel -- whichever is cheaper
          // (per-lane samples: (32 + 2 rho) w / 32 + w per pass, w^2 direct)
          counted = true;
          int k = 0;
          for (unsigned rem = pending; rem; ++k) {
            float l2, h2;
            rem &= ~greedy(rem, l2, h2);
          }
          if ((float)k * (float)((32 + 2 * rho) * w / 32 + w) > (float)(w * w)) {
            if ((pending >> lane) & 1u) {
              const PixelResult res = fallback_direct<N>(a, img, x, y, al, be, th, sg);
              a.out[o] = res.g;
              if (a.d_kappa) a.d_kappa[o] = res.kappa;
              if (a.d_t2n) a.d_t2n[o] = res.t2n;
              if (a.d_code) a.d_code[o] = (unsigned char)(res.code | kCodeFallback);
            }
            __syncwarp();
            break;
          }
        }
      }
      const double cT = 0.5 * ((double)cl + (double)ch), halfr = 0.5 * ((double)ch - (double)cl);
      int e2 = 0;
      if (halfr > 0.0) frexp(halfr, &e2);
      const double invS = ldexp(1.0, -e2), mcs = -cT * invS;
      // column power sums over the window rows, lanes over the segment's columns
      for (int cc = lane; cc < Lc; cc += 32) {
        const float* col = img + reflect_index(min(x0 - rho + cc, W - 1 + rho), W);
        double V[NN];
#pragma unroll
        for (int q = 0; q < NN; ++q) V[q] = 0.0;
        const bool inside = y - rho >= 0 && y + rho <= H - 1;
        for (int dy0 = -rho; dy0 <= rho; dy0 += 4) {
          float fv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // loads ahead of the arithmetic
            const int yy = y + min(dy0 + k, rho);
            fv[k] = __ldg(col + (inside ? yy : reflect_index(yy, H)) * W);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (dy0 + k <= rho) {
              const double u = fma((double)fv[k], invS, mcs);
              double pu = u;
#pragma unroll
              for (int q = 0; q < N; ++q) {
                V[q] += pu;
                pu *= u;
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < N; ++q) Vw[q * Lc + cc] = V[q];
      }
      __syncwarp();
      bool served = false;
      if ((members >> lane) & 1u) {
        const double au = fma((double)al, invS, mcs), bu = fma((double)be, invS, mcs);
        const bool amplified = stretch_flagged(au, bu, a.flag_root_direct);
        if (!amplified || (lane == r0 && !first)) {
          PixelResult res;
          if (amplified) {
            res = fallback_direct<N>(a, img, x, y, al, be, th, sg);
          } else {
            double S[N + 1];
            S[0] = (double)(w * w);
#pragma unroll
            for (int q = 1; q <= N; ++q) S[q] = 0.0;
            for (int d = 0; d < w; ++d) {  // N independent chains
#pragma unroll
              for (int q = 1; q <= N; ++q) S[q] += Vw[(q - 1) * Lc + lane + d];
            }
            double nup[NN];
            nu_from_sums<N>(S, au, bu, nup, 1);
            float lam, t0;
            const int regime = range_params(al, be, th, sg, lam, t0);
            res = ghat_from_record<N>(nup, 1, th, sg, al, be, regime, a.flags, a.d_t2n != nullptr,
                                      (double)(w * w));
          }
          a.out[o] = res.g;
          if (a.d_kappa) a.d_kappa[o] = res.kappa;
          if (a.d_t2n) a.d_t2n[o] = res.t2n;
          if (a.d_code) a.d_code[o] = (unsigned char)(res.code | kCodeFallback);
          served = true;
        }
      }
      pending &= ~__ballot_sync(0xffffffffu, served);
      first = false;
      __syncwarp();  // Vw reused by the next cluster / segment
    }
  }
}

// ============================================================================
// NEXT-1: the paper's default spatial kernel, eq.(4): omega(j) =
// exp(-|j|^2 / 2 rho^2) on Omega = [-3 rho, 3 rho]^2.  The moments gamma_k =
// omega * f^k of Algorithm 1 line 6 are separable Gaussian convolutions
// (the paper used direct FIR, "imfilter"); here exact sampled
// FIR in fp64, separable, O(rho) per pixel and power.  One CTA per T x T tile:
//   stage the (T + 2R)^2 footprint (R = 3 rho, reflected borders); its min/max
//   give the tile-local centre c_T and power-of-two scale s_T (u exact);
//   for q = 1..N: P <- P u over the footprint, vertical FIR of P into V,
//   horizontal FIR of V into S_q (all fp64, shared memory);
//   per pixel: alpha, beta from k_bounds (half-width R: every j in Omega has
//   omega(j) > 0, so Lambda_i is the whole box), the stretch / fit / integrals /
//   ratio of fabf_device.cuh with nu_0 = sum omega; pixels whose centring
//   amplification is too large go to k_fallback_gauss (exact weighted sums).
__constant__ double c_gw[2 * 48 + 1];  // omega's 1-D factor exp(-d^2 / 2 rho^2), d = -R..R
constexpr float kGaussKappaBits = 36.0f;

template <int T>
__host__ __device__ constexpr size_t gauss_smem(int R, int N) {
  return sizeof(double) * ((size_t)(T + 2 * R) * (T + 2 * R) + (size_t)T * (T + 2 * R) + (size_t)(N > 0 ? N : 1) * T * T) +
         sizeof(float) * (size_t)(T + 2 * R) * (T + 2 * R);
}

template <int N, int T>
__global__ void __launch_bounds__(kThreads) k_gauss(FilterArgs a, int R, double nu0) {
  extern __shared__ __align__(16) unsigned char smg[];
  constexpr int NN = N > 0 ? N : 1;
  const int FS = T + 2 * R, H = a.H, W = a.W;
  double* P = reinterpret_cast<double*>(smg);  // [FS][FS] current power of u
  double* V = P + FS * FS;                     // [T][FS] vertical FIR of P
  double* S = V + T * FS;                      // [NN][T][T] moments
  float* F = reinterpret_cast<float*>(S + NN * T * T);  // [FS][FS]
  __shared__ float red_min[kThreads / 32], red_max[kThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int x0 = blockIdx.x * T, y0 = blockIdx.y * T, b = blockIdx.z;
  const size_t plane = (size_t)(a.b0 + b) * H * W;
  const float* src = a.img + plane;
  float lmin = CUDART_INF_F, lmax = -CUDART_INF_F;
  for (int t = tid; t < FS * FS; t += kThreads) {
    const int r = t / FS, cc = t - r * FS;
    const float v = __ldg(src + (size_t)reflect_index(y0 - R + r, H) * W + reflect_index(x0 - R + cc, W));
    F[t] = v;
    lmin = fminf(lmin, v);
    lmax = fmaxf(lmax, v);
  }
  for (int off = 16; off > 0; off >>= 1) {
    lmin = fminf(lmin, __shfl_xor_sync(0xffffffffu, lmin, off));
    lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, off));
  }
  if (lane == 0) red_min[warp] = lmin, red_max[warp] = lmax;
  __syncthreads();
  lmin = red_min[0], lmax = red_max[0];
  for (int i = 1; i < kThreads / 32; ++i) lmin = fminf(lmin, red_min[i]), lmax = fmaxf(lmax, red_max[i]);
  const double cT = 0.5 * ((double)lmin + (double)lmax), halfr = 0.5 * ((double)lmax - (double)lmin);
  int e2 = 0;
  if (halfr > 0.0) frexp(halfr, &e2);
  const double invS = ldexp(1.0, -e2), mcs = -cT * invS;  // u = f invS + mcs, exact
  for (int t = tid; t < FS * FS; t += kThreads) P[t] = 1.0;
  for (int q = 0; q < N; ++q) {
    __syncthreads();
    for (int t = tid; t < FS * FS; t += kThreads) P[t] *= fma((double)F[t], invS, mcs);
    __syncthreads();
    for (int t = tid; t < T * FS; t += kThreads) {  // vertical: rows r .. r + 2R of column cc
      const int r = t / FS, cc = t - r * FS;
      const double* col = P + r * FS + cc;
      double acc = 0.0;
      for (int d = 0; d <= 2 * R; ++d) acc = fma(c_gw[d], col[d * FS], acc);
      V[t] = acc;
    }
    __syncthreads();
    for (int t = tid; t < T * T; t += kThreads) {  // horizontal: columns x .. x + 2R of row r
      const int r = t / T, x = t - r * T;
      const double* row = V + r * FS + x;
      double acc = 0.0;
      for (int d = 0; d <= 2 * R; ++d) acc = fma(c_gw[d], row[d], acc);
      S[q * T * T + t] = acc;
    }
  }
  __syncthreads();
  const double n = nu0;  // sum omega, exact to fp64 rounding like the FIR sums (S_0 of the stretch)
  for (int t = tid; t < T * T; t += kThreads) {
    const int r = t / T, x = t - r * T, yy = y0 + r, xx = x0 + x;
    if (yy >= H || xx >= W) continue;
    const int o = (int)plane + yy * W + xx;
    const float al = __ldg(a.alpha + o), be = __ldg(a.beta + o);
    if (al == be) {  // P:204, Algorithm 1 lines 4-5
      a.out[o] = al;
      continue;
    }
    const double au = fma((double)al, invS, mcs), bu = fma((double)be, invS, mcs);
    if (stretch_flagged(au, bu, a.flag_root)) {
      const int slot = atomicAdd(a.fb_count, 1);
      a.fb_list[slot] = o;
      continue;
    }
    double Sq[N + 1], nup[NN];
    Sq[0] = n;
#pragma unroll
    for (int q = 1; q <= N; ++q) Sq[q] = S[(q - 1) * T * T + t];
    nu_from_sums<N>(Sq, au, bu, nup, 1);
    const float th = __ldg(a.theta + o), sg = __ldg(a.sigma + o);
    float lam, t0;
    const int regime = range_params(al, be, th, sg, lam, t0);
    const PixelResult res = ghat_from_record<N>(nup, 1, th, sg, al, be, regime, a.flags, false, n);
    // the moment rounding (eps64 times the centring amplification) reaches
    // g-hat multiplied by kappa: with Gaussian weights a window's effective
    // sample count is small and kappa large, so the amplification test is
    // repeated with kappa once it is known (2^kGaussKappaBits, ~1e-3 grey)
    const double m = 0.5 * (au + bu), h = 0.5 * (bu - au);
    const float amp_bits = (float)N * __log2f((float)((1.0 + fabs(m)) / h)) + __log2f(fmaxf(res.kappa, 1.0f));
    if (N > 0 && !(amp_bits <= kGaussKappaBits)) {
      const int slot = atomicAdd(a.fb_count, 1);
      a.fb_list[slot] = o;
      continue;
    }
    a.out[o] = res.g;
  }
}

// exact weighted moments for the flagged pixels of k_gauss (thread per pixel):
// nu_k = sum_j omega(j) P_k(w_j) with the pixel's own stretch (cf. k_fallback)
template <int N>
__global__ void __launch_bounds__(kThreads) k_fallback_gauss(FilterArgs a, int R, double nu0) {
  const int count = *a.fb_count;
  const int H = a.H, W = a.W;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const int o = a.fb_list[i];
    const int b = o / (H * W), rem = o - b * H * W, y = rem / W, x = rem - y * W;
    const float* img = a.img + (size_t)b * H * W;
    const float al = a.alpha[o], be = a.beta[o];
    const double mid = 0.5 * ((double)al + (double)be), ih = 2.0 / ((double)be - (double)al);
    double acc[N + 1];
#pragma unroll
    for (int k = 0; k <= N; ++k) acc[k] = 0.0;
    for (int dy = -R; dy <= R; ++dy) {
      const float* row = img + reflect_index(y + dy, H) * W;
      const double wy = c_gw[dy + R];
      for (int dx = -R; dx <= R; ++dx) {
        const double wgt = wy * c_gw[dx + R];
        const double sv = ((double)__ldg(row + reflect_index(x + dx, W)) - mid) * ih;
        double r0 = 1.0, r1 = sv;
        acc[0] += wgt;
        if (N >= 1) acc[1] += wgt * sv;
#pragma unroll
        for (int k = 1; k < N; ++k) {
          const double r2 = fma(-(double)(k * k) / (double)(4 * k * k - 1), r0, sv * r1);
          acc[k + 1] = fma(wgt, r2, acc[k + 1]);
          r0 = r1;
          r1 = r2;
        }
      }
    }
    double nu[N + 1];
#pragma unroll
    for (int k = 0; k <= N; ++k) nu[k] = (double)(2 * k + 1) * c_monic_scale[k] * acc[k];
    float lam, t0;
    const float th = a.theta[o], sg = a.sigma[o];
    const int regime = range_params(al, be, th, sg, lam, t0);
    const PixelResult res = ghat_from_record<N>(nu + 1, 1, th, sg, al, be, regime, a.flags, false, nu[0]);
    a.out[o] = res.g;
  }
}

// ============================================================================
// Mozerov & van de Weijer's uniform-prior filter (NEXT-4), the baseline the
// paper compares with (Fig.3): a degree-0 fit of the local
// histogram on [f(i), 2 fbar(i) - f(i)] (Delta = 0) instead of [alpha, beta],
// i.e. eq.(29) at N = 0 on that interval (identity when it is a point).  One
// CTA per T x T output tile: the (T + 2 rho)^2 footprint staged in shared
// memory (reflected borders), box sums by sliding windows in fp64 (rows, then
// columns), then the N = 0 integrals of fabf_device.cuh per pixel.
template <int T>
__global__ void __launch_bounds__(kThreads) k_mozerov(const float* __restrict__ img,
                                                       const float* __restrict__ theta,
                                                       const float* __restrict__ sigma, float* __restrict__ out,
                                                       int H, int W, int rho, unsigned flags) {
  extern __shared__ __align__(16) unsigned char smm[];
  const int w = 2 * rho + 1, FS = T + 2 * rho;
  double* Hs = reinterpret_cast<double*>(smm);                       // [FS][T]
  float* F = reinterpret_cast<float*>(smm + sizeof(double) * FS * T);  // [FS][FS]
  const int x0 = blockIdx.x * T, y0 = blockIdx.y * T, b = blockIdx.z;
  const size_t plane = (size_t)b * H * W;
  const float* src = img + plane;
  for (int t = threadIdx.x; t < FS * FS; t += kThreads) {
    const int r = t / FS, cc = t - r * FS;
    F[t] = __ldg(src + (size_t)reflect_index(y0 - rho + r, H) * W + reflect_index(x0 - rho + cc, W));
  }
  __syncthreads();
  for (int r = threadIdx.x; r < FS; r += kThreads) {  // horizontal window sums, sliding
    const float* Fr = F + r * FS;
    double acc = 0.0;
    for (int cc = 0; cc < w; ++cc) acc += Fr[cc];
    Hs[r * T] = acc;
    for (int x = 1; x < T; ++x) {
      acc += (double)Fr[x + w - 1] - (double)Fr[x - 1];
      Hs[r * T + x] = acc;
    }
  }
  __syncthreads();
  constexpr int SEG = T * T / kThreads;  // output rows per thread (column x, rows r0 .. r0 + SEG)
  const int x = threadIdx.x % T, r0 = (threadIdx.x / T) * SEG;
  double acc = 0.0;
  for (int dy = 0; dy < w; ++dy) acc += Hs[(r0 + dy) * T + x];
  const float n = (float)(w * w);
  for (int k = 0; k < SEG; ++k) {
    if (k > 0) acc += Hs[(r0 + k + w - 1) * T + x] - Hs[(r0 + k - 1) * T + x];
    const int yy = y0 + r0 + k, xx = x0 + x;
    if (yy >= H || xx >= W) continue;
    const size_t o = plane + (size_t)yy * W + xx;
    const double f = (double)F[(r0 + k + rho) * FS + x + rho];
    const double e = 2.0 * (acc / (double)n) - f;  // 2 fbar - f
    const float a = (float)fmin(f, e), bb = (float)fmax(f, e);
    if (!(bb > a)) {
      out[o] = (float)f;
      continue;
    }
    const float th = theta[o], sg = sigma[o];
    float lam, t0;
    const int regime = range_params(a, bb, th, sg, lam, t0);
    const PixelResult res = ghat_from_record<0>(nullptr, 1, th, sg, a, bb, regime, flags & kFlagLiteral, false, n);
    out[o] = res.g;
  }
}

// ============================================================================
// NEXT-2: the sharpening application's range-kernel maps, produced
// on the device from f alone so that only f crosses PCIe:
//   theta = f + (f - fbar), fbar = the box mean over Omega (half-width rho);
//   sigma = s_hi - (s_hi - s_lo) min(|LoG f| / l_sat, 1)         (reading R15)
// with LoG the sampled normalised Gaussian of scale s (|x| <= ceil(4 s)) and its
// analytic second derivative, separable: L = g''_x g_y + g_x g''_y.  One CTA per
// T x T tile: footprint staged in shared memory (reflected borders), box sums
// by sliding windows in fp64, the two LoG terms by separable fp32 passes.
constexpr int kMaxLogR = 16;
__constant__ float c_log_g[2 * kMaxLogR + 1], c_log_g2[2 * kMaxLogR + 1];

template <int T>
__global__ void __launch_bounds__(kThreads) k_sharpen_maps(const float* __restrict__ img,
                                                            float* __restrict__ theta, float* __restrict__ sigma,
                                                            int H, int W, int rho, int rl, float s_lo, float s_hi,
                                                            float inv_sat) {
  extern __shared__ __align__(16) unsigned char sms[];
  const int R = max(rho, rl), FS = T + 2 * R, w = 2 * rho + 1;
  double* Hs = reinterpret_cast<double*>(sms);                            // [T + 2 rho][T] box row sums
  float* F = reinterpret_cast<float*>(sms + sizeof(double) * (T + 2 * rho) * T);  // [FS][FS]
  float* Ga = F + FS * FS;                                                 // [T + 2 rl][T]: g_x * f
  float* Gb = Ga + (T + 2 * rl) * T;                                       // [T + 2 rl][T]: g''_x * f
  const int x0 = blockIdx.x * T, y0 = blockIdx.y * T, b = blockIdx.z;
  const size_t plane = (size_t)b * H * W;
  const float* src = img + plane;
  for (int t = threadIdx.x; t < FS * FS; t += kThreads) {
    const int r = t / FS, cc = t - r * FS;
    F[t] = __ldg(src + (size_t)reflect_index(y0 - R + r, H) * W + reflect_index(x0 - R + cc, W));
  }
  __syncthreads();
  // box: rows R - rho .. R + rho + T - 1 of the footprint, sliding sums
  for (int r = threadIdx.x; r < T + 2 * rho; r += kThreads) {
    const float* Fr = F + (r + R - rho) * FS + (R - rho);
    double acc = 0.0;
    for (int cc = 0; cc < w; ++cc) acc += Fr[cc];
    Hs[r * T] = acc;
    for (int x = 1; x < T; ++x) {
      acc += (double)Fr[x + w - 1] - (double)Fr[x - 1];
      Hs[r * T + x] = acc;
    }
  }
  // LoG, horizontal pass: rows R - rl .. R + rl + T - 1
  for (int t = threadIdx.x; t < (T + 2 * rl) * T; t += kThreads) {
    const int r = t / T, x = t - r * T;
    const float* Fr = F + (r + R - rl) * FS + (R - rl) + x;
    float a = 0.f, bb = 0.f;
    for (int k = 0; k <= 2 * rl; ++k) {  // tap k <-> offset dx = rl - k (convolution)
      const float v = Fr[2 * rl - k];
      a = fmaf(c_log_g[k], v, a);
      bb = fmaf(c_log_g2[k], v, bb);
    }
    Ga[t] = a;
    Gb[t] = bb;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < T * T; t += kThreads) {
    const int y = t / T, x = t - y * T;
    const int yy = y0 + y, xx = x0 + x;
    if (yy >= H || xx >= W) continue;
    double acc = 0.0;
    for (int dy = 0; dy < w; ++dy) acc += Hs[(y + dy) * T + x];
    float L = 0.f;
    for (int k = 0; k <= 2 * rl; ++k) {
      const int rr = (y + 2 * rl - k) * T + x;
      L = fmaf(c_log_g2[k], Ga[rr], fmaf(c_log_g[k], Gb[rr], L));
    }
    const double f = (double)F[(y + R) * FS + x + R];
    const size_t o = plane + (size_t)yy * W + xx;
    theta[o] = (float)(2.0 * f - acc / (double)(w * w));
    sigma[o] = s_hi - (s_hi - s_lo) * fminf(fabsf(L) * inv_sat, 1.0f);
  }
}

// ============================================================================
// NEXT-2, second application: the texture-filtering sigma map,
//   mRTV(i) = Delta(i) max_{W_i} |grad f| / (sum_{W_i} |grad f| + eps),
//   Delta(i) = max_{W_i} f - min_{W_i} f,
//   sigma = s_hi - (s_hi - s_lo) min(mRTV / m_sat, 1)              (reading R19)
// W_i = the box of half-width pr, grad f by forward differences with the image
// reflected at its borders (0 across the last column / row), a window position
// outside the image takes the pixel it reflects to.  One CTA per T x T tile: f
// and |grad f| (fp64: products and sum rounded separately, IEEE sqrt) of the
// (T + 2 pr)^2 footprint in shared memory, then the separable window max / min /
// sum (rows, then columns; pr is small: direct O(pr) scans).  Writes sigma,
// scale2 * sigma (the pipeline's second pass) and, if asked, mRTV.
constexpr int kMaxPatch = 16;
template <int T>
__global__ void __launch_bounds__(kThreads) k_texture_maps(const float* __restrict__ img,
                                                            float* __restrict__ sigma, float* __restrict__ sigma2,
                                                            float* __restrict__ mrtv, int H, int W, int pr,
                                                            float s_lo, float s_hi, double inv_sat, double eps,
                                                            float scale2) {
  extern __shared__ __align__(16) unsigned char smt[];
  const int FS = T + 2 * pr, k = 2 * pr + 1;
  double* G = reinterpret_cast<double*>(smt);  // [FS][FS] gradient magnitude
  double* Hs = G + FS * FS;                    // [FS][T] row-window sum of G
  double* Hm = Hs + FS * T;                    // [FS][T] row-window max of G
  float* F = reinterpret_cast<float*>(Hm + FS * T);  // [FS][FS]
  float* Hlo = F + FS * FS;                    // [FS][T] row-window min of f
  float* Hhi = Hlo + FS * T;                   // [FS][T] row-window max of f
  const int x0 = blockIdx.x * T, y0 = blockIdx.y * T, b = blockIdx.z;
  const size_t plane = (size_t)b * H * W;
  const float* src = img + plane;
  for (int t = threadIdx.x; t < FS * FS; t += kThreads) {
    const int r = t / FS, cc = t - r * FS;
    // (rows / columns past H - 1 + pr only feed outputs outside the image)
    const int yy = reflect_index(min(y0 - pr + r, H - 1 + pr), H), xx = reflect_index(min(x0 - pr + cc, W - 1 + pr), W);
    const float f = __ldg(src + (size_t)yy * W + xx);
    const double gx = (double)__ldg(src + (size_t)yy * W + reflect_index(xx + 1, W)) - (double)f;
    const double gy = (double)__ldg(src + (size_t)reflect_index(yy + 1, H) * W + xx) - (double)f;
    F[t] = f;
    G[t] = sqrt(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)));
  }
  __syncthreads();
  for (int t = threadIdx.x; t < FS * T; t += kThreads) {
    const int r = t / T, x = t - r * T;
    const double* Gr = G + r * FS + x;
    const float* Fr = F + r * FS + x;
    double sum = 0.0, gm = 0.0;
    float lo = CUDART_INF_F, hi = -CUDART_INF_F;
    for (int cc = 0; cc < k; ++cc) {
      sum += Gr[cc];
      gm = fmax(gm, Gr[cc]);
      lo = fminf(lo, Fr[cc]);
      hi = fmaxf(hi, Fr[cc]);
    }
    Hs[t] = sum;
    Hm[t] = gm;
    Hlo[t] = lo;
    Hhi[t] = hi;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < T * T; t += kThreads) {
    const int y = t / T, x = t - y * T;
    const int yy = y0 + y, xx = x0 + x;
    if (yy >= H || xx >= W) continue;
    double sum = 0.0, gm = 0.0;
    float lo = CUDART_INF_F, hi = -CUDART_INF_F;
    for (int dy = 0; dy < k; ++dy) {
      const int rr = (y + dy) * T + x;
      sum += Hs[rr];
      gm = fmax(gm, Hm[rr]);
      lo = fminf(lo, Hlo[rr]);
      hi = fmaxf(hi, Hhi[rr]);
    }
    const double m = ((double)hi - (double)lo) * gm / (sum + eps);
    const float sg = (float)((double)s_hi - ((double)s_hi - (double)s_lo) * fmin(m * inv_sat, 1.0));
    const size_t o = plane + (size_t)yy * W + xx;
    sigma[o] = sg;
    if (sigma2) sigma2[o] = scale2 * sg;
    if (mrtv) mrtv[o] = (float)m;
  }
}

// ============================================================================
// colour (NEXT-3): channel-interleaved images (B x H x W x C) <-> the planar
// batch (B C) x H x W the filter runs on, channel by channel as the paper
// filters colour images.  Pure data movement, coalesced on the
// interleaved side.
__global__ void __launch_bounds__(kThreads) k_deinterleave(const float* __restrict__ a,
                                                            const float* __restrict__ b,
                                                            const float* __restrict__ c, float* __restrict__ pa,
                                                            float* __restrict__ pb, float* __restrict__ pc,
                                                            long long HW, int C, long long total) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long px = t / C, ch = t - px * C, bi = px / HW, q = px - bi * HW;
    const long long o = (bi * C + ch) * HW + q;  // plane (b, ch), pixel q
    pa[o] = a[t];
    pb[o] = b[t];
    pc[o] = c[t];
  }
}
__global__ void __launch_bounds__(kThreads) k_interleave(const float* __restrict__ p, float* __restrict__ out,
                                                          long long HW, int C, long long total) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long px = t / C, ch = t - px * C, bi = px / HW, q = px - bi * HW;
    out[t] = p[(bi * C + ch) * HW + q];
  }
}

// sigma2 = scale * sigma (the texture application's second pass on a caller's map)
__global__ void __launch_bounds__(kThreads) k_scale(const float* __restrict__ x, float* __restrict__ y, float scale,
                                                     long long total) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x)
    y[t] = scale * x[t];
}

// ============================================================================
// FABF_FLAG_DEBUG: device-side check of the preconditions (include/fabf.h):
// f, theta finite, sigma finite and > 0.  Counts violations of the pixels
// [lo, lo + n) of each image b0 .. b0 + nb - 1 and keeps the smallest index.
__global__ void __launch_bounds__(kThreads) k_validate(const float* __restrict__ img,
                                                        const float* __restrict__ theta,
                                                        const float* __restrict__ sigma, size_t plane,
                                                        int b0, int nb, size_t lo, size_t n,
                                                        unsigned long long* dbg) {
  const size_t total = (size_t)nb * n;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t - threadIdx.x < total;
       t += (size_t)gridDim.x * blockDim.x) {
    bool bad = false;
    unsigned long long o = ~0ull;
    if (t < total) {
      const size_t b = t / n;
      o = (unsigned long long)((b0 + b) * plane + lo + (t - b * n));
      const float f = img[o], th = theta[o], sg = sigma[o];
      bad = !(isfinite(f) && isfinite(th) && isfinite(sg) && sg > 0.0f);
    }
    const unsigned m = __ballot_sync(0xffffffffu, bad);
    if (m) {
      unsigned long long first = bad ? o : ~0ull;
      for (int off = 16; off > 0; off >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, off));
      if ((threadIdx.x & 31) == 0) {
        atomicAdd(&dbg[0], (unsigned long long)__popc(m));
        atomicMin(&dbg[1], first);
      }
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
  if (dev < 0 || dev >= kMaxDevices) return fail(FABF_ERR_UNSUPPORTED, "device ordinal >= 64");
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

template <int RC>
fabf_status_t launch_bounds_rc(Plan* p, const float* img, int rho, float* alpha, float* beta,
                               int b0, int nb, int ty0, int ty1, cudaStream_t st) {
  const bool stage = bounds_smem<RC>(rho, true) <= (size_t)kMaxDynSmem;
  const size_t smem = bounds_smem<RC>(rho, stage);
  {  // the dynamic-shared-memory opt-in is a per-device function attribute
    static bool attr_set[kMaxDevices] = {};
    std::lock_guard<std::mutex> lk(g_launch_mu);
    if (!attr_set[p->device]) {
      FABF_CUDA(cudaFuncSetAttribute(k_bounds<RC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kMaxDynSmem),
                "cudaFuncSetAttribute(k_bounds)");
      FABF_CUDA(cudaFuncSetAttribute(k_bounds<RC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kMaxDynSmem),
                "cudaFuncSetAttribute(k_bounds)");
      attr_set[p->device] = true;
    }
  }
  // TMA descriptor for interior tiles (needs 16-byte row pitch); encoded
  // once per (image pointer, rho class) through the runtime's driver entry point
  if (stage && (p->tmap_ptr != img || p->tmap_rc != RC)) {
    p->tmap_ptr = img;
    p->tmap_rc = RC;
    p->tmap_ok = false;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    std::lock_guard<std::mutex> lk(g_launch_mu);
    if (!encode) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
      else
        cudaGetLastError();
    }
    constexpr cuuint32_t FPB = (cuuint32_t)BoundsGeom<RC>::FP, FRB = (cuuint32_t)BoundsGeom<RC>::FR;
    if (encode && p->W % 4 == 0 && FPB <= 256 && FRB <= 256) {
      const cuuint64_t dims[3] = {(cuuint64_t)p->W, (cuuint64_t)p->H, (cuuint64_t)p->B};
      const cuuint64_t strides[2] = {(cuuint64_t)p->W * 4, (cuuint64_t)p->W * p->H * 4};
      const cuuint32_t box[3] = {FPB, FRB, 1};
      const cuuint32_t es[3] = {1, 1, 1};
      p->tmap_ok = encode(&p->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(img), dims,
                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
  }
  const int use_tma = (stage && p->tmap_ok) ? 1 : 0;
  dim3 g((p->W + kBT - 1) / kBT, ty1 - ty0, nb);
  if (stage)
    k_bounds<RC, true><<<g, kThreads, smem, st>>>(img, p->H, p->W, rho, alpha, beta, p->blkmm, b0, ty0,
                                                  p->tmap, use_tma);
  else
    k_bounds<RC, false><<<g, kThreads, smem, st>>>(img, p->H, p->W, rho, alpha, beta, p->blkmm, b0,
                                                   ty0, p->tmap, 0);
  ++g_launches;
  FABF_CUDA(cudaGetLastError(), "k_bounds launch");
  return FABF_OK;
}

// the separable two-pass bounds (k_bounds_h + k_bounds_v) for rows
// [64 ty0, 64 ty1) of images [b0, b0 + nb)
template <int SEG, bool DIRECT>
fabf_status_t launch_bounds_sep_seg(Plan* p, const float* img, int rho, float* alpha, float* beta, int b0,
                                    int nb, int ty0, int ty1, cudaStream_t st) {
  const int r0 = ty0 * kBT, r1 = std::min(p->H, ty1 * kBT);
  const int h0 = std::max(0, r0 - rho), h1 = std::min(p->H, r1 + rho);  // rows the column pass reads
  const size_t smem = hpass_smem(rho);
  {
    static bool attr_set[kMaxDevices] = {};
    std::lock_guard<std::mutex> lk(g_launch_mu);
    if (!attr_set[p->device]) {
      FABF_CUDA(cudaFuncSetAttribute(k_bounds_h<SEG, DIRECT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kMaxDynSmem),
                "cudaFuncSetAttribute(k_bounds_h)");
      attr_set[p->device] = true;
    }
  }
  dim3 gh((p->W + kHW - 1) / kHW, (h1 - h0 + kHR - 1) / kHR, nb);
  k_bounds_h<SEG, DIRECT><<<gh, kThreads, smem, st>>>(img, p->H, p->W, rho, p->hmm, b0, h0, h1);
  ++g_launches;
  FABF_CUDA(cudaGetLastError(), "k_bounds_h launch");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((p->W + kBT - 1) / kBT, ty1 - ty0, nb);
  cfg.blockDim = dim3(kBT * kBT / SEG);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  FABF_CUDA(cudaLaunchKernelEx(&cfg, k_bounds_v<SEG, DIRECT>, (const float2*)p->hmm, p->H, p->W, rho, alpha, beta,
                               p->blkmm, b0, ty0),
            "k_bounds_v launch");
  ++g_launches;
  return FABF_OK;
}
fabf_status_t launch_bounds_sep(Plan* p, const float* img, int rho, float* alpha, float* beta, int b0, int nb,
                                int ty0, int ty1, cudaStream_t st) {
  const int w = 2 * rho + 1;
  if (w >= 32) return launch_bounds_sep_seg<32, false>(p, img, rho, alpha, beta, b0, nb, ty0, ty1, st);
  if (w >= 16) return launch_bounds_sep_seg<16, false>(p, img, rho, alpha, beta, b0, nb, ty0, ty1, st);
  if (w >= 8) return launch_bounds_sep_seg<8, false>(p, img, rho, alpha, beta, b0, nb, ty0, ty1, st);
  return launch_bounds_sep_seg<8, true>(p, img, rho, alpha, beta, b0, nb, ty0, ty1, st);
}

// bounds placement: the separable passes (default) or the 2-D tile kernel
// k_bounds (FABF_BOUNDS=tile: A/B switch)
// (default: the 64 x 128 in-place kernel k_bounds2 for 8 <= rho <= 24, the
// 64 x 64 tile kernel below, the separable passes above; FABF_BOUNDS=tile /
// sep / t2 forces one where it applies)
int g_bounds_mode = !getenv("FABF_BOUNDS") ? 0 : std::string(getenv("FABF_BOUNDS")) == "tile" ? 1
                    : std::string(getenv("FABF_BOUNDS")) == "sep" ? 2
                    : std::string(getenv("FABF_BOUNDS")) == "t2" ? 3 : 0;

template <int SEGH, int SEGV>
fabf_status_t launch_bounds2_seg(Plan* p, const float* img, int rho, float* alpha, float* beta, int b0, int nb,
                                 int ty0, int ty1, cudaStream_t st) {
  const size_t smem = bounds2_smem(rho);
  {
    static bool attr_set[kMaxDevices] = {};
    std::lock_guard<std::mutex> lk(g_launch_mu);
    if (!attr_set[p->device]) {
      FABF_CUDA(cudaFuncSetAttribute(k_bounds2<SEGH, SEGV>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem),
                "cudaFuncSetAttribute(k_bounds2)");
      attr_set[p->device] = true;
    }
  }
  dim3 g((p->W + kB2C - 1) / kB2C, (ty1 - ty0 + 1) / 2, nb);
  k_bounds2<SEGH, SEGV><<<g, kThreads, smem, st>>>(img, p->H, p->W, rho, alpha, beta, p->blkmm, b0, ty0, ty1);
  ++g_launches;
  FABF_CUDA(cudaGetLastError(), "k_bounds2 launch");
  return FABF_OK;
}
fabf_status_t launch_bounds2(Plan* p, const float* img, int rho, float* alpha, float* beta, int b0, int nb,
                             int ty0, int ty1, cudaStream_t st) {
  if (2 * rho + 1 >= 32) return launch_bounds2_seg<32, 32>(p, img, rho, alpha, beta, b0, nb, ty0, ty1, st);
  return launch_bounds2_seg<16, 16>(p, img, rho, alpha, beta, b0, nb, ty0, ty1, st);
}

// rows [64 ty0, 64 ty1) of images [b0, b0 + nb)
fabf_status_t launch_bounds(Plan* p, const float* img, int rho, float* alpha, float* beta, int b0,
                            int nb, int ty0, int ty1, cudaStream_t st) {
  prof_mark(0, st);
  fabf_status_t s;
  if ((g_bounds_mode == 0 || g_bounds_mode == 3) && rho >= 8 && rho <= 24) {
    s = launch_bounds2(p, img, rho, alpha, beta, b0, nb, ty0, ty1, st);
    if (s != FABF_OK) return s;
    prof_mark(1, st);
    prof_mark(2, st);
    return FABF_OK;
  }
  if (g_bounds_mode == 2 || (g_bounds_mode == 0 && rho > 24)) {
    s = launch_bounds_sep(p, img, rho, alpha, beta, b0, nb, ty0, ty1, st);
    if (s != FABF_OK) return s;
    prof_mark(1, st);
    prof_mark(2, st);
    return FABF_OK;
  }
  if (rho <= 8)
    s = launch_bounds_rc<8>(p, img, rho, alpha, beta, b0, nb, ty0, ty1, st);
  else if (rho <= 24)
    s = launch_bounds_rc<24>(p, img, rho, alpha, beta, b0, nb, ty0, ty1, st);
  else if (rho <= 48)
    s = launch_bounds_rc<48>(p, img, rho, alpha, beta, b0, nb, ty0, ty1, st);
  else
    s = launch_bounds_rc<kMaxRho>(p, img, rho, alpha, beta, b0, nb, ty0, ty1, st);
  if (s != FABF_OK) return s;
  prof_mark(1, st);
  prof_mark(2, st);
  return FABF_OK;
}

// pixels per thread per step: 2 when the (worst-case L = 16E) shared memory
// still fits two CTAs per SM, else 1
template <int N, int E, bool FB>
constexpr int ppt_for() {
  constexpr size_t NN = N > 0 ? N : 1;
  constexpr size_t L = (size_t)kSL * E;
  constexpr size_t ps2 = sizeof(double) * 4 * NN * (L + 2);
  constexpr size_t vs = sizeof(double) * (NN | 1) * L;
  constexpr size_t q2 = (sizeof(double) * NN + 4 + (FB ? 0 : 16)) * 2 * kThreads;
  // bounds rows (worst case over the rho this E serves, TW = 128):
  constexpr size_t bz = FB ? sizeof(float2) * 4 * (L + 2 * 128) : 0;
  return ps2 + vs + q2 + bz <= 114 * 1024 ? 2 : 1;
}
constexpr int kMaxCtaPerSm = 3;  // persistent grid cap (sizes the plan's bounds rings)

// bounds-ring elements (float2) one CTA needs for rho (TW as launch_filter_n picks it)
inline long long ring_elems_per_cta(int rho) {
  const int TW = (128 + 2 * rho <= 256) ? 128 : 64;
  return 2LL * (2 * rho + 1) * (TW + 2 * rho);
}

template <int N, int E, int TW, int WD, bool FB>
fabf_status_t launch_filter_fb(FilterArgs& fa, cudaStream_t st) {
#ifdef FABF_PPT
  constexpr int PPT = FABF_PPT;
#else
  constexpr int PPT = ppt_for<N, E, FB>();
#endif
  const int L = TW + 2 * fa.rho, QS = PPT * kThreads, RB = QS / TW;
  const size_t smem = FilterSmem<N, E>(L, RB, QS, TW, FB).total;
  if (smem > kMaxDynSmem) return fail(FABF_ERR_INVALID_ARGUMENT, "rho too large for shared memory");
  static int grid_cache[kMaxDevices] = {};  // resident CTAs per device (persistent schedule)
  static size_t smem_cache[kMaxDevices] = {};
  int dev = 0;
  FABF_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  std::unique_lock<std::mutex> lk(g_launch_mu);
  if (grid_cache[dev] == 0 || smem_cache[dev] != smem) {
    FABF_CUDA(cudaFuncSetAttribute(k_filter<N, E, TW, PPT, WD, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kMaxDynSmem),
              "cudaFuncSetAttribute(k_filter)");
    int per_sm = 0, sms = 0;
    FABF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_filter<N, E, TW, PPT, WD, FB>, kThreads, smem),
              "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    FABF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    grid_cache[dev] = std::min(std::max(1, per_sm), kMaxCtaPerSm) * sms;
    smem_cache[dev] = smem;
  }
  const long long strips = (long long)fa.B * ((fa.W + TW - 1) / TW) * (fa.r1 - fa.r0);
  long long grid_ll = std::min<long long>(grid_cache[dev], strips);
  if (FB) grid_ll = std::min<long long>(grid_ll, fa.ring_ctas);  // one bounds ring per CTA
  const int grid = (int)grid_ll;
  lk.unlock();
  FABF_CUDA(launch_pdl(k_filter<N, E, TW, PPT, WD, FB>, grid, kThreads, smem, st, fa), "k_filter launch");
  ++g_launches;
  return FABF_OK;
}

template <int N, int E, int TW, int WD = 0>
fabf_status_t launch_filter_net(FilterArgs& fa, cudaStream_t st) {
  return fa.fused ? launch_filter_fb<N, E, TW, WD, true>(fa, st) : launch_filter_fb<N, E, TW, WD, false>(fa, st);
}

template <int N>
fabf_status_t launch_filter_n(FilterArgs& fa, int B, cudaStream_t st) {
  (void)B;
  const int L128 = 128 + 2 * fa.rho;
  fabf_status_t s;
  // prefix rows of 16*E entries, E odd (conflict-free strided phase-B access)
  // (column owners: L = TW + 2 rho <= 256 threads)
  if (fa.rho <= 3) {  // direct window sums (see k_filter, phase B)
    switch (fa.rho) {
      case 0: s = launch_filter_net<N, 9, 128, 1>(fa, st); break;
      case 1: s = launch_filter_net<N, 9, 128, 3>(fa, st); break;
      case 2: s = launch_filter_net<N, 9, 128, 5>(fa, st); break;
      default: s = launch_filter_net<N, 9, 128, 7>(fa, st); break;
    }
  } else if (L128 <= 16 * 9)
    s = launch_filter_net<N, 9, 128>(fa, st);
  else if (L128 <= 16 * 11)
    s = launch_filter_net<N, 11, 128>(fa, st);
  else if (L128 <= 16 * 13)
    s = launch_filter_net<N, 13, 128>(fa, st);
  else if (L128 <= 16 * 15)
    s = launch_filter_net<N, 15, 128>(fa, st);
  else if (L128 <= 256)
    s = launch_filter_net<N, 17, 128>(fa, st);
  else
    s = launch_filter_net<N, 17, 64>(fa, st);
  if (s != FABF_OK) return s;
  prof_mark(3, st);
  {  // the exact-moment fallback by row segments
    const size_t smem = sizeof(double) * kSegWarps * (N > 0 ? N : 1) * (32 + 2 * fa.rho);
    static bool attr_set[kMaxDevices] = {};
    int dev = 0;
    FABF_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    {
      std::lock_guard<std::mutex> lk(g_launch_mu);
      if (!attr_set[dev]) {
        FABF_CUDA(cudaFuncSetAttribute(k_fallback_seg<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem),
                  "cudaFuncSetAttribute(k_fallback_seg)");
        attr_set[dev] = true;
      }
    }
    FABF_CUDA(launch_pdl(k_fallback_seg<N>, 148 * 4, 32 * kSegWarps, smem, st, fa), "k_fallback_seg launch");
    ++g_launches;
  }
  prof_mark(4, st);
  return FABF_OK;
}

fabf_status_t launch_filter(FilterArgs& fa, int N, int B, cudaStream_t st) {
#ifdef FABF_ONLY_N  // development builds: one degree only (fast compiles)
  if (N == FABF_ONLY_N) return launch_filter_n<FABF_ONLY_N>(fa, B, st);
  return fail(FABF_ERR_UNSUPPORTED, "library built with FABF_ONLY_N");
#else
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
#endif
}

// a plan's workspace lives on the device it was made on; calls must be made
// with that device current (the library never switches the caller's device)
fabf_status_t check_plan_device(Plan* p) {
  int dev = -1;
  FABF_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev != p->device)
    return fail(FABF_ERR_INVALID_ARGUMENT, "plan was made on device " + std::to_string(p->device) +
                                               " but device " + std::to_string(dev) + " is current");
  return FABF_OK;
}

fabf_status_t validate_common(Plan* p, int rho) {
  if (!p) return fail(FABF_ERR_INVALID_ARGUMENT, "plan is NULL");
  {
    fabf_status_t s = check_plan_device(p);
    if (s != FABF_OK) return s;
  }
  if (rho < 0) return fail(FABF_ERR_INVALID_ARGUMENT, "rho < 0");
  if (2 * rho + 1 > p->H || 2 * rho + 1 > p->W)
    return fail(FABF_ERR_INVALID_ARGUMENT, "2*rho+1 exceeds min(height, width)");
  if (rho > kMaxRho)
    return fail(FABF_ERR_INVALID_ARGUMENT, "rho > " + std::to_string(kMaxRho) + " not supported");
  return FABF_OK;
}

fabf_status_t validate_filter(Plan* p, const float* img, const float* theta, const float* sigma,
                              int rho, int N, float* out) {
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
  return FABF_OK;
}

// where the bounds run: FABF_FLAG_FUSED plans always in k_filter; otherwise
// in k_filter for rho <= g_fuse_rho (default kFuseRho) on small calls
// (<= kFusePixels), else in k_bounds.  FABF_FUSE_RHO overrides the rho
// crossover (experiments).
bool fused_choice(const Plan* p, int rho) {
  if (p->flags & FABF_FLAG_FUSED) return true;
  return rho <= g_fuse_rho && (long long)p->B * p->H * p->W <= kFusePixels &&
         p->ring_elems >= ring_elems_per_cta(rho);
}

// The three kernels for images [b0, b0 + nb), rows [64 ty0, min(H, 64 ty1)).
// Reads input rows up to rho outside the band (the caller guarantees they are
// in place); writes out, alpha, beta of the band only.
fabf_status_t filter_band(Plan* p, const float* img, const float* theta, const float* sigma, int rho,
                          int N, float* out, const fabf_diag_t* diag, int b0, int nb, int ty0,
                          int ty1, int fb_slot, cudaStream_t st) {
  p->last_stream = st;
  if (p->flags & FABF_FLAG_DEBUG) {  // preconditions of the band's own pixels
    const size_t lo = (size_t)ty0 * kBT * p->W, hi = (size_t)std::min(p->H, ty1 * kBT) * p->W;
    k_validate<<<148 * 4, kThreads, 0, st>>>(img, theta, sigma, (size_t)p->H * p->W, b0, nb, lo, hi - lo,
                                              p->dbg);
    ++g_launches;
    FABF_CUDA(cudaGetLastError(), "k_validate launch");
  }
  // bounds inside k_filter (north_star (e): each pixel crosses HBM once) or
  // from k_bounds' planes (the faster choice where k_filter is issue-bound,
  // DESIGN.md section 4): fused_choice()
  const bool fused = fused_choice(p, rho);
  fabf_status_t s = FABF_OK;
  if (fused)
    prof_mark(0, st), prof_mark(1, st), prof_mark(2, st);
  else
    s = launch_bounds(p, img, rho, p->alpha, p->beta, b0, nb, ty0, ty1, st);
  if (s != FABF_OK) return s;
  FilterArgs fa;
  fa.fused = fused ? 1 : 0;
  fa.alpha = p->alpha;
  fa.beta = p->beta;
  fa.blkmm = p->blkmm;
  fa.img = img;
  fa.theta = theta;
  fa.sigma = sigma;
  fa.alpha_w = p->alpha;
  fa.beta_w = p->beta;
  fa.out = out;
  fa.H = p->H;
  fa.W = p->W;
  fa.rho = rho;
  fa.B = nb;
  fa.b0 = b0;
  fa.r0 = ty0 * kBT;
  fa.r1 = std::min(p->H, ty1 * kBT);
  // segment cap (rows): fresh fp64 sums every few window heights
  fa.SH = std::max(g_seg_min, g_seg_w * (2 * rho + 1));
  fa.flags = p->flags;
  fa.ring = p->ring;
  fa.ring_cta = ring_elems_per_cta(rho);
  fa.ring_ctas = p->ring_elems / std::max(1LL, fa.ring_cta);
  {
    // fallback flag: amplification ((1+|m|)/h)^N times the magnitude of the
    // summed terms relative to n (prefix rows: L w / n; direct sums: 1) may
    // not exceed 2^kFlagBits ("Numerical envelope")
    const int w = 2 * rho + 1, L = (rho <= 64 ? 128 : 64) + 2 * rho;
    const double mag = rho <= 3 ? 1.0 : (double)L * w / ((double)w * w);
    const double bits = (double)kFlagBits - std::log2(mag);
    fa.flag_root = N > 0 ? std::pow(2.0, bits / N) : 1e300;
    fa.flag_root_direct = N > 0 ? std::pow(2.0, (double)kFlagBits / N) : 1e300;
  }
  fa.fb_count = p->fb_count + fb_slot;
  fa.fb_list = p->fb_list + ((size_t)b0 * p->H + fa.r0) * p->W;
  fa.WS = (p->W + 31) / 32;
  fa.fb_bits = p->fb_bits;
  fa.seg_count = p->seg_count + fb_slot;
  fa.seg_list = p->seg_list + ((size_t)b0 * p->H + fa.r0) * fa.WS;
  fa.d_alpha = diag ? diag->alpha : nullptr;
  fa.d_beta = diag ? diag->beta : nullptr;
  if (!fa.d_alpha || !fa.d_beta) fa.d_alpha = fa.d_beta = nullptr;
  if (!fused && diag) {  // the whole planes, not only the filtered pixels
    const size_t bytes = sizeof(float) * (size_t)p->B * p->H * p->W;
    if (diag->alpha)
      FABF_CUDA(cudaMemcpyAsync(diag->alpha, p->alpha, bytes, cudaMemcpyDeviceToDevice, st), "copy alpha");
    if (diag->beta)
      FABF_CUDA(cudaMemcpyAsync(diag->beta, p->beta, bytes, cudaMemcpyDeviceToDevice, st), "copy beta");
    fa.d_alpha = fa.d_beta = nullptr;
  }
  fa.d_kappa = diag ? diag->kappa : nullptr;
  fa.d_t2n = diag ? diag->t2n : nullptr;
  fa.d_code = diag ? diag->code : nullptr;
  return launch_filter(fa, N, nb, st);
}

// FABF_FLAG_DEBUG: a fresh status word per call (count 0, first index ~0)
fabf_status_t debug_reset(Plan* p, cudaStream_t st) {
  if (!(p->flags & FABF_FLAG_DEBUG)) return FABF_OK;
  FABF_CUDA(cudaMemsetAsync(p->dbg, 0, sizeof(unsigned long long), st), "cudaMemsetAsync(dbg)");
  FABF_CUDA(cudaMemsetAsync(p->dbg + 1, 0xff, sizeof(unsigned long long), st), "cudaMemsetAsync(dbg)");
  return FABF_OK;
}

// the bounds rings of k_filter: kMaxCtaPerSm CTAs per SM, each with room for
// the largest rho this shape admits (2 rho + 1 <= min(H, W), rho <= kMaxRho)
cudaError_t alloc_ring(Plan* p) {
  int sms = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  if (e != cudaSuccess) return e;
  int rho_max = std::min(kMaxRho, (std::min(p->H, p->W) - 1) / 2);
  if (!(p->flags & FABF_FLAG_FUSED)) rho_max = std::min(rho_max, std::max(0, g_fuse_rho));
  long long per = 1;
  for (int r = 0; r <= rho_max; ++r) per = std::max(per, ring_elems_per_cta(r));
  p->ring_elems = per * kMaxCtaPerSm * sms;
  return cudaMalloc(&p->ring, sizeof(float2) * (size_t)p->ring_elems);
}

// planar staging buffers (fabf_filter_host, fabf_filter_interleaved): three
// planes of px floats, each starting 16-byte aligned
size_t staging_pitch(size_t px) { return (px + 3) & ~(size_t)3; }

// NEXT-1 launches: k_gauss on T x T tiles (T = 32 for rho <= 10, else 16 so
// that the fp64 footprint fits), then the exact weighted fallback
constexpr int kMaxGaussRho = 16;
template <int N>
fabf_status_t launch_gauss(FilterArgs& fa, int R, double nu0, cudaStream_t st) {
  const bool big = R <= 30;
  const size_t smem = big ? gauss_smem<32>(R, N) : gauss_smem<16>(R, N);
  if (smem > (size_t)kMaxDynSmem) return fail(FABF_ERR_INVALID_ARGUMENT, "rho too large for the Gaussian tiles");
  int dev = 0;
  FABF_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  {
    static bool attr_set[kMaxDevices] = {};
    std::lock_guard<std::mutex> lk(g_launch_mu);
    if (!attr_set[dev]) {
      FABF_CUDA(cudaFuncSetAttribute(k_gauss<N, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem),
                "cudaFuncSetAttribute(k_gauss)");
      FABF_CUDA(cudaFuncSetAttribute(k_gauss<N, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem),
                "cudaFuncSetAttribute(k_gauss)");
      attr_set[dev] = true;
    }
  }
  const int T = big ? 32 : 16;
  dim3 g((fa.W + T - 1) / T, (fa.H + T - 1) / T, fa.B);
  prof_mark(2, st);
  if (big)
    k_gauss<N, 32><<<g, kThreads, smem, st>>>(fa, R, nu0);
  else
    k_gauss<N, 16><<<g, kThreads, smem, st>>>(fa, R, nu0);
  ++g_launches;
  FABF_CUDA(cudaGetLastError(), "k_gauss launch");
  prof_mark(3, st);
  k_fallback_gauss<N><<<148 * 4, kThreads, 0, st>>>(fa, R, nu0);
  ++g_launches;
  FABF_CUDA(cudaGetLastError(), "k_fallback_gauss launch");
  prof_mark(4, st);
  return FABF_OK;
}

// a fresh set of fallback counters per call
fabf_status_t fallback_reset(Plan* p, int slots, cudaStream_t st) {
  FABF_CUDA(cudaMemsetAsync(p->fb_count, 0, sizeof(int) * (size_t)slots, st), "cudaMemsetAsync(fb_count)");
  FABF_CUDA(cudaMemsetAsync(p->seg_count, 0, sizeof(int) * (size_t)slots, st), "cudaMemsetAsync(seg_count)");
  p->fb_slots = slots;
  return FABF_OK;
}

fabf_status_t filter_impl(Plan* p, const float* img, const float* theta, const float* sigma,
                          int rho, int N, float* out, const fabf_diag_t* diag, cudaStream_t st) {
  fabf_status_t s = validate_filter(p, img, theta, sigma, rho, N, out);
  if (s != FABF_OK) return s;
  g_launches = 0;
  struct Record {
    Plan* p;
    ~Record() { p->launches = g_launches; }
  } rec{p};
  s = debug_reset(p, st);
  if (s != FABF_OK) return s;
  s = fallback_reset(p, 1, st);
  if (s != FABF_OK) return s;
  return filter_band(p, img, theta, sigma, rho, N, out, diag, 0, p->B, 0,
                     (p->H + kBT - 1) / kBT, 0, st);
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
  if (flags & ~(unsigned)(FABF_FLAG_LITERAL | FABF_FLAG_CLAMP | FABF_FLAG_DEBUG | FABF_FLAG_FUSED))
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
      (e = cudaMalloc(&p->hmm, px * sizeof(float2))) != cudaSuccess ||
      (e = cudaMalloc(&p->blkmm, sizeof(float2) * (size_t)batch * ((height + kBT - 1) / kBT) *
                                     ((width + kBT - 1) / kBT))) != cudaSuccess ||
      (e = cudaMalloc(&p->fb_count, sizeof(int) * (size_t)batch * Plan::kMaxBandsPlan)) != cudaSuccess ||
      (e = cudaMalloc(&p->fb_list, px * sizeof(int))) != cudaSuccess ||
      (e = cudaMalloc(&p->fb_bits, sizeof(unsigned) * (size_t)batch * height * ((width + 31) / 32))) != cudaSuccess ||
      (e = cudaMemset(p->fb_bits, 0, sizeof(unsigned) * (size_t)batch * height * ((width + 31) / 32))) != cudaSuccess ||
      (e = cudaMalloc(&p->seg_list, sizeof(int) * (size_t)batch * height * ((width + 31) / 32))) != cudaSuccess ||
      (e = cudaMalloc(&p->seg_count, sizeof(int) * (size_t)batch * Plan::kMaxBandsPlan)) != cudaSuccess ||
      (e = alloc_ring(p)) != cudaSuccess ||
      ((flags & FABF_FLAG_DEBUG) &&
       (e = cudaMalloc(&p->dbg, 2 * sizeof(unsigned long long))) != cudaSuccess)) {
    fabf_destroy(p);
    return cuda_fail(e, "cudaMalloc(plan workspace)");
  }
  if (p->dbg) {  // no call yet: count 0, no index
    const unsigned long long init[2] = {0ull, ~0ull};
    if ((e = cudaMemcpy(p->dbg, init, sizeof(init), cudaMemcpyHostToDevice)) != cudaSuccess) {
      fabf_destroy(p);
      return cuda_fail(e, "cudaMemcpy(debug word)");
    }
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
  return launch_bounds(p, img, rho, alpha, beta, 0, p->B, 0, (p->H + kBT - 1) / kBT,
                       (cudaStream_t)stream);
}

fabf_status_t fabf_filter_host(fabf_plan_t plan, const float* img, const float* theta,
                               const float* sigma, int rho, int N, float* out, void* stream) {
  // Host buffers in and out, pipelined by row bands (multiples of the 64-row
  // bounds tiles): band k's inputs go up on a copy stream, its kernels run on
  // `stream` once bands k and k+1 (its rho-row halo) are resident, and its
  // output comes back on a second copy stream, so the PCIe transfers overlap
  // each other and the kernels.
  Plan* p = reinterpret_cast<Plan*>(plan);
  if (!p) return fail(FABF_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (!img || !theta || !sigma || !out) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  {
    fabf_status_t s0 = check_plan_device(p);
    if (s0 != FABF_OK) return s0;
  }
  const size_t px = (size_t)p->B * p->H * p->W, bytes = px * sizeof(float);
  if (!p->h_in) {
    cudaError_t e;
    if ((e = cudaMalloc(&p->h_in, 3 * sizeof(float) * staging_pitch(px))) != cudaSuccess)
      return cuda_fail(e, "cudaMalloc(staging)");
    if ((e = cudaMalloc(&p->h_out, bytes)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
  }
  if (!p->cs_in) {
    FABF_CUDA(cudaStreamCreateWithFlags(&p->cs_in, cudaStreamNonBlocking), "cudaStreamCreate");
    FABF_CUDA(cudaStreamCreateWithFlags(&p->cs_out, cudaStreamNonBlocking), "cudaStreamCreate");
    for (int i = 0; i < kMaxBands + 1; ++i) {
      FABF_CUDA(cudaEventCreateWithFlags(&p->ev_in[i], cudaEventDisableTiming), "cudaEventCreate");
      FABF_CUDA(cudaEventCreateWithFlags(&p->ev_done[i], cudaEventDisableTiming), "cudaEventCreate");
    }
  }
  g_launches = 0;
  struct Record {
    Plan* p;
    ~Record() { p->launches = g_launches; }
  } rec{p};
  float* dimg = p->h_in;
  float* dth = p->h_in + staging_pitch(px);
  float* dsg = p->h_in + 2 * staging_pitch(px);
  fabf_status_t s = validate_filter(p, dimg, dth, dsg, rho, N, p->h_out);
  if (s != FABF_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  s = debug_reset(p, st);
  if (s != FABF_OK) return s;
  s = fallback_reset(p, p->B * kMaxBands, st);
  if (s != FABF_OK) return s;
  const int H = p->H, W = p->W;
  const int ntile = (H + kBT - 1) / kBT;
  // bands of whole tiles, each at least rho + 1 rows (a band's halo then lies
  // in its two neighbours).  The last band is the smallest allowed (the
  // pipeline's tail after the final upload is its kernels plus its download);
  // the others split the remaining tiles evenly.
  const int minT = (rho + 1 + kBT - 1) / kBT;  // tiles for rho + 1 rows
  int nband = std::min(g_host_bands, std::max(1, ntile / 2));  // 2+ tiles per band on average
  int lastT = minT;
  while (nband > 1 && ((ntile - lastT) / (nband - 1) < minT || ntile - lastT < nband - 1)) --nband;
  if (nband == 1) lastT = ntile;
  int tb[kMaxBands + 1];
  for (int k = 0; k < nband; ++k) tb[k] = (int)((long long)(ntile - lastT) * k / std::max(1, nband - 1));
  tb[nband] = ntile;
  // the copy-in stream starts after work already queued on `stream`
  FABF_CUDA(cudaEventRecord(p->ev_in[kMaxBands], st), "cudaEventRecord");
  FABF_CUDA(cudaStreamWaitEvent(p->cs_in, p->ev_in[kMaxBands], 0), "cudaStreamWaitEvent");
  for (int b = 0; b < p->B; ++b) {
    const size_t plane = (size_t)b * H * W;
    auto rows = [&](int k, size_t& o, size_t& nbytes) {
      const int r0 = tb[k] * kBT, r1 = std::min(H, tb[k + 1] * kBT);
      o = plane + (size_t)r0 * W;
      nbytes = sizeof(float) * (size_t)(r1 - r0) * W;
    };
    size_t o, nbytes;
    rows(0, o, nbytes);
    FABF_CUDA(cudaMemcpyAsync(dimg + o, img + o, nbytes, cudaMemcpyHostToDevice, p->cs_in), "H2D img");
    for (int k = 0; k < nband; ++k) {
      // upload order f_{k+1}, theta_k, sigma_k: band k's kernels can start as
      // soon as its own parameters are up (its lower halo, f_{k+1}, came first)
      if (k + 1 < nband) {
        rows(k + 1, o, nbytes);
        FABF_CUDA(cudaMemcpyAsync(dimg + o, img + o, nbytes, cudaMemcpyHostToDevice, p->cs_in), "H2D img");
      }
      rows(k, o, nbytes);
      FABF_CUDA(cudaMemcpyAsync(dth + o, theta + o, nbytes, cudaMemcpyHostToDevice, p->cs_in), "H2D theta");
      FABF_CUDA(cudaMemcpyAsync(dsg + o, sigma + o, nbytes, cudaMemcpyHostToDevice, p->cs_in), "H2D sigma");
      FABF_CUDA(cudaEventRecord(p->ev_in[k], p->cs_in), "cudaEventRecord");
      FABF_CUDA(cudaStreamWaitEvent(st, p->ev_in[k], 0), "cudaStreamWaitEvent");
      s = filter_band(p, dimg, dth, dsg, rho, N, p->h_out, nullptr, b, 1, tb[k], tb[k + 1], b * kMaxBands + k,
                      st);
      if (s != FABF_OK) return s;
      FABF_CUDA(cudaEventRecord(p->ev_done[k], st), "cudaEventRecord");
      FABF_CUDA(cudaStreamWaitEvent(p->cs_out, p->ev_done[k], 0), "cudaStreamWaitEvent");
      FABF_CUDA(cudaMemcpyAsync(out + o, p->h_out + o, nbytes, cudaMemcpyDeviceToHost, p->cs_out), "D2H out");
    }
  }
  FABF_CUDA(cudaStreamSynchronize(p->cs_out), "cudaStreamSynchronize");
  FABF_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  return FABF_OK;
}

fabf_status_t fabf_filter_gauss(fabf_plan_t plan, const float* img, const float* theta, const float* sigma,
                                int rho, int N, float* out, void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  if (!p) return fail(FABF_ERR_INVALID_ARGUMENT, "plan is NULL");
  const int R = 3 * rho;
  if (rho < 0 || rho > kMaxGaussRho) return fail(FABF_ERR_INVALID_ARGUMENT, "Gaussian omega: 0 <= rho <= 16");
  fabf_status_t s = validate_filter(p, img, theta, sigma, R, N, out);  // the window is [-3 rho, 3 rho]^2
  if (s != FABF_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  p->last_stream = st;
  g_launches = 0;
  struct Record {
    Plan* p;
    ~Record() { p->launches = g_launches; }
  } rec{p};
  s = fallback_reset(p, 1, st);
  if (s != FABF_OK) return s;
  // omega's 1-D factor and sum omega = (sum_d g(d))^2 = nu_0 (eq.(4))
  double g[2 * 48 + 1] = {}, gs = 0.0;
  for (int d = -R; d <= R; ++d) gs += (g[d + R] = rho > 0 ? std::exp(-(double)d * d / (2.0 * rho * rho)) : 1.0);
  FABF_CUDA(cudaMemcpyToSymbolAsync(c_gw, g, sizeof(g), 0, cudaMemcpyHostToDevice, st), "c_gw");
  s = launch_bounds(p, img, R, p->alpha, p->beta, 0, p->B, 0, (p->H + kBT - 1) / kBT, st);  // step a1 on the box of R
  if (s != FABF_OK) return s;
  FilterArgs fa = {};
  fa.img = img;
  fa.theta = theta;
  fa.sigma = sigma;
  fa.alpha = fa.alpha_w = p->alpha;
  fa.beta = fa.beta_w = p->beta;
  fa.out = out;
  fa.B = p->B;
  fa.H = p->H;
  fa.W = p->W;
  fa.rho = R;
  fa.flags = p->flags;
  fa.flag_root = N > 0 ? std::pow(2.0, (double)kFlagBits / N) : 1e300;  // direct (FIR) sums: magnitude 1
  fa.fb_count = p->fb_count;
  fa.fb_list = p->fb_list;
  const double nu0 = gs * gs;
  switch (N) {
#define FABF_GAUSS_CASE(NV) \
  case NV: s = launch_gauss<NV>(fa, R, nu0, st); break;
    FABF_GAUSS_CASE(0) FABF_GAUSS_CASE(1) FABF_GAUSS_CASE(2) FABF_GAUSS_CASE(3) FABF_GAUSS_CASE(4)
    FABF_GAUSS_CASE(5) FABF_GAUSS_CASE(6) FABF_GAUSS_CASE(7) FABF_GAUSS_CASE(8) FABF_GAUSS_CASE(9)
    FABF_GAUSS_CASE(10)
#undef FABF_GAUSS_CASE
    default: return fail(FABF_ERR_UNSUPPORTED, "N > FABF_MAX_N");
  }
  return s;
}

fabf_status_t fabf_filter_mozerov(fabf_plan_t plan, const float* img, const float* theta,
                                  const float* sigma, int rho, float* out, void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  fabf_status_t s = validate_filter(p, img, theta, sigma, rho, 0, out);
  if (s != FABF_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const bool small = 32 + 2 * rho <= 128;  // 32 x 32 tiles up to rho = 48, else 16 x 16
  const int T = small ? 32 : 16, FS = T + 2 * rho;
  const size_t smem = sizeof(double) * FS * T + sizeof(float) * FS * FS;
  if (smem > (size_t)kMaxDynSmem) return fail(FABF_ERR_INVALID_ARGUMENT, "rho too large for shared memory");
  {
    static bool attr_set[kMaxDevices] = {};
    std::lock_guard<std::mutex> lk(g_launch_mu);
    if (!attr_set[p->device]) {
      FABF_CUDA(cudaFuncSetAttribute(k_mozerov<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem),
                "cudaFuncSetAttribute(k_mozerov)");
      FABF_CUDA(cudaFuncSetAttribute(k_mozerov<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem),
                "cudaFuncSetAttribute(k_mozerov)");
      attr_set[p->device] = true;
    }
  }
  dim3 g((p->W + T - 1) / T, (p->H + T - 1) / T, p->B);
  if (small)
    k_mozerov<32><<<g, kThreads, smem, st>>>(img, theta, sigma, out, p->H, p->W, rho, p->flags);
  else
    k_mozerov<16><<<g, kThreads, smem, st>>>(img, theta, sigma, out, p->H, p->W, rho, p->flags);
  FABF_CUDA(cudaGetLastError(), "k_mozerov launch");
  p->launches = 1;
  p->last_stream = st;
  return FABF_OK;
}

fabf_status_t fabf_sharpen_maps(fabf_plan_t plan, const float* img, int rho, const fabf_sharpen_t* prm,
                                float* theta, float* sigma, void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  fabf_status_t s = validate_common(p, rho);
  if (s != FABF_OK) return s;
  if (!img || !theta || !sigma || !prm) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!(prm->log_scale > 0.0f) || !(prm->log_sat > 0.0f) || !(prm->sigma_lo > 0.0f) ||
      !(prm->sigma_hi >= prm->sigma_lo))
    return fail(FABF_ERR_INVALID_ARGUMENT, "sharpen parameters: log_scale, log_sat, sigma_lo > 0, sigma_hi >= sigma_lo");
  const int rl = (int)ceilf(4.0f * prm->log_scale);
  if (rl > kMaxLogR || 2 * rl + 1 > p->H || 2 * rl + 1 > p->W)
    return fail(FABF_ERR_INVALID_ARGUMENT, "log_scale too large (ceil(4 s) <= 16 and its window inside the image)");
  const size_t bytes = sizeof(float) * (size_t)p->B * p->H * p->W;
  if (overlaps(theta, bytes, img, bytes) || overlaps(sigma, bytes, img, bytes) || overlaps(theta, bytes, sigma, bytes))
    return fail(FABF_ERR_INVALID_ARGUMENT, "outputs overlap");
  constexpr int T = 32;
  const int R = std::max(rho, rl), FS = T + 2 * R;
  const size_t smem = sizeof(double) * (T + 2 * rho) * T + sizeof(float) * ((size_t)FS * FS + 2 * (T + 2 * rl) * T);
  if (smem > (size_t)kMaxDynSmem) return fail(FABF_ERR_INVALID_ARGUMENT, "rho too large for the map producer");
  cudaStream_t st = (cudaStream_t)stream;
  {  // taps (host, double -> float), per call on the stream
    float hg[2 * kMaxLogR + 1] = {}, hg2[2 * kMaxLogR + 1] = {};
    double g[2 * kMaxLogR + 1], gs = 0.0, sc = prm->log_scale;
    for (int k = -rl; k <= rl; ++k) gs += (g[k + rl] = std::exp(-0.5 * k * k / (sc * sc)));
    for (int k = -rl; k <= rl; ++k) {
      hg[k + rl] = (float)(g[k + rl] / gs);
      hg2[k + rl] = (float)(((double)k * k - sc * sc) / (sc * sc * sc * sc) * g[k + rl] / gs);
    }
    FABF_CUDA(cudaMemcpyToSymbolAsync(c_log_g, hg, sizeof(hg), 0, cudaMemcpyHostToDevice, st), "taps");
    FABF_CUDA(cudaMemcpyToSymbolAsync(c_log_g2, hg2, sizeof(hg2), 0, cudaMemcpyHostToDevice, st), "taps");
  }
  {
    static bool attr_set[kMaxDevices] = {};
    std::lock_guard<std::mutex> lk(g_launch_mu);
    if (!attr_set[p->device]) {
      FABF_CUDA(cudaFuncSetAttribute(k_sharpen_maps<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem),
                "cudaFuncSetAttribute(k_sharpen_maps)");
      attr_set[p->device] = true;
    }
  }
  dim3 g((p->W + T - 1) / T, (p->H + T - 1) / T, p->B);
  k_sharpen_maps<T><<<g, kThreads, smem, st>>>(img, theta, sigma, p->H, p->W, rho, rl, prm->sigma_lo,
                                               prm->sigma_hi, 1.0f / prm->log_sat);
  FABF_CUDA(cudaGetLastError(), "k_sharpen_maps launch");
  ++g_launches;
  return FABF_OK;
}

fabf_status_t fabf_filter_sharpen(fabf_plan_t plan, const float* img, int rho, int N, const fabf_sharpen_t* prm,
                                  float* out, void* stream) {
  // the application pipeline: maps from f (plan-owned planes), then Algorithm 1
  Plan* p = reinterpret_cast<Plan*>(plan);
  if (!p) return fail(FABF_ERR_INVALID_ARGUMENT, "plan is NULL");
  {
    fabf_status_t s0 = check_plan_device(p);
    if (s0 != FABF_OK) return s0;
  }
  const size_t px = (size_t)p->B * p->H * p->W;
  if (!p->h_in) {  // planar staging (shared with fabf_filter_host), allocated on first use
    cudaError_t e;
    if ((e = cudaMalloc(&p->h_in, 3 * sizeof(float) * staging_pitch(px))) != cudaSuccess)
      return cuda_fail(e, "cudaMalloc(staging)");
    if ((e = cudaMalloc(&p->h_out, px * sizeof(float))) != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
  }
  float* th = p->h_in + staging_pitch(px);
  float* sg = p->h_in + 2 * staging_pitch(px);
  g_launches = 0;
  fabf_status_t s = fabf_sharpen_maps(plan, img, rho, prm, th, sg, stream);
  if (s != FABF_OK) return s;
  const int maps = g_launches;
  s = filter_impl(p, img, th, sg, rho, N, out, nullptr, (cudaStream_t)stream);
  if (s != FABF_OK) return s;
  p->launches += maps;
  return FABF_OK;
}

namespace {
fabf_status_t ensure_staging(Plan* p) {  // planar staging (shared with fabf_filter_host), on first use
  if (p->h_in) return FABF_OK;
  const size_t px = (size_t)p->B * p->H * p->W;
  cudaError_t e;
  if ((e = cudaMalloc(&p->h_in, 3 * sizeof(float) * staging_pitch(px))) != cudaSuccess)
    return cuda_fail(e, "cudaMalloc(staging)");
  if ((e = cudaMalloc(&p->h_out, px * sizeof(float))) != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
  return FABF_OK;
}

fabf_status_t texture_maps_impl(Plan* p, const float* img, const fabf_texture_t* prm, float* sigma,
                                float* sigma2, float* mrtv, cudaStream_t st) {
  if (!img || !sigma || !prm) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (prm->patch < 0 || prm->patch > kMaxPatch || 2 * prm->patch + 1 > p->H || 2 * prm->patch + 1 > p->W)
    return fail(FABF_ERR_INVALID_ARGUMENT, "patch must be in [0, 16] and its window inside the image");
  if (!(prm->mrtv_sat > 0.0f) || !(prm->eps > 0.0f) || !(prm->sigma_lo > 0.0f) || !(prm->sigma_hi >= prm->sigma_lo) ||
      !(prm->second_scale > 0.0f))
    return fail(FABF_ERR_INVALID_ARGUMENT,
                "texture parameters: mrtv_sat, eps, sigma_lo, second_scale > 0, sigma_hi >= sigma_lo");
  const size_t bytes = sizeof(float) * (size_t)p->B * p->H * p->W;
  if (overlaps(sigma, bytes, img, bytes) || (mrtv && (overlaps(mrtv, bytes, img, bytes) || overlaps(mrtv, bytes, sigma, bytes))))
    return fail(FABF_ERR_INVALID_ARGUMENT, "outputs overlap");
  constexpr int T = 32;
  const int FS = T + 2 * prm->patch;
  const size_t smem = (sizeof(double) + sizeof(float)) * ((size_t)FS * FS + 2 * (size_t)FS * T);
  {
    static bool attr_set[kMaxDevices] = {};
    std::lock_guard<std::mutex> lk(g_launch_mu);
    if (!attr_set[p->device]) {
      FABF_CUDA(cudaFuncSetAttribute(k_texture_maps<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem),
                "cudaFuncSetAttribute(k_texture_maps)");
      attr_set[p->device] = true;
    }
  }
  dim3 g((p->W + T - 1) / T, (p->H + T - 1) / T, p->B);
  k_texture_maps<T><<<g, kThreads, smem, st>>>(img, sigma, sigma2, mrtv, p->H, p->W, prm->patch, prm->sigma_lo,
                                               prm->sigma_hi, 1.0 / (double)prm->mrtv_sat, (double)prm->eps,
                                               prm->second_scale);
  FABF_CUDA(cudaGetLastError(), "k_texture_maps launch");
  ++g_launches;
  return FABF_OK;
}
}  // namespace

fabf_status_t fabf_texture_maps(fabf_plan_t plan, const float* img, const fabf_texture_t* prm, float* sigma,
                                float* mrtv, void* stream) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  fabf_status_t s = validate_common(p, 0);
  if (s != FABF_OK) return s;
  return texture_maps_impl(p, img, prm, sigma, nullptr, mrtv, (cudaStream_t)stream);
}

namespace {
// Algorithm 1 three times -- theta = f with the sigma map, again on
// the result with sigma scaled by second_scale (the same map), then the
// sharpening rule of P:620-630 on that.  The map comes from k_texture_maps
// (tprm) or from the caller (sigma_map, second_scale).
fabf_status_t texture_passes(Plan* p, const float* img, int rho, int N, const fabf_texture_t* tprm,
                             const float* sigma_map, float second_scale, int rho_sharpen,
                             const fabf_sharpen_t* sprm, float* out, float* pass1, float* pass2, cudaStream_t st) {
  fabf_status_t s = validate_common(p, rho);
  if (s != FABF_OK) return s;
  if (!img || !out || !sprm || (!tprm && !sigma_map)) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  const size_t px = (size_t)p->B * p->H * p->W, bytes = px * sizeof(float);
  if ((pass1 && (overlaps(pass1, bytes, img, bytes) || overlaps(pass1, bytes, out, bytes))) ||
      (pass2 && (overlaps(pass2, bytes, img, bytes) || overlaps(pass2, bytes, out, bytes))) ||
      (pass1 && pass2 && overlaps(pass1, bytes, pass2, bytes)))
    return fail(FABF_ERR_INVALID_ARGUMENT, "pass1 / pass2 overlap another buffer");
  if (sigma_map && (!(second_scale > 0.0f) || !aligned16(sigma_map) || overlaps(sigma_map, bytes, out, bytes) ||
                    (pass1 && overlaps(sigma_map, bytes, pass1, bytes)) ||
                    (pass2 && overlaps(sigma_map, bytes, pass2, bytes))))
    return fail(FABF_ERR_INVALID_ARGUMENT, "sigma map: second_scale > 0, 16-byte aligned, no overlap with an output");
  s = ensure_staging(p);
  if (s != FABF_OK) return s;
  const size_t pitch = staging_pitch(px);
  float* g1 = pass1 ? pass1 : p->h_in;
  float* g2 = pass2 ? pass2 : p->h_out;
  float* pa = p->h_in + pitch;      // sigma, then theta of the sharpening pass
  float* pb = p->h_in + 2 * pitch;  // second_scale * sigma, then sigma of the sharpening pass
  g_launches = 0;
  const float* sg1 = pa;
  if (sigma_map) {
    sg1 = sigma_map;
    const int grid = (int)std::min<long long>(148LL * 8, ((long long)px + kThreads - 1) / kThreads);
    k_scale<<<grid, kThreads, 0, st>>>(sigma_map, pb, second_scale, (long long)px);
    FABF_CUDA(cudaGetLastError(), "k_scale launch");
    ++g_launches;
  } else {
    s = texture_maps_impl(p, img, tprm, pa, pb, nullptr, st);
    if (s != FABF_OK) return s;
  }
  int total = g_launches;
  s = filter_impl(p, img, img, sg1, rho, N, g1, nullptr, st);
  if (s != FABF_OK) return s;
  total += p->launches;
  s = filter_impl(p, g1, g1, pb, rho, N, g2, nullptr, st);
  if (s != FABF_OK) return s;
  total += p->launches;
  g_launches = 0;
  s = fabf_sharpen_maps(p, g2, rho_sharpen, sprm, pa, pb, st);
  if (s != FABF_OK) return s;
  total += g_launches;
  s = filter_impl(p, g2, pa, pb, rho_sharpen, N, out, nullptr, st);
  if (s != FABF_OK) return s;
  p->launches += total;
  return FABF_OK;
}
}  // namespace

fabf_status_t fabf_filter_texture(fabf_plan_t plan, const float* img, int rho, int N, const fabf_texture_t* tprm,
                                  int rho_sharpen, const fabf_sharpen_t* sprm, float* out, float* pass1,
                                  float* pass2, void* stream) {
  if (!tprm) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  return texture_passes(reinterpret_cast<Plan*>(plan), img, rho, N, tprm, nullptr, 0.0f, rho_sharpen, sprm, out,
                        pass1, pass2, (cudaStream_t)stream);
}

fabf_status_t fabf_filter_texture_map(fabf_plan_t plan, const float* img, const float* sigma_map,
                                      float second_scale, int rho, int N, int rho_sharpen,
                                      const fabf_sharpen_t* sprm, float* out, float* pass1, float* pass2,
                                      void* stream) {
  if (!sigma_map) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  return texture_passes(reinterpret_cast<Plan*>(plan), img, rho, N, nullptr, sigma_map, second_scale, rho_sharpen,
                        sprm, out, pass1, pass2, (cudaStream_t)stream);
}

fabf_status_t fabf_filter_interleaved(fabf_plan_t plan, const float* img, const float* theta,
                                      const float* sigma, int channels, int rho, int N, float* out,
                                      void* stream) {
  // colour / multi-channel: the plan's batch counts planes, B = images x
  // channels; inputs and output are B/C x H x W x C interleaved device buffers
  Plan* p = reinterpret_cast<Plan*>(plan);
  if (!p) return fail(FABF_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (channels < 1 || p->B % channels != 0)
    return fail(FABF_ERR_INVALID_ARGUMENT, "channels must divide the plan's batch (images x channels)");
  if (!img || !theta || !sigma || !out) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  {
    fabf_status_t s0 = check_plan_device(p);
    if (s0 != FABF_OK) return s0;
  }
  const size_t px = (size_t)p->B * p->H * p->W, bytes = px * sizeof(float);
  if (overlaps(out, bytes, img, bytes) || overlaps(out, bytes, theta, bytes) || overlaps(out, bytes, sigma, bytes))
    return fail(FABF_ERR_INVALID_ARGUMENT, "out overlaps an input");
  if (!p->h_in) {  // planar staging (shared with fabf_filter_host), allocated on first use
    cudaError_t e;
    if ((e = cudaMalloc(&p->h_in, 3 * sizeof(float) * staging_pitch(px))) != cudaSuccess)
      return cuda_fail(e, "cudaMalloc(staging)");
    if ((e = cudaMalloc(&p->h_out, bytes)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
  }
  cudaStream_t st = (cudaStream_t)stream;
  const long long HW = (long long)p->H * p->W, total = (long long)px;
  const int grid = (int)std::min<long long>(148LL * 8, (total + kThreads - 1) / kThreads);
  const size_t pxp = staging_pitch(px);
  k_deinterleave<<<grid, kThreads, 0, st>>>(img, theta, sigma, p->h_in, p->h_in + pxp, p->h_in + 2 * pxp, HW,
                                             channels, total);
  FABF_CUDA(cudaGetLastError(), "k_deinterleave launch");
  fabf_status_t s = filter_impl(p, p->h_in, p->h_in + pxp, p->h_in + 2 * pxp, rho, N, p->h_out, nullptr, st);
  if (s != FABF_OK) return s;
  k_interleave<<<grid, kThreads, 0, st>>>(p->h_out, out, HW, channels, total);
  FABF_CUDA(cudaGetLastError(), "k_interleave launch");
  p->launches += 2;  // (filter_impl recorded its own kernels)
  return FABF_OK;
}

fabf_status_t fabf_last_fallback_count(fabf_plan_t plan, long long* count) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  if (!p || !count) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  std::vector<int> c((size_t)std::max(1, p->fb_slots), 0);
  if (p->fb_slots > 0) {
    FABF_CUDA(cudaMemcpyAsync(c.data(), p->fb_count, sizeof(int) * (size_t)p->fb_slots, cudaMemcpyDeviceToHost,
                              (cudaStream_t)p->last_stream),
              "read fallback count");
    FABF_CUDA(cudaStreamSynchronize((cudaStream_t)p->last_stream), "cudaStreamSynchronize");
  }
  long long total = 0;
  for (int v : c) total += v;
  *count = total;
  return FABF_OK;
}

fabf_status_t fabf_last_launch_count(fabf_plan_t plan, int* count) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  if (!p || !count) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  *count = p->launches;
  return FABF_OK;
}

fabf_status_t fabf_debug_status(fabf_plan_t plan, long long* bad_count, long long* first_bad) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  if (!p || !bad_count || !first_bad) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!(p->flags & FABF_FLAG_DEBUG)) return fail(FABF_ERR_INVALID_ARGUMENT, "plan made without FABF_FLAG_DEBUG");
  unsigned long long w[2] = {0ull, ~0ull};
  FABF_CUDA(cudaMemcpyAsync(w, p->dbg, sizeof(w), cudaMemcpyDeviceToHost, (cudaStream_t)p->last_stream),
            "read debug word");
  FABF_CUDA(cudaStreamSynchronize((cudaStream_t)p->last_stream), "cudaStreamSynchronize");
  *bad_count = (long long)w[0];
  *first_bad = w[0] ? (long long)w[1] : -1;
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

fabf_status_t fabf_filter_events(fabf_plan_t plan, const float* img, const float* theta,
                                 const float* sigma, int rho, int N, float* out, void* stream,
                                 void* const events[5]) {
  if (!events) return fail(FABF_ERR_INVALID_ARGUMENT, "events is NULL");
  cudaEvent_t ev[5];
  for (int i = 0; i < 5; ++i) {
    if (!events[i]) return fail(FABF_ERR_INVALID_ARGUMENT, "NULL event");
    ev[i] = (cudaEvent_t)events[i];
  }
  g_prof_ev = ev;
  fabf_status_t s = filter_impl(reinterpret_cast<Plan*>(plan), img, theta, sigma, rho, N, out,
                                nullptr, (cudaStream_t)stream);
  g_prof_ev = nullptr;
  return s;
}

fabf_status_t fabf_destroy(fabf_plan_t plan) {
  Plan* p = reinterpret_cast<Plan*>(plan);
  if (!p) return FABF_OK;
  cudaFree(p->alpha);
  cudaFree(p->beta);
  cudaFree(p->hmm);
  cudaFree(p->blkmm);
  cudaFree(p->ring);
  cudaFree(p->fb_count);
  cudaFree(p->fb_list);
  cudaFree(p->fb_bits);
  cudaFree(p->seg_list);
  cudaFree(p->seg_count);
  cudaFree(p->dbg);
  cudaFree(p->h_in);
  cudaFree(p->h_out);
  if (p->cs_in) {
    cudaStreamSynchronize(p->cs_in);
    cudaStreamSynchronize(p->cs_out);
    cudaStreamDestroy(p->cs_in);
    cudaStreamDestroy(p->cs_out);
    for (int i = 0; i < kMaxBands + 1; ++i) {
      cudaEventDestroy(p->ev_in[i]);
      cudaEventDestroy(p->ev_done[i]);
    }
  }
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

#ifdef FABF_EXP_TIMERS
// experiments: read (and reset) the per-phase clock64 sums of k_filter
int fabf_exp_timers(unsigned long long out[8]) {
  if (cudaDeviceSynchronize() != cudaSuccess) return 1;
  if (cudaMemcpyFromSymbol(out, g_exp_timers, 8 * sizeof(unsigned long long)) != cudaSuccess) return 1;
  const unsigned long long z[8] = {};
  return cudaMemcpyToSymbol(g_exp_timers, z, sizeof(z)) != cudaSuccess;
}
#endif

int fabf_version(void) { return FABF_VERSION; }

}  // extern "C"
