// microbench.cu -- measure the B200 pipe peaks the roofline needs and that
// MEASURED_PEAKS.json does not hold: FP64 FMA, FP32 FMA and MUFU.EX2 throughput.
// Each thread runs 8 independent FMA chains; grid = 148 x 8 CTAs of 256 threads.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void fma_chain(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void ex2_chain(float* out, int iters) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = exp2f(-x0) ; x1 = exp2f(-x1); x2 = exp2f(-x2); x3 = exp2f(-x3);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}

template <typename F>
float time_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  const int blocks = sms * 8, threads = 256, iters = 2000;
  double* dd; float* df; cudaMalloc(&dd, blocks * threads * 8); cudaMalloc(&df, blocks * threads * 4);
  double n_fma = (double)blocks * threads * iters * 16 * 8;
  float t64 = time_ms([&] { fma_chain<double><<<blocks, threads>>>(dd, iters, 0.999999, 1e-7); });
  float t32 = time_ms([&] { fma_chain<float><<<blocks, threads>>>(df, iters, 0.999999f, 1e-7f); });
  double n_ex2 = (double)blocks * threads * iters * 16 * 4;
  float tex = time_ms([&] { ex2_chain<<<blocks, threads>>>(df, iters / 4); });
  n_ex2 /= 4;
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d, "
         "\"fp64_fma_per_s\": %.4e, \"fp64_tflops\": %.3f, "
         "\"fp32_fma_per_s\": %.4e, \"fp32_tflops\": %.3f, \"mufu_ex2_per_s\": %.4e}\n",
         p.name, sms, p.clockRate, n_fma / (t64 * 1e-3), 2 * n_fma / (t64 * 1e-3) / 1e12,
         n_fma / (t32 * 1e-3), 2 * n_fma / (t32 * 1e-3) / 1e12, n_ex2 / (tex * 1e-3));
  return 0;
}
