// latbench.cu -- dependent-chain latencies on the B200 (one warp)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat_dfma(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_dadd(double* out, long long* cyc, int iters, double a) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x = x + a;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_ffma(float* out, long long* cyc, int iters, float a, float b) {
  float x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x = fmaf(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_shfl(double* out, long long* cyc, int iters) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_lds(double* out, long long* cyc, int iters) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) s[i] = (i + 1) & 1023;
  __syncwarp();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) p = s[p];
  }
  long long t1 = clock64();
  out[threadIdx.x] = p; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_rcp(double* out, long long* cyc, int iters) {
  double x = 1.5 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x = __drcp_rn(x) + 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* d; float* f; long long* c; long long h;
  cudaMalloc(&d, 1024); cudaMalloc(&f, 1024); cudaMalloc(&c, 8);
  const int it = 1000; const double n = it * 32.0;
  lat_dfma<<<1, 32>>>(d, c, it, 0.999, 1e-3); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DFMA %.2f\n", h / n);
  lat_dadd<<<1, 32>>>(d, c, it, 1e-3); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DADD %.2f\n", h / n);
  lat_ffma<<<1, 32>>>(f, c, it, 0.999f, 1e-3f); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("FFMA %.2f\n", h / n);
  lat_shfl<<<1, 32>>>(d, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("SHFL.f64+DADD %.2f\n", h / n);
  lat_lds<<<1, 32>>>(d, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("LDS %.2f\n", h / n);
  lat_rcp<<<1, 32>>>(d, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DRCP_RN+DADD %.2f\n", h / n);
  return 0;
}
