// Latency microbenchmarks on the B200 (one warp, clock64): dependent fp64
// add / fma chains, f32->f64 conversion, and pointer chases that hit L1,
// L2 and DRAM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_dadd(double* out, long long* cyc, double a, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + a; x = x + a; x = x + a; x = x + a; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dfma(double* out, long long* cyc, double a, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __fma_rn(x, a, a); x = __fma_rn(x, a, a); x = __fma_rn(x, a, a); x = __fma_rn(x, a, a); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_f2f(double* out, long long* cyc, float a, int n) {
  float x = a; double y = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { y = (double)x; x = (float)(y * 1.0000001); y = (double)x; x = (float)(y * 1.0000001); }
  long long t1 = clock64();
  out[threadIdx.x] = y; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_chase(const int* __restrict__ p, int start, int n, long long* cyc, int* sink) {
  int j = start;
  for (int i = 0; i < 64; ++i) j = __ldg(p + j);  // warm
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) j = __ldg(p + j);
  long long t1 = clock64();
  sink[threadIdx.x] = j; if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* dout; long long* dcyc; int* sink;
  cudaMalloc(&dout, 1024 * 8); cudaMalloc(&dcyc, 8); cudaMalloc(&sink, 4096);
  long long cyc;
  int n = 4096;
  k_dadd<<<1, 32>>>(dout, dcyc, 1e-9, n); cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
  k_dadd<<<1, 32>>>(dout, dcyc, 1e-9, n); cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", (double)cyc / (4.0 * n));
  k_dfma<<<1, 32>>>(dout, dcyc, 0.5, n); cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)cyc / (4.0 * n));
  k_f2f<<<1, 32>>>(dout, dcyc, 0.5f, n); cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
  printf("F2F.F64.F32 + DMUL + F2F.F32.F64 round trip: %.2f cycles\n", (double)cyc / (2.0 * n));
  size_t sizes[] = {16 << 10, 128 << 10, 8 << 20, 64 << 20, 1024ull << 20};
  for (size_t bytes : sizes) {
    size_t m = bytes / 4;
    std::vector<int> h(m);
    // random cyclic permutation with 128-B stride granularity
    size_t lines = m / 32;
    std::vector<size_t> perm(lines);
    for (size_t i = 0; i < lines; ++i) perm[i] = i;
    srand(1);
    for (size_t i = lines - 1; i > 0; --i) { size_t k = rand() % (i + 1); std::swap(perm[i], perm[k]); }
    for (size_t i = 0; i < lines; ++i) h[perm[i] * 32] = (int)(perm[(i + 1) % lines] * 32);
    int* d; cudaMalloc(&d, bytes); cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
    int steps = 20000;
    k_chase<<<1, 1>>>(d, (int)(perm[0] * 32), steps, dcyc, sink);
    k_chase<<<1, 1>>>(d, (int)(perm[0] * 32), steps, dcyc, sink);
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    printf("pointer chase %8zu KB: %.1f cycles/load\n", bytes >> 10, (double)cyc / steps);
    cudaFree(d);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr: %d kHz\n", clk);
  return 0;
}
