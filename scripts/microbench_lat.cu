// Dependent-chain latency of the ops on the trace step's critical path, one
// warp on one SM (cycles per op, clock64 around 512 dependent ops):
//   DADD, DMUL, DFMA, F2F.F64.F32 (+ F2F.F32.F64 back), DADD.RZ + lo word,
//   FFMA, IMAD, LDG.128 pointer chase in L1 and in L2.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/mlat scripts/microbench_lat.cu
#include <cstdio>

constexpr int N = 512;

__global__ void k_alu(const double* in, double* out, long long* cyc) {
  double a = in[threadIdx.x], b = in[threadIdx.x + 32];
  float fa = (float)a, fb = (float)b;
  int ia = (int)threadIdx.x, ib = (int)in[threadIdx.x + 1] + 2;
  long long t0, t1;
  // DADD
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) a = __dadd_rn(a, b);
  t1 = clock64(); cyc[0] = t1 - t0;
  // DMUL
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) a = __dmul_rn(a, b);
  t1 = clock64(); cyc[1] = t1 - t0;
  // DFMA
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) a = __fma_rn(a, b, b);
  t1 = clock64(); cyc[2] = t1 - t0;
  // F2F.F32.F64 + F2F.F64.F32 pair
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) a = (double)__double2float_rn(a);
  t1 = clock64(); cyc[3] = t1 - t0;
  // DADD.RZ then lo word -> int -> back into the chain (IADD + I2F? no: DADD with hi/lo rebuild)
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) {
    double big = __dadd_rz(a, 6755399441055744.0);
    a = __hiloint2double(__double2hiint(big), __double2loint(big) + ib);
  }
  t1 = clock64(); cyc[4] = t1 - t0;
  // FFMA
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) fa = __fmaf_rn(fa, fb, fb);
  t1 = clock64(); cyc[5] = t1 - t0;
  // IMAD
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) ia = ia * ib + 7;
  t1 = clock64(); cyc[6] = t1 - t0;
  // F2F.F64.F32 alone: float chain through a double (convert up, DADD-free down via hi word)
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) fa = __int_as_float(__double2hiint((double)fa) ^ ib);
  t1 = clock64(); cyc[7] = t1 - t0;
  out[threadIdx.x] = a + (double)fa + ia;
}

__global__ void k_chase(const unsigned* next, int steps, unsigned start, unsigned* out, long long* cyc) {
  unsigned p = start;
  // warm
  for (int i = 0; i < steps; ++i) p = __ldg(next + p);
  p = start + (p & 0);  // restart: the timed pass re-reads the warmed lines
  const long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = __ldg(next + p);
  const long long t1 = clock64();
  *out = p;
  *cyc = t1 - t0;
}

int main() {
  double h[64];
  for (int i = 0; i < 64; ++i) h[i] = 1.0 + 1e-9 * i;
  double *din, *dout; long long* dc; long long hc[8];
  cudaMalloc(&din, sizeof h); cudaMemcpy(din, h, sizeof h, cudaMemcpyHostToDevice);
  cudaMalloc(&dout, 32 * 8); cudaMalloc(&dc, 8 * 8);
  for (int r = 0; r < 2; ++r) k_alu<<<1, 32>>>(din, dout, dc);
  cudaMemcpy(hc, dc, sizeof hc, cudaMemcpyDeviceToHost);
  const char* nm[8] = {"DADD", "DMUL", "DFMA", "F2F f64->f32->f64 pair", "DADD.RZ + lo/hi rebuild",
                       "FFMA", "IMAD", "F2F.F64.F32 + hi word"};
  for (int i = 0; i < 8; ++i) printf("%-28s %.1f cyc/op\n", nm[i], (double)hc[i] / N);
  // pointer chase: stride 4 KB (distinct lines), footprint 64 KB (L1) and 64 MB (L2)
  for (long long foot : {64LL << 10, 64LL << 20}) {
    const unsigned n = (unsigned)(foot / 4), stride = 1024 + 32;  // words
    unsigned* hn = new unsigned[n];
    for (unsigned i = 0; i < n; ++i) hn[i] = (i + stride) % n;
    unsigned* dn; cudaMalloc(&dn, foot);
    cudaMemcpy(dn, hn, foot, cudaMemcpyHostToDevice);
    unsigned* dres; cudaMalloc(&dres, 4);
    const int steps = foot < (1 << 20) ? 15 : 4096;  // 64 KB: 15 lines
    k_chase<<<1, 1>>>(dn, steps, 0, dres, dc);
    cudaMemcpy(hc, dc, 8, cudaMemcpyDeviceToHost);
    printf("LDG chase footprint %lld KB: %.1f cyc/load\n", foot >> 10, (double)hc[0] / steps);
    cudaFree(dn); cudaFree(dres); delete[] hn;
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
