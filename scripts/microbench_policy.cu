// Latency / throughput of one policy_accumulate batch (32 lanes, converged)
// on the B200: W warps per SM (one CTA of W warps per SM), each warp runs
// NB batches back to back.  Prints cycles per batch per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -I../paper_2301_08068_b200/csrc
#include <cstdio>
#include <cstdlib>
#include "rmpb_device.cuh"
using namespace rmpb;

__global__ void k_bench(PolicyParams p, int nb, const double* __restrict__ in, double* out,
                        long long* cyc) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  double d = in[(blockIdx.x * blockDim.x + threadIdx.x) & 1023];
  const long long t0 = clock64();
  for (int b = 0; b < nb; ++b) {
    Acc a;
    a.zero();
    // a closing in-radius beam: dir (-0.6, 0.48, 0.64), v (1, -0.5, -0.5) -> toward < 0 ...
    policy_accumulate(a, -0.6, 0.48, 0.64, d, -1.0, 0.5, 0.9, p);
    acc += a.a00 + a.b0;
    d = d * 0.999 + 1e-3 * (double)(lane & 7);  // dependent next input
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (lane == 0) cyc[blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)] = t1 - t0;
}

int main() {
  PolicyParams p{};
  p.eta_rep = 1.2; p.nu_rep = 1.5; p.eta_damp = 3.0; p.nu_damp = 1.0; p.eps_p = 1e-6;
  p.radius = 1.3; p.c = 1.0; p.min_range = 0.3;
  recip_dd(p.nu_rep, p.rnr_h, p.rnr_l); recip_dd(p.nu_damp, p.rnd_h, p.rnd_l);
  recip_dd(p.radius, p.rr_h, p.rr_l); p.rr2 = p.radius * p.radius; recip_dd(p.rr2, p.rr2_h, p.rr2_l);
  double h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = 0.35 + 0.9 * (i % 97) / 97.0;
  double *din, *dout; long long* dc;
  cudaMalloc(&din, sizeof h); cudaMemcpy(din, h, sizeof h, cudaMemcpyHostToDevice);
  cudaMalloc(&dout, 148 * 1024 * 8); cudaMalloc(&dc, 148 * 32 * 8);
  const int nb = 200;
  for (int W : {1, 4, 8, 16, 32}) {
    k_bench<<<148, W * 32>>>(p, nb, din, dout, dc);
    cudaDeviceSynchronize();
    long long c[148 * 32];
    cudaMemcpy(c, dc, 148 * W * 8, cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < 148 * W; ++i) s += c[i];
    printf("warps/SM %2d: %.0f cycles per batch per warp, %.1f batches/kcycle/SM\n", W,
           s / (148 * W) / nb, 1000.0 * W * nb / (s / (148 * W)));
  }
  return 0;
}
