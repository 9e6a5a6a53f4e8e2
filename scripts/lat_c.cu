// Host-path latency floor of the single-pose C ABI call (no Python):
// empty-kernel launch+sync, rmpb_ray_policy at ~0 range and at 10 m.
// Inputs (raw files written by scripts/probe_lat_c.py): C1 grid f32, bundle
// f64, 10 poses (x, v).  Build: nvcc -O2 -I include scripts/lat_c.cu
// -L paper_2301_08068_b200 -lrmpb -o /tmp/lat_c
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <algorithm>
#include <chrono>
#include <vector>
#include "rmpb.h"

__global__ void k_empty() {}
__global__ void k_flag(volatile unsigned* f, unsigned v) { if (threadIdx.x == 0 && blockIdx.x == 0) { __threadfence_system(); *f = v; } }

static double now_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}
template <class F> static double med(F f, int n = 400) {
  for (int i = 0; i < 20; ++i) f(i);
  std::vector<double> t(n);
  for (int i = 0; i < n; ++i) { double a = now_us(); f(i); t[i] = now_us() - a; }
  std::sort(t.begin(), t.end());
  return t[n / 2];
}
static std::vector<char> rd(const char* p) {
  FILE* f = fopen(p, "rb"); fseek(f, 0, SEEK_END); long n = ftell(f); fseek(f, 0, SEEK_SET);
  std::vector<char> b(n); fread(b.data(), 1, n, f); fclose(f); return b;
}
int main() {
  auto vals = rd("/tmp/lat_vals.f32"), dirs = rd("/tmp/lat_dirs.f64"), poses = rd("/tmp/lat_poses.f64");
  rmpb_grid* g; rmpb_bundle* b;
  if (rmpb_grid_create(vals.data(), RMPB_F32, 200, 200, 100, 0, 0, 0, 0.1, RMPB_STORE_AUTO,
                       RMPB_LAYOUT_AUTO, 0, &g)) { printf("grid: %s\n", rmpb_last_error()); return 1; }
  if (rmpb_bundle_create((const double*)dirs.data(), (int64_t)(dirs.size() / 24), RMPB_ORDER_MORTON, 0, &b)) {
    printf("bundle: %s\n", rmpb_last_error()); return 1; }
  const double* P = (const double*)poses.data();
  const double prm[7] = {88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2};
  double slot[13], acc[3];
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  double e0 = med([&](int) { k_empty<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); });
  double e1 = med([&](int) { k_empty<<<256, 256, 0, s>>>(); cudaStreamSynchronize(s); });
  volatile unsigned* hflag; cudaHostAlloc((void**)&hflag, 64, cudaHostAllocMapped);
  unsigned* dflag; cudaHostGetDevicePointer((void**)&dflag, (void*)hflag, 0);
  *hflag = 0; unsigned ep = 0;
  double e2 = med([&](int) { ++ep; k_flag<<<1, 32, 0, s>>>(dflag, ep); while (*hflag != ep) {} });
  double e3 = med([&](int) { k_empty<<<1, 32, 0, s>>>(); while (cudaStreamQuery(s) == cudaErrorNotReady) {} });
  double e4 = med([&](int) { k_empty<<<1, 32, 0, s>>>(); });
  cudaStreamSynchronize(s);
  auto call = [&](int i, double mr, void* st) {
    const double* x = P + 6 * (i % 10);
    int rc = rmpb_ray_policy(g, b, x, x + 3, prm, mr, 0.05, 0.9, slot, acc, nullptr, nullptr, nullptr, st);
    if (rc) { printf("err %s\n", rmpb_last_error()); exit(1); }
  };
  double r0 = med([&](int i) { call(i, 1e-6, nullptr); });
  double r10 = med([&](int i) { call(i, 10.0, nullptr); });
  double r0s = med([&](int i) { call(i, 1e-6, s); });
  double r10s = med([&](int i) { call(i, 10.0, s); });
  double r24 = med([&](int i) { call(i, 2.4, nullptr); });  // policy-only range (radius)
  rmpb_set_option("l2_window", 0);
  double r24w = med([&](int i) { call(i, 2.4, nullptr); });
  double r0w = med([&](int i) { call(i, 1e-6, nullptr); });
  rmpb_set_option("l2_window", 1);
  rmpb_set_option("seg_rays", 512);
  double r24s = med([&](int i) { call(i, 2.4, nullptr); });
  rmpb_set_option("seg_rays", 1024);
  double r24s2 = med([&](int i) { call(i, 2.4, nullptr); });
  rmpb_set_option("seg_rays", 0);
  printf("{\"abi_range2.4_no_l2window_us\": %.2f, \"abi_range0_no_l2window_us\": %.2f, "
         "\"abi_range2.4_seg512_us\": %.2f, \"abi_range2.4_seg1024_us\": %.2f}\n", r24w, r0w, r24s, r24s2);
  printf("{\"flag_spin_us\": %.2f, \"query_spin_us\": %.2f, \"launch_only_us\": %.2f, ", e2, e3, e4);
  printf("{\"empty_1x32_us\": %.2f, \"empty_256x256_us\": %.2f, \"abi_range0_us\": %.2f, "
         "\"abi_range10_us\": %.2f, \"abi_range0_stream_us\": %.2f, \"abi_range10_stream_us\": %.2f, "
         "\"abi_range2.4_us\": %.2f}\n",
         e0, e1, r0, r10, r0s, r10s, r24);
  return 0;
}
