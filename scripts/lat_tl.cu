// Device timeline of the single-pose lean kernel (librmpb built with
// -DRMPB_DBG_TIMELINE; scripts/gpu_lat_tl.sh): CTA start -> last trace end ->
// last CTA past the ticket -> fold done -> slot written, medians of 200 calls.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <algorithm>
#include <chrono>
#include <vector>
#include "rmpb.h"
extern "C" int rmpb_debug_timeline(unsigned long long out[8]);

static std::vector<char> rd(const char* p) {
  FILE* f = fopen(p, "rb"); fseek(f, 0, SEEK_END); long n = ftell(f); fseek(f, 0, SEEK_SET);
  std::vector<char> b(n); if (fread(b.data(), 1, n, f) != (size_t)n) exit(1); fclose(f); return b;
}
static double med(std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; }
int main() {
  auto vals = rd("/tmp/lat_vals.f32"), dirs = rd("/tmp/lat_dirs.f64"), poses = rd("/tmp/lat_poses.f64");
  rmpb_grid* g; rmpb_bundle* b;
  if (rmpb_grid_create(vals.data(), RMPB_F32, 200, 200, 100, 0, 0, 0, 0.1, RMPB_STORE_AUTO,
                       RMPB_LAYOUT_AUTO, 0, &g)) return 1;
  if (rmpb_bundle_create((const double*)dirs.data(), (int64_t)(dirs.size() / 24), RMPB_ORDER_MORTON, 0, &b)) return 1;
  const double* P = (const double*)poses.data();
  const double prm[7] = {88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2};
  double slot[13], acc[3];
  unsigned long long tl[8];
  for (double mr : {1e-6, 2.4, 10.0}) {
    std::vector<double> tr, red, fold, wr, tot, host;
    for (int i = 0; i < 220; ++i) {
      const double* x = P + 6 * (i % 10);
      rmpb_debug_timeline(tl);
      auto a = std::chrono::steady_clock::now();
      if (rmpb_ray_policy(g, b, x, x + 3, prm, mr, 0.05, 0.9, slot, acc, nullptr, nullptr, nullptr, nullptr)) return 2;
      auto c = std::chrono::steady_clock::now();
      rmpb_debug_timeline(tl);
      if (i < 20) continue;
      tr.push_back((tl[1] - tl[0]) * 1e-3); red.push_back((tl[2] - tl[1]) * 1e-3);
      fold.push_back((tl[3] - tl[2]) * 1e-3); wr.push_back((tl[4] - tl[3]) * 1e-3);
      tot.push_back((tl[4] - tl[0]) * 1e-3);
      host.push_back(std::chrono::duration<double, std::micro>(c - a).count());
    }
    printf("{\"max_range\": %g, \"trace_us\": %.2f, \"reduce_ticket_us\": %.2f, \"fold_us\": %.2f, "
           "\"write_slot_us\": %.2f, \"first_cta_to_slot_us\": %.2f, \"host_call_us\": %.2f}\n",
           mr, med(tr), med(red), med(fold), med(wr), med(tot), med(host));
  }
  return 0;
}
