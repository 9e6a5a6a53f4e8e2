// rmpb_kernels.cuh -- the hot-path kernels (K1 fused ray policy, K2 LiDAR-
// direct policy, K3 = K1 batched over poses) and the fixed-order fold.
//
// One CTA processes one "unit" = (pose, ray segment).  Each thread traces its
// rays in a fixed order and accumulates the per-ray policy into registers; the
// CTA reduces with a fixed butterfly/warp-order tree (rmpb_device.cuh).  If a
// pose has one segment the CTA resolves it directly (3x3 pinv on device);
// otherwise each CTA writes a 10-double partial and the LAST CTA of the pose
// (atomic ticket) folds the partials in segment order and resolves.  All
// orders are fixed, so results are bitwise reproducible run to run.
#pragma once
#include "rmpb_device.cuh"

namespace rmpb {

struct PoseIO {
  const double* __restrict__ x;   // [P][3] positions
  const double* __restrict__ v;   // [P][3] velocities
  double* __restrict__ slot;      // [P][13] (may be null when only partials wanted)
  double* __restrict__ accel;     // [P][3]  (null: skip pinv)
  double* __restrict__ partials;  // [P*segs][10] when segs > 1
  unsigned* __restrict__ tickets; // [P] zero-initialised, self-resetting
  double* __restrict__ seg_out;   // [P*segs][10] raw segment partials (ray-split), or null
  double x0[3], v0[3];            // single pose by value when x / v are null
  __device__ __forceinline__ void pose(int p, double& a, double& b, double& c) const {
    if (x) { a = x[3 * p]; b = x[3 * p + 1]; c = x[3 * p + 2]; } else { a = x0[0]; b = x0[1]; c = x0[2]; }
  }
  __device__ __forceinline__ void vel(int p, double& a, double& b, double& c) const {
    if (v) { a = v[3 * p]; b = v[3 * p + 1]; c = v[3 * p + 2]; } else { a = v0[0]; b = v0[1]; c = v0[2]; }
  }
};

struct RayOut {  // optional per-ray parity outputs (indexed by ORIGINAL ray index)
  double* __restrict__ t;
  int* __restrict__ cell;   // [N][3]
  int* __restrict__ steps;  // [N]
  unsigned long long* __restrict__ step_total;  // optional global step counter
};

struct Bundle {
  const double* __restrict__ dx;
  const double* __restrict__ dy;
  const double* __restrict__ dz;
  const int* __restrict__ perm;  // stored index -> original index (null = identity)
  int n;
};

__device__ __forceinline__ void acc_to_arr(const Acc& a, double* o) {
  o[0] = a.a00; o[1] = a.a01; o[2] = a.a02; o[3] = a.a11; o[4] = a.a12;
  o[5] = a.a22; o[6] = a.b0; o[7] = a.b1; o[8] = a.b2; o[9] = (double)a.cnt;
}

// Finish a unit: reduce the CTA, then either resolve the pose or publish a
// partial and let the last CTA of the pose fold + resolve.
__device__ __forceinline__ void finish_unit(Acc& acc, const PoseIO& io, int pose, int seg,
                                            int segs) {
  __shared__ double sm[kWarps * kAcc];
  __shared__ int s_last;
  block_reduce(acc, sm);
  if (io.seg_out && threadIdx.x == 0) acc_to_arr(acc, io.seg_out + (size_t)(pose * segs + seg) * kAcc);
  if (segs == 1) {
    if (threadIdx.x == 0 && io.slot)
      write_slot(acc, io.slot + (size_t)pose * 13, io.accel ? io.accel + (size_t)pose * 3 : nullptr);
    return;
  }
  if (!io.slot) return;
  if (threadIdx.x == 0) {
    acc_to_arr(acc, io.partials + (size_t)(pose * segs + seg) * kAcc);
    __threadfence();
    unsigned prev = atomicAdd(io.tickets + pose, 1u);
    s_last = (prev == (unsigned)(segs - 1));
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // Fixed-order fold of this pose's partials: thread j sums segments
  // j, j+kBlock, ... sequentially, then the fixed block tree.
  Acc f;
  f.zero();
  double cnt = 0.0;
  const double* base = io.partials + (size_t)pose * segs * kAcc;
  for (int j = threadIdx.x; j < segs; j += kBlock) {
    const double* q = base + (size_t)j * kAcc;
    f.a00 += __ldcg(q + 0); f.a01 += __ldcg(q + 1); f.a02 += __ldcg(q + 2);
    f.a11 += __ldcg(q + 3); f.a12 += __ldcg(q + 4); f.a22 += __ldcg(q + 5);
    f.b0 += __ldcg(q + 6); f.b1 += __ldcg(q + 7); f.b2 += __ldcg(q + 8);
    cnt += __ldcg(q + 9);
  }
  f.cnt = (int)cnt;
  block_reduce(f, sm);
  if (threadIdx.x == 0) {
    write_slot(f, io.slot + (size_t)pose * 13, io.accel ? io.accel + (size_t)pose * 3 : nullptr);
    io.tickets[pose] = 0u;  // self-reset: graph replays / next call start clean
  }
}

// K1 / K3: fused sphere trace + per-ray policy + reduction (+ pinv).
// grid: P * segs CTAs of kBlock threads; segment = seg_rays consecutive
// stored rays of the bundle.
template <class G>
__global__ void __launch_bounds__(kBlock)
k_ray_policy(G grid, GridGeom g, Bundle b, PoseIO io, PolicyParams p, double max_range,
             double eps, double step_scale, int segs, int seg_rays, RayOut ro) {
  const int unit = blockIdx.x;
  const int pose = unit / segs, seg = unit - pose * segs;
  double sx, sy, sz, vx, vy, vz;
  io.pose(pose, sx, sy, sz);
  io.vel(pose, vx, vy, vz);
  Acc acc;
  acc.zero();
  const int begin = seg * seg_rays;
  const int end = min(begin + seg_rays, b.n);
  int my_steps = 0;
  for (int i = begin + threadIdx.x; i < end; i += kBlock) {
    const double dx = b.dx[i], dy = b.dy[i], dz = b.dz[i];
    TraceResult r = trace_ray(grid, g, sx, sy, sz, dx, dy, dz, max_range, eps, step_scale);
    policy_accumulate(acc, dx, dy, dz, r.t, vx, vy, vz, p);
    my_steps += r.steps;
    if (ro.t) {
      const int o = b.perm ? b.perm[i] : i;
      ro.t[o] = r.t;
      if (ro.cell) { ro.cell[3 * o] = r.cx; ro.cell[3 * o + 1] = r.cy; ro.cell[3 * o + 2] = r.cz; }
      if (ro.steps) ro.steps[o] = r.steps;
    }
  }
  if (ro.step_total) {
    int s = warp_sum_i(my_steps);
    if ((threadIdx.x & 31) == 0) atomicAdd(ro.step_total, (unsigned long long)s);
  }
  finish_unit(acc, io, pose, seg, segs);
}

// K2: LiDAR-direct policy (policies.py:195-205, rays.py:172-173).  Beam k of
// scan s: world dir = R_s * d_k (rows of R dotted with d, fixed order),
// distance = ranges[s][k] if valid else +inf, min_range skip.
struct ScanIO {
  const double* __restrict__ dirs;   // [N][3] sensor (or world when R null)
  const double* __restrict__ R;      // [S][9] row-major or null
  const double* __restrict__ ranges; // [S][N]
  const unsigned char* __restrict__ valid;  // [S][N] or null (all valid)
  int n;
};

__global__ void __launch_bounds__(kBlock)
k_lidar_policy(ScanIO sc, PoseIO io, PolicyParams p, int segs, int seg_rays) {
  const int unit = blockIdx.x;
  const int scan = unit / segs, seg = unit - scan * segs;
  double vx, vy, vz;
  io.vel(scan, vx, vy, vz);
  double R[9];
  const bool rot = sc.R != nullptr;
  if (rot) {
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = sc.R[9 * scan + k];
  }
  const double* rg = sc.ranges + (size_t)scan * sc.n;
  const unsigned char* vl = sc.valid ? sc.valid + (size_t)scan * sc.n : nullptr;
  Acc acc;
  acc.zero();
  const int begin = seg * seg_rays;
  const int end = min(begin + seg_rays, sc.n);
  for (int i = begin + threadIdx.x; i < end; i += kBlock) {
    double d = rg[i];
    if (vl && !vl[i]) d = CUDART_INF;
    if (d != d || d == CUDART_INF || d < p.min_range) continue;
    double ex = sc.dirs[3 * i], ey = sc.dirs[3 * i + 1], ez = sc.dirs[3 * i + 2];
    double wx = ex, wy = ey, wz = ez;
    if (rot) {  // directions @ orientation.T  (rays.py:172-173)
      wx = ex * R[0] + ey * R[1] + ez * R[2];
      wy = ex * R[3] + ey * R[4] + ez * R[5];
      wz = ex * R[6] + ey * R[7] + ez * R[8];
    }
    policy_accumulate(acc, wx, wy, wz, d, vx, vy, vz, p);
  }
  finish_unit(acc, io, scan, seg, segs);
}

// K2b: LiDAR-direct from raw sensor-frame points (no map, no lattice): the
// beam direction is p/|p| and its range |p|; zero / non-finite points are
// invalid.  Float32 xyz as delivered by the sensor driver.
struct PointsIO {
  const float* __restrict__ xyz;  // [S][N][3]
  const double* __restrict__ R;   // [S][9] or null
  int n;
};

__global__ void __launch_bounds__(kBlock)
k_lidar_points(PointsIO pt, PoseIO io, PolicyParams p, int segs, int seg_rays) {
  const int unit = blockIdx.x;
  const int scan = unit / segs, seg = unit - scan * segs;
  double vx, vy, vz;
  io.vel(scan, vx, vy, vz);
  double R[9];
  const bool rot = pt.R != nullptr;
  if (rot) {
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = pt.R[9 * scan + k];
  }
  const float* P = pt.xyz + (size_t)scan * pt.n * 3;
  Acc acc;
  acc.zero();
  const int begin = seg * seg_rays;
  const int end = min(begin + seg_rays, pt.n);
  for (int i = begin + threadIdx.x; i < end; i += kBlock) {
    double px = P[3 * i], py = P[3 * i + 1], pz = P[3 * i + 2];
    double d = sqrt(px * px + py * py + pz * pz);
    if (!(d > 0.0)) continue;  // zero ("no return") or NaN point: invalid beam
    // d == inf / d < min_range are skipped (and not counted) by policy_accumulate
    double ex = px / d, ey = py / d, ez = pz / d;
    double wx = ex, wy = ey, wz = ez;
    if (rot) {
      wx = ex * R[0] + ey * R[1] + ez * R[2];
      wy = ex * R[3] + ey * R[4] + ez * R[5];
      wz = ex * R[6] + ey * R[7] + ez * R[8];
    }
    policy_accumulate(acc, wx, wy, wz, d, vx, vy, vz, p);
  }
  finish_unit(acc, io, scan, seg, segs);
}

// Unfused parity entry (ckern.policy_reduce, ckern.py:80-93): reduce given
// (dirs, dists) -- AoS host layout -- into a slot.
__global__ void __launch_bounds__(kBlock)
k_policy_reduce(const double* __restrict__ dirs, const double* __restrict__ dists, int n,
                PoseIO io, PolicyParams p, int segs, int seg_rays) {
  const int seg = blockIdx.x;
  double vx, vy, vz;
  io.vel(0, vx, vy, vz);
  Acc acc;
  acc.zero();
  const int begin = seg * seg_rays;
  const int end = min(begin + seg_rays, n);
  for (int i = begin + threadIdx.x; i < end; i += kBlock)
    policy_accumulate(acc, dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2], dists[i], vx, vy, vz, p);
  finish_unit(acc, io, 0, seg, segs);
}

// Unfused parity entry (ckern.grid_trace, ckern.py:49-62): AoS dirs.
template <class G>
__global__ void __launch_bounds__(kBlock)
k_grid_trace(G grid, GridGeom g, const double* __restrict__ dirs, int n, double sx, double sy,
             double sz, double max_range, double eps, double step_scale, RayOut ro) {
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n) return;
  TraceResult r = trace_ray(grid, g, sx, sy, sz, dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2],
                            max_range, eps, step_scale);
  ro.t[i] = r.t;
  if (ro.cell) { ro.cell[3 * i] = r.cx; ro.cell[3 * i + 1] = r.cy; ro.cell[3 * i + 2] = r.cz; }
  if (ro.steps) ro.steps[i] = r.steps;
}

// Resolve already-reduced slots: fixed pairwise fold (the reference's
// pairwise_fold shape, _pool.py:61-72) of `n` 13-slots followed by pinv.
// Used for ray ranges split across GPUs (each rank contributes one slot).
__global__ void k_fold_resolve(const double* __restrict__ slots, int n, double* __restrict__ out_slot,
                               double* __restrict__ out_accel) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  // pairwise fold with an in-register stack is awkward for arbitrary n;
  // n is small (number of GPUs), so fold in a local buffer.
  double buf[64 * 13];
  int m = n < 64 ? n : 64;
  for (int i = 0; i < m * 13; ++i) buf[i] = slots[i];
  while (m > 1) {
    int half = m / 2;
    for (int k = 0; k < half; ++k)
      for (int j = 0; j < 13; ++j) buf[k * 13 + j] = buf[2 * k * 13 + j] + buf[(2 * k + 1) * 13 + j];
    if (m % 2)
      for (int j = 0; j < 13; ++j) buf[half * 13 + j] = buf[(m - 1) * 13 + j];
    m = half + (m % 2);
  }
  for (int j = 0; j < 13; ++j) out_slot[j] = buf[j];
  if (out_accel) {
    double m9[9], f[3];
    for (int k = 0; k < 9; ++k) m9[k] = buf[k];
    f[0] = buf[9]; f[1] = buf[10]; f[2] = buf[11];
    pinv_apply(m9, f, out_accel);
  }
}

// pinv_psd of a batch of 3x3 metrics (core.py:103-115), returns the matrix.
__global__ void k_pinv_psd(const double* __restrict__ a, int n, double* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double m[3][3], V[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) m[r][c] = 0.5 * (a[9 * i + 3 * r + c] + a[9 * i + 3 * c + r]);
  jacobi3(m, V);
  double lam[3] = {m[0][0], m[1][1], m[2][2]};
  double lmax = fmax(fmax(lam[0], lam[1]), lam[2]);
  double cut = 1e-8 * (lmax > 0.0 ? lmax : 0.0);
  double inv[3];
  for (int k = 0; k < 3; ++k) inv[k] = lam[k] > cut ? 1.0 / lam[k] : 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      out[9 * i + 3 * r + c] = V[r][0] * inv[0] * V[c][0] + V[r][1] * inv[1] * V[c][1] +
                               V[r][2] * inv[2] * V[c][2];
}

}  // namespace rmpb
