// rmpb_dda.cuh -- K5: per-ray 3D DDA (Amanatides-Woo) over a bit-packed
// occupancy grid, the traversal north_star names.  NOT the reference's
// algorithm (the reference sphere-traces the ESDF): it is a
// separate, opt-in traversal, checked bit-for-bit against its own CPU
// definition (oracle/rmp_oracle.c orc_dda_trace) and never mixed with the
// reference-parity claims.
//
// Occupancy = node value <= 0 (rmpnav/geometry.py:312-315); the voxel of
// node (i,j,k) is the res-cube centred on it.  One bit per voxel, 32 voxels
// of a z-column per word: the C1 map is 500 KB -- L1/L2 resident.  The march
// is float32 with no contraction and IEEE division (this file is compiled
// with -fmad=false), so the CPU and GPU visit the same voxels and report the
// same entry distance bit-for-bit.
#pragma once
#include "rmpb_kernels.cuh"

namespace rmpb {

struct Occupancy {
  const uint32_t* __restrict__ bits;
  int nx, ny, nz, nzw;   // nzw = ceil(nz / 32)
  float ox, oy, oz, inv; // origin (f32) and 1/res (f32)
  __device__ __forceinline__ bool occ(int i, int j, int k) const {
    return (__ldg(bits + ((unsigned)(i * ny + j) * nzw + (k >> 5))) >> (k & 31)) & 1u;
  }
};

// Node values -> occupancy bits, one 32-voxel word per thread.
template <class G>
__global__ void k_occ_build(G grid, int nx, int ny, int nz, int nzw, uint32_t* __restrict__ bits) {
  long long n = (long long)nx * ny * nzw;
  long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; w < n; w += stride) {
    const int kw = (int)(w % nzw);
    const long long r = w / nzw;
    const int j = (int)(r % ny), i = (int)(r / ny);
    uint32_t word = 0;
    for (int b = 0; b < 32; ++b) {
      const int k = kw * 32 + b;
      if (k >= nz) break;
      const int ci = min(i, nx - 2), cj = min(j, ny - 2), ck = min(k, nz - 2);
      Corners c = grid.load(ci, cj, ck);
      const int a = i - ci, bb = j - cj, d = k - ck;
      const double v = a ? (bb ? (d ? c.v111 : c.v110) : (d ? c.v101 : c.v100))
                         : (bb ? (d ? c.v011 : c.v010) : (d ? c.v001 : c.v000));
      if (v <= 0.0) word |= 1u << b;
    }
    bits[w] = word;
  }
}

struct DdaResult {
  float t;          // entry distance of the first occupied voxel, +inf on miss
  int vx, vy, vz;   // its index (-1 on miss)
  int steps;        // voxels visited
};

// March state of one ray (scalars: indexing per-axis arrays with the
// data-dependent axis would put them on the stack).
struct DdaState {
  int vx, vy, vz, sx, sy, sz;
  float tmx, tmy, tmz, tdx, tdy, tdz, t, t1;
};

// Ray set-up of orc_dda_trace; false = the ray misses the grid.
__device__ __forceinline__ bool dda_setup(const Occupancy& o, float sx, float sy, float sz,
                                          float dx, float dy, float dz, float max_range,
                                          DdaState& q) {
  const int n[3] = {o.nx, o.ny, o.nz};
  float u[3], dv[3];
  {
    const float st[3] = {sx, sy, sz}, org[3] = {o.ox, o.oy, o.oz}, d[3] = {dx, dy, dz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float p = st[a] - org[a];
      p = p * o.inv;
      u[a] = p + 0.5f;
      dv[a] = d[a] * o.inv;
    }
  }
  float t0 = 0.0f, t1 = max_range;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (dv[a] != 0.0f) {
      float ta = (0.0f - u[a]) / dv[a];
      float tb = ((float)n[a] - u[a]) / dv[a];
      if (tb < ta) { float tmp = ta; ta = tb; tb = tmp; }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
    } else if (u[a] < 0.0f || u[a] >= (float)n[a]) {
      return false;
    }
  }
  if (t0 > t1) return false;
  int vox[3], stp[3];
  float tmax[3], tdel[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float pa = dv[a] * t0;
    pa = u[a] + pa;
    int ia = (int)floorf(pa);
    ia = ia < 0 ? 0 : (ia > n[a] - 1 ? n[a] - 1 : ia);
    vox[a] = ia;
    if (dv[a] > 0.0f) {
      stp[a] = 1;
      tmax[a] = ((float)(ia + 1) - u[a]) / dv[a];
      tdel[a] = 1.0f / dv[a];
    } else if (dv[a] < 0.0f) {
      stp[a] = -1;
      tmax[a] = ((float)ia - u[a]) / dv[a];
      tdel[a] = -1.0f / dv[a];
    } else {
      stp[a] = 0;
      tmax[a] = CUDART_INF_F;
      tdel[a] = CUDART_INF_F;
    }
  }
  q.vx = vox[0]; q.vy = vox[1]; q.vz = vox[2];
  q.sx = stp[0]; q.sy = stp[1]; q.sz = stp[2];
  q.tmx = tmax[0]; q.tmy = tmax[1]; q.tmz = tmax[2];
  q.tdx = tdel[0]; q.tdy = tdel[1]; q.tdz = tdel[2];
  q.t = t0; q.t1 = t1;
  return true;
}

// One voxel visit of orc_dda_trace's loop: 1 = hit (q.t is the entry
// distance), -1 = left the range / grid, 0 = continue.  Axis choice, t and
// the tMax update are those of orc_dda_trace exactly:
// a = 0; if (tmax[1] < tmax[a]) a = 1; if (tmax[2] < tmax[a]) a = 2.
__device__ __forceinline__ int dda_step(const Occupancy& o, DdaState& q) {
  if (o.occ(q.vx, q.vy, q.vz)) return 1;
  const bool y_lt = q.tmy < q.tmx;
  const float m = y_lt ? q.tmy : q.tmx;
  const bool az = q.tmz < m, ay = !az && y_lt, ax = !az && !y_lt;
  q.t = az ? q.tmz : m;
  if (!(q.t <= q.t1)) return -1;
  q.vx += ax ? q.sx : 0;
  q.vy += ay ? q.sy : 0;
  q.vz += az ? q.sz : 0;
  if (((unsigned)q.vx >= (unsigned)o.nx) | ((unsigned)q.vy >= (unsigned)o.ny) |
      ((unsigned)q.vz >= (unsigned)o.nz))
    return -1;
  q.tmx = ax ? q.tmx + q.tdx : q.tmx;
  q.tmy = ay ? q.tmy + q.tdy : q.tmy;
  q.tmz = az ? q.tmz + q.tdz : q.tmz;
  return 0;
}

__device__ __forceinline__ DdaResult dda_ray(const Occupancy& o, float sx, float sy, float sz,
                                             float dx, float dy, float dz, float max_range) {
  DdaResult res;
  res.t = CUDART_INF_F; res.vx = res.vy = res.vz = -1; res.steps = 0;
  DdaState q;
  if (!dda_setup(o, sx, sy, sz, dx, dy, dz, max_range, q)) return res;
  while (true) {
    ++res.steps;
    const int r = dda_step(o, q);
    if (r > 0) { res.t = q.t; res.vx = q.vx; res.vy = q.vy; res.vz = q.vz; break; }
    if (r < 0) break;
  }
  return res;
}

__global__ void __launch_bounds__(kBlock)
k_dda_trace(Occupancy o, const double* __restrict__ dirs, int n, float sx, float sy, float sz,
            float max_range, float* __restrict__ out_t, int* __restrict__ out_vox,
            int* __restrict__ out_steps) {
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= n) return;
  DdaResult r = dda_ray(o, sx, sy, sz, (float)dirs[3 * i], (float)dirs[3 * i + 1],
                        (float)dirs[3 * i + 2], max_range);
  out_t[i] = r.t;
  out_vox[3 * i] = r.vx; out_vox[3 * i + 1] = r.vy; out_vox[3 * i + 2] = r.vz;
  if (out_steps) out_steps[i] = r.steps;
}

// Fused DDA + per-ray policy (distance = voxel entry distance) + reduction,
// same unit / fold structure as the sphere-trace kernels.  The policy is
// deferred like k_ray_policy2's: closing hits inside the activation radius
// (the only rays policy_accumulate adds to) are queued per warp and evaluated
// 32 at a time, converged; the hit count is lane-private.  Queue order is
// data-determined, so results are bitwise reproducible.
struct DdaSmem {
  double acc[kWarps][9];
  double qt[kWarps][kQueue];
  int qr[kWarps][kQueue];
};

#ifndef RMPB_DDA_MINB
#define RMPB_DDA_MINB 4
#endif
__global__ void __launch_bounds__(kBlock, RMPB_DDA_MINB)
k_ray_policy_dda(Occupancy o, Bundle b, PoseIO io, PolicyParams p, float max_range, int segs,
                 int seg_rays) {
  __shared__ DdaSmem sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
  const int unit = blockIdx.x;
  const int pose = unit / segs, seg = unit - pose * segs;
  double sx, sy, sz, vx, vy, vz;
  io.pose(pose, sx, sy, sz);
  io.vel(pose, vx, vy, vz);
  if (lane < 9) sm.acc[warp][lane] = 0.0;
  __syncwarp();
  double* qt = sm.qt[warp];
  int* qr = sm.qr[warp];
  int qn = 0, cnt = 0;
  const int begin = seg * seg_rays;
  const int end = min(begin + seg_rays, b.n);
  // One ray per thread per pass (a lane-refill variant with per-lane set-up
  // measured 1.8x slower: the fp32 IEEE divisions of the set-up then run
  // once per refill round instead of once per converged pass).
  const int iters = (end - begin + kBlock - 1) / kBlock;  // warp-uniform trip count
  for (int k = 0; k < iters; ++k) {
    const int i = begin + k * kBlock + threadIdx.x;
    bool enq = false;
    double d = 0.0;
    if (i < end) {
      const double dx = b.dx[i], dy = b.dy[i], dz = b.dz[i];
      const DdaResult r = dda_ray(o, (float)sx, (float)sy, (float)sz, (float)dx, (float)dy,
                                  (float)dz, max_range);
      d = (double)r.t;
      // policy_accumulate's filters, same expressions and order
      const bool counted = !(d != d || d == CUDART_INF || d < p.min_range);
      cnt += counted;
      enq = counted && d < p.radius && (dx * vx + dy * vy + dz * vz) > 0.0;
    }
    const unsigned em = __ballot_sync(FULL, enq);
    if (em) {
      if (enq) {
        const int pos = qn + __popc(em & lt);
        qt[pos] = d;
        qr[pos] = i;
      }
      qn += __popc(em);
      if (qn >= 32) {
        __syncwarp();
        policy_flush(sm, warp, lane, true, b, qr[lane], qt[lane], vx, vy, vz, p);
        __syncwarp();
        if (lane < qn - 32) { qt[lane] = qt[lane + 32]; qr[lane] = qr[lane + 32]; }
        qn -= 32;
        __syncwarp();
      }
    }
  }
  __syncwarp();
  if (qn > 0) {
    const bool valid = lane < qn;
    policy_flush(sm, warp, lane, valid, b, valid ? qr[lane] : 0, valid ? qt[lane] : 0.0, vx, vy,
                 vz, p);
  }
  cnt = warp_sum_i(cnt);
  __syncwarp();
  Acc acc;
  acc.zero();
  if (lane == 0) {
    acc.a00 = sm.acc[warp][0]; acc.a01 = sm.acc[warp][1]; acc.a02 = sm.acc[warp][2];
    acc.a11 = sm.acc[warp][3]; acc.a12 = sm.acc[warp][4]; acc.a22 = sm.acc[warp][5];
    acc.b0 = sm.acc[warp][6]; acc.b1 = sm.acc[warp][7]; acc.b2 = sm.acc[warp][8];
    acc.cnt = cnt;
  }
  finish_unit(acc, io, pose, seg, segs);
}

}  // namespace rmpb
