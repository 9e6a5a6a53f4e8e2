// rmpb_rollout.cuh -- row f1: the closed-loop rollout step on device for a
// batch of robots (rmpnav/sim.py:155-161 step, 196-306 rollout).
//
// Per control tick and per active robot, in the reference's order:
//   checks at t = k dt: collision (analytic scene distance <= robot radius),
//   goal reached, time-out, stuck (mean speed over the window);
//   obstacle policy = fused ray policy (k_ray_policy2, masked to active);
//   command = combine([attractor(x, goal), obstacle])  (core.py:130-144):
//       accel = pinv(I + M) (f_att + M a_obs),  M = sum A_i (symmetric);
//   clamp |accel| to max_accel; semi-implicit Euler; speed window update.
// No host round trip per tick: the host launches ticks back to back.
#pragma once
#include "rmpb_aux.cuh"
#include "rmpb_device.cuh"

namespace rmpb {

enum Outcome : int { OUT_RUNNING = 0, OUT_SUCCESS = 1, OUT_COLLISION = 2, OUT_TIMEOUT = 3,
                     OUT_STUCK = 4 };

struct RolloutCfg {
  double dt, max_time, robot_radius, goal_tol, max_accel, stuck_speed;
  double alpha, beta, c;  // attractor (policies.py:127-132)
  int window;             // stuck window in ticks
  int max_steps;
  int hold;               // hold_mode: no goal / stuck termination, time-out = success
  int record;             // ticks recorded per robot (0 = none)
};

struct RolloutState {
  double* x;        // [P][3]
  double* v;        // [P][3]
  const double* goal;  // [P][3]
  int* k;           // [P] ticks done
  int* active;      // [P] 1 while running
  int* outcome;     // [P]
  int* n_clamped;   // [P]
  double* speeds;   // [P][window] ring
  int* sp_count;    // [P] valid entries in the ring (<= window)
  int* sp_head;     // [P] next write position
  double* rec;      // [P][record+1][9]: x, v, accel per recorded tick
  unsigned* n_active;  // running count (device)
};

__device__ __forceinline__ double norm3(double a, double b, double c) {
  return sqrt(a * a + b * b + c * c);
}

__device__ inline void record_sample(const RolloutState& s, const RolloutCfg& cfg, int p, int k,
                                     const double* x, const double* v, const double* a) {
  if (!s.rec || k > cfg.record) return;
  double* r = s.rec + ((size_t)p * (cfg.record + 1) + k) * 9;
  for (int i = 0; i < 3; ++i) { r[i] = x[i]; r[3 + i] = v[i]; r[6 + i] = a[i]; }
}

// Termination checks at the start of a tick (sim.py:236-250).  One warp per
// robot: the analytic scene distance (a sequential fold over the scene's
// primitives) is computed 32 primitives at a time (scene_sd_warp, bitwise
// scene_sd); lane 0 does the rest.
constexpr int kCheckBlock = 128;
__global__ void __launch_bounds__(kCheckBlock)
k_rollout_check(ScenePack scene, RolloutState s, RolloutCfg cfg, int P) {
  const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= P || !s.active[p]) return;  // warp-uniform
  const int k = s.k[p];
  const double t = (double)k * cfg.dt;
  const double* x = s.x + 3 * p;
  const double* g = s.goal + 3 * p;
  const double sd = scene_sd_warp(scene, t, x[0], x[1], x[2]);
  if ((threadIdx.x & 31) != 0) return;
  int out = OUT_RUNNING;
  if (sd <= cfg.robot_radius) {
    out = OUT_COLLISION;
  } else if (!cfg.hold && norm3(x[0] - g[0], x[1] - g[1], x[2] - g[2]) <= cfg.goal_tol) {
    out = OUT_SUCCESS;
  } else if (k >= cfg.max_steps) {
    out = cfg.hold ? OUT_SUCCESS : OUT_TIMEOUT;
  } else if (!cfg.hold && s.sp_count[p] == cfg.window) {
    double sum = 0.0;
    const double* sp = s.speeds + (size_t)p * cfg.window;
    const int h = s.sp_head[p];  // oldest entry when the ring is full
    for (int i = 0; i < cfg.window; ++i) sum += sp[(h + i) % cfg.window];
    if (sum / (double)cfg.window < cfg.stuck_speed) out = OUT_STUCK;
  }
  if (out != OUT_RUNNING) {
    s.outcome[p] = out;
    s.active[p] = 0;
    const double zero[3] = {0.0, 0.0, 0.0};
    record_sample(s, cfg, p, k, x, s.v + 3 * p, zero);  // terminal sample
  } else {
    atomicAdd(s.n_active, 1u);
  }
}

// (I + M)^-1 f for symmetric PSD M: I + M is SPD with eigenvalues >= 1, so
// pinv_psd's cutoff never applies (core.py:103-115) and a Cholesky solve is
// the same operator.
__device__ inline void spd_solve3(const double m[9], const double f[3], double out[3]) {
  double a00 = 1.0 + m[0], a01 = m[1], a02 = m[2], a11 = 1.0 + m[4], a12 = m[5], a22 = 1.0 + m[8];
  double l00 = sqrt(a00);
  double l10 = a01 / l00, l20 = a02 / l00;
  double l11 = sqrt(a11 - l10 * l10);
  double l21 = (a12 - l20 * l10) / l11;
  double l22 = sqrt(a22 - l20 * l20 - l21 * l21);
  double y0 = f[0] / l00;
  double y1 = (f[1] - l10 * y0) / l11;
  double y2 = (f[2] - l20 * y0 - l21 * y1) / l22;
  out[2] = y2 / l22;
  out[1] = (y1 - l21 * out[2]) / l11;
  out[0] = (y0 - l10 * out[1] - l20 * out[2]) / l00;
}

// combine + clamp + step (sim.py:262-285, core.py:130-144, policies.py:127-132).
__global__ void k_rollout_update(RolloutState s, RolloutCfg cfg, const double* __restrict__ slots,
                                 const double* __restrict__ accels, int P) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P || !s.active[p]) return;
  double* x = s.x + 3 * p;
  double* v = s.v + 3 * p;
  const double* g = s.goal + 3 * p;
  const double* sl = slots + 13 * p;
  const double* ao = accels + 3 * p;
  // attractor: alpha * soft_normalize(goal - x, c) - beta * v  (core.py:86-100)
  double e[3] = {g[0] - x[0], g[1] - x[1], g[2] - x[2]};
  double n = norm3(e[0], e[1], e[2]);
  double den = n + cfg.c * log1p(exp(-2.0 * cfg.c * n));
  double fa[3];
  for (int i = 0; i < 3; ++i) fa[i] = cfg.alpha * (e[i] / den) - cfg.beta * v[i];
  // obstacle policy metric (symmetrised, core.py:47-56) and metric-weighted accel
  double m[9];
  for (int r = 0; r < 3; ++r)
    for (int q = 0; q < 3; ++q) m[3 * r + q] = 0.5 * (sl[3 * r + q] + sl[3 * q + r]);
  double f[3];
  for (int i = 0; i < 3; ++i) f[i] = fa[i] + (m[3 * i] * ao[0] + m[3 * i + 1] * ao[1] + m[3 * i + 2] * ao[2]);
  double a[3];
  spd_solve3(m, f, a);
  const double mag = norm3(a[0], a[1], a[2]);
  if (mag > cfg.max_accel) {
    const double sc = cfg.max_accel / mag;
    a[0] *= sc; a[1] *= sc; a[2] *= sc;
    s.n_clamped[p] += 1;
  }
  const int k = s.k[p];
  record_sample(s, cfg, p, k, x, v, a);
  for (int i = 0; i < 3; ++i) v[i] = v[i] + a[i] * cfg.dt;  // velocity first (sim.py:155-161)
  for (int i = 0; i < 3; ++i) x[i] = x[i] + v[i] * cfg.dt;
  double* sp = s.speeds + (size_t)p * cfg.window;
  sp[s.sp_head[p]] = norm3(v[0], v[1], v[2]);
  s.sp_head[p] = (s.sp_head[p] + 1) % cfg.window;
  if (s.sp_count[p] < cfg.window) s.sp_count[p] += 1;
  s.k[p] = k + 1;
}

}  // namespace rmpb
