/*
 * rmpb.h -- C ABI of the B200-native raycasting-RMP evaluator (librmpb.so).
 *
 * This is the drop-in boundary for the reference's kernel-backend protocol
 * (rmpnav/_kernels/__init__.py:17-59; the "compiled" backend
 * rmpnav/_kernels/ckern.py:19-93 and its NumPy twin npkern.py:21-221).  A
 * backend there is a module with 7 functions; each is served here by one
 * or more entry points (paths relative to /root/reference/pkg/src/):
 *
 *   grid_trace        (ckern.py:49-62)  -> rmpb_grid_trace            [unfused parity]
 *   policy_reduce     (ckern.py:80-93)  -> rmpb_policy_reduce         [unfused parity]
 *   ray_policy        (policies.py:182-192: grid_trace+policy_reduce+pinv_psd)
 *                                       -> rmpb_ray_policy            [fused K1]
 *   lidar_policy      (policies.py:195-205) -> rmpb_lidar_policy      [K2]
 *   pinv_psd          (core.py:103-115) -> rmpb_pinv_psd
 *   bake_values       (ckern.py:25-35)  -> rmpb_bake / rmpb_bake_grid [row f2]
 *   scene_distance_many (ckern.py:19-23)-> rmpb_scene_distance        [row f3]
 *   scene_trace       (ckern.py:65-77)  -> rmpb_scene_trace           [row f3]
 *   esdf_sample_many  (ckern.py:38-46)  -> rmpb_esdf_sample           [row f4]
 *
 * plus batched / device-resident entries the reference does not have
 * (multi-pose K3, ray-range partials + fixed-order fold for GPU splits,
 * LiDAR from raw points, device-side Halton bundles).
 *
 * Conventions
 *   - Plain C: pointers, sizes, doubles.  No C++ or torch types.
 *   - Every function returns int status: RMPB_OK (0) or a negative code;
 *     rmpb_last_error() gives a thread-local message.  The reference raises
 *     ValueError for bad arguments (rmpnav/_kernels/__init__.py:45-48 and
 *     Cython buffer checks); the Python host layer maps RMPB_ERR_INVALID to
 *     ValueError and everything else to RuntimeError.
 *   - Host-buffer entries copy inputs in, run, copy results out and return
 *     when results are on the host (the caller owns all host buffers).
 *   - *_device entries take device pointers (e.g. torch tensors' data_ptr)
 *     and are asynchronous on `stream`.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls on
 *     distinct streams are thread-safe.
 *   - Handles (grid, bundle, scene) are library-owned device objects bound
 *     to one CUDA device.
 *   - Params are the reference kernel argument order (policies.py:80-83):
 *     {eta_rep, nu_rep, eta_damp, nu_damp, epsilon, radius, c}.
 *   - Slots are the reference's 13-double layout (ckern.py:91-93, before
 *     reshaping): [A (3x3 row-major, symmetric), A f (3), n_hits].
 */
#ifndef RMPB_H
#define RMPB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define RMPB_EXPORT __attribute__((visibility("default")))
#else
#define RMPB_EXPORT
#endif

#define RMPB_API_VERSION 1

enum {
  RMPB_OK = 0,
  RMPB_ERR_INVALID = -1,     /* bad argument (ValueError in the reference) */
  RMPB_ERR_CUDA = -2,        /* CUDA runtime / launch failure */
  RMPB_ERR_NOMEM = -3,       /* device or pinned allocation failed */
  RMPB_ERR_UNSUPPORTED = -4  /* option not available for this handle */
};

enum { RMPB_F32 = 0, RMPB_F64 = 1 };                              /* value dtypes */
enum { RMPB_STORE_AUTO = 0, RMPB_STORE_F32 = 1, RMPB_STORE_F64 = 2 }; /* grid storage */
enum { RMPB_LAYOUT_LINEAR = 0, RMPB_LAYOUT_QUAD = 1, RMPB_LAYOUT_BRICK = 2,
       RMPB_LAYOUT_PAIR64 = 4, RMPB_LAYOUT_AUTO = -1 };
enum { RMPB_ORDER_IDENTITY = 0, RMPB_ORDER_MORTON = 1 };          /* bundle evaluation order */
/* EXACT: bit-identical to the reference (fp64, its operation order).  FAST:
 * fp32 march with FMA, opt-in, NOT reference-exact (grazing rays may differ;
 * deviation measured in tests/test_gpu_parity.py). */
enum { RMPB_MODE_EXACT = 0, RMPB_MODE_FAST = 1 };

typedef struct rmpb_grid rmpb_grid;
typedef struct rmpb_bundle rmpb_bundle;
typedef struct rmpb_scene rmpb_scene;

/* ---- library ---------------------------------------------------------- */
RMPB_EXPORT const char* rmpb_last_error(void);
RMPB_EXPORT int rmpb_api_version(void);
RMPB_EXPORT int rmpb_device_count(int* n);
/* Number of kernels this library has launched (all devices, since load). */
RMPB_EXPORT uint64_t rmpb_launch_count(void);
/* Tuning knobs: "seg_rays" (rays per CTA unit, 0 = heuristic), "kernel"
 * (0 auto, 1 one ray per thread, 2 lane refill), "lidar_warps" (target warp
 * units per LiDAR launch), "lidar_persist" (0/1: persistent LiDAR warps
 * claiming units from a counter), "l2_window" (0/1: the map's L2 access-policy
 * window), "graphs" (0/1: CUDA-graph rollout ticks), "carveout" (-1 or the
 * shared-memory carveout % of the trace kernel).  Results do not depend on
 * them beyond the last bits of the sums (fixed per setting). */
RMPB_EXPORT int rmpb_set_option(const char* name, int64_t value);

/* ---- maps (EsdfGrid, rmpnav/geometry.py:215-255) ------------------------ */
/* values: nx*ny*nz C-order (z fastest), dtype RMPB_F32/RMPB_F64, host memory.
 * STORE_AUTO keeps f32 iff every value is exactly f32-representable (so the
 * trace stays bit-identical to the f64 reference); STORE_F32 on values that
 * are not f32-exact fails with RMPB_ERR_INVALID.  BRICK layout allocates
 * only 8^3 bricks containing a value != `fill` (see rmpb_grid_create_brick). */
RMPB_EXPORT int rmpb_grid_create(const void* values, int dtype, int64_t nx, int64_t ny, int64_t nz,
                     double ox, double oy, double oz, double res,
                     int storage, int layout, int device, rmpb_grid** out);
/* Same, values already in device memory (e.g. a torch tensor) on `device`. */
RMPB_EXPORT int rmpb_grid_create_device(const void* d_values, int dtype, int64_t nx, int64_t ny, int64_t nz,
                            double ox, double oy, double oz, double res,
                            int storage, int layout, int device, rmpb_grid** out);
/* Block-hashed (BRICK) map: bricks whose 8^3 nodes all equal `fill` (the
 * TSDF truncation value for unobserved space) are not stored. */
RMPB_EXPORT int rmpb_grid_create_brick(const void* values, int dtype, int64_t nx, int64_t ny, int64_t nz,
                           double ox, double oy, double oz, double res, double fill,
                           int storage, int device, rmpb_grid** out);
/* Re-upload all values into an existing grid (same shape), in place: every
 * holder of the handle sees the new map (a QUAD grid whose new values are
 * not f32-exact switches to the f64 layout; a BRICK grid is unsupported). */
RMPB_EXPORT int rmpb_grid_update(rmpb_grid* g, const void* values, int dtype);
/* Overwrite the node sub-box [i0, i0+ni) x [j0, j0+nj) x [k0, k0+nk) of an
 * existing LINEAR / QUAD / PAIR64 grid with `values` (f64, C-order, ni*nj*nk)
 * in place: only those nodes cross PCIe.  RMPB_ERR_UNSUPPORTED (grid left
 * unchanged) for a BRICK grid or an f32 grid and values that are not
 * f32-exact: recreate the grid then.  Synchronous; the caller orders it
 * after in-flight launches that read the grid.  Replaces the reference's
 * in-place edit of EsdfGrid.values (rmpnav/geometry.py:215-240, re-read by
 * every grid_trace call, rmpnav/_kernels/ckern.py:49-62). */
RMPB_EXPORT int rmpb_grid_update_region(rmpb_grid* g, const void* values, int dtype, int64_t i0,
                                        int64_t j0, int64_t k0, int64_t ni, int64_t nj, int64_t nk);
/* Host-only: *out = 1 when the 2-op exact division (q = fma(a, yhi, a*ylo))
 * is proven correctly rounded for divisor `res` (every normal |a| >=
 * 2^-960); maps with such a resolution trace with it.  Exactness is the
 * same either way (rmpnav/_kernels/_ckern.pyx:92-135 divides with IEEE /). */
RMPB_EXPORT int rmpb_div2_exact(double res, int* out);
RMPB_EXPORT int rmpb_grid_info(const rmpb_grid* g, int* storage, int* layout, int64_t* device_bytes,
                   int64_t* allocated_bricks);
RMPB_EXPORT int rmpb_grid_destroy(rmpb_grid* g);

/* ---- ray bundles (RayBundle / sample_directions, rmpnav/rays.py:63-96) -- */
RMPB_EXPORT int rmpb_bundle_create(const double* dirs, int64_t n, int order, int device, rmpb_bundle** out);
/* Halton bundle generated on device: i = 1..n, polar = acos(1-2 h2), az = 2 pi h3. */
RMPB_EXPORT int rmpb_bundle_halton(int64_t n, int order, int device, rmpb_bundle** out);
/* Spherical-grid bundle generated on device: the LiDAR lattice of
 * rmpnav/rays.py:176-199 (scan_pattern(rows, cols, vfov_deg)), row-major. */
RMPB_EXPORT int rmpb_bundle_lattice(int64_t rows, int64_t cols, double vfov_deg, int order, int device,
                        rmpb_bundle** out);
RMPB_EXPORT int64_t rmpb_bundle_size(const rmpb_bundle* b);
/* Directions back to host in ORIGINAL order (n x 3). */
RMPB_EXPORT int rmpb_bundle_directions(const rmpb_bundle* b, double* out);
RMPB_EXPORT int rmpb_bundle_destroy(rmpb_bundle* b);

/* ---- fused map-based policy (K1/K3) ------------------------------------- */
/* ray_policy (policies.py:182-192): trace + per-ray policy + reduce + pinv in
 * one launch.  eps / step_scale as rays.py:117-120 (0.5*res, 0.9).  Optional
 * per-ray outputs in ORIGINAL ray order: t (+inf = miss), hit cell (3 int32,
 * -1 on miss), interpolation steps.
 * Policy-only callers (who use the slot's sums / the acceleration, not the
 * per-ray outputs or slot[12]) may pass max_range = min(max_range, radius),
 * radius = params[5]: a hit at d >= radius has activation weight 0
 * (_ckern.pyx:300-306), so the sums are those of the full range while every
 * ray stops at the radius (Python: policy_only=True, rays.policy_range). */
RMPB_EXPORT int rmpb_ray_policy(const rmpb_grid* g, const rmpb_bundle* b, const double x[3], const double v[3],
                    const double params[7], double max_range, double eps, double step_scale,
                    double out_slot[13], double out_accel[3],
                    double* opt_t, int32_t* opt_cell, int32_t* opt_steps, void* stream);
/* P poses against one map and bundle (config C4); host buffers x, v: P x 3;
 * out_slot: P x 13; out_accel: P x 3. */
RMPB_EXPORT int rmpb_ray_policy_batch(const rmpb_grid* g, const rmpb_bundle* b, const double* x,
                          const double* v, int64_t P, const double params[7], double max_range,
                          double eps, double step_scale, double* out_slot, double* out_accel,
                          void* stream);
/* Same with device pointers; asynchronous.  opt_step_total (device u64, may
 * be NULL) accumulates the number of voxel-steps executed. */
RMPB_EXPORT int rmpb_ray_policy_batch_device(const rmpb_grid* g, const rmpb_bundle* b, const double* d_x,
                                 const double* d_v, int64_t P, const double params[7],
                                 double max_range, double eps, double step_scale, double* d_slot,
                                 double* d_accel, uint64_t* opt_step_total, void* stream);
/* Same with an explicit mode (RMPB_MODE_EXACT / RMPB_MODE_FAST). */
RMPB_EXPORT int rmpb_ray_policy_batch_device_mode(const rmpb_grid* g, const rmpb_bundle* b,
                                      const double* d_x, const double* d_v, int64_t P,
                                      const double params[7], double max_range, double eps,
                                      double step_scale, int mode, double* d_slot,
                                      double* d_accel, uint64_t* opt_step_total, void* stream);
/* Partial slot of stored rays [ray_begin, ray_end) of one pose (no pinv):
 * the per-GPU share of a ray-split pose (config C5).  Device pointers. */
RMPB_EXPORT int rmpb_ray_policy_range_device(const rmpb_grid* g, const rmpb_bundle* b, const double* d_x,
                                 const double* d_v, int64_t ray_begin, int64_t ray_end,
                                 const double params[7], double max_range, double eps,
                                 double step_scale, double* d_slot, void* stream);
/* Fixed-order pairwise fold (rmpnav/_kernels/_pool.py:61-72 shape) of n
 * 13-slots + pinv.  Device pointers (n <= 64). */
RMPB_EXPORT int rmpb_fold_resolve_device(const double* d_slots, int64_t n, double* d_slot, double* d_accel,
                             void* stream);

/* ---- latency server (single-pose ray_policy without per-call launches) -- */
/* One resident cooperative kernel on its own stream serves ray_policy
 * requests (the reference's control-loop call, policies.py:182-192) posted
 * through pinned mapped host memory: no kernel launch and no stream
 * synchronisation per call.  Results are bitwise those of rmpb_ray_policy
 * (same kernel body and segmentation).  The kernel holds its CTAs' SM
 * resources while it runs and exits after idle_timeout_s without a request
 * (the next eval relaunches it) or at rmpb_server_stop.  One caller thread
 * per server. */
typedef struct rmpb_server rmpb_server;
RMPB_EXPORT int rmpb_server_start(const rmpb_grid* g, const rmpb_bundle* b, const double params[7],
                      double max_range, double eps, double step_scale, double idle_timeout_s,
                      rmpb_server** out);
RMPB_EXPORT int rmpb_server_eval(rmpb_server* s, const double x[3], const double v[3],
                     double out_slot[13], double out_accel[3]);
RMPB_EXPORT int rmpb_server_stop(rmpb_server* s);

/* ---- fused ray-split exchange over peer memory (K4; config C5) --------- */
/* The all-gather + fold of the ray-split path (rmpnav/_kernels/_pool.py:
 * 61-72 partial-slot contract) done inside the trace kernel's epilogue: each
 * rank's final CTA stores its 13-slot into every rank's mailbox over NVLink
 * (P2P through CUDA IPC), publishes an epoch, waits for all `world` epochs
 * and folds in rank order + solves.  One mailbox per rank (device memory);
 * ranks exchange the 64-byte IPC handles once (e.g. all_gather_object) and
 * open each other's mailboxes; same-process peers use rmpb_peer_attach. */
#define RMPB_IPC_HANDLE_BYTES 64
typedef struct rmpb_peer rmpb_peer;
RMPB_EXPORT int rmpb_peer_create(int world, int rank, int device, void* ipc_handle_out, rmpb_peer** out);
RMPB_EXPORT int rmpb_peer_open_ipc(rmpb_peer* p, int peer_rank, const void* ipc_handle);
RMPB_EXPORT int rmpb_peer_attach(rmpb_peer* p, int peer_rank, const rmpb_peer* other);
/* 1 if a wait gave up (a peer never published its epoch within 10 s; the
 * slot / accel of that call are NaN). */
RMPB_EXPORT int rmpb_peer_error(rmpb_peer* p, int* timed_out);
RMPB_EXPORT int rmpb_peer_destroy(rmpb_peer* p);
/* This rank's rays [ray_begin, ray_end) of one pose + the exchange + fold +
 * pinv in ONE launch; every rank passes the same epoch (>= 1, +1 per call).
 * mode: 3 = post + wait (production); 1 = post only, 2 = wait only (lets
 * one-GPU tests run the ranks one after another, never concurrently). */
RMPB_EXPORT int rmpb_ray_policy_range_exchange(const rmpb_grid* g, const rmpb_bundle* b, const double* d_x,
                                   const double* d_v, int64_t ray_begin, int64_t ray_end,
                                   const double params[7], double max_range, double eps,
                                   double step_scale, rmpb_peer* peer, uint64_t epoch, int mode,
                                   double* d_slot, double* d_accel, void* stream);

/* ---- LiDAR-direct policy (K2; policies.py:195-205) ----------------------- */
/* dirs: n x 3 sensor-frame directions (world when R == NULL); R: 3x3
 * row-major sensor orientation (world = dirs @ R^T, rays.py:172-173);
 * valid: n bytes or NULL; min_range default 0.3 (policies.py:39). */
RMPB_EXPORT int rmpb_lidar_policy(const double* dirs, const double* R, const double* ranges,
                      const uint8_t* valid, int64_t n, const double v[3], const double params[7],
                      double min_range, double out_slot[13], double out_accel[3], void* stream);
/* Same with the sensor lattice kept on device as a bundle (IDENTITY order). */
RMPB_EXPORT int rmpb_lidar_policy_bundle(const rmpb_bundle* pattern, const double* R, const double* ranges,
                             const uint8_t* valid, const double v[3], const double params[7],
                             double min_range, double out_slot[13], double out_accel[3],
                             void* stream);
/* S scans per launch, device pointers: dirs n x 3 (shared), R S x 9 (or
 * NULL), ranges S x n, valid S x n (or NULL), v S x 3. */
RMPB_EXPORT int rmpb_lidar_policy_batch_device(const double* d_dirs, const double* d_R, const double* d_ranges,
                                   const uint8_t* d_valid, int64_t n, int64_t S, const double* d_v,
                                   const double params[7], double min_range, double* d_slot,
                                   double* d_accel, void* stream);
/* Same with a mode: RMPB_MODE_EXACT, or RMPB_MODE_FAST = the per-beam policy
 * math (exp / log1p / divisions) in fp32 with fp64 accumulation -- the same
 * beams contribute (the count / radius / closing tests stay fp64), each with
 * ~1e-7 relative error (north_star's bar for the sums: 1e-5); opt-in, NOT
 * reference-exact. */
RMPB_EXPORT int rmpb_lidar_policy_batch_device_mode(const double* d_dirs, const double* d_R,
                                   const double* d_ranges, const uint8_t* d_valid, int64_t n,
                                   int64_t S, const double* d_v, const double params[7],
                                   double min_range, double* d_slot, double* d_accel, void* stream,
                                   int mode);
/* Raw sensor-frame points (f32 xyz, S x n x 3): dir = p * (1/|p|), range = |p|;
 * zero or non-finite points are invalid. */
RMPB_EXPORT int rmpb_lidar_points(const float* xyz, const double* R, int64_t n, const double v[3],
                      const double params[7], double min_range, double out_slot[13],
                      double out_accel[3], void* stream);
RMPB_EXPORT int rmpb_lidar_points_batch_device(const float* d_xyz, const double* d_R, int64_t n, int64_t S,
                                   const double* d_v, const double params[7], double min_range,
                                   double* d_slot, double* d_accel, void* stream);
RMPB_EXPORT int rmpb_lidar_points_batch_device_mode(const float* d_xyz, const double* d_R, int64_t n,
                                   int64_t S, const double* d_v, const double params[7],
                                   double min_range, double* d_slot, double* d_accel, void* stream,
                                   int mode);

/* ---- unfused protocol entries (parity) ---------------------------------- */
RMPB_EXPORT int rmpb_grid_trace(const rmpb_grid* g, const double* dirs, int64_t n, const double start[3],
                    double max_range, double eps, double step_scale, double* out_t,
                    int32_t* out_cell, int32_t* out_steps, void* stream);
RMPB_EXPORT int rmpb_policy_reduce(const double* dirs, const double* dists, int64_t n, const double v[3],
                       const double params[7], double min_range, double out_slot[13],
                       void* stream);
/* n symmetric 3x3 matrices (row-major) -> their PSD pseudo-inverses. */
RMPB_EXPORT int rmpb_pinv_psd(const double* a, int64_t n, double* out, void* stream);
/* Same with the reference's rcond argument (core.py:103-115: eigenvalues at
 * or below rcond * max(lambda_max, 0) are dropped); rmpb_pinv_psd = 1e-8. */
RMPB_EXPORT int rmpb_pinv_psd_rcond(const double* a, int64_t n, double rcond, double* out,
                                    void* stream);

/* ---- analytic scene + map construction (rows f2-f4) --------------------- */
/* Scene pack as rmpnav/geometry.py:177-197: kinds (0 sphere, 1 box), ops
 * (0 union, 1 subtract), centers/sizes/velocities P x 3, empty distance. */
RMPB_EXPORT int rmpb_scene_create(const int8_t* kinds, const int8_t* ops, const double* centers,
                      const double* sizes, const double* velocities, int64_t n, double empty,
                      int device, rmpb_scene** out);
RMPB_EXPORT int rmpb_scene_destroy(rmpb_scene* s);
RMPB_EXPORT int rmpb_scene_distance(const rmpb_scene* s, const double* pts, int64_t n, double t, double* out,
                        void* stream);
RMPB_EXPORT int rmpb_scene_trace(const rmpb_scene* s, const double start[3], const double* dirs, int64_t n,
                     double max_range, double eps, double t, double step_scale, double* out,
                     void* stream);
/* bake_values (_ckern.pyx:71-87) into a host f64 array nx*ny*nz. */
RMPB_EXPORT int rmpb_bake(const rmpb_scene* s, double ox, double oy, double oz, double res, int64_t nx,
              int64_t ny, int64_t nz, double* out_values, void* stream);
/* Bake straight into a device grid; storage RMPB_STORE_F32 ROUNDS to f32. */
RMPB_EXPORT int rmpb_bake_grid(const rmpb_scene* s, double ox, double oy, double oz, double res, int64_t nx,
                   int64_t ny, int64_t nz, int storage, int layout, int device, rmpb_grid** out);
/* Truncated bake for TSDF maps (config C5): values clamp(sd, -tau, tau),
 * brick-culled (exact w.r.t. the unculled bake + clamp); storage F32 rounds
 * once to f32; layout BRICK (default) stores only bricks != +tau. */
RMPB_EXPORT int rmpb_bake_grid_tsdf(const rmpb_scene* s, double ox, double oy, double oz, double res,
                        int64_t nx, int64_t ny, int64_t nz, double tau, int storage, int layout,
                        int device, rmpb_grid** out);
/* Node values of any grid back to the host as f64, C-order (nx*ny*nz). */
RMPB_EXPORT int rmpb_grid_values(const rmpb_grid* g, double* out);
RMPB_EXPORT int rmpb_esdf_sample(const rmpb_grid* g, const double* pts, int64_t n, double* out_d,
                     double* out_g, uint8_t* out_flag, void* stream);

/* ---- batched closed-loop rollouts on device (row f1; sim.py:155-306) ----- */
/* P robots from start[P*3] toward goal[P*3] on one map / bundle / scene:
 * per tick the collision / goal / time-out / stuck checks, the fused ray
 * policy, combine with the goal attractor {alpha, beta, c}, the |a| clamp
 * and the semi-implicit Euler step run on the GPU with no host round trip.
 * cfg = {dt, max_time, robot_radius, goal_tolerance, max_accel,
 * stuck_window, stuck_speed, max_range, hold_mode} (RolloutConfig,
 * sim.py:102-134).  record_ticks > 0 keeps (x, v, accel) of the first ticks. */
typedef struct rmpb_rollout rmpb_rollout;
RMPB_EXPORT int rmpb_rollout_create(const rmpb_grid* g, const rmpb_bundle* b, const rmpb_scene* scene,
                        int64_t P, const double* start, const double* goal,
                        const double attractor[3], const double params[7], const double cfg[9],
                        int64_t record_ticks, rmpb_rollout** out);
/* Advance up to max_ticks control ticks (stops early once every robot is done). */
RMPB_EXPORT int rmpb_rollout_run(rmpb_rollout* r, int64_t max_ticks, int64_t* active_left, void* stream);
/* outcome: 0 running, 1 SUCCESS, 2 COLLISION, 3 TIMEOUT, 4 STUCK (sim.py:51-55). */
RMPB_EXPORT int rmpb_rollout_result(const rmpb_rollout* r, int32_t* outcome, int64_t* steps,
                        int64_t* n_clamped, double* x, double* v);
/* rec: P x (record_ticks + 1) x 9 doubles (x, v, accel per tick). */
RMPB_EXPORT int rmpb_rollout_trajectory(const rmpb_rollout* r, double* rec);
RMPB_EXPORT int rmpb_rollout_destroy(rmpb_rollout* r);

/* ---- K5: Amanatides-Woo DDA over bit-packed occupancy ------------------
 * The traversal north_star names; NOT the reference's (sphere tracing,
 * SPEC.md:228), so it is opt-in and reported separately.  Occupied = node
 * value <= 0 (geometry.py:312-315), voxel of node (i,j,k) = res-cube centred
 * on it.  float32 march, bit-exact against oracle/rmp_oracle.c
 * orc_dda_trace: entry distance of the first occupied voxel (+inf = miss)
 * and its index (-1 = miss). */
typedef struct rmpb_occupancy rmpb_occupancy;
RMPB_EXPORT int rmpb_occupancy_create(const rmpb_grid* g, rmpb_occupancy** out);
RMPB_EXPORT int rmpb_occupancy_destroy(rmpb_occupancy* o);
/* nx*ny*ceil(nz/32) words, bit k%32 of word (i*ny + j)*nzw + k/32. */
RMPB_EXPORT int rmpb_occupancy_bits(const rmpb_occupancy* o, uint32_t* out);
RMPB_EXPORT int rmpb_dda_trace(const rmpb_occupancy* o, const double* dirs, int64_t n, const double start[3],
                   double max_range, float* out_t, int32_t* out_voxel, int32_t* out_steps,
                   void* stream);
/* Fused DDA + per-ray policy + reduction + pinv for P poses (device ptrs). */
RMPB_EXPORT int rmpb_ray_policy_dda_batch_device(const rmpb_occupancy* o, const rmpb_bundle* b,
                                     const double* d_x, const double* d_v, int64_t P,
                                     const double params[7], double max_range, double* d_slot,
                                     double* d_accel, void* stream);

/* ---- measurement helper (not part of the reference interface) ----------
 * L2 bandwidth probe over a caller-owned device buffer (keep it well below
 * the 126 MB L2): mode 0 streams 16-B reads, mode 1 issues independent
 * pseudo-random 16-B reads (the trace kernel's gather shape).  Enqueued on
 * `stream`; the caller times it.  *bytes_read = bytes the launch requests. */
RMPB_EXPORT int rmpb_l2_probe(const void* d_buf, int64_t bytes, int reps, int mode,
                              int64_t* bytes_read, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RMPB_H */
