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
#include <type_traits>

#include "rmpb_device.cuh"

namespace rmpb {

// ---------------------------------------------------------------------------
// K4 fused: ray-split partial -> peer-memory exchange -> fold -> solve, in the
// epilogue of the trace kernel (config C5).  Every rank owns
// one mailbox in its device memory: flags [2][world] (u64 epochs) then slots
// [2][world][16] doubles, double-buffered on the epoch parity.  Warp 0 of
// the pose's final CTA stores the 13-slot into mailbox[rank] of EVERY rank
// (lane r -> rank r: NVLink P2P stores through IPC-mapped pointers), fences
// at system scope and publishes the epoch flag (relaxed store after the
// fence), then polls all `world` flags of its own mailbox (lane r -> flag r),
// fences, and folds the slots in rank order with the reference's pairwise
// shape (_pool.py:61-72; lane j -> component j) -- the same result as the
// all-gather path, identical on every rank.  Parity double-buffering makes reuse safe: a rank
// can only start epoch e+2 (same parity) after every rank published e+1,
// i.e. finished reading epoch e.
constexpr int kMaxPeers = 8;
constexpr int kMbox = 16;  // doubles per slot record (13 used)
enum : int { EX_POST = 1, EX_WAIT = 2 };

struct PeerEx {
  double* slots[kMaxPeers];               // each rank's [2][world][kMbox]
  unsigned long long* flags[kMaxPeers];   // each rank's [2][world]
  int world, rank;
  unsigned* err;                          // device word: 1 = wait timed out
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Fence-based flag protocol (PTX memory model: data stores; fence; relaxed
// flag store || relaxed flag load; fence; data loads): one system-scope
// fence per side instead of an implied fence per flag.
__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Last-arriver tickets: every arriver publishes its partial with a RELEASE
// atomic (orders its prior stores; no L1 invalidation), and only the last
// arriver issues an ACQUIRE fence before reading the others' partials.  The
// former __threadfence() + atomicAdd emitted MEMBAR.SC.GPU + CCTL.IVALL at
// every arrival, invalidating the whole SM's L1 (the map / lattice lines
// the other CTAs were using) once per unit.
__device__ __forceinline__ unsigned ticket_add_release(unsigned* p) {
  unsigned old;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}
__device__ __forceinline__ void fence_acquire_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Fixed pairwise fold (rmpnav/_kernels/_pool.py:61-72: s[2k] + s[2k+1], odd
// tail carried) of n <= MAXN 13-slots at `stride` doubles; one thread.
// (The buffer is thread-local: keep MAXN small where it is inlined into the
// trace kernels -- it sizes their stack frame.)
template <int MAXN>
__device__ inline void fold_slots(const double* slots, int n, int stride, bool bypass_l1,
                                  double out[13]) {
  double buf[MAXN * 13];
  int m = n < MAXN ? n : MAXN;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < 13; ++j)
      buf[i * 13 + j] = bypass_l1 ? __ldcg(slots + (size_t)i * stride + j) : slots[(size_t)i * stride + j];
  while (m > 1) {
    int half = m / 2;
    for (int k = 0; k < half; ++k)
      for (int j = 0; j < 13; ++j) buf[k * 13 + j] = buf[2 * k * 13 + j] + buf[(2 * k + 1) * 13 + j];
    if (m % 2)
      for (int j = 0; j < 13; ++j) buf[half * 13 + j] = buf[(m - 1) * 13 + j];
    m = half + (m % 2);
  }
  for (int j = 0; j < 13; ++j) out[j] = buf[j];
}

// The same fold for n <= kMaxPeers (8) slots held in registers: every index
// is a compile-time constant (no local-memory buffer in the trace kernels).
__device__ __forceinline__ double fold8(const double* p, int n, int stride) {
  double v[kMaxPeers];
#pragma unroll
  for (int i = 0; i < kMaxPeers; ++i) v[i] = i < n ? __ldcg(p + (size_t)i * stride) : 0.0;
  int m = n;
#pragma unroll
  for (int level = 0; level < 3; ++level) {  // 8 -> 4 -> 2 -> 1
    const int half = m >> 1, odd = m & 1;
    double last = 0.0;
#pragma unroll
    for (int i = 0; i < kMaxPeers; ++i)
      if (i == m - 1) last = v[i];
#pragma unroll
    for (int k = 0; k < kMaxPeers / 2; ++k)
      v[k] = k < half ? v[2 * k] + v[2 * k + 1] : (k == half && odd ? last : v[k]);
    m = half + odd;
  }
  return v[0];
}

#ifdef RMPB_DBG_TIMELINE
// (timing probe builds only) [0] min CTA start, [1] max trace end, [2] last
// CTA after the ticket, [3] after the fold, [4] after write_slot
__device__ unsigned long long g_tl[8];
#define RMPB_TL_MIN(k) atomicMin(&g_tl[k], globaltimer_ns())
#define RMPB_TL_MAX(k) atomicMax(&g_tl[k], globaltimer_ns())
#else
#define RMPB_TL_MIN(k)
#define RMPB_TL_MAX(k)
#endif

struct ExArgs {  // per-call exchange arguments (kernel parameter of the lean kernel)
  const PeerEx* ex;
  unsigned long long epoch;
  int mode;  // EX_POST | EX_WAIT (split only for one-GPU tests)
};

struct PoseIO;
__device__ void exchange_emit_warp(const Acc& s, const PoseIO& io, const ExArgs& xa);

struct PoseIO {
  const double* __restrict__ x;   // [P][3] positions
  const double* __restrict__ v;   // [P][3] velocities
  double* __restrict__ slot;      // [P][13] (may be null when only partials wanted)
  double* __restrict__ accel;     // [P][3]  (null: skip pinv)
  double* __restrict__ partials;  // [P*segs][10] when segs > 1
  unsigned* __restrict__ tickets; // [P] zero-initialised, self-resetting
  double* __restrict__ seg_out;   // [P*segs][10] raw segment partials (ray-split), or null
  double x0[3], v0[3];            // single pose by value when x / v are null
  const int* __restrict__ active; // [P] skip poses whose flag is 0 (rollouts), or null
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
  const int* __restrict__ perm;    // stored index -> original index (null = identity)
  int n;
};

__device__ __forceinline__ void acc_to_arr(const Acc& a, double* o) {
  o[0] = a.a00; o[1] = a.a01; o[2] = a.a02; o[3] = a.a11; o[4] = a.a12;
  o[5] = a.a22; o[6] = a.b0; o[7] = a.b1; o[8] = a.b2; o[9] = (double)a.cnt;
}

// Finish a unit: reduce the CTA, then either resolve the pose or publish a
// partial and let the last CTA of the pose fold + resolve.
// Returns true in the one thread that wrote the pose's final slot.  EX: the
// K4 exchange epilogue is compiled in (only the lean kernel serves it; the
// throughput kernel stays free of its code and registers).
template <bool EX = false, int NW = kWarps>
__device__ __forceinline__ bool finish_unit(Acc& acc, const PoseIO& io, int pose, int seg,
                                            int segs, const ExArgs* xa = nullptr) {
  __shared__ double sm[NW * kAcc];
  __shared__ int s_last;
  block_reduce<NW>(acc, sm);
  if (threadIdx.x == 0) RMPB_TL_MAX(1);
  if (io.seg_out && threadIdx.x == 0) acc_to_arr(acc, io.seg_out + (size_t)(pose * segs + seg) * kAcc);
  if (segs == 1) {
    if (EX) {  // warp 0 runs the exchange (lane 0 holds the total)
      if (threadIdx.x < 32 && io.slot) {
        exchange_emit_warp(acc, io, *xa);
        return threadIdx.x == 0;
      }
      return false;
    }
    if (threadIdx.x == 0 && io.slot) {
      write_slot(acc, io.slot + (size_t)pose * 13, io.accel ? io.accel + (size_t)pose * 3 : nullptr);
      return true;
    }
    return false;
  }
  if (!io.slot) return false;
  if (threadIdx.x == 0) {
    RMPB_CHECK(seg >= 0 && seg < segs && pose >= 0);
    acc_to_arr(acc, io.partials + (size_t)(pose * segs + seg) * kAcc);
    const unsigned prev = ticket_add_release(io.tickets + pose);
    s_last = (prev == (unsigned)(segs - 1));
    if (s_last) fence_acquire_gpu();  // the other segments' partials are visible
    if (s_last) RMPB_TL_MAX(2);
  }
  __syncthreads();
  if (!s_last) return false;
  // Fixed-order fold of this pose's partials: thread j sums segments
  // j, j+kBlock, ... sequentially, then the fixed block tree.
  Acc f;
  f.zero();
  double cnt = 0.0;
  const double* base = io.partials + (size_t)pose * segs * kAcc;
  for (int j = threadIdx.x; j < segs; j += NW * 32) {
    const double* q = base + (size_t)j * kAcc;
    f.a00 += __ldcg(q + 0); f.a01 += __ldcg(q + 1); f.a02 += __ldcg(q + 2);
    f.a11 += __ldcg(q + 3); f.a12 += __ldcg(q + 4); f.a22 += __ldcg(q + 5);
    f.b0 += __ldcg(q + 6); f.b1 += __ldcg(q + 7); f.b2 += __ldcg(q + 8);
    cnt += __ldcg(q + 9);
  }
  f.cnt = (int)cnt;
  block_reduce<NW>(f, sm);
  if (EX) {
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) io.tickets[pose] = 0u;  // self-reset
      exchange_emit_warp(f, io, *xa);
      return threadIdx.x == 0;
    }
    return false;
  }
  if (threadIdx.x == 0) {
    RMPB_TL_MAX(3);
    io.tickets[pose] = 0u;  // self-reset: graph replays / next call start clean
    write_slot(f, io.slot + (size_t)pose * 13, io.accel ? io.accel + (size_t)pose * 3 : nullptr);
    RMPB_TL_MAX(4);
    return true;
  }
  return false;
}

// The K4 epilogue run by warp 0 of the pose's final CTA (lane 0 holds the
// slot): lane r posts to rank r and polls rank r's flag, lane j < 13 folds
// component j over the ranks (fixed pairwise order, _pool.py:61-72), lane 0
// writes the slot and runs the pinv.  The single-thread form serialised ~13
// us of dependent memory operations per call (scripts/profile_k4.py).
__device__ void exchange_emit_warp(const Acc& s, const PoseIO& io, const ExArgs& xa) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const PeerEx& ex = *xa.ex;
  const int W = ex.world, par = (int)(xa.epoch & 1ull);
  if (xa.mode & EX_POST) {
    const double r0[13] = {s.a00, s.a01, s.a02, s.a01, s.a11, s.a12, s.a02, s.a12, s.a22,
                           s.b0,  s.b1,  s.b2,  (double)s.cnt};
    double rec[13];
#pragma unroll
    for (int j = 0; j < 13; ++j) rec[j] = __shfl_sync(FULL, r0[j], 0);
    if (lane < W) {
      double* dst = ex.slots[lane] + ((size_t)par * W + ex.rank) * kMbox;
#pragma unroll
      for (int j = 0; j < 13; ++j) __stcg(dst + j, rec[j]);
      fence_acq_rel_sys();  // this slot before its flag
      st_relaxed_sys(ex.flags[lane] + (size_t)par * W + ex.rank, xa.epoch);
    }
  }
  if (!(xa.mode & EX_WAIT)) return;
  bool ok = true;
  if (lane < W) {
    const unsigned long long* fl = ex.flags[ex.rank] + (size_t)par * W + lane;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_relaxed_sys(fl) != xa.epoch) {
      if (globaltimer_ns() - t0 > 10000000000ull) { ok = false; break; }  // 10 s: a peer is gone
      __nanosleep(32);
    }
    fence_acq_rel_sys();  // rank `lane`'s slot is visible
  }
  ok = __all_sync(FULL, ok);
  __syncwarp();  // memory ordering: every lane's loads after every lane's acquire fence
  double outj = CUDART_NAN;
  if (ok && lane < 13) outj = fold8(ex.slots[ex.rank] + (size_t)par * W * kMbox + lane, W, kMbox);
  double out[13];
#pragma unroll
  for (int j = 0; j < 13; ++j) out[j] = __shfl_sync(FULL, outj, j);
  if (lane != 0) return;
  if (!ok) atomicExch(ex.err, 1u);
  for (int j = 0; j < 13; ++j) io.slot[j] = out[j];
  if (io.accel) {
    double m9[9] = {out[0], out[1], out[2], out[3], out[4], out[5], out[6], out[7], out[8]};
    double f[3] = {out[9], out[10], out[11]};
    if (ok) pinv_apply(m9, f, io.accel);
    else io.accel[0] = io.accel[1] = io.accel[2] = CUDART_NAN;
  }
}

// K1 latency kernel: one ray per thread per pass, no refill bookkeeping --
// used when every thread owns a single ray (small batches, e.g. one pose),
// where the longest ray's dependent chain is the whole story.
// grid: P * segs CTAs of kBlock threads; segment = seg_rays consecutive
// stored rays of the bundle.
template <class G, bool EX = false>
__device__ __forceinline__ bool lean_unit(const G& grid, const GridGeom& g, const Bundle& b,
                                          const PoseIO& io, const PolicyParams& p,
                                          double max_range, double eps, double step_scale,
                                          int segs, int seg_rays, const RayOut& ro, int unit,
                                          const ExArgs* xa = nullptr);

// EX: with the K4 peer-exchange epilogue (config C5 ray split).
template <class G, bool EX = false>
__global__ void __launch_bounds__(kBlock)
k_ray_policy(G grid, GridGeom g, Bundle b, PoseIO io, PolicyParams p, double max_range,
             double eps, double step_scale, int segs, int seg_rays, RayOut ro, ExArgs xa) {
  lean_unit<G, EX>(grid, g, b, io, p, max_range, eps, step_scale, segs, seg_rays, ro,
                   (int)blockIdx.x, &xa);
}

// One CTA's unit of the lean kernel; true in the thread that wrote the
// pose's final slot.
template <class G, bool EX>
__device__ __forceinline__ bool lean_unit(const G& grid, const GridGeom& g, const Bundle& b,
                                          const PoseIO& io, const PolicyParams& p,
                                          double max_range, double eps, double step_scale,
                                          int segs, int seg_rays, const RayOut& ro, int unit,
                                          const ExArgs* xa) {
  const int pose = unit / segs, seg = unit - pose * segs;
  if (threadIdx.x == 0) RMPB_TL_MIN(0);
  double sx, sy, sz, vx, vy, vz;
  io.pose(pose, sx, sy, sz);
  io.vel(pose, vx, vy, vz);
  Acc acc;
  acc.zero();
  const int begin = seg * seg_rays;
  const int end = min(begin + seg_rays, b.n);
  int my_steps = 0;
  if (io.active && !io.active[pose]) return false;
  // a pose inside the domain: its first step (t = 0) is shared by all rays
  // (k_ray_policy2's shared first step), one dependent step off every chain
  const bool inside =
      sx >= g.ox && sx <= g.hx && sy >= g.oy && sy <= g.hy && sz >= g.oz && sz <= g.hz;
  bool skip1 = false;
  double t1s = 0.0;
  if (inside) {
    int cx, cy, cz;
    const double d0 = interp_fast(grid, g, sx, sy, sz, cx, cy, cz);
    const bool negz = (sx == 0.0 && signbit(sx)) || (sy == 0.0 && signbit(sy)) ||
                      (sz == 0.0 && signbit(sz));
    skip1 = !(d0 < eps) && !negz;
    t1s = 0.0 + step_scale * d0;
  }
  for (int i = begin + threadIdx.x; i < end; i += kBlock) {
    const double dx = b.dx[i], dy = b.dy[i], dz = b.dz[i];
    TraceResult r = inside ? trace_ray_inside(grid, g, sx, sy, sz, dx, dy, dz, max_range, eps,
                                              step_scale, skip1, t1s)
                           : trace_ray_fast(grid, g, sx, sy, sz, dx, dy, dz, max_range, eps,
                                            step_scale);
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
  return finish_unit<EX>(acc, io, pose, seg, segs, xa);
}

// ---------------------------------------------------------------------------
// Latency server: ONE resident (cooperative) launch serving single-pose
// ray_policy requests posted through pinned, mapped host memory -- the
// control-loop use without a kernel launch + completion per
// call.  Per request: CTA 0 polls the host mailbox, copies the pose to
// device memory and publishes the epoch; every CTA runs its unit of the
// lean kernel (identical segmentation, hence bitwise the rmpb_ray_policy
// result); the CTA that folds the pose writes slot + accel to host memory,
// fences at system scope and publishes done = epoch.  The host posts the
// next request only after `done`, so the partial / ticket buffers are free.
// CTA 0 ends the loop on `stop` or after idle_ns without a request.
struct alignas(16) ServerMail {           // pinned host memory (mapped)
  unsigned long long req;                 // host: request epoch (after x, v)
  unsigned long long stop;                // host: 1 = exit (same 16 B: one PCIe read polls both)
  double x[3], v[3];                      // 16-B aligned: three 16-B reads
  double slot[13], accel[3];              // device: results
  unsigned long long done;                // device: epoch of the results
  unsigned long long exited;              // device: 1 once the loop ended
};
struct ServerDev {                        // device memory
  unsigned long long go;                  // epoch being served, ~0 = exit
  double xv[6];
};
constexpr unsigned long long kServerExit = ~0ull;

// 16-B reads of host-written mailbox words, re-fetched on every call (asm
// volatile: never hoisted out of a polling loop, unlike __ldcv)
__device__ __forceinline__ ulonglong2 ld_sys_u64x2(const void* p) {
  ulonglong2 r;
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ double2 ld_sys_f64x2(const void* p) {
  double2 r;
  asm volatile("ld.volatile.global.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p) : "memory");
  return r;
}

template <class G>
__global__ void __launch_bounds__(kBlock)
k_ray_server(G grid, GridGeom g, Bundle b, PolicyParams p, double max_range, double eps,
             double step_scale, int seg_rays, ServerMail* mail, ServerDev* dev,
             double* partials, unsigned* tickets, unsigned long long idle_ns,
             unsigned long long first_epoch) {
  __shared__ unsigned long long s_epoch;
  __shared__ double s_xv[6];
  unsigned long long last = first_epoch;  // requests already served before this launch
  PoseIO io{};
  io.x = nullptr; io.v = nullptr;  // the pose travels by value (x0 / v0) per request
  io.slot = mail->slot; io.accel = mail->accel;
  io.partials = partials; io.tickets = tickets;
  const RayOut ro{};
  while (true) {
    if (threadIdx.x == 0) {
      unsigned long long e;
      if (blockIdx.x == 0) {
        // each poll is one PCIe round trip: read (req, stop) as one 16-B word
        const unsigned long long t0 = globaltimer_ns();
        while (true) {
          const ulonglong2 rs = ld_sys_u64x2(&mail->req);
          e = rs.x;
          if (e != last) break;  // a posted request is served before any exit
          if (rs.y || globaltimer_ns() - t0 > idle_ns) { e = kServerExit; break; }
        }
        if (e != kServerExit) {
          // the pose: three independent 16-B reads (in flight together);
          // the host wrote it before `req`
          const char* xv = reinterpret_cast<const char*>(mail) + offsetof(ServerMail, x);
          const double2 a = ld_sys_f64x2(xv), b2 = ld_sys_f64x2(xv + 16), c = ld_sys_f64x2(xv + 32);
          dev->xv[0] = a.x; dev->xv[1] = a.y; dev->xv[2] = b2.x;
          dev->xv[3] = b2.y; dev->xv[4] = c.x; dev->xv[5] = c.y;
          __threadfence();
        }
        st_release_gpu(&dev->go, e);
      } else {
        const unsigned long long t0 = globaltimer_ns();
        while ((e = ld_acquire_gpu(&dev->go)) == last) {
          if (globaltimer_ns() - t0 > idle_ns + 1000000000ull) { e = kServerExit; break; }
          __nanosleep(64);
        }
      }
      s_epoch = e;
      if (e != kServerExit)
        for (int k = 0; k < 6; ++k) s_xv[k] = __ldcg(dev->xv + k);  // L2: never a stale L1 line
    }
    __syncthreads();
    const unsigned long long e = s_epoch;
    if (e == kServerExit) break;
    last = e;
    for (int k = 0; k < 3; ++k) { io.x0[k] = s_xv[k]; io.v0[k] = s_xv[3 + k]; }
    const bool wrote = lean_unit(grid, g, b, io, p, max_range, eps, step_scale, (int)gridDim.x,
                                 seg_rays, ro, (int)blockIdx.x);
    if (wrote) st_release_sys(&mail->done, e);  // orders this thread's slot / accel writes
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    *(volatile unsigned long long*)&mail->exited = 1ull;
  }
}

// K1/K3 v2: the production trace kernel.
//
// * exact arithmetic via interp_fast (no MUFU, no F2I/I2F on the step) and
//   the reference's IEEE slab divisions;
// * work split: a unit's rays are cut into 32-ray chunks (consecutive in the
//   Morton-ordered bundle) dealt round-robin to the CTA's warps, which keeps
//   the warps' total march lengths balanced;
// * ray preparation (direction, slab interval, start / end t) is done for a
//   whole chunk at once by all 32 lanes (converged) into a per-warp shared
//   buffer; rays that miss the map domain are retired right there;
// * lane refill: a lane whose ray finishes pops the next prepared ray
//   (ballot + prefix popc), so lanes never idle behind the warp's longest
//   ray.  The ray -> lane schedule depends only on the data: deterministic;
// * deferred policy: hits inside the activation radius are queued per warp
//   and evaluated 32 at a time by the whole warp (no divergent
//   transcendentals inside the march); each batch is reduced with a fixed
//   butterfly and added to the warp's accumulator in batch order, then the
//   CTA reduces warps in warp order: bitwise reproducible.
constexpr int kQueue = 64;
constexpr int kPrep = 32;

template <int NW>
struct K2Smem {
  double acc[NW][9];
  double qt[NW][kQueue];
  int qr[NW][kQueue];
  double pt[NW][kPrep], pe[NW][kPrep];
  double px[NW][kPrep], py[NW][kPrep], pz[NW][kPrep];
  int pr[NW][kPrep];
};

// Evaluates queue entry `lane` (when `valid`) and adds the warp's batch sum
// to the warp accumulator (lane 0).
template <class SM>
__device__ __forceinline__ void policy_flush(SM& sm, int warp, int lane, bool valid,
                                             const Bundle& b, int ray, double d, double vx,
                                             double vy, double vz, const PolicyParams& p) {
  Acc a;
  a.zero();
  if (valid) policy_accumulate(a, b.dx[ray], b.dy[ray], b.dz[ray], d, vx, vy, vz, p);
  const bool nz = a.a00 != 0.0 || a.a11 != 0.0 || a.a22 != 0.0 || a.b0 != 0.0 || a.b1 != 0.0 ||
                  a.b2 != 0.0 || a.a01 != 0.0 || a.a02 != 0.0 || a.a12 != 0.0;
  if (!__any_sync(0xffffffffu, nz)) return;
  double v[9] = {a.a00, a.a01, a.a02, a.a11, a.a12, a.a22, a.b0, a.b1, a.b2};
#pragma unroll
  for (int k = 0; k < 9; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 9; ++k) sm.acc[warp][k] += v[k];
  }
}

#ifndef RMPB_MINB
#define RMPB_MINB 4
#endif
#ifndef RMPB_UNROLL
#define RMPB_UNROLL 4  // steps per lane between bookkeeping rounds (r02: 3 -> 4 with the
#endif                 // shorter exdiv2 step, 12.64 -> 12.48 ms with REFILL 4)
#ifndef RMPB_REFILL
#define RMPB_REFILL 4  // refill when at least this many lanes are idle (or none alive)
#endif
#ifndef RMPB_TOWARD_FILTER
#define RMPB_TOWARD_FILTER 1  // queue only hits closing on the obstacle (toward > 0)
#endif
#ifndef RMPB_LANE_COUNT
#define RMPB_LANE_COUNT 1  // lane-private hit count (no per-round ballot)
#endif

// Prepare the warp's next 32-ray chunk into its shared buffer: direction,
// slab interval [t0, t1] (max_range applied), shared-first-step start, ray
// id with the closing / first-step flags; rays that miss the map retire here.
template <class G, bool RAYOUT, bool INSIDE, int NW>
__device__ __forceinline__ void prep_chunk(K2Smem<NW>& sm, const GridGeom& g, const Bundle& b,
                                           const PoseIO& io, const RayOut& ro, int pose, int begin,
                                           int end, int lane, int warp, unsigned lt, double sx,
                                           double sy, double sz, double max_range, bool skip1,
                                           double t1s, int& chunk, int& pcount, int& phead) {
  const unsigned FULL = 0xffffffffu;
  const int r = begin + (chunk << 5) + lane;
  chunk += NW;
  bool ok = r < end, first = false;
  double ex = 0, ey = 0, ez = 0, t0 = 0, t1 = 0;
  if (ok) {
    ex = b.dx[r]; ey = b.dy[r]; ez = b.dz[r];
    if (INSIDE) {
      double thi = CUDART_INF;
      if (ex != 0.0) {
        const double tb = slab_div((ex > 0.0 ? g.hx : g.ox) - sx, ex);
        thi = tb < thi ? tb : thi;
      }
      if (ey != 0.0) {
        const double tb = slab_div((ey > 0.0 ? g.hy : g.oy) - sy, ey);
        thi = tb < thi ? tb : thi;
      }
      if (ez != 0.0) {
        const double tb = slab_div((ez > 0.0 ? g.hz : g.oz) - sz, ez);
        thi = tb < thi ? tb : thi;
      }
      t0 = 0.0;
      t1 = thi < max_range ? thi : max_range;
      ok = !(t0 > t1);
      // shared first step: rays with a finite direction start at t1s
      // (1 step done); those with t1s > t_end end there (a miss)
      if (skip1 && ok && isfinite(ex) && isfinite(ey) && isfinite(ez)) {
        t0 = t1s;
        first = true;
        ok = t1s <= t1;  // !(t > t_end): NaN ends the ray
      }
    } else {
      ok = box_span(g, sx, sy, sz, ex, ey, ez, t0, t1);
      if (ok) {
        t0 = t0 > 0.0 ? t0 : 0.0;
        t1 = t1 < max_range ? t1 : max_range;
        ok = !(t0 > t1);
      }
    }
    if (RAYOUT && !ok && ro.t) {
      const int o = b.perm ? b.perm[r] : r;
      ro.t[o] = CUDART_INF;
      if (ro.cell) { ro.cell[3 * o] = -1; ro.cell[3 * o + 1] = -1; ro.cell[3 * o + 2] = -1; }
      if (ro.steps) ro.steps[o] = first ? 1 : 0;
    }
  }
  const unsigned m = __ballot_sync(FULL, ok);
  if (ok) {
    const int pos = __popc(m & lt);
    RMPB_CHECK(pos < kPrep && r >= begin && r < end && r < b.n);
    sm.pt[warp][pos] = t0; sm.pe[warp][pos] = t1;
    sm.px[warp][pos] = ex; sm.py[warp][pos] = ey; sm.pz[warp][pos] = ez;
#if RMPB_TOWARD_FILTER
    // policy_accumulate adds nothing for toward <= 0 (_ckern.pyx:295-299):
    // flag the ray (sign bit) so only closing hits are queued.  Same
    // expression and rounding as policy_accumulate's test.
    double vx, vy, vz;
    io.vel(pose, vx, vy, vz);
    const double toward = ex * vx + ey * vy + ez * vz;
    sm.pr[warp][pos] = (int)((unsigned)r | (toward > 0.0 ? 0x80000000u : 0u) |
                             (first ? 0x40000000u : 0u));
#else
    sm.pr[warp][pos] = (int)((unsigned)r | (first ? 0x40000000u : 0u));
#endif
  }
  pcount = __popc(m);
  phead = 0;
  __syncwarp();
}

// RAYOUT: per-ray parity outputs (t, cell, steps) and the step counter.
// FAST: fp32 march (opt-in, not reference-exact; see interp_f).
// INSIDE: the pose lies inside the map domain (CTA-uniform: one pose per
// CTA), so the body is compiled without the per-refill domain test
// (13.78 -> 13.55 ms per 4096-pose C1 step).
template <class G, bool RAYOUT, bool FAST, bool INSIDE, int NW, bool EX = false>
__device__ __forceinline__ void ray_policy2_body(K2Smem<NW>& sm, const G& grid, const GridGeom& g,
                                                 const Bundle& b, const PoseIO& io,
                                                 const PolicyParams& p, double max_range,
                                                 double eps, double step_scale, int segs,
                                                 int seg_rays, const RayOut& ro, int pose, int seg,
                                                 double sx, double sy, double sz,
                                                 const ExArgs* xa = nullptr) {
  using real = typename std::conditional<FAST, float, double>::type;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  const int begin = seg * seg_rays;
  const int end = min(begin + seg_rays, b.n);
  const int nchunks = (end - begin + 31) >> 5;
  double* qt = sm.qt[warp];
  int* qr = sm.qr[warp];

  int chunk = warp, pcount = 0, phead = 0, qn = 0, cnt = 0, my_steps = 0;
  int ray = 0, steps = 0;
  bool alive = false;
  real dx = 0, dy = 0, dz = 0, t = 0, tend = 0;
  const GeomF gf{(float)g.ox, (float)g.oy, (float)g.oz, (float)(1.0 / g.res), g.nx - 2, g.ny - 2,
                 g.nz - 2};
  (void)gf;
  // Shared first step (exact): a pose inside the domain starts every ray at
  // t = 0, where p = s + 0 * d = s for any finite direction, so step 1 is the
  // same interpolation for all rays of the pose (_ckern.pyx:236-246).  It is
  // evaluated once here; each ray then starts at t1 = 0 + step * d0 with one
  // step counted.  Not taken when the pose is in an obstacle (d0 < eps: every
  // ray hits at t = 0) or a coordinate is -0.0 (s + (+/-0) could flip the
  // sign of that zero per ray).  ~1 of the ~7 steps per ray on C1.
  bool skip1 = false;
  double t1s = 0.0;
  if constexpr (INSIDE && !FAST) {
    int cx, cy, cz;
    const double d0 = interp_fast(grid, g, sx, sy, sz, cx, cy, cz);
    const bool negz = (sx == 0.0 && signbit(sx)) || (sy == 0.0 && signbit(sy)) ||
                      (sz == 0.0 && signbit(sz));
    skip1 = !(d0 < eps) && !negz;
    t1s = 0.0 + step_scale * d0;
  }
  __syncwarp();
  while (true) {
    // ---- refill from the prepared-ray buffer (prepare a chunk when empty);
    // only once enough lanes idle, so the refill cost is amortised
    unsigned need = __ballot_sync(FULL, !alive);
    const bool drained = pcount == 0 && chunk >= nchunks;
    if (need == FULL && drained) break;
    if ((__popc(need) < RMPB_REFILL && need != FULL) || drained) need = 0u;
    while (need != 0u && (pcount > 0 || chunk < nchunks)) {
      if (pcount == 0) {
        prep_chunk<G, RAYOUT, INSIDE, NW>(sm, g, b, io, ro, pose, begin, end, lane, warp, lt, sx,
                                          sy, sz, max_range, skip1, t1s, chunk, pcount, phead);
        continue;
      }
      const int rank = __popc(need & lt);
      if (!alive && rank < pcount) {
        const int e = phead + rank;
        t = (real)sm.pt[warp][e]; tend = (real)sm.pe[warp][e];
        dx = (real)sm.px[warp][e]; dy = (real)sm.py[warp][e]; dz = (real)sm.pz[warp][e];
        ray = sm.pr[warp][e];
        alive = true;
        if (RAYOUT) steps = (ray >> 30) & 1;  // 1 when the shared first step was taken
      }
      const int take = min(pcount, __popc(need));
      phead += take;
      pcount -= take;
      need = __ballot_sync(FULL, !alive);
      if (need == FULL && pcount == 0 && chunk >= nchunks) break;
    }
    if (need == FULL) break;  // (only reachable once every ray is done)
    // ---- RMPB_UNROLL sphere-trace steps per live lane between bookkeeping
    // rounds (a lane that finishes idles for the rest of the round).  Steps
    // carry only (t, alive, hit); the end-of-ray bookkeeping runs once per
    // round for the lanes whose ray ended in it.
    const bool was_alive = alive;
    bool hit_now = false;
    int hx = -1, hy = -1, hz = -1;
#pragma unroll
    for (int u = 0; u < RMPB_UNROLL; ++u) {
      if (alive) {
        int ix = -1, iy = -1, iz = -1;
        real d;
        if constexpr (FAST) {
          const float px = (float)sx, py = (float)sy, pz = (float)sz;
          d = interp_f(grid, gf, __fmaf_rn(t, dx, px), __fmaf_rn(t, dy, py), __fmaf_rn(t, dz, pz));
        } else {
          // pose in (uniform) registers: no shared-memory reload per step
          d = interp_fast(grid, g, sx + t * dx, sy + t * dy, sz + t * dz, ix, iy, iz);
        }
        if (RAYOUT) { ++steps; hx = ix; hy = iy; hz = iz; }
        hit_now = d < (real)eps;
        real tn;
        if constexpr (FAST) tn = __fmaf_rn((float)step_scale, d, t);
        else tn = t + step_scale * d;
        if (!hit_now) t = tn;
        alive = !hit_now && t <= tend;  // !(t > tend); a NaN t ends the ray
      }
    }
#if RMPB_TOWARD_FILTER
    const bool enq = hit_now && (double)t < p.radius && ray < 0;
#else
    const bool enq = hit_now && (double)t < p.radius;
#endif
    const int rid = ray & 0x3fffffff;  // bit 31: closing, bit 30: first step shared
    if (RAYOUT && was_alive && !alive) {
      my_steps += steps;
      if (ro.t) {
        const int o = b.perm ? b.perm[rid] : rid;
        ro.t[o] = hit_now ? (double)t : CUDART_INF;
        if (ro.cell) {
          ro.cell[3 * o] = hit_now ? hx : -1; ro.cell[3 * o + 1] = hit_now ? hy : -1;
          ro.cell[3 * o + 2] = hit_now ? hz : -1;
        }
        if (ro.steps) ro.steps[o] = steps;
      }
    }
    // ---- queue policy work; evaluate in full-warp batches of 32
#if RMPB_LANE_COUNT
    cnt += hit_now;  // lane-private; min_range = 0: every hit counts
#else
    cnt += __popc(__ballot_sync(FULL, hit_now));  // warp-uniform; min_range = 0: every hit counts
#endif
    const unsigned em = __ballot_sync(FULL, enq);
    if (em) {
      if (enq) {
        const int pos = qn + __popc(em & lt);
        RMPB_CHECK(pos < kQueue && rid < b.n);
        qt[pos] = (double)t;
        qr[pos] = rid;
      }
      qn += __popc(em);
      if (qn >= 32) {
        __syncwarp();
        double vx, vy, vz;
        io.vel(pose, vx, vy, vz);
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
    double vx, vy, vz;
    io.vel(pose, vx, vy, vz);
    const bool valid = lane < qn;
    policy_flush(sm, warp, lane, valid, b, valid ? qr[lane] : 0, valid ? qt[lane] : 0.0, vx, vy,
                 vz, p);
  }
  if (RAYOUT && ro.step_total) {
    int s = warp_sum_i(my_steps);
    if (lane == 0) atomicAdd(ro.step_total, (unsigned long long)s);
  }
#if RMPB_LANE_COUNT
  cnt = warp_sum_i(cnt);
#endif
  __syncwarp();
  Acc acc;
  acc.zero();
  if (lane == 0) {
    acc.a00 = sm.acc[warp][0]; acc.a01 = sm.acc[warp][1]; acc.a02 = sm.acc[warp][2];
    acc.a11 = sm.acc[warp][3]; acc.a12 = sm.acc[warp][4]; acc.a22 = sm.acc[warp][5];
    acc.b0 = sm.acc[warp][6]; acc.b1 = sm.acc[warp][7]; acc.b2 = sm.acc[warp][8];
    acc.cnt = cnt;  // warp-uniform count: contributed once per warp
  }
  finish_unit<EX, NW>(acc, io, pose, seg, segs, xa);
}

// NW warps per CTA (kTraceWarps): one (pose, ray segment) unit per CTA.
// (Measured, round 2: a whole pose per 16- / 32-warp CTA raises the L1 hit
// rate 26.7 -> 32 % but the wider CTAs' tails cost more: 13.72 / 14.07 ms
// vs 13.39 ms per 4096-pose C1 step.)
#ifndef RMPB_NW
#define RMPB_NW 8
#endif
#ifndef RMPB_TRACE_MINB
#define RMPB_TRACE_MINB (RMPB_MINB * kWarps / RMPB_NW)
#endif
constexpr int kTraceWarps = RMPB_NW;
// EX: with the K4 peer-exchange epilogue (config C5 ray split; exact only).
template <class G, bool RAYOUT, bool FAST = false, int NW = kTraceWarps, bool EX = false>
__global__ void __launch_bounds__(NW * 32, RMPB_TRACE_MINB)
k_ray_policy2(G grid, GridGeom g, Bundle b, PoseIO io, PolicyParams p, double max_range,
              double eps, double step_scale, int segs, int seg_rays, RayOut ro, ExArgs xa) {
  // dynamic: sizeof(K2Smem<32>) = 72 KB exceeds the 48 KB static limit
  extern __shared__ __align__(16) unsigned char k2_dsm[];
  K2Smem<NW>& sm = *reinterpret_cast<K2Smem<NW>*>(k2_dsm);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int unit = blockIdx.x;
  const int pose = unit / segs, seg = unit - pose * segs;
  if (io.active && !io.active[pose]) return;  // whole CTA: finished rollout
  double sx, sy, sz;
  io.pose(pose, sx, sy, sz);
  // Inside the domain every axis' entry quotient is <= 0, so the reference's
  // t = max(t0, 0) is exactly 0 and only the exit side is needed:
  // (hi - s)/d for d > 0, (lo - s)/d for d < 0 (_ckern.pyx:171-212).
  const bool inside =
      sx >= g.ox && sx <= g.hx && sy >= g.oy && sy <= g.hy && sz >= g.oz && sz <= g.hz;
  if (lane < 9) sm.acc[warp][lane] = 0.0;
  __syncthreads();
  if (inside)
    ray_policy2_body<G, RAYOUT, FAST, true, NW, EX>(sm, grid, g, b, io, p, max_range, eps,
                                                step_scale, segs, seg_rays, ro, pose, seg, sx, sy,
                                                sz, &xa);
  else
    ray_policy2_body<G, RAYOUT, FAST, false, NW, EX>(sm, grid, g, b, io, p, max_range, eps,
                                                 step_scale, segs, seg_rays, ro, pose, seg, sx,
                                                 sy, sz, &xa);
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

// K2 v3 (and K2b): warp units.  A warp owns `seg` consecutive beams of one scan (no
// CTA-wide barrier anywhere: warps never wait for each other).  Streaming:
// each lane loads 4 consecutive beams per group (2 x 16-B range loads + one
// 4-B validity word).  Beams inside the activation
// radius go to a stage-1 ring; a stage-1 batch of 32 gathers the lattice
// directions, rotates them and keeps the beams closing on the obstacle
// (toward > 0) in a stage-2 ring; only stage-2 batches of 32 run the
// transcendental policy.  Each stage has ONE call site (the kernel's code
// stays small: warps at different points of the loop share the I-cache).
// Per-warp partials (10 doubles) are folded in warp order by the last warp of
// the scan (atomic ticket), which also resolves.  Every order is
// data-determined: bitwise reproducible.
constexpr int kRing1 = 32 + 4 * 32;  // < 32 left + one group's pushes (4 beams x 32 lanes)
constexpr int kRing2 = 64;
template <bool F32>
struct LidarQ2 {  // stage-2 ring: range + world direction of the closing beams
  double d[kRing2], x[kRing2], y[kRing2], z[kRing2];
};
template <>
struct LidarQ2<true> {  // fast mode: the policy math is fp32 anyway (1 KB less per warp)
  float4 e[kRing2];     // (d, x, y, z)
};
template <bool F32 = false>
struct LidarWarpSmemT {
  double acc[9][32];  // per-lane running sums (lane l owns column l)
  double R[9], v[3];  // this warp's scan orientation (row-major) and velocity
  double q1d[kRing1];
  int q1i[kRing1];
  LidarQ2<F32> q2;
};
using LidarWarpSmem = LidarWarpSmemT<false>;

// K2b: raw sensor-frame points (no map, no lattice): the
// beam direction is p * (1/|p|) and its range |p|; zero / non-finite points are
// invalid.  Float32 xyz as delivered by the sensor driver.
struct PointsIO {
  const float* __restrict__ xyz;  // [S][N][3]
  const double* __restrict__ R;   // [S][9] or null
  int n;
};


// Bulk L2 prefetch (cp.async.bulk.prefetch.L2): 16-B aligned address, size a
// multiple of 16.  Non-binding; the data are read later by ordinary loads.
__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

#ifndef RMPB_LIDAR_PF
#define RMPB_LIDAR_PF 0  // groups of 128 beams prefetched ahead into L2 (0 = off)
#endif

// Beam sources of the warp-unit kernel: a lattice scan (sensor directions +
// ranges + validity, policies.py:195-205) or raw sensor-frame points (K2b).
struct LatticeSrc {
  ScanIO sc;
  const double* rg;
  const unsigned char* vl;
  bool vec;
  __device__ __forceinline__ const double* rot() const { return sc.R; }
  __device__ __forceinline__ int count() const { return sc.n; }
  __device__ __forceinline__ void bind(int scan) {
    rg = sc.ranges + (size_t)scan * sc.n;
    vl = sc.valid ? sc.valid + (size_t)scan * sc.n : nullptr;
    vec = ((reinterpret_cast<uintptr_t>(rg) & 15) == 0) &&
          (!vl || (reinterpret_cast<uintptr_t>(vl) & 3) == 0);
  }
  // beams i0..i0+3: 2 x 16-B range loads + one 4-B validity word (scalar
  // fallback for misaligned rows and the ragged tail); invalid -> +inf
  __device__ __forceinline__ void load4(int i0, int end, double (&o)[4]) const {
    if (vec && i0 + 3 < end) {
      const double2 x0 = __ldcs(reinterpret_cast<const double2*>(rg + i0));
      const double2 x1 = __ldcs(reinterpret_cast<const double2*>(rg + i0 + 2));
      o[0] = x0.x; o[1] = x0.y; o[2] = x1.x; o[3] = x1.y;
      if (vl) {
        const unsigned m = __ldcs(reinterpret_cast<const unsigned*>(vl + i0));
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (!((m >> (8 * j)) & 0xffu)) o[j] = CUDART_INF;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = i0 + j;
        o[j] = (i < end && (!vl || vl[i])) ? rg[i] : CUDART_INF;
      }
    }
  }
  __device__ __forceinline__ void dir(int i, double, double& ex, double& ey, double& ez) const {
    ex = sc.dirs[3 * i]; ey = sc.dirs[3 * i + 1]; ez = sc.dirs[3 * i + 2];
  }
  // L2 prefetch of the 128-beam group at i0 (one bulk prefetch per array;
  // issued by one lane, no registers held): aligned full groups only
  __device__ __forceinline__ void prefetch(int i0, int end) const {
    if (!vec || i0 + 128 > end) return;
    l2_prefetch(rg + i0, 128 * sizeof(double));
    if (vl && ((reinterpret_cast<uintptr_t>(vl + i0) & 15) == 0)) l2_prefetch(vl + i0, 128);
  }
};

struct PointSrc {
  PointsIO pt;
  const float* P;
  bool vec;
  __device__ __forceinline__ const double* rot() const { return pt.R; }
  __device__ __forceinline__ int count() const { return pt.n; }
  __device__ __forceinline__ void bind(int scan) {
    P = pt.xyz + (size_t)scan * pt.n * 3;
    vec = (reinterpret_cast<uintptr_t>(P) & 15) == 0;
  }
  static __device__ __forceinline__ double range(float x, float y, float z) {
    const double px = x, py = y, pz = z;
    const double d = sqrt(px * px + py * py + pz * pz);
    return d > 0.0 ? d : CUDART_INF;  // zero ("no return") or NaN point: invalid beam
  }
  // points i0..i0+3 (48 B = 3 x 16-B loads when aligned); range = |p|
  __device__ __forceinline__ void load4(int i0, int end, double (&o)[4]) const {
    if (vec && i0 + 3 < end) {
      const float4* q = reinterpret_cast<const float4*>(P + 3 * (size_t)i0);
      const float4 a = __ldcs(q), b = __ldcs(q + 1), c = __ldcs(q + 2);
      o[0] = range(a.x, a.y, a.z); o[1] = range(a.w, b.x, b.y);
      o[2] = range(b.z, b.w, c.x); o[3] = range(c.y, c.z, c.w);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = i0 + j;
        o[j] = i < end ? range(P[3 * i], P[3 * i + 1], P[3 * i + 2]) : CUDART_INF;
      }
    }
  }
  // direction p * (1/|p|): one fp64 division per point instead of three
  // (within 1 ulp of p / |p|; C3 points 0.74 -> 0.69 ms)
  __device__ __forceinline__ void dir(int i, double d, double& ex, double& ey, double& ez) const {
    const double r = 1.0 / d;
    ex = (double)P[3 * i] * r; ey = (double)P[3 * i + 1] * r; ez = (double)P[3 * i + 2] * r;
  }
  __device__ __forceinline__ void prefetch(int i0, int end) const {
    if (!vec || i0 + 128 > end) return;
    l2_prefetch(P + 3 * (size_t)i0, 128 * 12);
  }
};

// End of a LiDAR warp unit (lane 0 holds the unit's sums): resolve directly
// when the scan is one unit; else publish the partial, and the last unit of
// the scan (atomic ticket) folds the partials in unit order and resolves.
__device__ __forceinline__ void lidar_unit_finish(const Acc& a, const PoseIO& io, int scan,
                                                  int wu, int wps, int lane) {
  const unsigned FULL = 0xffffffffu;
  if (wps == 1) {
    if (lane == 0 && io.slot)
      write_slot(a, io.slot + (size_t)scan * 13, io.accel ? io.accel + (size_t)scan * 3 : nullptr);
    return;
  }
  unsigned prev = 0;
  if (lane == 0) {
    RMPB_CHECK(wu >= 0 && wu < wps && scan >= 0);
    acc_to_arr(a, io.partials + ((size_t)scan * wps + wu) * kAcc);
    prev = ticket_add_release(io.tickets + scan);
    if (prev == (unsigned)(wps - 1)) fence_acquire_gpu();  // the other units' partials
  }
  prev = __shfl_sync(FULL, prev, 0);
  if (prev != (unsigned)(wps - 1)) return;
  __syncwarp();
  double f[kAcc];
#pragma unroll
  for (int k = 0; k < kAcc; ++k) f[k] = 0.0;
  const double* pb = io.partials + (size_t)scan * wps * kAcc;
  for (int j = lane; j < wps; j += 32) {
#pragma unroll
    for (int k = 0; k < kAcc; ++k) f[k] += __ldcg(pb + (size_t)j * kAcc + k);
  }
#pragma unroll
  for (int k = 0; k < kAcc; ++k) f[k] = warp_sum(f[k]);
  if (lane == 0) {
    Acc t;
    t.a00 = f[0]; t.a01 = f[1]; t.a02 = f[2]; t.a11 = f[3]; t.a12 = f[4]; t.a22 = f[5];
    t.b0 = f[6]; t.b1 = f[7]; t.b2 = f[8]; t.cnt = (int)f[9];
    if (io.slot)
      write_slot(t, io.slot + (size_t)scan * 13, io.accel ? io.accel + (size_t)scan * 3 : nullptr);
    io.tickets[scan] = 0u;  // self-reset
  }
}


#ifndef RMPB_LIDAR_MINB
#define RMPB_LIDAR_MINB 4
#endif
template <class Src, bool F32 = false>
__device__ __forceinline__ void lidar_warp_unit(Src src, const PoseIO& io, const PolicyParams& p,
                                                int wps, int seg, long long unit,
                                                LidarWarpSmemT<F32>& w) {
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
  const int scan = (int)(unit / wps), wu = (int)(unit - (long long)scan * wps);
  __syncwarp();  // the previous unit's reads of w are done
  const double* Rall = src.rot();
  const bool rot = Rall != nullptr;
  if (rot && lane < 9) w.R[lane] = Rall[9 * scan + lane];
  if (lane == 0) io.vel(scan, w.v[0], w.v[1], w.v[2]);
#pragma unroll
  for (int k = 0; k < 9; ++k) w.acc[k][lane] = 0.0;
  src.bind(scan);
  const int begin = wu * seg;
  const int end = min(begin + seg, src.count());
  int h1 = 0, q1n = 0, h2 = 0, q2n = 0, cnt = 0;
  int base = begin;
  if (RMPB_LIDAR_PF > 1 && lane > 0 && lane < RMPB_LIDAR_PF)  // the first groups
    src.prefetch(base + lane * 128, end);
  __syncwarp();
  while (true) {
    const bool draining = base >= end;
    if (!draining) {
      // ---- stream one group, then count + push the in-radius beams to
      // ring 1 (no flush here).  (Prefetching the next group into registers
      // measured slower: 0.58 vs 0.50 ms on C3 -- more spills.)
      if (RMPB_LIDAR_PF > 0 && lane == 0) src.prefetch(base + RMPB_LIDAR_PF * 128, end);
      double cur[4];
      src.load4(base + 4 * lane, end, cur);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double d = cur[j];
        const bool counted = !(d != d || d == CUDART_INF || d < p.min_range);
        cnt += counted;
        const bool enq = counted && d < p.radius;
        const unsigned em = __ballot_sync(FULL, enq);
        if (enq) {
          int pos = h1 + q1n + __popc(em & lt);
          if (pos >= kRing1) pos -= kRing1;
          RMPB_CHECK(pos >= 0 && pos < kRing1 && q1n + __popc(em) <= kRing1);
          w.q1d[pos] = d;
          w.q1i[pos] = base + 4 * lane + j;
        }
        q1n += __popc(em);
      }
      base += 128;
    }
    __syncwarp();
    // ---- stage 1 (one call site): direction gather, rotation, closing test
    while (q1n >= 32 || (draining && (q1n > 0 || q2n > 0))) {
      const int take = min(q1n, 32);
      bool keep = false;
      double d = 0, wx = 0, wy = 0, wz = 0;
      if (lane < take) {
        int e = h1 + lane;
        if (e >= kRing1) e -= kRing1;
        const int i = w.q1i[e];
        d = w.q1d[e];
        RMPB_CHECK(i >= begin && i < end);
        double ex, ey, ez;
        src.dir(i, d, ex, ey, ez);
        wx = ex; wy = ey; wz = ez;
        if (rot) {  // directions @ orientation.T  (rays.py:172-173)
          wx = ex * w.R[0] + ey * w.R[1] + ez * w.R[2];
          wy = ex * w.R[3] + ey * w.R[4] + ez * w.R[5];
          wz = ex * w.R[6] + ey * w.R[7] + ez * w.R[8];
        }
        keep = wx * w.v[0] + wy * w.v[1] + wz * w.v[2] > 0.0;  // policy_accumulate's test
      }
      h1 += take;
      if (h1 >= kRing1) h1 -= kRing1;
      q1n -= take;
      const unsigned km = __ballot_sync(FULL, keep);
      if (keep) {
        const int pos = (h2 + q2n + __popc(km & lt)) & (kRing2 - 1);
        RMPB_CHECK(q2n + __popc(km) <= kRing2);
        if constexpr (F32)
          w.q2.e[pos] = make_float4((float)d, (float)wx, (float)wy, (float)wz);
        else {
          w.q2.d[pos] = d; w.q2.x[pos] = wx; w.q2.y[pos] = wy; w.q2.z[pos] = wz;
        }
      }
      q2n += __popc(km);
      __syncwarp();
      // ---- stage 2 (one call site): transcendental policy, 32 at a time
      const bool last = draining && q1n == 0;
      if (q2n >= 32 || (last && q2n > 0)) {
        const int t2 = min(q2n, 32);
        Acc a;
        a.zero();
        if (lane < t2) {
          const int e = (h2 + lane) & (kRing2 - 1);
          if constexpr (F32) {
            const float4 q = w.q2.e[e];
            policy_accumulate_f32(a, q.y, q.z, q.w, q.x, w.v[0], w.v[1], w.v[2], p);
          } else {
            policy_accumulate(a, w.q2.x[e], w.q2.y[e], w.q2.z[e], w.q2.d[e], w.v[0], w.v[1],
                              w.v[2], p);
          }
        }
        h2 = (h2 + t2) & (kRing2 - 1);
        q2n -= t2;
        if (lane < t2) {  // lane-private running sums: no shuffles per batch
          w.acc[0][lane] += a.a00; w.acc[1][lane] += a.a01; w.acc[2][lane] += a.a02;
          w.acc[3][lane] += a.a11; w.acc[4][lane] += a.a12; w.acc[5][lane] += a.a22;
          w.acc[6][lane] += a.b0; w.acc[7][lane] += a.b1; w.acc[8][lane] += a.b2;
        }
        __syncwarp();
      }
    }
    if (draining) break;
  }
  __syncwarp();
  cnt = warp_sum_i(cnt);
  // ---- warp partial (fixed butterfly over the lane sums); the last warp of
  // the scan folds the partials in warp order and resolves
  double ws[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) ws[k] = warp_sum(w.acc[k][lane]);
  Acc a;
  a.a00 = ws[0]; a.a01 = ws[1]; a.a02 = ws[2]; a.a11 = ws[3]; a.a12 = ws[4];
  a.a22 = ws[5]; a.b0 = ws[6]; a.b1 = ws[7]; a.b2 = ws[8]; a.cnt = cnt;
  lidar_unit_finish(a, io, scan, wu, wps, lane);
}

// F32: the opt-in fp32 policy math (policy_accumulate_f32).
#ifndef RMPB_LIDAR_MINB_FAST
#define RMPB_LIDAR_MINB_FAST 5  // fast mode: smaller rings -> 5 CTAs of 8 warps per SM
#endif
template <class Src, bool F32 = false>
__global__ void __launch_bounds__(kBlock, F32 ? RMPB_LIDAR_MINB_FAST : RMPB_LIDAR_MINB)
k_lidar_warp(Src src, PoseIO io, PolicyParams p, int wps, int seg, long long nunits,
             unsigned long long* __restrict__ sched) {
  extern __shared__ __align__(16) unsigned char lidar_dsm[];  // kWarps x LidarWarpSmemT<F32>
  LidarWarpSmemT<F32>* smw = reinterpret_cast<LidarWarpSmemT<F32>*>(lidar_dsm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (sched == nullptr) {  // one unit per warp (the hardware block scheduler balances)
    const long long unit = (long long)blockIdx.x * kWarps + warp;
    if (unit < nunits) lidar_warp_unit<Src, F32>(src, io, p, wps, seg, unit, smw[warp]);
    return;
  }
  // Persistent warps claiming units from a counter (sched[0]); a unit's
  // result does not depend on which warp runs it, so this is bitwise the
  // one-unit-per-warp schedule.  sched[1] counts finished warps; the last
  // one resets both (graph replays / the next call start at zero).
  while (true) {
    unsigned long long u = 0;
    if (lane == 0) u = atomicAdd(sched, 1ull);
    u = __shfl_sync(0xffffffffu, u, 0);
    if ((long long)u >= nunits) break;
    lidar_warp_unit<Src, F32>(src, io, p, wps, seg, (long long)u, smw[warp]);
  }
  if (lane == 0) {
    const unsigned long long W = (unsigned long long)gridDim.x * kWarps;
    if (atomicAdd(sched + 1, 1ull) == W - 1) { sched[0] = 0ull; sched[1] = 0ull; }
  }
}


// (Measured, round 2: a warp-specialised variant -- per CTA, filter warps
// streaming through a TMA stage ring into shared-memory queues and paired
// policy warps running stages 1 and 2 -- is bitwise equal to this kernel
// but slower on C3: 0.62-0.70 ms vs 0.51 ms per 1024 scans (commit ae35050,
// profiles/README.md).  Half the warps stream, and the pairs' per-unit
// latency, not the byte stream, bounds it.)

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
  // n is small (number of GPUs): fold in a local buffer.
  double buf[13];
  fold_slots<64>(slots, n, 13, false, buf);
  for (int j = 0; j < 13; ++j) out_slot[j] = buf[j];
  if (out_accel) {
    double m9[9], f[3];
    for (int k = 0; k < 9; ++k) m9[k] = buf[k];
    f[0] = buf[9]; f[1] = buf[10]; f[2] = buf[11];
    pinv_apply(m9, f, out_accel);
  }
}

// pinv_psd of a batch of 3x3 metrics (core.py:103-115), returns the matrix.
__global__ void k_pinv_psd(const double* __restrict__ a, int n, double rcond,
                           double* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double m[3][3], V[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) m[r][c] = 0.5 * (a[9 * i + 3 * r + c] + a[9 * i + 3 * c + r]);
  jacobi3(m, V);
  double lam[3] = {m[0][0], m[1][1], m[2][2]};
  double lmax = fmax(fmax(lam[0], lam[1]), lam[2]);
  double cut = rcond * (lmax > 0.0 ? lmax : 0.0);  // core.py:111: rcond * max(w.max(), 0)
  double inv[3];
  for (int k = 0; k < 3; ++k) inv[k] = lam[k] > cut ? 1.0 / lam[k] : 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      out[9 * i + 3 * r + c] = V[r][0] * inv[0] * V[c][0] + V[r][1] * inv[1] * V[c][1] +
                               V[r][2] * inv[2] * V[c][2];
}

}  // namespace rmpb
