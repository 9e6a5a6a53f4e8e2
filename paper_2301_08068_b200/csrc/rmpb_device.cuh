// rmpb_device.cuh -- device-side building blocks of the raycasting-RMP path.
//
// Everything in the EXACT path is IEEE fp64 in the reference's operation
// order and this translation unit family is compiled
// with `-fmad=false`, so every a*b+c stays a separate DMUL/DADD exactly as
// the reference's scalar SSE2 build (no FMA) computes it.  Division is the
// IEEE correctly-rounded `/`.  Reference anchors (relative to
// /root/reference/pkg/src/rmpnav/):
//   interp ........ _kernels/_ckern.pyx:92-135
//   box_span ...... _kernels/_ckern.pyx:171-212
//   sphere trace .. _kernels/_ckern.pyx:217-248, rays.py:99-124
//   ray policy .... _kernels/_ckern.pyx:278-321, policies.py:175-205
//   pinv_psd ...... core.py:103-115
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>
#include <math_constants.h>

// Debug build (make checked -> librmpb_checked.so): device-side bounds
// checks on every map / ring / partial index (a failed check prints its
// location and traps).  compute-sanitizer is not available on the GPU pool
// this was built on; this build plus the GPU test-suite stands in for it.
#ifdef RMPB_CHECKED
#include <cstdio>
#define RMPB_CHECK(c)                                                               \
  do {                                                                             \
    if (!(c)) {                                                                    \
      printf("RMPB_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
             #c, (int)blockIdx.x, (int)threadIdx.x);                               \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define RMPB_CHECK(c) \
  do {                \
  } while (0)
#endif

namespace rmpb {

constexpr int kBlock = 256;       // threads per CTA for the policy kernels
#ifndef RMPB_SPEC_LOAD
#define RMPB_SPEC_LOAD 1  // gather before the boundary branch (interp_fast; r02: 12.47 -> 12.43 ms)
#endif
constexpr int kWarps = kBlock / 32;
constexpr int kAcc = 10;          // a00 a01 a02 a11 a12 a22 b0 b1 b2 cnt

// ---------------------------------------------------------------------------
// Grid storage.  Node (i,j,k) sits at origin + (i,j,k)*res (geometry.py:215-221).
//   LINEAR: values[(i*ny + j)*nz + k]                      (reference layout)
//   QUAD  : quad[(i*(ny-1) + j)*(nz-1) + k] = {v[i,j,k], v[i,j,k+1],
//           v[i,j+1,k], v[i,j+1,k+1]}: the 4 z/y corners of a cell column as
//           one 16-B (f32) vector, so one trace step is 2 vector loads
//           (x-planes i and i+1) instead of 8 scalar gathers.
//   BRICK : 8^3 bricks behind a dense brick-index table (block-hashed TSDF,
//           unallocated bricks read as `fill`).
// Values are copied verbatim (f32 storage only when every value is exactly
// representable in f32), so all layouts interpolate bit-identically.
//   PAIR64: f64 z-pairs {v[i,j,k], v[i,j,k+1]} (double2): 4 aligned 16-B loads
//           per step and no f32->f64 conversions.
enum Layout : int { LAYOUT_LINEAR = 0, LAYOUT_QUAD = 1, LAYOUT_BRICK = 2,
                    LAYOUT_PAIR64 = 4 };  // (3: the 2x2x2-blocked QUADB of round 1, removed)

struct GridGeom {
  int nx, ny, nz;
  double ox, oy, oz, res;
  double mx, my, mz;     // n - 1.0 (the clamp bounds)
  double hx, hy, hz;     // origin + (n-1)*res (the slab bounds)
  double rhi, rlo;       // double-double 1/res for the exact division (exdiv)
  double dx2, dy2, dz2;  // (double)(n - 2): the clamped cell's base
  int nxm2, nym2, nzm2;  // n - 2: the last cell index (per-step boundary test)
  int div2;              // 1: exdiv2 is proven exact for divisor res (div2_exact)
};

// Exact a / b for a divisor with precomputed yhi = RN(1/b),
// ylo = RN(fma(-b, yhi, 1) * yhi): q0 = RN(a (yhi + ylo)) is within half an
// ulp (+2^-105 rel) of a/b, hence faithful, and Markstein's correction
// q = RN(q0 + (a - b q0) yhi) is the correctly rounded quotient -- bit-identical
// to IEEE a / b (no exact rounding ties exist for a non-power-of-two divisor;
// for a power of two every step is exact).  4 fp64 ops, no MUFU, no branch.
// Validated: oracle/check_exact_div.c, tests/test_exact_division.py.
__device__ __forceinline__ double exdiv(double a, double b, double yhi, double ylo) {
  double q0 = __fma_rn(a, yhi, __dmul_rn(a, ylo));
  double r = __fma_rn(-q0, b, a);
  return __fma_rn(r, yhi, q0);
}

// The first two operations of exdiv alone, q0 = RN(a yhi + RN(a ylo)), are
// the correctly rounded a / b for every normal |a| >= 2^-960 whenever the
// divisor passes div2_exact() (rmpb_api.cu): the error of q0 is below
// 1.5 * 2^-105 |a/b|, so only quotients within that of a rounding midpoint
// can round the wrong way, and for a fixed b those are the solutions A of
// 2^s A - D == 0 (mod B) with |D| <= 6 (s = 53, 54; A, B the integer
// mantissas) -- a handful per D, each checked directly (window |D| <= 64).
// Every map resolution tried (0.01-0.9, and 98 % of random divisors) passes.
// 2 dependent fp64 ops instead of 4 on the trace step's critical chain.
__device__ __forceinline__ double exdiv2(double a, double yhi, double ylo) {
  return __fma_rn(a, yhi, __dmul_rn(a, ylo));
}

__host__ __device__ inline void recip_dd(double b, double& hi, double& lo) {
  hi = 1.0 / b;
#ifdef __CUDA_ARCH__
  double e = __fma_rn(-b, hi, 1.0);
#else
  double e = __builtin_fma(-b, hi, 1.0);
#endif
  lo = e * hi;
}

__host__ inline GridGeom make_geom(int64_t nx, int64_t ny, int64_t nz, double ox, double oy,
                                   double oz, double res) {
  GridGeom g;
  g.nx = (int)nx; g.ny = (int)ny; g.nz = (int)nz;
  g.ox = ox; g.oy = oy; g.oz = oz; g.res = res;
  g.mx = (double)nx - 1.0; g.my = (double)ny - 1.0; g.mz = (double)nz - 1.0;
  // rmpnav/_kernels/_ckern.pyx:224-226: ox + (nx - 1) * res
  g.hx = ox + (double)(nx - 1) * res;
  g.hy = oy + (double)(ny - 1) * res;
  g.hz = oz + (double)(nz - 1) * res;
  recip_dd(res, g.rhi, g.rlo);
  g.dx2 = (double)(nx - 2); g.dy2 = (double)(ny - 2); g.dz2 = (double)(nz - 2);
  g.nxm2 = (int)nx - 2; g.nym2 = (int)ny - 2; g.nzm2 = (int)nz - 2;
  g.div2 = 0;  // set by the library after div2_exact(res) (rmpb_api.cu)
  return g;
}

// 8 corner values of cell (ix,iy,iz), in the reference's naming v{x}{y}{z}.
struct Corners { double v000, v001, v010, v011, v100, v101, v110, v111; };

template <typename T>
struct LinearGrid {
  static constexpr bool kDiv2 = false;
  const T* __restrict__ v;
  int sy, sx;  // strides: nz, ny*nz (node counts < 2^31 checked at create)
  unsigned lim;  // node count (RMPB_CHECKED builds)
  __device__ __forceinline__ Corners load(int ix, int iy, int iz) const {
    RMPB_CHECK(ix >= 0 && iy >= 0 && iz >= 0 &&
               (unsigned)(ix * sx + iy * sy + iz) + (unsigned)(sx + sy + 1) < lim);
    const T* b = v + (unsigned)(ix * sx + iy * sy + iz);  // < 2^31 nodes (checked at create)
    Corners c;
    c.v000 = (double)__ldg(b);           c.v001 = (double)__ldg(b + 1);
    c.v010 = (double)__ldg(b + sy);      c.v011 = (double)__ldg(b + sy + 1);
    c.v100 = (double)__ldg(b + sx);      c.v101 = (double)__ldg(b + sx + 1);
    c.v110 = (double)__ldg(b + sx + sy); c.v111 = (double)__ldg(b + sx + sy + 1);
    return c;
  }
};

// QUAD: f32 quads {v[i,j,k], v[i,j,k+1], v[i,j+1,k], v[i,j+1,k+1]} stored
// x-fastest, index (iy*(nz-1) + iz)*nx + ix, so the two x-planes a step
// reads are adjacent 16 B records (one 32 B sector when ix is even).  The
// z-fastest order ((ix*(ny-1) + iy)*(nz-1) + iz) measured 12.40-12.58 ms on
// the bench workload vs 12.19-12.22 ms for this one (profiles/README.md).
struct QuadGridF32 {
  static constexpr bool kDiv2 = false;  // see QuadGridF32Div2
  const float4* __restrict__ q;
  int qy, qx;    // qy = nz-1, qx = nx (quads per x row)
  unsigned lim;  // quad count (RMPB_CHECKED builds)
  __device__ __forceinline__ unsigned idx(int ix, int iy, int iz) const {
    return (unsigned)((iy * qy + iz) * qx + ix);
  }
  __device__ __forceinline__ unsigned xstep() const { return 1u; }
  __device__ __forceinline__ Corners load(int ix, int iy, int iz) const {
    RMPB_CHECK(ix >= 0 && iy >= 0 && iz >= 0 && iz < qy && idx(ix, iy, iz) + xstep() < lim);
    const float4* b = q + idx(ix, iy, iz);
    float4 a = __ldg(b), c = __ldg(b + xstep());
    Corners k;
    k.v000 = a.x; k.v001 = a.y; k.v010 = a.z; k.v011 = a.w;
    k.v100 = c.x; k.v101 = c.y; k.v110 = c.z; k.v111 = c.w;
    return k;
  }
};

// The default f32 map when its resolution passes div2_exact(): the same
// loads, and the trace step divides with exdiv2 (bitwise the same quotient).
struct QuadGridF32Div2 : QuadGridF32 {
  static constexpr bool kDiv2 = true;
};
// ... and with the map origin at exactly (0, 0, 0): p - o == p bitwise
// (-0.0 - 0.0 == -0.0, NaN stays NaN), so the subtraction leaves the chain.
struct QuadGridF32Div2O0 : QuadGridF32Div2 {
  static constexpr bool kOrigin0 = true;
};
template <class G, class = void>
struct origin0 { static constexpr bool value = false; };
template <class G>
struct origin0<G, decltype((void)G::kOrigin0)> { static constexpr bool value = G::kOrigin0; };

struct PairGridF64 {
  static constexpr bool kDiv2 = false;
  const double2* __restrict__ q;
  int py, px, pz;  // strides in pairs: y nz-1, x ny*(nz-1), z 1
  int nzm1;        // nz - 1 (RMPB_CHECKED builds)
  unsigned lim;    // pair count (RMPB_CHECKED builds)
  __device__ __forceinline__ Corners load(int ix, int iy, int iz) const {
    RMPB_CHECK(ix >= 0 && iy >= 0 && iz >= 0 && iz < nzm1 &&
               (unsigned)(ix * px + iy * py + iz * pz) + (unsigned)(px + py) < lim);
    const double2* b = q + (unsigned)(ix * px + iy * py + iz * pz);
    double2 a0 = __ldg(b), a1 = __ldg(b + (unsigned)py);
    double2 c0 = __ldg(b + (unsigned)px), c1 = __ldg(b + (unsigned)(px + py));
    Corners k;
    k.v000 = a0.x; k.v001 = a0.y; k.v010 = a1.x; k.v011 = a1.y;
    k.v100 = c0.x; k.v101 = c0.y; k.v110 = c1.x; k.v111 = c1.y;
    return k;
  }
};
// f64 maps whose resolution passes div2_exact() / with the origin at +0: the
// same 2-op division and origin-0 forms as the QUAD accessors.
struct PairGridF64Div2 : PairGridF64 {
  static constexpr bool kDiv2 = true;
};
struct PairGridF64Div2O0 : PairGridF64Div2 {
  static constexpr bool kOrigin0 = true;
};

// Block-hashed sparse grid: bricks of B^3 nodes; brick (bi,bj,bk) ->
// table[(bi*bny + bj)*bnz + bk] = brick slot or -1 (unallocated -> fill).
template <typename T>
struct BrickGrid {
  static constexpr bool kDiv2 = false;
  const T* __restrict__ pool;          // slot * B^3 + ((li*B)+lj)*B + lk
  const int32_t* __restrict__ table;
  int bny, bnz;
  T fill;
  unsigned tlim, plim;  // table entries, allocated bricks (RMPB_CHECKED builds)
  static constexpr int B = 8;
  __device__ __forceinline__ double at(int i, int j, int k) const {
    RMPB_CHECK(i >= 0 && j >= 0 && k >= 0 &&
               (unsigned)(((i >> 3) * bny + (j >> 3)) * bnz + (k >> 3)) < tlim);
    int s = __ldg(table + ((i >> 3) * bny + (j >> 3)) * bnz + (k >> 3));
    RMPB_CHECK(s < (int)plim);
    if (s < 0) return (double)fill;
    return (double)__ldg(pool + (int64_t)s * 512 + (((i & 7) << 6) | ((j & 7) << 3) | (k & 7)));
  }
  __device__ __forceinline__ Corners load(int ix, int iy, int iz) const {
    Corners c;
    if (((ix & 7) < 7) & ((iy & 7) < 7) & ((iz & 7) < 7)) {
      // all 8 corners in one brick (343 of 512 cells): one table lookup
      RMPB_CHECK(ix >= 0 && iy >= 0 && iz >= 0 &&
                 (unsigned)(((ix >> 3) * bny + (iy >> 3)) * bnz + (iz >> 3)) < tlim);
      const int sl = __ldg(table + ((ix >> 3) * bny + (iy >> 3)) * bnz + (iz >> 3));
      RMPB_CHECK(sl < (int)plim);
      if (sl < 0) {
        const double f = (double)fill;
        c.v000 = c.v001 = c.v010 = c.v011 = c.v100 = c.v101 = c.v110 = c.v111 = f;
        return c;
      }
      const T* q = pool + (int64_t)sl * 512 + (((ix & 7) << 6) | ((iy & 7) << 3) | (iz & 7));
      c.v000 = (double)__ldg(q);      c.v001 = (double)__ldg(q + 1);
      c.v010 = (double)__ldg(q + 8);  c.v011 = (double)__ldg(q + 9);
      c.v100 = (double)__ldg(q + 64); c.v101 = (double)__ldg(q + 65);
      c.v110 = (double)__ldg(q + 72); c.v111 = (double)__ldg(q + 73);
      return c;
    }
    c.v000 = at(ix, iy, iz);         c.v001 = at(ix, iy, iz + 1);
    c.v010 = at(ix, iy + 1, iz);     c.v011 = at(ix, iy + 1, iz + 1);
    c.v100 = at(ix + 1, iy, iz);     c.v101 = at(ix + 1, iy, iz + 1);
    c.v110 = at(ix + 1, iy + 1, iz); c.v111 = at(ix + 1, iy + 1, iz + 1);
    return c;
  }
};

// Block-hashed f32 map, bricks of 8^3 CELLS stored as QUAD records with a
// one-node apron: brick (bi, bj, bk) holds, for li in 0..8 and lj, lk in
// 0..7, the record {v[i,j,k], v[i,j,k+1], v[i,j+1,k], v[i,j+1,k+1]} of node
// (i, j, k) = 8 (bi, bj, bk) + (li, lj, lk) at (lj*8 + lk)*9 + li -- so every
// cell whose base lies in the brick reads its 8 corners as two adjacent
// 16-B records of ONE brick: a table lookup + 2 gathers per step (the
// scalar-pool layout needed a lookup + 8 gathers, and 8 lookups at brick
// faces).  A brick is allocated when any node of its 9^3 apron box differs
// from `fill`, so an unallocated brick's cells have every corner == fill.
struct BrickQuadF32 {
  static constexpr bool kDiv2 = false;
  const float4* __restrict__ pool;    // slot * 576 + (lj*8 + lk)*9 + li
  const int32_t* __restrict__ table;  // (bi*bny + bj)*bnz + bk -> slot or -1
  int bny, bnz;
  float fill;
  unsigned tlim, plim;  // table entries, allocated bricks (RMPB_CHECKED builds)
  __device__ __forceinline__ Corners load(int ix, int iy, int iz) const {
    RMPB_CHECK(ix >= 0 && iy >= 0 && iz >= 0 &&
               (unsigned)(((ix >> 3) * bny + (iy >> 3)) * bnz + (iz >> 3)) < tlim);
    const int sl = __ldg(table + ((ix >> 3) * bny + (iy >> 3)) * bnz + (iz >> 3));
    RMPB_CHECK(sl < (int)plim);
    Corners k;
    if (sl < 0) {
      const double f = (double)fill;
      k.v000 = k.v001 = k.v010 = k.v011 = k.v100 = k.v101 = k.v110 = k.v111 = f;
      return k;
    }
    const float4* b = pool + (size_t)sl * 576 + ((((iy & 7) << 3) | (iz & 7)) * 9 + (ix & 7));
    const float4 a = __ldg(b), c = __ldg(b + 1);
    k.v000 = a.x; k.v001 = a.y; k.v010 = a.z; k.v011 = a.w;
    k.v100 = c.x; k.v101 = c.y; k.v110 = c.z; k.v111 = c.w;
    return k;
  }
};
struct BrickQuadF32Div2 : BrickQuadF32 {
  static constexpr bool kDiv2 = true;
};
struct BrickQuadF32Div2O0 : BrickQuadF32Div2 {
  static constexpr bool kOrigin0 = true;
};

// ---------------------------------------------------------------------------
// Exact interpolation (rmpnav/_kernels/_ckern.pyx:92-135).
template <class G>
__device__ __forceinline__ double interp(const G& grid, const GridGeom& g, double px, double py,
                                         double pz, int& ix, int& iy, int& iz) {
  double ux = (px - g.ox) / g.res;
  double uy = (py - g.oy) / g.res;
  double uz = (pz - g.oz) / g.res;
  if (ux < 0.0) ux = 0.0; else if (ux > g.mx) ux = g.mx;
  if (uy < 0.0) uy = 0.0; else if (uy > g.my) uy = g.my;
  if (uz < 0.0) uz = 0.0; else if (uz > g.mz) uz = g.mz;
  // (uint) makes a NaN coordinate (undefined in the reference) a safe index.
  ix = (int)floor(ux); iy = (int)floor(uy); iz = (int)floor(uz);
  ix = min(max(ix, 0), g.nx - 2);
  iy = min(max(iy, 0), g.ny - 2);
  iz = min(max(iz, 0), g.nz - 2);
  double fx = ux - (double)ix, fy = uy - (double)iy, fz = uz - (double)iz;
  Corners c = grid.load(ix, iy, iz);
  double c00 = c.v000 + fz * (c.v001 - c.v000);
  double c01 = c.v010 + fz * (c.v011 - c.v010);
  double c10 = c.v100 + fz * (c.v101 - c.v100);
  double c11 = c.v110 + fz * (c.v111 - c.v110);
  double c0 = c00 + fy * (c01 - c00);
  double c1 = c10 + fy * (c11 - c10);
  return c0 + fx * (c1 - c0);
}

// Cell coordinate of one axis, identical to the reference's
//   u = clamp(u, 0, n-1); i = min((int64)floor(u), n-2); f = u - (double)i
// without the XU pipe and without selects on the common path: with
// M = 1.5 * 2^52 (ulp 1 on [2^52, 2^53)) and |u| < 2^51, RZ(u + M) - M is
// exactly floor(u) (the sum is positive, so round-toward-zero rounds down),
// and the low mantissa word of RZ(u + M) is floor(u) as a two's-complement
// int.  Then f = u - floor(u) is the reference's f whenever floor(u) lies in
// [0, n-2]; otherwise the reference clamped u: see cell_fix (rare, only at
// the map boundary).
__device__ __forceinline__ void cell_floor(double u, int& i, double& f) {
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  const double big = __dadd_rz(u, M);
  i = __double2loint(big);
  f = u - (big - M);
}
// u < 0 -> (0, 0); u >= n-1 -> (n-2, (n-1) - (n-2) = 1).
__device__ __forceinline__ void cell_fix(int nm2, int& i, double& f) {
  if ((unsigned)i > (unsigned)nm2) {
    if (i < 0) { i = 0; f = 0.0; } else { i = nm2; f = 1.0; }
  }
}

// Cell of a point (the reference's clamp + floor + fraction, before the
// boundary fix): exdiv2 / origin-0 forms per accessor type.
template <class G>
__device__ __forceinline__ void locate(const GridGeom& g, double px, double py, double pz,
                                       int& ix, int& iy, int& iz, double& fx, double& fy,
                                       double& fz) {
  if constexpr (origin0<G>::value) {
    cell_floor(exdiv2(px, g.rhi, g.rlo), ix, fx);
    cell_floor(exdiv2(py, g.rhi, g.rlo), iy, fy);
    cell_floor(exdiv2(pz, g.rhi, g.rlo), iz, fz);
  } else if constexpr (G::kDiv2) {
    cell_floor(exdiv2(px - g.ox, g.rhi, g.rlo), ix, fx);
    cell_floor(exdiv2(py - g.oy, g.rhi, g.rlo), iy, fy);
    cell_floor(exdiv2(pz - g.oz, g.rhi, g.rlo), iz, fz);
  } else {
    cell_floor(exdiv(px - g.ox, g.res, g.rhi, g.rlo), ix, fx);
    cell_floor(exdiv(py - g.oy, g.res, g.rhi, g.rlo), iy, fy);
    cell_floor(exdiv(pz - g.oz, g.res, g.rhi, g.rlo), iz, fz);
  }
}
__device__ __forceinline__ bool out_of_cells(const GridGeom& g, int ix, int iy, int iz) {
  return ((unsigned)ix > (unsigned)g.nxm2) | ((unsigned)iy > (unsigned)g.nym2) |
         ((unsigned)iz > (unsigned)g.nzm2);
}
// The reference's trilinear interpolation order (_ckern.pyx:126-135).
__device__ __forceinline__ double lerp8(const Corners& c, double fx, double fy, double fz) {
  double c00 = c.v000 + fz * (c.v001 - c.v000);
  double c01 = c.v010 + fz * (c.v011 - c.v010);
  double c10 = c.v100 + fz * (c.v101 - c.v100);
  double c11 = c.v110 + fz * (c.v111 - c.v110);
  double c0 = c00 + fy * (c01 - c00);
  double c1 = c10 + fy * (c11 - c10);
  return c0 + fx * (c1 - c0);
}

// interp with exdiv + cell_floor / cell_fix: bit-identical to interp() above.
template <class G>
__device__ __forceinline__ double interp_fast(const G& grid, const GridGeom& g, double px,
                                              double py, double pz, int& ix, int& iy, int& iz) {
  double fx, fy, fz;
  locate<G>(g, px, py, pz, ix, iy, iz, fx, fy, fz);
#if RMPB_SPEC_LOAD
  // The gather issues right after the floor, with the indices clamped into
  // the map (unsigned min: in bounds whatever they are); only a step outside
  // the clamp range -- the map boundary, rare -- fixes the cell (reference
  // clamps) and gathers again.  Keeps the boundary test's compare + branch
  // off the dependent chain in front of the L2 gather.
  const bool oob = out_of_cells(g, ix, iy, iz);
  Corners c = grid.load((int)min((unsigned)ix, (unsigned)g.nxm2),
                        (int)min((unsigned)iy, (unsigned)g.nym2),
                        (int)min((unsigned)iz, (unsigned)g.nzm2));
  if (oob) {
    cell_fix(g.nxm2, ix, fx);
    cell_fix(g.nym2, iy, fy);
    cell_fix(g.nzm2, iz, fz);
    c = grid.load(ix, iy, iz);
  }
#else
  // one (rarely taken) branch for all three boundary clamps
  if (out_of_cells(g, ix, iy, iz)) {
    cell_fix(g.nxm2, ix, fx);
    cell_fix(g.nym2, iy, fy);
    cell_fix(g.nzm2, iz, fz);
  }
  Corners c = grid.load(ix, iy, iz);
#endif
  return lerp8(c, fx, fy, fz);
}

// ---------------------------------------------------------------------------
// FAST mode (opt-in, NOT reference-exact): the same stepping rule in fp32
// with FMA -- about half the instructions and twice the pipe rate of the
// exact fp64 step.  Hit masks / distances can differ from the reference for
// rays grazing a surface (SURVEY.md §7 hard parts); the deviation is
// measured in tests/test_gpu_parity.py and reported, never mixed with the
// exact path's parity claims.
struct CornersF { float v000, v001, v010, v011, v100, v101, v110, v111; };

template <class G>
__device__ __forceinline__ CornersF load_f(const G& grid, int ix, int iy, int iz) {
  if constexpr (std::is_base_of<QuadGridF32, G>::value) {  // f32 corners straight from the quads
    const float4* b = grid.q + grid.idx(ix, iy, iz);
    const float4 a = __ldg(b), c = __ldg(b + grid.xstep());
    return CornersF{a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
  } else {
    const Corners c = grid.load(ix, iy, iz);
    return CornersF{(float)c.v000, (float)c.v001, (float)c.v010, (float)c.v011,
                    (float)c.v100, (float)c.v101, (float)c.v110, (float)c.v111};
  }
}
struct GeomF {
  float ox, oy, oz, inv;
  int nx2, ny2, nz2;
};

__device__ __forceinline__ void cell_floor_f(float u, int nm2, int& i, float& f) {
  const float M = 12582912.0f;  // 1.5 * 2^23: RZ(u + M) - M = floor(u), |u| < 2^22
  const float big = __fadd_rz(u, M);
  i = __float_as_int(big) - 0x4B400000;
  f = u - (big - M);
  if ((unsigned)i > (unsigned)nm2) {
    if (i < 0) { i = 0; f = 0.0f; } else { i = nm2; f = 1.0f; }
  }
}

template <class G>
__device__ __forceinline__ float interp_f(const G& grid, const GeomF& g, float px, float py,
                                          float pz) {
  int ix, iy, iz;
  float fx, fy, fz;
  cell_floor_f((px - g.ox) * g.inv, g.nx2, ix, fx);
  cell_floor_f((py - g.oy) * g.inv, g.ny2, iy, fy);
  cell_floor_f((pz - g.oz) * g.inv, g.nz2, iz, fz);
  const CornersF c = load_f(grid, ix, iy, iz);
  const float c00 = __fmaf_rn(fz, c.v001 - c.v000, c.v000);
  const float c01 = __fmaf_rn(fz, c.v011 - c.v010, c.v010);
  const float c10 = __fmaf_rn(fz, c.v101 - c.v100, c.v100);
  const float c11 = __fmaf_rn(fz, c.v111 - c.v110, c.v110);
  const float c0 = __fmaf_rn(fy, c01 - c00, c00);
  const float c1 = __fmaf_rn(fy, c11 - c10, c10);
  return __fmaf_rn(fx, c1 - c0, c0);
}

// Slab quotient (bound - s) / d: the reference's IEEE division
// (_ckern.pyx:171-212), bit-identical for every input (tiny numerators,
// subnormal direction components, overflowing quotients included).
// (r2: a per-ray double-double reciprocal with exdiv and an IEEE fallback
// branch was SLOWER than the native division here -- 12.19 vs 11.3 ms per
// 4096-pose step; it is once per ray, off the step chain.)
__device__ __forceinline__ double slab_div(double a, double d) { return a / d; }

// Slab interval against the node domain (rmpnav/_kernels/_ckern.pyx:171-212).
__device__ __forceinline__ bool box_span(const GridGeom& g, double sx, double sy, double sz,
                                         double dx, double dy, double dz, double& t0, double& t1) {
  double tlo = -CUDART_INF, thi = CUDART_INF, ta, tb, tmp;
  if (dx != 0.0) {
    ta = (g.ox - sx) / dx; tb = (g.hx - sx) / dx;
    if (tb < ta) { tmp = ta; ta = tb; tb = tmp; }
    if (ta > tlo) tlo = ta;
    if (tb < thi) thi = tb;
  } else if (sx < g.ox || sx > g.hx) {
    return false;
  }
  if (dy != 0.0) {
    ta = (g.oy - sy) / dy; tb = (g.hy - sy) / dy;
    if (tb < ta) { tmp = ta; ta = tb; tb = tmp; }
    if (ta > tlo) tlo = ta;
    if (tb < thi) thi = tb;
  } else if (sy < g.oy || sy > g.hy) {
    return false;
  }
  if (dz != 0.0) {
    ta = (g.oz - sz) / dz; tb = (g.hz - sz) / dz;
    if (tb < ta) { tmp = ta; ta = tb; tb = tmp; }
    if (ta > tlo) tlo = ta;
    if (tb < thi) thi = tb;
  } else if (sz < g.oz || sz > g.hz) {
    return false;
  }
  t0 = tlo; t1 = thi;
  return true;
}

struct TraceResult {
  double t;     // hit distance, +inf on miss
  int cx, cy, cz;  // cell of the terminating interpolation (valid on hit)
  int steps;    // interpolation calls ("voxel-steps")
};

// Sphere trace (rmpnav/_kernels/_ckern.pyx:217-248).
template <class G>
__device__ __forceinline__ TraceResult trace_ray(const G& grid, const GridGeom& g, double sx,
                                                 double sy, double sz, double dx, double dy,
                                                 double dz, double max_range, double eps,
                                                 double step_scale) {
  TraceResult r;
  r.t = CUDART_INF; r.cx = r.cy = r.cz = -1; r.steps = 0;
  double t0, t1;
  if (!box_span(g, sx, sy, sz, dx, dy, dz, t0, t1)) return r;
  double t = t0 > 0.0 ? t0 : 0.0;
  double t_end = t1 < max_range ? t1 : max_range;
  if (t > t_end) return r;
  int ix, iy, iz;
  while (true) {
    double d = interp(grid, g, sx + t * dx, sy + t * dy, sz + t * dz, ix, iy, iz);
    ++r.steps;
    if (d < eps) { r.t = t; r.cx = ix; r.cy = iy; r.cz = iz; break; }
    t += step_scale * d;
    if (!(t <= t_end)) break;  // NaN-safe form of (t > t_end)
  }
  return r;
}

// Sphere trace with the exact fast arithmetic (interp_fast): bit-identical
// to trace_ray.
template <class G>
__device__ __forceinline__ TraceResult trace_ray_fast(const G& grid, const GridGeom& g, double sx,
                                                      double sy, double sz, double dx, double dy,
                                                      double dz, double max_range, double eps,
                                                      double step_scale) {
  TraceResult r;
  r.t = CUDART_INF; r.cx = r.cy = r.cz = -1; r.steps = 0;
  double t0, t1;
  if (!box_span(g, sx, sy, sz, dx, dy, dz, t0, t1)) return r;
  double t = t0 > 0.0 ? t0 : 0.0;
  const double t_end = t1 < max_range ? t1 : max_range;
  if (t > t_end) return r;
  int ix, iy, iz;
  while (true) {
    const double d = interp_fast(grid, g, sx + t * dx, sy + t * dy, sz + t * dz, ix, iy, iz);
    ++r.steps;
    if (d < eps) { r.t = t; r.cx = ix; r.cy = iy; r.cz = iz; break; }
    t += step_scale * d;
    if (!(t <= t_end)) break;
  }
  return r;
}

// trace_ray_fast for a start inside the node domain, given the pose's first
// step (d0 = interp at the start, shared by every ray of the pose): the
// entry side drops out (t0 = 0 exactly) and, with `skip1` (d0 >= eps and no
// -0.0 coordinate, as k_ray_policy2), a ray with a finite direction starts
// at t = 0 + step * d0 with one step counted -- bitwise trace_ray_fast.
template <class G>
__device__ __forceinline__ TraceResult trace_ray_inside(const G& grid, const GridGeom& g,
                                                        double sx, double sy, double sz,
                                                        double dx, double dy, double dz,
                                                        double max_range,
                                                        double eps, double step_scale, bool skip1,
                                                        double t1s) {
  TraceResult r;
  r.t = CUDART_INF; r.cx = r.cy = r.cz = -1; r.steps = 0;
  double thi = CUDART_INF;
  if (dx != 0.0) {
    const double tb = slab_div((dx > 0.0 ? g.hx : g.ox) - sx, dx);
    thi = tb < thi ? tb : thi;
  }
  if (dy != 0.0) {
    const double tb = slab_div((dy > 0.0 ? g.hy : g.oy) - sy, dy);
    thi = tb < thi ? tb : thi;
  }
  if (dz != 0.0) {
    const double tb = slab_div((dz > 0.0 ? g.hz : g.oz) - sz, dz);
    thi = tb < thi ? tb : thi;
  }
  const double t_end = thi < max_range ? thi : max_range;
  double t = 0.0;
  if (t > t_end) return r;
  if (skip1 && isfinite(dx) && isfinite(dy) && isfinite(dz)) {
    r.steps = 1;
    t = t1s;
    if (!(t <= t_end)) return r;
  }
  int ix, iy, iz;
  while (true) {
    const double d = interp_fast(grid, g, sx + t * dx, sy + t * dy, sz + t * dz, ix, iy, iz);
    ++r.steps;
    if (d < eps) { r.t = t; r.cx = ix; r.cy = iy; r.cz = iz; break; }
    t += step_scale * d;
    if (!(t <= t_end)) break;
  }
  return r;
}

// ---------------------------------------------------------------------------
// Per-ray obstacle policy (rmpnav/_kernels/_ckern.pyx:290-316).  `dir` is the
// cast direction; r = -dir points away from the obstacle (policies.py:550-552).
struct PolicyParams {
  double eta_rep, nu_rep, eta_damp, nu_damp, eps_p, radius, c;  // as_tuple order, policies.py:80-83
  double min_range;
  // double-double reciprocals of the constant divisors (exdiv): nu_rep,
  // nu_damp, radius and RN(radius * radius)
  double rnr_h, rnr_l, rnd_h, rnd_l, rr_h, rr_l, rr2, rr2_h, rr2_l;
};

struct Acc {
  double a00, a01, a02, a11, a12, a22, b0, b1, b2;
  int cnt;
  __device__ __forceinline__ void zero() {
    a00 = a01 = a02 = a11 = a12 = a22 = b0 = b1 = b2 = 0.0;
    cnt = 0;
  }
};

// Adds ray (dir, dist) to `acc`.  Rays with a == 0 add nothing but the count
// (x + 0 == x exactly), so the transcendental work is only done where the
// metric weight can be nonzero: d < radius AND toward > 0 (w == 0 or g == 0
// give fdamp*... == 0 and a == (w*smag)*smag == 0 exactly).
__device__ __forceinline__ void policy_accumulate(Acc& acc, double dx, double dy, double dz,
                                                  double d, double vx, double vy, double vz,
                                                  const PolicyParams& p) {
  if (d != d || d == CUDART_INF || d < p.min_range) return;
  acc.cnt += 1;
  double toward = dx * vx + dy * vy + dz * vz;
  if (!(d < p.radius) || !(toward > 0.0)) return;
  double rx = -dx, ry = -dy, rz = -dz;
  // Divisions by the constant parameters: exdiv2 (within half an ulp + 2^-105
  // of the quotient, usually the correctly rounded one).  The policy sums are
  // compared at 1e-9 relative (libm exp / log1p differ by ulps anyway), and
  // the shorter chain is what bounds a 32-lane policy batch.
  double frep = p.eta_rep * exp(exdiv2(-d, p.rnr_h, p.rnr_l));
  double g = toward;
  double fdamp = p.eta_damp / (exdiv2(d, p.rnd_h, p.rnd_l) + p.eps_p) * g * g;
  double w = exdiv2(d * d, p.rr2_h, p.rr2_l) - exdiv2(2.0 * d, p.rr_h, p.rr_l) + 1.0;
  double smag = fdamp / (fdamp + p.c * log1p(exp(-2.0 * p.c * fdamp)));
  double a = w * smag * smag;
  if (a != 0.0) {
    acc.a00 += a * rx * rx; acc.a01 += a * rx * ry; acc.a02 += a * rx * rz;
    acc.a11 += a * ry * ry; acc.a12 += a * ry * rz; acc.a22 += a * rz * rz;
    double bf = a * (frep + fdamp);
    acc.b0 += bf * rx; acc.b1 += bf * ry; acc.b2 += bf * rz;
  }
}

// policy_accumulate with the per-beam transcendental math in fp32 (opt-in
// LiDAR "fast" mode, NOT reference-exact): the counted / in-radius /
// closing decisions are the fp64 ones, so the same beams contribute; each
// contribution carries ~1e-7 relative error (north_star's bar for the sums
// is 1e-5 relative in fp32) and is accumulated in fp64.
__device__ __forceinline__ void policy_accumulate_f32(Acc& acc, double dx, double dy, double dz,
                                                      double d, double vx, double vy, double vz,
                                                      const PolicyParams& p) {
  if (d != d || d == CUDART_INF || d < p.min_range) return;
  acc.cnt += 1;
  const double toward = dx * vx + dy * vy + dz * vz;
  if (!(d < p.radius) || !(toward > 0.0)) return;
  const float df = (float)d, gf = (float)toward;
  const float frep = (float)p.eta_rep * __expf(-df * (float)p.rnr_h);
  const float fdamp = __fdividef((float)p.eta_damp, df * (float)p.rnd_h + (float)p.eps_p) * gf * gf;
  const float x = 1.0f - df * (float)p.rr_h;  // w = (1 - d/r)^2
  const float w = x * x;
  const float cf = (float)p.c;
  const float smag = __fdividef(fdamp, fdamp + cf * log1pf(__expf(-2.0f * cf * fdamp)));
  const float a = w * smag * smag;
  if (a != 0.0f) {
    const double ad = (double)a, rx = -dx, ry = -dy, rz = -dz;
    acc.a00 += ad * rx * rx; acc.a01 += ad * rx * ry; acc.a02 += ad * rx * rz;
    acc.a11 += ad * ry * ry; acc.a12 += ad * ry * rz; acc.a22 += ad * rz * rz;
    const double bf = (double)(a * (frep + fdamp));
    acc.b0 += bf * rx; acc.b1 += bf * ry; acc.b2 += bf * rz;
  }
}

// ---------------------------------------------------------------------------
// Deterministic block reduction: butterfly shuffles inside each warp (fixed
// pairing), then warp partials summed in warp order.  The result does not
// depend on timing, so repeated launches are bitwise identical.
__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ int warp_sum_i(int x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Returns the block total in thread 0 (other threads: undefined).
// `sm` must hold NW*kAcc doubles (NW = warps per CTA).
template <int NW = kWarps>
__device__ __forceinline__ void block_reduce(Acc& acc, double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  bool any = __any_sync(0xffffffffu, acc.a00 != 0.0 || acc.a11 != 0.0 || acc.a22 != 0.0 ||
                                         acc.b0 != 0.0 || acc.b1 != 0.0 || acc.b2 != 0.0 ||
                                         acc.a01 != 0.0 || acc.a02 != 0.0 || acc.a12 != 0.0);
  double v[kAcc];
  v[0] = acc.a00; v[1] = acc.a01; v[2] = acc.a02; v[3] = acc.a11; v[4] = acc.a12;
  v[5] = acc.a22; v[6] = acc.b0; v[7] = acc.b1; v[8] = acc.b2;
  if (any) {
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = warp_sum(v[k]);
  }
  v[9] = (double)warp_sum_i(acc.cnt);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kAcc; ++k) sm[warp * kAcc + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s[kAcc];
#pragma unroll
    for (int k = 0; k < kAcc; ++k) s[k] = sm[k];
    for (int w = 1; w < NW; ++w) {
#pragma unroll
      for (int k = 0; k < kAcc; ++k) s[k] += sm[w * kAcc + k];
    }
    acc.a00 = s[0]; acc.a01 = s[1]; acc.a02 = s[2]; acc.a11 = s[3]; acc.a12 = s[4];
    acc.a22 = s[5]; acc.b0 = s[6]; acc.b1 = s[7]; acc.b2 = s[8]; acc.cnt = (int)s[9];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// pinv_psd (rmpnav/core.py:103-115): eigen-decomposition of the symmetric 3x3
// metric by cyclic Jacobi in fp64; eigenvalues <= 1e-8 * max(lambda_max, 0)
// are dropped; accel = V diag(1/lambda) V^T Af.
__device__ __forceinline__ void jacobi3(double a[3][3], double V[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 32; ++sweep) {
    double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    double diag = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]);
    if (off == 0.0 || off <= 1e-300 || off < 1e-18 * diag) break;
    // fully unrolled rotations (0,1), (0,2), (1,2): every index is a
    // compile-time constant, so a and V stay in registers
#pragma unroll
    for (int p = 0; p < 2; ++p) {
#pragma unroll
      for (int q = p + 1; q < 3; ++q) {
        double apq = a[p][q];
        if (apq == 0.0) continue;
        double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        if (!isfinite(theta)) t = 0.5 / theta;  // |theta| huge: t ~ 1/(2 theta)
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
#pragma unroll
        for (int k = 0; k < 3; ++k) {  // A <- A J
          double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {  // A <- J^T A
          double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        a[p][q] = a[q][p] = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {  // V <- V J
          double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = c * vkp - s * vkq;
          V[k][q] = s * vkp + c * vkq;
        }
      }
    }
  }
}

// Fast path: a Cholesky solve when the (PSD) metric is provably far from the
// pinv_psd cutoff.  Every pivot d_i is positive and at most tr (d_i <= m_ii),
// and det = d0 d1 d2 = l0 l1 l2; so det >= 1e-6 tr^3 gives
//   lambda_min >= det / (l_mid l_max) >= det / tr^2 >= 1e-6 tr >= 1e-6 lambda_max,
// 100x above pinv_psd's 1e-8 * lambda_max cutoff: nothing is dropped and
// pinv(M) f = M^-1 f, which the solve gives to ~cond(M) * 2^-53 <= 1e-10
// relative (~30 dependent fp64 ops instead of Jacobi sweeps: 4.4 -> ~1 us on
// one pose's final CTA).  Returns false otherwise (rank-deficient or badly
// conditioned metrics: the Jacobi path).
__device__ inline bool chol_solve3(const double m[9], const double f[3], double out[3]) {
  const double tr = m[0] + m[4] + m[8];
  if (!(tr > 1e-90) || !(tr < 1e90)) return false;  // (tr^3 and det stay normal)
  const double d0 = m[0];
  if (!(d0 > 0.0)) return false;
  const double l00 = sqrt(d0);
  const double l10 = m[3] / l00, l20 = m[6] / l00;
  const double d1 = m[4] - l10 * l10;
  if (!(d1 > 0.0)) return false;
  const double l11 = sqrt(d1);
  const double l21 = (m[7] - l20 * l10) / l11;
  const double d2 = m[8] - l20 * l20 - l21 * l21;
  if (!(d2 > 0.0) || !(d0 * d1 * d2 >= 1e-6 * tr * tr * tr)) return false;
  const double l22 = sqrt(d2);
  const double y0 = f[0] / l00;
  const double y1 = (f[1] - l10 * y0) / l11;
  const double y2 = (f[2] - l20 * y0 - l21 * y1) / l22;
  out[2] = y2 / l22;
  out[1] = (y1 - l21 * out[2]) / l11;
  out[0] = (y0 - l10 * out[1] - l20 * out[2]) / l00;
  return true;
}

// m: symmetric metric (row-major 9), f: weighted sum (3) -> accel (3).
__device__ inline void pinv_apply(const double m[9], const double f[3], double out[3]) {
  if (chol_solve3(m, f, out)) return;
  double a[3][3], V[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) a[i][j] = 0.5 * (m[3 * i + j] + m[3 * j + i]);
  jacobi3(a, V);
  double lam[3] = {a[0][0], a[1][1], a[2][2]};
  double lmax = fmax(fmax(lam[0], lam[1]), lam[2]);
  double cut = 1e-8 * (lmax > 0.0 ? lmax : 0.0);
  double y[3];
  for (int k = 0; k < 3; ++k) {
    double vf = V[0][k] * f[0] + V[1][k] * f[1] + V[2][k] * f[2];
    y[k] = lam[k] > cut ? vf / lam[k] : 0.0;
  }
  for (int i = 0; i < 3; ++i) out[i] = V[i][0] * y[0] + V[i][1] * y[1] + V[i][2] * y[2];
}

// 13-slot layout of ckern.policy_reduce before reshaping (ckern.py:91-93):
// [A (9, symmetric duplicated), Af (3), count].
__device__ __forceinline__ void write_slot(const Acc& s, double* slot, double* accel) {
  double m[9] = {s.a00, s.a01, s.a02, s.a01, s.a11, s.a12, s.a02, s.a12, s.a22};
  double f[3] = {s.b0, s.b1, s.b2};
  for (int k = 0; k < 9; ++k) slot[k] = m[k];
  slot[9] = f[0]; slot[10] = f[1]; slot[11] = f[2];
  slot[12] = (double)s.cnt;
  if (accel) pinv_apply(m, f, accel);
}

}  // namespace rmpb
