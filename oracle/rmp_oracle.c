/*
 * rmp_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.  The
 * product (paper_2301_08068_b200) never links, imports or calls this file.
 *
 * Restates SURVEY.md Appendix A, which in turn follows the reference
 * (paths relative to /root/reference/pkg/src/rmpnav/):
 *   - node-grid trilinear interpolation ........ _kernels/_ckern.pyx:92-135
 *   - ray / node-domain slab interval .......... _kernels/_ckern.pyx:171-212
 *   - sphere trace on the grid ................. _kernels/_ckern.pyx:217-248
 *   - per-ray obstacle policy + 13-slot sum .... _kernels/_ckern.pyx:278-321
 *   - fixed 2048-ray chunks + pairwise fold .... _kernels/_pool.py:14,31-33,61-72
 *   - analytic scene signed distance ........... _kernels/_ckern.pyx:21-56
 *   - bake / scene trace / esdf sample ......... _kernels/_ckern.pyx:71-87,251-273,138-166
 *
 * Parity pinning: every function here is checked bit-for-bit against the
 * reference's own compiled module (oracle/_ref, built by build_ref.py from
 * the reference .pyx) and against the committed golden vectors under
 * tests/golden/ (tests/test_oracle.py).
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (see oracle/Makefile).  No
 * FMA contraction: the reference module is scalar SSE2 fp64 with no FMA.
 *
 * Extra outputs the reference does not have (defined by this build, see
 * DESIGN.md): the hit cell (ix,iy,iz) used by the terminating interpolation,
 * and the number of interpolation calls ("voxel-steps") per ray.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define ORC_CHUNK 2048

typedef struct {
    const double *v;
    int64_t nx, ny, nz;
    double ox, oy, oz, res;
} orc_grid;

/* _ckern.pyx:92-135 -- clamp u to [0, n-1], cell <= n-2, lerps z -> y -> x. */
static double orc_interp(const orc_grid *g, double px, double py, double pz,
                         int64_t *cx, int64_t *cy, int64_t *cz)
{
    double ux = (px - g->ox) / g->res;
    double uy = (py - g->oy) / g->res;
    double uz = (pz - g->oz) / g->res;
    double mx = (double)g->nx - 1.0, my = (double)g->ny - 1.0, mz = (double)g->nz - 1.0;
    if (ux < 0.0) ux = 0.0; else if (ux > mx) ux = mx;
    if (uy < 0.0) uy = 0.0; else if (uy > my) uy = my;
    if (uz < 0.0) uz = 0.0; else if (uz > mz) uz = mz;
    int64_t ix = (int64_t)floor(ux), iy = (int64_t)floor(uy), iz = (int64_t)floor(uz);
    if (ix > g->nx - 2) ix = g->nx - 2;
    if (iy > g->ny - 2) iy = g->ny - 2;
    if (iz > g->nz - 2) iz = g->nz - 2;
    double fx = ux - (double)ix, fy = uy - (double)iy, fz = uz - (double)iz;
    const int64_t sy = g->nz, sx = g->ny * g->nz;
    const double *b = g->v + ix * sx + iy * sy + iz;
    double v000 = b[0], v001 = b[1];
    double v010 = b[sy], v011 = b[sy + 1];
    double v100 = b[sx], v101 = b[sx + 1];
    double v110 = b[sx + sy], v111 = b[sx + sy + 1];
    double c00 = v000 + fz * (v001 - v000);
    double c01 = v010 + fz * (v011 - v010);
    double c10 = v100 + fz * (v101 - v100);
    double c11 = v110 + fz * (v111 - v110);
    double c0 = c00 + fy * (c01 - c00);
    double c1 = c10 + fy * (c11 - c10);
    if (cx) { *cx = ix; *cy = iy; *cz = iz; }
    return c0 + fx * (c1 - c0);
}

/* _ckern.pyx:171-212 -- slab test, axes in x, y, z order; zero-direction branch. */
static int orc_box_span(const double s[3], const double d[3], const double lo[3],
                        const double hi[3], double *t0, double *t1)
{
    double tlo = -INFINITY, thi = INFINITY;
    for (int a = 0; a < 3; ++a) {
        if (d[a] != 0.0) {
            double ta = (lo[a] - s[a]) / d[a];
            double tb = (hi[a] - s[a]) / d[a];
            if (tb < ta) { double tmp = ta; ta = tb; tb = tmp; }
            if (ta > tlo) tlo = ta;
            if (tb < thi) thi = tb;
        } else if (s[a] < lo[a] || s[a] > hi[a]) {
            return 0;
        }
    }
    *t0 = tlo;
    *t1 = thi;
    return 1;
}

/* _ckern.pyx:217-248 (+ rays.py:99-124 for eps / step_scale).
 * out_t[i] = hit distance or +inf.  Optional: out_cell (3 per ray, -1 on
 * miss), out_steps (interp calls per ray). */
void orc_grid_trace(const double *values, int64_t nx, int64_t ny, int64_t nz,
                    double ox, double oy, double oz, double res,
                    double sx, double sy, double sz,
                    const double *dirs, int64_t s, int64_t e,
                    double max_range, double eps, double step_scale,
                    double *out_t, int32_t *out_cell, int32_t *out_steps)
{
    orc_grid g = {values, nx, ny, nz, ox, oy, oz, res};
    const double lo[3] = {ox, oy, oz};
    const double hi[3] = {ox + (double)(nx - 1) * res, oy + (double)(ny - 1) * res,
                          oz + (double)(nz - 1) * res};
    const double st[3] = {sx, sy, sz};
    for (int64_t i = s; i < e; ++i) {
        const double *d = dirs + 3 * i;
        double t0, t1, t, t_end;
        int32_t steps = 0;
        int64_t cx = -1, cy = -1, cz = -1;
        out_t[i] = INFINITY;
        int hit = 0;
        if (orc_box_span(st, d, lo, hi, &t0, &t1)) {
            t = t0 > 0.0 ? t0 : 0.0;
            t_end = t1 < max_range ? t1 : max_range;
            if (!(t > t_end)) {
                for (;;) {
                    double dist = orc_interp(&g, sx + t * d[0], sy + t * d[1], sz + t * d[2],
                                             &cx, &cy, &cz);
                    ++steps;
                    if (dist < eps) { out_t[i] = t; hit = 1; break; }
                    t += step_scale * dist;
                    if (t > t_end) break;
                }
            }
        }
        if (out_cell) {
            out_cell[3 * i + 0] = hit ? (int32_t)cx : -1;
            out_cell[3 * i + 1] = hit ? (int32_t)cy : -1;
            out_cell[3 * i + 2] = hit ? (int32_t)cz : -1;
        }
        if (out_steps) out_steps[i] = steps;
    }
}

/* _ckern.pyx:278-321 -- sequential accumulation over [s, e) into one slot:
 * [A (9, symmetric duplicated), Af (3), count]. */
void orc_policy_reduce_chunk(const double *dirs, const double *dists, int64_t s, int64_t e,
                             const double v[3], const double p[7], double min_range,
                             double slot[13])
{
    const double eta_rep = p[0], nu_rep = p[1], eta_damp = p[2], nu_damp = p[3];
    const double eps_p = p[4], radius = p[5], c = p[6];
    double a00 = 0, a01 = 0, a02 = 0, a11 = 0, a12 = 0, a22 = 0;
    double b0 = 0, b1 = 0, b2 = 0, cnt = 0;
    for (int64_t i = s; i < e; ++i) {
        double d = dists[i];
        if (d != d || d == INFINITY || d < min_range) continue;
        cnt += 1;
        const double *q = dirs + 3 * i;
        double rx = -q[0], ry = -q[1], rz = -q[2];
        double toward = q[0] * v[0] + q[1] * v[1] + q[2] * v[2];
        double frep = eta_rep * exp(-d / nu_rep);
        double g = toward > 0.0 ? toward : 0.0;
        double fdamp = eta_damp / (d / nu_damp + eps_p) * g * g;
        double w = d < radius ? d * d / (radius * radius) - 2.0 * d / radius + 1.0 : 0.0;
        double smag = fdamp / (fdamp + c * log1p(exp(-2.0 * c * fdamp)));
        double a = w * smag * smag;
        if (a != 0.0) {
            a00 += a * rx * rx; a01 += a * rx * ry; a02 += a * rx * rz;
            a11 += a * ry * ry; a12 += a * ry * rz; a22 += a * rz * rz;
            double bf = a * (frep + fdamp);
            b0 += bf * rx; b1 += bf * ry; b2 += bf * rz;
        }
    }
    slot[0] = a00; slot[1] = a01; slot[2] = a02;
    slot[3] = a01; slot[4] = a11; slot[5] = a12;
    slot[6] = a02; slot[7] = a12; slot[8] = a22;
    slot[9] = b0; slot[10] = b1; slot[11] = b2;
    slot[12] = cnt;
}

/* _pool.py:61-72 -- fixed-shape pairwise fold along axis 0 (in place). */
void orc_pairwise_fold(double *slots, int64_t n, int64_t width, double *out)
{
    while (n > 1) {
        int64_t half = n / 2;
        for (int64_t k = 0; k < half; ++k)
            for (int64_t j = 0; j < width; ++j)
                slots[k * width + j] = slots[2 * k * width + j] + slots[(2 * k + 1) * width + j];
        if (n % 2)
            memmove(slots + half * width, slots + (n - 1) * width, (size_t)width * sizeof(double));
        n = half + (n % 2);
    }
    memcpy(out, slots, (size_t)width * sizeof(double));
}

/* ckern.py:80-93 + _pool.py -- whole reduction: 2048-ray chunks, then fold.
 * `scratch` must hold ceil(n/2048) * 13 doubles (at least 13). */
void orc_policy_reduce(const double *dirs, const double *dists, int64_t n,
                       const double v[3], const double p[7], double min_range,
                       double *scratch, double out[13])
{
    int64_t spans = n > 0 ? (n + ORC_CHUNK - 1) / ORC_CHUNK : 1;
    memset(scratch, 0, (size_t)spans * 13 * sizeof(double));
    for (int64_t k = 0; k * ORC_CHUNK < n; ++k) {
        int64_t s = k * ORC_CHUNK, e = s + ORC_CHUNK < n ? s + ORC_CHUNK : n;
        orc_policy_reduce_chunk(dirs, dists, s, e, v, p, min_range, scratch + 13 * k);
    }
    orc_pairwise_fold(scratch, spans, 13, out);
}

/* _ckern.pyx:21-56 -- ordered union / subtract of moving spheres and boxes. */
double orc_scene_sd(const int8_t *kinds, const int8_t *ops, const double *centers,
                    const double *sizes, const double *vels, int64_t n, double empty,
                    double t, double px, double py, double pz)
{
    double d = empty;
    for (int64_t i = 0; i < n; ++i) {
        double dx = px - (centers[3 * i + 0] + vels[3 * i + 0] * t);
        double dy = py - (centers[3 * i + 1] + vels[3 * i + 1] * t);
        double dz = pz - (centers[3 * i + 2] + vels[3 * i + 2] * t);
        double dp;
        if (kinds[i] == 0) {
            dp = sqrt(dx * dx + dy * dy + dz * dz) - sizes[3 * i];
        } else {
            double qx = fabs(dx) - sizes[3 * i + 0];
            double qy = fabs(dy) - sizes[3 * i + 1];
            double qz = fabs(dz) - sizes[3 * i + 2];
            double mx = qx;
            if (qy > mx) mx = qy;
            if (qz > mx) mx = qz;
            double ex = qx > 0.0 ? qx : 0.0, ey = qy > 0.0 ? qy : 0.0, ez = qz > 0.0 ? qz : 0.0;
            dp = sqrt(ex * ex + ey * ey + ez * ez) + (mx < 0.0 ? mx : 0.0);
        }
        if (ops[i] == 0) { if (dp < d) d = dp; }
        else { if (-dp > d) d = -dp; }
    }
    return d;
}

void orc_scene_distance(const int8_t *kinds, const int8_t *ops, const double *centers,
                        const double *sizes, const double *vels, int64_t n, double empty,
                        double t, const double *pts, int64_t s, int64_t e, double *out)
{
    for (int64_t i = s; i < e; ++i)
        out[i] = orc_scene_sd(kinds, ops, centers, sizes, vels, n, empty, t,
                              pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
}

/* _ckern.pyx:71-87 -- node (ix,iy,iz) at origin + res * index, x-slabs [s, e). */
void orc_bake(const int8_t *kinds, const int8_t *ops, const double *centers,
              const double *sizes, const double *vels, int64_t n, double empty,
              double ox, double oy, double oz, double res,
              int64_t nx, int64_t ny, int64_t nz, int64_t s, int64_t e, double *out)
{
    (void)nx;
    for (int64_t ix = s; ix < e; ++ix) {
        double px = ox + res * (double)ix;
        for (int64_t iy = 0; iy < ny; ++iy) {
            double py = oy + res * (double)iy;
            for (int64_t iz = 0; iz < nz; ++iz) {
                double pz = oz + res * (double)iz;
                out[(ix * ny + iy) * nz + iz] =
                    orc_scene_sd(kinds, ops, centers, sizes, vels, n, empty, 0.0, px, py, pz);
            }
        }
    }
}

/* _ckern.pyx:251-273 -- analytic sphere trace from t = 0 (no box clip). */
void orc_scene_trace(const int8_t *kinds, const int8_t *ops, const double *centers,
                     const double *sizes, const double *vels, int64_t n, double empty,
                     double tm, double sx, double sy, double sz, const double *dirs,
                     int64_t s, int64_t e, double max_range, double eps, double step_scale,
                     double *out)
{
    for (int64_t i = s; i < e; ++i) {
        const double *d = dirs + 3 * i;
        double t = 0.0;
        out[i] = INFINITY;
        for (;;) {
            double dist = orc_scene_sd(kinds, ops, centers, sizes, vels, n, empty, tm,
                                       sx + t * d[0], sy + t * d[1], sz + t * d[2]);
            if (dist < eps) { out[i] = t; break; }
            t += step_scale * dist;
            if (t > max_range) break;
        }
    }
}

/* _ckern.pyx:138-166 -- distance + normalised central-difference gradient. */
void orc_esdf_sample(const double *values, int64_t nx, int64_t ny, int64_t nz,
                     double ox, double oy, double oz, double res,
                     const double *pts, int64_t s, int64_t e,
                     double *out_d, double *out_g, uint8_t *out_flag)
{
    orc_grid g = {values, nx, ny, nz, ox, oy, oz, res};
    for (int64_t i = s; i < e; ++i) {
        double px = pts[3 * i], py = pts[3 * i + 1], pz = pts[3 * i + 2];
        double ux = (px - ox) / res, uy = (py - oy) / res, uz = (pz - oz) / res;
        out_flag[i] = (ux < 0.0 || ux > (double)nx - 1.0 || uy < 0.0 || uy > (double)ny - 1.0 ||
                       uz < 0.0 || uz > (double)nz - 1.0);
        out_d[i] = orc_interp(&g, px, py, pz, 0, 0, 0);
        double gx = (orc_interp(&g, px + res, py, pz, 0, 0, 0) -
                     orc_interp(&g, px - res, py, pz, 0, 0, 0)) / (2.0 * res);
        double gy = (orc_interp(&g, px, py + res, pz, 0, 0, 0) -
                     orc_interp(&g, px, py - res, pz, 0, 0, 0)) / (2.0 * res);
        double gz = (orc_interp(&g, px, py, pz + res, 0, 0, 0) -
                     orc_interp(&g, px, py, pz - res, 0, 0, 0)) / (2.0 * res);
        double nrm = sqrt(gx * gx + gy * gy + gz * gz);
        if (nrm < 1e-9) {
            out_g[3 * i] = 0.0; out_g[3 * i + 1] = 0.0; out_g[3 * i + 2] = 0.0;
        } else {
            out_g[3 * i] = gx / nrm; out_g[3 * i + 1] = gy / nrm; out_g[3 * i + 2] = gz / nrm;
        }
    }
}

/* ------------------------------------------------------------------------
 * K5 (north_star "per-ray 3D DDA (Amanatides-Woo) through the occupancy
 * grid"): NOT a reference function -- the reference sphere-traces
 * (SPEC.md:228).  This is the CPU definition the CUDA DDA is checked
 * against bit-for-bit; see DESIGN.md §K5.  Occupancy = node value <= 0
 * (rmpnav/geometry.py:312-315); the voxel of node (i,j,k) is the res-cube
 * centred on it.  All arithmetic is float32, no contraction, IEEE division,
 * so CPU and GPU agree bitwise.  Outputs: entry distance t of the first
 * occupied voxel (+inf = miss), its index, and the voxels visited.
 */
static int orc_occ(const uint32_t *bits, int64_t ny, int64_t nzw, int64_t i, int64_t j, int64_t k)
{
    return (bits[(i * ny + j) * nzw + (k >> 5)] >> (k & 31)) & 1u;
}

void orc_occupancy_bits(const double *values, int64_t nx, int64_t ny, int64_t nz, uint32_t *bits)
{
    int64_t nzw = (nz + 31) / 32;
    memset(bits, 0, (size_t)(nx * ny * nzw) * sizeof(uint32_t));
    for (int64_t i = 0; i < nx; ++i)
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t k = 0; k < nz; ++k)
                if (values[(i * ny + j) * nz + k] <= 0.0)
                    bits[(i * ny + j) * nzw + (k >> 5)] |= 1u << (k & 31);
}

void orc_dda_trace(const uint32_t *bits, int64_t nx, int64_t ny, int64_t nz,
                   double ox, double oy, double oz, double res,
                   double sx, double sy, double sz, const double *dirs, int64_t s, int64_t e,
                   double max_range, float *out_t, int32_t *out_vox, int32_t *out_steps)
{
    const int64_t nzw = (nz + 31) / 32;
    const int n[3] = {(int)nx, (int)ny, (int)nz};
    const float inv = 1.0f / (float)res;
    const float o[3] = {(float)ox, (float)oy, (float)oz};
    const float st[3] = {(float)sx, (float)sy, (float)sz};
    const float tr = (float)max_range;
    for (int64_t r = s; r < e; ++r) {
        float u[3], dv[3];
        for (int a = 0; a < 3; ++a) {
            float p = st[a] - o[a];
            p = p * inv;
            u[a] = p + 0.5f;
            float d = (float)dirs[3 * r + a];
            dv[a] = d * inv;
        }
        float t0 = 0.0f, t1 = tr;
        int ok = 1;
        for (int a = 0; a < 3 && ok; ++a) {
            if (dv[a] != 0.0f) {
                float ta = (0.0f - u[a]) / dv[a];
                float tb = ((float)n[a] - u[a]) / dv[a];
                if (tb < ta) { float tmp = ta; ta = tb; tb = tmp; }
                if (ta > t0) t0 = ta;
                if (tb < t1) t1 = tb;
            } else if (u[a] < 0.0f || u[a] >= (float)n[a]) {
                ok = 0;
            }
        }
        out_t[r] = INFINITY;
        out_vox[3 * r] = out_vox[3 * r + 1] = out_vox[3 * r + 2] = -1;
        int steps = 0;
        if (ok && !(t0 > t1)) {
            int vox[3], stp[3];
            float tmax[3], tdel[3];
            for (int a = 0; a < 3; ++a) {
                float pa = dv[a] * t0;
                pa = u[a] + pa;
                int ia = (int)floorf(pa);
                if (ia < 0) ia = 0;
                if (ia > n[a] - 1) ia = n[a] - 1;
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
                    tmax[a] = INFINITY;
                    tdel[a] = INFINITY;
                }
            }
            float t = t0;
            for (;;) {
                ++steps;
                if (orc_occ(bits, ny, nzw, vox[0], vox[1], vox[2])) {
                    out_t[r] = t;
                    out_vox[3 * r] = vox[0]; out_vox[3 * r + 1] = vox[1]; out_vox[3 * r + 2] = vox[2];
                    break;
                }
                int a = 0;
                if (tmax[1] < tmax[a]) a = 1;
                if (tmax[2] < tmax[a]) a = 2;
                t = tmax[a];
                if (!(t <= t1)) break;
                vox[a] += stp[a];
                if (vox[a] < 0 || vox[a] >= n[a]) break;
                tmax[a] = tmax[a] + tdel[a];
            }
        }
        if (out_steps) out_steps[r] = steps;
    }
}
