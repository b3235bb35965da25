/*
 * pic_oracle.c -- CPU ORACLE for the PIC macro-particle hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library,
 * and only as the checker (or the timed CPU baseline), never as the product.
 *
 * A plain-C restatement of the reference "taskpic" (/root/reference/pkg/src/
 * taskpic).  Every arithmetic expression keeps the reference's association
 * order and the file is compiled with -ffp-contract=off (numba emits no FMA,
 * SURVEY.md §0/App. A), so 2D results are bit-identical to the reference:
 *   - gather_fields      kernels.py:51-121
 *   - boris_push         kernels.py:124-162
 *   - flag_boundaries    kernels.py:165-178
 *   - esirkepov_project  kernels.py:181-266
 *   - deposit_rho        kernels.py:269-298
 *   - reduce_bin_currents fields.py:101-114 (rint of each (patch,species,bin)
 *     subgrid at quantum 2^-44, integer-added)
 *   - ghost fold / pull  exchange.py:23-156 (expressed on one whole-domain
 *     array with 3 ghost layers: an integer fold commutes, and a pulled ghost
 *     equals sign x owner value, so the global form is exactly equivalent)
 *   - maxwell            fields.py:130-190 with ghosts refreshed between the
 *     sub-steps ("reference + synced-Yee harness fix")
 *   - BC + migration + canonical (bin, id) re-sort
 *                        exchange.py:163-258, arena.py:59-95
 * Parity pin: the tests/golden npz fixtures produced by running the reference itself
 * (tests/golden/make_golden.py).  The 3D functions (suffix _3d) are the
 * builder's generalisation of the same formulas; the reference is 2D-only,
 * so 3D parity is pinned by invariants only.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define G 3
#define J_SCALE 17592186044416.0 /* 2^44, fields.py:28-30 */
#define INV_J_SCALE (1.0 / J_SCALE)

enum { FLAG_X_NEG = 1, FLAG_X_POS = 2, FLAG_Y_NEG = 4, FLAG_Y_POS = 8, FLAG_Z_NEG = 16, FLAG_Z_POS = 32 };

/* error codes shared with the device library (include/b200pic.h) */
enum { OK = 0, ERR_NONFINITE = 1, ERR_COURANT = 2, ERR_INVARIANT = 3, ERR_ARG = 4, ERR_CAPACITY = 5 };

typedef struct {
    int32_t dim;   /* 2 or 3 */
    int32_t L[3];  /* cells per axis */
    int32_t pn[3]; /* patch extent in cells */
    int32_t np[3]; /* patches per axis */
    int32_t bx;    /* bin_x_size */
    int32_t bc[3]; /* 0 periodic, 1 reflective */
    double d[3];
    double dt;
} o_cfg;

/* staggering (dual flags) per component, fields.py:33-44 (2D) and the 3D Yee cell */
enum { C_EX, C_EY, C_EZ, C_BX, C_BY, C_BZ, C_JX, C_JY, C_JZ, C_RHO };
static const int DUAL[10][3] = {
    {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, /* ex ey ez */
    {0, 1, 1}, {1, 0, 1}, {1, 1, 0}, /* bx by bz */
    {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, /* jx jy jz */
    {0, 0, 0}};                      /* rho */

static inline int dual_of(const o_cfg *c, int comp, int axis) {
    /* in 2D the z staggering collapses: ez/jz primal, bx/by dual only in-plane (fields.py:33-44) */
    if (c->dim == 2 && axis == 2) return 0;
    return DUAL[comp][axis];
}

static inline int64_t ext_of(const o_cfg *c, int a) { return a < c->dim ? (int64_t)c->L[a] + 1 + 2 * G : 1; }
static inline int64_t gidx(const o_cfg *c, int64_t i, int64_t j, int64_t k) {
    return (i * ext_of(c, 1) + j) * ext_of(c, 2) + k;
}

/* exchange.py:23-61 mapping of a global node to its owner node (and sign) */
static inline int64_t wrap_node(int64_t node, int64_t L, int periodic, int dual, int *sign) {
    *sign = 1;
    if (periodic) return ((node % L) + L) % L;
    if (dual) {
        if (node < 0) return -node - 1;
        if (node >= L) return 2 * L - node - 1;
        return node;
    }
    if (node < 0) { *sign = -1; return -node; }
    if (node > L) { *sign = -1; return 2 * L - node; }
    return node;
}

/* owned index range [G, hi) of a component along an axis (fields.py:117-127); walls own node L */
static inline int64_t owned_hi(const o_cfg *c, int comp, int a) {
    if (a >= c->dim) return 1;
    int64_t hi = G + c->L[a];
    if (c->bc[a] != 0 && !dual_of(c, comp, a)) hi += 1;
    return hi;
}

/* bc 2 (absorbing, beyond the reference): fold drops ghost currents (-1), pull copies the nearest owned node */
static inline int64_t ghost_owner(int64_t node, int64_t L, int bc, int dual, int fold, int *sign) {
    if (bc != 2) return wrap_node(node, L, bc == 0, dual, sign);
    *sign = 1;
    if (fold) {
        int64_t hi = dual ? L - 1 : L;
        return (node < 0 || node > hi) ? -1 : node;
    }
    int64_t hi = dual ? L - 1 : L;
    return node < 0 ? 0 : (node > hi ? hi : node);
}

static inline double sq(double t) { return t * t; }
/* order-2 spline weights, kernels.py:40-48 / 76-87 */
static inline void spl(double d, double w[3]) {
    w[0] = 0.5 * sq(0.5 - d);
    w[1] = 0.75 - d * d;
    w[2] = 0.5 * sq(0.5 + d);
}

/* ===================================================================== */
/* 2D kernels (exact restatement)                                        */
/* ===================================================================== */

static inline double interp2(const double *f, int64_t e1, int64_t a, int64_t b, const double wx[3], const double wy[3]) {
    const double *r0 = f + (a - 1) * e1 + b, *r1 = f + a * e1 + b, *r2 = f + (a + 1) * e1 + b;
    return wx[0] * (wy[0] * r0[-1] + wy[1] * r0[0] + wy[2] * r0[1]) +
           wx[1] * (wy[0] * r1[-1] + wy[1] * r1[0] + wy[2] * r1[1]) +
           wx[2] * (wy[0] * r2[-1] + wy[1] * r2[0] + wy[2] * r2[1]);
}

/* kernels.py:51-121; field arrays have row length e1 (C order, x slow) */
void o_gather_2d(int64_t n, const double *x, const double *y, const double *const f[6], int64_t e1,
                 int64_t *cix, int64_t *ciy, double *dlx, double *dly, double *const out[6],
                 double inv_dx, double inv_dy, int64_t cell0x, int64_t cell0y) {
    for (int64_t p = 0; p < n; ++p) {
        double xn = x[p] * inv_dx, yn = y[p] * inv_dy;
        int64_t ip = (int64_t)(xn + 0.5), jp = (int64_t)(yn + 0.5);
        double dxp = xn - ip, dyp = yn - jp;
        int64_t idu = (int64_t)xn, jdu = (int64_t)yn;
        double dxd = xn - 0.5 - idu, dyd = yn - 0.5 - jdu;
        cix[p] = ip; ciy[p] = jp; dlx[p] = dxp; dly[p] = dyp;
        double wxp[3], wyp[3], wxd[3], wyd[3];
        spl(dxp, wxp); spl(dyp, wyp); spl(dxd, wxd); spl(dyd, wyd);
        int64_t ap = ip - cell0x + G, bp = jp - cell0y + G, ad = idu - cell0x + G, bd = jdu - cell0y + G;
        out[0][p] = interp2(f[0], e1, ad, bp, wxd, wyp);
        out[1][p] = interp2(f[1], e1, ap, bd, wxp, wyd);
        out[2][p] = interp2(f[2], e1, ap, bp, wxp, wyp);
        out[3][p] = interp2(f[3], e1, ap, bd, wxp, wyd);
        out[4][p] = interp2(f[4], e1, ad, bp, wxd, wyp);
        out[5][p] = interp2(f[5], e1, ad, bd, wxd, wyd);
    }
}

/* kernels.py:124-162; z may be NULL (2D3V: z untracked).  Returns first bad index or -1. */
int64_t o_push(int64_t n, double *x, double *y, double *z, double *px, double *py, double *pz,
               const double *const e[6], double charge, double mass, double dt) {
    double qd2 = charge * dt * 0.5;
    double inv_m2 = 1.0 / (mass * mass);
    int64_t bad = -1;
    for (int64_t p = 0; p < n; ++p) {
        double ex = e[0][p], ey = e[1][p], ez = e[2][p];
        double pxm = px[p] + qd2 * ex, pym = py[p] + qd2 * ey, pzm = pz[p] + qd2 * ez;
        double gm = sqrt(1.0 + (pxm * pxm + pym * pym + pzm * pzm) * inv_m2);
        double tf = qd2 / (gm * mass);
        double tx = tf * e[3][p], ty = tf * e[4][p], tz = tf * e[5][p];
        double sf = 2.0 / (1.0 + tx * tx + ty * ty + tz * tz);
        double sx = tx * sf, sy = ty * sf, sz = tz * sf;
        double ppx = pxm + (pym * tz - pzm * ty);
        double ppy = pym + (pzm * tx - pxm * tz);
        double ppz = pzm + (pxm * ty - pym * tx);
        double pxn = pxm + (ppy * sz - ppz * sy) + qd2 * ex;
        double pyn = pym + (ppz * sx - ppx * sz) + qd2 * ey;
        double pzn = pzm + (ppx * sy - ppy * sx) + qd2 * ez;
        double gn = sqrt(1.0 + (pxn * pxn + pyn * pyn + pzn * pzn) * inv_m2);
        px[p] = pxn; py[p] = pyn; pz[p] = pzn;
        double adv = dt / (gn * mass);
        x[p] += pxn * adv;
        y[p] += pyn * adv;
        if (z) z[p] += pzn * adv;
        if (bad < 0 && !(isfinite(pxn) && isfinite(pyn) && isfinite(pzn))) bad = p;
    }
    return bad;
}

/* kernels.py:165-178 (+ z bits in 3D); bounds = xmin,xmax,ymin,ymax[,zmin,zmax] */
void o_flag(int64_t n, const double *x, const double *y, const double *z, uint8_t *flags, const double *bd) {
    for (int64_t p = 0; p < n; ++p) {
        int f = 0;
        if (x[p] < bd[0]) f |= FLAG_X_NEG; else if (x[p] >= bd[1]) f |= FLAG_X_POS;
        if (y[p] < bd[2]) f |= FLAG_Y_NEG; else if (y[p] >= bd[3]) f |= FLAG_Y_POS;
        if (z) { if (z[p] < bd[4]) f |= FLAG_Z_NEG; else if (z[p] >= bd[5]) f |= FLAG_Z_POS; }
        flags[p] = (uint8_t)f;
    }
}

/* kernels.py:181-266; subgrid arrays with row length e1.  Returns first Courant violator or -1. */
int64_t o_project_2d(int64_t n, const double *x, const double *y, const double *px, const double *py,
                     const double *pz, const double *w, const int64_t *cix, const int64_t *ciy,
                     const double *dlx, const double *dly, double *jx, double *jy, double *jz, int64_t e1,
                     double charge, double mass, double inv_dx, double inv_dy, double dx_over_dt,
                     double dy_over_dt, int64_t sub_cell0x, int64_t sub_cell0y) {
    const double inv_m2 = 1.0 / (mass * mass), third = 1.0 / 3.0, sixth = 1.0 / 6.0;
    for (int64_t p = 0; p < n; ++p) {
        int64_t i0 = cix[p], j0 = ciy[p];
        double xn = x[p] * inv_dx, yn = y[p] * inv_dy;
        int64_t i1 = (int64_t)(xn + 0.5), j1 = (int64_t)(yn + 0.5);
        int64_t shx = i1 - i0, shy = j1 - j0;
        if (shx < -1 || shx > 1 || shy < -1 || shy > 1) return p;
        double d0x = dlx[p], d0y = dly[p], d1x = xn - i1, d1y = yn - j1;
        double s0x[5] = {0}, s1x[5] = {0}, s0y[5] = {0}, s1y[5] = {0};
        spl(d0x, s0x + 1); spl(d0y, s0y + 1); spl(d1x, s1x + 1 + shx); spl(d1y, s1y + 1 + shy);
        double qw = charge * w[p];
        double gam = sqrt(1.0 + (px[p] * px[p] + py[p] * py[p] + pz[p] * pz[p]) * inv_m2);
        double fx = qw * dx_over_dt, fy = qw * dy_over_dt, fz = qw * pz[p] / (gam * mass);
        int64_t bi = i0 - 2 - sub_cell0x + G, bj = j0 - 2 - sub_cell0y + G;
        if (fz != 0.0) {
            for (int ky = 0; ky < 5; ++ky) {
                double sy0 = s0y[ky], sy1 = s1y[ky];
                double cyx = 0.5 * (sy0 + sy1);
                double za = fz * (sy0 * third + sy1 * sixth), zb = fz * (sy0 * sixth + sy1 * third);
                double acc = 0.0;
                for (int kx = 0; kx < 4; ++kx) {
                    acc -= fx * (s1x[kx] - s0x[kx]) * cyx;
                    jx[(bi + kx) * e1 + bj + ky] += acc;
                    jz[(bi + kx) * e1 + bj + ky] += s0x[kx] * za + s1x[kx] * zb;
                }
                jz[(bi + 4) * e1 + bj + ky] += s0x[4] * za + s1x[4] * zb;
            }
        } else {
            for (int ky = 0; ky < 5; ++ky) {
                double cyx = 0.5 * (s0y[ky] + s1y[ky]);
                double acc = 0.0;
                for (int kx = 0; kx < 4; ++kx) {
                    acc -= fx * (s1x[kx] - s0x[kx]) * cyx;
                    jx[(bi + kx) * e1 + bj + ky] += acc;
                }
            }
        }
        for (int kx = 0; kx < 5; ++kx) {
            double cxy = 0.5 * (s0x[kx] + s1x[kx]);
            double acc = 0.0;
            for (int ky = 0; ky < 4; ++ky) {
                acc -= fy * (s1y[ky] - s0y[ky]) * cxy;
                jy[(bi + kx) * e1 + bj + ky] += acc;
            }
        }
    }
    return -1;
}

/* kernels.py:269-298 */
void o_deposit_rho_2d(int64_t n, const double *x, const double *y, const double *w, double *rho, int64_t e1,
                      double charge, double inv_dx, double inv_dy, int64_t cell0x, int64_t cell0y) {
    for (int64_t p = 0; p < n; ++p) {
        double xn = x[p] * inv_dx, yn = y[p] * inv_dy;
        int64_t ip = (int64_t)(xn + 0.5), jp = (int64_t)(yn + 0.5);
        double wx[3], wy[3];
        spl(xn - ip, wx); spl(yn - jp, wy);
        double qw = charge * w[p];
        int64_t a = ip - cell0x + G, b = jp - cell0y + G;
        for (int u = 0; u < 3; ++u)
            for (int v = 0; v < 3; ++v) rho[(a - 1 + u) * e1 + (b - 1 + v)] += qw * wx[u] * wy[v];
    }
}

/* ===================================================================== */
/* 3D kernels (builder's generalisation of the 2D formulas)              */
/* ===================================================================== */

static inline double interp3(const double *f, int64_t e1, int64_t e2, int64_t a, int64_t b, int64_t c,
                             const double wx[3], const double wy[3], const double wz[3]) {
    double sx = 0.0;
    for (int u = 0; u < 3; ++u) {
        double sy = 0.0;
        for (int v = 0; v < 3; ++v) {
            const double *r = f + ((a - 1 + u) * e1 + (b - 1 + v)) * e2 + (c - 1);
            double sz = wz[0] * r[0] + wz[1] * r[1] + wz[2] * r[2];
            sy = (v == 0) ? wy[0] * sz : sy + wy[v] * sz;
        }
        sx = (u == 0) ? wx[0] * sy : sx + wx[u] * sy;
    }
    return sx;
}

void o_gather_3d(int64_t n, const double *x, const double *y, const double *z, const double *const f[6],
                 int64_t e1, int64_t e2, int64_t *ci, double *dl, double *const out[6], double inv_dx,
                 double inv_dy, double inv_dz, int64_t cell0x, int64_t cell0y, int64_t cell0z) {
    /* ci/dl: [3*n] interleaved per particle (i,j,k) */
    for (int64_t p = 0; p < n; ++p) {
        double xn = x[p] * inv_dx, yn = y[p] * inv_dy, zn = z[p] * inv_dz;
        int64_t ip = (int64_t)(xn + 0.5), jp = (int64_t)(yn + 0.5), kp = (int64_t)(zn + 0.5);
        int64_t idu = (int64_t)xn, jdu = (int64_t)yn, kdu = (int64_t)zn;
        double dxp = xn - ip, dyp = yn - jp, dzp = zn - kp;
        double dxd = xn - 0.5 - idu, dyd = yn - 0.5 - jdu, dzd = zn - 0.5 - kdu;
        ci[3 * p] = ip; ci[3 * p + 1] = jp; ci[3 * p + 2] = kp;
        dl[3 * p] = dxp; dl[3 * p + 1] = dyp; dl[3 * p + 2] = dzp;
        double wxp[3], wyp[3], wzp[3], wxd[3], wyd[3], wzd[3];
        spl(dxp, wxp); spl(dyp, wyp); spl(dzp, wzp); spl(dxd, wxd); spl(dyd, wyd); spl(dzd, wzd);
        int64_t ap = ip - cell0x + G, bp = jp - cell0y + G, cp = kp - cell0z + G;
        int64_t ad = idu - cell0x + G, bd = jdu - cell0y + G, cd = kdu - cell0z + G;
        out[0][p] = interp3(f[0], e1, e2, ad, bp, cp, wxd, wyp, wzp); /* ex: dual x */
        out[1][p] = interp3(f[1], e1, e2, ap, bd, cp, wxp, wyd, wzp); /* ey: dual y */
        out[2][p] = interp3(f[2], e1, e2, ap, bp, cd, wxp, wyp, wzd); /* ez: dual z */
        out[3][p] = interp3(f[3], e1, e2, ap, bd, cd, wxp, wyd, wzd); /* bx: dual y,z */
        out[4][p] = interp3(f[4], e1, e2, ad, bp, cd, wxd, wyp, wzd); /* by: dual x,z */
        out[5][p] = interp3(f[5], e1, e2, ad, bd, cp, wxd, wyd, wzp); /* bz: dual x,y */
    }
}

/* 3D Esirkepov, order 2 (builder's restatement; the reference is 2D-only).
 * W_x(u,v,q) = P_x[u] * wyz(v,q), P_x[u] = -q w dx/dt * cumsum(S1x - S0x)[u] (the prefix form of the
 * 2D jx loop, kernels.py:244-250) and wyz = S0y(S0z/3 + S1z/6) + S1y(S0z/6 + S1z/3) (the time-averaged
 * transverse weight, the 3D form of kernels.py:244-246); cyclic for y and z. */
int64_t o_project_3d(int64_t n, const double *x, const double *y, const double *z, const double *px,
                     const double *py, const double *pz, const double *w, const int64_t *ci, const double *dl,
                     double *jx, double *jy, double *jz, int64_t e1, int64_t e2, double charge, double mass,
                     double inv_dx, double inv_dy, double inv_dz, double dx_over_dt, double dy_over_dt,
                     double dz_over_dt, int64_t sub_cell0x, int64_t sub_cell0y, int64_t sub_cell0z) {
    const double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
    (void)px; (void)py; (void)pz; (void)mass;
    for (int64_t p = 0; p < n; ++p) {
        double xn[3] = {x[p] * inv_dx, y[p] * inv_dy, z[p] * inv_dz};
        double s0[3][5], s1[3][5], P[3][4];
        int64_t i0[3];
        double qw = charge * w[p];
        double f[3] = {qw * dx_over_dt, qw * dy_over_dt, qw * dz_over_dt};
        for (int a = 0; a < 3; ++a) {
            i0[a] = ci[3 * p + a];
            int64_t i1 = (int64_t)(xn[a] + 0.5);
            int64_t sh = i1 - i0[a];
            if (sh < -1 || sh > 1) return p;
            for (int k = 0; k < 5; ++k) { s0[a][k] = 0.0; s1[a][k] = 0.0; }
            spl(dl[3 * p + a], s0[a] + 1);
            spl(xn[a] - i1, s1[a] + 1 + sh);
            double pref = 0.0;
            for (int u = 0; u < 4; ++u) { pref -= f[a] * (s1[a][u] - s0[a][u]); P[a][u] = pref; }
        }
        int64_t bi = i0[0] - 2 - sub_cell0x + G, bj = i0[1] - 2 - sub_cell0y + G, bk = i0[2] - 2 - sub_cell0z + G;
#define JIDX(u, v, q) (((bi + (u)) * e1 + (bj + (v))) * e2 + (bk + (q)))
        for (int v = 0; v < 5; ++v)
            for (int q = 0; q < 5; ++q) {
                double wyz = s0[1][v] * (s0[2][q] * third + s1[2][q] * sixth) + s1[1][v] * (s0[2][q] * sixth + s1[2][q] * third);
                for (int u = 0; u < 4; ++u) jx[JIDX(u, v, q)] += P[0][u] * wyz;
            }
        for (int u = 0; u < 5; ++u)
            for (int q = 0; q < 5; ++q) {
                double wxz = s0[0][u] * (s0[2][q] * third + s1[2][q] * sixth) + s1[0][u] * (s0[2][q] * sixth + s1[2][q] * third);
                for (int v = 0; v < 4; ++v) jy[JIDX(u, v, q)] += P[1][v] * wxz;
            }
        for (int u = 0; u < 5; ++u)
            for (int v = 0; v < 5; ++v) {
                double wxy = s0[0][u] * (s0[1][v] * third + s1[1][v] * sixth) + s1[0][u] * (s0[1][v] * sixth + s1[1][v] * third);
                for (int q = 0; q < 4; ++q) jz[JIDX(u, v, q)] += P[2][q] * wxy;
            }
#undef JIDX
    }
    return -1;
}

void o_deposit_rho_3d(int64_t n, const double *x, const double *y, const double *z, const double *w, double *rho,
                      int64_t e1, int64_t e2, double charge, double inv_dx, double inv_dy, double inv_dz,
                      int64_t cell0x, int64_t cell0y, int64_t cell0z) {
    for (int64_t p = 0; p < n; ++p) {
        double xn = x[p] * inv_dx, yn = y[p] * inv_dy, zn = z[p] * inv_dz;
        int64_t ip = (int64_t)(xn + 0.5), jp = (int64_t)(yn + 0.5), kp = (int64_t)(zn + 0.5);
        double wx[3], wy[3], wz[3];
        spl(xn - ip, wx); spl(yn - jp, wy); spl(zn - kp, wz);
        double qw = charge * w[p];
        int64_t a = ip - cell0x + G, b = jp - cell0y + G, c = kp - cell0z + G;
        for (int u = 0; u < 3; ++u)
            for (int v = 0; v < 3; ++v)
                for (int q = 0; q < 3; ++q)
                    rho[((a - 1 + u) * e1 + (b - 1 + v)) * e2 + (c - 1 + q)] += qw * wx[u] * wy[v] * wz[q];
    }
}

/* ===================================================================== */
/* Step-level oracle on whole-domain arrays                              */
/* ===================================================================== */

typedef struct {
    double *x, *y, *z, *px, *py, *pz, *w;
    int64_t *id;
    int64_t n;
    int64_t *offsets; /* [n_patches * n_bins + 1], canonical (patch, bin, id) order */
    double charge, mass;
} o_species;

static inline int64_t n_patches(const o_cfg *c) { return (int64_t)c->np[0] * c->np[1] * (c->dim == 3 ? c->np[2] : 1); }
static inline int64_t n_bins(const o_cfg *c) { return c->pn[0] / c->bx; }
static inline void patch_coords(const o_cfg *c, int64_t flat, int64_t pc[3]) {
    if (c->dim == 3) {
        pc[2] = flat % c->np[2]; flat /= c->np[2];
    } else pc[2] = 0;
    pc[1] = flat % c->np[1];
    pc[0] = flat / c->np[1];
}

/* Add a subgrid (origin = global node org[], extent se[]) into the owner-folded int64 accumulator
 * at quantum 2^-44 with rint (fields.py:101-114 + exchange.py:134-147). */
static void fold_subgrid(const o_cfg *c, int comp, const double *sub, const int64_t se[3], const int64_t org[3],
                         int64_t *acc) {
    for (int64_t u = 0; u < se[0]; ++u) {
        int s0; int64_t gi = ghost_owner(org[0] + u, c->L[0], c->bc[0], dual_of(c, comp, 0), 1, &s0);
        for (int64_t v = 0; v < se[1]; ++v) {
            int s1; int64_t gj = ghost_owner(org[1] + v, c->L[1], c->bc[1], dual_of(c, comp, 1), 1, &s1);
            for (int64_t q = 0; q < se[2]; ++q) {
                int s2 = 1; int64_t gk = 0;
                if (c->dim == 3) {
                    gk = ghost_owner(org[2] + q, c->L[2], c->bc[2], dual_of(c, comp, 2), 1, &s2);
                    if (gk < 0) continue;
                    gk += G;
                }
                if (gi < 0 || gj < 0) continue;  /* beyond an absorbing wall */
                double val = sub[(u * se[1] + v) * se[2] + q];
                if (val == 0.0) continue;
                int64_t iv = llrint(val * J_SCALE);
                int64_t t = gidx(c, gi + G, gj + G, gk);
                int64_t add = (s0 * s1 * s2 > 0) ? iv : -iv;
#pragma omp atomic
                acc[t] += add;
            }
        }
    }
}

/* Particle phase: interpolate/push/pre-BC/project per (patch, bin) + reduction, for n_species
 * species.  Each (patch, bin) subgrid is rounded to 2^-44 and folded once after ALL the species
 * given have deposited into it: n_species = 1 is the reference's per-(patch, species, bin) reduction
 * (fields.py:101-114); n_species = 2 restates the device's merged work items (one tile per
 * (patch, bin) over both species, csrc/sort.cu merged_items) -- not in the reference.
 * fields: ex,ey,ez,bx,by,bz global arrays (ghosts synced).  jacc: 3 owner-folded int64 arrays.
 * flags[s][n] written.  Returns 0 or an error code with *bad_id. */
int o_particle_phase_multi(const o_cfg *c, o_species *const *ss, int n_species, const double *const f[6],
                           int64_t *const jacc[3], uint8_t *const *flagss, int64_t *bad_id) {
    const int64_t NP = n_patches(c), NB = n_bins(c);
    const int dim = c->dim;
    const double inv_dx = 1.0 / c->d[0], inv_dy = 1.0 / c->d[1], inv_dz = dim == 3 ? 1.0 / c->d[2] : 1.0;
    const double dxdt = c->d[0] / c->dt, dydt = c->d[1] / c->dt, dzdt = dim == 3 ? c->d[2] / c->dt : 0.0;
    const int64_t e1 = ext_of(c, 1), e2 = ext_of(c, 2);
    int err = OK;
    int64_t err_id = INT64_MAX;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t pf = 0; pf < NP; ++pf) {
        int64_t pc[3]; patch_coords(c, pf, pc);
        int64_t cell0[3] = {pc[0] * c->pn[0], pc[1] * c->pn[1], dim == 3 ? pc[2] * c->pn[2] : 0};
        int64_t se[3] = {c->bx + 1 + 2 * G, c->pn[1] + 1 + 2 * G, dim == 3 ? c->pn[2] + 1 + 2 * G : 1};
        int64_t sub_n = se[0] * se[1] * se[2];
        double *sub = malloc(sizeof(double) * 3 * sub_n);
        double bounds[6];
        for (int a = 0; a < 3; ++a) {
            bounds[2 * a] = cell0[a] * c->d[a];                 /* domain.py:26-29 */
            bounds[2 * a + 1] = (cell0[a] + c->pn[a]) * c->d[a];
        }
        for (int64_t b = 0; b < NB; ++b) {
            int64_t xs = b * c->bx;
            int64_t sub0[3] = {cell0[0] + xs, cell0[1], cell0[2]};
            int any = 0, failed = 0;
            memset(sub, 0, sizeof(double) * 3 * sub_n);
            for (int sp = 0; sp < n_species; ++sp) {
                o_species *s = ss[sp];
                uint8_t *flags = flagss[sp];
                int64_t s0 = s->offsets[pf * NB + b], s1 = s->offsets[pf * NB + b + 1], n = s1 - s0;
                if (n == 0) continue;
                any = 1;
                int64_t *ci = malloc(sizeof(int64_t) * 3 * n);
                double *dl = malloc(sizeof(double) * 3 * n);
                double *buf = malloc(sizeof(double) * 6 * n);
                double *out[6];
                for (int k = 0; k < 6; ++k) out[k] = buf + k * n;
                int64_t bad_push, bad_proj;
                if (dim == 2) {
                    o_gather_2d(n, s->x + s0, s->y + s0, f, e1, ci, ci + n, dl, dl + n, out, inv_dx, inv_dy, 0, 0);
                    bad_push = o_push(n, s->x + s0, s->y + s0, NULL, s->px + s0, s->py + s0, s->pz + s0,
                                      (const double *const *)out, s->charge, s->mass, c->dt);
                    o_flag(n, s->x + s0, s->y + s0, NULL, flags + s0, bounds);
                    bad_proj = o_project_2d(n, s->x + s0, s->y + s0, s->px + s0, s->py + s0, s->pz + s0, s->w + s0,
                                            ci, ci + n, dl, dl + n, sub, sub + sub_n, sub + 2 * sub_n, se[1],
                                            s->charge, s->mass, inv_dx, inv_dy, dxdt, dydt, sub0[0], sub0[1]);
                } else {
                    o_gather_3d(n, s->x + s0, s->y + s0, s->z + s0, f, e1, e2, ci, dl, out, inv_dx, inv_dy, inv_dz,
                                0, 0, 0);
                    bad_push = o_push(n, s->x + s0, s->y + s0, s->z + s0, s->px + s0, s->py + s0, s->pz + s0,
                                      (const double *const *)out, s->charge, s->mass, c->dt);
                    o_flag(n, s->x + s0, s->y + s0, s->z + s0, flags + s0, bounds);
                    bad_proj = o_project_3d(n, s->x + s0, s->y + s0, s->z + s0, s->px + s0, s->py + s0,
                                            s->pz + s0, s->w + s0, ci, dl, sub, sub + sub_n, sub + 2 * sub_n, se[1],
                                            se[2], s->charge, s->mass, inv_dx, inv_dy, inv_dz, dxdt, dydt, dzdt,
                                            sub0[0], sub0[1], sub0[2]);
                }
                free(ci); free(dl); free(buf);
                if (bad_push >= 0 || bad_proj >= 0) {
#pragma omp critical
                    {
                        int64_t id = s->id[s0 + (bad_push >= 0 ? bad_push : bad_proj)];
                        int e = bad_push >= 0 ? ERR_NONFINITE : ERR_COURANT;
                        if (id < err_id) { err_id = id; err = e; }
                    }
                    failed = 1;
                }
            }
            if (!any || failed) continue;
            int64_t org[3] = {sub0[0] - G, sub0[1] - G, dim == 3 ? sub0[2] - G : 0};
            for (int k = 0; k < 3; ++k) fold_subgrid(c, C_JX + k, sub + k * sub_n, se, org, jacc[k]);
        }
        free(sub);
    }
    if (err) *bad_id = err_id;
    return err;
}

/* One species (the reference's granularity). */
int o_particle_phase(const o_cfg *c, o_species *s, const double *const f[6], int64_t *const jacc[3],
                     uint8_t *flags, int64_t *bad_id) {
    return o_particle_phase_multi(c, &s, 1, f, jacc, &flags, bad_id);
}

/* fields.py:77-81 on owned indices; ghosts stay 0 (exchange.py:140-147) */
void o_currents(const o_cfg *c, int64_t *const jacc[3], double *const j[3]) {
    int64_t e0 = ext_of(c, 0), e1 = ext_of(c, 1), e2 = ext_of(c, 2), tot = e0 * e1 * e2;
    for (int k = 0; k < 3; ++k)
        for (int64_t t = 0; t < tot; ++t) j[k][t] = jacc[k][t] * INV_J_SCALE;
}

/* exchange.py:99-123 / 150-156 on one whole-domain array: x sweep, then y, then z */
void o_sync_component(const o_cfg *c, int comp, double *f) {
    int64_t e[3] = {ext_of(c, 0), ext_of(c, 1), ext_of(c, 2)};
    for (int a = 0; a < c->dim; ++a) {
        int64_t hi = owned_hi(c, comp, a);
        for (int64_t i = 0; i < e[a]; ++i) {
            if (i >= G && i < hi) continue;
            int sg; int64_t src = ghost_owner(i - G, c->L[a], c->bc[a], dual_of(c, comp, a), 0, &sg) + G;
            for (int64_t u = 0; u < (a == 0 ? 1 : e[0]); ++u)
                for (int64_t v = 0; v < (a == 1 ? 1 : e[1]); ++v)
                    for (int64_t q = 0; q < (a == 2 ? 1 : e[2]); ++q) {
                        int64_t di[3] = {u, v, q}, si[3] = {u, v, q};
                        di[a] = i; si[a] = src;
                        f[(di[0] * e[1] + di[1]) * e[2] + di[2]] = sg * f[(si[0] * e[1] + si[1]) * e[2] + si[2]];
                    }
        }
    }
}

void o_sync_fields(const o_cfg *c, double *const f[6]) {
    for (int k = 0; k < 6; ++k) o_sync_component(c, C_EX + k, f[k]);
}

/* fields.py:146-155 (2D) and its 3D generalisation */
static void half_b(const o_cfg *c, double *const f[6]) {
    const int64_t e1 = ext_of(c, 1), e2 = ext_of(c, 2);
    const double hdt[3] = {0.5 * c->dt / c->d[0], 0.5 * c->dt / c->d[1], c->dim == 3 ? 0.5 * c->dt / c->d[2] : 0.0};
    double *ex = f[0], *ey = f[1], *ez = f[2], *bx = f[3], *by = f[4], *bz = f[5];
    const int64_t sx = e1 * e2, sy = e2, sz = 1;
    for (int comp = C_BX; comp <= C_BZ; ++comp) {
        int64_t hx = owned_hi(c, comp, 0), hy = owned_hi(c, comp, 1), hz = c->dim == 3 ? owned_hi(c, comp, 2) : 1;
        int64_t lz = c->dim == 3 ? G : 0;
        for (int64_t i = G; i < hx; ++i)
            for (int64_t j = G; j < hy; ++j)
                for (int64_t k = lz; k < hz; ++k) {
                    int64_t t = (i * e1 + j) * e2 + k;
                    if (c->dim == 2) {
                        if (comp == C_BX) bx[t] -= hdt[1] * (ez[t + sy] - ez[t]);
                        else if (comp == C_BY) by[t] += hdt[0] * (ez[t + sx] - ez[t]);
                        else bz[t] -= hdt[0] * (ey[t + sx] - ey[t]) - hdt[1] * (ex[t + sy] - ex[t]);
                    } else {
                        if (comp == C_BX) bx[t] -= hdt[1] * (ez[t + sy] - ez[t]) - hdt[2] * (ey[t + sz] - ey[t]);
                        else if (comp == C_BY) by[t] -= hdt[2] * (ex[t + sz] - ex[t]) - hdt[0] * (ez[t + sx] - ez[t]);
                        else bz[t] -= hdt[0] * (ey[t + sx] - ey[t]) - hdt[1] * (ex[t + sy] - ex[t]);
                    }
                }
    }
}

/* fields.py:158-170 (2D) and its 3D generalisation */
static void full_e(const o_cfg *c, double *const f[6], const double *const j[3]) {
    const int64_t e1 = ext_of(c, 1), e2 = ext_of(c, 2);
    const double dt = c->dt;
    const double dtd[3] = {dt / c->d[0], dt / c->d[1], c->dim == 3 ? dt / c->d[2] : 0.0};
    double *ex = f[0], *ey = f[1], *ez = f[2], *bx = f[3], *by = f[4], *bz = f[5];
    const int64_t sx = e1 * e2, sy = e2, sz = 1;
    for (int comp = C_EX; comp <= C_EZ; ++comp) {
        int64_t hx = owned_hi(c, comp, 0), hy = owned_hi(c, comp, 1), hz = c->dim == 3 ? owned_hi(c, comp, 2) : 1;
        int64_t lz = c->dim == 3 ? G : 0;
        for (int64_t i = G; i < hx; ++i)
            for (int64_t jj = G; jj < hy; ++jj)
                for (int64_t k = lz; k < hz; ++k) {
                    int64_t t = (i * e1 + jj) * e2 + k;
                    if (c->dim == 2) {
                        if (comp == C_EX) ex[t] += dtd[1] * (bz[t] - bz[t - sy]) - dt * j[0][t];
                        else if (comp == C_EY) ey[t] += -dtd[0] * (bz[t] - bz[t - sx]) - dt * j[1][t];
                        else ez[t] += dtd[0] * (by[t] - by[t - sx]) - dtd[1] * (bx[t] - bx[t - sy]) - dt * j[2][t];
                    } else {
                        if (comp == C_EX) ex[t] += dtd[1] * (bz[t] - bz[t - sy]) - dtd[2] * (by[t] - by[t - sz]) - dt * j[0][t];
                        else if (comp == C_EY) ey[t] += dtd[2] * (bx[t] - bx[t - sz]) - dtd[0] * (bz[t] - bz[t - sx]) - dt * j[1][t];
                        else ez[t] += dtd[0] * (by[t] - by[t - sx]) - dtd[1] * (bx[t] - bx[t - sy]) - dt * j[2][t];
                    }
                }
    }
}

/* fields.py:173-190: tangential E and normal B pinned on reflective walls */
static void pin_walls(const o_cfg *c, double *const f[6]) {
    int64_t e[3] = {ext_of(c, 0), ext_of(c, 1), ext_of(c, 2)};
    static const int PIN[3][3] = {{C_EY, C_EZ, C_BX}, {C_EX, C_EZ, C_BY}, {C_EX, C_EY, C_BZ}};
    for (int a = 0; a < c->dim; ++a) {
        if (c->bc[a] != 1) continue;
        int64_t walls[2] = {G, G + c->L[a]};
        for (int wi = 0; wi < 2; ++wi)
            for (int m = 0; m < 3; ++m) {
                double *arr = f[PIN[a][m]];
                for (int64_t u = 0; u < (a == 0 ? 1 : e[0]); ++u)
                    for (int64_t v = 0; v < (a == 1 ? 1 : e[1]); ++v)
                        for (int64_t q = 0; q < (a == 2 ? 1 : e[2]); ++q) {
                            int64_t di[3] = {u, v, q};
                            di[a] = walls[wi];
                            arr[(di[0] * e[1] + di[1]) * e[2] + di[2]] = 0.0;
                        }
            }
    }
}

/* first-order Silver-Mueller wall on absorbing x boundaries (device twin: fields.cu k_silver_muller_x) */
static void silver_muller(const o_cfg *c, double *const f[6]) {
    if (c->bc[0] != 2) return;
    int64_t e1 = ext_of(c, 1), e2 = ext_of(c, 2), sx = e1 * e2;
    double *ey = f[C_EY], *ez = f[C_EZ], *by = f[C_BY], *bz = f[C_BZ];
    for (int64_t r = 0; r < sx; ++r) {
        int64_t q0 = G * sx + r, qL = (G + c->L[0]) * sx + r;
        bz[q0 - sx] = -2.0 * ey[q0] - bz[q0];
        by[q0 - sx] = 2.0 * ez[q0] - by[q0];
        bz[qL] = 2.0 * ey[qL] - bz[qL - sx];
        by[qL] = -2.0 * ez[qL] - by[qL - sx];
    }
}

/* Synced Yee step: half-B, sync, full-E, sync, half-B, walls, sync (+ Silver-Mueller on absorbing x). */
void o_maxwell(const o_cfg *c, double *const f[6], const double *const j[3]) {
    half_b(c, f);
    o_sync_fields(c, f);
    silver_muller(c, f);
    full_e(c, f, j);
    o_sync_fields(c, f);
    half_b(c, f);
    pin_walls(c, f);
    o_sync_fields(c, f);
    silver_muller(c, f);
}

/* maxwell_step exactly as shipped (fields.py:130-143, scheduler.py:478-484): every patch runs the three
 * sub-steps on its OWN ghosted array whose ghosts hold the values of the last sync_field_ghosts (so the
 * ghosts read by full-E are half a step stale and those read by the second half-B a full step), then one
 * sync.  Restated literally: each patch's window (owned + 3 ghost layers) is copied out of the synced
 * whole-domain arrays, stepped with the patch's own owned ranges (owned_slices, fields.py:117-127: a patch
 * owns the wall node only as the last patch of a non-periodic axis), and its owned nodes are written
 * back; walls are pinned and ghosts refreshed afterwards. */
void o_maxwell_lagged(const o_cfg *c, double *const f[6], const double *const j[3]) {
    o_cfg lc = *c;
    for (int a = 0; a < 3; ++a) lc.L[a] = a < c->dim ? c->pn[a] : 1;
    const int64_t le[3] = {ext_of(&lc, 0), ext_of(&lc, 1), ext_of(&lc, 2)};
    const int64_t ge[3] = {ext_of(c, 0), ext_of(c, 1), ext_of(c, 2)};
    const int64_t ln = le[0] * le[1] * le[2], gn = ge[0] * ge[1] * ge[2];
    double *loc = (double *)malloc(sizeof(double) * 9 * ln);
    double *out = (double *)malloc(sizeof(double) * 6 * gn);
    double *lf[6], *lj[3];
    for (int k = 0; k < 6; ++k) {
        lf[k] = loc + k * ln;
        memcpy(out + k * gn, f[k], sizeof(double) * gn);
    }
    for (int k = 0; k < 3; ++k) lj[k] = loc + (6 + k) * ln;
    const int64_t npz = c->dim == 3 ? c->np[2] : 1;
    for (int64_t px = 0; px < c->np[0]; ++px)
        for (int64_t py = 0; py < c->np[1]; ++py)
            for (int64_t pz = 0; pz < npz; ++pz) {
                const int64_t pc[3] = {px, py, pz};
                int64_t o[3];
                for (int a = 0; a < 3; ++a) {
                    o[a] = a < c->dim ? pc[a] * c->pn[a] : 0;  /* whole-domain index of local index 0 */
                    /* the patch owns the wall node only as the last patch of a non-periodic axis */
                    lc.bc[a] = (a < c->dim && c->bc[a] != 0 && pc[a] == c->np[a] - 1) ? c->bc[a] : 0;
                }
                for (int64_t u = 0; u < le[0]; ++u)
                    for (int64_t v = 0; v < le[1]; ++v)
                        for (int64_t q = 0; q < le[2]; ++q) {
                            const int64_t lt = (u * le[1] + v) * le[2] + q;
                            const int64_t gt = ((o[0] + u) * ge[1] + o[1] + v) * ge[2] + o[2] + q;
                            for (int k = 0; k < 6; ++k) lf[k][lt] = f[k][gt];
                            for (int k = 0; k < 3; ++k) lj[k][lt] = j[k][gt];
                        }
                half_b(&lc, lf);
                full_e(&lc, lf, (const double *const *)lj);
                half_b(&lc, lf);
                for (int k = 0; k < 6; ++k) {
                    const int comp = C_EX + k;
                    const int64_t hx = owned_hi(&lc, comp, 0), hy = owned_hi(&lc, comp, 1);
                    const int64_t lz = c->dim == 3 ? G : 0, hz = c->dim == 3 ? owned_hi(&lc, comp, 2) : 1;
                    for (int64_t u = G; u < hx; ++u)
                        for (int64_t v = G; v < hy; ++v)
                            for (int64_t q = lz; q < hz; ++q)
                                out[k * gn + ((o[0] + u) * ge[1] + o[1] + v) * ge[2] + o[2] + q] =
                                    lf[k][(u * le[1] + v) * le[2] + q];
                }
            }
    for (int k = 0; k < 6; ++k) memcpy(f[k], out + k * gn, sizeof(double) * gn);
    free(loc);
    free(out);
    pin_walls(c, f);
    o_sync_fields(c, f);
}

/* One sub-step at a time (for unit tests of K2) */
void o_half_b(const o_cfg *c, double *const f[6]) { half_b(c, f); }
void o_full_e(const o_cfg *c, double *const f[6], const double *const j[3]) { full_e(c, f, j); }
void o_pin_walls(const o_cfg *c, double *const f[6]) { pin_walls(c, f); }

/* ---------------------------------------------------------------------- */
/* BC + migration + canonical re-sort (exchange.py:163-258, arena.py:59-95) */
/* ---------------------------------------------------------------------- */

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return x < y ? -1 : x > y;
}

/* In: species s (canonical order, offsets) + flags.  Out: arrays in `o` (capacity >= s->n) in canonical order
 * with offsets.  Returns OK or ERR_INVARIANT (*bad_id = particle id). */
int o_migrate_sort(const o_cfg *c, const o_species *s, const uint8_t *flags, o_species *o, int64_t *bad_id) {
    const int64_t NP = n_patches(c), NB = n_bins(c), NK = NP * NB, n = s->offsets[NK];
    const int dim = c->dim;
    const double inv[3] = {1.0 / c->d[0], 1.0 / c->d[1], dim == 3 ? 1.0 / c->d[2] : 1.0};
    const double Lw[3] = {c->L[0] * c->d[0], c->L[1] * c->d[1], dim == 3 ? c->L[2] * c->d[2] : 0.0};
    double *pos[3] = {s->x, s->y, s->z}, *mom[3] = {s->px, s->py, s->pz};
    int64_t *key = malloc(sizeof(int64_t) * (n ? n : 1));
    /* new position/momentum copies (BC applies to movers only) */
    double *nx_[3], *np_[3];
    for (int a = 0; a < 3; ++a) {
        nx_[a] = pos[a] ? malloc(sizeof(double) * (n ? n : 1)) : NULL;
        np_[a] = malloc(sizeof(double) * (n ? n : 1));
        if (pos[a]) memcpy(nx_[a], pos[a], sizeof(double) * n);
        memcpy(np_[a], mom[a], sizeof(double) * n);
    }
    int err = OK;
    int64_t err_id = INT64_MAX;
#pragma omp parallel for schedule(static)
    for (int64_t pf = 0; pf < NP; ++pf) {
        int64_t pc[3]; patch_coords(c, pf, pc);
        int last[3], first[3];
        for (int a = 0; a < 3; ++a) { first[a] = pc[a] == 0; last[a] = pc[a] == c->np[a] - 1; }
        for (int64_t i = s->offsets[pf * NB]; i < s->offsets[pf * NB + NB]; ++i) {
            int64_t dest[3] = {pc[0], pc[1], pc[2]};
            int fl = flags[i];
            if (fl) {
                int absorbed = 0;
                for (int a = 0; a < dim; ++a) {
                    int fneg = 1 << (2 * a), fpos = 2 << (2 * a);
                    if (c->bc[a] == 2 && ((last[a] && (fl & fpos)) || (first[a] && (fl & fneg)))) absorbed = 1;
                }
                if (absorbed) { key[i] = NK; continue; }  /* deleted (beyond the reference) */
                for (int a = 0; a < dim; ++a) {
                    int fneg = 1 << (2 * a), fpos = 2 << (2 * a);
                    /* exchange.py:163-193 (x last, x first, y last, y first, ...) */
                    if (last[a] && (fl & fpos)) {
                        if (c->bc[a] == 0) nx_[a][i] -= Lw[a];
                        else { nx_[a][i] = fmin(2.0 * Lw[a] - nx_[a][i], nextafter(Lw[a], 0.0)); np_[a][i] = -np_[a][i]; }
                    }
                    if (first[a] && (fl & fneg)) {
                        if (c->bc[a] == 0) nx_[a][i] += Lw[a];
                        else { nx_[a][i] = -nx_[a][i]; np_[a][i] = -np_[a][i]; }
                    }
                }
                /* exchange.py:223-230 */
                for (int a = 0; a < dim; ++a) {
                    int64_t cell = (int64_t)floor(nx_[a][i] * inv[a]);
                    if (cell < 0) cell = 0;
                    if (cell > c->L[a] - 1) cell = c->L[a] - 1;
                    dest[a] = cell / c->pn[a];
                }
            }
            /* arena.py:59-75: x cell relative to the destination patch */
            int64_t cx = (int64_t)floor(nx_[0][i] * inv[0]) - dest[0] * c->pn[0];
            if (cx < 0 || cx > c->pn[0]) {
#pragma omp critical
                { if (s->id[i] < err_id) { err_id = s->id[i]; err = ERR_INVARIANT; } }
            }
            if (cx < 0) cx = 0;
            if (cx > c->pn[0] - 1) cx = c->pn[0] - 1;
            int64_t df = dim == 3 ? (dest[0] * c->np[1] + dest[1]) * c->np[2] + dest[2] : dest[0] * c->np[1] + dest[1];
            key[i] = df * NB + cx / c->bx;
        }
    }
    if (err) {
        *bad_id = err_id;
    } else {
        /* stable counting sort by key, then ascending id within each (patch, bin) */
        int64_t *cnt = calloc(NK + 2, sizeof(int64_t));
        for (int64_t i = 0; i < n; ++i) cnt[key[i] + 1]++;  /* key NK: absorbed, sorted past the end */
        for (int64_t k = 0; k < NK; ++k) cnt[k + 1] += cnt[k];
        memcpy(o->offsets, cnt, sizeof(int64_t) * (NK + 1));
        int64_t *perm = malloc(sizeof(int64_t) * (n ? n : 1));
        int64_t *pos_ = malloc(sizeof(int64_t) * (NK + 2));
        memcpy(pos_, cnt, sizeof(int64_t) * (NK + 1));
        pos_[NK + 1] = 0;
        for (int64_t i = 0; i < n; ++i) if (key[i] < NK) perm[pos_[key[i]]++] = i;
        const int64_t kept = cnt[NK];
        /* sort each bucket by id: build (id, index) pairs */
        int64_t *pair = malloc(sizeof(int64_t) * 2 * (n ? n : 1));
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t k = 0; k < NK; ++k) {
            int64_t a0 = cnt[k], a1 = cnt[k + 1];
            for (int64_t t = a0; t < a1; ++t) { pair[2 * t] = s->id[perm[t]]; pair[2 * t + 1] = perm[t]; }
            qsort(pair + 2 * a0, a1 - a0, 2 * sizeof(int64_t), cmp_i64);
        }
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < kept; ++t) {
            int64_t i = pair[2 * t + 1];
            o->x[t] = nx_[0][i]; o->y[t] = nx_[1][i];
            if (dim == 3) o->z[t] = nx_[2][i];
            o->px[t] = np_[0][i]; o->py[t] = np_[1][i]; o->pz[t] = np_[2][i];
            o->w[t] = s->w[i]; o->id[t] = s->id[i];
        }
        o->n = kept;
        free(cnt); free(perm); free(pos_); free(pair);
    }
    free(key);
    for (int a = 0; a < 3; ++a) { free(nx_[a]); free(np_[a]); }
    return err;
}

/* Canonical sort of freshly injected particles (harness injection + arena.py:78-95):
 * every particle is routed like a mover without BC (patch from clip(floor(x/dx))), then (bin, id). */
int o_initial_sort(const o_cfg *c, const o_species *s, o_species *o, int64_t *bad_id) {
    const int64_t NK = n_patches(c) * n_bins(c), n = s->n;
    o_species tmp = *s;
    int64_t *offs = calloc(NK + 1, sizeof(int64_t));
    for (int64_t k = 1; k <= NK; ++k) offs[k] = n; /* all in (patch 0, bin 0) */
    tmp.offsets = offs;
    uint8_t *fl = malloc(n ? n : 1);
    memset(fl, 0x40, n ? n : 1); /* non-zero (=> rerouted) but no BC bit set */
    int r = o_migrate_sort(c, &tmp, fl, o, bad_id);
    free(fl);
    free(offs);
    return r;
}

int o_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void o_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
