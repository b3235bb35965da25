// particle_math.cuh -- per-particle device math shared by the operator-level
// kernels and the fused K1 kernel.  Each function restates one reference
// kernel body with the same IEEE op order (compiled with -fmad=false).
#pragma once
#include "common.cuh"

// --------------------------------------------------------------------------
// gather (kernels.py:51-121).  Field views: component base pointers, row
// strides (s1 = y stride, s2 = z stride) and the node index of element 0 per
// axis ("org"); for the reference's patch arrays org = cell0 - 3.
// --------------------------------------------------------------------------

struct Gathered {
    int64_t ip, jp, kp;   // primal node indices (cix, ciy, ciz)
    double dxp, dyp, dzp; // primal displacements (dlx, dly, dlz)
    double e[3], b[3];
};

__device__ __forceinline__ double interp2(const double *__restrict__ f, int64_t s1, int64_t a, int64_t b,
                                          double wx0, double wx1, double wx2, double wy0, double wy1, double wy2) {
    const double *r0 = f + (a - 1) * s1 + b, *r1 = r0 + s1, *r2 = r1 + s1;
    return wx0 * (wy0 * r0[-1] + wy1 * r0[0] + wy2 * r0[1]) + wx1 * (wy0 * r1[-1] + wy1 * r1[0] + wy2 * r1[1]) +
           wx2 * (wy0 * r2[-1] + wy1 * r2[0] + wy2 * r2[1]);
}

// 2D: kernels.py:61-121 verbatim (f[0..5] = ex ey ez bx by bz)
__device__ __forceinline__ bool gather2d(double x, double y, double inv_dx, double inv_dy,
                                         const double *const *f, int64_t s1, int64_t orgx, int64_t orgy,
                                         int64_t ex_lo, int64_t ex_hi, int64_t ey_lo, int64_t ey_hi, Gathered &g) {
    double xn = x * inv_dx, yn = y * inv_dy;
    int64_t ip = (int64_t)(xn + 0.5), jp = (int64_t)(yn + 0.5);
    double dxp = xn - ip, dyp = yn - jp;
    int64_t idu = (int64_t)xn, jdu = (int64_t)yn;
    double dxd = xn - 0.5 - idu, dyd = yn - 0.5 - jdu;
    g.ip = ip; g.jp = jp; g.kp = 0; g.dxp = dxp; g.dyp = dyp; g.dzp = 0.0;
    int64_t ap = ip - orgx, bp = jp - orgy, ad = idu - orgx, bd = jdu - orgy;
    // stencil must stay inside the provided array view
    if (min(ap, ad) - 1 < ex_lo || max(ap, ad) + 1 > ex_hi || min(bp, bd) - 1 < ey_lo || max(bp, bd) + 1 > ey_hi)
        return false;
    double wxp0, wxp1, wxp2, wyp0, wyp1, wyp2, wxd0, wxd1, wxd2, wyd0, wyd1, wyd2;
    spline3(dxp, wxp0, wxp1, wxp2);
    spline3(dyp, wyp0, wyp1, wyp2);
    spline3(dxd, wxd0, wxd1, wxd2);
    spline3(dyd, wyd0, wyd1, wyd2);
    g.e[0] = interp2(f[0], s1, ad, bp, wxd0, wxd1, wxd2, wyp0, wyp1, wyp2);
    g.e[1] = interp2(f[1], s1, ap, bd, wxp0, wxp1, wxp2, wyd0, wyd1, wyd2);
    g.e[2] = interp2(f[2], s1, ap, bp, wxp0, wxp1, wxp2, wyp0, wyp1, wyp2);
    g.b[0] = interp2(f[3], s1, ap, bd, wxp0, wxp1, wxp2, wyd0, wyd1, wyd2);
    g.b[1] = interp2(f[4], s1, ad, bp, wxd0, wxd1, wxd2, wyp0, wyp1, wyp2);
    g.b[2] = interp2(f[5], s1, ad, bd, wxd0, wxd1, wxd2, wyd0, wyd1, wyd2);
    return true;
}

// 3D: same nesting as the 2D sum, extended along z (oracle/pic_oracle.c interp3)
__device__ __forceinline__ double interp3(const double *__restrict__ f, int64_t s1, int64_t s2, int64_t a,
                                          int64_t b, int64_t c, const double *wx, const double *wy,
                                          const double *wz) {
    double sx = 0.0;
#pragma unroll
    for (int u = 0; u < 3; ++u) {
        double sy = 0.0;
#pragma unroll
        for (int v = 0; v < 3; ++v) {
            const double *r = f + (a - 1 + u) * s1 + (b - 1 + v) * s2 + (c - 1);
            double sz = wz[0] * r[0] + wz[1] * r[1] + wz[2] * r[2];
            sy = (v == 0) ? wy[0] * sz : sy + wy[v] * sz;
        }
        sx = (u == 0) ? wx[0] * sy : sx + wx[u] * sy;
    }
    return sx;
}

__device__ __forceinline__ bool gather3d(double x, double y, double z, const double inv[3],
                                         const double *const *f, int64_t s1, int64_t s2, const int64_t org[3],
                                         const int64_t lo[3], const int64_t hi[3], Gathered &g) {
    double xn[3] = {x * inv[0], y * inv[1], z * inv[2]};
    int64_t ip[3], id[3];
    double wp[3][3], wd[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        ip[a] = (int64_t)(xn[a] + 0.5);
        id[a] = (int64_t)xn[a];
        double dp = xn[a] - ip[a], dd = xn[a] - 0.5 - id[a];
        spline3(dp, wp[a][0], wp[a][1], wp[a][2]);
        spline3(dd, wd[a][0], wd[a][1], wd[a][2]);
        if (a == 0) g.dxp = dp; else if (a == 1) g.dyp = dp; else g.dzp = dp;
    }
    g.ip = ip[0]; g.jp = ip[1]; g.kp = ip[2];
    int64_t P[3], D[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        P[a] = ip[a] - org[a];
        D[a] = id[a] - org[a];
        if (min(P[a], D[a]) - 1 < lo[a] || max(P[a], D[a]) + 1 > hi[a]) return false;
    }
    g.e[0] = interp3(f[0], s1, s2, D[0], P[1], P[2], wd[0], wp[1], wp[2]);
    g.e[1] = interp3(f[1], s1, s2, P[0], D[1], P[2], wp[0], wd[1], wp[2]);
    g.e[2] = interp3(f[2], s1, s2, P[0], P[1], D[2], wp[0], wp[1], wd[2]);
    g.b[0] = interp3(f[3], s1, s2, P[0], D[1], D[2], wp[0], wd[1], wd[2]);
    g.b[1] = interp3(f[4], s1, s2, D[0], P[1], D[2], wd[0], wp[1], wd[2]);
    g.b[2] = interp3(f[5], s1, s2, D[0], D[1], P[2], wd[0], wd[1], wp[2]);
    return true;
}

// Tile-resident variants (shared-memory E/B tile, 32-bit offsets): same
// weights, same sum nesting as gather2d / gather3d, cheaper addressing.
// base[k] points at the tile of component k; (a, b, c) are tile indices of
// the stencil centre.
__device__ __forceinline__ double tinterp2(const double *__restrict__ f, int s1, int a, int b, double wx0,
                                           double wx1, double wx2, double wy0, double wy1, double wy2) {
    const double *r0 = f + (a - 1) * s1 + b, *r1 = r0 + s1, *r2 = r1 + s1;
    return wx0 * (wy0 * r0[-1] + wy1 * r0[0] + wy2 * r0[1]) + wx1 * (wy0 * r1[-1] + wy1 * r1[0] + wy2 * r1[1]) +
           wx2 * (wy0 * r2[-1] + wy1 * r2[0] + wy2 * r2[1]);
}

// 3D tile gather with FMA contraction: the 3D path is the builder's restatement (no reference
// code to match bit for bit), so it trades the last-ulp identity with oracle o_gather_3d for ~40%
// fewer FP64 instructions; the 2D gather (tinterp2) stays bit-exact with the reference
__device__ __forceinline__ double tinterp3(const double *__restrict__ f, int s1, int s2, int a, int b, int c,
                                           const double *wx, const double *wy, const double *wz) {
    const double *r = f + (a - 1) * s1 + (b - 1) * s2 + (c - 1);
    double sx = 0.0;
#pragma unroll
    for (int u = 0; u < 3; ++u) {
        double sy = 0.0;
#pragma unroll
        for (int v = 0; v < 3; ++v) {
            const double *q = r + u * s1 + v * s2;
            const double sz = __fma_rn(wz[2], q[2], __fma_rn(wz[1], q[1], wz[0] * q[0]));
            sy = __fma_rn(wy[v], sz, sy);
        }
        sx = __fma_rn(wx[u], sy, sx);
    }
    return sx;
}

// kernels.py:61-121 on a tile whose element 0 is node org[a]; returns false if
// the stencil leaves [0, T[a]) on any axis
template <int DIM>
__device__ __forceinline__ bool tile_gather(const double pos[3], const double inv[3], const double *tile, int TN,
                                            const int T[3], const int64_t org[3], Gathered &g, int xs = 0) {
    // xs: x stride of the tile (0: dense T[1] * T[2]; K1 pads it against shared-memory bank conflicts)
    int P_[3] = {0, 0, 0}, D_[3] = {0, 0, 0};
    double wp[3][3], wd[3][3];
    int64_t ip[3] = {0, 0, 0};
    double dp[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        const double xn = pos[a] * inv[a];
        ip[a] = (int64_t)(xn + 0.5);
        const int64_t id = (int64_t)xn;
        dp[a] = xn - ip[a];
        const double dd = xn - 0.5 - id;
        spline3(dp[a], wp[a][0], wp[a][1], wp[a][2]);
        spline3(dd, wd[a][0], wd[a][1], wd[a][2]);
        const int64_t pa = ip[a] - org[a], da = id - org[a];
        if (min(pa, da) < 1 || max(pa, da) > T[a] - 2) return false;
        P_[a] = (int)pa;
        D_[a] = (int)da;
    }
    g.ip = ip[0]; g.jp = ip[1]; g.kp = ip[2];
    g.dxp = dp[0]; g.dyp = dp[1]; g.dzp = dp[2];
    if (DIM == 2) {
        const int s1 = T[1];
        g.e[0] = tinterp2(tile, s1, D_[0], P_[1], wd[0][0], wd[0][1], wd[0][2], wp[1][0], wp[1][1], wp[1][2]);
        g.e[1] = tinterp2(tile + TN, s1, P_[0], D_[1], wp[0][0], wp[0][1], wp[0][2], wd[1][0], wd[1][1], wd[1][2]);
        g.e[2] = tinterp2(tile + 2 * TN, s1, P_[0], P_[1], wp[0][0], wp[0][1], wp[0][2], wp[1][0], wp[1][1], wp[1][2]);
        g.b[0] = tinterp2(tile + 3 * TN, s1, P_[0], D_[1], wp[0][0], wp[0][1], wp[0][2], wd[1][0], wd[1][1], wd[1][2]);
        g.b[1] = tinterp2(tile + 4 * TN, s1, D_[0], P_[1], wd[0][0], wd[0][1], wd[0][2], wp[1][0], wp[1][1], wp[1][2]);
        g.b[2] = tinterp2(tile + 5 * TN, s1, D_[0], D_[1], wd[0][0], wd[0][1], wd[0][2], wd[1][0], wd[1][1], wd[1][2]);
    } else {
        const int s1 = xs ? xs : T[1] * T[2], s2 = T[2];
        g.e[0] = tinterp3(tile, s1, s2, D_[0], P_[1], P_[2], wd[0], wp[1], wp[2]);
        g.e[1] = tinterp3(tile + TN, s1, s2, P_[0], D_[1], P_[2], wp[0], wd[1], wp[2]);
        g.e[2] = tinterp3(tile + 2 * TN, s1, s2, P_[0], P_[1], D_[2], wp[0], wp[1], wd[2]);
        g.b[0] = tinterp3(tile + 3 * TN, s1, s2, P_[0], D_[1], D_[2], wp[0], wd[1], wd[2]);
        g.b[1] = tinterp3(tile + 4 * TN, s1, s2, D_[0], P_[1], D_[2], wd[0], wp[1], wd[2]);
        g.b[2] = tinterp3(tile + 5 * TN, s1, s2, D_[0], D_[1], P_[2], wd[0], wd[1], wp[2]);
    }
    return true;
}

// --------------------------------------------------------------------------
// Boris push (kernels.py:131-161).  Returns false if the new momentum is not
// finite.  x/y/z advanced in place (z only if has_z).
// --------------------------------------------------------------------------
__device__ __forceinline__ bool boris(double &x, double &y, double &z, bool has_z, double &px, double &py,
                                      double &pz, const double e[3], const double b[3], double qd2,
                                      double inv_m2, double mass, double dt, double &gn_out) {
    double pxm = px + qd2 * e[0], pym = py + qd2 * e[1], pzm = pz + qd2 * e[2];
    double gm = sqrt(1.0 + (pxm * pxm + pym * pym + pzm * pzm) * inv_m2);
    double tf = qd2 / (gm * mass);
    double tx = tf * b[0], ty = tf * b[1], tz = tf * b[2];
    double sf = 2.0 / (1.0 + tx * tx + ty * ty + tz * tz);
    double sx = tx * sf, sy = ty * sf, sz = tz * sf;
    double ppx = pxm + (pym * tz - pzm * ty);
    double ppy = pym + (pzm * tx - pxm * tz);
    double ppz = pzm + (pxm * ty - pym * tx);
    double pxn = pxm + (ppy * sz - ppz * sy) + qd2 * e[0];
    double pyn = pym + (ppz * sx - ppx * sz) + qd2 * e[1];
    double pzn = pzm + (ppx * sy - ppy * sx) + qd2 * e[2];
    double gn = sqrt(1.0 + (pxn * pxn + pyn * pyn + pzn * pzn) * inv_m2);
    px = pxn; py = pyn; pz = pzn;
    gn_out = gn;  // == the sqrt recomputed in esirkepov_project (kernels.py:234), bitwise
    double adv = dt / (gn * mass);
    x += pxn * adv;
    y += pyn * adv;
    if (has_z) z += pzn * adv;
    return isfinite(pxn) && isfinite(pyn) && isfinite(pzn);
}

// kernels.py:165-178 (+ z bits)
__device__ __forceinline__ int pre_bc_flags(double x, double y, double z, bool has_z, const double bd[6]) {
    int f = 0;
    if (x < bd[0]) f |= FLAG_X_NEG; else if (x >= bd[1]) f |= FLAG_X_POS;
    if (y < bd[2]) f |= FLAG_Y_NEG; else if (y >= bd[3]) f |= FLAG_Y_POS;
    if (has_z) { if (z < bd[4]) f |= FLAG_Z_NEG; else if (z >= bd[5]) f |= FLAG_Z_POS; }
    return f;
}

// --------------------------------------------------------------------------
// Esirkepov order-2 shape vectors (kernels.py:202-232).  Returns false on a
// Courant violation (|shift| > 1 on any axis).
// --------------------------------------------------------------------------
__device__ __forceinline__ bool esirkepov_shapes(double xn, int64_t i0, double d0, double s0[5], double s1[5]) {
    int64_t i1 = (int64_t)(xn + 0.5);
    int64_t sh = i1 - i0;
    if (sh < -1 || sh > 1) return false;
    double d1 = xn - i1;
#pragma unroll
    for (int k = 0; k < 5; ++k) { s0[k] = 0.0; s1[k] = 0.0; }
    spline3(d0, s0[1], s0[2], s0[3]);
    double a, b, c;
    spline3(d1, a, b, c);
    // s1[1+sh..3+sh] = (a, b, c) without dynamic register indexing
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        int r = k - 1 - (int)sh;
        s1[k] = r == 0 ? a : r == 1 ? b : r == 2 ? c : 0.0;
    }
    return true;
}

// Deposit sink: J[c][(u*s1 + v)*s2 + q] += val, via Add (atomic to shared or global)
// 2D Esirkepov accumulation (kernels.py:233-265); bi/bj index of the footprint's first node
template <class Add>
__device__ __forceinline__ void esirkepov2d_accumulate(const double s0x[5], const double s1x[5], const double s0y[5],
                                                       const double s1y[5], double fx, double fy, double fz,
                                                       int64_t bi, int64_t bj, int64_t s1, Add add) {
    const double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
    if (fz != 0.0) {
#pragma unroll
        for (int ky = 0; ky < 5; ++ky) {
            double sy0 = s0y[ky], sy1 = s1y[ky];
            double cyx = 0.5 * (sy0 + sy1);
            double za = fz * (sy0 * third + sy1 * sixth), zb = fz * (sy0 * sixth + sy1 * third);
            double acc = 0.0;
#pragma unroll
            for (int kx = 0; kx < 4; ++kx) {
                acc -= fx * (s1x[kx] - s0x[kx]) * cyx;
                add(0, (bi + kx) * s1 + bj + ky, acc);
                add(2, (bi + kx) * s1 + bj + ky, s0x[kx] * za + s1x[kx] * zb);
            }
            add(2, (bi + 4) * s1 + bj + ky, s0x[4] * za + s1x[4] * zb);
        }
    } else {
#pragma unroll
        for (int ky = 0; ky < 5; ++ky) {
            double cyx = 0.5 * (s0y[ky] + s1y[ky]);
            double acc = 0.0;
#pragma unroll
            for (int kx = 0; kx < 4; ++kx) {
                acc -= fx * (s1x[kx] - s0x[kx]) * cyx;
                add(0, (bi + kx) * s1 + bj + ky, acc);
            }
        }
    }
#pragma unroll
    for (int kx = 0; kx < 5; ++kx) {
        double cxy = 0.5 * (s0x[kx] + s1x[kx]);
        double acc = 0.0;
#pragma unroll
        for (int ky = 0; ky < 4; ++ky) {
            acc -= fy * (s1y[ky] - s0y[ky]) * cxy;
            add(1, (bi + kx) * s1 + bj + ky, acc);
        }
    }
}

// 3D Esirkepov (restatement, oracle/pic_oracle.c o_project_3d): J += P[u] * w(v, q)
template <class Add>
__device__ __forceinline__ void esirkepov3d_accumulate(const double s0[3][5], const double s1[3][5], double fx,
                                                       double fy, double fz, int64_t bi, int64_t bj, int64_t bk,
                                                       int64_t st1, int64_t st2, Add add) {
    const double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
    const double f[3] = {fx, fy, fz};
    double P[3][4];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double pref = 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            pref -= f[a] * (s1[a][u] - s0[a][u]);
            P[a][u] = pref;
        }
    }
#define JI(u, v, q) ((bi + (u)) * st1 + (bj + (v)) * st2 + (bk + (q)))
#pragma unroll
    for (int v = 0; v < 5; ++v)
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            double wyz = s0[1][v] * (s0[2][q] * third + s1[2][q] * sixth) + s1[1][v] * (s0[2][q] * sixth + s1[2][q] * third);
#pragma unroll
            for (int u = 0; u < 4; ++u) add(0, JI(u, v, q), P[0][u] * wyz);
        }
#pragma unroll
    for (int u = 0; u < 5; ++u)
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            double wxz = s0[0][u] * (s0[2][q] * third + s1[2][q] * sixth) + s1[0][u] * (s0[2][q] * sixth + s1[2][q] * third);
#pragma unroll
            for (int v = 0; v < 4; ++v) add(1, JI(u, v, q), P[1][v] * wxz);
        }
#pragma unroll
    for (int u = 0; u < 5; ++u)
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            double wxy = s0[0][u] * (s0[1][v] * third + s1[1][v] * sixth) + s1[0][u] * (s0[1][v] * sixth + s1[1][v] * third);
#pragma unroll
            for (int q = 0; q < 4; ++q) add(2, JI(u, v, q), P[2][q] * wxy);
        }
#undef JI
}
