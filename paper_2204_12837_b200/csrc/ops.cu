// ops.cu -- operator-level device kernels with the reference kernels' own
// signatures (kernels.py:51-298, fields.py:101-114), for the _Engine drop-in
// (scheduler.py:113-170).  One thread per particle of [s0, s1).  These share
// the per-particle math of the fused K1 kernel (particle_math.cuh).
#include <math_constants.h>

#include "particle_math.cuh"

namespace {

struct F6 {
    const double *p[6];
};
struct O6 {
    double *p[6];
};

__global__ void k_gather2d(const double *__restrict__ x, const double *__restrict__ y, int64_t s0, int64_t s1,
                           F6 f, int64_t e1, int64_t *cix, int64_t *ciy, double *dlx, double *dly, O6 out,
                           double inv_dx, double inv_dy, int64_t orgx, int64_t orgy, int64_t ex_hi, int64_t ey_hi) {
    int64_t n = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= s1) return;
    Gathered g;
    // the reference indexes without bounds checks (numba boundscheck off): out-of-view stencils
    // are reported as NaN instead of reading out of bounds
    if (!gather2d(x[n], y[n], inv_dx, inv_dy, f.p, e1, orgx, orgy, 0, ex_hi, 0, ey_hi, g)) {
        for (int c = 0; c < 3; ++c) { g.e[c] = CUDART_NAN; g.b[c] = CUDART_NAN; }
    }
    cix[n] = g.ip; ciy[n] = g.jp; dlx[n] = g.dxp; dly[n] = g.dyp;
    for (int c = 0; c < 3; ++c) { out.p[c][n] = g.e[c]; out.p[3 + c][n] = g.b[c]; }
}

__global__ void k_push(double *x, double *y, double *z, double *px, double *py, double *pz, int64_t s0, int64_t s1,
                       F6 gth, double qd2, double inv_m2, double mass, double dt, unsigned long long *bad) {
    int64_t n = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= s1) return;
    double e[3] = {gth.p[0][n], gth.p[1][n], gth.p[2][n]}, b[3] = {gth.p[3][n], gth.p[4][n], gth.p[5][n]};
    double xx = x[n], yy = y[n], zz = z ? z[n] : 0.0, a = px[n], bb = py[n], c = pz[n], gn;
    bool ok = boris(xx, yy, zz, z != nullptr, a, bb, c, e, b, qd2, inv_m2, mass, dt, gn);
    x[n] = xx; y[n] = yy; if (z) z[n] = zz;
    px[n] = a; py[n] = bb; pz[n] = c;
    if (!ok) atomicMin(bad, (unsigned long long)n);  // first bad index (kernels.py:160-161)
}

__global__ void k_flag(const double *x, const double *y, const double *z, int64_t s0, int64_t s1, uint8_t *flags,
                       double b0, double b1, double b2, double b3, double b4, double b5) {
    int64_t n = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= s1) return;
    const double bd[6] = {b0, b1, b2, b3, b4, b5};
    flags[n] = (uint8_t)pre_bc_flags(x[n], y[n], z ? z[n] : 0.0, z != nullptr, bd);
}

// kernels.py:181-266 with the reference's summation order: one CTA walks the slice's particles in order
// and, per particle, one thread per (component, node) of its stencil (20 Jx + 20 Jy + 25 Jz nodes, all
// distinct) adds that particle's contribution -- every node then receives its contributions in particle
// order, the same float sum as the sequential numba loop, bit for bit.  A Courant violator stops the walk
// where the reference returns (kernels.py:208-211): earlier particles deposited, later ones not.
__global__ void k_project2d_ordered(const double *x, const double *y, const double *px, const double *py,
                                    const double *pz, const double *w, int64_t s0, int64_t s1, const int64_t *cix,
                                    const int64_t *ciy, const double *dlx, const double *dly, double *jx,
                                    double *jy, double *jz, int64_t e1, double charge, double mass, double inv_dx,
                                    double inv_dy, double dxdt, double dydt, int64_t sub_cell0x, int64_t sub_cell0y,
                                    unsigned long long *bad) {
    const int t = threadIdx.x;
    const double inv_m2 = 1.0 / (mass * mass);
    const double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
    for (int64_t n = s0; n < s1; ++n) {
        double s0x[5], s1x[5], s0y[5], s1y[5];
        const int64_t i0 = cix[n], j0 = ciy[n];
        if (!esirkepov_shapes(x[n] * inv_dx, i0, dlx[n], s0x, s1x) ||
            !esirkepov_shapes(y[n] * inv_dy, j0, dly[n], s0y, s1y)) {
            if (t == 0) *bad = (unsigned long long)n;
            return;  // (uniform: every thread sees the same particle)
        }
        const double qw = charge * w[n];
        const double gam = sqrt(1.0 + (px[n] * px[n] + py[n] * py[n] + pz[n] * pz[n]) * inv_m2);
        const double fx = qw * dxdt, fy = qw * dydt, fz = qw * pz[n] / (gam * mass);
        const int64_t bi = i0 - 2 - sub_cell0x + G, bj = j0 - 2 - sub_cell0y + G;
        if (t < 20) {  // Jx(kx, ky): running prefix over k <= kx
            const int kx = t & 3, ky = t >> 2;
            const double cyx = 0.5 * (s0y[ky] + s1y[ky]);
            double acc = 0.0;
            for (int k = 0; k <= kx; ++k) acc -= fx * (s1x[k] - s0x[k]) * cyx;
            jx[(bi + kx) * e1 + bj + ky] += acc;
        } else if (t < 40) {  // Jy(kx, ky): running prefix over k <= ky
            const int u = t - 20, ky = u & 3, kx = u >> 2;
            const double cxy = 0.5 * (s0x[kx] + s1x[kx]);
            double acc = 0.0;
            for (int k = 0; k <= ky; ++k) acc -= fy * (s1y[k] - s0y[k]) * cxy;
            jy[(bi + kx) * e1 + bj + ky] += acc;
        } else if (t < 65 && fz != 0.0) {  // Jz(kx, ky)
            const int u = t - 40, kx = u % 5, ky = u / 5;
            const double sy0 = s0y[ky], sy1 = s1y[ky];
            const double za = fz * (sy0 * third + sy1 * sixth), zb = fz * (sy0 * sixth + sy1 * third);
            jz[(bi + kx) * e1 + bj + ky] += s0x[kx] * za + s1x[kx] * zb;
        }
        __syncthreads();
    }
}

// kernels.py:269-298 in the reference's order (one CTA, 9 nodes per particle, particle after particle)
__global__ void k_rho2d_ordered(const double *x, const double *y, const double *w, int64_t s0, int64_t s1,
                                double *rho, int64_t e1, double charge, double inv_dx, double inv_dy, int64_t cell0x,
                                int64_t cell0y) {
    const int t = threadIdx.x;
    for (int64_t n = s0; n < s1; ++n) {
        if (t < 9) {
            const double xn = x[n] * inv_dx, yn = y[n] * inv_dy;
            const int64_t ip = (int64_t)(xn + 0.5), jp = (int64_t)(yn + 0.5);
            double wx[3], wy[3];
            spline3(xn - ip, wx[0], wx[1], wx[2]);
            spline3(yn - jp, wy[0], wy[1], wy[2]);
            const double qw = charge * w[n];
            const int u = t / 3, v = t - 3 * u;
            const int64_t a = ip - cell0x + G, b = jp - cell0y + G;
            rho[(a - 1 + u) * e1 + (b - 1 + v)] += qw * wx[u] * wy[v];
        }
        __syncthreads();
    }
}

__global__ void k_reduce_subgrid(double *sub, int64_t n, int64_t e1, int64_t *acc, int64_t x_shift) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    double v = sub[t];
    int64_t i = t / e1, j = t % e1;
    acc[(x_shift + i) * e1 + j] += __double2ll_rn(v * J_SCALE);  // np.rint (fields.py:108-114)
    sub[t] = 0.0;
}

__global__ void k_bad_to_index(unsigned long long *bad) {
    // ~0ull (none) -> -1, like the reference's sentinel
    if (*bad == ~0ull) *bad = (unsigned long long)(-1ll);
}

inline unsigned nblk(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

extern "C" {

int b200pic_gather_fields_2d(const double *x, const double *y, int64_t s0, int64_t s1,
                             const double *const fields[6], int64_t e1, int64_t *cix, int64_t *ciy, double *dlx,
                             double *dly, double *const gathered[6], double inv_dx, double inv_dy, int64_t cell0x,
                             int64_t cell0y, void *stream) {
    if (s1 <= s0) return B200PIC_OK;
    F6 f;
    O6 o;
    for (int c = 0; c < 6; ++c) { f.p[c] = fields[c]; o.p[c] = gathered[c]; }
    // the array's row count is not passed by the reference signature; bound the x stencil loosely
    k_gather2d<<<nblk(s1 - s0, 128), 128, 0, (cudaStream_t)stream>>>(
        x, y, s0, s1, f, e1, cix, ciy, dlx, dly, o, inv_dx, inv_dy, cell0x - G, cell0y - G, INT64_MAX / 4, e1 - 1);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

int b200pic_boris_push(double *x, double *y, double *z, double *px, double *py, double *pz, int64_t s0, int64_t s1,
                       const double *const gathered[6], double charge, double mass, double dt, int64_t *bad_dev,
                       void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    CUDA_TRY(cudaMemsetAsync(bad_dev, 0xff, sizeof(int64_t), s));
    if (s1 > s0) {
        F6 g;
        for (int c = 0; c < 6; ++c) g.p[c] = gathered[c];
        double qd2 = charge * dt * 0.5, inv_m2 = 1.0 / (mass * mass);  // kernels.py:131-132
        k_push<<<nblk(s1 - s0, 128), 128, 0, s>>>(x, y, z, px, py, pz, s0, s1, g, qd2, inv_m2, mass, dt,
                                                   (unsigned long long *)bad_dev);
        LAUNCH_CHECK();
    }
    k_bad_to_index<<<1, 1, 0, s>>>((unsigned long long *)bad_dev);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

int b200pic_flag_boundaries(const double *x, const double *y, const double *z, int64_t s0, int64_t s1,
                            uint8_t *flags, const double *bounds, void *stream) {
    if (s1 <= s0) return B200PIC_OK;
    double b4 = z ? bounds[4] : 0.0, b5 = z ? bounds[5] : 0.0;
    k_flag<<<nblk(s1 - s0, 256), 256, 0, (cudaStream_t)stream>>>(x, y, z, s0, s1, flags, bounds[0], bounds[1],
                                                                   bounds[2], bounds[3], b4, b5);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

int b200pic_esirkepov_project_2d(const double *x, const double *y, const double *px, const double *py,
                                 const double *pz, const double *weight, int64_t s0, int64_t s1, const int64_t *cix,
                                 const int64_t *ciy, const double *dlx, const double *dly, double *jx, double *jy,
                                 double *jz, int64_t e1, double charge, double mass, double inv_dx, double inv_dy,
                                 double dx_over_dt, double dy_over_dt, int64_t sub_cell0x, int64_t sub_cell0y,
                                 int64_t *bad_dev, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    CUDA_TRY(cudaMemsetAsync(bad_dev, 0xff, sizeof(int64_t), s));
    if (s1 > s0) {
        k_project2d_ordered<<<1, 96, 0, s>>>(x, y, px, py, pz, weight, s0, s1, cix, ciy, dlx, dly, jx, jy, jz, e1,
                                             charge, mass, inv_dx, inv_dy, dx_over_dt, dy_over_dt, sub_cell0x,
                                             sub_cell0y, (unsigned long long *)bad_dev);
        LAUNCH_CHECK();
    }
    k_bad_to_index<<<1, 1, 0, s>>>((unsigned long long *)bad_dev);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

int b200pic_deposit_rho_2d(const double *x, const double *y, const double *weight, int64_t s0, int64_t s1,
                           double *rho, int64_t e1, double charge, double inv_dx, double inv_dy, int64_t cell0x,
                           int64_t cell0y, void *stream) {
    if (s1 <= s0) return B200PIC_OK;
    k_rho2d_ordered<<<1, 32, 0, (cudaStream_t)stream>>>(x, y, weight, s0, s1, rho, e1, charge, inv_dx, inv_dy, cell0x,
                                                        cell0y);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

int b200pic_reduce_subgrid(double *sub, int64_t sub_rows, int64_t e1, int64_t *acc, int64_t x_shift, void *stream) {
    int64_t n = sub_rows * e1;
    if (n <= 0) return B200PIC_OK;
    k_reduce_subgrid<<<nblk(n, 256), 256, 0, (cudaStream_t)stream>>>(sub, n, e1, acc, x_shift);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

}  // extern "C"
