// diag.cu -- K7: device diagnostics (diagnostics.py:30-87) without a host
// round trip: field energy, kinetic energy, charge density and the Gauss
// residual div E - rho.  Reductions: per-block tree, one fp64 atomic per block
// (sums) or an integer atomicMax on the bit pattern of |r| (non-negative
// doubles order like their bit patterns).
#include "fields.cuh"
#include "particle_math.cuh"
#include "sort.cuh"

namespace {

constexpr int DT = 256;

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[DT / 32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < DT / 32 ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    __syncthreads();
    return t;  // valid in thread 0
}

struct Owned {
    int64_t lo[3], n[3], st[3];
};

__host__ __device__ inline Owned owned_box(const b200pic_config &c, int comp) {
    Owned o;
    for (int a = 0; a < 3; ++a) {
        o.lo[a] = a < c.dim ? G : 0;
        o.n[a] = a < c.dim ? owned_hi(c, comp, a) - G : 1;
    }
    o.st[2] = 1;
    o.st[1] = zpitch(c);
    o.st[0] = ext_of(c, 1) * zpitch(c);
    return o;
}

// 0.5 * sum over owned nodes of F^2 (diagnostics.py:60-83)
__global__ void k_field_energy(b200pic_config c, const double *f, int comp, double *out) {
    Owned o = owned_box(c, comp);
    const int64_t total = o.n[0] * o.n[1] * o.n[2];
    double acc = 0.0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / (o.n[1] * o.n[2]), r = t - i * o.n[1] * o.n[2], j = r / o.n[2], k = r - j * o.n[2];
        const double v = f[(i + o.lo[0]) * o.st[0] + (j + o.lo[1]) * o.st[1] + (k + o.lo[2])];
        acc += v * v;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) atomicAdd(out, 0.5 * acc);
}

// mass * sum w (gamma - 1) (diagnostics.py:84-87)
__global__ void k_kinetic(const double *px, const double *py, const double *pz, const double *w, const int64_t *n_dev,
                          const int32_t *perm, double mass, double *out) {
    const int64_t n = *n_dev;
    const double inv_m2 = 1.0 / (mass * mass);
    double acc = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = perm[j];  // live particles are the sorted slots
        const double g = sqrt(1.0 + (px[i] * px[i] + py[i] * py[i] + pz[i] * pz[i]) * inv_m2);
        acc += w[i] * (g - 1.0);
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) atomicAdd(out, mass * acc);
}

// order-2 charge at primal nodes (kernels.py:269-298) into a whole-domain array (ghosts folded below)
template <int DIM>
__global__ void k_rho(b200pic_config c, const double *x, const double *y, const double *z, const double *w,
                      const int64_t *n_dev, const int32_t *perm, double charge, double *rho) {
    const int64_t n = *n_dev;
    const int64_t s1 = ext_of(c, 1) * zpitch(c), s2 = zpitch(c);
    const double inv[3] = {1.0 / c.d[0], 1.0 / c.d[1], DIM == 3 ? 1.0 / c.d[2] : 1.0};
    const int64_t x0 = slab_x0(c);
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = perm[j];
        const double pos[3] = {x[p], y[p], DIM == 3 ? z[p] : 0.0};
        double wt[3][3];
        int64_t ip[3] = {0, 0, 0};
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            const double xn = pos[a] * inv[a];
            ip[a] = (int64_t)(xn + 0.5);
            spline3(xn - ip[a], wt[a][0], wt[a][1], wt[a][2]);
        }
        const double qw = charge * w[p];
        const int64_t a0 = ip[0] - x0 + G, b0 = ip[1] + G, c0 = DIM == 3 ? ip[2] + G : 0;
        for (int u = 0; u < 3; ++u)
            for (int v = 0; v < 3; ++v) {
                if (DIM == 2) {
                    atomicAdd(rho + (a0 - 1 + u) * s1 + (b0 - 1 + v), qw * wt[0][u] * wt[1][v]);
                } else {
                    for (int q = 0; q < 3; ++q)
                        atomicAdd(rho + (a0 - 1 + u) * s1 + (b0 - 1 + v) * s2 + (c0 - 1 + q),
                                  qw * wt[0][u] * wt[1][v] * wt[2][q]);
                }
            }
    }
}

// float ghost fold of rho along one axis (exchange.py:64-96 / fold_grid_ghosts, primal component)
__global__ void k_fold_rho_axis(b200pic_config c, double *rho, int a) {
    const int64_t e[3] = {ext_of(c, 0), ext_of(c, 1), ext_of(c, 2)};
    const int64_t st[3] = {e[1] * zpitch(c), zpitch(c), 1};
    const int b0 = a == 0 ? 1 : 0, b1 = a == 2 ? 1 : 2;
    const int64_t n_other = e[b0] * e[b1];
    const int64_t hi = owned_hi(c, C_RHO, a);
    const int64_t nh = e[a] - (hi - G);
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nh * n_other; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / n_other, r = t - k * n_other;
        const int64_t i1 = r / e[b1], i2 = r - i1 * e[b1];
        const int64_t h = k < G ? k : hi + (k - G);
        int sign;
        const int64_t wo = ghost_owner(h - G, c.L[a], c.bc[a], 0, true, &sign);
        const int64_t base = i1 * st[b0] + i2 * st[b1];
        const double v = rho[base + h * st[a]];
        if (v != 0.0 && wo >= 0) atomicAdd(rho + base + (wo + G) * st[a], sign * v);
        rho[base + h * st[a]] = 0.0;
    }
}

// r = div E - rho at owned primal nodes (backward differences, diagnostics.py:43-57); max |r - r0|
template <int DIM>
__global__ void k_gauss(b200pic_config c, const double *ex, const double *ey, const double *ez, const double *rho,
                        const double *r0, double *r_out, unsigned long long *maxbits) {
    Owned o = owned_box(c, C_RHO);
    const int64_t total = o.n[0] * o.n[1] * o.n[2];
    const double inv[3] = {1.0 / c.d[0], 1.0 / c.d[1], DIM == 3 ? 1.0 / c.d[2] : 1.0};
    unsigned long long m = 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / (o.n[1] * o.n[2]), r = t - i * o.n[1] * o.n[2], j = r / o.n[2], k = r - j * o.n[2];
        const int64_t q = (i + o.lo[0]) * o.st[0] + (j + o.lo[1]) * o.st[1] + (k + o.lo[2]);
        double div = (ex[q] - ex[q - o.st[0]]) * inv[0] + (ey[q] - ey[q - o.st[1]]) * inv[1];
        if (DIM == 3) div += (ez[q] - ez[q - 1]) * inv[2];
        double res = div - rho[q];
        if (r_out) r_out[t] = res;
        if (r0) res -= r0[t];
        const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(res));
        m = bits > m ? bits : m;
    }
    for (int s = 16; s > 0; s >>= 1) {
        unsigned long long o2 = __shfl_xor_sync(0xffffffffu, m, s);
        m = o2 > m ? o2 : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(maxbits, m);
}

int grid_n(int64_t n) {
    int64_t b = (n + DT - 1) / DT;
    return (int)(b < 1 ? 1 : (b > 148 * 8 ? 148 * 8 : b));
}

}  // namespace

extern "C" {

int b200pic_energy(b200pic_state *st, double *out_dev, void *stream) {
    if (!st || !out_dev) return B200PIC_ERR_ARG;
    const b200pic_config &c = st->cfg;
    cudaStream_t s = (cudaStream_t)stream;
    CUDA_TRY(cudaMemsetAsync(out_dev, 0, 2 * sizeof(double), s));
    for (int k = 0; k < 6; ++k) {
        Owned o = owned_box(c, C_EX + k);
        k_field_energy<<<grid_n(o.n[0] * o.n[1] * o.n[2]), DT, 0, s>>>(c, st->f.e[k], C_EX + k, out_dev);
        LAUNCH_CHECK();
    }
    Workspace w = carve(*st);
    for (int i = 0; i < c.n_species; ++i) {
        const b200pic_species &a = st->sp[i];
        k_kinetic<<<grid_n(a.capacity), DT, 0, s>>>(a.px, a.py, a.pz, a.w, a.n_dev, w.perm[i], c.mass[i], out_dev + 1);
        LAUNCH_CHECK();
    }
    return B200PIC_OK;
}

int b200pic_charge_density(b200pic_state *st, double *rho, void *stream) {
    if (!st || !rho) return B200PIC_ERR_ARG;
    const b200pic_config &c = st->cfg;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t tot = ext_of(c, 0) * ext_of(c, 1) * ext_of(c, 2);
    CUDA_TRY(cudaMemsetAsync(rho, 0, field_elems(c) * sizeof(double), s));
    Workspace w = carve(*st);
    for (int i = 0; i < c.n_species; ++i) {
        const b200pic_species &a = st->sp[i];
        if (c.dim == 2)
            k_rho<2><<<grid_n(a.capacity), DT, 0, s>>>(c, a.x, a.y, a.z, a.w, a.n_dev, w.perm[i], c.charge[i], rho);
        else
            k_rho<3><<<grid_n(a.capacity), DT, 0, s>>>(c, a.x, a.y, a.z, a.w, a.n_dev, w.perm[i], c.charge[i], rho);
        LAUNCH_CHECK();
    }
    for (int a = c.slab ? 1 : 0; a < c.dim; ++a) {
        const int64_t n_other = tot / ext_of(c, a);
        k_fold_rho_axis<<<grid_n((G + 4) * n_other), DT, 0, s>>>(c, rho, a);
        LAUNCH_CHECK();
    }
    return B200PIC_OK;
}

int b200pic_gauss_residual(b200pic_state *st, const double *rho, const double *r0, double *r_out,
                           double *max_dev, void *stream) {
    if (!st || !rho || !max_dev) return B200PIC_ERR_ARG;
    const b200pic_config &c = st->cfg;
    cudaStream_t s = (cudaStream_t)stream;
    CUDA_TRY(cudaMemsetAsync(max_dev, 0, sizeof(double), s));
    Owned o = owned_box(c, C_RHO);
    const int g = grid_n(o.n[0] * o.n[1] * o.n[2]);
    if (c.dim == 2)
        k_gauss<2><<<g, DT, 0, s>>>(c, st->f.e[0], st->f.e[1], st->f.e[2], rho, r0, r_out, (unsigned long long *)max_dev);
    else
        k_gauss<3><<<g, DT, 0, s>>>(c, st->f.e[0], st->f.e[1], st->f.e[2], rho, r0, r_out, (unsigned long long *)max_dev);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

}  // extern "C"
