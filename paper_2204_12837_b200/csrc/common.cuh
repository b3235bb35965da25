// common.cuh -- shared device helpers for the B200 PIC hot path (sm_100a).
//
// Numerics contract: the library is compiled with -fmad=false so that every
// expression in gather / push / Yee keeps the reference's IEEE op order
// (numba emits no FMA); where contraction is wanted (the
// deposit, which is bounded by the J tolerance) it is written explicitly.
#pragma once
#include <cuda_runtime.h>
#include <string.h>
#include <stdint.h>

#include "../../include/b200pic.h"

#define G 3
#define J_SCALE 17592186044416.0  // 2^44, fields.py:28-30
#define INV_J_SCALE (1.0 / J_SCALE)

enum { FLAG_X_NEG = 1, FLAG_X_POS = 2, FLAG_Y_NEG = 4, FLAG_Y_POS = 8, FLAG_Z_NEG = 16, FLAG_Z_POS = 32 };
enum { C_EX, C_EY, C_EZ, C_BX, C_BY, C_BZ, C_JX, C_JY, C_JZ, C_RHO };

#define CUDA_TRY(x)                                   \
    do {                                              \
        cudaError_t e_ = (x);                         \
        if (e_ != cudaSuccess) return B200PIC_ERR_CUDA; \
    } while (0)
// every kernel launch site ends in LAUNCH_CHECK(), which also counts it
// (b200pic_launch_count(): the bench reports launches inside its timed region)
extern long long g_b200pic_launches;
#define LAUNCH_CHECK()             \
    do {                           \
        ++g_b200pic_launches;      \
        CUDA_TRY(cudaGetLastError()); \
    } while (0)

__host__ __device__ inline int dual_of(int dim, int comp, int axis) {
    // Yee staggering: 2D follows fields.py:33-44 (z collapses to primal)
    const int D[10][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {0, 1, 1}, {1, 0, 1},
                          {1, 1, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {0, 0, 0}};
    if (dim == 2 && axis == 2) return 0;
    return D[comp][axis];
}

__host__ __device__ inline int64_t ext_of(const b200pic_config &c, int a) {
    return a < c.dim ? (int64_t)c.L[a] + 1 + 2 * G : 1;
}

// z pitch of the whole-domain field arrays: the z extent rounded up to an even number of doubles, so that
// every (x, y) row starts 16-byte aligned (the TMA tensor maps of K1's E/B staging need 16-byte strides);
// the padding node is never read as data
__host__ __device__ inline int64_t zpitch(const b200pic_config &c) {
    const int64_t e = ext_of(c, 2);
    return c.dim == 3 ? (e + 1) & ~1ll : 1;
}
__host__ __device__ inline int64_t field_elems(const b200pic_config &c) { return ext_of(c, 0) * ext_of(c, 1) * zpitch(c); }

// exchange.py:23-61: owner node of a global node (+ sign on reflective primal axes)
__host__ __device__ inline int64_t wrap_node(int64_t node, int64_t L, int periodic, int dual, int *sign) {
    *sign = 1;
    if (periodic) {
        int64_t r = node % L;
        return r < 0 ? r + L : r;
    }
    if (dual) {
        if (node < 0) return -node - 1;
        if (node >= L) return 2 * L - node - 1;
        return node;
    }
    if (node < 0) { *sign = -1; return -node; }
    if (node > L) { *sign = -1; return 2 * L - node; }
    return node;
}

// owned index range [G, hi) along an axis (fields.py:117-127); an x-slab owns [G, G + L) (periodic x);
// walls (reflective, absorbing) own the primal wall node L
__host__ __device__ inline int64_t owned_hi(const b200pic_config &c, int comp, int a) {
    if (a >= c.dim) return 1;
    if (a == 0 && c.slab) return G + c.L[0];
    int64_t hi = G + c.L[a];
    if (c.bc[a] != B200PIC_BC_PERIODIC && !dual_of(c.dim, comp, a)) hi += 1;
    return hi;
}

// owner node of a ghost node for the halo sweeps: periodic / reflective as exchange.py:23-61; on an
// absorbing wall the fold drops ghost currents (returns -1) and the pull copies the nearest owned node
__host__ __device__ inline int64_t ghost_owner(int64_t node, int64_t L, int bc, int dual, bool fold, int *sign) {
    if (bc != B200PIC_BC_ABSORBING) return wrap_node(node, L, bc == B200PIC_BC_PERIODIC, dual, sign);
    *sign = 1;
    if (fold) return -1;
    const int64_t hi = dual ? L - 1 : L;
    return node < 0 ? 0 : (node > hi ? hi : node);
}

// global x geometry (an x-slab sees cells [x0, x0 + L[0]) of gL0)
__host__ __device__ inline int64_t slab_x0(const b200pic_config &c) { return c.slab ? c.x0 : 0; }
__host__ __device__ inline int64_t global_L0(const b200pic_config &c) { return c.slab ? c.gL0 : c.L[0]; }
__host__ __device__ inline int64_t global_np0(const b200pic_config &c) { return c.slab ? c.gnp0 : c.np[0]; }

__host__ __device__ inline int64_t n_patches(const b200pic_config &c) {
    return (int64_t)c.np[0] * c.np[1] * (c.dim == 3 ? c.np[2] : 1);
}
__host__ __device__ inline int64_t n_bins(const b200pic_config &c) { return c.pn[0] / c.bx; }
// Sort key = ((patch * n_bins + bin) * anchors_per_bin + anchor): the bin of the
// reference's canonical order (arena.py:59-95) refined by the particle's nearest
// primal node (its Esirkepov stencil anchor, kernels.py:206-207), so that runs of
// same-anchor particles deposit through register accumulation (K1).
__host__ __device__ inline int64_t anchors_per_bin(const b200pic_config &c) {
    return (int64_t)(c.bx + 1) * (c.pn[1] + 1) * (c.dim == 3 ? c.pn[2] + 1 : 1);
}
__host__ __device__ inline int64_t n_bin_keys(const b200pic_config &c) { return n_patches(c) * n_bins(c); }
__host__ __device__ inline int64_t n_keys(const b200pic_config &c) { return n_bin_keys(c) * anchors_per_bin(c); }

// key of a particle at (post-BC) position pos in destination patch dest (arena.py:59-75 + anchor)
// floor(a / b) for 0 <= a < 2^31 without the int64 division subroutine: (a + 1/2) / b is at least
// 1/(2b) away from an integer, far beyond the rounding of the product (inv_b = 1.0 / b)
__host__ __device__ __forceinline__ int64_t fdiv(int64_t a, double inv_b) {
    return (int64_t)((double)a * inv_b + 0.5 * inv_b);
}

// dest: patch coordinates local to the slab; x0: global cell of the slab's first cell
template <int DIM>
__host__ __device__ __forceinline__ int64_t particle_key_t(const b200pic_config &c, const double pos[3],
                                                           const double inv[3], const int64_t dest[3],
                                                           int64_t cx_local, int64_t x0 = 0) {
    const int64_t nb = c.pn[0] / c.bx;
    const int64_t bin = fdiv(cx_local, 1.0 / c.bx);
    const int64_t flat = DIM == 3 ? (dest[0] * c.np[1] + dest[1]) * c.np[2] + dest[2] : dest[0] * c.np[1] + dest[1];
    const int64_t lo[3] = {x0 + dest[0] * c.pn[0] + bin * c.bx, dest[1] * c.pn[1], dest[2] * c.pn[2]};
    const int64_t ext[3] = {c.bx, c.pn[1], c.pn[2]};
    int64_t an[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        int64_t v = (int64_t)(pos[a] * inv[a] + 0.5) - lo[a];
        an[a] = v < 0 ? 0 : (v > ext[a] ? ext[a] : v);
    }
    const int64_t anchor = DIM == 3 ? (an[0] * (c.pn[1] + 1) + an[1]) * (c.pn[2] + 1) + an[2]
                                    : an[0] * (c.pn[1] + 1) + an[1];
    return (flat * nb + bin) * anchors_per_bin(c) + anchor;
}

__host__ __device__ inline int64_t particle_key(const b200pic_config &c, const double pos[3], const double inv[3],
                                                const int64_t dest[3], int64_t cx_local, int64_t x0 = 0) {
    const int64_t nb = c.pn[0] / c.bx;
    const int64_t bin = cx_local / c.bx;
    int64_t flat = c.dim == 3 ? (dest[0] * c.np[1] + dest[1]) * c.np[2] + dest[2] : dest[0] * c.np[1] + dest[1];
    int64_t lo[3] = {x0 + dest[0] * c.pn[0] + bin * c.bx, dest[1] * c.pn[1], dest[2] * c.pn[2]};
    int64_t ext[3] = {c.bx, c.pn[1], c.pn[2]};
    int64_t an[3] = {0, 0, 0};
    for (int a = 0; a < c.dim; ++a) {
        int64_t v = (int64_t)(pos[a] * inv[a] + 0.5) - lo[a];
        an[a] = v < 0 ? 0 : (v > ext[a] ? ext[a] : v);
    }
    int64_t anchor = c.dim == 3 ? (an[0] * (c.pn[1] + 1) + an[1]) * (c.pn[2] + 1) + an[2] : an[0] * (c.pn[1] + 1) + an[1];
    return (flat * nb + bin) * anchors_per_bin(c) + anchor;
}

// order-2 spline weights (kernels.py:40-48); d*d products, no FMA
__device__ __forceinline__ void spline3(double d, double &w0, double &w1, double &w2) {
    double a = 0.5 - d, b = 0.5 + d;
    w0 = 0.5 * (a * a);
    w1 = 0.75 - d * d;
    w2 = 0.5 * (b * b);
}

// sticky error record (device int64[8]): err[0] = bitmask of codes seen,
// err[code] = smallest particle id that raised `code` (INT64_MAX if none)
__device__ __forceinline__ void raise_error(int64_t *err, int code, int64_t id) {
    atomicOr((unsigned long long *)err, 1ull << code);
    atomicMin((long long *)(err + code), (long long)id);
}

template <typename T>
__host__ __device__ inline T ceil_div(T a, T b) { return (a + b - 1) / b; }
