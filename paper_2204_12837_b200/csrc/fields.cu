// fields.cu -- K2 (Yee), K3 (J ghost fold), K4 (E/B ghost pull) on
// whole-domain arrays with 3 ghost layers.
//
// The reference keeps one ghosted array per patch and exchanges ghosts
// between patch objects (exchange.py:64-156); on one GPU the patches are
// index ranges of a single array, so only the domain-edge ghosts remain:
//   K3 folds edge-ghost J into its periodic/mirror owner (integer adds,
//      exactly sum_current_ghosts' result), x sweep then y then z;
//   K4 pulls E/B edge ghosts from owners with the PEC sign rule
//      (_pull_axis, exchange.py:99-123), x then y then z;
//   K2 is maxwell_step (fields.py:130-190) with ghosts refreshed between the
//      sub-steps ("synced Yee"); full-E also converts the
//      int64 accumulators to float J (fields.py:77-81) and clears them.
// Stencil expressions keep the reference's op order (-fmad=false build).
#include <stdlib.h>

#include "fields.cuh"

namespace {

struct Geo {
    int64_t e[3];    // array extents
    int64_t st[3];   // strides
};

__host__ __device__ inline Geo geo(const b200pic_config &c) {
    Geo g;
    for (int a = 0; a < 3; ++a) g.e[a] = ext_of(c, a);
    g.st[2] = 1;
    g.st[1] = zpitch(c);
    g.st[0] = g.e[1] * g.st[1];
    return g;
}

// number of non-owned indices along axis a for component comp
__host__ __device__ inline int64_t n_halo(const b200pic_config &c, int comp, int a) {
    return ext_of(c, a) - (owned_hi(c, comp, a) - G);
}
// k-th non-owned index along axis a: [0, G) then [hi, ext)
__device__ inline int64_t halo_index(const b200pic_config &c, int comp, int a, int64_t k) {
    return k < G ? k : owned_hi(c, comp, a) + (k - G);
}

struct Ptrs9 {
    double *f[9];
    int64_t *acc[3];
};

// fold (acc) or pull (fields) along one axis for up to 6 components at once
template <bool FOLD>
__global__ void k_halo_axis(b200pic_config c, Ptrs9 P, int comp0, int ncomp, int a) {
    Geo g = geo(c);
    const int b0 = a == 0 ? 1 : 0, b1 = a == 2 ? 1 : 2;  // the two other axes
    const int64_t n_other = g.e[b0] * g.e[b1];
    for (int ci = 0; ci < ncomp; ++ci) {
        const int comp = comp0 + ci;
        const int64_t nh = n_halo(c, comp, a);
        const int64_t total = nh * n_other;
        const int dual = dual_of(c.dim, comp, a);
        // 32-bit index split (halo sets stay far below 2^32 elements); for the z axis (the contiguous
        // one) the halo index runs fastest so that neighbouring threads touch neighbouring doubles
        const uint32_t nh32 = (uint32_t)nh, e1_32 = (uint32_t)g.e[b1], no32 = (uint32_t)n_other;
        for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
             t += (int64_t)gridDim.x * blockDim.x) {
            const uint32_t tt = (uint32_t)t;
            uint32_t k32, r32;
            if (a == 2) {
                r32 = tt / nh32;
                k32 = tt - r32 * nh32;
            } else {
                k32 = tt / no32;
                r32 = tt - k32 * no32;
            }
            const uint32_t i1_32 = r32 / e1_32;
            const int64_t k = k32, i1 = i1_32, i2 = r32 - i1_32 * e1_32;
            int64_t h = halo_index(c, comp, a, k);
            int sign;
            const int64_t wo = ghost_owner(h - G, c.L[a], c.bc[a], dual, FOLD, &sign);
            int64_t w = wo + G;
            int64_t base = i1 * g.st[b0] + i2 * g.st[b1];
            int64_t src = base + h * g.st[a], dst = base + w * g.st[a];
            if (FOLD) {
                int64_t *acc = P.acc[comp - C_JX];
                int64_t v = acc[src];
                if (v) {
                    // absorbing wall: current deposited beyond the wall leaves the domain
                    if (wo >= 0) atomicAdd((unsigned long long *)(acc + dst), (unsigned long long)(sign > 0 ? v : -v));
                    acc[src] = 0;
                }
            } else {
                double *f = P.f[comp];
                f[src] = sign * f[dst];  // dst is the owner here
            }
        }
    }
}

// fields.py:146-155 (2D) / 3D generalisation; all three B components
// x range [ilo, ihi) in array indices; xfree: every x plane of the range is updated (an x-slab's
// redundant halo update, maxwell_slab), else only owned x nodes
template <int DIM>
__global__ void k_half_b(b200pic_config c, Ptrs9 P, double hx, double hy, double hz, int ilo, int ihi, int xfree) {
    Geo g = geo(c);
    double *ex = P.f[0], *ey = P.f[1], *ez = P.f[2], *bx = P.f[3], *by = P.f[4], *bz = P.f[5];
    const int64_t sx = g.st[0], sy = g.st[1], sz = g.st[2];
    const int64_t n0 = ihi - ilo, n1 = c.L[1] + 1, n2 = DIM == 3 ? c.L[2] + 1 : 1;
    const int64_t total = n0 * n1 * n2;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        // (32-bit index split: grids stay below 2^31 nodes, and 64-bit division is a long subroutine)
        const uint32_t tt = (uint32_t)t, plane = (uint32_t)(n1 * n2);
        const uint32_t i32 = tt / plane, r32 = tt - i32 * plane, j32 = r32 / (uint32_t)n2;
        int64_t i = i32, j = j32, k = r32 - j32 * (uint32_t)n2;
        i += ilo; j += G; k += DIM == 3 ? G : 0;
        const int64_t q = i * sx + j * sy + k * sz;
        auto own = [&](int comp) {
            return (xfree || i < owned_hi(c, comp, 0)) && j < owned_hi(c, comp, 1) && (DIM == 2 || k < owned_hi(c, comp, 2));
        };
        if (DIM == 2) {
            if (own(C_BX)) bx[q] -= hy * (ez[q + sy] - ez[q]);
            if (own(C_BY)) by[q] += hx * (ez[q + sx] - ez[q]);
            if (own(C_BZ)) bz[q] -= hx * (ey[q + sx] - ey[q]) - hy * (ex[q + sy] - ex[q]);
        } else {
            if (own(C_BX)) bx[q] -= hy * (ez[q + sy] - ez[q]) - hz * (ey[q + sz] - ey[q]);
            if (own(C_BY)) by[q] -= hz * (ex[q + sz] - ex[q]) - hx * (ez[q + sx] - ez[q]);
            if (own(C_BZ)) bz[q] -= hx * (ey[q + sx] - ey[q]) - hy * (ex[q + sy] - ex[q]);
        }
    }
}

// fields.py:158-170 (2D) / 3D; J = acc * 2^-44 (fields.py:77-81), acc cleared
template <int DIM>
__global__ void k_full_e(b200pic_config c, Ptrs9 P, double dt, double dtx, double dty, double dtz, int ilo, int ihi,
                         int xfree) {
    Geo g = geo(c);
    double *ex = P.f[0], *ey = P.f[1], *ez = P.f[2], *bx = P.f[3], *by = P.f[4], *bz = P.f[5];
    const int64_t sx = g.st[0], sy = g.st[1], sz = g.st[2];
    const int64_t n0 = ihi - ilo, n1 = c.L[1] + 1, n2 = DIM == 3 ? c.L[2] + 1 : 1;
    const int64_t total = n0 * n1 * n2;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        // (32-bit index split: grids stay below 2^31 nodes, and 64-bit division is a long subroutine)
        const uint32_t tt = (uint32_t)t, plane = (uint32_t)(n1 * n2);
        const uint32_t i32 = tt / plane, r32 = tt - i32 * plane, j32 = r32 / (uint32_t)n2;
        int64_t i = i32, j = j32, k = r32 - j32 * (uint32_t)n2;
        i += ilo; j += G; k += DIM == 3 ? G : 0;
        const int64_t q = i * sx + j * sy + k * sz;
        auto own = [&](int comp) {
            return (xfree || i < owned_hi(c, comp, 0)) && j < owned_hi(c, comp, 1) && (DIM == 2 || k < owned_hi(c, comp, 2));
        };
        double J[3];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
            if (own(C_JX + m)) {
                J[m] = (double)P.acc[m][q] * INV_J_SCALE;
                P.f[6 + m][q] = J[m];
                P.acc[m][q] = 0;
            }
        }
        if (DIM == 2) {
            if (own(C_EX)) ex[q] += dty * (bz[q] - bz[q - sy]) - dt * J[0];
            if (own(C_EY)) ey[q] += -dtx * (bz[q] - bz[q - sx]) - dt * J[1];
            if (own(C_EZ)) ez[q] += dtx * (by[q] - by[q - sx]) - dty * (bx[q] - bx[q - sy]) - dt * J[2];
        } else {
            if (own(C_EX)) ex[q] += dty * (bz[q] - bz[q - sy]) - dtz * (by[q] - by[q - sz]) - dt * J[0];
            if (own(C_EY)) ey[q] += dtz * (bx[q] - bx[q - sz]) - dtx * (bz[q] - bz[q - sx]) - dt * J[1];
            if (own(C_EZ)) ez[q] += dtx * (by[q] - by[q - sx]) - dty * (bx[q] - bx[q - sy]) - dt * J[2];
        }
    }
}

// fields.py:173-190: tangential E and normal B pinned to 0 on reflective walls
__global__ void k_pin(b200pic_config c, Ptrs9 P, int a) {
    Geo g = geo(c);
    const int PIN[3][3] = {{C_EY, C_EZ, C_BX}, {C_EX, C_EZ, C_BY}, {C_EX, C_EY, C_BZ}};
    const int b0 = a == 0 ? 1 : 0, b1 = a == 2 ? 1 : 2;
    const int64_t n_other = g.e[b0] * g.e[b1];
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < 2 * n_other; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t wsel = t / n_other, r = t - wsel * n_other;
        int64_t i1 = r / g.e[b1], i2 = r - i1 * g.e[b1];
        int64_t wi = wsel == 0 ? G : G + c.L[a];
        int64_t q = i1 * g.st[b0] + i2 * g.st[b1] + wi * g.st[a];
        for (int m = 0; m < 3; ++m) P.f[PIN[a][m]][q] = 0.0;
    }
}

// first-order Silver-Mueller wall on absorbing x boundaries (beyond the reference, BASELINE config 1):
// the outgoing-wave condition E + c n x B = 0 at the wall node, with B at the node taken as the mean of
// its two dual neighbours, sets the ghost B half a cell outside:
//   x = 0 (n = -x):  Bz(-1/2) = -2 Ey(0) - Bz(1/2),   By(-1/2) =  2 Ez(0) - By(1/2)
//   x = L (n = +x):  Bz(L+1/2) = 2 Ey(L) - Bz(L-1/2), By(L+1/2) = -2 Ez(L) - By(L-1/2)
__global__ void k_silver_muller_x(b200pic_config c, Ptrs9 P) {
    Geo g = geo(c);
    const int64_t n_other = g.st[0];  // one x plane, z padding included (harmless: padding maps to padding)
    double *ey = P.f[C_EY], *ez = P.f[C_EZ], *by = P.f[C_BY], *bz = P.f[C_BZ];
    const int64_t sx = g.st[0];
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < 2 * n_other;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t side = t / n_other, r = t - side * n_other;
        if (side == 0) {
            const int64_t q0 = G * sx + r;  // node 0 (primal) == dual index of +1/2
            bz[q0 - sx] = -2.0 * ey[q0] - bz[q0];
            by[q0 - sx] = 2.0 * ez[q0] - by[q0];
        } else {
            const int64_t qL = (G + c.L[0]) * sx + r;  // node L; dual L+1/2 has the same index, L-1/2 one less
            bz[qL] = 2.0 * ey[qL] - bz[qL - sx];
            by[qL] = -2.0 * ez[qL] - by[qL - sx];
        }
    }
}

// ---- fused Yee step (K2f; every axis periodic, whole domain): half-B, full-E, half-B in one kernel ----
// One CTA per tile of T owned nodes reads E0 / B0 over the nodes [o - 1, o + T + 2) per axis (the
// sub-steps' dependency cone: B1 needs E0 at n, n + 1; E1 needs B1 at n, n - 1; B2 needs E1 at n, n + 1)
// into shared memory (8-byte cp.async, all in flight), runs the sub-steps there -- B1 on [o - 1, o + T + 1),
// E1 on [o, o + T + 1), B2 on the tile -- recomputing the cone's margin from the same inputs as its owner
// (bit-identical: the stencil expressions and their association order are k_half_b / k_full_e's), and
// writes E, B of the tile into the OTHER field set (a neighbour tile still reads this tile's old values as
// its margin) and float J.  The J accumulators are read, not cleared (a neighbour reads the margin's J):
// the caller clears them after the kernel, refreshes the new set's ghost images and swaps the sets.
// 21 array passes per node (read E0 B0 acc, write E B J, clear acc) against 36 for the three-pass step.
struct Out6 {
    double *f[6];
};
template <int DIM, int TX, int TY, int TZ>
__global__ void __launch_bounds__(256) k_yee_fused(b200pic_config c, Ptrs9 P, Out6 O, double hx, double hy, double hz,
                                                   double dt, double dtx, double dty, double dtz) {
    constexpr int RX = TX + 3, RY = TY + 3, RZ = DIM == 3 ? TZ + 3 : 1;
    constexpr int RN = RX * RY * RZ;
    constexpr int sx = RY * RZ, sy = RZ, sz = 1;
    extern __shared__ double sm[];
    double *ex = sm, *ey = sm + RN, *ez = sm + 2 * RN, *bx = sm + 3 * RN, *by = sm + 4 * RN, *bz = sm + 5 * RN;
    Geo g = geo(c);
    const int64_t L0 = c.L[0], L1 = c.L[1], L2 = DIM == 3 ? c.L[2] : 1;
    const int64_t nty = (L1 + TY - 1) / TY, ntz = DIM == 3 ? (L2 + TZ - 1) / TZ : 1;
    const int64_t b = blockIdx.x;
    const int64_t o0 = (b / (nty * ntz)) * TX, o1 = ((b / ntz) % nty) * TY, o2 = DIM == 3 ? (b % ntz) * TZ : 0;
    // stage nodes [o - 1, o + T + 2) (array index node + G); nodes past the array are never used
    for (int t = threadIdx.x; t < RN; t += blockDim.x) {
        const int u = t / sx, v = (t / sy) % RY, w = t % RZ;
        const int64_t n0 = o0 - 1 + u, n1 = o1 - 1 + v, n2 = DIM == 3 ? o2 - 1 + w : -G;
        if (n0 > L0 + G || n1 > L1 + G || (DIM == 3 && n2 > L2 + G)) continue;
        const int64_t q = (n0 + G) * g.st[0] + (n1 + G) * g.st[1] + (n2 + G) * g.st[2];
#pragma unroll
        for (int k = 0; k < 6; ++k)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(sm + k * RN + t)),
                         "l"(P.f[k] + q)
                         : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // B1 on local [0, T + 2) (fields.py:146-155 / k_half_b)
    constexpr int AX = TX + 2, AY = TY + 2, AZ = DIM == 3 ? TZ + 2 : 1;
    for (int t = threadIdx.x; t < AX * AY * AZ; t += blockDim.x) {
        const int u = t / (AY * AZ), v = (t / AZ) % AY, w = t % AZ;
        const int q = u * sx + v * sy + w * sz;
        if (DIM == 2) {
            bx[q] -= hy * (ez[q + sy] - ez[q]);
            by[q] += hx * (ez[q + sx] - ez[q]);
            bz[q] -= hx * (ey[q + sx] - ey[q]) - hy * (ex[q + sy] - ex[q]);
        } else {
            bx[q] -= hy * (ez[q + sy] - ez[q]) - hz * (ey[q + sz] - ey[q]);
            by[q] -= hz * (ex[q + sz] - ex[q]) - hx * (ez[q + sx] - ez[q]);
            bz[q] -= hx * (ey[q + sx] - ey[q]) - hy * (ex[q + sy] - ex[q]);
        }
    }
    __syncthreads();
    // E1 on local [1, T + 2) (fields.py:158-170 / k_full_e); J of a margin node past L is its periodic image's
    constexpr int FX = TX + 1, FY = TY + 1, FZ = DIM == 3 ? TZ + 1 : 1;
    for (int t = threadIdx.x; t < FX * FY * FZ; t += blockDim.x) {
        const int u = 1 + t / (FY * FZ), v = 1 + (t / FZ) % FY, w = (DIM == 3 ? 1 : 0) + t % FZ;
        const int64_t n0 = o0 - 1 + u, n1 = o1 - 1 + v, n2 = DIM == 3 ? o2 - 1 + w : -G;
        if (n0 > L0 || n1 > L1 || (DIM == 3 && n2 > L2)) continue;
        const int64_t m0 = n0 >= L0 ? n0 - L0 : n0, m1 = n1 >= L1 ? n1 - L1 : n1, m2 = DIM == 3 && n2 >= L2 ? n2 - L2 : n2;
        const int64_t gj = (m0 + G) * g.st[0] + (m1 + G) * g.st[1] + (m2 + G) * g.st[2];
        const double J0 = (double)P.acc[0][gj] * INV_J_SCALE, J1 = (double)P.acc[1][gj] * INV_J_SCALE,
                     J2 = (double)P.acc[2][gj] * INV_J_SCALE;
        const int q = u * sx + v * sy + w * sz;
        if (DIM == 2) {
            ex[q] += dty * (bz[q] - bz[q - sy]) - dt * J0;
            ey[q] += -dtx * (bz[q] - bz[q - sx]) - dt * J1;
            ez[q] += dtx * (by[q] - by[q - sx]) - dty * (bx[q] - bx[q - sy]) - dt * J2;
        } else {
            ex[q] += dty * (bz[q] - bz[q - sy]) - dtz * (by[q] - by[q - sz]) - dt * J0;
            ey[q] += dtz * (bx[q] - bx[q - sz]) - dtx * (bz[q] - bz[q - sx]) - dt * J1;
            ez[q] += dtx * (by[q] - by[q - sx]) - dty * (bx[q] - bx[q - sy]) - dt * J2;
        }
        if (u <= TX && v <= TY && (DIM == 2 || w <= TZ) && n0 < L0 && n1 < L1 && (DIM == 2 || n2 < L2)) {
            P.f[6][gj] = J0;  // float J of the owned nodes (fields.py:77-81)
            P.f[7][gj] = J1;
            P.f[8][gj] = J2;
        }
    }
    __syncthreads();
    // B2 on the tile; E and B of the tile into the other field set
    constexpr int OZ = DIM == 3 ? TZ : 1;
    for (int t = threadIdx.x; t < TX * TY * OZ; t += blockDim.x) {
        const int u = 1 + t / (TY * OZ), v = 1 + (t / OZ) % TY, w = (DIM == 3 ? 1 : 0) + t % OZ;
        const int64_t n0 = o0 - 1 + u, n1 = o1 - 1 + v, n2 = DIM == 3 ? o2 - 1 + w : -G;
        if (n0 >= L0 || n1 >= L1 || (DIM == 3 && n2 >= L2)) continue;
        const int q = u * sx + v * sy + w * sz;
        double b0, b1, b2;
        if (DIM == 2) {
            b0 = bx[q] - hy * (ez[q + sy] - ez[q]);
            b1 = by[q] + hx * (ez[q + sx] - ez[q]);
            b2 = bz[q] - (hx * (ey[q + sx] - ey[q]) - hy * (ex[q + sy] - ex[q]));
        } else {
            b0 = bx[q] - (hy * (ez[q + sy] - ez[q]) - hz * (ey[q + sz] - ey[q]));
            b1 = by[q] - (hz * (ex[q + sz] - ex[q]) - hx * (ez[q + sx] - ez[q]));
            b2 = bz[q] - (hx * (ey[q + sx] - ey[q]) - hy * (ex[q + sy] - ex[q]));
        }
        const int64_t gq = (n0 + G) * g.st[0] + (n1 + G) * g.st[1] + (n2 + G) * g.st[2];
        O.f[0][gq] = ex[q];
        O.f[1][gq] = ey[q];
        O.f[2][gq] = ez[q];
        O.f[3][gq] = b0;
        O.f[4][gq] = b1;
        O.f[5][gq] = b2;
    }
}

// ---- lagged-ghost compatibility (maxwell_step as shipped, fields.py:130-143 + scheduler.py:478-484) ----
// Every reference patch steps its own ghosted array whose ghosts were filled by the last
// sync_field_ghosts, so a sub-step reads a neighbour's node as it was at the start of the step.  On the
// whole-domain arrays: a read node that lies in the updating patch's owned slice of its component
// (owned_slices, fields.py:117-127) comes from the live array, any other node (a neighbour patch's node,
// or a domain-edge ghost) from the snapshot S taken before the step.
// patch coordinate along axis a owning node n of a component (dual: staggered along a); -1: a ghost
__device__ inline int64_t node_patch(const b200pic_config &c, int a, int64_t n, int dual) {
    if (n < 0) return -1;
    if (n < c.L[a]) return n / c.pn[a];
    if (n == c.L[a] && !dual && c.bc[a] != B200PIC_BC_PERIODIC) return c.np[a] - 1;  // the wall node
    return -1;
}
struct Snap6 {
    const double *f[6];
};
template <int DIM>
struct LagReader {
    const b200pic_config &c;
    const Ptrs9 &P;
    const Snap6 &S;
    int64_t node[3];  // the updated node (0-based node indices)
    int64_t pc[3];    // its patch
    __device__ LagReader(const b200pic_config &c_, const Ptrs9 &P_, const Snap6 &S_, int comp, int64_t i, int64_t j,
                         int64_t k)
        : c(c_), P(P_), S(S_) {
        node[0] = i - G;
        node[1] = j - G;
        node[2] = DIM == 3 ? k - G : 0;
        for (int a = 0; a < 3; ++a) pc[a] = a < DIM ? node_patch(c, a, node[a], dual_of(DIM, comp, a)) : 0;
    }
    // component comp at the updated node + off along axis a (off 0: the node itself), array index q
    __device__ double operator()(int comp, int64_t q, int a, int off) const {
        bool own = true;
        for (int b = 0; b < DIM; ++b) {
            const int64_t n = node[b] + (b == a ? off : 0);
            own = own && node_patch(c, b, n, dual_of(DIM, comp, b)) == pc[b];
        }
        return own ? P.f[comp][q] : S.f[comp][q];
    }
};

template <int DIM>
__global__ void k_half_b_lag(b200pic_config c, Ptrs9 P, Snap6 S, double hx, double hy, double hz) {
    Geo g = geo(c);
    const int64_t sx = g.st[0], sy = g.st[1], sz = g.st[2];
    const int64_t n0 = c.L[0] + 1, n1 = c.L[1] + 1, n2 = DIM == 3 ? c.L[2] + 1 : 1;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n0 * n1 * n2; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / (n1 * n2) + G, j = (t / n2) % n1 + G, k = t % n2 + (DIM == 3 ? G : 0);
        const int64_t q = i * sx + j * sy + k * sz;
        auto own = [&](int comp) {
            return i < owned_hi(c, comp, 0) && j < owned_hi(c, comp, 1) && (DIM == 2 || k < owned_hi(c, comp, 2));
        };
        if (own(C_BX)) {
            LagReader<DIM> r(c, P, S, C_BX, i, j, k);
            if (DIM == 2) P.f[C_BX][q] -= hy * (r(C_EZ, q + sy, 1, 1) - r(C_EZ, q, 1, 0));
            else P.f[C_BX][q] -= hy * (r(C_EZ, q + sy, 1, 1) - r(C_EZ, q, 1, 0)) - hz * (r(C_EY, q + sz, 2, 1) - r(C_EY, q, 2, 0));
        }
        if (own(C_BY)) {
            LagReader<DIM> r(c, P, S, C_BY, i, j, k);
            if (DIM == 2) P.f[C_BY][q] += hx * (r(C_EZ, q + sx, 0, 1) - r(C_EZ, q, 0, 0));
            else P.f[C_BY][q] -= hz * (r(C_EX, q + sz, 2, 1) - r(C_EX, q, 2, 0)) - hx * (r(C_EZ, q + sx, 0, 1) - r(C_EZ, q, 0, 0));
        }
        if (own(C_BZ)) {
            LagReader<DIM> r(c, P, S, C_BZ, i, j, k);
            P.f[C_BZ][q] -= hx * (r(C_EY, q + sx, 0, 1) - r(C_EY, q, 0, 0)) - hy * (r(C_EX, q + sy, 1, 1) - r(C_EX, q, 1, 0));
        }
    }
}

template <int DIM>
__global__ void k_full_e_lag(b200pic_config c, Ptrs9 P, Snap6 S, double dt, double dtx, double dty, double dtz) {
    Geo g = geo(c);
    const int64_t sx = g.st[0], sy = g.st[1], sz = g.st[2];
    const int64_t n0 = c.L[0] + 1, n1 = c.L[1] + 1, n2 = DIM == 3 ? c.L[2] + 1 : 1;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n0 * n1 * n2; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / (n1 * n2) + G, j = (t / n2) % n1 + G, k = t % n2 + (DIM == 3 ? G : 0);
        const int64_t q = i * sx + j * sy + k * sz;
        auto own = [&](int comp) {
            return i < owned_hi(c, comp, 0) && j < owned_hi(c, comp, 1) && (DIM == 2 || k < owned_hi(c, comp, 2));
        };
        double J[3];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
            if (own(C_JX + m)) {
                J[m] = (double)P.acc[m][q] * INV_J_SCALE;
                P.f[6 + m][q] = J[m];
                P.acc[m][q] = 0;
            }
        }
        if (own(C_EX)) {
            LagReader<DIM> r(c, P, S, C_EX, i, j, k);
            if (DIM == 2) P.f[C_EX][q] += dty * (r(C_BZ, q, 1, 0) - r(C_BZ, q - sy, 1, -1)) - dt * J[0];
            else P.f[C_EX][q] += dty * (r(C_BZ, q, 1, 0) - r(C_BZ, q - sy, 1, -1)) - dtz * (r(C_BY, q, 2, 0) - r(C_BY, q - sz, 2, -1)) - dt * J[0];
        }
        if (own(C_EY)) {
            LagReader<DIM> r(c, P, S, C_EY, i, j, k);
            if (DIM == 2) P.f[C_EY][q] += -dtx * (r(C_BZ, q, 0, 0) - r(C_BZ, q - sx, 0, -1)) - dt * J[1];
            else P.f[C_EY][q] += dtz * (r(C_BX, q, 2, 0) - r(C_BX, q - sz, 2, -1)) - dtx * (r(C_BZ, q, 0, 0) - r(C_BZ, q - sx, 0, -1)) - dt * J[1];
        }
        if (own(C_EZ)) {
            LagReader<DIM> r(c, P, S, C_EZ, i, j, k);
            P.f[C_EZ][q] += dtx * (r(C_BY, q, 0, 0) - r(C_BY, q - sx, 0, -1)) - dty * (r(C_BX, q, 1, 0) - r(C_BX, q - sy, 1, -1)) - dt * J[2];
        }
    }
}

int grid_of(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return (int)b;
}

Ptrs9 ptrs(const b200pic_state &st) {
    Ptrs9 P;
    for (int k = 0; k < 6; ++k) P.f[k] = st.f.e[k];
    for (int k = 0; k < 3; ++k) {
        P.f[6 + k] = st.f.j[k];
        P.acc[k] = st.f.jacc[k];
    }
    return P;
}

int halo_sweeps(const b200pic_state &st, bool fold, int comp0, int ncomp, int axis_mask, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    Geo g = geo(c);
    Ptrs9 P = ptrs(st);
    for (int a = 0; a < c.dim; ++a) {
        if (!(axis_mask & (1 << a))) continue;
        int64_t n_other = (a == 0 ? g.e[1] * g.e[2] : a == 1 ? g.e[0] * g.e[2] : g.e[0] * g.e[1]);
        int64_t n = (G + 4) * n_other;
        if (n >= (1ll << 32)) return B200PIC_ERR_ARG;  // k_halo_axis splits indices in 32 bits
        if (fold) k_halo_axis<true><<<grid_of(n), 256, 0, s>>>(c, P, comp0, ncomp, a);
        else k_halo_axis<false><<<grid_of(n), 256, 0, s>>>(c, P, comp0, ncomp, a);
        LAUNCH_CHECK();
    }
    return B200PIC_OK;
}

}  // namespace

// in an x-slab the x ghosts belong to the neighbour ranks: the host exchanges them first
static int local_axes(const b200pic_config &c) { return c.slab ? 6 : 7; }

int fold_currents(const b200pic_state &st, cudaStream_t s) {
    return halo_sweeps(st, true, C_JX, 3, local_axes(st.cfg), s);
}

int sync_fields(const b200pic_state &st, int comp0, int ncomp, cudaStream_t s) {
    return halo_sweeps(st, false, comp0, ncomp, local_axes(st.cfg), s);
}

int sync_axes(const b200pic_state &st, int comp0, int ncomp, int axis_mask, cudaStream_t s) {
    return halo_sweeps(st, false, comp0, ncomp, axis_mask, s);
}

int fold_axes(const b200pic_state &st, int axis_mask, cudaStream_t s) {
    return halo_sweeps(st, true, C_JX, 3, axis_mask, s);
}

static int half_b_range(const b200pic_state &st, int ilo, int ihi, int xfree, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    Ptrs9 P = ptrs(st);
    const double dt = c.dt;
    const double hx = 0.5 * dt / c.d[0], hy = 0.5 * dt / c.d[1], hz = c.dim == 3 ? 0.5 * dt / c.d[2] : 0.0;
    const int64_t n = (int64_t)(ihi - ilo) * (c.L[1] + 1) * (c.dim == 3 ? c.L[2] + 1 : 1);
    if (n >= (1ll << 31)) return B200PIC_ERR_ARG;  // the stencil kernels split indices in 32 bits
    if (c.dim == 2) k_half_b<2><<<grid_of(n), 256, 0, s>>>(c, P, hx, hy, hz, ilo, ihi, xfree);
    else k_half_b<3><<<grid_of(n), 256, 0, s>>>(c, P, hx, hy, hz, ilo, ihi, xfree);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

static int full_e_range(const b200pic_state &st, int ilo, int ihi, int xfree, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    Ptrs9 P = ptrs(st);
    const double dt = c.dt;
    const double dtx = dt / c.d[0], dty = dt / c.d[1], dtz = c.dim == 3 ? dt / c.d[2] : 0.0;
    const int64_t n = (int64_t)(ihi - ilo) * (c.L[1] + 1) * (c.dim == 3 ? c.L[2] + 1 : 1);
    if (n >= (1ll << 31)) return B200PIC_ERR_ARG;  // the stencil kernels split indices in 32 bits
    if (c.dim == 2) k_full_e<2><<<grid_of(n), 256, 0, s>>>(c, P, dt, dtx, dty, dtz, ilo, ihi, xfree);
    else k_full_e<3><<<grid_of(n), 256, 0, s>>>(c, P, dt, dtx, dty, dtz, ilo, ihi, xfree);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

int yee_half_b(const b200pic_state &st, cudaStream_t s) { return half_b_range(st, G, G + st.cfg.L[0] + 1, 0, s); }

int yee_full_e(const b200pic_state &st, cudaStream_t s) { return full_e_range(st, G, G + st.cfg.L[0] + 1, 0, s); }

// One Yee step of an x-slab with a single x exchange per step: the sub-steps also run on the x ghost
// planes (redundantly with the neighbours, from the same inputs -- bit-identical values): with E / B
// valid on all 2G + L + 1 planes at the start (the end-of-step refresh) and J summed on every plane
// (b200pic_xplanes_unpack of the J planes), B_half on [0, L+6), E_full on [1, L+6) and B_half on
// [1, L+5) leave E / B valid on [1, L+5] / [1, L+4] -- every plane K1 reads ([2, L+4]) -- and the x
// ghosts are refreshed once afterwards, beside the next step's K1 (slab.py).  y / z ghosts: local sweeps.
int maxwell_slab(const b200pic_state &st, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    if (!c.slab || c.L[0] < 2 * G + 1) return B200PIC_ERR_ARG;
    const int L = c.L[0];
    int rc;
    if ((rc = half_b_range(st, 0, L + 2 * G, 1, s))) return rc;
    if ((rc = sync_axes(st, C_BX, 3, 6, s))) return rc;
    if ((rc = full_e_range(st, 1, L + 2 * G, 1, s))) return rc;
    // accumulator planes the conversion did not visit: cleared for the next K1
    const int64_t plane = ext_of(c, 1) * zpitch(c);
    for (int k = 0; k < 3; ++k) {
        CUDA_TRY(cudaMemsetAsync(st.f.jacc[k], 0, plane * sizeof(int64_t), s));
        CUDA_TRY(cudaMemsetAsync(st.f.jacc[k] + (int64_t)(L + 2 * G) * plane, 0, plane * sizeof(int64_t), s));
    }
    if ((rc = sync_axes(st, C_EX, 3, 6, s))) return rc;
    if ((rc = half_b_range(st, 1, L + 2 * G - 1, 1, s))) return rc;
    bool walls = false;
    for (int a = 1; a < c.dim; ++a) walls = walls || c.bc[a] == B200PIC_BC_REFLECTIVE;
    if (walls && (rc = yee_pin_walls(st, s))) return rc;
    return walls ? sync_axes(st, C_EX, 6, 6, s) : sync_axes(st, C_BX, 3, 6, s);
}

int yee_pin_walls(const b200pic_state &st, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    Ptrs9 P = ptrs(st);
    Geo g = geo(c);
    for (int a = 0; a < c.dim; ++a) {
        if (c.bc[a] != B200PIC_BC_REFLECTIVE || (a == 0 && c.slab)) continue;
        int64_t n_other = (a == 0 ? g.e[1] * g.e[2] : a == 1 ? g.e[0] * g.e[2] : g.e[0] * g.e[1]);
        k_pin<<<grid_of(2 * n_other), 256, 0, s>>>(c, P, a);
        LAUNCH_CHECK();
    }
    return B200PIC_OK;
}

int silver_muller(const b200pic_state &st, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    if (c.bc[0] != B200PIC_BC_ABSORBING || c.slab) return B200PIC_OK;
    Geo g = geo(c);
    k_silver_muller_x<<<grid_of(2 * g.e[1] * g.e[2]), 256, 0, s>>>(c, ptrs(st));
    LAUNCH_CHECK();
    return B200PIC_OK;
}

// ---------------------------------------------------------------------------
// x planes of an x-slab's exchanges (whole planes are contiguous: x is the slowest axis)
//   which 0, J accumulators (int64): planes [0, 2G+1) go left, [L, L+2G+1) go right; on receipt they are
//     added to the same planes, so both sides of a face hold the full sum on all 2G+1 shared planes
//     (exchange.py:64-96 with the redundant halo update of maxwell_slab);
//   which 1, E / B (double), all ghosts: owned planes [G, 2G+1) go left (its right ghosts [L+G, L+2G+1)),
//     owned [L, L+G) go right (its left ghosts [0, G)); copied on receipt (exchange.py:99-123);
//   which 2, E / B, the planes maxwell_slab leaves stale: [G+2, G+4) go left (its ghosts [L+5, L+7)),
//     [L, L+1) goes right (its ghost 0) -- planes K1 never reads, so this exchange may overlap it.
// Message: the components' plane blocks back to back, 2G+1 planes each (E / B: G+1 / 2 planes each).
// ---------------------------------------------------------------------------
namespace {
struct Dst3 {
    int64_t *p[3];
};
__global__ void k_add_planes3(Dst3 dst, const int64_t *src, int64_t block) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < 3 * block; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / block, r = t - k * block;
        dst.p[k][r] += src[t];
    }
}
}  // namespace

size_t xplanes_bytes(const b200pic_config &c, int which) {
    const int64_t plane = ext_of(c, 1) * zpitch(c);
    if (which == 0) return (size_t)3 * (2 * G + 1) * plane * sizeof(int64_t);
    return (size_t)6 * (which == 1 ? G + 1 : 2) * plane * sizeof(double);
}

int xplanes_pack(const b200pic_state &st, int which, void *to_left, void *to_right, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    if (!c.slab || c.L[0] < 2 * G + 1) return B200PIC_ERR_ARG;
    const int64_t plane = ext_of(c, 1) * zpitch(c), L = c.L[0];
    if (which == 0) {
        const int64_t blk = (2 * G + 1) * plane;
        for (int k = 0; k < 3; ++k) {
            CUDA_TRY(cudaMemcpyAsync((int64_t *)to_left + k * blk, st.f.jacc[k], blk * 8, cudaMemcpyDeviceToDevice, s));
            CUDA_TRY(cudaMemcpyAsync((int64_t *)to_right + k * blk, st.f.jacc[k] + L * plane, blk * 8,
                                     cudaMemcpyDeviceToDevice, s));
        }
    } else {
        const int64_t np = which == 1 ? G + 1 : 2, blk = np * plane;
        const int64_t l0 = which == 1 ? G : G + 2, nr = which == 1 ? G : 1;
        for (int k = 0; k < 6; ++k) {
            CUDA_TRY(cudaMemcpyAsync((double *)to_left + k * blk, st.f.e[k] + l0 * plane, blk * 8,
                                     cudaMemcpyDeviceToDevice, s));
            CUDA_TRY(cudaMemcpyAsync((double *)to_right + k * blk, st.f.e[k] + L * plane, nr * plane * 8,
                                     cudaMemcpyDeviceToDevice, s));
        }
    }
    return B200PIC_OK;
}

int xplanes_unpack(const b200pic_state &st, int which, const void *from_left, const void *from_right, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    if (!c.slab || c.L[0] < 2 * G + 1) return B200PIC_ERR_ARG;
    const int64_t plane = ext_of(c, 1) * zpitch(c), L = c.L[0];
    if (which == 0) {
        const int64_t blk = (2 * G + 1) * plane;
        Dst3 lo, hi;
        for (int k = 0; k < 3; ++k) {
            lo.p[k] = st.f.jacc[k];
            hi.p[k] = st.f.jacc[k] + L * plane;
        }
        k_add_planes3<<<grid_of(3 * blk), 256, 0, s>>>(lo, (const int64_t *)from_left, blk);
        LAUNCH_CHECK();
        k_add_planes3<<<grid_of(3 * blk), 256, 0, s>>>(hi, (const int64_t *)from_right, blk);
        LAUNCH_CHECK();
    } else {
        const int64_t np = which == 1 ? G + 1 : 2, blk = np * plane;
        const int64_t nl = which == 1 ? G : 1, r0 = which == 1 ? L + G : L + G + 2;
        for (int k = 0; k < 6; ++k) {
            // left ghosts [0, nl) <- the left neighbour's owned planes it sends to the right
            CUDA_TRY(cudaMemcpyAsync(st.f.e[k], (const double *)from_left + k * blk, nl * plane * 8,
                                     cudaMemcpyDeviceToDevice, s));
            // right ghosts [r0, L + 2G + 1) <- the right neighbour's owned planes it sends to the left
            CUDA_TRY(cudaMemcpyAsync(st.f.e[k] + r0 * plane, (const double *)from_right + k * blk, np * plane * 8,
                                     cudaMemcpyDeviceToDevice, s));
        }
    }
    return B200PIC_OK;
}

// maxwell_step as shipped (the lagged-ghost compatibility mode): snapshot, three sub-steps reading
// non-owned nodes from the snapshot, wall pins, one ghost refresh (scheduler.py:478-484).  The reference's
// boundary kinds only (periodic / reflective), whole domain only.
int maxwell_lagged(const b200pic_state &st, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    if (c.slab) return B200PIC_ERR_ARG;
    for (int a = 0; a < c.dim; ++a)
        if (c.bc[a] == B200PIC_BC_ABSORBING) return B200PIC_ERR_ARG;
    const int64_t n = field_elems(c);
    const int64_t nodes = (int64_t)(c.L[0] + 1) * (c.L[1] + 1) * (c.dim == 3 ? c.L[2] + 1 : 1);
    double *snap = nullptr;
    CUDA_TRY(cudaMallocAsync((void **)&snap, 6 * n * sizeof(double), s));
    Snap6 S;
    for (int k = 0; k < 6; ++k) {
        CUDA_TRY(cudaMemcpyAsync(snap + k * n, st.f.e[k], n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        S.f[k] = snap + k * n;
    }
    Ptrs9 P = ptrs(st);
    const double dt = c.dt;
    const double hx = 0.5 * dt / c.d[0], hy = 0.5 * dt / c.d[1], hz = c.dim == 3 ? 0.5 * dt / c.d[2] : 0.0;
    const double dtx = dt / c.d[0], dty = dt / c.d[1], dtz = c.dim == 3 ? dt / c.d[2] : 0.0;
    for (int sub = 0; sub < 3; ++sub) {
        if (c.dim == 2) {
            if (sub == 1) k_full_e_lag<2><<<grid_of(nodes), 256, 0, s>>>(c, P, S, dt, dtx, dty, dtz);
            else k_half_b_lag<2><<<grid_of(nodes), 256, 0, s>>>(c, P, S, hx, hy, hz);
        } else {
            if (sub == 1) k_full_e_lag<3><<<grid_of(nodes), 256, 0, s>>>(c, P, S, dt, dtx, dty, dtz);
            else k_half_b_lag<3><<<grid_of(nodes), 256, 0, s>>>(c, P, S, hx, hy, hz);
        }
        LAUNCH_CHECK();
    }
    CUDA_TRY(cudaFreeAsync(snap, s));
    int rc;
    if ((rc = yee_pin_walls(st, s))) return rc;
    return sync_fields(st, C_EX, 6, s);
}

template <int DIM, int TX, int TY, int TZ>
static int yee_fused(b200pic_state &st, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    constexpr int RN = (TX + 3) * (TY + 3) * (DIM == 3 ? TZ + 3 : 1);
    constexpr int smem = 6 * RN * (int)sizeof(double);
    static bool attr = false;  // per instantiation; the value is a constant
    if (!attr) {
        CUDA_TRY(cudaFuncSetAttribute(k_yee_fused<DIM, TX, TY, TZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    const int64_t tiles = ((c.L[0] + TX - 1) / TX) * ((c.L[1] + TY - 1) / TY) * (DIM == 3 ? (c.L[2] + TZ - 1) / TZ : 1);
    const double dt = c.dt;
    const double hx = 0.5 * dt / c.d[0], hy = 0.5 * dt / c.d[1], hz = DIM == 3 ? 0.5 * dt / c.d[2] : 0.0;
    const double dtx = dt / c.d[0], dty = dt / c.d[1], dtz = DIM == 3 ? dt / c.d[2] : 0.0;
    Out6 O;
    for (int k = 0; k < 6; ++k) O.f[k] = st.f.e_alt[k];
    k_yee_fused<DIM, TX, TY, TZ><<<(unsigned)tiles, 256, smem, s>>>(c, ptrs(st), O, hx, hy, hz, dt, dtx, dty, dtz);
    LAUNCH_CHECK();
    const int64_t n = field_elems(c);
    for (int k = 0; k < 3; ++k) CUDA_TRY(cudaMemsetAsync(st.f.jacc[k], 0, n * sizeof(int64_t), s));
    for (int k = 0; k < 6; ++k) {  // the new set becomes the current fields
        double *t = st.f.e[k];
        st.f.e[k] = st.f.e_alt[k];
        st.f.e_alt[k] = t;
    }
    return sync_fields(st, C_EX, 6, s);  // periodic ghost images of the new E and B
}

// the fused step applies: every axis periodic, whole domain, a second field set bound
bool yee_fused_applies(const b200pic_state &st) {
    const b200pic_config &c = st.cfg;
    if (c.slab || getenv("B200PIC_YEE_3PASS")) return false;  // (the env switch: A/B and tests)
    for (int a = 0; a < c.dim; ++a)
        if (c.bc[a] != B200PIC_BC_PERIODIC) return false;
    for (int k = 0; k < 6; ++k)
        if (!st.f.e_alt[k]) return false;
    return true;
}

int maxwell(b200pic_state &st, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    if (c.slab) return B200PIC_ERR_ARG;  // x ghosts need the neighbour exchange between sub-steps
    if (yee_fused_applies(st)) return c.dim == 3 ? yee_fused<3, 8, 8, 8>(st, s) : yee_fused<2, 16, 32, 1>(st, s);
    int rc;
    if ((rc = yee_half_b(st, s))) return rc;
    if ((rc = sync_fields(st, C_BX, 3, s))) return rc;
    if ((rc = silver_muller(st, s))) return rc;  // after the pull: it owns the first ghost layer
    if ((rc = yee_full_e(st, s))) return rc;
    if ((rc = sync_fields(st, C_EX, 3, s))) return rc;
    if ((rc = yee_half_b(st, s))) return rc;
    bool walls = false;
    for (int a = 0; a < c.dim; ++a) walls = walls || c.bc[a] == B200PIC_BC_REFLECTIVE;
    if (walls && (rc = yee_pin_walls(st, s))) return rc;
    // final ghost refresh: B always; E only if walls changed owned E values
    rc = walls ? sync_fields(st, C_EX, 6, s) : sync_fields(st, C_BX, 3, s);
    if (rc) return rc;
    return silver_muller(st, s);
}
