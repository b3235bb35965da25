// k1_particles.cu -- K1: the fused macro-particle kernel.
//
// One persistent kernel replaces the reference's whole particle phase
// (scheduler.py:442-468).  Each CTA pulls work items = (species, patch, bin,
// chunk) from an atomic queue (the device form of the paper's dynamic task
// scheduling: dense bins are split into chunks, idle SMs take the next item)
// and, for its particles:
//   Phase A (lane = particle): interpolate (kernels.py:51-121), Boris push
//     (kernels.py:124-162), pre-BC flags (kernels.py:165-178), Esirkepov
//     shape factors (kernels.py:202-237), then the global BC + destination
//     sort key of the exchange step (exchange.py:163-230, arena.py:59-75);
//   Phase B (lane = stencil column): the projection (kernels.py:238-265)
//     into a shared-memory J tile.  Particles arrive sorted by stencil anchor
//     (nearest primal node), so a lane accumulates its column of a run of
//     same-anchor particles in registers and touches shared memory only when
//     the anchor changes -- lanes of one warp always hit distinct addresses.
// The J tile is 64-bit fixed point at a finer quantum 2^-(44+F) updated with
// native 32-bit shared atomics (lo/hi words + carry); at the end of the item
// it is rounded half-to-even to the reference's 2^-44 grid and added to the
// int64 accumulators (reduce_bin_currents, fields.py:101-114) with global
// atomics.  Integer adds commute, so the tile is order-independent and the
// serialised reduction of the paper's Algorithm 2 is gone.
//
// Variant 1 (cfg.k1_variant = 1) keeps the straightforward per-particle
// shared-memory atomics for A/B comparisons.
#include <cudaTypedefs.h>
#include <stdlib.h>
#include <type_traits>

#include "k1.cuh"
#include "sort.cuh"

namespace {

constexpr int NWARPS = K1_THREADS / 32;

struct TileGeom {
    int64_t o[3];   // global node of tile element 0 per axis
    int T[3];       // tile extent per axis
    int64_t pc[3];  // patch coordinates (x: local to the slab)
    int64_t gpc0;   // global x patch index
    double bd[6];   // patch bounds (domain.py:26-29)
};

template <int DIM>
__device__ __forceinline__ void decode_item(const K1Params &P, int64_t bin_key, TileGeom &g) {
    const b200pic_config &c = P.cfg;
    int64_t nb = c.pn[0] / c.bx;
    int64_t flat = bin_key / nb, bin = bin_key % nb;
    if (DIM == 3) {
        g.pc[2] = flat % c.np[2];
        flat /= c.np[2];
    } else {
        g.pc[2] = 0;
    }
    g.pc[1] = flat % c.np[1];
    g.pc[0] = flat / c.np[1];
    g.gpc0 = g.pc[0] + slab_x0(c) / c.pn[0];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        int64_t cell0 = g.pc[a] * c.pn[a] + (a == 0 ? slab_x0(c) : 0);  // global cell
        g.bd[2 * a] = cell0 * c.d[a];
        g.bd[2 * a + 1] = (cell0 + c.pn[a]) * c.d[a];
        if (a < DIM) {
            int64_t lo = a == 0 ? cell0 + bin * c.bx : cell0;
            int ext = a == 0 ? c.bx : c.pn[a];
            g.o[a] = lo - 2;
            g.T[a] = ext + 5;
        } else {
            g.o[a] = 0;
            g.T[a] = 1;
        }
    }
}

// J tile: 64-bit fixed point (quantum 2^-(44+F)) held as two 32-bit words so that every update is a
// native shared-memory atomic (fp64 shared atomics are CAS loops on sm_100a); the carry out of the low
// word is added to the high word, which keeps the pair an exact 64-bit modular sum
// (branch-free so that the independent updates of one flush pipeline)
__device__ __forceinline__ void tile_add(unsigned *lo, unsigned *hi, int idx, long long iv) {
    const unsigned l = (unsigned)iv;
    const unsigned old = atomicAdd(lo + idx, l);
    const unsigned h = (unsigned)((unsigned long long)iv >> 32) + ((old + l) < old ? 1u : 0u);
    atomicAdd(hi + idx, h);
}

// v (already scaled by 2^(44+F), |v| < 2^51) rounded half-even to an integer: adding 1.5 * 2^52
// puts the integer in the low mantissa bits (ulp 1), exactly (host keeps |v| < 2^51,
// engine.j_fine_bits).  Terms rounded alone sum exactly in int64, in any order.
constexpr double kUnitMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr long long kUnitMagicBits = 0x4338000000000000ll;
__device__ __forceinline__ long long fx_units(double v) {
    return __double_as_longlong(__dadd_rn(v, kUnitMagic)) - kUnitMagicBits;
}
__device__ __forceinline__ long long fma_units(double a, double b) {  // round(a * b), one rounding
    return __double_as_longlong(__fma_rn(a, b, kUnitMagic)) - kUnitMagicBits;
}

// consumer run sums (3D): exact integer units per term (default), or (WS_FP64RUN) a float sum per run in
// tile units, rounded to an integer once at the run's flush (tuning switch)
#ifndef WS_FP64RUN
#define WS_FP64RUN 0
#endif
__device__ __forceinline__ void acc_term(long long &a, double p, double w) { a += fma_units(p, w); }
__device__ __forceinline__ void acc_term(double &a, double p, double w) { a = __fma_rn(p, w, a); }
__device__ __forceinline__ long long acc_units(long long a) { return a; }
__device__ __forceinline__ long long acc_units(double a) { return __double2ll_rn(a); }

// round-half-even of v / 2^F (np.rint semantics, fields.py:108-114, on the fixed-point sum)
__device__ __forceinline__ long long rshift_rne(long long v, int F) {
    if (F == 0) return v;
    const long long q = v >> F;  // floor
    const long long r = v - (q << F);
    const long long half = 1ll << (F - 1);
    return (r > half || (r == half && (q & 1))) ? q + 1 : q;
}

// global BC + destination key (exchange.py:163-230, arena.py:59-75); updates pos/mom.
// In an x-slab, a destination patch outside the slab gets the outgoing key n_keys + 0 (left) / + 1 (right).
template <int DIM>
__device__ __forceinline__ int64_t bc_and_key(const K1Params &P, const TileGeom &g, int fl, double pos[3],
                                              double mom[3], bool &invariant_ok) {
    const b200pic_config &c = P.cfg;
    const int64_t gpc[3] = {g.gpc0, g.pc[1], g.pc[2]};
    const int64_t gnp[3] = {global_np0(c), c.np[1], c.np[2]};
    const int64_t gL[3] = {global_L0(c), c.L[1], c.L[2]};
    int64_t dest[3] = {g.gpc0, g.pc[1], g.pc[2]};  // global patch coordinates
    if (fl) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            const int fneg = 1 << (2 * a), fpos = 2 << (2 * a);
            const bool out_hi = gpc[a] == gnp[a] - 1 && (fl & fpos), out_lo = gpc[a] == 0 && (fl & fneg);
            if (c.bc[a] == B200PIC_BC_ABSORBING && (out_hi || out_lo)) {
                invariant_ok = true;
                return P.n_keys + 2;  // absorbed: dropped by the re-sort
            }
            if (out_hi) {
                if (c.bc[a] == B200PIC_BC_PERIODIC) pos[a] -= P.Lw[a];
                else { pos[a] = fmin(2.0 * P.Lw[a] - pos[a], nextafter(P.Lw[a], 0.0)); mom[a] = -mom[a]; }
            }
            if (out_lo) {
                if (c.bc[a] == B200PIC_BC_PERIODIC) pos[a] += P.Lw[a];
                else { pos[a] = -pos[a]; mom[a] = -mom[a]; }
            }
        }
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            int64_t cell = (int64_t)floor(pos[a] * P.inv[a]);
            cell = cell < 0 ? 0 : (cell > gL[a] - 1 ? gL[a] - 1 : cell);
            dest[a] = fdiv(cell, P.inv_pn[a]);
        }
    }
    const int64_t pslab0 = slab_x0(c) / c.pn[0];
    if (dest[0] < pslab0 || dest[0] >= pslab0 + c.np[0]) {  // leaves the slab (only in slab mode)
        invariant_ok = true;
        return P.n_keys + ((fl & FLAG_X_NEG) ? 0 : 1);
    }
    int64_t cx = (int64_t)floor(pos[0] * P.inv[0]) - dest[0] * c.pn[0];
    invariant_ok = !(cx < 0 || cx > c.pn[0]);
    cx = cx < 0 ? 0 : (cx > c.pn[0] - 1 ? c.pn[0] - 1 : cx);
    const int64_t ldest[3] = {dest[0] - pslab0, dest[1], dest[2]};
    return particle_key_t<DIM>(c, pos, P.inv, ldest, cx, slab_x0(c));
}

// ---------------------------------------------------------------------------
// Phase-B descriptors, AoS in shared memory (one 16-byte aligned record per
// particle, so Phase B reads (s0[k], s1[k]) pairs with one 128-bit load):
// 2D (NF = 30): 0-9 (s0x[k], s1x[k]) pairs, 10-19 (s0y, s1y) pairs,
//     20-23 dX[k] = fx*(s1x-s0x)[k], 24-27 dY[k] = fy*(s1y-s0y)[k], 28 fz
//     (kernels.py:221-265)
// 3D (NF = 42): 10a + 2k: (s0[a][k], s1[a][k]) pairs, 30 + 4a + u: P[a][u] =
//     -f_a * cumsum(s1 - s0)[u]                        (oracle o_project_3d);
//     variant 2 stores z as (A, B) = (s0/3 + s1/6, s0/6 + s1/3) pairs at 20 + 2k
// ---------------------------------------------------------------------------
template <int DIM>
struct Desc {
    static constexpr int NF = DIM == 2 ? 30 : 42;
};

template <int DIM, int VARIANT, bool STAGE>
__global__ void __launch_bounds__(K1_THREADS) k1_fused(const __grid_constant__ K1Params P) {
    extern __shared__ __align__(128) double smem[];
    __shared__ int s_item;
    __shared__ int s_fbits;
    __shared__ double s_fscale;
    if (threadIdx.x == 0) {
        s_fbits = *P.fbits_dev;
        s_fscale = *P.fscale_dev;
    }
    __syncthreads();
    __shared__ int s_anchor[NWARPS][32];  // J-tile flat index of each particle's stencil anchor, -1 = skip
    const b200pic_config &c = P.cfg;
    constexpr bool has_z = DIM == 3;
    constexpr int NF = Desc<DIM>::NF;
    const int64_t e1 = ext_of(c, 1), e2 = zpitch(c);
    const int64_t X0 = slab_x0(c);
    const int n_items = *P.n_items;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int la = lane / 5, lb = lane - 5 * (lane / 5);  // stencil column of this lane (lane < 25)

    for (int round = 0;; ++round) {
        // dynamic: pull the next work item from the queue (the paper's task scheduling, Algorithm 2);
        // static ("tasks off", Algorithm 1 without the shared patch queue): fixed round-robin
        if (threadIdx.x == 0) s_item = c.k1_static ? (int)(blockIdx.x + (int64_t)round * gridDim.x) : atomicAdd(P.queue, 1);
        __syncthreads();
        const int it = s_item;
        if (it >= n_items) break;
        unsigned long long t_begin = 0;
        if (P.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
        const K1Item item = P.items[it];
        TileGeom g;
        decode_item<DIM>(P, item.key, g);
        // J tile: extent n+5 from node cell0-2 (stencil i0-2..i0+2, i0 in [cell0, cell0+n]);
        // E/B tile: extent n+4 from the same origin (primal i0+-1, dual idu-1..idu+1, idu >= cell0-1)
        const int TN = g.T[0] * g.T[1] * g.T[2];
        const int ts1 = g.T[1] * g.T[2], ts2 = g.T[2];
        const int FT[3] = {g.T[0] - 1, DIM >= 2 ? g.T[1] - 1 : 1, DIM == 3 ? g.T[2] - 1 : 1};
        const int FN = FT[0] * FT[1] * FT[2];
        const int fts1 = FT[1] * FT[2], fts2 = FT[2];
        double *sJ = smem;                                                // 3 * TN (as 2 x 3 * TN words)
        unsigned *sJlo = reinterpret_cast<unsigned *>(smem), *sJhi = sJlo + 3 * TN;
        double *sDall = smem + ((3 * TN + 1) & ~1);                       // NWARPS * 32 * NF (16B aligned)
        double *sD = sDall + (VARIANT == 0 ? warp * 32 * NF : 0);
        double *sF = sDall + (VARIANT == 0 ? NWARPS * 32 * NF : 0);       // 6 * FN if STAGE
        // species record: compile-time indices into the parameter block (a runtime index would copy it to the stack)
        K1Species S = P.sp[0];
#pragma unroll
        for (int k = 1; k < B200PIC_MAX_SPECIES; ++k)
            if (item.species == k) S = P.sp[k];
        // warp-contiguous segment of the item (keeps anchor runs inside one warp)
        // (equal shares, not rounded to whole batches: the barrier after Phase B waits for the slowest warp)
        const int64_t seg = ((int64_t)item.count + NWARPS - 1) / NWARPS;
        const int64_t w0 = item.start + warp * seg;
        const int64_t w1 = min(w0 + seg, item.start + (int64_t)item.count);
        // software pipeline: the particle record of the next batch is in flight while the current
        // batch is deposited (and the first one while the E/B tile is staged)
        double nx_ = 0, ny_ = 0, nz_ = 0, npx_ = 0, npy_ = 0, npz_ = 0, nw_ = 0;
        int64_t nid_ = 0;
        // the permutation entry is loaded one batch ahead of the record it addresses, so the
        // record loads never wait on it
        int32_t perm_next = (w0 + lane < w1) ? __ldcs(S.perm + w0 + lane) : 0;
        auto prefetch = [&](int64_t nn) {
            const int32_t m = perm_next;
            if (nn + 32 < w1) perm_next = __ldcs(S.perm + nn + 32);
            if (nn < w1) {
                // gathered through perm: neighbouring slots are read by other lanes / warps soon after,
                // so keep the default (evict-normal) L2 policy for the records
                nx_ = __ldg(S.x + m); ny_ = __ldg(S.y + m); nz_ = has_z ? __ldg(S.z + m) : 0.0;
                npx_ = __ldg(S.px + m); npy_ = __ldg(S.py + m); npz_ = __ldg(S.pz + m); nw_ = __ldg(S.w + m);
                nid_ = __ldg(S.id + m);
            }
        };
        prefetch(w0 + lane);
        // ---- stage E/B tile (optional), zero J tile ----
        if (STAGE) {
            for (int t = threadIdx.x; t < FN; t += blockDim.x) {
                int u = t / fts1, r = t - u * fts1, v = r / fts2, q = r - v * fts2;
                int64_t gi = ((g.o[0] - X0 + u + G) * e1 + (g.o[1] + v + G)) * e2 + (DIM == 3 ? g.o[2] + q + G : 0);
#pragma unroll
                for (int k = 0; k < 6; ++k) sF[k * FN + t] = __ldg(P.e[k] + gi);
            }
        }
        for (int t = threadIdx.x; t < 3 * TN; t += blockDim.x) sJ[t] = 0.0;
        __syncthreads();
        const double qd2 = S.qd2, inv_m2 = S.inv_m2, mass = S.mass, charge = S.charge;
        double ax[4] = {0, 0, 0, 0}, ay[4] = {0, 0, 0, 0}, az[4] = {0, 0, 0, 0};
        int cur_anchor = -1;
        // add this lane's column sums of the finished anchor run to the tile; lanes of a warp
        // always address distinct nodes
        auto flush_run = [&](int anc) {
            if (P.ablate & 1) return;
            const double sc = s_fscale;
            if (DIM == 2) {
                tile_add(sJlo, sJhi, 2 * TN + anc + la * ts1 + lb, __double2ll_rn(az[0] * sc));
                if (la < 4) {
                    tile_add(sJlo, sJhi, anc + la * ts1 + lb, __double2ll_rn(ax[0] * sc));
                    tile_add(sJlo, sJhi, TN + anc + lb * ts1 + la, __double2ll_rn(ay[0] * sc));
                }
            } else {
                // all 12 low-word atomics first (independent round trips in flight), then the
                // carry-propagating high words
                int idx[12];
                long long iv[12];
                unsigned old[12];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    idx[k] = anc + k * ts1 + la * ts2 + lb;
                    idx[4 + k] = TN + anc + la * ts1 + k * ts2 + lb;
                    idx[8 + k] = 2 * TN + anc + la * ts1 + lb * ts2 + k;
                    iv[k] = __double2ll_rn(ax[k] * sc);
                    iv[4 + k] = __double2ll_rn(ay[k] * sc);
                    iv[8 + k] = __double2ll_rn(az[k] * sc);
                }
#pragma unroll
                for (int m = 0; m < 12; ++m) old[m] = atomicAdd(sJlo + idx[m], (unsigned)iv[m]);
#pragma unroll
                for (int m = 0; m < 12; ++m) {
                    const unsigned l = (unsigned)iv[m];
                    atomicAdd(sJhi + idx[m], (unsigned)((unsigned long long)iv[m] >> 32) + ((old[m] + l) < old[m] ? 1u : 0u));
                }
            }
        };
        // 3D z-step: the column sums at z-offset 0 leave the window of the next anchor (az + 1):
        // Jx/Jy columns (.., q = 0) -> lanes lb == 0, Jz value q = 0 of every lane; the rest shifts
        // one z-plane down (Jx/Jy: from lane + 1, Jz: within the lane)
        auto z_step = [&](int anc) {
            if (!(P.ablate & 1) && lane < 25) {
                const double sc = s_fscale;
                if (lb == 0) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        tile_add(sJlo, sJhi, anc + k * ts1 + la * ts2, __double2ll_rn(ax[k] * sc));
                        tile_add(sJlo, sJhi, TN + anc + la * ts1 + k * ts2, __double2ll_rn(ay[k] * sc));
                    }
                }
                tile_add(sJlo, sJhi, 2 * TN + anc + la * ts1 + lb * ts2, __double2ll_rn(az[0] * sc));
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double nx = __shfl_down_sync(0xffffffffu, ax[k], 1);
                const double ny = __shfl_down_sync(0xffffffffu, ay[k], 1);
                ax[k] = (lb == 4 || lane >= 24) ? 0.0 : nx;
                ay[k] = (lb == 4 || lane >= 24) ? 0.0 : ny;
            }
            az[0] = az[1];
            az[1] = az[2];
            az[2] = az[3];
            az[3] = 0.0;
        };

        for (int64_t base = w0; base < w1; base += 32) {
            const int64_t n = base + lane;
            // ================= Phase A: lane = particle =================
            int my_anchor = -1;
            if (n < w1) {
                double x = nx_, y = ny_, z = nz_;
                double px = npx_, py = npy_, pz = npz_;
                const double w = nw_;
                const int64_t pid = nid_;
                // every sorted slot is written (dst is the next step's storage), errors included
                auto store = [&](const double q[3], const double m[3]) {
                    S.dx[n] = q[0];
                    S.dy[n] = q[1];
                    if (has_z) S.dz[n] = q[2];
                    S.dpx[n] = m[0];
                    S.dpy[n] = m[1];
                    S.dpz[n] = m[2];
                    S.dw[n] = w;
                    S.did[n] = pid;
                };
                Gathered gt;
                bool ok;
                if (STAGE) {
                    const double pos[3] = {x, y, z};
                    ok = tile_gather<DIM>(pos, P.inv, sF, FN, FT, g.o, gt);
                } else {
                    const double *fptr[6] = {P.e[0], P.e[1], P.e[2], P.e[3], P.e[4], P.e[5]};
                    const int64_t forg[3] = {X0 - G, DIM >= 2 ? -G : 0, DIM == 3 ? -G : 0};
                    const int64_t flo[3] = {g.o[0] - X0 + G, g.o[1] + G, DIM == 3 ? g.o[2] + G : 0};
                    const int64_t fhi[3] = {flo[0] + FT[0] - 1, flo[1] + FT[1] - 1, DIM == 3 ? flo[2] + FT[2] - 1 : 0};
                    if (DIM == 2)
                        ok = gather2d(x, y, P.inv[0], P.inv[1], fptr, e1, forg[0], forg[1], flo[0], fhi[0], flo[1],
                                      fhi[1], gt);
                    else
                        ok = gather3d(x, y, z, P.inv, fptr, e1 * e2, e2, forg, flo, fhi, gt);
                }
                int64_t key = item.key * P.anchors;
                if (!ok) {
                    raise_error(P.err, B200PIC_ERR_INVARIANT, pid);
                    const double q0[3] = {x, y, z}, m0[3] = {px, py, pz};
                    store(q0, m0);
                } else {
                    double gn;
                    if (!boris(x, y, z, has_z, px, py, pz, gt.e, gt.b, qd2, inv_m2, mass, c.dt, gn))
                        raise_error(P.err, B200PIC_ERR_NONFINITE, pid);
                    const int fl = pre_bc_flags(x, y, z, has_z, g.bd);
                    double s0[3][5], s1[3][5];
                    bool cour = esirkepov_shapes(x * P.inv[0], gt.ip, gt.dxp, s0[0], s1[0]) &&
                                esirkepov_shapes(y * P.inv[1], gt.jp, gt.dyp, s0[1], s1[1]);
                    if (DIM == 3) cour = cour && esirkepov_shapes(z * P.inv[2], gt.kp, gt.dzp, s0[2], s1[2]);
                    const int bi = (int)(gt.ip - 2 - g.o[0]), bj = (int)(gt.jp - 2 - g.o[1]);
                    const int bk = DIM == 3 ? (int)(gt.kp - 2 - g.o[2]) : 0;
                    if (!cour) {
                        raise_error(P.err, B200PIC_ERR_COURANT, pid);
                    } else if (bi < 0 || bi > g.T[0] - 5 || bj < 0 || bj > g.T[1] - 5 ||
                               (DIM == 3 && (bk < 0 || bk > g.T[2] - 5))) {
                        raise_error(P.err, B200PIC_ERR_INVARIANT, pid);
                    } else {
                        const double qw = charge * w;
                        if (VARIANT == 1) {
                            auto add = [&](int cc, int64_t idx, double v) {
                                tile_add(sJlo, sJhi, cc * TN + (int)idx, __double2ll_rn(v * s_fscale));
                            };
                            if (DIM == 2) {
                                const double fz = qw * pz / (gn * mass);  // gam == gn (kernels.py:234-237)
                                esirkepov2d_accumulate(s0[0], s1[0], s0[1], s1[1], qw * P.d_over_dt[0],
                                                       qw * P.d_over_dt[1], fz, bi, bj, ts1, add);
                            } else {
                                esirkepov3d_accumulate(s0, s1, qw * P.d_over_dt[0], qw * P.d_over_dt[1],
                                                       qw * P.d_over_dt[2], bi, bj, bk, ts1, ts2, add);
                            }
                        } else {
                            double *d = sD + lane * NF;
                            if (DIM == 2) {
                                const double fx = qw * P.d_over_dt[0], fy = qw * P.d_over_dt[1];
#pragma unroll
                                for (int k = 0; k < 5; ++k) {
                                    d[2 * k] = s0[0][k];
                                    d[2 * k + 1] = s1[0][k];
                                    d[10 + 2 * k] = s0[1][k];
                                    d[10 + 2 * k + 1] = s1[1][k];
                                }
#pragma unroll
                                for (int k = 0; k < 4; ++k) {
                                    d[20 + k] = fx * (s1[0][k] - s0[0][k]);  // kernels.py:249
                                    d[24 + k] = fy * (s1[1][k] - s0[1][k]);  // kernels.py:264
                                }
                                d[28] = qw * pz / (gn * mass);  // fz (kernels.py:237, gam == gn)
                                my_anchor = bi * ts1 + bj;
                            } else {
#pragma unroll
                                for (int a = 0; a < 3; ++a) {
                                    const double f = qw * P.d_over_dt[a];
                                    double pref = 0.0;
#pragma unroll
                                    for (int k = 0; k < 5; ++k) {
                                        d[10 * a + 2 * k] = s0[a][k];
                                        d[10 * a + 2 * k + 1] = s1[a][k];
                                        if (k < 4) {  // P[u] = -f * cumsum(s1 - s0)[u]
                                            pref -= f * (s1[a][k] - s0[a][k]);
                                            d[30 + 4 * a + k] = pref;
                                        }
                                    }
                                }
                                my_anchor = bi * ts1 + bj * ts2 + bk;
                            }
                        }
                    }
                    double pos[3] = {x, y, z}, mom[3] = {px, py, pz};
                    bool inv_ok;
                    key = bc_and_key<DIM>(P, g, fl, pos, mom, inv_ok);
                    if (!inv_ok) raise_error(P.err, B200PIC_ERR_INVARIANT, pid);
                    store(pos, mom);
                }
                if (key < 0 || key > P.n_keys + 2) {  // only reachable with non-finite positions
                    raise_error(P.err, B200PIC_ERR_INVARIANT, pid);
                    key = item.key * P.anchors;
                }
                S.key[n] = (int32_t)key;
            }
            prefetch(n + 32);
            if (VARIANT == 1 || (P.ablate & 2)) continue;
            // ================= Phase B: lane = stencil column =================
            // Runs of equal anchors (particles are anchor-sorted) are found with one ballot;
            // inside a run there is no per-particle branch, two particles per iteration.
            s_anchor[warp][lane] = my_anchor;
            __syncwarp();
            const int np_ = (int)min((int64_t)32, w1 - base);
            const int prev = __shfl_up_sync(0xffffffffu, my_anchor, 1);
            const unsigned bounds =
                __ballot_sync(0xffffffffu, lane < np_ && (lane == 0 ? my_anchor != cur_anchor : my_anchor != prev));
#pragma unroll 1
            for (int p = 0; p < np_;) {
                const unsigned rest = p >= 31 ? 0u : (bounds & ~((2u << p) - 1u));
                const int q = rest ? __ffs(rest) - 1 : np_;
                const int anc = s_anchor[warp][p];
                if (anc != cur_anchor) {
                    if (DIM == 3 && cur_anchor >= 0 && anc == cur_anchor + 1 && !(P.ablate & 8)) {
                        // z-step of the anchor (keys are z-fastest): slide the register window
                        // instead of flushing it -- only the z-plane that leaves is written out
                        z_step(cur_anchor);
                    } else {
                        // flush the previous run: lanes of the warp hit distinct addresses
                        if (cur_anchor >= 0 && lane < 25) flush_run(cur_anchor);
#pragma unroll
                        for (int k = 0; k < 4; ++k) { ax[k] = 0.0; ay[k] = 0.0; az[k] = 0.0; }
                    }
                    cur_anchor = anc;
                }
                if (anc >= 0 && lane < 25) {
                    if (DIM == 2) {
                        // kernels.py:240-265, one (kx = la, ky = lb) column per lane
#pragma unroll 1
                        for (int r = p; r < q; ++r) {
                            const double *d = sD + r * NF;
                            const double2 xa = *reinterpret_cast<const double2 *>(d + 2 * la);
                            const double2 yb = *reinterpret_cast<const double2 *>(d + 10 + 2 * lb);
                            const double fz = d[28];
                            if (fz != 0.0) {
                                const double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
                                const double za = fz * (yb.x * third + yb.y * sixth);
                                const double zb = fz * (yb.x * sixth + yb.y * third);
                                az[0] += xa.x * za + xa.y * zb;
                            }
                            if (la < 4) {
                                const double2 dx01 = *reinterpret_cast<const double2 *>(d + 20);
                                const double2 dx23 = *reinterpret_cast<const double2 *>(d + 22);
                                const double2 dy01 = *reinterpret_cast<const double2 *>(d + 24);
                                const double2 dy23 = *reinterpret_cast<const double2 *>(d + 26);
                                const double dX[4] = {dx01.x, dx01.y, dx23.x, dx23.y};
                                const double dY[4] = {dy01.x, dy01.y, dy23.x, dy23.y};
                                // Jx(la, lb): running prefix over kx <= la (kernels.py:247-250)
                                const double cyx = 0.5 * (yb.x + yb.y);
                                double acc = 0.0;
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    if (k <= la) acc -= dX[k] * cyx;
                                ax[0] += acc;
                                // Jy(lb, la): running prefix over ky <= la (kernels.py:260-265)
                                const double2 xb = *reinterpret_cast<const double2 *>(d + 2 * lb);
                                const double cxy = 0.5 * (xb.x + xb.y);
                                double accy = 0.0;
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    if (k <= la) accy -= dY[k] * cxy;
                                ay[0] += accy;
                            }
                        }
                    } else {
                        // 3D: w(v,q) = S0(S0'/3 + S1'/6) + S1(S0'/6 + S1'/3), J += P[u] * w (FMA: the
                        // deposit is bounded by the J tolerance, not bit-pinned)
                        const double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
                        auto column = [&](const double *d, double (&cx)[4], double (&cy)[4], double (&cz)[4]) {
                            const double2 xa = *reinterpret_cast<const double2 *>(d + 2 * la);
                            const double2 ya = *reinterpret_cast<const double2 *>(d + 10 + 2 * la);
                            const double2 yb = *reinterpret_cast<const double2 *>(d + 10 + 2 * lb);
                            const double2 zb = *reinterpret_cast<const double2 *>(d + 20 + 2 * lb);
                            const double Az = __fma_rn(zb.y, sixth, zb.x * third), Bz = __fma_rn(zb.y, third, zb.x * sixth);
                            const double Ay = __fma_rn(yb.y, sixth, yb.x * third), By = __fma_rn(yb.y, third, yb.x * sixth);
                            const double wyz = __fma_rn(ya.y, Bz, ya.x * Az);  // Jx column (v = la, q = lb)
                            const double wxz = __fma_rn(xa.y, Bz, xa.x * Az);  // Jy column (u = la, q = lb)
                            const double wxy = __fma_rn(xa.y, By, xa.x * Ay);  // Jz column (u = la, v = lb)
                            const double2 px01 = *reinterpret_cast<const double2 *>(d + 30);
                            const double2 px23 = *reinterpret_cast<const double2 *>(d + 32);
                            const double2 py01 = *reinterpret_cast<const double2 *>(d + 34);
                            const double2 py23 = *reinterpret_cast<const double2 *>(d + 36);
                            const double2 pz01 = *reinterpret_cast<const double2 *>(d + 38);
                            const double2 pz23 = *reinterpret_cast<const double2 *>(d + 40);
                            cx[0] = __fma_rn(px01.x, wyz, cx[0]);
                            cx[1] = __fma_rn(px01.y, wyz, cx[1]);
                            cx[2] = __fma_rn(px23.x, wyz, cx[2]);
                            cx[3] = __fma_rn(px23.y, wyz, cx[3]);
                            cy[0] = __fma_rn(py01.x, wxz, cy[0]);
                            cy[1] = __fma_rn(py01.y, wxz, cy[1]);
                            cy[2] = __fma_rn(py23.x, wxz, cy[2]);
                            cy[3] = __fma_rn(py23.y, wxz, cy[3]);
                            cz[0] = __fma_rn(pz01.x, wxy, cz[0]);
                            cz[1] = __fma_rn(pz01.y, wxy, cz[1]);
                            cz[2] = __fma_rn(pz23.x, wxy, cz[2]);
                            cz[3] = __fma_rn(pz23.y, wxy, cz[3]);
                        };
                        int r = p;
                        if (r + 1 < q) {
                            // second accumulator set for the odd particles: independent FMA chains
                            double bx[4] = {0, 0, 0, 0}, by[4] = {0, 0, 0, 0}, bz[4] = {0, 0, 0, 0};
#pragma unroll 1
                            for (; r + 1 < q; r += 2) {
                                column(sD + r * NF, ax, ay, az);
                                column(sD + (r + 1) * NF, bx, by, bz);
                            }
#pragma unroll
                            for (int k = 0; k < 4; ++k) { ax[k] += bx[k]; ay[k] += by[k]; az[k] += bz[k]; }
                        }
                        if (r < q) column(sD + r * NF, ax, ay, az);
                    }
                }
                p = q;
            }
            __syncwarp();
        }
        if (VARIANT == 0 && cur_anchor >= 0 && lane < 25) flush_run(cur_anchor);
        __syncthreads();
        // ---- flush: rint(tile * 2^44) into the int64 accumulators (fields.py:108-114) ----
        for (int t = threadIdx.x; t < ((P.ablate & 4) ? 0 : TN); t += blockDim.x) {
            int u = t / ts1, r = t - u * ts1, v = r / ts2, q = r - v * ts2;
            int64_t gi = ((g.o[0] - X0 + u + G) * e1 + (g.o[1] + v + G)) * e2 + (DIM == 3 ? g.o[2] + q + G : 0);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const unsigned long long raw =
                    ((unsigned long long)sJhi[k * TN + t] << 32) | (unsigned long long)sJlo[k * TN + t];
                const long long iv = rshift_rne((long long)raw, s_fbits);
                if (iv) atomicAdd((unsigned long long *)(P.jacc[k] + gi), (unsigned long long)iv);
            }
        }
        __syncthreads();
        if (P.trace && threadIdx.x == 0 && it < P.trace_rows) {
            // row (B200PIC_TRACE_WORDS): begin ns, end ns (%globaltimer), SM, CTA, species, key, start, count
            unsigned long long t_end;
            unsigned smid;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            ulonglong2 *row = reinterpret_cast<ulonglong2 *>(P.trace + B200PIC_TRACE_WORDS * (int64_t)it);
            row[0] = make_ulonglong2(t_begin, t_end);  // one role per warp: both phases span the item
            row[1] = make_ulonglong2(t_begin, t_end);
            row[2] = make_ulonglong2(((unsigned long long)smid << 32) | blockIdx.x,
                                     ((unsigned long long)item.species << 32) | (unsigned)item.key);
            row[3] = make_ulonglong2(item.start, item.count);
        }
    }
}

// ===========================================================================
// Variant 2: warp-specialised K1 (512 threads).  Warps 0-7 run Phase A
// (producers), warps 8-15 run Phase B (consumers); producer p and consumer
// 8 + p share segment p of the item and a double-buffered descriptor slot pair
// in shared memory, handed over with mbarriers (full / empty per slot).  Phase
// A of batch k + 1 then overlaps Phase B of batch k on the same SM, and the
// register file is split by setmaxnreg: producers need the wide gather / push /
// shape state, consumers only the column accumulators.
// ===========================================================================
constexpr int WS_THREADS = 512;
constexpr int WS_PAIRS = 8;
#ifndef WS_DECOUPLE
#define WS_DECOUPLE 1  // (with WS_OVERLAP) no CTA barrier at an item's end: producers claim and stage the
                       // next item while the consumers drain the last batches and flush the J tile
#endif
#ifndef WS_PRE_P
#define WS_PRE_P 1  // producers compute the 3D prefix sums before waiting for the slot (tuning switch)
#endif
#ifndef WS_PRE_AB
#define WS_PRE_AB 0  // producers compute the z (A, B) weights before waiting for the slot (tuning switch)
#endif
#ifndef WS_CPASYNC
#define WS_CPASYNC 1  // E/B tile staged with cp.async (all loads of an item in flight at once)
#endif
#ifndef WS_SPARSE_SHIFT
#define WS_SPARSE_SHIFT 8  // registers moved from producers to consumers in sparse plasma (k1_sparse)
#endif
#ifndef WS_LB
#define WS_LB 1  // interleaved items keep the reference's per-species J rounding (species-1 low-bits tile);
                 // 0 (A/B experiments only): one rounding over both species
#endif
// J units of the warp-specialised K1: DEVF = false takes F from the host (a kernel constant: the fast
// path), DEVF = true from this step's device bound (csrc/sort.cu k_jbits); both are launched every step and
// the one that does not apply exits at once (the device flag jsafe says whether the host's F is within
// this step's bound).  Same-box A/B: reading F from shared memory instead of the constant bank costs the
// scheduling of the whole kernel ~7 % (K1 66.6 -> 71.3 ms on config 2).
#define WS_FSCALE (DEVF ? sh.fscale : P.fscale_host)
#define WS_FBITS (DEVF ? sh.fbits : P.fbits_host)
#ifndef WS_LB_DBG
#define WS_LB_DBG 0  // (A/B experiments only) 1: no low-bits atomics
#endif
#ifndef WS_PREG
#define WS_PREG 168  // producer / consumer registers per thread: (168 + 88) * 256 = 65536
#endif
#ifndef WS_CREG
#define WS_CREG 88
#endif
static_assert(WS_PREG + WS_CREG <= 256 && WS_PREG % 8 == 0 && WS_CREG % 8 == 0, "setmaxnreg split");

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity), "n"(1000000)  // suspend-time hint (ns): sleep until the phase completes, don't spin
        : "memory");
}

// role barriers (named barriers 1 / 2): producers are warps 0-7, consumers warps 8-15
__device__ __forceinline__ void bar_producers() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void bar_consumers() { asm volatile("bar.sync 2, 256;" ::: "memory"); }

// ---- TMA (cp.async.bulk.tensor): one elected thread moves a 3D box of a field array into shared memory
// and the bytes land on an mbarrier's transaction count ----
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// ---------------------------------------------------------------------------
// BASELINE geometry (3D, 8^3 patches, bin_x_size 8 -- configs 2, 3, 4): the E/B stencil tile of a
// (patch, bin) item is staged per component at that component's own extent -- along an axis the primal
// nodes i0 - 1 .. i0 + 9 (11), the dual ones i0 - 1 .. i0 + 8 (10) -- as six regular 3D boxes of the
// whole-domain arrays, each one TMA load (csrc/common.cuh zpitch keeps the array rows 16-byte aligned; the
// box's z extent is rounded up to an even count for the same reason).  7,250 doubles instead of the 6 x
// 12^3 of the generic tile: less L2 -> SM traffic per item and room for the species-1 low-bits J tile of
// the interleaved items.  Compile-time extents: every stencil address is a register + immediate.
// ---------------------------------------------------------------------------
namespace g8 {
constexpr int N = 8;
__host__ __device__ constexpr bool dual(int comp, int a) { return comp < 3 ? comp == a : comp - 3 != a; }
__host__ __device__ constexpr int ext(int comp, int a) { return dual(comp, a) ? N + 2 : N + 3; }
__host__ __device__ constexpr int zext(int comp) { return (ext(comp, 2) + 1) & ~1; }
// y extent of a component's box (>= its stencil extent): padded rows move the x-neighbour plane of the
// gather off the same bank pair (Ex: 11 -> 14 rows, By: 11 -> 12; bank-conflict model of sorted particles,
// gather wavefronts x1.12 -> x1.04 at 16 particles per cell, x1.40 -> x1.29 at 4)
#ifndef G8_YPAD
#define G8_YPAD 1
#endif
__host__ __device__ constexpr int yext(int comp) {
    return G8_YPAD ? ext(comp, 1) + (comp == 0 ? 3 : comp == 4 ? 1 : 0) : ext(comp, 1);
}
__host__ __device__ constexpr int s1(int comp) { return yext(comp) * zext(comp); }
__host__ __device__ constexpr int s2(int comp) { return zext(comp); }
__host__ __device__ constexpr int size(int comp) { return ext(comp, 0) * s1(comp); }
__host__ __device__ constexpr int padded(int comp) { return (size(comp) + 15) & ~15; }  // 128-byte aligned tiles
__host__ __device__ constexpr int off(int comp) { return comp == 0 ? 0 : off(comp - 1) + padded(comp - 1); }
constexpr int TOTAL = off(5) + padded(5);  // doubles
__host__ __device__ constexpr unsigned bytes() {
    return 8u * (size(0) + size(1) + size(2) + size(3) + size(4) + size(5));
}
static_assert(TOTAL * 8 < 64 * 1024, "g8 E/B tiles");
}  // namespace g8

__host__ __device__ inline bool g8_geometry(const b200pic_config &c) {
    return c.dim == 3 && c.bx == g8::N && c.pn[0] == g8::N && c.pn[1] == g8::N && c.pn[2] == g8::N;
}

// kernels.py:61-121 (3D restatement) on the per-component tiles; org[a] = global node of element 0 of every
// tile along axis a (the item's first cell - 1).  A particle sits in [lo, lo + N) of its bin, except one
// left exactly on the far edge by a periodic wrap (x + L rounding to L; the reference keeps it in the last
// patch, arena.py:59-75): its dual stencil id - 1 .. id + 1 would reach one node past the tile with weight
// spline3(-1/2)[2] = 0, so it is taken one node lower with the offset + 1 -- the same two nodes, the same
// weights 1/2, 1/2 (a ~1e-28 weight is dropped if x * inv lands a hair above the edge).  false: the
// stencil leaves the tile otherwise (InvariantError, as arena.py:69-73).
__device__ __forceinline__ bool tile_gather8(const double pos[3], const double inv[3], const double *sF,
                                             const int64_t org[3], Gathered &g) {
    int P_[3], D_[3];
    double wp[3][3], wd[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double xn = pos[a] * inv[a];
        const int64_t ip = (int64_t)(xn + 0.5), id = (int64_t)xn;
        const double dp = xn - ip;
        double dd = xn - 0.5 - id;
        const int64_t pa = ip - org[a];
        int64_t da = id - org[a];
        if (da == g8::N + 1) { da = g8::N; dd += 1.0; }
        spline3(dp, wp[a][0], wp[a][1], wp[a][2]);
        spline3(dd, wd[a][0], wd[a][1], wd[a][2]);
        if (pa < 1 || pa > g8::N + 1 || da < 1 || da > g8::N) return false;
        P_[a] = (int)pa;
        D_[a] = (int)da;
        if (a == 0) { g.ip = ip; g.dxp = dp; } else if (a == 1) { g.jp = ip; g.dyp = dp; } else { g.kp = ip; g.dzp = dp; }
    }
#define G8I(k, A, B, C, W0, W1, W2) tinterp3(sF + g8::off(k), g8::s1(k), g8::s2(k), A, B, C, W0, W1, W2)
    g.e[0] = G8I(0, D_[0], P_[1], P_[2], wd[0], wp[1], wp[2]);
    g.e[1] = G8I(1, P_[0], D_[1], P_[2], wp[0], wd[1], wp[2]);
    g.e[2] = G8I(2, P_[0], P_[1], D_[2], wp[0], wp[1], wd[2]);
    g.b[0] = G8I(3, P_[0], D_[1], D_[2], wp[0], wd[1], wd[2]);
    g.b[1] = G8I(4, D_[0], P_[1], D_[2], wd[0], wp[1], wd[2]);
    g.b[2] = G8I(5, D_[0], D_[1], P_[2], wd[0], wd[1], wp[2]);
#undef G8I
    return true;
}

constexpr int K1_SP1 = 1 << 30;  // (interleaved items) anchor flag of species-1 particles
#ifndef WS_JYT
#define WS_JYT 1  // (3D) Jy tile stored [x][z][y]: the 25 lanes of a run flush hit 25 distinct banks
#endif
// 3D run key: the J tile index of the stencil anchor in the [x][y][z] layout of Jx / Jz (bits 0-14) and, with
// WS_JYT, in the [x][z][y] layout of Jy (bits 15-29); tiles stay below 2^15 nodes
constexpr int K1_ANC_BITS = 15, K1_ANC_MASK = (1 << K1_ANC_BITS) - 1;

struct WsShared {
    int item[2];                   // the round's item (ring of two: producers run at most one round ahead)
    unsigned long long item_full;  // (WS_OVERLAP) producer thread 0 published sh.item for the round
    unsigned long long item_read;  // (WS_DECOUPLE) every consumer warp has read the round's sh.item
    unsigned long long tb[2];      // (WS_OVERLAP) claim time of the round's item (trace)
    unsigned long long td[2];      // (WS_DECOUPLE) producer thread 0 done with the round's batches (trace)
    int anchor[WS_PAIRS][2][32];
    unsigned long long full[WS_PAIRS][2], empty[WS_PAIRS][2];
    unsigned long long tma_bar;    // (g8) the round's six E/B boxes have landed
    int n_items;                   // work items of this launch (read once)
    int fbits;                     // this step's J tile fraction bits F and 2^(44 + F) (read once)
    double fscale;
    K1Species spec[2];             // (interleaved items) the two species' records, read per lane
};
static_assert(WS_PAIRS == K1_IL_PAIRS, "interleaved items carry one segment per producer/consumer pair");

// ---- interleaved items (k1_merge 2): a pair's segment is an anchor range of the item, walked anchor by
// anchor with both species' particles of an anchor back to back, so a consumer's anchor run spans both
// species (half the register flushes of a two-species plasma).  Virtual index v in [0, n) of the segment
// -> (species, sorted position) by a binary search over the anchors' merged prefix (global key offsets,
// L1-resident after the first batch; located one batch ahead). ----
struct IlSeg {
    const int64_t *o0, *o1;  // the bin's anchor-key offsets of species 0 / 1
    int a0, a1;              // the pair's anchors [a0, a1) (bin-local)
    int64_t b0, b1, n;       // o0[a0], o1[a0], particles of both species in the segment
};
__device__ __forceinline__ int64_t il_prefix(const IlSeg &g, int a) {
    return (__ldg(g.o0 + a) - g.b0) + (__ldg(g.o1 + a) - g.b1);
}
__device__ __forceinline__ void il_segment(const K1Params &P, const K1Item &it, int item_index, int pair, IlSeg &g) {
    const int64_t kA = (int64_t)it.key * P.anchors;
    g.o0 = P.sp[0].off + kA;
    g.o1 = P.sp[1].off + kA;
    const IlPair q = P.ilp[(int64_t)item_index * K1_IL_PAIRS + pair];
    g.a0 = q.a0;
    g.a1 = pair + 1 < K1_IL_PAIRS ? P.ilp[(int64_t)item_index * K1_IL_PAIRS + pair + 1].a0 : (int)it.start1;
    g.b0 = q.b0;
    g.b1 = q.b1;
    g.n = q.n;
}
__device__ __forceinline__ void il_locate(const IlSeg &g, int64_t v, int &s, int64_t &n) {
    int lo = g.a0, hi = g.a1 - 1;  // last anchor of the segment whose prefix is <= v
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (il_prefix(g, mid) <= v) lo = mid; else hi = mid - 1;
    }
    const int64_t o0 = __ldg(g.o0 + lo), o1 = __ldg(g.o1 + lo);
    const int64_t w = v - ((o0 - g.b0) + (o1 - g.b1));
    const int64_t c1 = __ldg(g.o1 + lo + 1) - o1;  // species 1 first within an anchor (see ws_consumer)
    if (w < c1) { s = 1; n = o1 + w; } else { s = 0; n = o0 + (w - c1); }
}
// warp-cooperative locate of v = base + lane (the 32 consecutive indices of a batch): lane j loads the
// key offsets of anchor cursor + j (one coalesced pair of loads), each lane binary-searches the window's
// merged prefix through shuffles; lanes past the window fall back to il_locate.  cursor: an anchor at or
// before the one holding index base; advanced to the anchor of the batch's last valid index.
__device__ __forceinline__ void il_locate_warp(const IlSeg &g, int64_t base, int lane, int &cursor, int &s,
                                               int64_t &n) {
    const int aj = min(cursor + lane, g.a1);
    const int64_t o0j = __ldg(g.o0 + aj), o1j = __ldg(g.o1 + aj);
    const int64_t pj = cursor + lane <= g.a1 ? (o0j - g.b0) + (o1j - g.b1) : INT64_MAX;  // prefix at anchor aj
    const int64_t v = base + lane;
    int lo = 0, hi = 31;  // largest window index j with prefix(j) <= v (prefix(0) <= base <= v)
#pragma unroll
    for (int it = 0; it < 5; ++it) {
        const int mid = (lo + hi + 1) >> 1;
        const int64_t pm = __shfl_sync(0xffffffffu, pj, mid);
        if (pm <= v) lo = mid; else hi = mid - 1;
    }
    const int64_t o0a = __shfl_sync(0xffffffffu, o0j, lo), o1a = __shfl_sync(0xffffffffu, o1j, lo);
    const int64_t o1b = __shfl_sync(0xffffffffu, o1j, min(lo + 1, 31));
    if (v < g.n) {
        if (lo < 31) {
            const int64_t w = v - ((o0a - g.b0) + (o1a - g.b1));
            const int64_t c1 = o1b - o1a;
            if (w < c1) { s = 1; n = o1a + w; } else { s = 0; n = o0a + (w - c1); }
        } else {
            il_locate(g, v, s, n);
        }
    }
    // the next batch starts at or after the anchor of this batch's last valid index
    const int last = (int)min((int64_t)31, g.n - 1 - base);
    const int lo_last = __shfl_sync(0xffffffffu, lo, last < 0 ? 0 : last);
    cursor = lo_last < 31 ? cursor + lo_last : cursor + 31;
}
// descriptor slots per pair: 2 (double-buffered) when they fit next to the J (and staged E/B) tile,
// else 1 (the producer still overlaps its gather + push with the consumer and waits only to write)
constexpr int WS_SMEM_LIMIT = 227 * 1024 - 4096;  // dynamic shared memory budget (static WsShared aside)

// dynamic shared memory of the warp-specialised K1, offsets in doubles:
//   J tile: 3 TN 64-bit fixed-point words, held as 3 TN low then 3 TN high 32-bit halves;
//   (interleaved items) species-1 low-bits tile: 3 TN 32-bit words, species 1's tile sum mod 2^32;
//   descriptor slots (16-byte aligned);
//   staged E/B tile (g8: the six per-component tiles, 128-byte aligned for TMA)
struct WsLayout {
    int desc, spec, ef;
};
// (one-species items) the species records, read by the producers from shared memory instead of being held
// in registers (a K1Species is 23 words: held per item it pushed the producers into spills)
constexpr int WS_SPEC_D = B200PIC_MAX_SPECIES * (int)(sizeof(K1Species) / sizeof(double));
static_assert(sizeof(K1Species) % sizeof(double) == 0, "K1Species is a whole number of doubles");
__host__ __device__ __forceinline__ WsLayout ws_layout(int TN, int ns, int nf, bool il, bool g8tiles) {
    int after = 3 * TN + (il && WS_LB ? (3 * TN + 1) / 2 : 0);
    WsLayout L;
    L.desc = (after + 1) & ~1;
    L.spec = L.desc + ns * WS_PAIRS * 32 * nf;
    const int end = L.spec + (il ? 0 : WS_SPEC_D);
    L.ef = g8tiles ? (end + 15) & ~15 : end;
    return L;
}

__device__ __forceinline__ K1Species pick_species(const K1Params &P, int s) {
    K1Species S = P.sp[0];
#pragma unroll
    for (int k = 1; k < B200PIC_MAX_SPECIES; ++k)
        if (s == k) S = P.sp[k];
    return S;
}

// item frame shared by both roles: fetch, geometry, E/B staging, J zeroing (ends with a CTA barrier)
__host__ __device__ constexpr int ws_fxs(int dense, int dim) {
    return dim == 3 ? dense + ((8 - dense % 16) + 16) % 16 : dense;
}

struct WsFrame {
    int it;
    K1Item item;
    TileGeom g;
    int TN, ts1, ts2, FN, fts1, fts2, FT[3];
    int fxs;  // x stride of the staged E/B tile: FT1 * FT2 padded to 8 mod 16 doubles (3D), so that
              // particles whose stencils differ by one x plane hit other shared-memory banks
    unsigned long long t_begin;
};

__device__ __forceinline__ int tile_nodes_dev(const b200pic_config &c) {
    return (c.bx + 5) * (c.pn[1] + 5) * (c.dim == 3 ? c.pn[2] + 5 : 1);
}

// ---- WS_OVERLAP frame: the consumers' J-tile flush of item r overlaps the producers' claim and E/B
// staging of item r + 1 (the E/B tile is producer-only, the J tile consumer-only); with WS_DECOUPLE
// (default) there is no CTA barrier at an item's end at all, only role barriers ----
template <int DIM>
__device__ __forceinline__ void ws_geom_only(const K1Params &P, WsFrame &f) {
    decode_item<DIM>(P, f.item.key, f.g);
    f.TN = f.g.T[0] * f.g.T[1] * f.g.T[2];
    f.ts1 = f.g.T[1] * f.g.T[2];
    f.ts2 = f.g.T[2];
    f.FT[0] = f.g.T[0] - 1;
    f.FT[1] = DIM >= 2 ? f.g.T[1] - 1 : 1;
    f.FT[2] = DIM == 3 ? f.g.T[2] - 1 : 1;
    f.fts1 = f.FT[1] * f.FT[2];
    f.fxs = ws_fxs(f.FT[1] * f.FT[2], DIM);
    f.FN = f.FT[0] * f.fxs;
    f.fts2 = f.FT[2];
}

template <int DIM, bool STAGE, int NS, bool IL, bool G8, bool DEVF>
__device__ __forceinline__ bool ws_produce_begin(const K1Params &P, WsShared &sh, double *smem, int round, WsFrame &f) {
    const b200pic_config &c = P.cfg;
    if (threadIdx.x == 0) {
        // (decoupled: the ring slot is free once every consumer warp has read the previous round's item
        // -- producers finished that round's batches, so the consumers are at most there)
        if (WS_DECOUPLE && round >= 1) mbar_wait(&sh.item_read, (round - 1) & 1);
        sh.item[round & 1] = c.k1_static ? (int)(blockIdx.x + (int64_t)round * gridDim.x) : atomicAdd(P.queue, 1);
        unsigned long long t = 0;
        if (P.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        sh.tb[round & 1] = t;
        mbar_arrive(&sh.item_full);
    }
    bar_producers();  // (decoupled: also every producer is done with the previous item's E/B tile)
    f.it = sh.item[round & 1];
    if (f.it >= sh.n_items) return false;
    f.item = P.items[f.it];
    ws_geom_only<DIM>(P, f);
    if (G8) {
        // six TMA boxes, one per component, issued by one thread; every producer waits for the bytes
        double *sF = smem + ws_layout(f.TN, NS, Desc<DIM>::NF, IL, true).ef;
        if (threadIdx.x == 0) {
            const int cz = (int)(f.g.o[2] + 1 + G), cy = (int)(f.g.o[1] + 1 + G);
            const int cx = (int)(f.g.o[0] + 1 - slab_x0(c) + G);
            mbar_expect_tx(&sh.tma_bar, g8::bytes());
#pragma unroll
            for (int k = 0; k < 6; ++k) tma_load_3d(sF + g8::off(k), &P.tmap[k], cz, cy, cx, &sh.tma_bar);
        }
        mbar_wait(&sh.tma_bar, round & 1);
    } else if (STAGE) {
        const int64_t e1 = ext_of(c, 1), e2 = zpitch(c);
        const int64_t X0 = slab_x0(c);
        double *sF = smem + ws_layout(f.TN, NS, Desc<DIM>::NF, IL, false).ef;
        for (int t = threadIdx.x; t < f.FT[0] * f.fts1; t += 256) {
            int u = t / f.fts1, r = t - u * f.fts1, v = r / f.fts2, q = r - v * f.fts2;
            int64_t gi = ((f.g.o[0] - X0 + u + G) * e1 + (f.g.o[1] + v + G)) * e2 + (DIM == 3 ? f.g.o[2] + q + G : 0);
#pragma unroll
            for (int k = 0; k < 6; ++k) {
#if WS_CPASYNC
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sF + k * f.FN + u * f.fxs + r)),
                             "l"(P.e[k] + gi)
                             : "memory");
#else
                sF[k * f.FN + u * f.fxs + r] = __ldg(P.e[k] + gi);
#endif
            }
        }
#if WS_CPASYNC
        asm volatile("cp.async.wait_all;" ::: "memory");
#endif
        bar_producers();
    }
    return true;
}

template <int DIM>
__device__ __forceinline__ bool ws_consume_begin(const K1Params &P, WsShared &sh, int round, WsFrame &f) {
    mbar_wait(&sh.item_full, round & 1);
    f.it = sh.item[round & 1];
    if (WS_DECOUPLE) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&sh.item_read);
    }
    if (f.it >= sh.n_items) return false;
    f.item = P.items[f.it];
    ws_geom_only<DIM>(P, f);
    return true;
}

// rne(T0 / 2^F) + rne(T1 / 2^F) for a tile sum T = T0 + T1 of which only T1 mod 2^32 (l1) is known
// separately: the reference rounds each species' bin subgrid on its own (fields.py:101-114).  Both
// roundings depend only on the low F + 1 bits of T0 and T1, and T - r0 - r1 is an exact multiple of 2^F.
__device__ __forceinline__ long long rne_species_split(long long T, unsigned l1, int F) {
    if (F == 0) return T;
    const unsigned mask = (1u << F) - 1u, half = 1u << (F - 1);
    const unsigned l0 = (unsigned)T - l1;  // T0 mod 2^32
    const unsigned r0 = l0 & mask, r1 = l1 & mask;
    const long long up0 = (r0 > half || (r0 == half && ((l0 >> F) & 1u))) ? 1 : 0;
    const long long up1 = (r1 > half || (r1 == half && ((l1 >> F) & 1u))) ? 1 : 0;
    return ((T - (long long)r0 - (long long)r1) >> F) + up0 + up1;
}

template <int DIM, bool IL, bool DEVF>
__device__ __forceinline__ void ws_consume_end(const K1Params &P, WsShared &sh, double *smem, int round, const WsFrame &f,
                                               unsigned long long t_cbegin, unsigned long long t_done) {
    const b200pic_config &c = P.cfg;
    const int64_t e1 = ext_of(c, 1), e2 = zpitch(c);
    const int64_t X0 = slab_x0(c);
    unsigned *sJlo = reinterpret_cast<unsigned *>(smem), *sJhi = sJlo + 3 * f.TN, *sLB = sJhi + 3 * f.TN;
    const int ct = threadIdx.x - 256;
    for (int t = ct; t < f.TN; t += 256) {
        int u = t / f.ts1, r = t - u * f.ts1, v = r / f.ts2, q = r - v * f.ts2;
        int64_t gi = ((f.g.o[0] - X0 + u + G) * e1 + (f.g.o[1] + v + G)) * e2 + (DIM == 3 ? f.g.o[2] + q + G : 0);
        // (WS_JYT) element t of the Jy tile is node (u, y = r % T1, z = r / T1)
        const int T1 = f.g.T[1];
        const int qy = r / T1, vy = r - qy * T1;
        const int64_t giy = ((f.g.o[0] - X0 + u + G) * e1 + (f.g.o[1] + vy + G)) * e2 + (DIM == 3 ? f.g.o[2] + qy + G : 0);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const unsigned long long raw =
                ((unsigned long long)sJhi[k * f.TN + t] << 32) | (unsigned long long)sJlo[k * f.TN + t];
            sJlo[k * f.TN + t] = 0u;  // zeroed for the next item
            sJhi[k * f.TN + t] = 0u;
            long long iv;
            if (IL && WS_LB) {  // the two species rounded apart, as the reference's per-species reduction
                iv = rne_species_split((long long)raw, sLB[k * f.TN + t], WS_FBITS);
                sLB[k * f.TN + t] = 0u;
            } else {
                iv = rshift_rne((long long)raw, WS_FBITS);
            }
            const int64_t gk = (WS_JYT && DIM == 3 && k == 1) ? giy : gi;
            if (iv && !(P.ablate & 4)) atomicAdd((unsigned long long *)(P.jacc[k] + gk), (unsigned long long)iv);
        }
    }
    bar_consumers();
    if (P.trace && ct == 0 && f.it < P.trace_rows) {
        unsigned long long t_end;
        unsigned smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        ulonglong2 *row = reinterpret_cast<ulonglong2 *>(P.trace + B200PIC_TRACE_WORDS * (int64_t)f.it);
        // producers: claim .. both roles done with the batches; consumers: item start .. tile flushed
        row[0] = make_ulonglong2(sh.tb[round & 1], t_done);
        row[1] = make_ulonglong2(t_cbegin, t_end);
        row[2] = make_ulonglong2(((unsigned long long)smid << 32) | blockIdx.x,
                                 ((unsigned long long)f.item.species << 32) | (unsigned)f.item.key);
        row[3] = make_ulonglong2(f.item.start, (unsigned long long)f.item.count + f.item.count1);
    }
}

// ---- producer: Phase A (lane = particle) ----
template <int DIM, bool STAGE, int NS, bool IL, bool G8, bool DEVF>
__device__ void ws_producer(const K1Params &P, WsShared &sh, double *smem) {
    const b200pic_config &c = P.cfg;
    constexpr bool has_z = DIM == 3;
    constexpr int NF = Desc<DIM>::NF;
    const int64_t e1 = ext_of(c, 1), e2 = zpitch(c);
    const int64_t X0 = slab_x0(c);
    const int lane = threadIdx.x & 31, pair = threadIdx.x >> 5;
    unsigned use = 0;  // batches handed over so far (slot = use & 1, parity = (use >> 1) & 1)
    WsFrame f;
    for (int round = 0; ws_produce_begin<DIM, STAGE, NS, IL, G8, DEVF>(P, sh, smem, round, f); ++round) {
        const TileGeom &g = f.g;
        const WsLayout lay = ws_layout(f.TN, NS, NF, IL, G8);
        double *sDall = smem + lay.desc;
        double *sF = smem + lay.ef;
        int spc = 0;
        int64_t w0 = 0, w1 = 0;
        IlSeg ilg;
        if (IL) {
            il_segment(P, f.item, f.it, pair, ilg);
            w1 = ilg.n;  // virtual indices [0, n) of the segment
        } else {
            item_segment(f.item, pair, WS_PAIRS, spc, w0, w1);
        }
        // (one-species items) the item's species record in shared memory (IL: sh.spec, per lane)
        const K1Species &Sreg = reinterpret_cast<const K1Species *>(smem + lay.spec)[IL ? 0 : spc];
        const double qd2_ = Sreg.qd2, inv_m2_ = Sreg.inv_m2, mass_ = Sreg.mass, charge_ = Sreg.charge;
        double nx_ = 0, ny_ = 0, nz_ = 0, npx_ = 0, npy_ = 0, npz_ = 0, nw_ = 0;
        int64_t nid_ = 0;
        int ns_ = 0;       // (interleaved) this batch: species and sorted position of this lane's particle
        int64_t nn_ = 0;
        int ps_next = 0;   // (interleaved) the same for the batch after, located one batch ahead
        int64_t pn_next = 0;
        int32_t perm_next = 0;
        int il_cursor = IL ? ilg.a0 : 0;
        if (IL) {
            if (w1 > 0) {
                il_locate_warp(ilg, 0, lane, il_cursor, ps_next, pn_next);
                if (lane < w1) perm_next = __ldcs(sh.spec[ps_next].perm + pn_next);
            }
        } else if (w0 + lane < w1) {
            perm_next = __ldcs(Sreg.perm + w0 + lane);
        }
        auto prefetch = [&](int64_t nn) {
            const int32_t m = perm_next;
            if (IL) {
                // records of index nn (located and permuted one batch ago); locate nn + 32 meanwhile
                ns_ = ps_next;
                nn_ = pn_next;
                if (nn + 32 - lane < w1) {  // (warp-uniform: the next batch has particles)
                    il_locate_warp(ilg, nn + 32 - lane, lane, il_cursor, ps_next, pn_next);
                    if (nn + 32 < w1) perm_next = __ldcs(sh.spec[ps_next].perm + pn_next);
                }
                if (nn < w1) {
                    const K1Species *Q = &sh.spec[ns_];
                    nx_ = __ldg(Q->x + m); ny_ = __ldg(Q->y + m); nz_ = has_z ? __ldg(Q->z + m) : 0.0;
                    npx_ = __ldg(Q->px + m); npy_ = __ldg(Q->py + m); npz_ = __ldg(Q->pz + m); nw_ = __ldg(Q->w + m);
                    nid_ = __ldg(Q->id + m);
                }
            } else {
                if (nn + 32 < w1) perm_next = __ldcs(Sreg.perm + nn + 32);
                if (nn < w1) {
                    nx_ = __ldg(Sreg.x + m); ny_ = __ldg(Sreg.y + m); nz_ = has_z ? __ldg(Sreg.z + m) : 0.0;
                    npx_ = __ldg(Sreg.px + m); npy_ = __ldg(Sreg.py + m); npz_ = __ldg(Sreg.pz + m);
                    nw_ = __ldg(Sreg.w + m);
                    nid_ = __ldg(Sreg.id + m);
                }
            }
        };
        prefetch(w0 + lane);
        for (int64_t base = w0; base < w1; base += 32, ++use) {
            const int slot = use % NS;
            const unsigned free_parity = ((use / NS) & 1) ^ 1;
            const int64_t vi = base + lane;      // this lane's index in the segment
            const int64_t n = IL ? nn_ : vi;     // its sorted position (in its species)
            const int ps = ns_;
#define SPF(f) (IL ? sh.spec[ps].f : Sreg.f)  // this lane's species record field
            const double qd2 = IL ? sh.spec[ps].qd2 : qd2_, inv_m2 = IL ? sh.spec[ps].inv_m2 : inv_m2_;
            const double mass = IL ? sh.spec[ps].mass : mass_, charge = IL ? sh.spec[ps].charge : charge_;
            double *d = sDall + ((pair * NS + slot) * 32 + lane) * NF;
            // double-buffered: the slot was read by the consumer two batches ago -- wait up front;
            // single slot: gather and push first, wait just before the descriptor is written
            if (NS == 2) mbar_wait(&sh.empty[pair][slot], free_parity);
            int my_anchor = -1;
            // state carried past the hand-over: the BC, key and particle store run after the consumer
            // already has this batch (they do not feed the deposit)
            bool tail = false;
            double x = nx_, y = ny_, z = nz_;
            double px = npx_, py = npy_, pz = npz_;
            const double w = nw_;
            const int64_t pid = nid_;
            int fl = 0;
            auto store = [&](const double q[3], const double m[3]) {
                SPF(dx)[n] = q[0];
                SPF(dy)[n] = q[1];
                if (has_z) SPF(dz)[n] = q[2];
                SPF(dpx)[n] = m[0];
                SPF(dpy)[n] = m[1];
                SPF(dpz)[n] = m[2];
                SPF(dw)[n] = w;
                SPF(did)[n] = pid;
            };
            if (vi < w1) {
                Gathered gt;
                bool ok;
                if (G8) {
                    const double pos[3] = {x, y, z};
                    const int64_t org[3] = {g.o[0] + 1, g.o[1] + 1, g.o[2] + 1};
                    ok = tile_gather8(pos, P.inv, sF, org, gt);

                } else if (STAGE) {
                    const double pos[3] = {x, y, z};
                    ok = tile_gather<DIM>(pos, P.inv, sF, f.FN, f.FT, g.o, gt, f.fxs);
                } else {
                    const double *fptr[6] = {P.e[0], P.e[1], P.e[2], P.e[3], P.e[4], P.e[5]};
                    const int64_t forg[3] = {X0 - G, DIM >= 2 ? -G : 0, DIM == 3 ? -G : 0};
                    const int64_t flo[3] = {g.o[0] - X0 + G, g.o[1] + G, DIM == 3 ? g.o[2] + G : 0};
                    const int64_t fhi[3] = {flo[0] + f.FT[0] - 1, flo[1] + f.FT[1] - 1, DIM == 3 ? flo[2] + f.FT[2] - 1 : 0};
                    if (DIM == 2)
                        ok = gather2d(x, y, P.inv[0], P.inv[1], fptr, e1, forg[0], forg[1], flo[0], fhi[0], flo[1],
                                      fhi[1], gt);
                    else
                        ok = gather3d(x, y, z, P.inv, fptr, e1 * e2, e2, forg, flo, fhi, gt);
                }
                if (!ok) {
                    raise_error(P.err, B200PIC_ERR_INVARIANT, pid);
                    const double q0[3] = {x, y, z}, m0[3] = {px, py, pz};
                    store(q0, m0);
                    SPF(key)[n] = (int32_t)(f.item.key * P.anchors);
                } else {
                    double gn;
                    if (!boris(x, y, z, has_z, px, py, pz, gt.e, gt.b, qd2, inv_m2, mass, c.dt, gn))
                        raise_error(P.err, B200PIC_ERR_NONFINITE, pid);
                    fl = pre_bc_flags(x, y, z, has_z, g.bd);
                    double s0[3][5], s1[3][5];
                    bool cour = esirkepov_shapes(x * P.inv[0], gt.ip, gt.dxp, s0[0], s1[0]) &&
                                esirkepov_shapes(y * P.inv[1], gt.jp, gt.dyp, s0[1], s1[1]);
                    if (DIM == 3) cour = cour && esirkepov_shapes(z * P.inv[2], gt.kp, gt.dzp, s0[2], s1[2]);
                    const int bi = (int)(gt.ip - 2 - g.o[0]), bj = (int)(gt.jp - 2 - g.o[1]);
                    const int bk = DIM == 3 ? (int)(gt.kp - 2 - g.o[2]) : 0;
                    if (!cour) {
                        raise_error(P.err, B200PIC_ERR_COURANT, pid);
                    } else if (bi < 0 || bi > g.T[0] - 5 || bj < 0 || bj > g.T[1] - 5 ||
                               (DIM == 3 && (bk < 0 || bk > g.T[2] - 5))) {
                        raise_error(P.err, B200PIC_ERR_INVARIANT, pid);
                    } else {
                        const double qw = charge * w;
#if WS_PRE_P
                        // 3D prefix sums computed before the wait for the slot: the consumer idles only
                        // for the stores
                        double pp[3][4];
                        if (DIM == 3) {
#pragma unroll
                            for (int a = 0; a < 3; ++a) {
                                const double fa = (qw * P.d_over_dt[a]) * WS_FSCALE;  // exact: 2^(44+F)
                                pp[a][0] = -(fa * (s1[a][0] - s0[a][0]));
                                pp[a][1] = pp[a][0] - fa * (s1[a][1] - s0[a][1]);
                                pp[a][2] = pp[a][1] - fa * (s1[a][2] - s0[a][2]);
                                pp[a][3] = pp[a][2] - fa * (s1[a][3] - s0[a][3]);
                            }
                        }
#endif
#if WS_PRE_AB
                        double zab[5][2];
                        if (DIM == 3) {
                            const double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
#pragma unroll
                            for (int k = 0; k < 5; ++k) {
                                zab[k][0] = __fma_rn(s1[2][k], sixth, s0[2][k] * third);
                                zab[k][1] = __fma_rn(s1[2][k], third, s0[2][k] * sixth);
                            }
                        }
#endif
                        if (NS == 1) mbar_wait(&sh.empty[pair][slot], free_parity);
                        double2 *d2 = reinterpret_cast<double2 *>(d);  // 128-bit descriptor stores
                        if (DIM == 2) {
                            // pre-scaled to tile units by 2^(44+F) (exact): the consumer rounds each term to a unit
                            const double fx = (qw * P.d_over_dt[0]) * WS_FSCALE, fy = (qw * P.d_over_dt[1]) * WS_FSCALE;
#pragma unroll
                            for (int k = 0; k < 5; ++k) {
                                d2[k] = make_double2(s0[0][k], s1[0][k]);
                                d2[5 + k] = make_double2(s0[1][k], s1[1][k]);
                            }
                            d2[10] = make_double2(fx * (s1[0][0] - s0[0][0]), fx * (s1[0][1] - s0[0][1]));  // kernels.py:249
                            d2[11] = make_double2(fx * (s1[0][2] - s0[0][2]), fx * (s1[0][3] - s0[0][3]));
                            d2[12] = make_double2(fy * (s1[1][0] - s0[1][0]), fy * (s1[1][1] - s0[1][1]));  // kernels.py:264
                            d2[13] = make_double2(fy * (s1[1][2] - s0[1][2]), fy * (s1[1][3] - s0[1][3]));
                            d[28] = (qw * pz / (gn * mass)) * WS_FSCALE;  // fz (kernels.py:237, gam == gn), tile units
                            my_anchor = bi * f.ts1 + bj;
                        } else {
                            // z enters the deposit only through A = S0/3 + S1/6, B = S0/6 + S1/3 (the
                            // consumer's weights): stored instead of (S0, S1), once per particle
                            const double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
#pragma unroll
                            for (int k = 0; k < 5; ++k) {
                                d2[k] = make_double2(s0[0][k], s1[0][k]);
                                d2[5 + k] = make_double2(s0[1][k], s1[1][k]);
#if WS_PRE_AB
                                d2[10 + k] = make_double2(zab[k][0], zab[k][1]);
#else
                                d2[10 + k] = make_double2(__fma_rn(s1[2][k], sixth, s0[2][k] * third),
                                                          __fma_rn(s1[2][k], third, s0[2][k] * sixth));
#endif
                            }
#pragma unroll
                            for (int a = 0; a < 3; ++a) {  // P[u] = -f * cumsum(s1 - s0)[u]
#if WS_PRE_P
                                d2[15 + 2 * a] = make_double2(pp[a][0], pp[a][1]);
                                d2[16 + 2 * a] = make_double2(pp[a][2], pp[a][3]);
#else
                                const double fa = (qw * P.d_over_dt[a]) * WS_FSCALE;  // exact: 2^(44+F)
                                const double p0 = -(fa * (s1[a][0] - s0[a][0]));
                                const double p1 = p0 - fa * (s1[a][1] - s0[a][1]);
                                const double p2 = p1 - fa * (s1[a][2] - s0[a][2]);
                                const double p3 = p2 - fa * (s1[a][3] - s0[a][3]);
                                d2[15 + 2 * a] = make_double2(p0, p1);
                                d2[16 + 2 * a] = make_double2(p2, p3);
#endif
                            }
                            my_anchor = bi * f.ts1 + bj * f.ts2 + bk;
                            if (WS_JYT) my_anchor |= (bi * f.ts1 + bk * g.T[1] + bj) << K1_ANC_BITS;
                        }
                    }
                    tail = true;
                }
            }
            if (NS == 1) mbar_wait(&sh.empty[pair][slot], free_parity);  // (returns at once if waited above)
            // (interleaved) species-1 particles carry the K1_SP1 flag: a species change is a run boundary for
            // the consumers, which round species 1's share of the J tile apart (species-1 low-bits tile)
            sh.anchor[pair][slot][lane] = (IL && WS_LB && ps == 1 && my_anchor >= 0) ? (my_anchor | K1_SP1) : my_anchor;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh.full[pair][slot]);
            if (tail) {  // global BC + destination key (exchange.py:163-230), particle store
                double pos[3] = {x, y, z}, mom[3] = {px, py, pz};
                bool inv_ok;
                int64_t key = bc_and_key<DIM>(P, g, fl, pos, mom, inv_ok);
                if (!inv_ok) raise_error(P.err, B200PIC_ERR_INVARIANT, pid);
                store(pos, mom);
                if (key < 0 || key > P.n_keys + 2) {  // only reachable with non-finite positions
                    raise_error(P.err, B200PIC_ERR_INVARIANT, pid);
                    key = f.item.key * P.anchors;
                }
                SPF(key)[n] = (int32_t)key;
            }
            prefetch(vi + 32);
#undef SPF
        }
        if (WS_DECOUPLE) {
            if (P.trace && threadIdx.x == 0) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                sh.td[round & 1] = t;
            }
        } else {
            __syncthreads();  // item end: both roles done (the consumers flush while the producers move on)
        }
    }
}

// ---- consumer: Phase B (lane = stencil column) ----
template <int DIM, bool STAGE, int NS, bool IL, bool G8, bool DEVF>
__device__ void ws_consumer(const K1Params &P, WsShared &sh, double *smem) {
    constexpr int NF = Desc<DIM>::NF;
    const int lane = threadIdx.x & 31, pair = (threadIdx.x >> 5) - WS_PAIRS;
    const int la = lane / 5, lb = lane - 5 * (lane / 5);
    unsigned use = 0;
    WsFrame f;
    for (int t = threadIdx.x - 256; t < ws_layout(tile_nodes_dev(P.cfg), NS, NF, IL, G8).desc; t += 256)
        smem[t] = 0.0;  // J tile (+ species-1 low-bits tile)
    bar_consumers();
    for (int round = 0; ws_consume_begin<DIM>(P, sh, round, f); ++round) {
        unsigned long long t_cbegin = 0;
        if (P.trace && threadIdx.x == 256) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_cbegin));
        const int TN = f.TN, ts1 = f.ts1, ts2 = f.ts2;
        unsigned *sJlo = reinterpret_cast<unsigned *>(smem), *sJhi = sJlo + 3 * TN, *sLB = sJhi + 3 * TN;
        const double *sDall = smem + ws_layout(TN, NS, NF, IL, G8).desc;
        int spc = 0;
        int64_t w0 = 0, w1 = 0;
        if (IL) w1 = P.ilp[(int64_t)f.it * K1_IL_PAIRS + pair].n;  // virtual indices of the pair's segment
        else item_segment(f.item, pair, WS_PAIRS, spc, w0, w1);
        // run sums in units of the tile quantum 2^-(44+F), exact: every term is rounded to the unit on
        // its own (the descriptor carries values pre-scaled by 2^(44+F); fma(.., .., 1.5 * 2^52) leaves
        // the rounded integer in the low mantissa bits), so the sum does not depend on the order of
        // the particles inside a key -- K5 needs no canonical order for the step to be deterministic
        using RunAcc = typename std::conditional<(WS_FP64RUN && DIM == 3), double, long long>::type;
        RunAcc ax[4] = {0, 0, 0, 0}, ay[4] = {0, 0, 0, 0}, az[4] = {0, 0, 0, 0};
        // (interleaved items) the item's flush rounds the two species apart like the reference
        // (rne_species_split), from species 1's share of the tile mod 2^32.  Within an anchor the walk puts
        // species 1 first, so a run's sums are species 1's alone until its first species-0 particle: their
        // low 32 bits go to the low-bits tile there (sw), or at the flush when the run never switches.
        // run1: the run holds species-1 particles.
        bool run1 = false, sw = false;
        int cur_anchor = -1, cur_key = -1;  // the run's anchor; the last segment's flagged anchor
        const int T1 = f.g.T[1];
        // node of lane (la, lb)'s Jy column entry k ([x][z][y] tile with WS_JYT, else [x][y][z])
        auto jy_idx = [&](int anc, int k) {
            return WS_JYT && DIM == 3 ? TN + (anc >> K1_ANC_BITS) + la * ts1 + lb * T1 + k
                                      : TN + anc + la * ts1 + k * ts2 + lb;
        };
        auto lb_add = [&](int key) {  // low bits of the run sums (lanes of a warp hit distinct nodes)
            if (!WS_LB || (P.ablate & 17)) return;
            const int anc = WS_JYT && DIM == 3 ? key & K1_ANC_MASK : key;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                atomicAdd(sLB + anc + k * ts1 + la * ts2 + lb, (unsigned)acc_units(ax[k]));
                atomicAdd(sLB + jy_idx(key, k), (unsigned)acc_units(ay[k]));
                atomicAdd(sLB + 2 * TN + anc + la * ts1 + lb * ts2 + k, (unsigned)acc_units(az[k]));
            }
        };
        auto flush_run = [&](int key) {
            if (P.ablate & 1) return;
            const int anc = WS_JYT && DIM == 3 ? key & K1_ANC_MASK : key;
            if (DIM == 2) {
                tile_add(sJlo, sJhi, 2 * TN + anc + la * ts1 + lb, az[0]);
                if (la < 4) {
                    tile_add(sJlo, sJhi, anc + la * ts1 + lb, ax[0]);
                    tile_add(sJlo, sJhi, TN + anc + lb * ts1 + la, ay[0]);
                }
            } else {
                int idx[12];
                long long iv[12];
                unsigned old[12];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    idx[k] = anc + k * ts1 + la * ts2 + lb;
                    idx[4 + k] = jy_idx(key, k);
                    idx[8 + k] = 2 * TN + anc + la * ts1 + lb * ts2 + k;
                    iv[k] = acc_units(ax[k]);
                    iv[4 + k] = acc_units(ay[k]);
                    iv[8 + k] = acc_units(az[k]);
                }
#pragma unroll
                for (int m = 0; m < 12; ++m) old[m] = atomicAdd(sJlo + idx[m], (unsigned)iv[m]);
#pragma unroll
                for (int m = 0; m < 12; ++m) {
                    const unsigned l = (unsigned)iv[m];
                    atomicAdd(sJhi + idx[m], (unsigned)((unsigned long long)iv[m] >> 32) + ((old[m] + l) < old[m] ? 1u : 0u));
                }
                if (IL && WS_LB && run1 && !sw && !(P.ablate & 16)) {  // a run of species 1 only
#pragma unroll
                    for (int m = 0; m < 12; ++m) atomicAdd(sLB + idx[m], (unsigned)iv[m]);
                }
            }
        };
        for (int64_t base = w0; base < w1; base += 32, ++use) {
            const int slot = use % NS;
            mbar_wait(&sh.full[pair][slot], (use / NS) & 1);
            const double *sD = sDall + (pair * NS + slot) * 32 * NF;
            const int my_anchor = sh.anchor[pair][slot][lane];
            const int np_ = (int)min((int64_t)32, w1 - base);
            const int prev = __shfl_up_sync(0xffffffffu, my_anchor, 1);
            const unsigned bounds =
                __ballot_sync(0xffffffffu, lane < np_ && (lane == 0 ? my_anchor != cur_key : my_anchor != prev));
            if (!(P.ablate & 2)) {
#pragma unroll 1
                for (int p = 0; p < np_;) {
                    const unsigned rest = p >= 31 ? 0u : (bounds & ~((2u << p) - 1u));
                    const int q = rest ? __ffs(rest) - 1 : np_;
                    const int key = sh.anchor[pair][slot][p];
                    const int anc = (IL && WS_LB && key >= 0) ? (key & ~K1_SP1) : key;
                    if (anc != cur_anchor) {
                        if (cur_anchor >= 0 && lane < 25) flush_run(cur_anchor);
#pragma unroll
                        for (int k = 0; k < 4; ++k) { ax[k] = 0; ay[k] = 0; az[k] = 0; }
                        run1 = IL && WS_LB && key != anc;
                        sw = false;
                        cur_anchor = anc;
                    } else if (IL && WS_LB && key != cur_key && run1 && !sw) {
                        // species 1 -> 0 within the run (species 1 leads within an anchor): the sums so far
                        // are species 1's alone
                        if (lane < 25 && WS_LB_DBG == 0) lb_add(anc);
                        sw = true;
                    }
                    cur_key = key;
                    if (anc >= 0 && lane < 25) {
                        if (DIM == 2) {
#pragma unroll 1
                            for (int r = p; r < q; ++r) {
                                const double *d = sD + r * NF;
                                const double2 xa = *reinterpret_cast<const double2 *>(d + 2 * la);
                                const double2 yb = *reinterpret_cast<const double2 *>(d + 10 + 2 * lb);
                                const double fz = d[28];
                                if (fz != 0.0) {
                                    const double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
                                    const double za = fz * (yb.x * third + yb.y * sixth);
                                    const double zb = fz * (yb.x * sixth + yb.y * third);
                                    az[0] += fx_units(xa.x * za + xa.y * zb);
                                }
                                if (la < 4) {
                                    const double2 dx01 = *reinterpret_cast<const double2 *>(d + 20);
                                    const double2 dx23 = *reinterpret_cast<const double2 *>(d + 22);
                                    const double2 dy01 = *reinterpret_cast<const double2 *>(d + 24);
                                    const double2 dy23 = *reinterpret_cast<const double2 *>(d + 26);
                                    const double dX[4] = {dx01.x, dx01.y, dx23.x, dx23.y};
                                    const double dY[4] = {dy01.x, dy01.y, dy23.x, dy23.y};
                                    const double cyx = 0.5 * (yb.x + yb.y);
                                    double acc = 0.0;
#pragma unroll
                                    for (int k = 0; k < 4; ++k)
                                        if (k <= la) acc -= dX[k] * cyx;
                                    ax[0] += fx_units(acc);
                                    const double2 xb = *reinterpret_cast<const double2 *>(d + 2 * lb);
                                    const double cxy = 0.5 * (xb.x + xb.y);
                                    double accy = 0.0;
#pragma unroll
                                    for (int k = 0; k < 4; ++k)
                                        if (k <= la) accy -= dY[k] * cxy;
                                    ay[0] += fx_units(accy);
                                }
                            }
                        } else {
                            const double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
                            // one particle's 12 column terms
                            auto deposit = [&](int r) {
                                const double *d = sD + r * NF;
                                const double2 xa = *reinterpret_cast<const double2 *>(d + 2 * la);
                                const double2 ya = *reinterpret_cast<const double2 *>(d + 10 + 2 * la);
                                const double2 yb = *reinterpret_cast<const double2 *>(d + 10 + 2 * lb);
                                const double2 zab = *reinterpret_cast<const double2 *>(d + 20 + 2 * lb);  // (Az, Bz)
                                const double Az = zab.x, Bz = zab.y;
                                const double Ay = __fma_rn(yb.y, sixth, yb.x * third), By = __fma_rn(yb.y, third, yb.x * sixth);
                                const double wyz = __fma_rn(ya.y, Bz, ya.x * Az);
                                const double wxz = __fma_rn(xa.y, Bz, xa.x * Az);
                                const double wxy = __fma_rn(xa.y, By, xa.x * Ay);
                                const double2 px01 = *reinterpret_cast<const double2 *>(d + 30);
                                const double2 px23 = *reinterpret_cast<const double2 *>(d + 32);
                                const double2 py01 = *reinterpret_cast<const double2 *>(d + 34);
                                const double2 py23 = *reinterpret_cast<const double2 *>(d + 36);
                                const double2 pz01 = *reinterpret_cast<const double2 *>(d + 38);
                                const double2 pz23 = *reinterpret_cast<const double2 *>(d + 40);
                                // (one rounding per term: the sums are exact; summing raw bits with the
                                // bias taken off at the flush, or pairs of particles per 3-input add,
                                // measured slower)
                                acc_term(ax[0], px01.x, wyz);
                                acc_term(ax[1], px01.y, wyz);
                                acc_term(ax[2], px23.x, wyz);
                                acc_term(ax[3], px23.y, wyz);
                                acc_term(ay[0], py01.x, wxz);
                                acc_term(ay[1], py01.y, wxz);
                                acc_term(ay[2], py23.x, wxz);
                                acc_term(ay[3], py23.y, wxz);
                                acc_term(az[0], pz01.x, wxy);
                                acc_term(az[1], pz01.y, wxy);
                                acc_term(az[2], pz23.x, wxy);
                                acc_term(az[3], pz23.y, wxy);
                            };
#pragma unroll 1
                            for (int r = p; r < q; ++r) deposit(r);
                        }
                    }
                    p = q;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh.empty[pair][slot]);
        }
        if (cur_anchor >= 0 && lane < 25) flush_run(cur_anchor);
        unsigned long long t_done = 0;
        if (WS_DECOUPLE) {
            bar_consumers();  // every consumer done with the J tile (the producers may be an item ahead)
            if (P.trace && threadIdx.x == 256) t_done = *(volatile unsigned long long *)&sh.td[round & 1];
        } else {
            __syncthreads();  // item end: both roles done
            if (P.trace && threadIdx.x == 256) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_done));
        }
        ws_consume_end<DIM, IL, DEVF>(P, sh, smem, round, f, t_cbegin, t_done);
    }
}

template <int DIM, bool STAGE, int NS, bool IL, bool SPARSE = false, bool G8 = false, bool DEVF = false>
__global__ void __launch_bounds__(WS_THREADS, 1) k1_ws(const __grid_constant__ K1Params P) {
    // the fast (host F) and the safe (device F) instantiation are both launched: one of them returns here
    if ((*P.jsafe_dev != 0) == DEVF) return;
    extern __shared__ __align__(128) double smem[];
    __shared__ WsShared sh;
    if (threadIdx.x < WS_PAIRS * 2) {
        mbar_init(&sh.full[threadIdx.x >> 1][threadIdx.x & 1], 1);
        mbar_init(&sh.empty[threadIdx.x >> 1][threadIdx.x & 1], 1);
    }
    if (threadIdx.x == 0) {
        mbar_init(&sh.item_full, 1);
        mbar_init(&sh.item_read, WS_PAIRS);  // one arrival per consumer warp
        mbar_init(&sh.tma_bar, 1);
        sh.n_items = *P.n_items;
        sh.fbits = *P.fbits_dev;
        sh.fscale = *P.fscale_dev;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");  // visible to the async proxy (TMA)
    }
    if (IL && threadIdx.x < 2) sh.spec[threadIdx.x] = P.sp[threadIdx.x];
    if (!IL && threadIdx.x < P.cfg.n_species)
        reinterpret_cast<K1Species *>(smem + ws_layout(tile_nodes_dev(P.cfg), NS, Desc<DIM>::NF, false, G8).spec)[threadIdx.x] =
            P.sp[threadIdx.x];
    __syncthreads();
    if ((threadIdx.x >> 5) < WS_PAIRS) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(SPARSE ? WS_PREG - WS_SPARSE_SHIFT : WS_PREG));
        ws_producer<DIM, STAGE, NS, IL, G8, DEVF>(P, sh, smem);
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(SPARSE ? WS_CREG + WS_SPARSE_SHIFT : WS_CREG));
        ws_consumer<DIM, STAGE, NS, IL, G8, DEVF>(P, sh, smem);
    }
}

int tile_nodes(const b200pic_config &c) {
    return (c.bx + 5) * (c.pn[1] + 5) * (c.dim == 3 ? c.pn[2] + 5 : 1);
}
int field_tile_nodes(const b200pic_config &c) {
    return (c.bx + 4) * (c.pn[1] + 4) * (c.dim == 3 ? c.pn[2] + 4 : 1);
}

typedef void (*K1Fn)(K1Params);

// the warp-specialised K1 stages E/B per component with TMA on the BASELINE geometry (g8) for the items
// interleaving both species, whose species-1 low-bits tile needs the shared memory the compact tiles free
// (one-species items keep the generic staged tile: same-box A/B on config 3, K1 15.2 vs 17.2 ms)
bool use_g8(const b200pic_config &c, bool il) {
    static const bool off = getenv("B200PIC_NO_G8") != nullptr;  // (A/B experiments only)
    return il && c.k1_variant == 2 && c.k1_stage_fields && g8_geometry(c) && !off;
}

int64_t ws_bytes(const b200pic_config &c, int ns, bool il) {
    const int nf = c.dim == 2 ? Desc<2>::NF : Desc<3>::NF;
    const bool g8t = use_g8(c, il);
    int64_t d = ws_layout(tile_nodes(c), ns, nf, il, g8t).ef;
    const int fy = c.pn[1] + 4, fz = c.dim == 3 ? c.pn[2] + 4 : 1;
    if (c.k1_stage_fields) d += g8t ? g8::TOTAL : 6 * (int64_t)(c.bx + 4) * ws_fxs(fy * fz, c.dim);
    return d * 8;
}

int ws_slots(const b200pic_config &c) { return ws_bytes(c, 2, merged_items(c) == 2) <= WS_SMEM_LIMIT ? 2 : 1; }



struct K1Pick {
    K1Fn fn;           // the warp-specialised kernels: J units from the host (fast path) ...
    K1Fn fn_safe;      // ... and from this step's device bound (launched too; one of the two exits at once)
    const char *name;  // the instantiation (b200pic_k1_kernel_name: tests assert the benchmarked one is covered)
};
// k1_ws<DIM, STAGE, NS, IL, SPARSE, G8> in both J-units flavours
#define K1W(D, ST, NS, IL, SP, G8) \
    K1Pick{k1_ws<D, ST, NS, IL, SP, G8, false>, k1_ws<D, ST, NS, IL, SP, G8, true>, \
           "k1_ws<" #D ", " #ST ", " #NS ", " #IL ", " #SP ", " #G8 ">"}
#define K1F(...) K1Pick{__VA_ARGS__, nullptr, #__VA_ARGS__}

K1Pick pick_named(const b200pic_config &c) {
    const bool st = c.k1_stage_fields != 0;
    if (c.k1_variant == 2) {
        const bool two = ws_slots(c) == 2;
        if (c.dim == 2)
            return st ? (two ? K1W(2, true, 2, false, false, false) : K1W(2, true, 1, false, false, false))
                      : (two ? K1W(2, false, 2, false, false, false) : K1W(2, false, 1, false, false, false));
        const bool il = merged_items(c) == 2;
        if (use_g8(c, il) && !two)  // BASELINE geometry, interleaved items: per-component E/B tiles by TMA
            return c.k1_sparse ? K1W(3, true, 1, true, true, true) : K1W(3, true, 1, true, false, true);
        if (c.k1_sparse && st && !two)  // sparse plasma: more consumer registers (flush-heavy runs)
            return il ? K1W(3, true, 1, true, true, false) : K1W(3, true, 1, false, true, false);
        if (il)  // both species interleaved by anchor (3D only)
            return st ? (two ? K1W(3, true, 2, true, false, false) : K1W(3, true, 1, true, false, false))
                      : (two ? K1W(3, false, 2, true, false, false) : K1W(3, false, 1, true, false, false));
        return st ? (two ? K1W(3, true, 2, false, false, false) : K1W(3, true, 1, false, false, false))
                  : (two ? K1W(3, false, 2, false, false, false) : K1W(3, false, 1, false, false, false));
    }
    const int v = c.k1_variant == 1 ? 1 : 0;
    if (c.dim == 2) {
        if (v == 0) return st ? K1F(k1_fused<2, 0, true>) : K1F(k1_fused<2, 0, false>);
        return st ? K1F(k1_fused<2, 1, true>) : K1F(k1_fused<2, 1, false>);
    }
    if (v == 0) return st ? K1F(k1_fused<3, 0, true>) : K1F(k1_fused<3, 0, false>);
    return st ? K1F(k1_fused<3, 1, true>) : K1F(k1_fused<3, 1, false>);
}
#undef K1W
#undef K1F

K1Fn pick(const b200pic_config &c) { return pick_named(c).fn; }

// TMA descriptors of the six field arrays for the g8 staging: 3D (z, y, x) with the padded z pitch, one
// box per component at its own extent (g8::ext, z rounded up to even)
int make_field_tmaps(K1Params &P) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return B200PIC_ERR_CUDA;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const b200pic_config &c = P.cfg;
    const cuuint64_t dims[3] = {(cuuint64_t)ext_of(c, 2), (cuuint64_t)ext_of(c, 1), (cuuint64_t)ext_of(c, 0)};
    const cuuint64_t strides[2] = {(cuuint64_t)zpitch(c) * 8, (cuuint64_t)(ext_of(c, 1) * zpitch(c)) * 8};
    const cuuint32_t estr[3] = {1, 1, 1};
    for (int k = 0; k < 6; ++k) {
        const cuuint32_t box[3] = {(cuuint32_t)g8::zext(k), (cuuint32_t)g8::yext(k), (cuuint32_t)g8::ext(k, 0)};
        const CUresult r = encode(&P.tmap[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)P.e[k], dims, strides, box,
                                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return B200PIC_ERR_CUDA;
    }
    return B200PIC_OK;
}

}  // namespace

int k1_il_fits(const b200pic_config &c) { return ws_bytes(c, 1, true) <= WS_SMEM_LIMIT; }

// stage the E/B tile when the staged kernel fits in shared memory next to its static part (WS_SMEM_LIMIT
// keeps 4 KB of the 227 KB opt-in for it)
int k1_stage_default(const b200pic_config &c0) {
    b200pic_config c = c0;
    c.k1_stage_fields = 1;
    return k1_smem_bytes(c) <= WS_SMEM_LIMIT;
}

int k1_smem_bytes(const b200pic_config &c) {
    const int64_t T = tile_nodes(c);
    const int64_t nf = c.dim == 2 ? Desc<2>::NF : Desc<3>::NF;
    if (c.k1_variant == 2) return (int)ws_bytes(c, ws_slots(c), merged_items(c) == 2);
    int64_t bytes = ((3 * T + 1) & ~1ll) * 8;
    if (c.k1_variant != 1) bytes += (int64_t)NWARPS * 32 * nf * 8;
    if (c.k1_stage_fields) bytes += 6 * (int64_t)field_tile_nodes(c) * 8;
    return (int)bytes;
}

int launch_k1(const K1Params &P0, int grid, cudaStream_t s) {
    const int smem = k1_smem_bytes(P0.cfg);
    K1Fn fn = pick(P0.cfg);
    K1Params P = P0;
    if (use_g8(P.cfg, merged_items(P.cfg) == 2) && ws_slots(P.cfg) == 1) {
        const int rc = make_field_tmaps(P);
        if (rc) return rc;
    }
    const K1Fn fns[2] = {fn, pick_named(P0.cfg).fn_safe};
    for (int k = 0; k < 2; ++k) {
        if (!fns[k]) continue;
        if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(fns[k], cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        fns[k]<<<grid, P.cfg.k1_variant == 2 ? WS_THREADS : K1_THREADS, smem, s>>>(P);
        LAUNCH_CHECK();
    }
    return B200PIC_OK;
}

const char *k1_kernel_name(const b200pic_config &c) { return pick_named(c).name; }

int k1_grid(const b200pic_config &c) {
    const int smem = k1_smem_bytes(c);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    K1Fn fn = pick(c);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, c.k1_variant == 2 ? WS_THREADS : K1_THREADS, smem);
    if (per_sm < 1) per_sm = 1;
    return sms * per_sm;
}
