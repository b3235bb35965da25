// k1_particles.cu -- K1: the fused macro-particle kernel.
//
// One persistent kernel replaces the reference's whole particle phase
// (scheduler.py:442-468): for every work item = (species, patch, bin, chunk)
// pulled from an atomic queue it
//   1. stages the item's E/B stencil tile in shared memory,
//   2. per particle: interpolate (kernels.py:51-121), Boris push
//      (kernels.py:124-162), pre-BC flags (kernels.py:165-178), Esirkepov
//      projection into a shared-memory J tile (kernels.py:181-266), then the
//      global BC + destination (patch, bin) key of the exchange step
//      (exchange.py:163-230, arena.py:59-75) so the re-sort (K5) needs no
//      second pass over positions,
//   3. flushes the tile as rint(J * 2^44) into the int64 accumulators
//      (reduce_bin_currents, fields.py:101-114) with global atomics.
// The per-(patch, species, bin) task chain of the paper's Algorithm 2 is
// program order inside one thread; the serialised reduction becomes integer
// atomics, which commute (fields.py:16-20).
#include "k1.cuh"

namespace {

template <int DIM>
struct TileGeom {
    int64_t o[3];  // node of tile element 0 per axis
    int T[3];      // tile extent per axis
    int64_t pc[3]; // patch coordinates
    double bd[6];  // patch bounds (domain.py:26-29)
};

template <int DIM>
__device__ __forceinline__ void decode_item(const K1Params &P, int key, TileGeom<DIM> &g) {
    const b200pic_config &c = P.cfg;
    int64_t nb = c.pn[0] / c.bx;
    int64_t flat = key / nb, bin = key % nb;
    if (DIM == 3) {
        g.pc[2] = flat % c.np[2];
        flat /= c.np[2];
    } else {
        g.pc[2] = 0;
    }
    g.pc[1] = flat % c.np[1];
    g.pc[0] = flat / c.np[1];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        int64_t cell0 = g.pc[a] * c.pn[a];
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

template <int DIM>
__global__ void __launch_bounds__(K1_THREADS) k1_fused(K1Params P) {
    extern __shared__ double smem[];
    __shared__ int s_item;
    const b200pic_config &c = P.cfg;
    const bool has_z = DIM == 3;
    const int64_t e1 = ext_of(c, 1), e2 = ext_of(c, 2);
    const int n_items = *P.n_items;
    const int64_t NB = c.pn[0] / c.bx;

    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(P.queue, 1);
        __syncthreads();
        const int it = s_item;
        if (it >= n_items) break;
        const K1Item item = P.items[it];
        TileGeom<DIM> g;
        decode_item<DIM>(P, item.key, g);
        const int TN = g.T[0] * g.T[1] * g.T[2];
        const int ts1 = g.T[1] * g.T[2], ts2 = g.T[2];
        double *sF = smem;            // 6 * TN
        double *sJ = smem + 6 * TN;   // 3 * TN
        // ---- stage E/B tile, zero J tile ----
        for (int t = threadIdx.x; t < TN; t += blockDim.x) {
            int u = t / ts1, r = t - u * ts1, v = r / ts2, q = r - v * ts2;
            int64_t gi = ((g.o[0] + u + G) * e1 + (g.o[1] + v + G)) * e2 + (DIM == 3 ? g.o[2] + q + G : 0);
#pragma unroll
            for (int k = 0; k < 6; ++k) sF[k * TN + t] = __ldg(P.e[k] + gi);
#pragma unroll
            for (int k = 0; k < 3; ++k) sJ[k * TN + t] = 0.0;
        }
        __syncthreads();
        const K1Species &S = P.sp[item.species];
        const double *fptr[6] = {sF, sF + TN, sF + 2 * TN, sF + 3 * TN, sF + 4 * TN, sF + 5 * TN};
        const int64_t pend = item.start + item.count;
        for (int64_t n = item.start + threadIdx.x; n < pend; n += blockDim.x) {
            double x = S.x[n], y = S.y[n], z = has_z ? S.z[n] : 0.0;
            double px = S.px[n], py = S.py[n], pz = S.pz[n], w = S.w[n];
            Gathered gt;
            bool ok;
            if (DIM == 2) {
                ok = gather2d(x, y, P.inv[0], P.inv[1], fptr, ts1, g.o[0], g.o[1], 0, g.T[0] - 1, 0, g.T[1] - 1, gt);
            } else {
                const int64_t lo[3] = {0, 0, 0}, hi[3] = {g.T[0] - 1, g.T[1] - 1, g.T[2] - 1};
                ok = gather3d(x, y, z, P.inv, fptr, ts1, ts2, g.o, lo, hi, gt);
            }
            if (!ok) {
                raise_error(P.err, B200PIC_ERR_INVARIANT, S.id[n]);
                S.key[n] = item.key;  // keep the sort consistent; the sticky error aborts the run
                continue;
            }
            double gn;
            if (!boris(x, y, z, has_z, px, py, pz, gt.e, gt.b, S.qd2, S.inv_m2, S.mass, c.dt, gn))
                raise_error(P.err, B200PIC_ERR_NONFINITE, S.id[n]);
            const int fl = pre_bc_flags(x, y, z, has_z, g.bd);
            // ---- projection (pre-BC post-push position, kernels.py:181-266) ----
            double s0[3][5], s1[3][5];
            bool cour = esirkepov_shapes(x * P.inv[0], gt.ip, gt.dxp, s0[0], s1[0]) &&
                        esirkepov_shapes(y * P.inv[1], gt.jp, gt.dyp, s0[1], s1[1]);
            if (DIM == 3) cour = cour && esirkepov_shapes(z * P.inv[2], gt.kp, gt.dzp, s0[2], s1[2]);
            if (!cour) {
                raise_error(P.err, B200PIC_ERR_COURANT, S.id[n]);
            } else {
                const int64_t bi = gt.ip - 2 - g.o[0], bj = gt.jp - 2 - g.o[1], bk = DIM == 3 ? gt.kp - 2 - g.o[2] : 0;
                if (bi < 0 || bi > g.T[0] - 5 || bj < 0 || bj > g.T[1] - 5 || (DIM == 3 && (bk < 0 || bk > g.T[2] - 5))) {
                    raise_error(P.err, B200PIC_ERR_INVARIANT, S.id[n]);
                } else {
                    const double qw = S.charge * w;
                    auto add = [&](int cc, int64_t idx, double v) { atomicAdd(sJ + cc * TN + idx, v); };
                    if (DIM == 2) {
                        // fz = qw * pz / (gam * mass) with gam == gn (kernels.py:234-237)
                        const double fz = qw * pz / (gn * S.mass);
                        esirkepov2d_accumulate(s0[0], s1[0], s0[1], s1[1], qw * P.d_over_dt[0], qw * P.d_over_dt[1],
                                               fz, bi, bj, ts1, add);
                    } else {
                        esirkepov3d_accumulate(s0, s1, qw * P.d_over_dt[0], qw * P.d_over_dt[1], qw * P.d_over_dt[2],
                                               bi, bj, bk, ts1, ts2, add);
                    }
                }
            }
            // ---- global BC + destination key (exchange.py:196-230, arena.py:59-75) ----
            double pos[3] = {x, y, z}, mom[3] = {px, py, pz};
            int64_t dest[3] = {g.pc[0], g.pc[1], g.pc[2]};
            if (fl) {
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    const int fneg = 1 << (2 * a), fpos = 2 << (2 * a);
                    if (g.pc[a] == c.np[a] - 1 && (fl & fpos)) {
                        if (c.bc[a] == B200PIC_BC_PERIODIC) pos[a] -= P.Lw[a];
                        else { pos[a] = fmin(2.0 * P.Lw[a] - pos[a], nextafter(P.Lw[a], 0.0)); mom[a] = -mom[a]; }
                    }
                    if (g.pc[a] == 0 && (fl & fneg)) {
                        if (c.bc[a] == B200PIC_BC_PERIODIC) pos[a] += P.Lw[a];
                        else { pos[a] = -pos[a]; mom[a] = -mom[a]; }
                    }
                }
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    int64_t cell = (int64_t)floor(pos[a] * P.inv[a]);
                    cell = cell < 0 ? 0 : (cell > c.L[a] - 1 ? c.L[a] - 1 : cell);
                    dest[a] = cell / c.pn[a];
                }
            }
            int64_t cx = (int64_t)floor(pos[0] * P.inv[0]) - dest[0] * c.pn[0];
            if (cx < 0 || cx > c.pn[0]) raise_error(P.err, B200PIC_ERR_INVARIANT, S.id[n]);
            cx = cx < 0 ? 0 : (cx > c.pn[0] - 1 ? c.pn[0] - 1 : cx);
            int64_t dflat = DIM == 3 ? (dest[0] * c.np[1] + dest[1]) * c.np[2] + dest[2] : dest[0] * c.np[1] + dest[1];
            int64_t key = dflat * NB + cx / c.bx;
            if (key < 0 || key >= n_patches(c) * NB) {  // only reachable with non-finite positions
                raise_error(P.err, B200PIC_ERR_INVARIANT, S.id[n]);
                key = item.key;
            }
            S.key[n] = (int32_t)key;
            S.x[n] = pos[0];
            S.y[n] = pos[1];
            if (has_z) S.z[n] = pos[2];
            S.px[n] = mom[0];
            S.py[n] = mom[1];
            S.pz[n] = mom[2];
        }
        __syncthreads();
        // ---- flush: rint(tile * 2^44) into the int64 accumulators (fields.py:108-114) ----
        for (int t = threadIdx.x; t < TN; t += blockDim.x) {
            int u = t / ts1, r = t - u * ts1, v = r / ts2, q = r - v * ts2;
            int64_t gi = ((g.o[0] + u + G) * e1 + (g.o[1] + v + G)) * e2 + (DIM == 3 ? g.o[2] + q + G : 0);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                double v = sJ[k * TN + t];
                if (v != 0.0) {
                    long long iv = __double2ll_rn(v * J_SCALE);
                    if (iv) atomicAdd((unsigned long long *)(P.jacc[k] + gi), (unsigned long long)iv);
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace

int k1_smem_bytes(const b200pic_config &c) {
    int64_t T = (int64_t)(c.bx + 5) * (c.pn[1] + 5) * (c.dim == 3 ? c.pn[2] + 5 : 1);
    return (int)(9 * T * sizeof(double));
}

int launch_k1(const K1Params &P, int grid, cudaStream_t s) {
    int smem = k1_smem_bytes(P.cfg);
    if (P.cfg.dim == 2) {
        if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(k1_fused<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k1_fused<2><<<grid, K1_THREADS, smem, s>>>(P);
    } else {
        if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(k1_fused<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k1_fused<3><<<grid, K1_THREADS, smem, s>>>(P);
    }
    LAUNCH_CHECK();
    return B200PIC_OK;
}

int k1_grid(const b200pic_config &c) {
    int smem = k1_smem_bytes(c);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (c.dim == 2) {
        cudaFuncSetAttribute(k1_fused<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1_fused<2>, K1_THREADS, smem);
    } else {
        cudaFuncSetAttribute(k1_fused<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1_fused<3>, K1_THREADS, smem);
    }
    if (per_sm < 1) per_sm = 1;
    return sms * per_sm;
}
