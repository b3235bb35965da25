// sort.cu -- K5: (patch, bin, anchor) re-sort + K1 work-item build.
//
// Replaces apply_particle_bc_and_migrate's mailbox/concatenate/argsort
// (exchange.py:196-258) and sort_into_bins (arena.py:78-95): K1 already wrote
// every particle's destination key (after the global BC), so the re-sort is
// a counting sort: warp-aggregated histogram -> exclusive scan -> warp-
// aggregated scatter of a 4-byte permutation (sorted position -> storage
// slot).  No particle record moves here: the next K1 reads through the
// permutation and writes the updated records contiguously into the other
// buffer.  Inside a key the permutation is then sorted by particle id
// (k_seg_tiles / k_seg_warp / k_seg_long), so the order -- and with it every double sum of
// K1 -- is canonical: identical runs are bit-identical.
#include "sort.cuh"

namespace {

constexpr int SCAN_BLOCK = 1024;  // threads; 2 elements per thread

// exclusive scan of one 2048-element block (256 threads x 8 consecutive elements: thread-local scan,
// warp shuffles, one pass over the 8 warp totals); writes the block total
constexpr int SCAN_THREADS = 2 * SCAN_BLOCK / 8;
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_blocks(const int64_t *in, int64_t *out, int64_t n,
                                                             int64_t *block_sums) {
    __shared__ int64_t wsum[SCAN_THREADS / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * 2 * SCAN_BLOCK + 8 * t;
    int64_t v[8];
    if (i0 + 8 <= n) {
        const longlong2 *q = reinterpret_cast<const longlong2 *>(in + i0);  // (n-aligned: i0 % 8 == 0)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const longlong2 a = q[u];
            v[2 * u] = a.x;
            v[2 * u + 1] = a.y;
        }
    } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = i0 + u < n ? in[i0 + u] : 0;
    }
    int64_t tot = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) tot += v[u];
    int64_t incl = tot;  // warp inclusive scan of the thread totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int64_t wpre = 0, btot = 0;
#pragma unroll
    for (int w = 0; w < SCAN_THREADS / 32; ++w) {
        const int64_t x = wsum[w];
        if (w < warp) wpre += x;
        btot += x;
    }
    int64_t run = wpre + incl - tot;  // exclusive prefix of this thread's first element
    if (i0 + 8 <= n) {
        longlong2 *q = reinterpret_cast<longlong2 *>(out + i0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t a = run;
            run += v[2 * u];
            const int64_t b = run;
            run += v[2 * u + 1];
            q[u] = make_longlong2(a, b);
        }
    } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (i0 + u < n) out[i0 + u] = run;
            run += v[u];
        }
    }
    if (t == 0) block_sums[blockIdx.x] = btot;
}

// serial-carry exclusive scan of block sums (one block, any length)
__global__ void k_scan_sums(int64_t *sums, int64_t nb) {
    __shared__ int64_t carry;
    __shared__ int64_t sh[SCAN_BLOCK];
    if (threadIdx.x == 0) carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += SCAN_BLOCK) {
        __syncthreads();
        int64_t i = b0 + threadIdx.x;
        int64_t v = i < nb ? sums[i] : 0;
        sh[threadIdx.x] = v;
        __syncthreads();
        // Hillis-Steele inclusive
        for (int o = 1; o < SCAN_BLOCK; o <<= 1) {
            int64_t add = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
            __syncthreads();
            sh[threadIdx.x] += add;
            __syncthreads();
        }
        if (i < nb) sums[i] = carry + sh[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == SCAN_BLOCK - 1) carry += sh[SCAN_BLOCK - 1];
    }
}

__global__ void k_scan_add(int64_t *out, int64_t n, const int64_t *sums) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] += sums[i / (2 * SCAN_BLOCK)];
}

// ---------------------------------------------------------------------------

struct SortSpecies {
    const int32_t *key;
    int32_t *perm;
    const int64_t *n_dev;
};

struct SortParams {
    SortSpecies sp[B200PIC_MAX_SPECIES];
    int n_species;
    int64_t nk;        // keys per species
    int64_t *counts;   // [S][nk+1]
    int64_t *cursor;   // [S][nk]
};

// Warp aggregation by runs of equal keys: K1 writes every particle at its sorted position, so the keys of
// consecutive slots mostly repeat (particles that keep their (patch, bin, anchor)); each run's head lane does
// one atomic for the run (equal keys in separate runs just do separate atomics).  Cheaper than a match_any.
__device__ __forceinline__ unsigned run_heads(int32_t k, int lane) {
    const int32_t prev = __shfl_up_sync(0xffffffffu, k, 1);
    return __ballot_sync(0xffffffffu, lane == 0 || k != prev);
}

__global__ void k_histogram(SortParams P, int s) {
    const SortSpecies &S = P.sp[s];
    const int64_t n = *S.n_dev;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const int64_t i = i0 + threadIdx.x;
        const int32_t k = i < n ? S.key[i] : -1;
        const bool act = k >= 0 && k < P.nk;  // outgoing (slab) keys >= nk are not sorted
        const unsigned heads = run_heads(act ? k : -1, lane);
        if (act && ((heads >> lane) & 1u)) {
            const unsigned after = lane == 31 ? 0u : heads >> (lane + 1);
            const int len = after ? __ffs(after) : 32 - lane;
            atomicAdd((unsigned long long *)(P.counts + s * (P.nk + 1) + k), (unsigned long long)len);
        }
    }
}

// perm[pos] = i: the sorted position of storage slot i (K1 reads through perm, so no particle moves here).
// Four warp-rows of keys per iteration: their run heads' cursor atomics (which return the base) are in
// flight together instead of one round trip after another.
constexpr int SCATTER_ROWS = 4;
__global__ void k_perm_scatter(SortParams P, int s) {
    const SortSpecies &S = P.sp[s];
    const int64_t n = *S.n_dev;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * SCATTER_ROWS;
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x * SCATTER_ROWS; i0 < n; i0 += stride) {
        int32_t k[SCATTER_ROWS];
        int head[SCATTER_ROWS];
        unsigned long long base[SCATTER_ROWS];
#pragma unroll
        for (int u = 0; u < SCATTER_ROWS; ++u) {
            const int64_t i = i0 + (int64_t)u * blockDim.x + threadIdx.x;
            k[u] = i < n ? S.key[i] : -1;
            if (!(k[u] >= 0 && k[u] < P.nk)) k[u] = -1;  // outgoing (slab) keys >= nk are not sorted
        }
#pragma unroll
        for (int u = 0; u < SCATTER_ROWS; ++u) {
            const unsigned heads = run_heads(k[u], lane);
            head[u] = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));  // this lane's run head
            base[u] = 0;
            if (k[u] >= 0 && head[u] == lane) {
                const unsigned after = lane == 31 ? 0u : heads >> (lane + 1);
                const int len = after ? __ffs(after) : 32 - lane;
                base[u] = atomicAdd((unsigned long long *)(P.cursor + s * P.nk + k[u]), (unsigned long long)len);
            }
        }
#pragma unroll
        for (int u = 0; u < SCATTER_ROWS; ++u) {
            const unsigned long long b = __shfl_sync(0xffffffffu, base[u], head[u]);
            if (k[u] >= 0) S.perm[(int64_t)b + (lane - head[u])] = (int32_t)(i0 + (int64_t)u * blockDim.x + threadIdx.x);
        }
    }
}

// ---- canonical order inside a key: ascending id --------------------------------------
// The scatter above leaves the order inside a key to the atomics (run to run nondeterministic).
// K1's anchor-run accumulation sums in double in that order, so J would differ in the last
// fine quantum between identical runs.  Sorting each key's slice of perm by (id, slot) makes the
// whole step a pure function of its input (SPEC.md "byte-stable for identical config, seed"),
// independent of rank count and history (the reference's (bin, id) order, arena.py:78-95,
// refined by the anchor).  Keys hold ~ppc particles, so:
//   k_seg_tiles  CTA per RANK_TILE sorted positions; key extents from a max-scan of key heads; a
//                key wholly inside the tile and no longer than RANK_MAX is ranked in shared memory
//                (rank = #smaller (id, slot) in the key)
//   k_seg_warp   a warp per remaining key of <= 32 (keys straddling a tile edge)
//   k_seg_long   a CTA per remaining longer key (bitonic tiles in shared memory + merge ranks)
// Each pass writes only the perm slices of the keys it owns, and reads only what it writes.
constexpr int RANK_TILE = 1024;
constexpr int RANK_THREADS = 256;
constexpr int RANK_MAX = 64;
#ifndef SEG_TILE_N
#define SEG_TILE_N 1024
#endif
#ifndef SEG_THREADS_N
#define SEG_THREADS_N 128
#endif
// long-key pass: small CTAs, many in flight per SM (one key each; most long keys hold a few hundred)
constexpr int SEG_TILE = SEG_TILE_N;  // bitonic tile (shared memory)
constexpr int SEG_THREADS = SEG_THREADS_N;

struct SegSpecies {
    const int64_t *offsets;
    const int32_t *key;  // destination key per storage slot (K1 / initial keys)
    const int64_t *id;
    int32_t *perm;
    int32_t *list;       // keys of <= 32 left to k_seg_warp
    int32_t *list2;      // longer keys left to k_seg_long
    int64_t *scr_id, *scr_slot;  // long-key scratch (the idle alt buffers)
};
struct SegParams {
    SegSpecies sp[B200PIC_MAX_SPECIES];
    int64_t nk;
    int32_t *long_n;     // [2][species]: entries of list, list2; [2 * MAX_SPECIES]: keys valid
};
// the passes read the destination key of every storage slot: valid from a sort until a compaction
__device__ __forceinline__ bool seg_keys_valid(const SegParams &P) {
    return P.long_n[2 * B200PIC_MAX_SPECIES] != 0;
}
// species record by compile-time index (a runtime index into the parameter block spills it)
__device__ __forceinline__ SegSpecies seg_species(const SegParams &P, int s) {
    SegSpecies r = P.sp[0];
#pragma unroll
    for (int k = 1; k < B200PIC_MAX_SPECIES; ++k)
        if (s == k) r = P.sp[k];
    return r;
}

__device__ __forceinline__ bool pair_less(int64_t ia, int32_t pa, int64_t ib, int32_t pb) {
    return ia < ib || (ia == ib && pa < pb);
}

// blockIdx.y = species.  Key boundaries come from the keys of neighbouring positions (the slice
// is sorted by key), with one extra key on each side of the tile to detect keys crossing its edges.
__global__ void __launch_bounds__(RANK_THREADS) k_seg_tiles(SegParams P) {
    if (!seg_keys_valid(P)) return;
    constexpr int EPT = RANK_TILE / RANK_THREADS;  // consecutive positions per thread (one 16-byte perm load)
    constexpr int NW = RANK_THREADS / 32;
    __shared__ int64_t si[RANK_TILE];
    __shared__ int32_t sp[RANK_TILE];
    __shared__ int32_t sk[RANK_TILE + 2];  // sk[j + 1] = key at position t0 + j, j in [-1, m]
    __shared__ int16_t kend[RANK_TILE];    // at a key's first tile position: one past its last
    __shared__ int16_t kst[RANK_TILE];     // first tile position of each position's key
    __shared__ int32_t wmax[NW];
    const int s = blockIdx.y;
    const SegSpecies S = seg_species(P, s);
    const int64_t n = S.offsets[P.nk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t t0 = (int64_t)blockIdx.x * RANK_TILE; t0 < n; t0 += (int64_t)gridDim.x * RANK_TILE) {
        const int m = (int)min((int64_t)RANK_TILE, n - t0);
        const int tb = threadIdx.x * EPT;
        int32_t slot[EPT];
        if (tb + EPT <= m && ((t0 + tb) & 3) == 0) {
            const int4 q = *reinterpret_cast<const int4 *>(S.perm + t0 + tb);
            slot[0] = q.x; slot[1] = q.y; slot[2] = q.z; slot[3] = q.w;
        } else {
#pragma unroll
            for (int u = 0; u < EPT; ++u) slot[u] = tb + u < m ? S.perm[t0 + tb + u] : 0;
        }
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int t = tb + u;
            if (t < m) {
                si[t] = __ldg(S.id + slot[u]);
                sp[t] = slot[u];
                sk[t + 1] = __ldg(S.key + slot[u]);
            }
        }
        if (threadIdx.x == 0) sk[0] = t0 > 0 ? __ldg(S.key + S.perm[t0 - 1]) : -1;
        if (threadIdx.x == RANK_THREADS - 1) sk[m + 1] = t0 + m < n ? __ldg(S.key + S.perm[t0 + m]) : -1;
        __syncthreads();
        // start of each position's key inside the tile: inclusive max-scan of (head ? t : 0)
        int st[EPT];
        int run = 0;
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int t = tb + u;
            if (t < m && (t == 0 || sk[t] != sk[t + 1])) run = t;
            st[u] = run;
        }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl = max(incl, v);
        }
        int excl = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) excl = 0;
        if (lane == 31) wmax[warp] = incl;
        __syncthreads();
        int wpre = 0;
        for (int w = 0; w < warp; ++w) wpre = max(wpre, wmax[w]);
        const int pre = max(excl, wpre);
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            st[u] = max(st[u], pre);
            const int t = tb + u;
            if (t < m && (t == m - 1 || sk[t + 1] != sk[t + 2])) kend[st[u]] = (int16_t)(t + 1);  // key's last
            if (t < m) kst[t] = (int16_t)st[u];
        }
        __syncthreads();
        // ranking with consecutive positions on consecutive lanes: lanes of one key loop equally long
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int t = threadIdx.x + u * RANK_THREADS;
            if (t >= m) continue;
            const int32_t k = sk[t + 1];
            const int j0 = kst[t], j1 = kend[j0];
            const bool left = j0 == 0 && sk[0] == k, right = j1 == m && sk[m + 1] == k;
            if (!left && !right && j1 - j0 <= RANK_MAX) {
                if (j1 - j0 >= 2) {
                    const int64_t vid = si[t];
                    const int32_t vs = sp[t];
                    int r = 0;
                    for (int q = j0; q < j1; ++q) r += pair_less(si[q], sp[q], vid, vs);
                    S.perm[t0 + j0 + r] = vs;
                }
            } else if (t == j0 && !left) {
                // straddles the tile's right edge or longer than RANK_MAX: keys of <= 32 go to the warp pass,
                // longer ones to the CTA pass (separate lists: neither pass walks the other's entries)
                const int64_t len = S.offsets[k + 1] - S.offsets[k];
                if (len <= 32) S.list[atomicAdd(P.long_n + s, 1)] = k;
                else S.list2[atomicAdd(P.long_n + B200PIC_MAX_SPECIES + s, 1)] = k;
            }
        }
        __syncthreads();
    }
}

// a warp per listed key of <= 32: lane j holds element j, rank by comparing against all lanes
__global__ void k_seg_warp(SegParams P) {
    if (!seg_keys_valid(P)) return;
    const int s = blockIdx.y;
    const SegSpecies S = seg_species(P, s);
    const int lane = threadIdx.x & 31;
    const int nl = P.long_n[s];
    for (int l = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; l < nl; l += (gridDim.x * blockDim.x) >> 5) {
        const int64_t k = S.list[l];
        const int64_t kb = S.offsets[k];
        const int len = (int)min((int64_t)33, S.offsets[k + 1] - kb);
        if (len > 32) continue;
        int32_t slot = INT32_MAX;
        int64_t vid = INT64_MAX;
        if (lane < len) {
            slot = S.perm[kb + lane];
            vid = __ldg(S.id + slot);
        }
        int r = 0;
        for (int j = 0; j < len; ++j) {
            const int64_t oi = __shfl_sync(0xffffffffu, vid, j);
            const int32_t op = __shfl_sync(0xffffffffu, slot, j);
            r += pair_less(oi, op, vid, slot);
        }
        __syncwarp();
        if (lane < len) S.perm[kb + r] = slot;
    }
}

// bitonic sort of n <= SEG_TILE (id, slot) pairs in shared memory (padded with +inf)
__device__ void tile_sort(int64_t *si, int32_t *sp, int n) {
    int m = 1;
    while (m < n) m <<= 1;
    for (int t = n + threadIdx.x; t < m; t += blockDim.x) { si[t] = INT64_MAX; sp[t] = INT32_MAX; }
    __syncthreads();
    for (int size = 2; size <= m; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < m / 2; t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                if (pair_less(si[hi], sp[hi], si[lo], sp[lo]) == up) {
                    const int64_t a = si[lo]; si[lo] = si[hi]; si[hi] = a;
                    const int32_t c = sp[lo]; sp[lo] = sp[hi]; sp[hi] = c;
                }
            }
            __syncthreads();
        }
}

// one CTA per listed key of > 32: tiles of SEG_TILE sorted in shared memory into scratch, then
// each element's final rank = its rank in its tile + lower bounds in the others
__global__ void __launch_bounds__(SEG_THREADS) k_seg_long(SegParams P) {
    if (!seg_keys_valid(P)) return;
    __shared__ int64_t si[SEG_TILE];
    __shared__ int32_t sp[SEG_TILE];
    const int s = blockIdx.y;
    const SegSpecies S = seg_species(P, s);
    const int nl = P.long_n[B200PIC_MAX_SPECIES + s];
    for (int l = blockIdx.x; l < nl; l += gridDim.x) {
        const int64_t k = S.list2[l];
        const int64_t b = S.offsets[k], len = S.offsets[k + 1] - b;
        const int64_t ntile = (len + SEG_TILE - 1) / SEG_TILE;
        for (int64_t t0 = 0; t0 < len; t0 += SEG_TILE) {
            const int n = (int)min((int64_t)SEG_TILE, len - t0);
            for (int t = threadIdx.x; t < n; t += blockDim.x) {
                const int32_t q = S.perm[b + t0 + t];
                sp[t] = q;
                si[t] = __ldg(S.id + q);
            }
            tile_sort(si, sp, n);
            if (ntile == 1) {
                for (int t = threadIdx.x; t < n; t += blockDim.x) S.perm[b + t] = sp[t];
            } else {
                for (int t = threadIdx.x; t < n; t += blockDim.x) {
                    S.scr_id[b + t0 + t] = si[t];
                    S.scr_slot[b + t0 + t] = sp[t];
                }
            }
            __syncthreads();
        }
        if (ntile == 1) continue;
        for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
            const int64_t vi = S.scr_id[b + e];
            const int32_t vp = (int32_t)S.scr_slot[b + e];
            const int64_t mine = e / SEG_TILE;
            int64_t rank = e - mine * SEG_TILE;
            for (int64_t t = 0; t < ntile; ++t) {
                if (t == mine) continue;
                int64_t lo = t * SEG_TILE, hi = min(len, lo + SEG_TILE);  // lower bound of (vi, vp)
                const int64_t first = lo;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (pair_less(S.scr_id[b + mid], (int32_t)S.scr_slot[b + mid], vi, vp)) lo = mid + 1; else hi = mid;
                }
                rank += lo - first;
            }
            S.perm[b + rank] = vp;
        }
        __syncthreads();
    }
}

// offsets_s[k] = scanned[s*(nk+1)+k] - scanned[s*(nk+1)]; cursor = offsets
// scanned: block-local exclusive scans (k_scan_blocks); bsum: the scanned block totals (k_scan_sums)
__global__ void k_finish_offsets(const int64_t *scanned, const int64_t *bsum, int64_t nk, int s, int64_t *offsets,
                                 int64_t *cursor, int32_t *long_n) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k == 0) {
        long_n[s] = 0;
        long_n[B200PIC_MAX_SPECIES + s] = 0;
        long_n[2 * B200PIC_MAX_SPECIES] = 1;  // keys match the storage slots again
    }
    if (k > nk) return;
    const int64_t i = s * (nk + 1) + k, i0 = s * (nk + 1);
    const int64_t base = scanned[i0] + bsum[i0 / (2 * SCAN_BLOCK)];
    const int64_t v = scanned[i] + bsum[i / (2 * SCAN_BLOCK)] - base;
    offsets[k] = v;
    if (k < nk) cursor[s * nk + k] = v;
}

__global__ void k_set_n_from_offsets(const int64_t *offsets, int64_t nk, int64_t *n_dev) { *n_dev = offsets[nk]; }

// initial keys: patch from clip(floor(x/dx)) (harness injection), bin from the local x cell,
// anchor from the nearest primal node (csrc/common.cuh particle_key)
__global__ void k_initial_keys(b200pic_config c, const double *x, const double *y, const double *z,
                               const int64_t *n_dev, int32_t *key, const int64_t *first_dev) {
    const int64_t first = first_dev ? *first_dev : 0;
    const int64_t n = *n_dev;
    const double inv[3] = {1.0 / c.d[0], 1.0 / c.d[1], c.dim == 3 ? 1.0 / c.d[2] : 1.0};
    const int64_t x0 = slab_x0(c);
    for (int64_t i = first + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double pos[3] = {x[i], y[i], z ? z[i] : 0.0};
        int64_t cell[3] = {0, 0, 0}, dest[3] = {0, 0, 0};
        for (int a = 0; a < c.dim; ++a) {
            int64_t cc = (int64_t)floor(pos[a] * inv[a]) - (a == 0 ? x0 : 0);  // slab-local cell
            cc = cc < 0 ? 0 : (cc > c.L[a] - 1 ? c.L[a] - 1 : cc);
            cell[a] = cc;
            dest[a] = cc / c.pn[a];
        }
        key[i] = (int32_t)particle_key(c, pos, inv, dest, cell[0] - dest[0] * c.pn[0], x0);
    }
}

// chunks per (species, key)
struct OffPtrs {
    const int64_t *p[B200PIC_MAX_SPECIES];
};

// chunks per (species, bin key); offsets are per (bin, anchor) key, stride A per bin.  Merged mode
// (k1_merge): one entry per bin key, pieces over both species
__global__ void k_count_chunks(OffPtrs offsets, int n_species, int merged, int64_t nbk, int64_t A, int64_t chunk,
                               int64_t *nch) {
    const int64_t m = merged ? nbk : n_species * nbk;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m + 1) return;
    if (t == m) { nch[t] = 0; return; }
    int s = merged ? 0 : (int)(t / nbk);
    int64_t k = t - s * nbk;
    int64_t cnt = offsets.p[s][(k + 1) * A] - offsets.p[s][k * A];
    if (merged) cnt += offsets.p[1][(k + 1) * A] - offsets.p[1][k * A];
    nch[t] = (cnt + chunk - 1) / chunk;
}

// j-th of the n - 1 inner cuts of a bin's range [ko[0], ko[A]): the even cut moved to the next
// anchor-key boundary when one lies within chunk / 2, so every piece holds whole keys (which particles
// a piece holds -- and so its tile's rounding to 2^-44 -- does not depend on the order inside a key)
__device__ __forceinline__ int64_t bin_cut(const int64_t *ko, int64_t A, int64_t j, int64_t n, int64_t chunk) {
    const int64_t a = ko[0], b = ko[A];
    if (j <= 0) return a;
    if (j >= n) return b;
    const int64_t t = a + ((b - a) * j) / n;  // even cut
    int64_t lo = 0, hi = A;                   // first key boundary >= t
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ko[mid] < t) lo = mid + 1; else hi = mid;
    }
    return ko[lo] - t <= chunk / 2 ? ko[lo] : t;
}

// merged prefix of a bin's two species over anchors [0, a)
__device__ __forceinline__ int64_t bin_m(const int64_t *k0, const int64_t *k1, int64_t a) {
    return (k0[a] - k0[0]) + (k1[a] - k1[0]);
}
// first anchor boundary in [lo, hi] whose merged prefix is >= t
__device__ __forceinline__ int64_t bin_m_lb(const int64_t *k0, const int64_t *k1, int64_t lo, int64_t hi, int64_t t) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (bin_m(k0, k1, mid) < t) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void k_emit_items(OffPtrs off, int n_species, int merged, int64_t nk, int64_t A, int64_t chunk,
                             const int64_t *nch_scan, K1Item *items, IlPair *ilp, int32_t *n_items) {
    const int64_t m = merged ? nk : n_species * nk;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0) *n_items = (int32_t)nch_scan[m];
    if (t >= m) return;
    int s = merged ? 0 : (int)(t / nk);
    int64_t k = t - s * nk;
    // a dense bin is cut into n = ceil(cnt / chunk) about equal pieces, not chunk-sized pieces plus a
    // small remainder: every item carries its tile staging and flush
    const int64_t base = nch_scan[t], n = nch_scan[t + 1] - base;
    const int64_t *ko = off.p[s] + k * A;  // anchor-key offsets of this bin: ko[0] .. ko[A]
    const int64_t *ko1 = merged ? off.p[1] + k * A : ko;
    if (merged == 2) {
        // pieces = anchor ranges of about equal merged count (every anchor, both species, in one piece);
        // inside a piece the same for the K1_IL_PAIRS producer/consumer pairs
        const int64_t tot = bin_m(ko, ko1, A);
        int64_t a0 = 0;
        for (int64_t j = 0; j < n; ++j) {
            const int64_t a1 = j + 1 < n ? bin_m_lb(ko, ko1, a0, A, (tot * (j + 1)) / n) : A;
            K1Item it;
            it.start = a0;
            it.start1 = a1;
            it.count = (int32_t)(ko[a1] - ko[a0]);
            it.count1 = (int32_t)(ko1[a1] - ko1[a0]);
            it.key = (int32_t)k;
            it.species = -2;
            items[base + j] = it;
            const int64_t m0 = bin_m(ko, ko1, a0), mt = bin_m(ko, ko1, a1) - m0;
            int64_t c = a0;
            for (int p = 0; p < K1_IL_PAIRS; ++p) {
                const int64_t c1 = p + 1 < K1_IL_PAIRS ? bin_m_lb(ko, ko1, c, a1, m0 + (mt * (p + 1)) / K1_IL_PAIRS) : a1;
                IlPair q;
                q.b0 = ko[c];
                q.b1 = ko1[c];
                q.a0 = (int32_t)c;
                q.n = (int32_t)(bin_m(ko, ko1, c1) - bin_m(ko, ko1, c));
                ilp[(base + j) * K1_IL_PAIRS + p] = q;
                c = c1;
            }
            a0 = a1;
        }
        return;
    }
    for (int64_t j = 0; j < n; ++j) {
        K1Item it;
        int64_t c0 = bin_cut(ko, A, j, n, chunk), c1 = bin_cut(ko, A, j + 1, n, chunk);
        c1 = c1 < c0 ? c0 : c1;
        it.start = c0;
        it.count = (int32_t)(c1 - c0);
        it.start1 = 0;
        it.count1 = 0;
        if (merged) {
            int64_t d0 = bin_cut(ko1, A, j, n, chunk), d1 = bin_cut(ko1, A, j + 1, n, chunk);
            d1 = d1 < d0 ? d0 : d1;
            it.start1 = d0;
            it.count1 = (int32_t)(d1 - d0);
        }
        it.key = (int32_t)k;
        it.species = merged ? -1 : s;
        items[base + j] = it;
    }
}

// J tile range, per step: a tile node only receives current from particles whose stencil anchor lies
// within 2 nodes of it (kernels.py:202-232: the 5-point stencil around the pre-push nearest node), so
// |node sum| <= window * max over anchors of sum_s count_s j_bound_s (window 5^dim).  jw <- that max.
struct JbArgs {
    const int64_t *off[B200PIC_MAX_SPECIES];
    double c[B200PIC_MAX_SPECIES];
    int n_species;
    int64_t nk;
    unsigned long long *jw;
};
__global__ void k_jbound(JbArgs A) {
    double m = 0.0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < A.nk; k += (int64_t)gridDim.x * blockDim.x) {
        double w = 0.0;
        for (int s = 0; s < A.n_species; ++s) w += (double)(A.off[s][k + 1] - A.off[s][k]) * A.c[s];
        m = fmax(m, w);
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    // non-negative doubles order like their bit patterns
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(A.jw, (unsigned long long)__double_as_longlong(m));
}
// F = min(16, F_term, largest F whose window bound fits 2^62 units); 2^(44+F).  F_term: every single term
// is rounded to the unit with the 1.5 * 2^52 trick, which needs |term| 2^(44+F) < 2^51 (cmax = max j_bound).
// jsafe: the host's F (fhost) is at most this F, so K1's fast path (host constants) is exact
__global__ void k_jbits(const unsigned long long *jw, int window, double cmax, int fhost, int *fbits, double *fscale,
                        int *jsafe, int64_t *err) {
    const double B = window * __longlong_as_double((long long)*jw);
    int F = 16;
    if (cmax > 0.0) {
        const int ft = (int)ceil(51.0 - 44.0 - log2(cmax * (1.0 + 1e-12))) - 1;
        F = ft < F ? ft : F;
    }
    if (B > 0.0) {
        const int ft = (int)floor(62.0 - 44.0 - log2(B));
        F = ft < F ? ft : F;
    }
    if (F < 0) {  // a stencil window dense enough to overflow the 64-bit tile even at the reference's quantum
        raise_error(err, B200PIC_ERR_CAPACITY, -1);
        F = 0;
    }
    *fbits = F;
    *fscale = ldexp(1.0, 44 + F);
    *jsafe = fhost <= F ? 1 : 0;
}

}  // namespace

// ---------------------------------------------------------------------------

int scan_exclusive(const int64_t *in, int64_t *out, int64_t n, int64_t *tmp, cudaStream_t s) {
    if (n <= 0) return B200PIC_OK;
    int64_t nb = (n + 2 * SCAN_BLOCK - 1) / (2 * SCAN_BLOCK);
    k_scan_blocks<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, out, n, tmp);
    LAUNCH_CHECK();
    if (nb > 1) {
        k_scan_sums<<<1, SCAN_BLOCK, 0, s>>>(tmp, nb);
        LAUNCH_CHECK();
        k_scan_add<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, n, tmp);
        LAUNCH_CHECK();
    }
    return B200PIC_OK;
}

size_t scan_tmp_elems(int64_t n) { return (size_t)((n + 2 * SCAN_BLOCK - 1) / (2 * SCAN_BLOCK)) + 1; }

Workspace carve(const b200pic_state &st) {
    const b200pic_config &c = st.cfg;
    Workspace w;
    char *p = (char *)st.work;
    auto take = [&](size_t bytes) {
        bytes = (bytes + 255) & ~size_t(255);
        char *r = p;
        p += bytes;
        return (void *)r;
    };
    int64_t nk = n_keys(c);
    int S = c.n_species;
    w.nk = nk;
    for (int s = 0; s < S; ++s) w.key[s] = (int32_t *)take(sizeof(int32_t) * (size_t)(st.sp[s].capacity > 0 ? st.sp[s].capacity : 1));
    for (int s = 0; s < S; ++s) w.perm[s] = (int32_t *)take(sizeof(int32_t) * (size_t)(st.sp[s].capacity > 0 ? st.sp[s].capacity : 1));
    w.counts = (int64_t *)take(sizeof(int64_t) * S * (nk + 1));
    w.scanned = (int64_t *)take(sizeof(int64_t) * S * (nk + 1));
    w.cursor = (int64_t *)take(sizeof(int64_t) * S * nk);
    const int64_t nbk = n_bin_keys(c);
    w.nch = (int64_t *)take(sizeof(int64_t) * (S * nbk + 1));
    w.nch_scan = (int64_t *)take(sizeof(int64_t) * (S * nbk + 1));
    w.scan_tmp = (int64_t *)take(sizeof(int64_t) * scan_tmp_elems(S * (nk + 1) + 1));
    int64_t max_items = S * nbk + 1;
    for (int s = 0; s < S; ++s) max_items += st.sp[s].capacity / (c.chunk > 0 ? c.chunk : 1) + 1;
    w.max_items = max_items;
    w.items = (K1Item *)take(sizeof(K1Item) * max_items);
    w.ilp = (IlPair *)take(sizeof(IlPair) * K1_IL_PAIRS * (merged_items(c) == 2 ? max_items : 1));
    w.n_items = (int32_t *)take(sizeof(int32_t) * 4);
    w.aux = (int64_t *)take(sizeof(int64_t) * B200PIC_MAX_SPECIES);
    w.queue = w.n_items + 1;
    w.long_n = (int32_t *)take(sizeof(int32_t) * (2 * B200PIC_MAX_SPECIES + 1));
    w.jw = (unsigned long long *)take(sizeof(unsigned long long));
    w.fbits = (int32_t *)take(sizeof(int32_t));
    w.fscale = (double *)take(sizeof(double));
    w.jsafe = (int32_t *)take(sizeof(int32_t));
    w.bytes = (size_t)(p - (char *)st.work);
    return w;
}

static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

static int grid_for(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t want = (n + 255) / 256;
    int64_t cap = (int64_t)sms * 8;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

// sort species by the keys already in w.key into alt; swap sp <-> alt data pointers
int sort_by_keys(b200pic_state &st, const Workspace &w, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    const int S = c.n_species;
    const int64_t nk = w.nk;
    SortParams P;
    P.n_species = S;
    P.nk = nk;
    P.counts = w.counts;
    P.cursor = w.cursor;
    for (int i = 0; i < S; ++i) {
        SortSpecies &q = P.sp[i];
        q.key = w.key[i];
        q.perm = w.perm[i];
        q.n_dev = st.sp[i].n_dev;
    }
    CUDA_TRY(cudaMemsetAsync(w.counts, 0, sizeof(int64_t) * S * (nk + 1), s));
    int64_t cap = 0;
    for (int i = 0; i < S; ++i) cap = st.sp[i].capacity > cap ? st.sp[i].capacity : cap;
    const int grid = grid_for(cap);
    for (int i = 0; i < S; ++i) {
        k_histogram<<<grid, 256, 0, s>>>(P, i);
        LAUNCH_CHECK();
    }
    {
        // block scans + scanned block totals; k_finish_offsets adds the two (no separate add pass)
        const int64_t m = S * (nk + 1);
        const int64_t nb = (m + 2 * SCAN_BLOCK - 1) / (2 * SCAN_BLOCK);
        k_scan_blocks<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(w.counts, w.scanned, m, w.scan_tmp);
        LAUNCH_CHECK();
        k_scan_sums<<<1, SCAN_BLOCK, 0, s>>>(w.scan_tmp, nb);
        LAUNCH_CHECK();
    }
    for (int i = 0; i < S; ++i) {
        k_finish_offsets<<<(unsigned)((nk + 1 + 255) / 256), 256, 0, s>>>(w.scanned, w.scan_tmp, nk, i,
                                                                         st.sp[i].offsets, w.cursor, w.long_n);
        LAUNCH_CHECK();
    }
    for (int i = 0; i < S; ++i) {
        k_perm_scatter<<<grid, 256, 0, s>>>(P, i);
        LAUNCH_CHECK();
    }
    {  // absorbed / outgoing particles are dropped and received ones appended: the count may change
        for (int i = 0; i < S; ++i) {
            k_set_n_from_offsets<<<1, 1, 0, s>>>(st.sp[i].offsets, nk, st.sp[i].n_dev);
            LAUNCH_CHECK();
        }
    }
    return B200PIC_OK;
}

void swap_buffers(b200pic_state &st) {
    for (int i = 0; i < st.cfg.n_species; ++i) {
        b200pic_species &a = st.sp[i], &b = st.alt[i];
        double **pa[7] = {&a.x, &a.y, &a.z, &a.px, &a.py, &a.pz, &a.w};
        double **pb[7] = {&b.x, &b.y, &b.z, &b.px, &b.py, &b.pz, &b.w};
        for (int f = 0; f < 7; ++f) { double *t = *pa[f]; *pa[f] = *pb[f]; *pb[f] = t; }
        int64_t *t = a.id; a.id = b.id; b.id = t;
    }
}

int initial_keys(b200pic_state &st, const Workspace &w, cudaStream_t s) {
    for (int i = 0; i < st.cfg.n_species; ++i) {
        const b200pic_species &a = st.sp[i];
        k_initial_keys<<<grid_for(a.capacity), 256, 0, s>>>(st.cfg, a.x, a.y, a.z, a.n_dev, w.key[i], nullptr);
        LAUNCH_CHECK();
    }
    return B200PIC_OK;
}

int merged_items(const b200pic_config &c) {
    // k1_merge 1 (pairs split by species) is retired: it rounded the J tile over both species; 1 and 2 both
    // select the interleaved items, which keep the reference's per-species rounding (species-1 low-bits tile)
    if (!(c.k1_merge && c.dim == 3 && c.n_species == 2 && c.k1_variant == 2)) return 0;
    return k1_il_fits(c) ? 2 : 0;
}

int j_bits(const b200pic_state &st, const Workspace &w, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    JbArgs A;
    memset(&A, 0, sizeof(A));
    A.n_species = c.n_species;
    for (int i = 0; i < c.n_species; ++i) {
        A.off[i] = st.sp[i].offsets;
        A.c[i] = c.j_bound[i] > 0.0 ? c.j_bound[i] : 0.0;
    }
    A.nk = w.nk;
    A.jw = w.jw;
    CUDA_TRY(cudaMemsetAsync(w.jw, 0, sizeof(unsigned long long), s));
    k_jbound<<<grid_for(w.nk), 256, 0, s>>>(A);
    LAUNCH_CHECK();
    double cmax = 0.0;
    for (int i = 0; i < c.n_species; ++i) cmax = c.j_bound[i] > cmax ? c.j_bound[i] : cmax;
    const int fhost = c.j_fine_bits < 0 ? 0 : (c.j_fine_bits > 16 ? 16 : c.j_fine_bits);
    k_jbits<<<1, 1, 0, s>>>(w.jw, c.dim == 3 ? 125 : 25, cmax, fhost, w.fbits, w.fscale, w.jsafe, st.err);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

int build_items(b200pic_state &st, const Workspace &w, cudaStream_t s) {
    const b200pic_config &c = st.cfg;
    const int S = c.n_species;
    const int merged = merged_items(c);
    const int64_t nbk = n_bin_keys(c), A = anchors_per_bin(c), chunk = c.chunk > 0 ? c.chunk : (1ll << 30);
    OffPtrs op;
    for (int i = 0; i < B200PIC_MAX_SPECIES; ++i) op.p[i] = i < S ? st.sp[i].offsets : nullptr;
    int64_t m = (merged ? 1 : S) * nbk + 1;
    k_count_chunks<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(op, S, merged, nbk, A, chunk, w.nch);
    LAUNCH_CHECK();
    int rc = scan_exclusive(w.nch, w.nch_scan, m, w.scan_tmp, s);
    if (rc) return rc;
    k_emit_items<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(op, S, merged, nbk, A, chunk, w.nch_scan, w.items,
                                                             w.ilp, w.n_items);
    LAUNCH_CHECK();
    return j_bits(st, w, s);  // this step's J tile fraction bits from the current counts
}

// ---------------------------------------------------------------------------
// x-slab migration: pack particles keyed n_keys + dir into send buffers; append received ones
// ---------------------------------------------------------------------------
namespace {

struct PackArgs {
    const double *src[7];
    const int64_t *id;
    const int32_t *key;
    const int64_t *n_dev;
    double *dst[2];
    int64_t cap, nk;
    int64_t *counts[2];  // per direction (left, right)
    int64_t *err;
    int has_z;
};

__global__ void k_pack_outgoing(PackArgs A) {
    const int64_t n = *A.n_dev;
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        const int64_t k = i < n ? A.key[i] : -1;
        const int dir = (k >= A.nk) ? (int)(k - A.nk) : -1;
        const unsigned mask = __match_any_sync(0xffffffffu, dir);
        const int leader = __ffs(mask) - 1;
        unsigned long long base = 0;
        if (dir >= 0 && lane == leader) base = atomicAdd((unsigned long long *)A.counts[dir], (unsigned long long)__popc(mask));
        base = __shfl_sync(mask, base, leader);
        if (dir < 0) continue;
        const int64_t pos = (int64_t)base + __popc(mask & ((1u << lane) - 1));
        if (pos >= A.cap) {
            raise_error(A.err, B200PIC_ERR_CAPACITY, A.id[i]);
            continue;
        }
        double *d = A.dst[dir];
#pragma unroll
        for (int f = 0; f < 7; ++f) d[f * A.cap + pos] = (f == 2 && !A.has_z) ? 0.0 : A.src[f][i];
        d[7 * A.cap + pos] = __longlong_as_double(A.id[i]);
    }
}

__global__ void k_append(b200pic_species sp, const double *recv, int64_t count, int64_t cap, int has_z,
                         int64_t *err, const int64_t *first_dev) {
    const int64_t n0 = *first_dev;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = n0 + t;
        if (i >= sp.capacity) {
            raise_error(err, B200PIC_ERR_CAPACITY, __double_as_longlong(recv[7 * cap + t]));
            continue;
        }
        sp.x[i] = recv[t];
        sp.y[i] = recv[cap + t];
        if (has_z) sp.z[i] = recv[2 * cap + t];
        sp.px[i] = recv[3 * cap + t];
        sp.py[i] = recv[4 * cap + t];
        sp.pz[i] = recv[5 * cap + t];
        sp.w[i] = recv[6 * cap + t];
        sp.id[i] = __double_as_longlong(recv[7 * cap + t]);
    }
}

__global__ void k_note_count(const int64_t *n_dev, int64_t *first_dev) { *first_dev = *n_dev; }

// the received count read on the device (a fixed-capacity message: no host read of the count), clamped
__global__ void k_append_dev(b200pic_species sp, const double *recv, const int64_t *count_dev, int64_t cap, int has_z,
                             int64_t *err, const int64_t *first_dev) {
    const int64_t count = min(*count_dev, cap);
    const int64_t n0 = *first_dev;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = n0 + t;
        if (i >= sp.capacity) {
            raise_error(err, B200PIC_ERR_CAPACITY, __double_as_longlong(recv[7 * cap + t]));
            continue;
        }
        sp.x[i] = recv[t];
        sp.y[i] = recv[cap + t];
        if (has_z) sp.z[i] = recv[2 * cap + t];
        sp.px[i] = recv[3 * cap + t];
        sp.py[i] = recv[4 * cap + t];
        sp.pz[i] = recv[5 * cap + t];
        sp.w[i] = recv[6 * cap + t];
        sp.id[i] = __double_as_longlong(recv[7 * cap + t]);
    }
}

__global__ void k_bump_count_dev(int64_t *n_dev, const int64_t *first_dev, const int64_t *count_dev, int64_t cap,
                                 int64_t capacity, int64_t *err) {
    const int64_t c = *count_dev;
    if (c > cap) raise_error(err, B200PIC_ERR_CAPACITY, -1);  // the sender overflowed its message
    const int64_t v = *first_dev + (c < cap ? c : cap);
    *n_dev = v > capacity ? capacity : v;
}

__global__ void k_bump_count(int64_t *n_dev, const int64_t *first_dev, int64_t count, int64_t capacity) {
    int64_t v = *first_dev + count;
    *n_dev = v > capacity ? capacity : v;
}

}  // namespace

int pack_outgoing(b200pic_state &st, const Workspace &w, int s, double *left, double *right, int64_t cap,
                  int64_t *counts_dev, cudaStream_t stream) {
    const b200pic_species &a = st.sp[s];
    PackArgs A;
    const double *src[7] = {a.x, a.y, a.z, a.px, a.py, a.pz, a.w};
    for (int f = 0; f < 7; ++f) A.src[f] = src[f];
    A.id = a.id;
    A.key = w.key[s];
    A.n_dev = a.n_dev;
    A.dst[0] = left;
    A.dst[1] = right;
    A.cap = cap;
    A.nk = w.nk;
    A.counts[0] = counts_dev;
    A.counts[1] = counts_dev + 1;
    A.err = st.err;
    A.has_z = st.cfg.dim == 3;
    CUDA_TRY(cudaMemsetAsync(counts_dev, 0, 2 * sizeof(int64_t), stream));
    k_pack_outgoing<<<grid_for(a.capacity), 256, 0, stream>>>(A);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

int append_particles(b200pic_state &st, const Workspace &w, int s, const double *recv, int64_t count, int64_t cap,
                     cudaStream_t stream) {
    if (count <= 0) return B200PIC_OK;
    const b200pic_species &a = st.sp[s];
    k_note_count<<<1, 1, 0, stream>>>(a.n_dev, w.aux + s);
    LAUNCH_CHECK();
    k_append<<<grid_for(count), 256, 0, stream>>>(a, recv, count, cap, st.cfg.dim == 3, st.err, w.aux + s);
    LAUNCH_CHECK();
    k_bump_count<<<1, 1, 0, stream>>>(a.n_dev, w.aux + s, count, a.capacity);
    LAUNCH_CHECK();
    // key the appended particles [first, first + count): patch/bin/anchor from their positions
    k_initial_keys<<<grid_for(count), 256, 0, stream>>>(st.cfg, a.x, a.y, a.z, a.n_dev, w.key[s], w.aux + s);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

// ---------------------------------------------------------------------------
// x-slab migration in one fixed-capacity message per direction, all species (no host read of counts):
// int64 counts[S], then per species [8][cap] doubles (x y z px py pz w id-bits)
// ---------------------------------------------------------------------------
size_t migrants_bytes(const b200pic_config &c, int64_t cap) {
    return (size_t)c.n_species * (1 + 8 * (size_t)cap) * sizeof(double);
}

int pack_migrants(b200pic_state &st, const Workspace &w, void *to_left, void *to_right, int64_t cap, cudaStream_t s) {
    const int S = st.cfg.n_species;
    CUDA_TRY(cudaMemsetAsync(to_left, 0, S * sizeof(int64_t), s));
    CUDA_TRY(cudaMemsetAsync(to_right, 0, S * sizeof(int64_t), s));
    for (int i = 0; i < S; ++i) {
        const b200pic_species &a = st.sp[i];
        PackArgs A;
        const double *src[7] = {a.x, a.y, a.z, a.px, a.py, a.pz, a.w};
        for (int f = 0; f < 7; ++f) A.src[f] = src[f];
        A.id = a.id;
        A.key = w.key[i];
        A.n_dev = a.n_dev;
        A.dst[0] = (double *)to_left + S + (int64_t)i * 8 * cap;
        A.dst[1] = (double *)to_right + S + (int64_t)i * 8 * cap;
        A.cap = cap;
        A.nk = w.nk;
        A.counts[0] = (int64_t *)to_left + i;
        A.counts[1] = (int64_t *)to_right + i;
        A.err = st.err;
        A.has_z = st.cfg.dim == 3;
        k_pack_outgoing<<<grid_for(a.capacity), 256, 0, s>>>(A);
        LAUNCH_CHECK();
    }
    return B200PIC_OK;
}

int unpack_migrants(b200pic_state &st, const Workspace &w, const void *from_left, const void *from_right, int64_t cap,
                    cudaStream_t s) {
    const int S = st.cfg.n_species;
    for (int i = 0; i < S; ++i) {
        const b200pic_species &a = st.sp[i];
        for (int d = 0; d < 2; ++d) {
            const double *msg = (const double *)(d ? from_right : from_left);
            const int64_t *cnt = (const int64_t *)msg + i;
            const double *recv = msg + S + (int64_t)i * 8 * cap;
            k_note_count<<<1, 1, 0, s>>>(a.n_dev, w.aux + i);
            LAUNCH_CHECK();
            k_append_dev<<<grid_for(cap), 256, 0, s>>>(a, recv, cnt, cap, st.cfg.dim == 3, st.err, w.aux + i);
            LAUNCH_CHECK();
            k_bump_count_dev<<<1, 1, 0, s>>>(a.n_dev, w.aux + i, cnt, cap, a.capacity, st.err);
            LAUNCH_CHECK();
            k_initial_keys<<<grid_for(cap), 256, 0, s>>>(st.cfg, a.x, a.y, a.z, a.n_dev, w.key[i], w.aux + i);
            LAUNCH_CHECK();
        }
    }
    return B200PIC_OK;
}

// ---------------------------------------------------------------------------
// compaction: materialise the sorted order (alt[j] = sp[perm[j]], perm = identity) so that the live
// particles are the prefix [0, n) of the current buffer (host downloads, diagnostics)
// ---------------------------------------------------------------------------
namespace {
__global__ void k_compact(b200pic_species src, b200pic_species dst, int32_t *perm, int has_z) {
    const int64_t n = *src.n_dev;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = perm[j];
        dst.x[j] = src.x[m];
        dst.y[j] = src.y[m];
        if (has_z) dst.z[j] = src.z[m];
        dst.px[j] = src.px[m];
        dst.py[j] = src.py[m];
        dst.pz[j] = src.pz[m];
        dst.w[j] = src.w[m];
        dst.id[j] = src.id[m];
        perm[j] = (int32_t)j;
    }
}
}  // namespace

// (patch, bin, anchor, id) order: every key's slice of perm sorted by particle id.  Not needed by
// the step (K1's J sums are exact integers, its items hold whole keys), so it runs only where a
// host sees the order: before a compaction.  No-op unless the keys match the slots (after a sort).
static int canonical_order(b200pic_state &st, const Workspace &w, cudaStream_t s) {
    const int S = st.cfg.n_species;
    const int64_t nk = w.nk;
    int64_t cap = 0;
    for (int i = 0; i < S; ++i) cap = st.sp[i].capacity > cap ? st.sp[i].capacity : cap;
    {
        // the cursors are dead after the scatter: their buffer holds the list of keys left to the
        // warp / CTA passes
        SegParams SG;
        memset(&SG, 0, sizeof(SG));
        SG.nk = nk;
        SG.long_n = w.long_n;
        for (int i = 0; i < S; ++i) {
            SegSpecies &q = SG.sp[i];
            q.offsets = st.sp[i].offsets;
            q.key = w.key[i];
            q.id = st.sp[i].id;
            q.perm = w.perm[i];
            q.list = reinterpret_cast<int32_t *>(w.cursor + (int64_t)i * nk);  // nk int64 = 2 nk int32 slots
            q.list2 = q.list + nk;
            q.scr_id = reinterpret_cast<int64_t *>(st.alt[i].x);
            q.scr_slot = reinterpret_cast<int64_t *>(st.alt[i].y);
        }
        const int sms = sm_count();
        const int64_t tiles = (cap + RANK_TILE - 1) / RANK_TILE;
        k_seg_tiles<<<dim3((unsigned)(tiles < 8 * sms ? (tiles < 1 ? 1 : tiles) : 8 * sms), S), RANK_THREADS, 0, s>>>(SG);
        LAUNCH_CHECK();
        k_seg_warp<<<dim3(sms * 4, S), 256, 0, s>>>(SG);
        LAUNCH_CHECK();
        k_seg_long<<<dim3(sms * (2048 / SEG_THREADS), S), SEG_THREADS, 0, s>>>(SG);
        LAUNCH_CHECK();
    }
    return B200PIC_OK;
}

// ---------------------------------------------------------------------------
// host-order mirror (drop-in calls on host buffers, engine.step_host): the host keeps a species' mutable
// fields in one fixed order; hmap[j] is the host slot of storage slot j of the current buffer.  The live
// storage slots are perm[p] for sorted positions p < n.
// ---------------------------------------------------------------------------
namespace {
__global__ void k_host_map_reset(int32_t *hmap, int64_t cap) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cap; j += (int64_t)gridDim.x * blockDim.x)
        hmap[j] = (int32_t)j;
}
// the map of the buffer the next K1 writes (storage slot = sorted position p): next[p] = hmap[perm[p]]
__global__ void k_host_map_advance(const int32_t *perm, const int64_t *n_dev, const int32_t *hmap, int32_t *next) {
    const int64_t n = *n_dev;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        next[p] = __ldg(hmap + __ldg(perm + p));
}
// to_host: stage[hmap[j]] = cur[j]; else cur[j] = stage[hmap[j]] (j = perm[p], p < n) for x y [z] px py pz
__global__ void k_host_exchange(b200pic_species cur, b200pic_species stage, const int32_t *perm, const int32_t *hmap,
                                int has_z, int to_host) {
    const int64_t n = *cur.n_dev;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = __ldg(perm + p), h = __ldg(hmap + j);
        double *c[6] = {cur.x, cur.y, cur.z, cur.px, cur.py, cur.pz};
        double *g[6] = {stage.x, stage.y, stage.z, stage.px, stage.py, stage.pz};
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            if (k == 2 && !has_z) continue;
            if (to_host) g[k][h] = c[k][j];
            else c[k][j] = g[k][h];
        }
    }
}
}  // namespace

int host_map_reset(b200pic_state &st, int s, int32_t *hmap, cudaStream_t stream) {
    k_host_map_reset<<<grid_for(st.sp[s].capacity), 256, 0, stream>>>(hmap, st.sp[s].capacity);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

int host_map_advance(b200pic_state &st, const Workspace &w, int s, const int32_t *hmap, int32_t *next,
                     cudaStream_t stream) {
    k_host_map_advance<<<grid_for(st.sp[s].capacity), 256, 0, stream>>>(w.perm[s], st.sp[s].n_dev, hmap, next);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

// the staging side is the alternate buffer set (free between steps: K1 writes it, the sort reads only keys)
int host_exchange(b200pic_state &st, const Workspace &w, int s, const int32_t *hmap, int to_host, cudaStream_t stream) {
    k_host_exchange<<<grid_for(st.sp[s].capacity), 256, 0, stream>>>(st.sp[s], st.alt[s], w.perm[s], hmap,
                                                                     st.cfg.dim == 3, to_host);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

__global__ void k_keys_stale(int32_t *long_n) { long_n[2 * B200PIC_MAX_SPECIES] = 0; }

int compact(b200pic_state &st, const Workspace &w, cudaStream_t s) {
    int rc = canonical_order(st, w, s);
    if (rc) return rc;
    for (int i = 0; i < st.cfg.n_species; ++i) {
        k_compact<<<grid_for(st.sp[i].capacity), 256, 0, s>>>(st.sp[i], st.alt[i], w.perm[i], st.cfg.dim == 3);
        LAUNCH_CHECK();
    }
    k_keys_stale<<<1, 1, 0, s>>>(w.long_n);  // slots moved, keys did not
    LAUNCH_CHECK();
    swap_buffers(st);
    return B200PIC_OK;
}
