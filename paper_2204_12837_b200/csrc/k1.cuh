// k1.cuh -- parameter blocks shared by the step-level kernels.
#pragma once
#include <cuda.h>  // CUtensorMap (TMA descriptors of the E/B staging)

#include "particle_math.cuh"

#ifndef K1_THREADS
#define K1_THREADS 256
#endif

struct K1Item {
    int64_t start;    // first particle of the chunk
    int64_t start1;   // (species == -1) first particle of species 1's part
    int32_t count;    // particles in the chunk (<= cfg.chunk)
    int32_t count1;   // (species == -1) particles of species 1
    int32_t key;      // patch_flat * n_bins + bin (exchange/arena canonical key)
    int32_t species;  // -1: both species share the item, pairs split by species (k1_merge 1);
                      // -2: both species interleaved by anchor (k1_merge 2): start / start1 hold the item's
                      // anchor range [a0, a1) inside the bin, count / count1 the two species' particles
};

// (k1_merge 2) per item, per producer/consumer pair: its anchor range starts at bin-local anchor a0 with
// sorted positions b0 / b1 of species 0 / 1 and holds n particles of both (cuts balanced by count,
// computed when the items are built, csrc/sort.cu k_emit_items)
struct IlPair {
    int64_t b0, b1;
    int32_t a0, n;
};
constexpr int K1_IL_PAIRS = 8;  // = WS_PAIRS

// merged items (species == -1): the 8 producer/consumer pairs are shared out between the two species
// in proportion to their counts (each pair works on one species; at least one pair per non-empty part)
__host__ __device__ __forceinline__ int merged_pairs0(int64_t c0, int64_t c1, int pairs) {
    if (c1 <= 0) return pairs;
    if (c0 <= 0) return 0;
    int n0 = (int)((2 * c0 * pairs + (c0 + c1)) / (2 * (c0 + c1)));  // round(pairs * c0 / (c0 + c1))
    return n0 < 1 ? 1 : (n0 > pairs - 1 ? pairs - 1 : n0);
}
// species and particle range [w0, w1) of pair p in an item
__host__ __device__ __forceinline__ void item_segment(const K1Item &it, int p, int pairs, int &s, int64_t &w0,
                                                      int64_t &w1) {
    int64_t start = it.start, count = it.count;
    int k = p, n = pairs;
    s = it.species;
    if (it.species < 0) {
        const int n0 = merged_pairs0(it.count, it.count1, pairs);
        if (p < n0) { s = 0; n = n0; }
        else { s = 1; k = p - n0; n = pairs - n0; start = it.start1; count = it.count1; }
    }
    const int64_t seg = (count + n - 1) / n;
    w0 = start + k * seg;
    w1 = w0 + seg < start + count ? w0 + seg : start + count;
}

// K1 reads a species through the sort permutation (src[perm[j]]) and writes the updated record
// contiguously at j of the other buffer (dst): the re-sort (K5) only builds perm
struct K1Species {
    const double *x, *y, *z, *px, *py, *pz, *w;
    const int64_t *id;
    double *dx, *dy, *dz, *dpx, *dpy, *dpz, *dw;
    int64_t *did;
    const int32_t *perm;
    const int64_t *off;  // sorted-position offsets per (bin, anchor) key (k1_merge 2 walks them)
    int32_t *key;
    double charge, mass, qd2, inv_m2;
};

struct K1Params {
    // (BASELINE geometry, csrc/k1_particles.cu g8) TMA descriptors of the six E/B arrays, one 3D box per
    // component; the kernel takes K1Params as a __grid_constant__ so their addresses are param space
    alignas(64) CUtensorMap tmap[6];
    b200pic_config cfg;
    K1Species sp[B200PIC_MAX_SPECIES];
    const double *e[6];
    int64_t *jacc[3];
    const K1Item *items;
    const IlPair *ilp;   // (k1_merge 2) K1_IL_PAIRS entries per item
    const int32_t *n_items;
    int32_t *queue;
    int64_t *err;
    double inv[3], d_over_dt[3], Lw[3];
    double inv_pn[3];  // 1 / patch extent (cheap integer division, common.cuh fdiv)
    const double *fscale_dev;  // 2^(44 + F): J tile fixed-point scale (F set per step by the item build,
    const int *fbits_dev;      // csrc/sort.cu k_jbits; K1 reads both once into shared memory)
    double fscale_host;        // the host's F (cfg.j_fine_bits) as kernel constants: the fast path, valid while
    int fbits_host;            // this step's device bound allows it ...
    const int *jsafe_dev;      // ... which k_jbits writes here (csrc/k1_particles.cu k1_ws DEVF)
    int ablate;       // profiling experiments only (env B200PIC_ABLATE): 1 no run flush, 2 no Phase B, 4 no tile flush,
                      // 16 no species-1 low-bits updates
    int64_t anchors;  // sort keys per bin (anchors_per_bin)
    int64_t n_keys;   // sort keys per species
    unsigned long long *trace;  // optional per-item trace rows (b200pic_step_particles_traced), else null
    int64_t trace_rows;
};

int k1_smem_bytes(const b200pic_config &c);
// 1 if K1 items may interleave both species (k1_merge 2): the instantiation, with its species-1 low-bits
// tile, fits in shared memory (csrc/sort.cu merged_items falls back to per-species items otherwise)
int k1_il_fits(const b200pic_config &c);
int k1_stage_default(const b200pic_config &c);
int k1_grid(const b200pic_config &c);
const char *k1_kernel_name(const b200pic_config &c);
int launch_k1(const K1Params &P, int grid, cudaStream_t s);
