// sort.cuh -- workspace layout and the K5 / item-build entry points.
#pragma once
#include "k1.cuh"

struct Workspace {
    int64_t nk;
    int32_t *key[B200PIC_MAX_SPECIES];  // destination key per particle (written by K1)
    int32_t *perm[B200PIC_MAX_SPECIES]; // sorted position -> storage slot (built by K5, read by K1)
    int64_t *counts, *scanned, *cursor; // counting sort
    int64_t *nch, *nch_scan;            // chunks per (species, key)
    int64_t *scan_tmp;
    K1Item *items;
    IlPair *ilp;                        // (k1_merge 2) K1_IL_PAIRS per item
    int64_t max_items;
    int32_t *n_items, *queue, *long_n;  // long_n[2][species]: K5 keys left to the warp / CTA passes
    int64_t *aux;                       // per-species scratch scalars (slab migration)
    unsigned long long *jw;             // max over stencil anchors of sum_s count_s j_bound_s (double bits)
    int32_t *fbits;                     // this step's J tile fraction bits F (k_jbits) ...
    double *fscale;                     // ... and 2^(44 + F)
    int32_t *jsafe;                     // 1: the host's F (cfg.j_fine_bits) is within this step's bound
    size_t bytes;
};

Workspace carve(const b200pic_state &st);
int scan_exclusive(const int64_t *in, int64_t *out, int64_t n, int64_t *tmp, cudaStream_t s);
int sort_by_keys(b200pic_state &st, const Workspace &w, cudaStream_t s);
void swap_buffers(b200pic_state &st);
int compact(b200pic_state &st, const Workspace &w, cudaStream_t s);
int host_map_reset(b200pic_state &st, int s, int32_t *hmap, cudaStream_t stream);
int host_map_advance(b200pic_state &st, const Workspace &w, int s, const int32_t *hmap, int32_t *next,
                     cudaStream_t stream);
int host_exchange(b200pic_state &st, const Workspace &w, int s, const int32_t *hmap, int to_host, cudaStream_t stream);
int initial_keys(b200pic_state &st, const Workspace &w, cudaStream_t s);
int build_items(b200pic_state &st, const Workspace &w, cudaStream_t s);
// K1 work items over both species: 0 no, 1 pairs split by species, 2 interleaved by anchor
int merged_items(const b200pic_config &c);
int pack_outgoing(b200pic_state &st, const Workspace &w, int s, double *left, double *right, int64_t cap,
                  int64_t *counts_dev, cudaStream_t stream);
int append_particles(b200pic_state &st, const Workspace &w, int s, const double *recv, int64_t count, int64_t cap,
                     cudaStream_t stream);
size_t migrants_bytes(const b200pic_config &c, int64_t cap);
int pack_migrants(b200pic_state &st, const Workspace &w, void *to_left, void *to_right, int64_t cap, cudaStream_t s);
int unpack_migrants(b200pic_state &st, const Workspace &w, const void *from_left, const void *from_right, int64_t cap,
                    cudaStream_t s);
