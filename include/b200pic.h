/*
 * b200pic.h -- C ABI of the B200 (sm_100a) PIC macro-particle hot path.
 *
 * Drop-in boundary for the reference "taskpic" operator path
 * (/root/reference/pkg/src/taskpic).  Every entry point takes plain device
 * pointers, sizes and scalars, runs asynchronously on the given CUDA stream
 * (NULL = legacy default stream) and returns an int status (B200PIC_OK = 0).
 * No torch or C++ types cross this boundary.
 *
 * Two layers:
 *  (1) operator level -- the reference kernels' own signatures, on device
 *      arrays, for the _Engine methods (scheduler.py:113-170):
 *        b200pic_gather_fields_2d   <- kernels.gather_fields    kernels.py:51-54
 *        b200pic_boris_push         <- kernels.boris_push       kernels.py:124-126
 *        b200pic_flag_boundaries    <- kernels.flag_boundaries  kernels.py:165-166
 *        b200pic_esirkepov_project_2d <- kernels.esirkepov_project kernels.py:181-184
 *        b200pic_deposit_rho_2d     <- kernels.deposit_rho      kernels.py:269-271
 *        b200pic_reduce_subgrid     <- fields.reduce_bin_currents fields.py:101-114
 *      Sentinels (first bad index, or -1) are written to a device int64 and
 *      read back by the host facade, which raises FloatingPointError like
 *      scheduler.py:135-139 / 162-166.
 *  (2) step level -- the fused device path replacing one run_simulation
 *      iteration body (scheduler.py:438-489):
 *        b200pic_step_particles  K1: interpolate+push+pre-BC+project+reduce for
 *                                all (species, patch, bin, chunk) work items
 *                                (replaces _OffDriver.work / the task graph)
 *        b200pic_sort_particles  K5: BC + migration + (patch, bin) re-sort
 *                                (exchange.apply_particle_bc_and_migrate, exchange.py:196-258)
 *        b200pic_fold_currents   K3: ghost fold of the int64 J accumulators
 *                                (exchange.sum_current_ghosts, exchange.py:134-147)
 *        b200pic_maxwell         K2: synced Yee step + field ghost sync
 *                                (fields.maxwell_step fields.py:130-190 + exchange.sync_field_ghosts 150-156)
 *        b200pic_sync_fields     K4: E/B ghost pull
 *        b200pic_step            all of the above, in order
 */
#ifndef B200PIC_H
#define B200PIC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B200PIC_MAX_SPECIES 8
#define B200PIC_GHOST 3
#define B200PIC_J_SCALE_BITS 44

enum {
    B200PIC_OK = 0,
    B200PIC_ERR_NONFINITE = 1, /* boris_push sentinel  -> FloatingPointError */
    B200PIC_ERR_COURANT = 2,   /* esirkepov sentinel   -> FloatingPointError */
    B200PIC_ERR_INVARIANT = 3, /* arena.py:69-73       -> InvariantError      */
    B200PIC_ERR_ARG = 4,
    B200PIC_ERR_CAPACITY = 5,
    B200PIC_ERR_CUDA = 6
};

/* periodic / reflective: the reference's kinds (config.py:20-22); absorbing (beyond the reference, BASELINE
 * config 1): particles leaving through the wall are deleted, fields see a first-order Silver-Mueller wall */
enum { B200PIC_BC_PERIODIC = 0, B200PIC_BC_REFLECTIVE = 1, B200PIC_BC_ABSORBING = 2 };

/* Grid/decomposition (config.py:93-190, plus z for 3D).  Field arrays are
 * whole-domain (or whole-slab) arrays with 3 ghost layers on every side:
 * extent L[a] + 1 + 2*3 per axis, C order, x slowest (fields.py:1-20). */
typedef struct b200pic_config {
    int32_t dim;     /* 2 (2D3V) or 3 */
    int32_t L[3];    /* cells per axis (L[2] = 1 in 2D) */
    int32_t pn[3];   /* patch extent in cells */
    int32_t np[3];   /* patches per axis */
    int32_t bx;      /* bin_x_size */
    int32_t bc[3];   /* B200PIC_BC_* per axis */
    double d[3];     /* dx, dy, dz */
    double dt;
    int32_t n_species;
    int32_t chunk;   /* max particles per K1 work item (dense bins are split) */
    int32_t k1_variant;      /* 2: warp-specialised producer/consumer K1 (default), 0: one role per warp, 1: per-particle shared atomics */
    int32_t k1_stage_fields; /* 1: stage the E/B stencil tile in shared memory, 0: gather through L1 */
    int32_t k1_static;       /* 1: "tasks off" analogue -- CTA b takes items b, b + grid, ... (no work queue);
                                0: persistent CTAs pull items from an atomic queue (the paper's dynamic tasks) */
    int32_t j_fine_bits;     /* K1 J tile: 64-bit fixed point at quantum 2^-(44+F); this is the largest F the host
                                allows (every single contribution c must keep |c| 2^(44+F) < 2^51); each step
                                the item build lowers F so that the densest stencil window's worst-case sum
                                fits the tile (see j_bound) */
    /* x-slab decomposition (multi-GPU): this rank owns global cells
     * [x0, x0 + L[0]) of a periodic-in-x domain of gL0 cells (gnp0 patches).  slab = 0: whole domain. */
    int32_t slab;
    int32_t x0;
    int32_t gL0;
    int32_t gnp0;
    int32_t k1_merge;        /* (3D, two species, variant 2) work items per (patch, bin) over both species:
                                0 no (items of one species, the reference's reduction granularity),
                                1 the producer/consumer pairs shared out by species,
                                2 both species interleaved by anchor (consumer runs span species) */
    int32_t k1_sparse;       /* 1: (3D warp-specialised K1) register split for sparse plasma: 160 / 96 per
                                producer / consumer thread instead of 168 / 88 (short anchor runs make the
                                consumers' flushes weigh more); the host sets it from particles per bin */
    double charge[B200PIC_MAX_SPECIES];
    double mass[B200PIC_MAX_SPECIES];
    /* largest current one particle of species s can add to one J node in a step: 0.75 |q_s| max w_s (the
     * Esirkepov prefix moves by at most |v| dt / d < 1 cell, times at most 0.75 of transverse weight) */
    double j_bound[B200PIC_MAX_SPECIES];
} b200pic_config;

/* One species' device SoA (arena.py:17-56) in canonical (patch, bin) order.
 * z == NULL in 2D.  offsets: device int64[n_patches*n_bins + 1].
 * n_dev: device int64 holding the live count (kept on device so the step can
 * be captured in a CUDA graph). */
typedef struct b200pic_species {
    double *x, *y, *z, *px, *py, *pz, *w;
    int64_t *id;
    int64_t *offsets;
    int64_t *n_dev;
    int64_t capacity;
} b200pic_species;

typedef struct b200pic_fields {
    double *e[6];        /* ex ey ez bx by bz */
    double *j[3];        /* jx jy jz (float currents, fields.py:77-81) */
    int64_t *jacc[3];    /* fixed-point accumulators, quantum 2^-44 (fields.py:63-75) */
    double *e_alt[6];    /* optional (NULL: unused) second E/B set of the same shape: with every axis periodic
                            and the whole domain, b200pic_maxwell runs the fused Yee step from e into e_alt and
                            swaps the two sets (e always names the current fields) */
} b200pic_fields;

/* Full device state of one rank.  `alt` is the ping-pong particle buffer used
 * by the re-sort; `work` is scratch of b200pic_workspace_bytes() bytes;
 * `err` is a device int64[8] sticky error record: err[0] = bitmask of codes
 * raised, err[code] = smallest offending particle id (INT64_MAX if none). */
typedef struct b200pic_state {
    b200pic_config cfg;
    b200pic_species sp[B200PIC_MAX_SPECIES];
    b200pic_species alt[B200PIC_MAX_SPECIES];
    b200pic_fields f;
    void *work;
    size_t work_bytes;
    int64_t *err;
} b200pic_state;

int b200pic_version(void);
const char *b200pic_error_string(int code);
/* number of kernels this library has launched so far (host-side counter) */
int64_t b200pic_launch_count(void);
/* sizeof of the ABI structs (0 config, 1 species, 2 fields, 3 state): lets a binding verify its layout */
size_t b200pic_abi_size(int which);
/* the K1 template instantiation b200pic_step_particles launches for this config (e.g.
 * "k1_ws<3, true, 1, true>"): lets tests assert that the benchmarked kernel is the one they cover */
const char *b200pic_k1_kernel_name(const b200pic_config *cfg);
/* K1 work items: 0 one species per item (the reference's granularity), 2 both species of a (patch, bin)
 * interleaved by stencil anchor (3D, two species; J still rounded per species) */
int b200pic_k1_items_mode(const b200pic_config *cfg);
/* persistent K1 CTAs per launch on the current device (the report's workers_per_collection) */
int b200pic_k1_grid(const b200pic_config *cfg);
/* 1 if K1 stages the E/B stencil tile in shared memory by default for this config (it fits) */
int b200pic_k1_stage_default(const b200pic_config *cfg);
/* scratch bytes needed by the step-level calls for these capacities */
size_t b200pic_workspace_bytes(const b200pic_config *cfg, const int64_t *capacity);

/* ---------------- operator level (reference kernel signatures) ---------- */
/* fields[6]: ex..bz arrays with row length e1 (C order); out-params as in kernels.py:51-54 */
int b200pic_gather_fields_2d(const double *x, const double *y, int64_t s0, int64_t s1,
                             const double *const fields[6], int64_t e1, int64_t *cix, int64_t *ciy,
                             double *dlx, double *dly, double *const gathered[6], double inv_dx,
                             double inv_dy, int64_t cell0x, int64_t cell0y, void *stream);
/* bad_dev: device int64, set to the first non-finite index or -1 (kernels.py:160-162); z may be NULL */
int b200pic_boris_push(double *x, double *y, double *z, double *px, double *py, double *pz, int64_t s0,
                       int64_t s1, const double *const gathered[6], double charge, double mass, double dt,
                       int64_t *bad_dev, void *stream);
/* bounds: xmin,xmax,ymin,ymax[,zmin,zmax] (host array); z may be NULL */
int b200pic_flag_boundaries(const double *x, const double *y, const double *z, int64_t s0, int64_t s1,
                            uint8_t *flags, const double *bounds, void *stream);
int b200pic_esirkepov_project_2d(const double *x, const double *y, const double *px, const double *py,
                                 const double *pz, const double *weight, int64_t s0, int64_t s1,
                                 const int64_t *cix, const int64_t *ciy, const double *dlx, const double *dly,
                                 double *jx, double *jy, double *jz, int64_t e1, double charge, double mass,
                                 double inv_dx, double inv_dy, double dx_over_dt, double dy_over_dt,
                                 int64_t sub_cell0x, int64_t sub_cell0y, int64_t *bad_dev, void *stream);
int b200pic_deposit_rho_2d(const double *x, const double *y, const double *weight, int64_t s0, int64_t s1,
                           double *rho, int64_t e1, double charge, double inv_dx, double inv_dy, int64_t cell0x,
                           int64_t cell0y, void *stream);
/* acc[x_shift + i, :] += rint(sub[i, :] * 2^44); sub zeroed (fields.py:101-114) */
int b200pic_reduce_subgrid(double *sub, int64_t sub_rows, int64_t e1, int64_t *acc, int64_t x_shift, void *stream);

/* ---------------- step level (fused device path) ------------------------- */
/* On-device loader for perf-size runs: ppc particles per cell over cells x in [x_cell0, x_cell0 + x_cells),
 * uniform in-cell positions, Gaussian momenta (sigma), equal weights, ids id0.. (counter-based RNG, seed).
 * Fills sp[species] from index 0 and sets its device count; follow with b200pic_initial_sort. */
int b200pic_load_uniform(b200pic_state *st, int species, int64_t ppc, double sigma, double weight, uint64_t seed,
                         int64_t x_cell0, int64_t x_cells, int64_t id0, void *stream);
/* Density-profile loader (BASELINE configs 1, 3, 4): lambda(cell) = max(floor, background (x range + linear
 * up-ramp) + Gaussian component + sphere component); per-cell count Poisson(lambda) or floor+Bernoulli.
 * Gaussian/sphere particles get (sigma_hot, drift), background ones sigma_bg.  Cells and lengths in cells. */
typedef struct b200pic_profile {
    double ppc_bg, bg_x0, bg_x1, ramp_cells, floor_ppc;
    double gauss_peak, gauss_c[3], gauss_s[3]; /* gauss_s[a] <= 0: uniform along a */
    double sphere_ppc, sphere_c[3], sphere_r;
    double sigma_bg, sigma_hot, drift[3];
    double weight;
    int32_t poisson;
    int32_t _pad;
} b200pic_profile;
/* pass 1: counts[c] for the slab's cells (C order over [x_cell0, x_cell0 + x_cells) x Ly x Lz) */
int b200pic_profile_count(b200pic_state *st, int species, const b200pic_profile *prof, uint64_t seed,
                          int64_t x_cell0, int64_t x_cells, int64_t *counts, void *stream);
/* pass 2: offsets = exclusive scan of counts (n_cells + 1 entries); writes sp[species] and its count.
 * ids = global cell index * 4096 + rank in cell (unique for < 4096 particles per cell, < 2^40) */
int b200pic_profile_fill(b200pic_state *st, int species, const b200pic_profile *prof, uint64_t seed,
                         int64_t x_cell0, int64_t x_cells, const int64_t *offsets, void *stream);
int b200pic_initial_sort(b200pic_state *st, void *stream);   /* canonical (patch, bin) order + offsets */
int b200pic_step_particles(b200pic_state *st, void *stream); /* K1 */
/* K1 with a per-work-item trace (the reference's TraceEvent, runtime.py:33-42 / scheduler.py:362-394):
 * row i (B200PIC_TRACE_WORDS u64, indexed by work item) = begin ns, end ns (%globaltimer), SM id, CTA,
 * species, key (patch * n_bins + bin), first particle, count; rows >= trace_rows are not written.
 * *n_items_out (device) receives the item count of this launch. */
#define B200PIC_TRACE_WORDS 8
int b200pic_step_particles_traced(b200pic_state *st, unsigned long long *trace, int64_t trace_rows,
                                  int32_t *n_items_out, void *stream);
int b200pic_sort_particles(b200pic_state *st, void *stream); /* K5 (swaps sp <-> alt) */
int b200pic_build_items(b200pic_state *st, void *stream);    /* K1 work items from sp[].offsets */
/* out_dev[0] (device int32) = the number of K1 work items the next b200pic_step_particles executes (the
 * reference report's executed_units, scheduler.py:68) */
int b200pic_n_items(b200pic_state *st, int32_t *out_dev, void *stream);
/* out_dev[0] = F, out_dev[1] = 2^(44+F): the J tile units the next K1 uses (set by the last item build) */
int b200pic_j_units(b200pic_state *st, double *out_dev, void *stream);
/* K5 only builds a permutation (sorted position -> storage slot) that the next K1 reads through;
 * b200pic_compact materialises it: afterwards the live particles are sp[s][0, n) in canonical order */
int b200pic_compact(b200pic_state *st, void *stream);
/* Host-order mirror for drop-in calls on host buffers (engine.Simulation.step_host): the host keeps one
 * species' mutable fields (x y [z] px py pz) in a fixed order, and the immutable w / id are never re-sent.
 * hmap (device int32[capacity], owned by the caller) maps each storage slot of the current buffer sp[s] to its
 * host slot; the live storage slots are perm[p], p < n.
 *   b200pic_host_map_reset:    hmap = identity (after b200pic_compact: host order = canonical order)
 *   b200pic_host_map_advance:  next = the map of the buffer the next K1 writes (next[p] = hmap[perm[p]])
 *   b200pic_host_exchange:     to_host 1: alt[hmap[j]] = sp[j]; 0: sp[j] = alt[hmap[j]] -- the alternate
 *                              buffer set is the host-order staging area (free between steps) */
int b200pic_host_map_reset(b200pic_state *st, int species, int32_t *hmap, void *stream);
int b200pic_host_map_advance(b200pic_state *st, int species, const int32_t *hmap, int32_t *next, void *stream);
int b200pic_host_exchange(b200pic_state *st, int species, const int32_t *hmap, int to_host, void *stream);
int b200pic_fold_currents(b200pic_state *st, void *stream);  /* K3 */
int b200pic_maxwell(b200pic_state *st, void *stream);        /* K2 (+ J convert, acc zero) */
/* K2 as shipped (compatibility mode, whole domain, periodic / reflective): maxwell_step fields.py:130-143
 * on every patch with the ghosts of the previous sync (stale by half / one step at the seams, SURVEY.md
 * §0.1 #3), then sync_field_ghosts (scheduler.py:478-484) */
int b200pic_maxwell_lagged(b200pic_state *st, void *stream);
int b200pic_sync_fields(b200pic_state *st, void *stream);    /* K4 */
/* The rest of a step after K1: K5 on `stream`, K3 + K2 on an auxiliary stream beside it (they touch
 * disjoint data), joined back into `stream` (capturable).  One b200pic_step = step_particles + this. */
int b200pic_step_rest(b200pic_state *st, void *stream);
int b200pic_step(b200pic_state *st, int n_steps, void *stream);

/* ---------------- K7 device diagnostics (diagnostics.py:30-87) ------------- */
/* out_dev[0] = field energy 0.5 sum F^2 over owned nodes, out_dev[1] = kinetic sum m w (gamma - 1) */
int b200pic_energy(b200pic_state *st, double *out_dev, void *stream);
/* order-2 rho at primal nodes into a whole-domain array (ghosts folded; x ghosts stay with a slab) */
int b200pic_charge_density(b200pic_state *st, double *rho, void *stream);
/* r = div E - rho on owned primal nodes (backward differences); r_out (optional) receives r, and
 * max_dev[0] = max |r - r0| (r0 optional) */
int b200pic_gauss_residual(b200pic_state *st, const double *rho, const double *r0, double *r_out, double *max_dev,
                           void *stream);

/* ---------------- x-slab pieces (multi-GPU; the host exchanges x planes over NCCL) ---------------- */
/* Yee sub-steps on owned nodes (fields.py:146-190); full-E also converts/clears the J accumulators */
int b200pic_yee_half_b(b200pic_state *st, void *stream);
int b200pic_yee_full_e(b200pic_state *st, void *stream);
int b200pic_yee_pin_walls(b200pic_state *st, void *stream);
/* ghost pull (E/B components [comp0, comp0+ncomp)) / J ghost fold along the axes in axis_mask (bit a = axis a),
 * in x, y, z order -- the host runs the x exchange first and passes axis_mask = 6 in slab mode */
int b200pic_sync_axes(b200pic_state *st, int comp0, int ncomp, int axis_mask, void *stream);
int b200pic_fold_axes(b200pic_state *st, int axis_mask, void *stream);
/* particles whose destination patch lies outside the slab (K1 key = n_keys + 0 left / + 1 right) are packed
 * into send[dir] (layout [8][cap] doubles: x y z px py pz w id-bits); counts_dev[2] receives the counts */
int b200pic_pack_outgoing(b200pic_state *st, int species, double *send_left, double *send_right, int64_t cap,
                          int64_t *counts_dev, void *stream);
/* append `count` received particles (same layout, row stride cap) after the live ones and key them */
int b200pic_append_particles(b200pic_state *st, int species, const double *recv, int64_t count, int64_t cap,
                             void *stream);
/* Device-driven slab exchange (two messages per step, no host read; slab.py):
 *  1. after K1: the migrants -- every species' outgoing particles in one fixed-capacity block per
 *     direction, int64 counts[S] then per species [8][cap] doubles (overflow raises B200PIC_ERR_CAPACITY,
 *     sticky) -- and the J accumulator x planes (which 0: 2G+1 planes per face, summed on receipt, so both
 *     sides of a face hold the full sums on the shared planes);
 *  2. after b200pic_maxwell_slab (the Yee step with the x halo updated redundantly): the E / B planes it
 *     leaves stale (which 2: two per face, planes K1 never reads -- the exchange may overlap the next K1).
 * which 1 refreshes every E / B ghost plane (start of a run). */
size_t b200pic_migrants_bytes(const b200pic_config *cfg, int64_t cap);
int b200pic_pack_migrants(b200pic_state *st, void *to_left, void *to_right, int64_t cap, void *stream);
int b200pic_unpack_migrants(b200pic_state *st, const void *from_left, const void *from_right, int64_t cap,
                            void *stream);
size_t b200pic_xplanes_bytes(const b200pic_config *cfg, int which);
int b200pic_xplanes_pack(b200pic_state *st, int which, void *to_left, void *to_right, void *stream);
int b200pic_xplanes_unpack(b200pic_state *st, int which, const void *from_left, const void *from_right,
                           void *stream);
int b200pic_maxwell_slab(b200pic_state *st, void *stream);
/* reads the sticky device error record (synchronises the stream) */
int b200pic_check_error(b200pic_state *st, void *stream, int64_t *bad_id);
/* frees the host-side resources the library keeps per state (the auxiliary stream of b200pic_step_rest);
 * call before freeing the state's workspace */
int b200pic_release(b200pic_state *st);
int b200pic_clear_error(b200pic_state *st, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* B200PIC_H */
