// step.cu -- step-level C ABI (include/b200pic.h): one run_simulation
// iteration body (scheduler.py:438-489) as K1 -> K5 -> K3 -> K2 on a stream.
#include "fields.cuh"
#include "sort.cuh"

#include <stdlib.h>

#include <map>
#include <mutex>
#include <string>
#include <tuple>

long long g_b200pic_launches = 0;

namespace {

bool valid(const b200pic_state *st) {
    if (!st) return false;
    const b200pic_config &c = st->cfg;
    if (c.dim != 2 && c.dim != 3) return false;
    if (c.n_species < 1 || c.n_species > B200PIC_MAX_SPECIES) return false;
    if (c.bx <= 0 || c.pn[0] % c.bx) return false;
    for (int a = 0; a < c.dim; ++a)
        if (c.L[a] <= 0 || c.pn[a] <= 0 || c.np[a] * c.pn[a] != c.L[a]) return false;
    if (c.bc[1] == B200PIC_BC_ABSORBING || c.bc[2] == B200PIC_BC_ABSORBING) return false;  // x only
    if (c.slab && (c.bc[0] != B200PIC_BC_PERIODIC || c.x0 < 0 || c.x0 % c.pn[0] || c.gnp0 * c.pn[0] != c.gL0 ||
                   c.x0 + c.L[0] > c.gL0))
        return false;
    if (!st->work || !st->err) return false;
    for (int k = 0; k < 6; ++k)
        if (!st->f.e[k]) return false;
    for (int s = 0; s < c.n_species; ++s) {
        const b200pic_species &a = st->sp[s], &b = st->alt[s];
        if (!a.x || !a.y || !a.px || !a.py || !a.pz || !a.w || !a.id || !a.offsets || !a.n_dev) return false;
        if (!b.x || !b.y || !b.px || !b.py || !b.pz || !b.w || !b.id) return false;
        if (c.dim == 3 && (!a.z || !b.z)) return false;
    }
    return true;
}

__global__ void k_j_units(const int32_t *fbits, const double *fscale, double *out) {
    out[0] = (double)*fbits;
    out[1] = *fscale;
}

__global__ void k_clear_err(int64_t *err) {
    int t = threadIdx.x;
    if (t < 8) err[t] = t == 0 ? 0 : INT64_MAX;
}

std::mutex g_host_mutex;  // the host-side caches below (several states / threads may step at once)

// K1 grid (SMs x resident CTAs) per (device, kernel instantiation, dynamic shared memory)
int k1_grid_cached(const b200pic_config &c) {
    static std::map<std::tuple<int, std::string, int>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(dev, std::string(k1_kernel_name(c)), k1_smem_bytes(c));
    std::lock_guard<std::mutex> lock(g_host_mutex);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    const int g = k1_grid(c);
    cache[key] = g;
    return g;
}

// auxiliary stream of one state (keyed by its workspace) for the field half of a step (K3 fold + K2
// Yee), which touches no particle data and so runs beside the K5 re-sort; fork / join by events
// (capturable).  Per state: two simulations stepping on different streams never share the events.
struct AuxStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
std::map<const void *, AuxStream> g_aux;

AuxStream *aux_stream(const b200pic_state *st) {
    std::lock_guard<std::mutex> lock(g_host_mutex);
    AuxStream &a = g_aux[st->work];
    if (!a.s) {
        if (cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming) != cudaSuccess) {
            g_aux.erase(st->work);
            return nullptr;
        }
    }
    return &a;
}

}  // namespace

extern "C" {

int b200pic_version(void) { return 100; }

int64_t b200pic_launch_count(void) { return g_b200pic_launches; }

const char *b200pic_k1_kernel_name(const b200pic_config *cfg) { return cfg ? k1_kernel_name(*cfg) : ""; }

int b200pic_k1_items_mode(const b200pic_config *cfg) { return cfg ? merged_items(*cfg) : 0; }

int b200pic_k1_grid(const b200pic_config *cfg) { return cfg ? k1_grid_cached(*cfg) : 0; }

int b200pic_k1_stage_default(const b200pic_config *cfg) { return cfg ? k1_stage_default(*cfg) : 0; }

size_t b200pic_abi_size(int which) {
    switch (which) {
        case 0: return sizeof(b200pic_config);
        case 1: return sizeof(b200pic_species);
        case 2: return sizeof(b200pic_fields);
        case 3: return sizeof(b200pic_state);
        default: return 0;
    }
}

const char *b200pic_error_string(int code) {
    switch (code) {
        case B200PIC_OK: return "ok";
        case B200PIC_ERR_NONFINITE: return "non-finite momentum";
        case B200PIC_ERR_COURANT: return "particle moved more than one cell per step (Courant violation)";
        case B200PIC_ERR_INVARIANT: return "particle outside its patch cell range (missed exchange?)";
        case B200PIC_ERR_ARG: return "invalid argument";
        case B200PIC_ERR_CAPACITY: return "capacity exceeded";
        case B200PIC_ERR_CUDA: return "CUDA error";
        default: return "unknown";
    }
}

size_t b200pic_workspace_bytes(const b200pic_config *cfg, const int64_t *capacity) {
    if (!cfg) return 0;
    b200pic_state st;
    memset(&st, 0, sizeof(st));
    st.cfg = *cfg;
    for (int s = 0; s < cfg->n_species && s < B200PIC_MAX_SPECIES; ++s) st.sp[s].capacity = capacity[s];
    st.work = (void *)0;
    Workspace w = carve(st);
    return w.bytes + 256;
}

int b200pic_release(b200pic_state *st) {
    if (!st) return B200PIC_ERR_ARG;
    std::lock_guard<std::mutex> lock(g_host_mutex);
    auto it = g_aux.find(st->work);
    if (it != g_aux.end()) {
        cudaStreamSynchronize(it->second.s);
        cudaStreamDestroy(it->second.s);
        cudaEventDestroy(it->second.fork);
        cudaEventDestroy(it->second.join);
        g_aux.erase(it);
    }
    return B200PIC_OK;
}

int b200pic_clear_error(b200pic_state *st, void *stream) {
    if (!st || !st->err) return B200PIC_ERR_ARG;
    k_clear_err<<<1, 32, 0, (cudaStream_t)stream>>>(st->err);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

int b200pic_check_error(b200pic_state *st, void *stream, int64_t *bad_id) {
    if (!st || !st->err) return B200PIC_ERR_ARG;
    int64_t h[8];
    CUDA_TRY(cudaMemcpyAsync(h, st->err, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    for (int code = 1; code < 8; ++code) {
        if (h[0] & (1ll << code)) {
            if (bad_id) *bad_id = h[code];
            return code;
        }
    }
    if (bad_id) *bad_id = -1;
    return B200PIC_OK;
}

int b200pic_initial_sort(b200pic_state *st, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    Workspace w = carve(*st);
    if (w.bytes > st->work_bytes) return B200PIC_ERR_CAPACITY;
    int rc;
    if ((rc = initial_keys(*st, w, s))) return rc;
    if ((rc = sort_by_keys(*st, w, s))) return rc;
    return build_items(*st, w, s);
}

static int step_particles(b200pic_state *st, unsigned long long *trace, int64_t trace_rows, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const b200pic_config &c = st->cfg;
    Workspace w = carve(*st);
    if (w.bytes > st->work_bytes) return B200PIC_ERR_CAPACITY;
    K1Params P;
    memset(&P, 0, sizeof(P));
    P.cfg = c;
    for (int i = 0; i < c.n_species; ++i) {
        const b200pic_species &a = st->sp[i], &b = st->alt[i];
        K1Species &k = P.sp[i];
        k.x = a.x; k.y = a.y; k.z = a.z; k.px = a.px; k.py = a.py; k.pz = a.pz; k.w = a.w;
        k.id = a.id;
        k.dx = b.x; k.dy = b.y; k.dz = b.z; k.dpx = b.px; k.dpy = b.py; k.dpz = b.pz; k.dw = b.w;
        k.did = b.id;
        k.perm = w.perm[i];
        k.off = a.offsets;
        k.key = w.key[i];
        k.charge = c.charge[i];
        k.mass = c.mass[i];
        k.qd2 = c.charge[i] * c.dt * 0.5;               // kernels.py:131
        k.inv_m2 = 1.0 / (c.mass[i] * c.mass[i]);       // kernels.py:132
    }
    for (int k = 0; k < 6; ++k) P.e[k] = st->f.e[k];
    for (int k = 0; k < 3; ++k) P.jacc[k] = st->f.jacc[k];
    P.items = w.items;
    P.ilp = w.ilp;
    P.n_items = w.n_items;
    P.queue = w.queue;
    P.err = st->err;
    for (int a = 0; a < 3; ++a) {
        bool on = a < c.dim;
        P.inv[a] = on ? 1.0 / c.d[a] : 1.0;              // scheduler.py:99-100
        P.d_over_dt[a] = on ? c.d[a] / c.dt : 0.0;       // scheduler.py:101-102
        P.Lw[a] = on ? (a == 0 ? global_L0(c) : c.L[a]) * c.d[a] : 0.0;  // config.py:180-186 (global extent)
        P.inv_pn[a] = 1.0 / (on ? c.pn[a] : 1);
    }
    P.fbits_dev = w.fbits;
    P.fscale_dev = w.fscale;
    P.fbits_host = c.j_fine_bits < 0 ? 0 : (c.j_fine_bits > 16 ? 16 : c.j_fine_bits);
    P.fscale_host = ldexp(1.0, 44 + P.fbits_host);
    P.jsafe_dev = w.jsafe;
    P.anchors = anchors_per_bin(c);
    {
        const char *ab = getenv("B200PIC_ABLATE");
        P.ablate = ab ? atoi(ab) : 0;
    }
    P.n_keys = n_keys(c);
    P.trace = trace;
    P.trace_rows = trace_rows;
    CUDA_TRY(cudaMemsetAsync(w.queue, 0, sizeof(int32_t), s));
    int rc = launch_k1(P, k1_grid_cached(c), s);
    if (rc) return rc;
    swap_buffers(*st);  // K1 wrote the updated particles, in sorted order, into alt
    return B200PIC_OK;
}

int b200pic_step_particles(b200pic_state *st, void *stream) { return step_particles(st, nullptr, 0, stream); }

int b200pic_step_particles_traced(b200pic_state *st, unsigned long long *trace, int64_t trace_rows,
                                  int32_t *n_items_out, void *stream) {
    if (!valid(st) || !trace || trace_rows < 0 || !n_items_out) return B200PIC_ERR_ARG;
    Workspace w = carve(*st);
    if (w.bytes > st->work_bytes) return B200PIC_ERR_CAPACITY;
    // the item count of this launch (items are rebuilt by the sort that precedes K1)
    CUDA_TRY(cudaMemcpyAsync(n_items_out, w.n_items, sizeof(int32_t), cudaMemcpyDeviceToDevice,
                             (cudaStream_t)stream));
    return step_particles(st, trace, trace_rows, stream);
}

int b200pic_sort_particles(b200pic_state *st, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    Workspace w = carve(*st);
    if (w.bytes > st->work_bytes) return B200PIC_ERR_CAPACITY;
    int rc;
    if ((rc = sort_by_keys(*st, w, s))) return rc;
    return build_items(*st, w, s);
}

int b200pic_n_items(b200pic_state *st, int32_t *out_dev, void *stream) {
    if (!valid(st) || !out_dev) return B200PIC_ERR_ARG;
    Workspace w = carve(*st);
    if (w.bytes > st->work_bytes) return B200PIC_ERR_CAPACITY;
    CUDA_TRY(cudaMemcpyAsync(out_dev, w.n_items, sizeof(int32_t), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return B200PIC_OK;
}

int b200pic_j_units(b200pic_state *st, double *out_dev, void *stream) {
    if (!valid(st) || !out_dev) return B200PIC_ERR_ARG;
    Workspace w = carve(*st);
    if (w.bytes > st->work_bytes) return B200PIC_ERR_CAPACITY;
    k_j_units<<<1, 1, 0, (cudaStream_t)stream>>>(w.fbits, w.fscale, out_dev);
    LAUNCH_CHECK();
    return B200PIC_OK;
}

int b200pic_compact(b200pic_state *st, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    Workspace w = carve(*st);
    if (w.bytes > st->work_bytes) return B200PIC_ERR_CAPACITY;
    return compact(*st, w, (cudaStream_t)stream);
}

static bool species_ok(const b200pic_state *st, int s) { return s >= 0 && s < st->cfg.n_species; }

int b200pic_host_map_reset(b200pic_state *st, int species, int32_t *hmap, void *stream) {
    if (!valid(st) || !species_ok(st, species) || !hmap) return B200PIC_ERR_ARG;
    return host_map_reset(*st, species, hmap, (cudaStream_t)stream);
}

int b200pic_host_map_advance(b200pic_state *st, int species, const int32_t *hmap, int32_t *next, void *stream) {
    if (!valid(st) || !species_ok(st, species) || !hmap || !next) return B200PIC_ERR_ARG;
    Workspace w = carve(*st);
    if (w.bytes > st->work_bytes) return B200PIC_ERR_CAPACITY;
    return host_map_advance(*st, w, species, hmap, next, (cudaStream_t)stream);
}

int b200pic_host_exchange(b200pic_state *st, int species, const int32_t *hmap, int to_host, void *stream) {
    if (!valid(st) || !species_ok(st, species) || !hmap) return B200PIC_ERR_ARG;
    Workspace w = carve(*st);
    if (w.bytes > st->work_bytes) return B200PIC_ERR_CAPACITY;
    return host_exchange(*st, w, species, hmap, to_host != 0, (cudaStream_t)stream);
}

int b200pic_build_items(b200pic_state *st, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    Workspace w = carve(*st);
    if (w.bytes > st->work_bytes) return B200PIC_ERR_CAPACITY;
    return build_items(*st, w, (cudaStream_t)stream);
}

int b200pic_fold_currents(b200pic_state *st, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    return fold_currents(*st, (cudaStream_t)stream);
}

int b200pic_maxwell(b200pic_state *st, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    for (int k = 0; k < 3; ++k)
        if (!st->f.j[k] || !st->f.jacc[k]) return B200PIC_ERR_ARG;
    return maxwell(*st, (cudaStream_t)stream);
}

int b200pic_maxwell_lagged(b200pic_state *st, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    for (int k = 0; k < 3; ++k)
        if (!st->f.j[k] || !st->f.jacc[k]) return B200PIC_ERR_ARG;
    return maxwell_lagged(*st, (cudaStream_t)stream);
}

int b200pic_sync_fields(b200pic_state *st, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    return sync_fields(*st, C_EX, 6, (cudaStream_t)stream);
}

int b200pic_step_rest(b200pic_state *st, void *stream) {
    int rc;
    if (!valid(st) || st->cfg.slab) return B200PIC_ERR_ARG;  // slabs exchange through the host driver
    AuxStream *aux = getenv("B200PIC_NO_AUX") ? nullptr : aux_stream(st);
    if (aux) {
        // K3 + K2 (fields only) on the auxiliary stream beside K5 (particles only); joined before the
        // next K1, which reads both
        CUDA_TRY(cudaEventRecord(aux->fork, (cudaStream_t)stream));
        CUDA_TRY(cudaStreamWaitEvent(aux->s, aux->fork, 0));
        if ((rc = b200pic_fold_currents(st, aux->s))) return rc;
        if ((rc = b200pic_maxwell(st, aux->s))) return rc;
        CUDA_TRY(cudaEventRecord(aux->join, aux->s));
        if ((rc = b200pic_sort_particles(st, stream))) return rc;
        CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, aux->join, 0));
        return B200PIC_OK;
    }
    if ((rc = b200pic_sort_particles(st, stream))) return rc;
    if ((rc = b200pic_fold_currents(st, stream))) return rc;
    return b200pic_maxwell(st, stream);
}

int b200pic_step(b200pic_state *st, int n_steps, void *stream) {
    int rc;
    if (st && st->cfg.slab) return B200PIC_ERR_ARG;  // slabs step through the host driver (x exchange)
    for (int i = 0; i < n_steps; ++i) {
        if ((rc = b200pic_step_particles(st, stream))) return rc;
        if ((rc = b200pic_step_rest(st, stream))) return rc;
    }
    return B200PIC_OK;
}

int b200pic_yee_half_b(b200pic_state *st, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    return yee_half_b(*st, (cudaStream_t)stream);
}

int b200pic_yee_full_e(b200pic_state *st, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    for (int k = 0; k < 3; ++k)
        if (!st->f.j[k] || !st->f.jacc[k]) return B200PIC_ERR_ARG;
    return yee_full_e(*st, (cudaStream_t)stream);
}

int b200pic_yee_pin_walls(b200pic_state *st, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    return yee_pin_walls(*st, (cudaStream_t)stream);
}

int b200pic_sync_axes(b200pic_state *st, int comp0, int ncomp, int axis_mask, void *stream) {
    if (!valid(st) || comp0 < 0 || ncomp < 0 || comp0 + ncomp > 6) return B200PIC_ERR_ARG;
    return sync_axes(*st, comp0, ncomp, axis_mask, (cudaStream_t)stream);
}

int b200pic_fold_axes(b200pic_state *st, int axis_mask, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    return fold_axes(*st, axis_mask, (cudaStream_t)stream);
}

int b200pic_pack_outgoing(b200pic_state *st, int species, double *send_left, double *send_right, int64_t cap,
                          int64_t *counts_dev, void *stream) {
    if (!valid(st) || species < 0 || species >= st->cfg.n_species || !send_left || !send_right || !counts_dev)
        return B200PIC_ERR_ARG;
    Workspace w = carve(*st);
    return pack_outgoing(*st, w, species, send_left, send_right, cap, counts_dev, (cudaStream_t)stream);
}

size_t b200pic_migrants_bytes(const b200pic_config *cfg, int64_t cap) { return cfg ? migrants_bytes(*cfg, cap) : 0; }

int b200pic_pack_migrants(b200pic_state *st, void *to_left, void *to_right, int64_t cap, void *stream) {
    if (!valid(st) || !st->cfg.slab || !to_left || !to_right || cap <= 0) return B200PIC_ERR_ARG;
    Workspace w = carve(*st);
    return pack_migrants(*st, w, to_left, to_right, cap, (cudaStream_t)stream);
}

int b200pic_unpack_migrants(b200pic_state *st, const void *from_left, const void *from_right, int64_t cap,
                            void *stream) {
    if (!valid(st) || !st->cfg.slab || !from_left || !from_right || cap <= 0) return B200PIC_ERR_ARG;
    Workspace w = carve(*st);
    return unpack_migrants(*st, w, from_left, from_right, cap, (cudaStream_t)stream);
}

size_t b200pic_xplanes_bytes(const b200pic_config *cfg, int which) {
    return cfg && which >= 0 && which <= 2 ? xplanes_bytes(*cfg, which) : 0;
}

int b200pic_xplanes_pack(b200pic_state *st, int which, void *to_left, void *to_right, void *stream) {
    if (!valid(st) || which < 0 || which > 2 || !to_left || !to_right) return B200PIC_ERR_ARG;
    return xplanes_pack(*st, which, to_left, to_right, (cudaStream_t)stream);
}

int b200pic_xplanes_unpack(b200pic_state *st, int which, const void *from_left, const void *from_right,
                           void *stream) {
    if (!valid(st) || which < 0 || which > 2 || !from_left || !from_right) return B200PIC_ERR_ARG;
    return xplanes_unpack(*st, which, from_left, from_right, (cudaStream_t)stream);
}

int b200pic_maxwell_slab(b200pic_state *st, void *stream) {
    if (!valid(st)) return B200PIC_ERR_ARG;
    for (int k = 0; k < 3; ++k)
        if (!st->f.j[k] || !st->f.jacc[k]) return B200PIC_ERR_ARG;
    return maxwell_slab(*st, (cudaStream_t)stream);
}

int b200pic_append_particles(b200pic_state *st, int species, const double *recv, int64_t count, int64_t cap,
                             void *stream) {
    if (!valid(st) || species < 0 || species >= st->cfg.n_species || count < 0 || (count > 0 && !recv))
        return B200PIC_ERR_ARG;
    Workspace w = carve(*st);
    return append_particles(*st, w, species, recv, count, cap, (cudaStream_t)stream);
}

}  // extern "C"
