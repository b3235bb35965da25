// loader.cu -- on-device particle loader for perf-size runs (BASELINE configs
// 2-4 hold 0.27-1.2 billion particles; generating them on the host and
// copying 17-74 GB over PCIe would dominate setup).  Counter-based RNG
// (splitmix64 of (seed, species, particle, draw)), so any slab of the domain
// can be generated independently and reproducibly.  Layout follows the
// harness loader (loaders.uniform_random_species): ppc particles per cell,
// cells in C order (x slowest), uniform in-cell positions, Gaussian momenta
// (Box-Muller), equal weights, id = creation index.
#include "common.cuh"

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double u01(uint64_t seed, uint64_t sp, uint64_t i, uint64_t k) {
    uint64_t h = mix64(seed ^ mix64(sp * 0x100000001B3ull ^ mix64(i * 8 + k)));
    return ((h >> 11) + 0.5) * (1.0 / 9007199254740992.0);  // (0, 1)
}

__global__ void k_load_uniform(b200pic_config c, b200pic_species sp, int species, int64_t ppc, double sigma,
                               double weight, uint64_t seed, int64_t x0, int64_t nxc, int64_t id0) {
    const int64_t ny = c.L[1], nz = c.dim == 3 ? c.L[2] : 1;
    const int64_t n = nxc * ny * nz * ppc;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t cell = i / ppc;
        int64_t cz = cell % nz, r = cell / nz, cy = r % ny, cx = r / ny + x0;
        int64_t gid = id0 + i;
        sp.x[i] = (cx + u01(seed, species, gid, 0)) * c.d[0];
        sp.y[i] = (cy + u01(seed, species, gid, 1)) * c.d[1];
        if (c.dim == 3) sp.z[i] = (cz + u01(seed, species, gid, 2)) * c.d[2];
        double u1 = u01(seed, species, gid, 3), u2 = u01(seed, species, gid, 4);
        double u3 = u01(seed, species, gid, 5), u4 = u01(seed, species, gid, 6);
        double r1 = sqrt(-2.0 * log(u1)), r2 = sqrt(-2.0 * log(u3));
        double s1, c1, s2, c2;
        sincospi(2.0 * u2, &s1, &c1);
        sincospi(2.0 * u4, &s2, &c2);
        sp.px[i] = sigma * r1 * c1;
        sp.py[i] = sigma * r1 * s1;
        sp.pz[i] = sigma * r2 * c2;
        sp.w[i] = weight;
        sp.id[i] = gid;
    }
}

__global__ void k_set_count(int64_t *n_dev, int64_t n) { *n_dev = n; }

}  // namespace

extern "C" int b200pic_load_uniform(b200pic_state *st, int species, int64_t ppc, double sigma, double weight,
                                    uint64_t seed, int64_t x_cell0, int64_t x_cells, int64_t id0, void *stream) {
    if (!st || species < 0 || species >= st->cfg.n_species || ppc < 0) return B200PIC_ERR_ARG;
    const b200pic_config &c = st->cfg;
    const b200pic_species &sp = st->sp[species];
    int64_t n = x_cells * (int64_t)c.L[1] * (c.dim == 3 ? c.L[2] : 1) * ppc;
    if (n > sp.capacity) return B200PIC_ERR_CAPACITY;
    cudaStream_t s = (cudaStream_t)stream;
    if (n > 0) {
        int64_t blocks = (n + 255) / 256;
        if (blocks > 148 * 32) blocks = 148 * 32;
        k_load_uniform<<<(unsigned)blocks, 256, 0, s>>>(c, sp, species, ppc, sigma, weight, seed, x_cell0, x_cells,
                                                       id0);
        LAUNCH_CHECK();
    }
    k_set_count<<<1, 1, 0, s>>>(sp.n_dev, n);
    LAUNCH_CHECK();
    return B200PIC_OK;
}
