// Shared-memory wavefronts per warp-wide load for the address patterns of K1 (ncu
// l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum / 32 warps / ITER loads):
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/ldsw scripts/diag/lds_wavefronts.cu
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum /tmp/ldsw
#include <cstdio>
constexpr int ITER = 256;
// pattern: address (in doubles) of lane l
__device__ __forceinline__ int addr(int pat, int l) {
    switch (pat) {
        case 0: return 0;                   // broadcast
        case 1: return (l / 11) * 40;       // 3 distinct (runs of ~11 lanes: three anchors in a warp)
        case 2: return (l / 5) * 2;         // la-indexed (5 lanes per value)
        case 3: return (l % 5) * 2;         // lb-indexed
        case 4: return l * 2;               // all distinct, contiguous (16 B apart)
        case 5: return (l / 8) * 40 + (l & 1) * 2;  // 4 anchors x parity
        // K1 gather-like: particles sorted by anchor (runs of R lanes), a dual stencil index that differs by
        // one node between particles of a run (hash of the lane), 16-byte pairs (x2 doubles)
        case 6: return (l / 16) * 40 + ((l * 7 + 3) % 5 < 2 ? 2 : 0);
        case 7: return (l / 11) * 40 + ((l * 7 + 3) % 5 < 2 ? 2 : 0);
        case 8: return ((l * 7 + 3) % 5 < 2 ? 2 : 0);
        case 9: return (l / 16) * 40 + ((l * 7 + 3) % 5 < 2 ? 1 : 0);  // 8-byte offsets (LDS.64 gather today)
        default: return 0;
    }
}
template <int PAT, int W>
__global__ void k(double *out) {
    __shared__ __align__(16) double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
    __syncthreads();
    const int a = addr(PAT, threadIdx.x & 31);
    double acc = 0;
#pragma unroll 8
    for (int i = 0; i < ITER; ++i) {
        const int o = a + ((i * 2) & 1023);
        if (W == 16) {
            const double2 v = *reinterpret_cast<const double2 *>(s + o);
            acc += v.x + v.y;
        } else {
            acc += s[o];
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    double *o;
    cudaMalloc(&o, 1 << 20);
#define RUN(P, W) k<P, W><<<1, 1024>>>(o); cudaDeviceSynchronize();
    RUN(0, 8) RUN(0, 16) RUN(1, 8) RUN(1, 16) RUN(2, 8) RUN(2, 16) RUN(3, 8) RUN(3, 16) RUN(4, 8) RUN(4, 16) RUN(5, 8) RUN(5, 16)
    RUN(6, 16) RUN(7, 16) RUN(8, 16) RUN(9, 8) RUN(7, 8)
    printf("done\n");
    return 0;
}
