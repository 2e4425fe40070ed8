// Microbenchmark (dev tool): cost of cooperative grid.sync, a custom barrier, and a
// flag-chain hop between CTAs on B200.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_gridsync(int iters, double *out) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
}
__device__ unsigned ld_acq(const unsigned *p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ void st_rel(unsigned *p, unsigned v) { asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ void red_rel(unsigned *p, unsigned v) { asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
// barrier: counter of arrivals (monotonic); wait until counter >= G*(i+1)
__global__ void k_mybar(int iters, unsigned *ctr) {
    const unsigned G = gridDim.x;
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            red_rel(ctr, 1u);
            const unsigned target = G * (unsigned)(i + 1);
            while (ld_acq(ctr) < target) {}
        }
        __syncthreads();
    }
}
// chain: CTA b waits for flag[b+1] (round r), then sets flag[b]
__global__ void k_chain(int rounds, unsigned *flags) {
    const int b = blockIdx.x, G = gridDim.x;
    for (int r = 1; r <= rounds; ++r) {
        if (threadIdx.x == 0) {
            if (b + 1 < G) while (ld_acq(&flags[b + 1]) != (unsigned)r) {}
            else if (r > 1) while (ld_acq(&flags[0]) != (unsigned)(r - 1)) {}
        }
        __syncthreads();
        if (threadIdx.x == 0) st_rel(&flags[b], (unsigned)r);
        __syncthreads();
    }
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
    int iters = 20000; double *dout; cudaMalloc(&dout, 8);
    for (int G : {8, 64, 148}) {
        void *args[] = {&iters, &dout};
        cudaLaunchCooperativeKernel((void*)k_gridsync, G, 512, args, 0, 0); cudaDeviceSynchronize();
        cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_gridsync, G, 512, args, 0, 0); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("cg grid.sync  G=%3d: %.3f us/sync\n", G, ms * 1e3 / iters);
        unsigned *ctr; cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4);
        void *a2[] = {&iters, &ctr};
        cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_mybar, G, 512, a2, 0, 0); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("custom barrier G=%3d: %.3f us/sync (%s)\n", G, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
        unsigned *fl; cudaMalloc(&fl, 4 * G); cudaMemset(fl, 0, 4 * G);
        int rounds = 200; void *a3[] = {&rounds, &fl};
        cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_chain, G, 512, a3, 0, 0); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("flag chain     G=%3d: %.3f us/hop\n", G, ms * 1e3 / (rounds * G));
    }
    return 0;
}
