// Does a cooperative launch with 2-CTA clusters work on B200 (grid.sync + DSMEM)?
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void __cluster_dims__(2, 1, 1) k(int *out, int iters)
{
    cg::grid_group grid = cg::this_grid();
    cg::cluster_group cl = cg::this_cluster();
    __shared__ int buf[32];
    const int r = cl.block_rank();
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x == 0) {
            int *peer = cl.map_shared_rank(buf, r ^ 1);
            peer[0] = blockIdx.x * 1000 + it;
        }
        cl.sync();
        if (threadIdx.x == 0) out[blockIdx.x] = buf[0];
        grid.sync();
    }
}
int main()
{
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int *d; cudaMalloc(&d, 4 * nsm);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nsm); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 0;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int iters = 1000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, k, d, iters);
    cudaEventRecord(e1);
    cudaError_t e2 = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int h[4]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("launch %s, sync %s, out %d %d %d %d, %.3f us/iter\n", cudaGetErrorString(err), cudaGetErrorString(e2), h[0], h[1], h[2], h[3], ms * 1e3 / iters);
    return 0;
}
