// Probe: can runtime-API kernels run in a green-context stream (SM partition) on memory from
// cudaMalloc (primary context)?  Prints the SMs used by a kernel in the partition.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o green_probe green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
__global__ void k_big(int *out)
{
    extern __shared__ int sm[];
    sm[threadIdx.x * 100] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = sm[100 * 5] + 1;
}
__global__ void k_smid(int *out, int n)
{
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = (int)s;
}
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *e; cuGetErrorString(r, &e); printf("%s -> %s\n", #x, e); return 1; } } while (0)
int main(int argc, char **argv)
{
    const int want = argc > 1 ? atoi(argv[1]) : 112;
    cudaFree(0);
    CUdevice dev; CK(cuDeviceGet(&dev, 0));
    CUdevResource all, part[2]; unsigned nparts = 1;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs: %u\n", all.sm.smCount);
    CUdevResource rem;
    CK(cuDevSmResourceSplitByCount(part, &nparts, &all, &rem, 0, want));
    printf("partition: %u groups of %u SMs, remaining %u\n", nparts, part[0].sm.smCount, rem.sm.smCount);
    CUdevResourceDesc desc; CK(cuDevResourceGenerateDesc(&desc, &part[0], 1));
    CUgreenCtx g; CK(cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream s; CK(cuGreenCtxStreamCreate(&s, g, CU_STREAM_NON_BLOCKING, 0));
    const int n = 1 << 22;
    int *d; cudaMalloc(&d, n * sizeof(int));
    k_smid<<<1184, 256, 0, (cudaStream_t)s>>>(d, n);
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)s);
    printf("launch in green stream: %s\n", cudaGetErrorString(e));
    int *h = new int[n]; cudaMemcpy(h, d, n * sizeof(int), cudaMemcpyDeviceToHost);
    std::set<int> sms(h, h + n);
    printf("distinct SMs used: %zu (min %d max %d)\n", sms.size(), *sms.begin(), *sms.rbegin());
    k_smid<<<1184, 256>>>(d, n);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, n * sizeof(int), cudaMemcpyDeviceToHost);
    std::set<int> sms2(h, h + n);
    printf("primary context: distinct SMs used: %zu\n", sms2.size());
    // dynamic smem > 48 KB (attribute set through the runtime in the primary context)
    cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    k_big<<<4, 256, 160 * 1024, (cudaStream_t)s>>>(d);
    printf("big-smem launch in green stream: %s / %s\n", cudaGetErrorString(cudaGetLastError()), cudaGetErrorString(cudaStreamSynchronize((cudaStream_t)s)));
    // events: primary event recorded on the green stream, waited on by a primary stream, and back
    cudaEvent_t ev; cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaStream_t ps; cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking);
    k_smid<<<148, 256, 0, (cudaStream_t)s>>>(d, n);
    cudaError_t e1 = cudaEventRecord(ev, (cudaStream_t)s);
    cudaError_t e2 = cudaStreamWaitEvent(ps, ev, 0);
    k_smid<<<148, 256, 0, ps>>>(d, n);
    cudaError_t e3 = cudaEventRecord(ev, ps);
    cudaError_t e4 = cudaStreamWaitEvent((cudaStream_t)s, ev, 0);
    cudaError_t e5 = cudaDeviceSynchronize();
    printf("events: record(green) %s, wait(primary) %s, record(primary) %s, wait(green) %s, sync %s\n",
           cudaGetErrorString(e1), cudaGetErrorString(e2), cudaGetErrorString(e3), cudaGetErrorString(e4), cudaGetErrorString(e5));
    // timing events on a green stream
    cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
    cudaEventRecord(t0, (cudaStream_t)s); k_smid<<<148, 256, 0, (cudaStream_t)s>>>(d, n); cudaEventRecord(t1, (cudaStream_t)s);
    cudaEventSynchronize(t1); float ms = -1; cudaError_t e6 = cudaEventElapsedTime(&ms, t0, t1);
    printf("timing events on green stream: %s %.3f ms\n", cudaGetErrorString(e6), ms);
    int pri_lo, pri_hi; cudaDeviceGetStreamPriorityRange(&pri_lo, &pri_hi);
    CUstream s2; CK(cuGreenCtxStreamCreate(&s2, g, CU_STREAM_NON_BLOCKING, pri_lo));
    printf("low-priority green stream ok\n");
    return 0;
}
