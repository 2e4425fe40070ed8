// Latency calibration of FP64 / shuffle / shared-memory / barrier operations (development tool).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double *out, long long *cyc, int n)
{
    __shared__ double sm[1024];
    const int tid = threadIdx.x;
    sm[tid] = tid * 1e-3;
    __syncthreads();
    double a = 1.0 + tid * 1e-9, b = 0.999999;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, 1e-12);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) a = __shfl_sync(0xffffffffu, a, (tid + 1) & 31);
    long long t2 = clock64();
    int idx = tid;
    for (int i = 0; i < n; ++i) { a += sm[idx & 1023]; idx = (int)a & 1; }
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) { __syncthreads(); }
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) a = sqrt(a);
    long long t5 = clock64();
    for (int i = 0; i < n; ++i) a = 1.0 / a;
    long long t6 = clock64();
    for (int i = 0; i < n; ++i) a = a + 1e-12;
    long long t7 = clock64();
    if (tid == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6; }
    out[tid] = a;
}
int main()
{
    double *o; long long *c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
    for (int nt : {32, 512}) {
        int n = 4096;
        lat<<<1, nt>>>(o, c, n); lat<<<1, nt>>>(o, c, n);
        long long h[8]; cudaMemcpy(h, c, 56, cudaMemcpyDeviceToHost);
        printf("threads=%d: DFMA %.1f, SHFL %.1f, LDS+DADD %.1f, BAR %.1f, sqrt %.1f, div %.1f, DADD %.1f cycles/op\n", nt,
               h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n, h[6] / (double)n);
    }
    return 0;
}
