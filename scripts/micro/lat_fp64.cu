// Dependent-chain latencies on this GPU (development probe): DFMA, DADD, double rsqrt/sqrt/div,
// float rcp, LDS round trip, 64-bit SHFL, __syncthreads with 256 threads.
#include <cstdio>
__global__ void k(double *out, long long *cyc, double x0, int n)
{
    __shared__ double sm[256];
    double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
    sm[threadIdx.x] = x;
    __syncthreads();
    long long t0, t1;
#define LAT(slot, body)                                            \
    t0 = clock64();                                                \
    for (int i = 0; i < n; ++i) { body; }                          \
    t1 = clock64();                                                \
    if (threadIdx.x == 0) cyc[slot] = (t1 - t0) / n;
    LAT(0, x = fma(x, y, 1e-30))
    LAT(1, x = x + 1e-30)
    LAT(2, x = rsqrt(x) + 0.5)
    LAT(3, x = sqrt(x) + 0.5)
    LAT(4, x = 1.0 / x + 0.5)
    LAT(5, x = (double)(1.0f / (float)x) + 0.5)
    LAT(6, x = sm[((int)x) & 1] + 0.5)
    LAT(7, x = __shfl_sync(0xffffffffu, x, 1) + 1e-30)
    LAT(8, __syncthreads(); x = x + 1e-30)
    LAT(9, x = x * 1.0000001)
    out[threadIdx.x] = x;
}
int main()
{
    double *o; long long *c, h[16];
    cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 16 * 8);
    k<<<1, 256>>>(o, c, 1.5, 1000);
    k<<<1, 256>>>(o, c, 1.5, 10000);
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    const char *nm[] = {"DFMA", "DADD", "rsqrt(d)+add", "sqrt(d)+add", "1/d+add", "f32 rcp cvt+add", "LDS.64+add", "SHFL64+add", "bar.sync+add (256 thr)", "DMUL"};
    for (int i = 0; i < 10; ++i) printf("%-24s %lld cycles\n", nm[i], h[i]);
    return 0;
}
