// Cycle cost of the solve chain's critical section (128x128 shared-memory mat-vec + publish).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int TB = 128, PNT = 512;
__device__ __forceinline__ void st_volatile64(unsigned long long *p, unsigned long long v)
{ asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__global__ void __launch_bounds__(PNT, 1) crit(double *vy, unsigned long long *yll, long long *cyc, int iters, int mode)
{
    extern __shared__ double dyn[];
    __shared__ double rhs[TB], cbv[TB], red[32];
    double *Dsm = dyn, *accg = dyn + TB * TB;
    const int tid = threadIdx.x, ri = tid & (TB - 1), grp = tid >> 7, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < TB * TB; i += PNT) Dsm[i] = 1e-3 * (i % 97);
    if (tid < TB) { rhs[tid] = 1.0; cbv[tid] = 2.0; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        double sa[4] = {0, 0, 0, 0};
#pragma unroll
        for (int m = 0; m < TB / 16; ++m)
#pragma unroll
            for (int u = 0; u < 4; ++u) { const int l = grp + 16 * m + 4 * u; sa[u] = fma(Dsm[l * TB + ri], rhs[l], sa[u]); }
        accg[grp * TB + ri] = (sa[0] + sa[1]) + (sa[2] + sa[3]);
        __syncthreads();
        double xv = 0;
        if (tid < TB) xv = cbv[tid] * 0.5 - ((accg[tid] + accg[TB + tid]) + (accg[2 * TB + tid] + accg[3 * TB + tid])) * 1e-9;
        if (mode >= 1) {
            const bool big = (tid < TB) && !(fabs(xv) <= 1e300);
            if (__syncthreads_or(big)) { red[0] = 1; }
            if (tid < TB) {
                vy[tid] = xv;
                if (mode >= 2) {
                    const unsigned long long b = (unsigned long long)__double_as_longlong(xv);
                    const unsigned long long e = (unsigned long long)(it + 1) << 32;
                    st_volatile64(yll + 2 * tid, e | (b & 0xffffffffull));
                    st_volatile64(yll + 2 * tid + 1, e | (b >> 32));
                }
            }
            __syncthreads();
            if (tid == 0) st_volatile64(yll + 1000, (unsigned long long)it);
        }
        if (tid < TB) rhs[tid] = xv * 1e-3 + 1.0;
        __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) cyc[0] = t1 - t0;
}
int main()
{
    double *vy; unsigned long long *yll; long long *c;
    cudaMalloc(&vy, 1024 * 8); cudaMalloc(&yll, 4096 * 8); cudaMalloc(&c, 8);
    const int smem = (TB * TB + 8 * TB) * 8;
    cudaFuncSetAttribute(crit, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 3; ++mode) {
        int iters = 2000;
        crit<<<1, PNT, smem>>>(vy, yll, c, iters, mode);
        crit<<<1, PNT, smem>>>(vy, yll, c, iters, mode);
        long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("mode %d: %.0f cycles per critical step (%.2f us at 1.965 GHz)\n", mode, (double)h / iters, h / iters / 1965.0);
    }
    return 0;
}
