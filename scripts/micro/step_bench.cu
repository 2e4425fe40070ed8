// Cycle cost of one Householder column step pattern (development tool).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
template <int RPT, int MODE>
__global__ void __launch_bounds__(512, 1) step_kernel(double *out, long long *cyc, int iters)
{
    __shared__ double part[2][16][8];
    __shared__ double rowc[2][8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, c8 = lane & 7, rq = lane >> 3;
    double val[RPT];
    for (int e = 0; e < RPT; ++e) val[e] = 1.0 + 0.001 * (tid + e);
    int buf = 0;
    long long c0 = clock64();
    unsigned long long g0 = gt();
    for (int it = 0; it < iters; ++it) {
        const int jc = it & 7;
        const int src = (rq << 3) | jc;
        double xr[RPT], sa0 = 0, sa1 = 0;
#pragma unroll
        for (int e = 0; e < RPT; ++e) {
            xr[e] = __shfl_sync(0xffffffffu, val[e], src);
            if (e & 1) sa1 = fma(val[e], xr[e], sa1); else sa0 = fma(val[e], xr[e], sa0);
        }
        double s = sa0 + sa1;
        s += __shfl_xor_sync(0xffffffffu, s, 8);
        s += __shfl_xor_sync(0xffffffffu, s, 16);
        if (rq == 0) part[buf][warp][c8] = s;
        if (warp == (it & 15) && rq == 0) rowc[buf][c8] = val[0];
        if (MODE >= 1) __syncthreads();
        double pr[16];
#pragma unroll
        for (int w = 0; w < 16; ++w) pr[w] = part[buf][w][c8];
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
            for (int w = 0; w < h; ++w) pr[w] += pr[w + h];
        const double S = pr[0];
        const double ss = __shfl_sync(0xffffffffu, S, jc);
        const double alpha = rowc[buf][jc];
        double tau = 0, scal = 0;
        if (MODE >= 2) {
            const double nrm = sqrt(alpha * alpha + ss * 1e-6);
            const double beta = alpha >= 0 ? -nrm : nrm;
            tau = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        } else { tau = 0.5; scal = 0.25; }
        const double wj = tau * (rowc[buf][c8] + scal * S);
        const double mx = (c8 > jc) ? -wj * scal * 1e-9 : 0.0;
#pragma unroll
        for (int e = 0; e < RPT; ++e) val[e] = fma(mx, xr[e], val[e]);
        buf ^= 1;
    }
    long long c1 = clock64();
    unsigned long long g1 = gt();
    if (tid == 0) { cyc[0] = c1 - c0; cyc[1] = (long long)(g1 - g0); }
    double t = 0; for (int e = 0; e < RPT; ++e) t += val[e];
    out[tid] = t;
}
template <int RPT, int MODE> void run(const char *name)
{
    double *o; long long *c; cudaMalloc(&o, 512 * 8); cudaMalloc(&c, 16);
    int iters = 10000;
    step_kernel<RPT, MODE><<<1, 512>>>(o, c, iters);
    step_kernel<RPT, MODE><<<1, 512>>>(o, c, iters);
    long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("%s RPT=%d: %.1f cycles/step, %.3f us/step, clock %.0f MHz\n", name, RPT, (double)h[0] / iters, h[1] * 1e-3 / iters, (double)h[0] / h[1] * 1e3);
}
int main()
{
    run<4, 0>("no-sync ");
    run<4, 1>("sync    ");
    run<4, 2>("sync+sqrt/div");
    run<8, 2>("sync+sqrt/div");
    run<2, 2>("sync+sqrt/div");
    return 0;
}
