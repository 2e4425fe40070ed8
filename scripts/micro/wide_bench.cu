// Cycle cost of the wide-layout Householder column step (development tool).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 wide_bench.cu -o wide_bench
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void house(double alpha, double ss, double &beta, double &tau, double &scal)
{
    const double N = fma(alpha, alpha, ss);
    const double r = rsqrt(N);
    const double nrm = N * r;
    beta = alpha >= 0.0 ? -nrm : nrm;
    tau = fma(fabs(alpha), r, 1.0);
    double it = (double)(1.0f / (float)tau);
    it = it * fma(-tau, it, 2.0);
    it = it * fma(-tau, it, 2.0);
    const double sc = r * it;
    scal = alpha >= 0.0 ? sc : -sc;
}
// FLAGS: 1 = house scalars, 2 = barrier, 4 = unroll 32, 8 = pivot via smem (else shfl)
template <int RPT, int FLAGS>
__global__ void __launch_bounds__(256, 1) k(double *out, long long *cyc, int iters)
{
    constexpr int NW = 8, PBW = 32;
    __shared__ double part[2][NW][PBW];
    __shared__ double rowc[2][PBW];
    __shared__ __align__(16) double pivs[2][NW * RPT];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, w0 = warp * RPT;
    double val[RPT];
    for (int e = 0; e < RPT; ++e) val[e] = 1.0 + 0.001 * (tid + e) + 0.01 * e * e;
    if (lane == 0) for (int e = 0; e < RPT; ++e) pivs[0][w0 + e] = val[e];
    __syncthreads();
    long long c0 = clock64();
    auto step = [&](int jj) {
        const int buf = jj & 1;
        double xr[RPT], sa[4] = {0, 0, 0, 0};
        if (FLAGS & 8) {
            const double2 *src = reinterpret_cast<const double2 *>(&pivs[buf][w0]);
#pragma unroll
            for (int e = 0; e < RPT; e += 2) { double2 t = src[e / 2]; xr[e] = t.x; xr[e + 1] = t.y; }
        } else {
#pragma unroll
            for (int e = 0; e < RPT; ++e) xr[e] = __shfl_sync(0xffffffffu, val[e], jj);
        }
#pragma unroll
        for (int e = 0; e < RPT; ++e) sa[e & 3] = fma(xr[e], val[e], sa[e & 3]);
        part[buf][warp][lane] = (sa[0] + sa[1]) + (sa[2] + sa[3]);
        if (warp == 0) rowc[buf][lane] = val[0];
        if (FLAGS & 2) __syncthreads();
        double pr[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) pr[w] = part[buf][w][lane];
#pragma unroll
        for (int h = NW / 2; h >= 1; h >>= 1)
#pragma unroll
            for (int w = 0; w < h; ++w) pr[w] += pr[w + h];
        const double S = pr[0];
        const double ss = __shfl_sync(0xffffffffu, S, jj);
        const double alpha = rowc[buf][jj];
        const double myrow = rowc[buf][lane];
        double tau = 0.5, scal = 0.25, beta = alpha;
        if (FLAGS & 1) house(alpha, ss, beta, tau, scal);
        const double wj = tau * (myrow + scal * S);
        const double mx = lane > jj ? -wj * scal * 1e-9 : 0.0;
#pragma unroll
        for (int e = 0; e < RPT; ++e) val[e] = fma(mx, xr[e], val[e]);
        if (FLAGS & 8) {
            if (lane == ((jj + 1) & 31)) {
                double2 *dst = reinterpret_cast<double2 *>(&pivs[buf ^ 1][w0]);
#pragma unroll
                for (int e = 0; e < RPT; e += 2) dst[e / 2] = make_double2(val[e], val[e + 1]);
            }
            __syncwarp();
        }
    };
    for (int it = 0; it < iters; ++it) {
        if (FLAGS & 4) {
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) step(jj);
        } else {
#pragma unroll 1
            for (int jj = 0; jj < 32; ++jj) step(jj);
        }
    }
    long long c1 = clock64();
    if (tid == 0) cyc[0] = c1 - c0;
    double t = 0;
    for (int e = 0; e < RPT; ++e) t += val[e];
    out[tid] = t;
}
template <int RPT, int FLAGS> void run()
{
    double *o; long long *c; cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 16);
    int iters = 200;
    k<RPT, FLAGS><<<1, 256>>>(o, c, iters);
    k<RPT, FLAGS><<<1, 256>>>(o, c, iters);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("RPT=%2d house=%d bar=%d unroll32=%d smem_pivot=%d: %.1f cycles/step\n", RPT, FLAGS & 1, (FLAGS >> 1) & 1,
           (FLAGS >> 2) & 1, (FLAGS >> 3) & 1, (double)h / (iters * 32));
}
int main()
{
    run<32, 0>(); run<32, 2>(); run<32, 3>(); run<32, 11>(); run<32, 15>(); run<32, 7>();
    run<16, 0>(); run<16, 2>(); run<16, 3>(); run<16, 11>(); run<16, 15>();
    run<8, 3>(); run<8, 11>();
    return 0;
}
