// Peak rate of warp-level FP64 MMA (mma.sync m8n8k4 / m16n8k4 / m16n8k8 f64) on this GPU: independent
// accumulator chains, no memory traffic.  Development tool (no tcgen05 kind::f64).
#include <cstdio>
__global__ void k884(double *out, int iters)
{
    double c[8][2];
    double a = threadIdx.x * 1e-3, b = 1.0 - a;
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}
__global__ void k1688(double *out, int iters)
{
    double c[8][4];
    double a0 = threadIdx.x * 1e-3, a1 = 0.5, a2 = 0.25, a3 = 0.125, b0 = 1.0 - a0, b1 = 0.3;
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                         : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.0) out[0] = s;
}
int main()
{
    double *o;
    cudaMalloc(&o, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 20000;
    for (int warps : {4, 8, 16, 32}) {
        for (int v = 0; v < 2; ++v) {
            const int grid = nsm, block = 32 * warps;
            if (v == 0) k884<<<grid, block>>>(o, 10); else k1688<<<grid, block>>>(o, 10);
            cudaEventRecord(e0);
            if (v == 0) k884<<<grid, block>>>(o, iters); else k1688<<<grid, block>>>(o, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flop = (double)grid * warps * iters * 8 * (v == 0 ? 2.0 * 8 * 8 * 4 : 2.0 * 16 * 8 * 8);
            printf("%s warps/SM=%2d: %.2f TFLOP/s\n", v == 0 ? "m8n8k4 " : "m16n8k8", warps, flop / ms * 1e-9);
        }
    }
    return 0;
}
