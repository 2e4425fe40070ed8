// Standalone timing of the band apply (ht_band_wy) and Qhat formation (development tool).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1710_08538_b200/csrc band_bench.cu -o band_bench
#include "../../paper_1710_08538_b200/csrc/ht_chain.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
int ht_cuda_fail(cudaError_t e, const char *what, const char *file, int line)
{
    fprintf(stderr, "CUDA error %s at %s:%d (%s)\n", cudaGetErrorString(e), file, line, what);
    return 2;
}
int main(int argc, char **argv)
{
    const int64_t n = 8192;
    const int p = argc > 1 ? atoi(argv[1]) : 256, q = argc > 2 ? atoi(argv[2]) : 128, cnt = argc > 3 ? atoi(argv[3]) : 128;
    const int left = argc > 4 ? atoi(argv[4]) : 0;
    double *X, *V, *T, *Qw;
    cudaMalloc(&X, (size_t)n * n * 8); cudaMemset(X, 0, (size_t)n * n * 8);
    cudaMalloc(&V, (size_t)p * q * 8); cudaMalloc(&T, (size_t)q * q * 8); cudaMalloc(&Qw, (size_t)p * p * 8);
    std::vector<double> h((size_t)p * q);
    for (auto &v : h) v = ((double)rand() / RAND_MAX - 0.5) * 0.1;
    cudaMemcpy(V, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(T, h.data(), (size_t)q * q * 8, cudaMemcpyHostToDevice);
    void *dd; cudaMalloc(&dd, 4096); void *hd; cudaMallocHost(&hd, 4096);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f, bestf = 1e30f;
    for (int it = 0; it < 20; ++it) {
        cudaEventRecord(e0);
        ht_band_wy(0, X, n, left, 4096, cnt, 4000, p, q, V, p, T, q);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (it > 2) best = ms < best ? ms : best;
        double *qp[1] = {Qw}; const double *vp[1] = {V}, *tp[1] = {T}; int pp[1] = {p}, qq[1] = {q};
        cudaEventRecord(e0);
        ht_form_qhat(0, 1, qp, pp, qq, vp, tp, dd, hd);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); if (it > 2) bestf = ms < bestf ? ms : bestf;
    }
    unsigned long long *dp; cudaMalloc(&dp, 64); cudaMemset(dp, 0, 64); cudaMemcpyToSymbol(g_bprof, &dp, sizeof(dp));
    ht_band_wy(0, X, n, left, 4096, cnt, 4000, p, q, V, p, T, q); cudaDeviceSynchronize();
    unsigned long long hp[8]; cudaMemcpy(hp, dp, 64, cudaMemcpyDeviceToHost);
    printf("  cycles: prologue+first wait %llu  later waits %llu  SV %llu  YT %llu  S-=Y2V' %llu\n", hp[4], hp[0], hp[1], hp[2], hp[3]);
    printf("band p=%d q=%d rows=%d left=%d: %.1f us   form Qhat: %.1f us  (%s)\n", p, q, cnt, left, best * 1e3, bestf * 1e3,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
