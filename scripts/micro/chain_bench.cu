// Standalone throughput of the chained window apply (development tool).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1710_08538_b200/csrc chain_bench.cu -o chain_bench
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
    const int64_t n = argc > 1 ? atoll(argv[1]) : 8192;
    const int p = argc > 2 ? atoi(argv[2]) : 256;
    const int nw = argc > 3 ? atoi(argv[3]) : 32;
    const int left = argc > 4 ? atoi(argv[4]) : 0;
    const int maxgrid = argc > 5 ? atoi(argv[5]) : 0;
    double *X, *Q;
    cudaMalloc(&X, (size_t)n * n * 8);
    cudaMalloc(&Q, (size_t)nw * p * p * 8);
    std::vector<double> h((size_t)p * p);
    srand(1);
    for (auto &v : h) v = ((double)rand() / RAND_MAX - 0.5) * 0.1;
    for (int i = 0; i < nw; ++i) cudaMemcpy(Q + (size_t)i * p * p, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(X, 0, (size_t)n * n * 8);
    const int k = p / 2;
    std::vector<ChainWin> w(nw);
    for (int i = 0; i < nw; ++i) w[i] = ChainWin{Q + (size_t)i * p * p, (int64_t)i * k, p, {0, 0, 0}, {n, n, n}};
    ChainWin *dw;
    cudaMalloc(&dw, nw * sizeof(ChainWin));
    cudaMemcpy(dw, w.data(), nw * sizeof(ChainWin), cudaMemcpyHostToDevice);
    ChainMat m{X, n, left, 0, n};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 6; ++it) {
        cudaEventRecord(e0);
        ht_chain_apply(0, &m, 1, dw, nw, p, maxgrid);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it) best = ms < best ? ms : best;
    }
    const double fl = 2.0 * (double)n * p * p * nw;
    printf("chain n=%lld p=%d nw=%d left=%d grid=%d: %.3f ms, %.2f TFLOP/s  (%s)\n", (long long)n, p, nw, left, maxgrid,
           best, fl / (best * 1e-3) * 1e-12, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
