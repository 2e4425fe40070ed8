// Micro-benchmark + self-check of the window factorization kernel (development tool).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1710_08538_b200/csrc
//        factor_bench.cu -o factor_bench
// Usage: ./factor_bench p q [reps] [rev] [transposed]
#ifndef HT_NO_STEP_PROF
#define HT_FACTOR_STEP_PROF 1
#endif
#include "../../paper_1710_08538_b200/csrc/ht_factor.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <algorithm>
int ht_cuda_fail(cudaError_t e, const char *what, const char *file, int line)
{
    fprintf(stderr, "CUDA error %s at %s:%d (%s)\n", cudaGetErrorString(e), file, line, what);
    return 2;
}
int main(int argc, char **argv)
{
    const int p = argc > 1 ? atoi(argv[1]) : 256, q = argc > 2 ? atoi(argv[2]) : 128;
    const int reps = argc > 3 ? atoi(argv[3]) : 10;
    const int rev = argc > 4 ? atoi(argv[4]) : 0;
    const int dense = argc > 5 ? atoi(argv[5]) : 0;  // staircase structure: view rows > dense + c of column c are 0
    std::vector<double> W0((size_t)p * q);
    srand(1);
    for (auto &x : W0) x = (double)rand() / RAND_MAX - 0.5;
    double *dW, *dV, *dtau, *dT, *dg;
    cudaMalloc(&dW, W0.size() * 8); cudaMalloc(&dV, (size_t)p * q * 8); cudaMalloc(&dtau, q * 8);
    cudaMalloc(&dT, (size_t)q * q * 8); cudaMalloc(&dg, 64 * 1024 * 8);
    FactorDesc hd;
    // view: rev -> reversed rows and columns (QL-type); W(i, j) = base[i*rs + j*cs]
    if (rev) hd = FactorDesc{dW + (p - 1) + (size_t)(q - 1) * p, -1, -(int64_t)p, p, q, 1, dV, p, dtau, dT, q};
    else hd = FactorDesc{dW, 1, p, p, q, 0, dV, p, dtau, dT, q};
    hd.dense = dense;
    if (dense > 0)
        for (int i = 0; i < p; ++i)
            for (int j = 0; j < q; ++j)
                if (i > dense + j) W0[rev ? (size_t)(p - 1 - i) + (size_t)(q - 1 - j) * p : (size_t)i + (size_t)j * p] = 0.0;
    FactorDesc *dd; cudaMalloc(&dd, sizeof(FactorDesc));
    cudaMemcpy(dd, &hd, sizeof(hd), cudaMemcpyHostToDevice);
    unsigned long long *dprof; cudaMalloc(&dprof, 32 * 8); cudaMemset(dprof, 0, 32 * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < reps + 1; ++it) {
        cudaMemcpy(dW, W0.data(), W0.size() * 8, cudaMemcpyHostToDevice);
        if (it == reps) cudaMemcpyToSymbol(g_fprof, &dprof, sizeof(dprof));
        cudaEventRecord(e0);
        int rc = ht_factor_run(0, dd, 1, dg, p);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        if (rc || cudaGetLastError() != cudaSuccess) { printf("launch failed\n"); return 1; }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (it < reps) best = ms < best ? ms : best;
    }
    unsigned long long hp[32]; cudaMemcpy(hp, dprof, sizeof(hp), cudaMemcpyDeviceToHost);
    printf("wide column step cycles/col (last warp): loads+dots %.0f bar %.0f partials+sum %.0f house %.0f update %.0f\n",
           hp[12] / (double)q, hp[13] / (double)q, hp[14] / (double)q, hp[15] / (double)q, hp[16] / (double)q);
    printf("column step cycles/col: warp0 [A %.0f bar1 %.0f B %.0f bar2 %.0f C %.0f]  warp15 [A %.0f bar1 %.0f B %.0f bar2 %.0f C %.0f]\n",
           hp[12] / (double)q, hp[13] / (double)q, hp[14] / (double)q, hp[15] / (double)q, hp[16] / (double)q,
           hp[17] / (double)q, hp[18] / (double)q, hp[19] / (double)q, hp[20] / (double)q, hp[21] / (double)q);
    printf("write split (us): stage %.1f R %.1f V+tau %.1f\n", hp[28] * 1e-3, hp[29] * 1e-3, hp[4] * 1e-3);
    printf("T recurrence: %.0f cycles per panel\n", (double)(long long)hp[27] / ((q + 31) / 32));
    printf("vt_times_panel: %llu calls, stage %.0f cycles/call, dmma %.0f cycles/call\n", hp[26], hp[24] / (double)(hp[26] ? hp[26] : 1), hp[25] / (double)(hp[26] ? hp[26] : 1));
    printf("p=%d q=%d rev=%d: best %.1f us | phases(us): load %.1f left[X %.1f TX %.1f upd %.1f] leafsteps %.1f leafupd %.1f write %.1f G %.1f T %.1f offT %.1f zero %.1f\n",
           p, q, rev, best * 1e3, hp[0] * 1e-3, hp[8] * 1e-3, hp[9] * 1e-3, hp[10] * 1e-3, hp[2] * 1e-3, hp[3] * 1e-3, hp[4] * 1e-3,
           hp[11] * 1e-3, hp[5] * 1e-3, hp[6] * 1e-3, hp[7] * 1e-3);
    // check: with the view W (p x q, view coordinates), Q = I - V T V^T (V in natural order);
    // natural-order window Wn0 = Q * Rn where Rn is the R written back through the view.
    std::vector<double> Wf(W0.size()), V((size_t)p * q), T((size_t)q * q);
    cudaMemcpy(Wf.data(), dW, Wf.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(V.data(), dV, V.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(T.data(), dT, T.size() * 8, cudaMemcpyDeviceToHost);
    // view accessors on host (natural storage index)
    auto vidx = [&](int i, int j) -> size_t { return rev ? (size_t)(p - 1 - i) + (size_t)(q - 1 - j) * p : (size_t)i + (size_t)j * p; };
    // Q = Q_0 Q_1 ..., Q_b = I - V_b T_b V_b^T (32-column blocks, view row order Vv(i,j) = V(nat(i), j));
    // X = R, then X <- Q_b X for b = last .. 0, compare with W0
    double maxres = 0, nrm = 0, maxlow = 0;
    std::vector<double> X((size_t)p * q);
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < q; ++j) {
            X[(size_t)j * p + i] = (i <= j) ? Wf[vidx(i, j)] : 0.0;
            if (i > j && Wf[vidx(i, j)] != 0.0) maxlow = fmax(maxlow, fabs(Wf[vidx(i, j)]));
        }
    auto Vv = [&](int i, int l) { return V[(size_t)l * p + (rev ? p - 1 - i : i)]; };
    const int nbk = (q + 31) / 32;
    for (int b = nbk - 1; b >= 0; --b) {
        const int j0 = 32 * b, nc = std::min(32, q - j0);
        for (int j = 0; j < q; ++j) {
            double y[32], z[32];
            for (int l = 0; l < nc; ++l) {
                double sacc = 0;
                for (int i = 0; i < p; ++i) sacc += Vv(i, j0 + l) * X[(size_t)j * p + i];
                y[l] = sacc;
            }
            for (int l = 0; l < nc; ++l) {
                double sacc = 0;
                for (int m = l; m < nc; ++m) sacc += T[(size_t)(j0 + m) * q + j0 + l] * y[m];
                z[l] = sacc;
            }
            for (int i = 0; i < p; ++i) {
                double sacc = 0;
                for (int l = 0; l < nc; ++l) sacc += Vv(i, j0 + l) * z[l];
                X[(size_t)j * p + i] -= sacc;
            }
        }
    }
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < q; ++j) {
            maxres = fmax(maxres, fabs(X[(size_t)j * p + i] - W0[vidx(i, j)]));
            nrm = fmax(nrm, fabs(W0[vidx(i, j)]));
        }
    printf("check: max |Q R - W0| / max|W0| = %.2e, nonzero below diag = %.2e\n", maxres / nrm, maxlow);
    return 0;
}
