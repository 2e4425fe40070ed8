// ht_gemm.cu -- FP64 GEMM on the B200 FP64 tensor pipe (mma.sync m8n8k4 f64 -> SASS DMMA).
//
// Used for every level-3 step of HouseHT (sec. 3.3): the staircase
// window applies C <- C*Qw / Qw^T*C (eq. commuteQ, commuteQ2 P:1083-1134),
// the W-updates and the Remark-2 GEMM.
// Note: sm_100a has no tcgen05 kind::f64; DMMA is the FP64 tensor path.
#include "ht_common.cuh"
#include <stdio.h>
#include <algorithm>

thread_local double g_ht_flops = 0.0;  // per calling thread: concurrent calls on different devices

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;
constexpr int LDS = BM + 8;  // 72 doubles: conflict-free fragment loads

__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// TA/TB: false = 'N' (column-major operand), true = 'T'
template <bool TA, bool TB>
__device__ __forceinline__ void gemm_tile(const double *__restrict__ A, int64_t lda, const double *__restrict__ B,
                                          int64_t ldb, double *__restrict__ C, int64_t ldc, int M, int N, int K,
                                          double alpha, double beta, int m0, int n0, double diag_add = 0.0)
{
    __shared__ __align__(16) double As[2][BK][LDS];
    __shared__ __align__(16) double Bs[2][BK][LDS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;  // 2 x 4 warps, warp tile 32 x 16
    const int g = lane >> 2, t = lane & 3;

    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    double ra[4], rb[4];
    auto load_a = [&](int k0) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            int m, k;
            if (!TA) { m = tid & 63; k = (tid >> 6) + 4 * e; }
            else     { k = tid & 15; m = (tid >> 4) + 16 * e; }
            int gm = m0 + m, gk = k0 + k;
            double v = 0.0;
            if (gm < M && gk < K) v = TA ? A[(size_t)gm * lda + gk] : A[(size_t)gk * lda + gm];
            ra[e] = v;
        }
    };
    auto load_b = [&](int k0) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            int n, k;
            if (TB) { n = tid & 63; k = (tid >> 6) + 4 * e; }
            else    { k = tid & 15; n = (tid >> 4) + 16 * e; }
            int gn = n0 + n, gk = k0 + k;
            double v = 0.0;
            if (gn < N && gk < K) v = TB ? B[(size_t)gk * ldb + gn] : B[(size_t)gn * ldb + gk];
            rb[e] = v;
        }
    };
    auto store_ab = [&](int buf) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            int m, k;
            if (!TA) { m = tid & 63; k = (tid >> 6) + 4 * e; }
            else     { k = tid & 15; m = (tid >> 4) + 16 * e; }
            As[buf][k][m] = ra[e];
            int n, kb;
            if (TB) { n = tid & 63; kb = (tid >> 6) + 4 * e; }
            else    { kb = tid & 15; n = (tid >> 4) + 16 * e; }
            Bs[buf][kb][n] = rb[e];
        }
    };

    const int nk = (K + BK - 1) / BK;
    if (nk > 0) {
        load_a(0);
        load_b(0);
        store_ab(0);
    }
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) {
            load_a((kt + 1) * BK);
            load_b((kt + 1) * BK);
        }
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = As[buf][kk + t][wm + 8 * i + g];
#pragma unroll
            for (int j = 0; j < 2; ++j) bf[j] = Bs[buf][kk + t][wn + 8 * j + g];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        if (kt + 1 < nk) store_ab(buf ^ 1);
        __syncthreads();
    }
    // epilogue: fragment (g, 2t + h) of each 8x8 tile
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                int gm = m0 + wm + 8 * i + g, gn = n0 + wn + 8 * j + 2 * t + h;
                if (gm < M && gn < N) {
                    double *cp = C + (size_t)gn * ldc + gm;
                    double v = alpha * acc[i][j][h];
                    if (beta != 0.0) v += beta * *cp;
                    if (gm == gn) v += diag_add;
                    *cp = v;
                }
            }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(NT) gemm_kernel(const double *A, int64_t lda, const double *B, int64_t ldb,
                                                  double *C, int64_t ldc, int M, int N, int K, double alpha,
                                                  double beta)
{
    gemm_tile<TA, TB>(A, lda, B, ldb, C, ldc, M, N, K, alpha, beta, blockIdx.x * BM, blockIdx.y * BN);
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(NT) gemm_batched_kernel(const GemmBatchItem *items)
{
    const GemmBatchItem it = items[blockIdx.z];
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    if (m0 >= it.M || n0 >= it.N) return;
    gemm_tile<TA, TB>(it.A, it.lda, it.B, it.ldb, it.C, it.ldc, it.M, it.N, it.K, it.alpha, it.beta, m0, n0,
                      it.diag_add);
}

// slice z of the K range: work[z] = A(:, K_z) B(K_z, :)  (M x N, column-major, ld M)
template <bool TA, bool TB>
__global__ void __launch_bounds__(NT) gemm_splitk_kernel(const double *A, int64_t lda, const double *B, int64_t ldb,
                                                         double *work, int M, int N, int K, int kchunk)
{
    const int z = blockIdx.z;
    const int64_t k0 = (int64_t)z * kchunk;
    const int kc = (int)((int64_t)kchunk < K - k0 ? (int64_t)kchunk : K - k0);
    const double *Az = TA ? A + k0 : A + k0 * lda;
    const double *Bz = TB ? B + k0 * ldb : B + k0;
    gemm_tile<TA, TB>(Az, lda, Bz, ldb, work + (size_t)z * M * N, M, M, N, kc, 1.0, 0.0, blockIdx.x * BM, blockIdx.y * BN);
}

// C = alpha * sum_z work[z] + beta * C, slices added in order z = 0, 1, ... (deterministic)
__global__ void splitk_reduce_kernel(const double *__restrict__ work, int nz, int M, int N, double alpha, double beta,
                                     double *C, int64_t ldc)
{
    const int64_t MN = (int64_t)M * N;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < MN; e += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int z = 0; z < nz; ++z) s += work[(size_t)z * MN + e];
        const int64_t gm = e % M, gn = e / M;
        double *cp = C + gn * ldc + gm;
        double v = alpha * s;
        if (beta != 0.0) v += beta * *cp;
        *cp = v;
    }
}

struct GemmBatch16 {
    GemmBatchItem it[16];
};

template <bool TA, bool TB>
__global__ void __launch_bounds__(NT) gemm_multi_kernel(const GemmBatch16 b)
{
    const GemmBatchItem &it = b.it[blockIdx.z];
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    if (m0 >= it.M || n0 >= it.N) return;
    gemm_tile<TA, TB>(it.A, it.lda, it.B, it.ldb, it.C, it.ldc, it.M, it.N, it.K, it.alpha, it.beta, m0, n0,
                      it.diag_add);
}

__global__ void copy2d_kernel(int64_t rows, int64_t cols, const double *src, int64_t lds, double *dst, int64_t ldd)
{
    for (int64_t j = blockIdx.y; j < cols; j += gridDim.y)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
            dst[j * ldd + i] = src[j * lds + i];
}

__global__ void fill2d_kernel(int64_t rows, int64_t cols, double *dst, int64_t ldd, double off, double dia)
{
    for (int64_t j = blockIdx.y; j < cols; j += gridDim.y)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
            dst[j * ldd + i] = (i == j) ? dia : off;
}

}  // namespace

int ht_gemm(cudaStream_t st, char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha,
            const double *A, int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc)
{
    if (M <= 0 || N <= 0) return 0;
    g_ht_flops += 2.0 * (double)M * (double)N * (double)K;
    dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN));
    const bool ta = (transA == 'T' || transA == 't'), tb = (transB == 'T' || transB == 't');
    if (!ta && !tb) gemm_kernel<false, false><<<grid, NT, 0, st>>>(A, lda, B, ldb, C, ldc, (int)M, (int)N, (int)K, alpha, beta);
    else if (!ta && tb) gemm_kernel<false, true><<<grid, NT, 0, st>>>(A, lda, B, ldb, C, ldc, (int)M, (int)N, (int)K, alpha, beta);
    else if (ta && !tb) gemm_kernel<true, false><<<grid, NT, 0, st>>>(A, lda, B, ldb, C, ldc, (int)M, (int)N, (int)K, alpha, beta);
    else gemm_kernel<true, true><<<grid, NT, 0, st>>>(A, lda, B, ldb, C, ldc, (int)M, (int)N, (int)K, alpha, beta);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

int ht_gemm_splitk(cudaStream_t st, char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha,
                   const double *A, int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
                   double *work, int64_t work_doubles)
{
    if (M <= 0 || N <= 0) return 0;
    const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
    // slices of >= 256 K, enough of them to give ~1 CTA per SM, bounded by the workspace
    int64_t nz = std::min<int64_t>((K + 255) / 256, std::max<int64_t>(1, 148 / tiles));
    nz = std::min<int64_t>(nz, work ? work_doubles / (M * N) : 0);
    if (nz < 2) return ht_gemm(st, transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    const int kchunk = (int)(((K + nz - 1) / nz + 3) & ~(int64_t)3);
    nz = (K + kchunk - 1) / kchunk;
    g_ht_flops += 2.0 * (double)M * (double)N * (double)K;
    dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN), (unsigned)nz);
    const bool ta = (transA == 'T' || transA == 't'), tb = (transB == 'T' || transB == 't');
    if (!ta && !tb) gemm_splitk_kernel<false, false><<<grid, NT, 0, st>>>(A, lda, B, ldb, work, (int)M, (int)N, (int)K, kchunk);
    else if (!ta && tb) gemm_splitk_kernel<false, true><<<grid, NT, 0, st>>>(A, lda, B, ldb, work, (int)M, (int)N, (int)K, kchunk);
    else if (ta && !tb) gemm_splitk_kernel<true, false><<<grid, NT, 0, st>>>(A, lda, B, ldb, work, (int)M, (int)N, (int)K, kchunk);
    else gemm_splitk_kernel<true, true><<<grid, NT, 0, st>>>(A, lda, B, ldb, work, (int)M, (int)N, (int)K, kchunk);
    HT_CUDA_TRY(cudaGetLastError());
    const int64_t MN = M * N;
    splitk_reduce_kernel<<<(unsigned)std::min<int64_t>((MN + 255) / 256, 148), 256, 0, st>>>(work, (int)nz, (int)M, (int)N,
                                                                                            alpha, beta, C, ldc);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

int ht_gemm_batched(cudaStream_t st, char transA, char transB, const GemmBatchItem *d_items, int nitems, int maxM,
                    int maxN)
{
    if (nitems <= 0 || maxM <= 0 || maxN <= 0) return 0;
    dim3 grid((unsigned)((maxM + BM - 1) / BM), (unsigned)((maxN + BN - 1) / BN), (unsigned)nitems);
    const bool ta = (transA == 'T' || transA == 't'), tb = (transB == 'T' || transB == 't');
    if (!ta && !tb) gemm_batched_kernel<false, false><<<grid, NT, 0, st>>>(d_items);
    else if (!ta && tb) gemm_batched_kernel<false, true><<<grid, NT, 0, st>>>(d_items);
    else if (ta && !tb) gemm_batched_kernel<true, false><<<grid, NT, 0, st>>>(d_items);
    else gemm_batched_kernel<true, true><<<grid, NT, 0, st>>>(d_items);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

int ht_gemm_multi(cudaStream_t st, char transA, char transB, const GemmBatchItem *items, int nitems)
{
    const bool ta = (transA == 'T' || transA == 't'), tb = (transB == 'T' || transB == 't');
    for (int base = 0; base < nitems; base += 16) {
        GemmBatch16 b;
        int cnt = 0, maxM = 0, maxN = 0;
        for (int i = base; i < nitems && i < base + 16; ++i) {
            if (items[i].M <= 0 || items[i].N <= 0) continue;
            b.it[cnt++] = items[i];
            maxM = items[i].M > maxM ? items[i].M : maxM;
            maxN = items[i].N > maxN ? items[i].N : maxN;
            g_ht_flops += 2.0 * items[i].M * (double)items[i].N * items[i].K;
        }
        if (cnt == 0) continue;
        dim3 grid((unsigned)((maxM + BM - 1) / BM), (unsigned)((maxN + BN - 1) / BN), (unsigned)cnt);
        if (!ta && !tb) gemm_multi_kernel<false, false><<<grid, NT, 0, st>>>(b);
        else if (!ta && tb) gemm_multi_kernel<false, true><<<grid, NT, 0, st>>>(b);
        else if (ta && !tb) gemm_multi_kernel<true, false><<<grid, NT, 0, st>>>(b);
        else gemm_multi_kernel<true, true><<<grid, NT, 0, st>>>(b);
        HT_CUDA_TRY(cudaGetLastError());
    }
    return 0;
}

int ht_copy2d(cudaStream_t st, int64_t rows, int64_t cols, const double *src, int64_t lds, double *dst, int64_t ldd)
{
    if (rows <= 0 || cols <= 0) return 0;
    dim3 grid((unsigned)((rows + 255) / 256 < 64 ? (rows + 255) / 256 : 64), (unsigned)(cols < 4096 ? cols : 4096));
    copy2d_kernel<<<grid, 256, 0, st>>>(rows, cols, src, lds, dst, ldd);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

int ht_fill2d(cudaStream_t st, int64_t rows, int64_t cols, double *dst, int64_t ldd, double offdiag, double diag)
{
    if (rows <= 0 || cols <= 0) return 0;
    dim3 grid((unsigned)((rows + 255) / 256 < 64 ? (rows + 255) / 256 : 64), (unsigned)(cols < 4096 ? cols : 4096));
    fill2d_kernel<<<grid, 256, 0, st>>>(rows, cols, dst, ldd, offdiag, diag);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}
