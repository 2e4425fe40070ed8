// ht_common.cuh -- shared device/host helpers of the B200 HouseHT library.
// (Product code.  Shares nothing with oracle/.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define HT_U 1.1102230246251565404e-16  // unit roundoff 2^-53

#define HT_CUDA_TRY(expr)                                   \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return ht_cuda_fail(_e, #expr, __FILE__, __LINE__); \
    } while (0)

int ht_cuda_fail(cudaError_t e, const char *what, const char *file, int line);

// column-major element access
#define CM(p, i, j, ld) ((p)[(size_t)(j) * (size_t)(ld) + (size_t)(i)])

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide sum; `red` must hold >= 32 doubles of shared memory. All threads get the result.
__device__ __forceinline__ double block_sum(double v, double *red)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t = (threadIdx.x < (unsigned)nw) ? red[threadIdx.x] : 0.0;
    if (wid == 0) {
        t = warp_sum(t);
        if (lane == 0) red[0] = t;
    }
    __syncthreads();
    double r = red[0];
    __syncthreads();
    return r;
}

// ------------------------------------------------------------------ GEMM
// C(MxN) = alpha * op(A)(MxK) * op(B)(KxN) + beta * C, column-major, like dgemm.
// trans = 'N' or 'T'.  Implemented with warp-level FP64 tensor-core MMA
// (mma.sync.m8n8k4.f64 -> SASS DMMA) in ht_gemm.cu.
struct GemmBatchItem {
    const double *A;
    const double *B;
    double *C;
    int64_t lda, ldb, ldc;
    int M, N, K;
    double alpha, beta;
    double diag_add;  // added to C(i,i) after the update (forms I - W V^T in one pass)
};
int ht_gemm(cudaStream_t st, char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha,
            const double *A, int64_t lda, const double *B, int64_t ldb, double beta, double *C,
            int64_t ldc);
// split-K for small outputs with a long K (e.g. the k x k spike U^T B): the K range
// is cut into slices whose partial products go to `work` (>= slices * M * N doubles), then added
// in slice order (deterministic).  Falls back to ht_gemm when the output alone fills the GPU.
int ht_gemm_splitk(cudaStream_t st, char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha,
                   const double *A, int64_t lda, const double *B, int64_t ldb, double beta, double *C,
                   int64_t ldc, double *work, int64_t work_doubles);
// batched: items live in device memory (d_items), all with the same transposition
int ht_gemm_batched(cudaStream_t st, char transA, char transB, const GemmBatchItem *d_items, int nitems,
                    int maxM, int maxN);
// by-value batch (no host->device descriptor copies); any count, launched in chunks of 16
int ht_gemm_multi(cudaStream_t st, char transA, char transB, const GemmBatchItem *items, int nitems);
// copy a (rows x cols) block: dst(i,j) = src(i,j)
int ht_copy2d(cudaStream_t st, int64_t rows, int64_t cols, const double *src, int64_t lds, double *dst,
              int64_t ldd);
int ht_fill2d(cudaStream_t st, int64_t rows, int64_t cols, double *dst, int64_t ldd, double offdiag,
              double diag);

// running flop counter (instrumentation, paper convention P:2161-2162)
extern thread_local double g_ht_flops;

// Per-device one-time setup (function attributes such as the dynamic shared-memory
// opt-in apply per device context): runs `f` once for each device it is called on.
// `done` is a bitmask over device ordinals, guarded by `mu`.
#include <mutex>
template <class F>
int ht_once_per_device(std::mutex &mu, unsigned long long &done, F f)
{
    int dev = 0;
    HT_CUDA_TRY(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    std::lock_guard<std::mutex> lk(mu);
    if (done & bit) return 0;
    const int rc = f();
    if (rc == 0) done |= bit;
    return rc;
}
