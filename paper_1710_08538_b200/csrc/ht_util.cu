// ht_util.cu -- small utility kernels of the B200 HouseHT library.
#include "ht_common.cuh"
#include "ht_internal.h"
#include <stdio.h>

namespace {

// ||M||_F^2 in a fixed order (bitwise reproducible run to run and rank to rank): block b
// sums columns b, b + FRO_BLOCKS, ... (each thread a fixed row stride, then a fixed tree),
// the partials are added by one block in index order (fro_final_kernel).
constexpr int FRO_BLOCKS = 592;  // 4 x 148 SMs
__global__ void fro_kernel(int64_t rows, int64_t cols, const double *M, int64_t ld, double *part)
{
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t j = blockIdx.x; j < cols; j += gridDim.x)
        for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
            const double v = M[j * ld + i];
            s = fma(v, v, s);
        }
    s = block_sum(s, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void fro_final_kernel(const double *part, int np, double *out)
{
    __shared__ double red[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
    s = block_sum(s, red);
    if (threadIdx.x == 0) *out = s;
}

// flags[0] |= non-finite in A or B; flags[1] |= nonzero strictly-lower entry of B;
// maxbits[0] = max |A|, maxbits[1] = max |B| (bit patterns of non-negative doubles order
// like the values, so an integer atomicMax is exact and order-independent)
__global__ void check_kernel(int64_t n, const double *A, int64_t lda, const double *B, int64_t ldb, int *flags,
                             unsigned long long *maxbits)
{
    int bad = 0, low = 0;
    double ma = 0.0, mb = 0.0;
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
            double a = A[j * lda + i], b = B[j * ldb + i];
            if (!isfinite(a) || !isfinite(b)) bad = 1;
            if (i > j && b != 0.0) low = 1;
            ma = fmax(ma, fabs(a));
            mb = fmax(mb, fabs(b));
        }
    if (bad) atomicOr(&flags[0], 1);
    if (low) atomicOr(&flags[1], 1);
    ma = warp_max(ma);
    mb = warp_max(mb);
    if ((threadIdx.x & 31) == 0) {
        if (ma > 0.0) atomicMax(&maxbits[0], (unsigned long long)__double_as_longlong(ma));
        if (mb > 0.0) atomicMax(&maxbits[1], (unsigned long long)__double_as_longlong(mb));
    }
}

// M <- M * s (s a power of two: exact)
__global__ void scale_kernel(int64_t rows, int64_t cols, double *M, int64_t ld, double s)
{
    for (int64_t j = blockIdx.y; j < cols; j += gridDim.y)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
            M[j * ld + i] *= s;
}

// End of a reduction: exact structural zeros of H (i > j+1) and T (i > j) (Alg. 2 "Set ... <- 0",
// P:2378) unless `partial`, the inverse power-of-two scaling of H and T, and a scan
// of H, T, Q, Z for non-finite entries (flag[0] |= 1).
__global__ void finish_kernel(int64_t n, double *A, int64_t lda, double *B, int64_t ldb, const double *Q,
                              int64_t ldq, const double *Z, int64_t ldz, double sa, double sb, int partial, int *flag)
{
    int bad = 0;
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
            double a = A[j * lda + i], b = B[j * ldb + i];
            if (!partial && i > j + 1) a = 0.0;
            if (!partial && i > j) b = 0.0;
            a *= sa;
            b *= sb;
            A[j * lda + i] = a;
            B[j * ldb + i] = b;
            bad |= !isfinite(a) || !isfinite(b);
            if (Q) bad |= !isfinite(Q[j * ldq + i]);
            if (Z) bad |= !isfinite(Z[j * ldz + i]);
        }
    if (bad) atomicOr(flag, 1);
}

// Counter-based normal draw (reading R-Z7): splitmix64 hash of (seed, key, row, ctr)
// -> two uniforms -> Box-Muller.  This generator is a shared SPEC (DESIGN.md R-Z7): the
// oracle implements the same counter-based generator in its own file; the two share no
// code.  The GPU keys draws by the panel start column, the oracle by the column.
__device__ __forceinline__ uint64_t mix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ double rho_draw(uint64_t seed, int64_t key, int64_t row, uint32_t ctr)
{
    uint64_t h = mix64(seed ^ mix64((uint64_t)key * 0x100000001B3ULL ^ mix64((uint64_t)row + ((uint64_t)ctr << 40))));
    uint64_t h2 = mix64(h);
    double u1 = ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    double u2 = ((double)(h2 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

// Desingularisation of tiny pivots of B(r0:n, r0:n) (Remark 1 P:135-139):
// |b_ii| < thresh -> repl * rho, |rho| >= 1/2 (readings R-Z6, R-Z7), persisted in B.
__global__ void desing_kernel(int64_t n, double *B, int64_t ldb, int64_t r0, double thresh, double repl,
                              uint64_t seed, int64_t key, int *count)
{
    for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double *d = B + i * ldb + i;
        if (fabs(*d) < thresh) {
            uint32_t ctr = 0;
            double rho;
            do { rho = rho_draw(seed, key, i, ctr++); } while (fabs(rho) < 0.5);
            *d = repl * rho;
            atomicAdd(count, 1);
        }
    }
}

// M(i, j) = 0 for i > j + diag_offset  (exact structural zeros)
__global__ void zero_lower_kernel(int64_t rows, int64_t cols, double *M, int64_t ld, int64_t off)
{
    for (int64_t j = blockIdx.y; j < cols; j += gridDim.y)
        for (int64_t i = j + off + 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
             i += (int64_t)gridDim.x * blockDim.x)
            if (i >= 0) M[j * ld + i] = 0.0;
}

// Column j of B exactly zero -> zc[j] = 1 (bitwise-zero test; sec. 3.5.1 deflates structural
// zeros only); any nonzero off-diagonal entry -> flags[0] |= 1 (B not diagonal)
__global__ void zero_cols_kernel(int64_t n, const double *B, int64_t ldb, int *zc, int *flags)
{
    __shared__ int any;
    for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
        if (threadIdx.x == 0) any = 0;
        __syncthreads();
        int nz = 0, off = 0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const double v = B[j * ldb + i];
            if (v != 0.0) {
                nz = 1;
                if (i != j) off = 1;
            }
        }
        if (nz) atomicOr(&any, 1);
        if (off) atomicOr(&flags[0], 1);
        __syncthreads();
        if (threadIdx.x == 0) zc[j] = any ? 0 : 1;
        __syncthreads();
    }
}

// dst(i, j) = src(perm_r[i], perm_c[j]) (perm_* null: identity)
__global__ void permute_kernel(int64_t rows, int64_t cols, const double *src, int64_t lds, double *dst, int64_t ldd,
                               const int64_t *perm_r, const int64_t *perm_c)
{
    for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
        const int64_t sj = perm_c ? perm_c[j] : j;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
            dst[j * ldd + i] = src[sj * lds + (perm_r ? perm_r[i] : i)];
    }
}

// M = the permutation matrix with columns e_{perm[j]} (M(perm[j], j) = 1)
__global__ void perm_matrix_kernel(int64_t n, double *M, int64_t ld, const int64_t *perm)
{
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
            M[j * ld + i] = (i == perm[j]) ? 1.0 : 0.0;
}

}  // namespace

int ht_zero_columns(cudaStream_t st, int64_t n, const double *B, int64_t ldb, int *d_zc, int *d_flags)
{
    HT_CUDA_TRY(cudaMemsetAsync(d_flags, 0, sizeof(int), st));
    if (n <= 0) return 0;
    zero_cols_kernel<<<(unsigned)(n < 4096 ? n : 4096), 256, 0, st>>>(n, B, ldb, d_zc, d_flags);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

int ht_permute(cudaStream_t st, int64_t rows, int64_t cols, const double *src, int64_t lds, double *dst, int64_t ldd,
               const int64_t *d_perm_r, const int64_t *d_perm_c)
{
    if (rows <= 0 || cols <= 0) return 0;
    dim3 grid((unsigned)((rows + 255) / 256 < 16 ? (rows + 255) / 256 : 16), (unsigned)(cols < 4096 ? cols : 4096));
    permute_kernel<<<grid, 256, 0, st>>>(rows, cols, src, lds, dst, ldd, d_perm_r, d_perm_c);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

int ht_perm_matrix(cudaStream_t st, int64_t n, double *M, int64_t ld, const int64_t *d_perm)
{
    if (n <= 0) return 0;
    dim3 grid((unsigned)((n + 255) / 256 < 16 ? (n + 255) / 256 : 16), (unsigned)(n < 4096 ? n : 4096));
    perm_matrix_kernel<<<grid, 256, 0, st>>>(n, M, ld, d_perm);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

int ht_cuda_fail(cudaError_t e, const char *what, const char *file, int line)
{
    fprintf(stderr, "[ht_b200] CUDA error %s (%s) at %s:%d: %s\n", cudaGetErrorName(e), cudaGetErrorString(e), file,
            line, what);
    return 2;  // HT_ECUDA
}

int ht_fro_norm_sq(cudaStream_t st, int64_t rows, int64_t cols, const double *M, int64_t ld, double *d_out,
                   double *d_part)
{
    HT_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(double), st));
    if (rows <= 0 || cols <= 0) return 0;
    fro_kernel<<<FRO_BLOCKS, 256, 0, st>>>(rows, cols, M, ld, d_part);
    HT_CUDA_TRY(cudaGetLastError());
    fro_final_kernel<<<1, 256, 0, st>>>(d_part, FRO_BLOCKS, d_out);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}
int ht_fro_scratch_size() { return FRO_BLOCKS; }

int ht_check_input(cudaStream_t st, int64_t n, const double *A, int64_t lda, const double *B, int64_t ldb, int *d_flags,
                   unsigned long long *d_maxbits)
{
    HT_CUDA_TRY(cudaMemsetAsync(d_flags, 0, 2 * sizeof(int), st));
    HT_CUDA_TRY(cudaMemsetAsync(d_maxbits, 0, 2 * sizeof(unsigned long long), st));
    if (n <= 0) return 0;
    dim3 grid(4, (unsigned)(n < 2048 ? n : 2048));
    check_kernel<<<grid, 256, 0, st>>>(n, A, lda, B, ldb, d_flags, d_maxbits);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

int ht_scale(cudaStream_t st, int64_t rows, int64_t cols, double *M, int64_t ld, double s)
{
    if (rows <= 0 || cols <= 0 || s == 1.0) return 0;
    dim3 grid((unsigned)((rows + 255) / 256 < 8 ? (rows + 255) / 256 : 8), (unsigned)(cols < 4096 ? cols : 4096));
    scale_kernel<<<grid, 256, 0, st>>>(rows, cols, M, ld, s);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

int ht_finish(cudaStream_t st, int64_t n, double *A, int64_t lda, double *B, int64_t ldb, const double *Q, int64_t ldq,
              const double *Z, int64_t ldz, double sa, double sb, int partial, int *d_flag)
{
    HT_CUDA_TRY(cudaMemsetAsync(d_flag, 0, sizeof(int), st));
    if (n <= 0) return 0;
    dim3 grid((unsigned)((n + 255) / 256 < 8 ? (n + 255) / 256 : 8), (unsigned)(n < 4096 ? n : 4096));
    finish_kernel<<<grid, 256, 0, st>>>(n, A, lda, B, ldb, Q, ldq, Z, ldz, sa, sb, partial, d_flag);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

int ht_desingularize(cudaStream_t st, int64_t n, double *B, int64_t ldb, int64_t r0, double thresh, double repl,
                     uint64_t seed, int64_t key, int *d_count)
{
    if (r0 >= n) return 0;
    int64_t m = n - r0;
    desing_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(n, B, ldb, r0, thresh, repl, seed, key, d_count);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

int ht_zero_lower(cudaStream_t st, int64_t rows, int64_t cols, double *M, int64_t ld, int64_t diag_offset)
{
    if (rows <= 0 || cols <= 0) return 0;
    dim3 grid((unsigned)((rows + 255) / 256 < 32 ? (rows + 255) / 256 : 32), (unsigned)(cols < 4096 ? cols : 4096));
    zero_lower_kernel<<<grid, 256, 0, st>>>(rows, cols, M, ld, diag_offset);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}
