// ht_factor.cu -- staircase window factorizations and their orthogonal factors.
//
// Every staircase step of the absorption (sec. 3.3) is a small QR or QL
// factorization of a window:
//   R1  QL of 2k x k windows of V2, top -> bottom       (sec. 3.3.1b, eq. lqdecomposition)
//   R3  RQ of k x 2k blocks of B, bottom -> top          (sec. 3.3.1 second "e)")
//   L1  QR of 2k x k windows of U2, bottom -> top        (sec. 3.3.2b, eq. qrdecomposition)
//   L3  QR of 2k x k blocks of B, top -> bottom          (sec. 3.3.2f)
// QL and RQ are computed as a Householder QR of a strided *view* of the window
// whose rows/columns are reversed (and, for RQ, transposed); the reflector
// vectors are written back in the natural order, so every window transform is
//   Qw = I - Vnat T Vnat^T   (compact WY, eq. compactWY)
// which is then formed explicitly (2k x 2k) and applied with the DMMA GEMM.
#include "ht_common.cuh"
#include "ht_internal.h"

namespace {

constexpr int FNT = 512;  // threads of the factor CTA

__global__ void __launch_bounds__(FNT) factor_qr_kernel(const FactorDesc *descs, int nd, double *gscratch,
                                                         int smem_doubles)
{
    extern __shared__ __align__(16) double fsm[];
    __shared__ double red[32];
    __shared__ double sc[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = FNT / 32;
    for (int di = 0; di < nd; ++di) {
        const FactorDesc d = descs[di];
        const int p = d.p, q = d.q;
        double *Wk = (p * q <= smem_doubles) ? fsm : gscratch;
        // load the view
        for (int idx = tid; idx < p * q; idx += FNT) {
            int i = idx % p, j = idx / p;
            Wk[idx] = d.W[(int64_t)i * d.rs + (int64_t)j * d.cs];
        }
        __syncthreads();
        for (int c = 0; c < q; ++c) {
            // Householder reflector of Wk(c:p, c) (dlarfg convention, reading R1)
            double ss = 0.0;
            for (int i = c + 1 + tid; i < p; i += FNT) {
                double v = Wk[c * p + i];
                ss += v * v;
            }
            ss = block_sum(ss, red);
            if (tid == 0) {
                double alpha = (c < p) ? Wk[c * p + c] : 0.0;
                double tau = 0.0, scal = 0.0, beta = alpha;
                if (ss > 0.0) {
                    double nrm = sqrt(alpha * alpha + ss);
                    beta = (alpha >= 0.0) ? -nrm : nrm;
                    tau = (beta - alpha) / beta;
                    scal = 1.0 / (alpha - beta);
                }
                sc[0] = tau;
                sc[1] = scal;
                sc[2] = beta;
                d.tau[c] = tau;
            }
            __syncthreads();
            const double tau = sc[0], scal = sc[1];
            if (tau != 0.0) {
                for (int i = c + 1 + tid; i < p; i += FNT) Wk[c * p + i] *= scal;
                __syncthreads();
                // apply (I - tau v v^T) to columns j > c
                for (int j = c + 1 + warp; j < q; j += nw) {
                    double w = 0.0;
                    for (int i = c + lane; i < p; i += 32) {
                        double vi = (i == c) ? 1.0 : Wk[c * p + i];
                        w += vi * Wk[j * p + i];
                    }
                    w = warp_sum(w) * tau;
                    for (int i = c + lane; i < p; i += 32) {
                        double vi = (i == c) ? 1.0 : Wk[c * p + i];
                        Wk[j * p + i] -= w * vi;
                    }
                }
            }
            __syncthreads();
            if (tid == 0 && c < p) Wk[c * p + c] = sc[2];
            __syncthreads();
        }
        // write back R (upper trapezoid of the view, exact zeros below) and Vnat
        for (int idx = tid; idx < p * q; idx += FNT) {
            int i = idx % p, j = idx / p;
            double r = (i <= j) ? Wk[idx] : 0.0;
            d.W[(int64_t)i * d.rs + (int64_t)j * d.cs] = r;
            double v = (i < j) ? 0.0 : (i == j ? 1.0 : Wk[idx]);
            if (i > j && d.tau[j] == 0.0) v = 0.0;
            int inat = d.rev ? (p - 1 - i) : i;
            d.V[(int64_t)j * d.ldv + inat] = v;
        }
        __threadfence();
        __syncthreads();
    }
}

// T from G = V^T V by the dlarft forward recurrence:
// T(c,c) = tau_c, T(0:c,c) = -tau_c T(0:c,0:c) G(0:c,c).  One CTA per window.
__global__ void larft_kernel(const LarftDesc *descs)
{
    const LarftDesc d = descs[blockIdx.x];
    const int q = d.q;
    for (int c = 0; c < q; ++c) {
        const double tc = d.tau[c];
        for (int i = threadIdx.x; i < c; i += blockDim.x) {
            double s = 0.0;
            for (int l = i; l < c; ++l) s += d.T[(int64_t)l * d.ldt + i] * d.G[(int64_t)c * d.ldg + l];
            d.T[(int64_t)c * d.ldt + i] = -tc * s;
        }
        if (threadIdx.x == 0) d.T[(int64_t)c * d.ldt + c] = tc;
        for (int i = c + 1 + threadIdx.x; i < q; i += blockDim.x) d.T[(int64_t)c * d.ldt + i] = 0.0;
        __syncthreads();
    }
}

}  // namespace

int ht_factor_run(cudaStream_t st, const FactorDesc *d_descs, int nd, double *gscratch, int maxpq)
{
    if (nd <= 0) return 0;
    static int smem_max = -1;
    if (smem_max < 0) {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        smem_max = v - 4096;
        cudaFuncSetAttribute(factor_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
    }
    int want = maxpq * 8;
    int smem = want <= smem_max ? want : 0;
    factor_qr_kernel<<<1, FNT, smem, st>>>(d_descs, nd, gscratch, smem / 8);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

int ht_larft_run(cudaStream_t st, const LarftDesc *d_descs, int nd)
{
    if (nd <= 0) return 0;
    larft_kernel<<<nd, 256, 0, st>>>(d_descs);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}
