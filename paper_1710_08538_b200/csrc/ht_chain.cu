// ht_chain.cu -- chained staircase-window applies with a carried slab.
//
// The absorption (sec. 3.3) multiplies tall strips of A, B, Z, Q by a
// CHAIN of overlapping window transforms: e.g. B(:, j+1:n) <- B * RV_1 ... RV_r
// (eq. commuteQ, steps P:819-825) where RV_i acts on the 2k-wide column
// window i and consecutive windows overlap by k columns.  Rows are independent
// under right multiplication (columns under left multiplication, eq. commuteQ2
// P:1083-1134), so one CTA owns a slab of h rows (or columns) and walks the whole
// chain, keeping the slab's current window in shared memory: columns leave the
// ring (written to HBM once) when the chain has moved past them and enter it once.
// Each window product  slab(h x p) <- slab(h x p) * Qhat_i(p x p)  runs on the FP64
// tensor pipe (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4) with Qhat_i streamed from L2
// in k-chunks (register-staged double buffering).
//
// Left applies X(rows, cols) <- Qhat^T X are the same operation on the transposed
// view (slab = columns, window dimension = rows).
#include "ht_common.cuh"
#include "ht_internal.h"

namespace {

constexpr int CNT = 512;  // threads (16 warps)
constexpr int SLAB_ELEMS = 16384;  // h * CAP doubles of the ring (128 KB)

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

struct ChainParams {
    ChainMat m[3];
    int nm;
    int h, cap;          // slab height, ring capacity (columns); both powers of two
    const ChainWin *wins;
    int nw;
};

template <int KC>
__global__ void __launch_bounds__(CNT, 1) chain_apply_kernel(const __grid_constant__ ChainParams P)
{
    extern __shared__ __align__(16) double csm[];
    const int h = P.h, cap = P.cap;
    constexpr int kc = KC;
    const int ldh = h + 8;          // == 8 mod 32: conflict-free A fragments
    const int ldq = cap + 8;        // == 8 mod 32: conflict-free B fragments
    double *Xs = csm;               // [cap][ldh]  ring of slab columns
    double *Qs = Xs + (size_t)cap * ldh;  // [2][kc][ldq]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;

    // slab tasks over all matrices; a capped grid loops over them (persistent style), so that
    // concurrent streams keep SMs free for the factorization chain
    int64_t ntask = 0;
    for (int q = 0; q < P.nm; ++q) ntask += (P.m[q].s_end - P.m[q].s_begin + h - 1) / h;
    for (int64_t task = blockIdx.x; task < ntask; task += gridDim.x) {
    __syncthreads();  // the ring of the previous task is no longer read
    int mi = 0;
    int64_t blk = task;
    for (; mi < P.nm; ++mi) {
        const int64_t ns = (P.m[mi].s_end - P.m[mi].s_begin + h - 1) / h;
        if (blk < ns) break;
        blk -= ns;
    }
    if (mi >= P.nm) continue;
    const ChainMat M = P.m[mi];
    const int64_t s0 = M.s_begin + blk * h;
    const int hs = (int)(M.s_end - s0 < (int64_t)h ? M.s_end - s0 : (int64_t)h);  // valid slab rows
    auto gaddr = [&](int s, int64_t c) -> double * {
        return M.left ? M.X + c + (s0 + s) * M.ld : M.X + (s0 + s) + c * M.ld;
    };
    const int capm = cap - 1;
    auto slot = [&](int64_t c) -> int { return (int)c & capm; };
    // move columns [c_lo, c_hi) between HBM and the ring (coalesced along the contiguous
    // direction: rows of a column for right applies, columns of a row for left applies)
    auto load_cols = [&](int64_t c_lo, int64_t c_hi) {
        const int nc = (int)(c_hi - c_lo);
        if (nc <= 0) return;
        if (M.left) {
            for (int s = warp; s < h; s += CNT / 32)
                for (int c = lane; c < nc; c += 32)
                    Xs[slot(c_lo + c) * ldh + s] = (s < hs) ? *gaddr(s, c_lo + c) : 0.0;
        } else {
            for (int c = warp; c < nc; c += CNT / 32)
                for (int s = lane; s < h; s += 32)
                    Xs[slot(c_lo + c) * ldh + s] = (s < hs) ? *gaddr(s, c_lo + c) : 0.0;
        }
    };
    auto store_cols = [&](int64_t c_lo, int64_t c_hi) {
        const int nc = (int)(c_hi - c_lo);
        if (nc <= 0) return;
        if (M.left) {
            for (int s = warp; s < hs; s += CNT / 32)
                for (int c = lane; c < nc; c += 32) *gaddr(s, c_lo + c) = Xs[slot(c_lo + c) * ldh + s];
        } else {
            for (int c = warp; c < nc; c += CNT / 32)
                for (int s = lane; s < hs; s += 32) *gaddr(s, c_lo + c) = Xs[slot(c_lo + c) * ldh + s];
        }
    };
    // padding columns [o + p, o + pp) of a window must read as zeros (their Qhat rows are 0,
    // but 0 * NaN would not be): they are dead ring slots, zeroed before the window runs
    auto zero_pad = [&](int64_t o, int p) {
        const int pp = (p + 31) & ~31;
        for (int idx = tid; idx < (pp - p) * ldh; idx += CNT) Xs[slot(o + p + idx / ldh) * ldh + idx % ldh] = 0.0;
    };

    {
        const ChainWin w0 = P.wins[0];
        load_cols(w0.o, (int64_t)w0.o + w0.p);
        zero_pad(w0.o, w0.p);
    }
    for (int wi = 0; wi < P.nw; ++wi) {
        const ChainWin W = P.wins[wi];
        const int p = W.p, pp = (p + 31) & ~31;
        const int64_t lo = W.lo[mi], hi = W.hi[mi];
        const bool active = (s0 < hi) && (s0 + hs > lo) && p > 0;
        __syncthreads();
        if (active) {
            const int nwr = h / 32, nwc = pp / 32;
            const int wr = warp % nwr, wc = warp / nwr;
            const bool wact = wc < nwc;
            double acc[4][4][2];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
            const int per = (kc * pp + CNT - 1) / CNT;  // staged elements per thread (<= 8)
            double rq[8];
            auto fetch = [&](int k0) {
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    if (e >= per) break;
                    const int idx = tid + e * CNT;
                    const int kr = idx % KC, c = idx / KC;
                    double v = 0.0;
                    if (c < p && k0 + kr < p) v = W.Qw[(size_t)(k0 + kr) + (size_t)c * p];
                    rq[e] = v;
                }
            };
            auto put = [&](int buf) {
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    if (e >= per) break;
                    const int idx = tid + e * CNT;
                    const int kr = idx % KC, c = idx / KC;
                    if (c < pp) Qs[(size_t)buf * kc * ldq + kr * ldq + c] = rq[e];
                }
            };
            const int nk = pp / kc + (pp % kc ? 1 : 0);
            fetch(0);
            put(0);
            __syncthreads();
            for (int kt = 0; kt < nk; ++kt) {
                const int buf = kt & 1;
                if (kt + 1 < nk) fetch((kt + 1) * kc);
                if (wact) {
                    const double *qb = Qs + (size_t)buf * kc * ldq;
#pragma unroll
                    for (int kk = 0; kk < KC; kk += 4) {
                        const int64_t cA = (int64_t)W.o + kt * kc + kk + t4;  // window column of A frag
                        const double *xa = Xs + slot(cA) * ldh + wr * 32 + g;
                        double af[4], bf[4];
#pragma unroll
                        for (int a = 0; a < 4; ++a) af[a] = xa[8 * a];
#pragma unroll
                        for (int b = 0; b < 4; ++b) bf[b] = qb[(kk + t4) * ldq + wc * 32 + 8 * b + g];
#pragma unroll
                        for (int a = 0; a < 4; ++a)
#pragma unroll
                            for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
                    }
                }
                if (kt + 1 < nk) put(buf ^ 1);
                __syncthreads();
            }
            // epilogue: slab(s, o + c) <- acc for s in [lo, hi), c < p
            if (wact) {
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const int s = wr * 32 + 8 * a + g;
                            const int c = wc * 32 + 8 * b + 2 * t4 + hh;
                            const int64_t sg = s0 + s;
                            if (c < p && sg >= lo && sg < hi && s < hs)
                                Xs[slot((int64_t)W.o + c) * ldh + s] = acc[a][b][hh];
                        }
            }
        }
        __syncthreads();
        // transition: flush columns leaving the chain, load columns entering it
        const int64_t a0 = W.o, a1 = (int64_t)W.o + W.p;
        if (wi + 1 < P.nw) {
            const ChainWin N = P.wins[wi + 1];
            const int64_t b0 = N.o, b1 = (int64_t)N.o + N.p;
            // leaving: [a0, a1) \ [b0, b1); entering: [b0, b1) \ [a0, a1)  (monotone chains)
            store_cols(a0, a1 < b0 ? a1 : b0);
            store_cols(a0 > b1 ? a0 : b1, a1);
            __syncthreads();
            load_cols(b0, b1 < a0 ? b1 : a0);
            load_cols(b0 > a1 ? b0 : a1, b1);
            __syncthreads();
            zero_pad(N.o, N.p);
        } else {
            store_cols(a0, a1);
        }
    }
    }  // task loop
}

}  // namespace

// Apply a chain of explicit window transforms to up to 3 matrices (one launch).
// d_wins: device array of nw windows (application order, monotone offsets).
int ht_chain_apply(cudaStream_t st, const ChainMat *mats, int nm, const ChainWin *d_wins, int nw, int pmax, int maxgrid)
{
    if (nm <= 0 || nw <= 0) return 0;
    ChainParams P;
    P.nm = nm;
    for (int i = 0; i < nm; ++i) P.m[i] = mats[i];
    const int pp = (pmax + 31) & ~31;
    P.cap = pp <= 256 ? 256 : 512;
    P.h = SLAB_ELEMS / P.cap;          // 64 (p <= 256) or 32 (p <= 512)
    if (pp <= 128) { P.cap = 128; P.h = 128; }
    P.wins = d_wins;
    P.nw = nw;
    int64_t nblk = 0;
    for (int i = 0; i < nm; ++i)
        if (mats[i].s_end > mats[i].s_begin) nblk += (mats[i].s_end - mats[i].s_begin + P.h - 1) / P.h;
    if (nblk == 0) return 0;
    const int kc = P.cap <= 256 ? 16 : 8;
    const size_t smem = ((size_t)P.cap * (P.h + 8) + 2 * (size_t)kc * (P.cap + 8)) * sizeof(double);
    static bool init = false;
    if (!init) {
        const int mx = (int)(SLAB_ELEMS + 8 * 512 + 2 * 16 * 264) * 8;
        HT_CUDA_TRY(cudaFuncSetAttribute(chain_apply_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        HT_CUDA_TRY(cudaFuncSetAttribute(chain_apply_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        init = true;
    }
    const unsigned grid = (unsigned)(maxgrid > 0 && nblk > maxgrid ? maxgrid : nblk);
    if (kc == 16) chain_apply_kernel<16><<<grid, CNT, smem, st>>>(P);
    else chain_apply_kernel<8><<<grid, CNT, smem, st>>>(P);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}
