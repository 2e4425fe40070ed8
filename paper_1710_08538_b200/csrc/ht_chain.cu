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
#include <algorithm>
#include "ht_common.cuh"
#include "ht_internal.h"

namespace {

constexpr int CNT = 512;  // threads (16 warps)
#ifndef CHAIN_PAD
#define CHAIN_PAD 4
#endif
constexpr int SLAB_ELEMS = 16384;  // h * CAP doubles of the ring (128 KB)

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double *dst, const double *src, bool ok)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

struct ChainParams {
    ChainMat m[3];
    int nm;
    int h, cap;          // slab height, ring capacity (columns); both powers of two
    const ChainWin *wins;  // null: the windows are inl[0 .. nw) (launch parameters, nw <= 4)
    int nw;
    ChainWin inl[4];
    __device__ __forceinline__ ChainWin win(int i) const { return wins ? wins[i] : inl[i]; }
};

#ifdef CHAIN_PROF
// development instrumentation (scripts/micro/chain_prof.py): per-CTA cycles in
// [0] first-window load, [1] k-chunk loop, [2] whole window product incl. epilogue, [3] transition, [4] barrier waits in the loop
__device__ unsigned long long g_chain_prof[256][8];
#define CPROF_T(v) const long long v = clock64()
#define CPROF_ADD(i, a, b) if (tid == 0) g_chain_prof[blockIdx.x][i] += (unsigned long long)((b) - (a))
#else
#define CPROF_T(v)
#define CPROF_ADD(i, a, b)
#endif

template <int KC>
__global__ void __launch_bounds__(CNT, 1) chain_apply_kernel(const __grid_constant__ ChainParams P)
{
    extern __shared__ __align__(16) double csm[];
    const int h = P.h, cap = P.cap;
    constexpr int kc = KC;
    const int ldh = h + CHAIN_PAD;    // == 4 mod 16 (in doubles): conflict-free 64-bit A fragments
    const int ldq = cap + CHAIN_PAD;  // (lanes t4*ld + g hit 16 distinct bank pairs per half-warp)
    double *Xs = csm;               // [cap][ldh]  ring of slab columns
    double *Qs = Xs + (size_t)cap * ldh;  // [2][kc][ldq]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;

    // Qhat chunks arrive by bulk copy (cp.async.bulk, one per Qhat row, completion counted on
    // the buffer's mbarrier) when the window's rows are 16-byte aligned; else by 8-byte cp.async
    __shared__ __align__(8) unsigned long long qbar[2], ebar;
    const unsigned qb0 = (unsigned)__cvta_generic_to_shared(&qbar[0]);
    const unsigned eb = (unsigned)__cvta_generic_to_shared(&ebar);  // entering columns (bulk path)
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(qb0) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(qb0 + 8) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(eb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // rows k >= p of a ragged last chunk are not rewritten: they meet zero slab columns, so
    // they must hold finite values -- zeros at start, earlier Qhat rows later
    for (int i = tid; i < 2 * KC * (cap + CHAIN_PAD); i += CNT) Qs[i] = 0.0;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    unsigned qpar = 0;  // bit b: parity of the next wait on Qhat buffer b
    unsigned epar = 0;  // parity of the next wait on ebar

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
    // (all loads of a thread are issued before its shared-memory stores: the entering columns of
    // a transition are ~16 independent HBM loads per thread, one latency instead of 16)
    auto load_cols = [&](int64_t c_lo, int64_t c_hi) {
        const int nc = (int)(c_hi - c_lo);
        if (nc <= 0) return;
        const int total = nc * h;
        constexpr int LB = 16;
        for (int base = 0; base < total; base += CNT * LB) {
            double v[LB];
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                const int idx = base + tid + q * CNT;
                v[q] = 0.0;
                if (idx < total) {
                    // right applies: rows fastest (a column is contiguous); left: columns fastest
                    const int s = M.left ? idx / nc : idx % h, c = M.left ? idx % nc : idx / h;
                    if (s < hs) v[q] = *gaddr(s, c_lo + c);
                }
            }
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                const int idx = base + tid + q * CNT;
                if (idx < total) {
                    const int s = M.left ? idx / nc : idx % h, c = M.left ? idx % nc : idx / h;
                    Xs[slot(c_lo + c) * ldh + s] = v[q];
                }
            }
        }
    };
    // the same movement issued as cp.async (no register staging; completes behind later work);
    // a handful of columns per call, so plain warp/lane loops (no division by runtime sizes)
    auto load_cols_async = [&](int64_t c_lo, int64_t c_hi) {
        const int nc = (int)(c_hi - c_lo);
        if (M.left) {  // columns fastest (contiguous in X), every lane busy
            const int total = nc * h;
            for (int idx = tid; idx < total; idx += CNT) {
                const int s = idx / nc, c = idx - s * nc;
                cp_async8(&Xs[slot(c_lo + c) * ldh + s], s < hs ? gaddr(s, c_lo + c) : M.X, s < hs);
            }
        } else {
            for (int c = warp; c < nc; c += CNT / 32)
                for (int s = lane; s < h; s += 32)
                    cp_async8(&Xs[slot(c_lo + c) * ldh + s], s < hs ? gaddr(s, c_lo + c) : M.X, s < hs);
        }
    };
    // right applies with 16-byte aligned slab columns: one bulk copy per entering column
    // (hs rows, contiguous in X), issued by warp 1's lanes, bytes counted on ebar
    auto load_cols_bulk = [&](int64_t c_lo, int64_t c_hi) {
        if (warp != 1) return;
        const int nc = (int)(c_hi - c_lo);
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;\n" ::"r"(eb), "r"((unsigned)(nc * hs * 8)) : "memory");
        }
        __syncwarp();
        for (int c = lane; c < nc; c += 32)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                         ::"r"((unsigned)__cvta_generic_to_shared(&Xs[slot(c_lo + c) * ldh])), "l"(gaddr(0, c_lo + c)),
                         "r"(hs * 8), "r"(eb) : "memory");
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
        CPROF_T(t0);
        const ChainWin w0 = P.win(0);
        load_cols(w0.o, (int64_t)w0.o + w0.p);
        zero_pad(w0.o, w0.p);
        CPROF_T(t1);
        CPROF_ADD(0, t0, t1);
    }
    for (int wi = 0; wi < P.nw; ++wi) {
        const ChainWin W = P.win(wi);
        const int p = W.p, pp = (p + 31) & ~31;
        const int64_t lo = W.lo[mi], hi = W.hi[mi];
        const bool active = (s0 < hi) && (s0 + hs > lo) && p > 0;
        const bool last = wi + 1 == P.nw;
        const int64_t a0 = W.o, a1 = (int64_t)W.o + W.p;
        int64_t b0 = a1, b1 = a1;
        if (!last) {
            const ChainWin N = P.win(wi + 1);
            b0 = N.o;
            b1 = (int64_t)N.o + N.p;
        }
        // Overlapped transition (forward chains, slab entirely inside the window's row range):
        // the leaving columns [a0, b0) are written to HBM straight from the accumulators, and
        // the entering columns are prefetched with cp.async into the ring slots of leaving
        // columns as soon as the k-loop has consumed them (slot(c) = slot(c - cap)), so the
        // slab's HBM traffic streams behind the DMMA work instead of stalling between windows.
        // Entering columns that overlap this window's zero padding [a1, a0 + pp) wait for the
        // transition (the padding must read as zeros until the window is done).
        const bool inside = active && s0 >= lo && s0 + hs <= hi;
        const bool early = inside && !last && b0 >= a0 && b1 >= a1 && b1 - b0 <= cap;
        const int direct = !inside ? 0 : last ? p : early ? (int)(b0 - a0 < p ? b0 - a0 : p) : 0;
        const bool ebulk = early && !M.left && (hs % 2) == 0 && (M.ld % 2) == 0 && (((uintptr_t)(M.X + s0)) & 15) == 0;
        const int64_t e_beg = a0 + pp > a1 ? a0 + pp : a1;  // first early-prefetchable entering column
        int64_t e_cur = e_beg;
        CPROF_T(tw0);
        // the ring's generic-proxy writes (epilogue, transition) before any bulk copy into it
        if (ebulk) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
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
            // k-chunk of Qhat (row-major, Qhat(k, c) at Qw[k p + c]) staged by cp.async into the
            // other buffer while this chunk computes; lanes run along c (coalesced, conflict-free)
            const int lcap = __ffs(cap) - 1;  // cap is a power of two
            const int per = (kc * cap) >> 9;  // staged elements per thread (<= 8; CNT = 512)
            const bool qbulk = (p % 2) == 0 && ((uintptr_t)W.Qw & 15) == 0;
            auto fetch = [&](int k0, int buf) {
                double *qd = Qs + (size_t)buf * kc * ldq;
                if (qbulk) {
                    // warp 0: lane 0 posts the byte count, then lane r copies Qhat row k0 + r
                    if (warp == 0) {
                        const int nr = p - k0 < kc ? p - k0 : kc;
                        const unsigned mb = qb0 + 8 * buf;
                        if (lane == 0) {
                            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                                         "r"((unsigned)(nr > 0 ? nr * p * 8 : 0)) : "memory");
                        }
                        __syncwarp();
                        if (lane < nr)
                            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                                         ::"r"((unsigned)__cvta_generic_to_shared(qd + lane * ldq)),
                                         "l"(W.Qw + (size_t)(k0 + lane) * p), "r"(p * 8), "r"(mb) : "memory");
                    }
                    return;
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    if (e >= per) break;
                    const int idx = tid + e * CNT;
                    const int kr = idx >> lcap, c = idx & (cap - 1);
                    const bool ok = c < p && k0 + kr < p;
                    cp_async8(qd + kr * ldq + c, ok ? W.Qw + (size_t)(k0 + kr) * p + c : W.Qw, ok);
                }
                cp_async_commit();
            };
            // wait for the chunk staged in `buf` (bulk: mbarrier phase; else cp.async groups)
            auto qwait = [&](int buf, bool pending_enter) {
                if (qbulk) {
                    const unsigned mb = qb0 + 8 * buf, par = (qpar >> buf) & 1u;
                    unsigned done = 0;
                    while (!done)
                        asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
                                     : "=r"(done) : "r"(mb), "r"(par) : "memory");
                    qpar ^= 1u << buf;
                }
                // entering-column groups: the newest may stay in flight
                if (pending_enter) cp_async_wait<1>(); else cp_async_wait<0>();
            };
            const int nk = pp / kc + (pp % kc ? 1 : 0);
            CPROF_T(tl0);
            fetch(0, 0);
            qwait(0, false);
            __syncthreads();
            for (int kt = 0; kt < nk; ++kt) {
                const int buf = kt & 1;
                if (kt + 1 < nk) fetch((kt + 1) * kc, buf ^ 1);
                if (early) {  // entering columns whose ring slots the k-loop has released
                    int64_t lim = a0 + (int64_t)kt * kc + cap;
                    if (lim > b1) lim = b1;
                    if (lim > e_cur) {
                        if (ebulk) load_cols_bulk(e_cur, lim);
                        else load_cols_async(e_cur, lim);
                        e_cur = lim;
                    }
                    if (!ebulk) cp_async_commit();
                }
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
                // the next Qhat chunk has landed; this chunk's entering columns may still fly
                const bool ecp = early && !ebulk;
                if (kt + 1 < nk) qwait(buf ^ 1, ecp);
                else if (ecp) cp_async_wait<1>();
                CPROF_T(tb0);
                __syncthreads();
                CPROF_T(tb1);
                CPROF_ADD(4, tb0, tb1);
            }
            CPROF_T(tl1);
            CPROF_ADD(1, tl0, tl1);
            if (ebulk && tid == 32)  // all entering copies of this window are issued
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(eb) : "memory");
            // epilogue: slab(s, o + c) <- acc for s in [lo, hi), c < p; the first `direct`
            // columns leave the chain here and go straight to HBM
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
                            if (c < p && sg >= lo && sg < hi && s < hs) {
                                if (c < direct)
                                    *gaddr(s, (int64_t)W.o + c) = acc[a][b][hh];
                                else
                                    Xs[slot((int64_t)W.o + c) * ldh + s] = acc[a][b][hh];
                            }
                        }
            }
        }
        cp_async_wait<0>();
        if (ebulk) {  // (ebulk implies active: the arrival above happened)
            unsigned done = 0;
            while (!done)
                asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
                             : "=r"(done) : "r"(eb), "r"(epar) : "memory");
            epar ^= 1u;
        }
        __syncthreads();
        CPROF_T(tt0);
        CPROF_ADD(2, tw0, tt0);
        // transition: flush columns leaving the chain, load columns entering it
        if (!last) {
            // leaving: [a0, a1) \ [b0, b1); entering: [b0, b1) \ [a0, a1)  (monotone chains)
            store_cols(a0 + direct, a1 < b0 ? a1 : b0);
            store_cols(a0 > b1 ? a0 : b1, a1);
            __syncthreads();
            if (early) {
                load_cols(a1, e_beg < b1 ? e_beg : b1);  // entering columns under the zero padding
                load_cols(e_cur, b1);
            } else {
                load_cols(b0, b1 < a0 ? b1 : a0);
                load_cols(b0 > a1 ? b0 : a1, b1);
            }
            __syncthreads();
            const ChainWin N = P.win(wi + 1);
            zero_pad(N.o, N.p);
        } else {
            store_cols(a0 + direct, a1);
        }
        CPROF_T(tt1);
        CPROF_ADD(3, tt0, tt1);
    }
    }  // task loop
}

// ---------------------------------------------------------------------------
// Band apply from the compact-WY factors (ht_band_wy): Qhat = Q_0 Q_1 ... with one
// 32-column panel block Q_b = I - V_b T_b V_b^T per factorization panel (only the
// diagonal 32x32 blocks of T are used), so that on the slab view S (8 slabs per CTA)
//   for b = 0, 1, ...:   Y = S V_b,  Y2 = Y T_b,  S -= Y2 V_b^T        (DMMA m8n8k4)
// With ident = 1 the slabs start as rows of the identity: the CTA rows of Qhat itself
// (the explicit window transform the chained applies stream, ht_chain_apply).
struct BandDesc {
    double *X;
    int64_t ld;
    int left, ident;
    int64_t s0;
    int cnt;
    int64_t o;
    int p, q;
    const double *V;
    int64_t ldv;
    const double *T;
    int64_t ldt;
};
constexpr int BPW = 32;  // panel width of the factorization (ht_factor.cu PBW)


// double-buffered V_b/T_b staging fits in shared memory for windows of up to 256 rows
__host__ __device__ __forceinline__ bool band_double_buffer(int p8) { return p8 <= 256; }

// smem layout (doubles): Ss [8][lds] | Yp [2][8][LDY] | Y2 [8][LDY] | Vb [nbuf][BPW][ldr] | Tb [nbuf][BPW][LDY]
// (ld == 4 mod 16 everywhere: conflict-free 64-bit fragments)
__device__ unsigned long long *g_bprof = nullptr;  // development: per-phase clock64 sums (thread 0, CTA 0)

__global__ void __launch_bounds__(256) band_wy_kernel(const BandDesc *descs, const __grid_constant__ BandDesc one)
{
    unsigned long long *bprof = (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) ? g_bprof : nullptr;
    long long bck = bprof ? clock64() : 0;
    auto BPROF = [&](int ph) {
        if (bprof) {
            const long long t = clock64();
            bprof[ph] += (unsigned long long)(t - bck);
            bck = t;
        }
    };
    extern __shared__ __align__(16) double bsm[];
    const BandDesc A = descs ? descs[blockIdx.y] : one;  // by value: registers, not generic loads
    if (8 * (int)blockIdx.x >= A.cnt) return;
    const int p = A.p, q = A.q;
    const int p8 = (p + 7) & ~7;
    const int lds = ((p8 + 31) & ~31) + 4;
    const int ldr = ((p8 + 15) & ~15) + 4;  // V_b block, column-major
    constexpr int LDY = BPW + 4;
    double *Ss = bsm;
    double *Yp = Ss + 8 * lds;
    double *Y2 = Yp + 16 * LDY;
    double *Vb = Y2 + 8 * LDY;             // [2][BPW][ldr]
    double *Tb = Vb + (band_double_buffer(p8) ? 2 : 1) * BPW * ldr;  // [nbuf][BPW][LDY]  T_b(k, n) at Tb[n * LDY + k]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
    const int64_t sb = A.s0 + 8 * (int64_t)blockIdx.x;
    const int ns = min(8, A.cnt - 8 * (int)blockIdx.x);
    auto xp = [&](int s, int c) -> double * {
        return A.left ? A.X + (sb + s) * A.ld + A.o + c : A.X + (A.o + c) * A.ld + sb + s;
    };
    const int nblk = (q + BPW - 1) / BPW;
    const bool dbl = band_double_buffer(p8);  // windows of <= 256 rows: prefetch the next block
    // Bulk-copy path (copy engine, one cp.async.bulk per column, completion on an mbarrier):
    // needs 16-byte aligned columns of whole 8-row multiples; else 8-byte cp.async.
#ifdef BAND_NOBULK
    const bool bulk = false;
#else
    const bool bulk = (p % 8) == 0 && (A.ldv % 2) == 0 && (A.ldt % 2) == 0 && ((uintptr_t)A.V & 15) == 0 &&
                      ((uintptr_t)A.T & 15) == 0;
#endif
    __shared__ __align__(8) unsigned long long mbar[2];
    const unsigned mb0 = (unsigned)__cvta_generic_to_shared(&mbar[0]);
    if (bulk && tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb0) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb0 + 8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    int uses[2] = {0, 0};  // completed phases per buffer (parity of the next wait)
    // stage V_b (p x 32, rows contiguous) and T_b (32 x 32, diagonal block) of block b
    auto stage = [&](int b) {
        const int j0 = b * BPW, nc = min(BPW, q - j0), bf = dbl ? (b & 1) : 0;
        double *vb = Vb + bf * BPW * ldr, *tb = Tb + bf * BPW * LDY;
        if (bulk) {
            for (int j = nc; j < BPW; ++j) {  // ragged block: columns beyond nc are zeros
                for (int r = tid; r < p8; r += 256) vb[j * ldr + r] = 0.0;
                if (tid < BPW) tb[j * LDY + tid] = 0.0;
            }
            if (warp == 0) {  // lane 0 posts the byte count; lane j copies column j of V_b and T_b
                const unsigned mb = mb0 + 8 * bf;
                const unsigned bytes = (unsigned)(nc * (p + BPW) * 8);
                if (lane == 0) {
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
                }
                __syncwarp();
                for (int j = lane; j < nc; j += 32) {
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                                 ::"r"((unsigned)__cvta_generic_to_shared(vb + j * ldr)), "l"(A.V + (int64_t)(j0 + j) * A.ldv),
                                 "r"(p * 8), "r"(mb) : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                                 ::"r"((unsigned)__cvta_generic_to_shared(tb + j * LDY)), "l"(A.T + (int64_t)(j0 + j) * A.ldt + j0),
                                 "r"(BPW * 8), "r"(mb) : "memory");
                }
            }
            return;
        }
        for (int j = 0; j < BPW; ++j)  // (no division by the runtime row count)
            for (int r = tid; r < p8; r += 256) {
                const bool ok = j < nc && r < p;
                cp_async8(vb + j * ldr + r, ok ? A.V + (int64_t)(j0 + j) * A.ldv + r : A.V, ok);
            }
        for (int i = tid; i < BPW * BPW; i += 256) {
            const int n = i / BPW, k = i % BPW;
            const bool ok = n < nc && k <= n;  // T_b upper: lower part read as 0
            cp_async8(tb + n * LDY + k, ok ? A.T + (int64_t)(j0 + n) * A.ldt + j0 + k : A.T, ok);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    // wait for block b's buffer (bulk: mbarrier phase; else cp.async groups, see the loop)
    auto bulk_wait = [&](int b) {
        const int bf = dbl ? (b & 1) : 0;
        const unsigned mb = mb0 + 8 * bf, par = (unsigned)(uses[bf] & 1);
        unsigned done = 0;
        while (!done)
            asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
                         : "=r"(done) : "r"(mb), "r"(par) : "memory");
        ++uses[bf];
    };
    if (dbl) stage(0);
    // the slab (8 x p): every thread issues all its loads before its shared-memory stores
    // (p8 <= 512: at most 16 elements per thread)
    {
        constexpr int ME = 16;
        double t[ME];
#pragma unroll
        for (int e = 0; e < ME; ++e) {
            const int i = tid + e * 256;
            t[e] = 0.0;
            if (i < 8 * p8) {
                int ss, c;
                if (A.left) { ss = i / p8; c = i - ss * p8; }  // contiguous along c
                else { c = i >> 3; ss = i & 7; }                // contiguous along s
                if (ss < ns && c < p) t[e] = A.ident ? ((sb + ss == A.o + c) ? 1.0 : 0.0) : *xp(ss, c);
            }
        }
#pragma unroll
        for (int e = 0; e < ME; ++e) {
            const int i = tid + e * 256;
            if (i < 8 * p8) {
                int ss, c;
                if (A.left) { ss = i / p8; c = i - ss * p8; }
                else { c = i >> 3; ss = i & 7; }
                Ss[ss * lds + c] = t[e];
            }
        }
    }
    for (int b = 0; b < nblk; ++b) {
        if (b > 0) __syncthreads();  // pass b-1 has finished reading the buffer staged next
        if (!dbl) {
            stage(b);
            if (bulk) bulk_wait(b);
            else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        } else if (b + 1 < nblk) {
            stage(b + 1);
            if (bulk) bulk_wait(b);
            else asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            if (bulk) bulk_wait(b);
            else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        BPROF(b == 0 ? 4 : 0);  // staging wait (4: first block, incl. the slab load)
        const int bf = dbl ? (b & 1) : 0;
        const double *vb = Vb + bf * BPW * ldr, *tb = Tb + bf * BPW * LDY;
        // Y = S V_b: warp = (n-tile, K half)
        {
            const int nt = warp & 3, kh = warp >> 2;
            const int half = (p8 / 2) & ~3;
            const int kb = kh ? half : 0, ke = kh ? p8 : half;
            const double *bcol = vb + (8 * nt + g) * ldr + t4;
            const double *arow = Ss + g * lds + t4;
            double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
            int k = kb;
            for (; k + 8 <= ke; k += 8) {
                dmma(c0, c1, arow[k], bcol[k]);
                dmma(d0, d1, arow[k + 4], bcol[k + 4]);
            }
            if (k < ke) dmma(c0, c1, arow[k], bcol[k]);
            Yp[(kh * 8 + g) * LDY + 8 * nt + 2 * t4] = c0 + d0;
            Yp[(kh * 8 + g) * LDY + 8 * nt + 2 * t4 + 1] = c1 + d1;
        }
        __syncthreads();
        BPROF(1);  // S V_b
        // Y2 = Y T_b: warps 0..3, one n-tile each
        if (warp < 4) {
            const int nt = warp;
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int k = 0; k < BPW; k += 4) {
                if (k < 8 * nt + 8) {
                    const int kr = k + t4;
                    const double av = Yp[g * LDY + kr] + Yp[(8 + g) * LDY + kr];
                    dmma(c0, c1, av, tb[(8 * nt + g) * LDY + kr]);
                }
            }
            Y2[g * LDY + 8 * nt + 2 * t4] = c0;
            Y2[g * LDY + 8 * nt + 2 * t4 + 1] = c1;
        }
        __syncthreads();
        BPROF(2);  // Y T_b
        // S -= Y2 V_b^T: B fragments V^T(k, n) = V_b(n, k)
        for (int nt = warp; nt < p8 / 8; nt += 8) {
            const int n = 8 * nt + g;
            double c0 = Ss[g * lds + 8 * nt + 2 * t4], c1 = Ss[g * lds + 8 * nt + 2 * t4 + 1];
#pragma unroll
            for (int u = 0; u < 8; ++u) dmma(c0, c1, -Y2[g * LDY + 4 * u + t4], vb[(4 * u + t4) * ldr + n]);
            Ss[g * lds + 8 * nt + 2 * t4] = c0;
            Ss[g * lds + 8 * nt + 2 * t4 + 1] = c1;
        }
        BPROF(3);  // S -= Y2 V_b^T (own warp)
    }
    __syncthreads();
    if (A.left) {
        for (int s = 0; s < ns; ++s)
            for (int c = tid; c < p; c += 256) *xp(s, c) = Ss[s * lds + c];
    } else {
        for (int i = tid; i < 8 * p8; i += 256) {
            const int c = i >> 3, s = i & 7;
            if (s < ns && c < p) *xp(s, c) = Ss[s * lds + c];
        }
    }
}

size_t band_smem(int pmax)
{
    const int p8 = (pmax + 7) & ~7;
    const int lds = ((p8 + 31) & ~31) + 4, ldr = ((p8 + 15) & ~15) + 4, ldy = BPW + 4;
    const int nbuf = band_double_buffer(p8) ? 2 : 1;
    return (size_t)(8 * lds + 24 * ldy + nbuf * BPW * ldr + nbuf * BPW * ldy) * sizeof(double);
}
int band_init()
{
    static std::mutex mu;
    static unsigned long long done = 0;
    return ht_once_per_device(mu, done, [] {
        HT_CUDA_TRY(cudaFuncSetAttribute(band_wy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        return 0;
    });
}

}  // namespace

int ht_band_wy(cudaStream_t st, double *X, int64_t ld, int left, int64_t s0, int64_t cnt, int64_t o, int p, int q,
               const double *V, int64_t ldv, const double *T, int64_t ldt)
{
    if (cnt <= 0 || p <= 0 || q <= 0) return 0;
    if (band_init()) return 2;
    BandDesc A{X, ld, left, 0, s0, (int)cnt, o, p, q, V, ldv, T, ldt};
    band_wy_kernel<<<(unsigned)((cnt + 7) / 8), 256, band_smem(p), st>>>(nullptr, A);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

// Explicit Qhat (p x p, row-major: Qhat(k, c) at [k p + c]) of nw windows: window i has Qw[i], V[i] (p x q, ld p), T[i]
// (diagonal 32x32 blocks, ld q).  d_descs: device scratch for nw descriptors, h_descs pinned.
int ht_form_qhat(cudaStream_t st, int nw, double *const *Qw, const int *p, const int *q, const double *const *V,
                 const double *const *T, void *d_descs, void *h_descs)
{
    if (nw <= 0) return 0;
    if (band_init()) return 2;
    BandDesc *hd = reinterpret_cast<BandDesc *>(h_descs);
    int pmax = 0;
    for (int i = 0; i < nw; ++i) {
        hd[i] = BandDesc{Qw[i], p[i], 1, 1, 0, p[i], 0, p[i], q[i], V[i], p[i], T[i], q[i]};  // row-major Qhat
        pmax = std::max(pmax, p[i]);
    }
    const dim3 grid((unsigned)((pmax + 7) / 8), (unsigned)nw);
    if (nw == 1) {  // by value: no host-to-device copy ahead of the kernel
        band_wy_kernel<<<grid, 256, band_smem(pmax), st>>>(nullptr, hd[0]);
    } else {
        HT_CUDA_TRY(cudaMemcpyAsync(d_descs, hd, nw * sizeof(BandDesc), cudaMemcpyHostToDevice, st));
        band_wy_kernel<<<grid, 256, band_smem(pmax), st>>>(reinterpret_cast<const BandDesc *>(d_descs), BandDesc{});
    }
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}
size_t ht_band_desc_size() { return sizeof(BandDesc); }

// Apply a chain of explicit window transforms to up to 3 matrices (one launch).
// d_wins: device array of nw windows (application order, monotone offsets).
int ht_chain_apply(cudaStream_t st, const ChainMat *mats, int nm, const ChainWin *d_wins, int nw, int pmax, int maxgrid,
                   const ChainWin *h_wins)
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
    if (h_wins && nw <= 4) {  // by value: d_wins is not read
        for (int i = 0; i < nw; ++i) P.inl[i] = h_wins[i];
        P.wins = nullptr;
    }
    int64_t nblk = 0;
    for (int i = 0; i < nm; ++i)
        if (mats[i].s_end > mats[i].s_begin) nblk += (mats[i].s_end - mats[i].s_begin + P.h - 1) / P.h;
    if (nblk == 0) return 0;
    const int kc = P.cap <= 256 ? 16 : 8;
    const size_t smem = ((size_t)P.cap * (P.h + CHAIN_PAD) + 2 * (size_t)kc * (P.cap + CHAIN_PAD)) * sizeof(double);
    static std::mutex mu;
    static unsigned long long done = 0;
    const int rc = ht_once_per_device(mu, done, [] {
        const int mx = (int)(SLAB_ELEMS + CHAIN_PAD * 512 + 2 * 16 * (256 + CHAIN_PAD)) * 8;
        HT_CUDA_TRY(cudaFuncSetAttribute(chain_apply_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        HT_CUDA_TRY(cudaFuncSetAttribute(chain_apply_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        return 0;
    });
    if (rc) return rc;
    const unsigned grid = (unsigned)(maxgrid > 0 && nblk > maxgrid ? maxgrid : nblk);
    if (kc == 16) chain_apply_kernel<16><<<grid, CNT, smem, st>>>(P);
    else chain_apply_kernel<8><<<grid, CNT, smem, st>>>(P);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

#ifdef CHAIN_PROF
extern "C" __attribute__((visibility("default"))) int ht_chain_prof_read(unsigned long long *out, int reset)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_chain_prof, sizeof(g_chain_prof));
    if (reset) {
        static unsigned long long z[256][8];
        cudaMemcpyToSymbol(g_chain_prof, z, sizeof(z));
    }
    return 0;
}
#endif
