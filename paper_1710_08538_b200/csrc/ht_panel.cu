// ht_panel.cu -- persistent cooperative panel kernel of HouseHT (sec. 3.2).
//
// One launch reduces one panel: columns j = s, s+1, ... of A (0-based s0) until
// kmax reflector pairs are accumulated or iterative refinement fails.  Per column
// (paper notation, sec. 3.2.2, Algorithm 1):
//   P1  a = A(s+1:n, j) - Y V(j,:)^T;  a -= U S^T U^T a           (sec. 3.2.2a)
//   P2  (u, beta) = House(a(j+1:n));  S <- [S, -beta S U^T u; 0, beta]  (sec. 3.2.2b)
//   P3  c~ = (I - U S U^T)[0; e1];  y~ = B^{-1} c~;  y = (I - V T V^T)^T y~;  x = y(j+1:n)
//                                                                   (sec. 3.2.2c steps 1-4, P:477-483;
//                                                                    k = 0: sec. 3.2.1)
//   P4  w = (I - V T V^T)[0; x];  w = B w;  w = (I - U S^T U^T) w;  r = e1 - w(j+1:n)
//       accept if ||r||/||x|| <= 2u||B||_F, else <= 10 IR corrections (sec. 2.3)
//       failure: restore column j of A, drop u, end the panel (Algorithm 1)
//   P5  (v, gamma) = House(x);  T <- [T, -gamma T V^T v; 0, gamma];
//       y = gamma (A v - Y V^T v)                                   (sec. 3.2.2d)
// Rows 1:s of Y and of the panel columns are deferred (Remark 2).
//
// B200 design: one CTA per SM, grid-wide barriers between
// phases, no host round trip per column (the IR loop and the fallback are
// decided on the device).  The triangular solve is a flag-chained block
// back-substitution over 128-row blocks: each block is solved with its
// pre-inverted diagonal block (held in shared memory for the solve), or, when
// the block is unsafe to invert (tiny pivots, config 4), by an overflow-safe
// sequential back-substitution; every block carries a power-of-two exponent
// (reading R-Z8), so y~ never overflows.  HBM-bound sweeps (B w, A v, the
// off-diagonal solve tiles) are issued with many independent loads per thread.
#include <cooperative_groups.h>
#include <vector>
#include <algorithm>
#include <mutex>
#include <cstdlib>
#include "ht_common.cuh"
#include "ht_internal.h"

namespace cg = cooperative_groups;

namespace {

constexpr int PNT = 512;   // threads per CTA
constexpr int NWP = PNT / 32;
constexpr int TB = 128;    // triangular-solve block size
constexpr int T4 = 256;    // trsv4: solve block rows (4-CTA clusters, 64-column slices)
constexpr int C4 = 4;
constexpr int NBMAX = 256; // max panel width supported
constexpr int RBMAX = 256; // max own rows per CTA (uniform slabs)
constexpr double BIG = 0x1p256;
// Per-CTA shared-memory copies of S and T (packed upper triangles, column c at c(c+1)/2) for
// panels of width <= STC_NB solved by trsv4: every column's small mat-vecs with S and T then
// read shared memory instead of L2 (each was a few dependent L2 round trips per column).  They
// sit above the staging areas of the phases (<= OFF_ST doubles); trsv_blocked's 128 x 128 tile
// overlaps them, so the 128-row solve keeps S and T in global memory.
constexpr int STC_NB = 128, STC_SZ = STC_NB * (STC_NB + 1) / 2, OFF_ST = 4608;
constexpr int DYN_DOUBLES = (TB * TB + 8 * TB) > (OFF_ST + 2 * STC_SZ) ? (TB * TB + 8 * TB) : (OFF_ST + 2 * STC_SZ);

struct __align__(16) PanelSmem {
    double sv1[NBMAX + 2];
    double sv2[NBMAX + 2];
    double sv3[NBMAX + 2];
    double snew[NBMAX + 2];  // new column of S
    double svx[NBMAX + 2];   // V^T x of the current solve (kept for P5's V^T v)
    double vloc[RBMAX];      // own-row vector cache
    double red[32];
    double pt[16];     // HT_PROFILE: per-phase seconds of CTA 0 (flushed to a.ptime at the end)
    double rhs[TB];
    double cbv[TB];
    double yrecv[TB];  // y~_{b+1} handed over by the partner CTA of the cluster (DSMEM)
    unsigned long long mbar;  // completes when the partner has written yrecv/erecv (TB remote arrivals)
    unsigned long long mbar4; // trsv4, cluster rank 0: the 3 partial-sum messages of a block have landed
    int ival[4];
    int es4[4];        // trsv4r: exponents of the four 64-row slices of a fetched block
    int erecv;
};

// Shared memory of the panel kernel, declared at namespace scope so that every access
// compiles to LDS/STS (a pointer kept in a struct would decay to generic loads).
__shared__ PanelSmem g_sm;
extern __shared__ __align__(16) double g_dyn[];

__device__ __forceinline__ unsigned long long gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
struct Ctx {
    const PanelArgs &a;
    unsigned mbpar = 0;  // parity of the next phase of g_sm.mbar (lo CTAs of the solve clusters)
    unsigned mb4par = 0; // parity of the next phase of g_sm.mbar4 (trsv4, cluster rank 0)
    int tbs;             // rows per solve block: 128 (trsv_blocked) or 256 (trsv4)
    int G, bid, tid, lane, warp;
    int64_t n, p0, M, rb0, rb1;
    int nr;
    double *part[2];
    int ph;
    __device__ Ctx(const PanelArgs &aa) : a(aa)
    {
        G = gridDim.x;
        bid = blockIdx.x;
        tid = threadIdx.x;
        lane = tid & 31;
        warp = tid >> 5;
        n = a.n;
        p0 = a.s0 + 1;
        M = n - p0;
        int64_t RB = (M + G - 1) / G;
        rb0 = p0 + (int64_t)bid * RB;
        if (rb0 > n) rb0 = n;
        rb1 = rb0 + RB < n ? rb0 + RB : n;
        nr = (int)(rb1 - rb0);
        part[0] = a.part;
        part[1] = a.part + (size_t)G * a.pw;
        ph = 0;
        tbs = a.solve4 == 2 ? 64 : (a.solve4 ? 256 : TB);
    }
    // partials are stored index-major: (CTA b, index c) at part[ph][c * G + b], so a gather
    // reads contiguous CTA runs
    __device__ void putpart(int c, double v) { part[ph & 1][(size_t)c * G + bid] = v; }
    __device__ double *curpart() { return part[ph & 1]; }

    // The helpers below are latency-bound (a CTA owns ~n/148 rows, k <= nb columns): each
    // one issues ALL loads of a batch before the first use (one memory round trip per
    // batch instead of one per loop iteration), with fixed summation orders (deterministic).
    //
    // out[c] = sum over own rows of X(r,c) * vloc[r - rb0], c < ncols -> partial (off + c).
    // Warps take 8 columns, lanes 2 x 32 rows per batch; lane partials through shared staging.
    __device__ void coltdot(const double *X, int64_t ldx, int ncols, int off)
    {
        double *stg = g_dyn;  // ncols x 33
        constexpr int CU = 8;
        for (int cb = warp * CU; cb < ncols; cb += NWP * CU) {
            double acc[CU];
#pragma unroll
            for (int u = 0; u < CU; ++u) acc[u] = 0.0;
            for (int r0 = 0; r0 < nr; r0 += 64) {
                double xv[2][CU], vv[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int rl = r0 + 32 * h + lane;
                    const bool ok = rl < nr;
                    vv[h] = ok ? g_sm.vloc[rl] : 0.0;
#pragma unroll
                    for (int u = 0; u < CU; ++u)
                        xv[h][u] = (ok && cb + u < ncols) ? X[(size_t)(cb + u) * ldx + rb0 + rl] : 0.0;
                }
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int u = 0; u < CU; ++u) acc[u] = fma(xv[h][u], vv[h], acc[u]);
            }
#pragma unroll
            for (int u = 0; u < CU; ++u)
                if (cb + u < ncols) stg[(cb + u) * 33 + lane] = acc[u];
        }
        __syncthreads();
        for (int c = tid; c < ncols; c += PNT) {
            double t = 0.0;
#pragma unroll 8
            for (int l = 0; l < 32; ++l) t += stg[c * 33 + l];
            putpart(off + c, t);
        }
        __syncthreads();
    }
    // returns (in g_dyn[rl]) sum_c X(rb0+rl, c) * coef[c] for own rows; warps split the
    // columns (c = warp + NWP t), lanes take 2 x 32 rows; 8 columns x 2 rows of loads in flight.
    __device__ void rowgemv(const double *X, int64_t ldx, int ncols, const double *coef)
    {
        double *stg = g_dyn + TB * 4;  // NWP x RBMAX
        constexpr int CU = 8;
        for (int rc = 0; rc < nr; rc += 64) {
            double s[2] = {0.0, 0.0};
            for (int c0 = warp; c0 < ncols; c0 += NWP * CU) {
                double xs[2][CU];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int rl = rc + 32 * h + lane;
#pragma unroll
                    for (int t = 0; t < CU; ++t) {
                        const int c = c0 + NWP * t;
                        xs[h][t] = (rl < nr && c < ncols) ? X[(size_t)c * ldx + rb0 + rl] : 0.0;
                    }
                }
#pragma unroll
                for (int t = 0; t < CU; ++t) {
                    const int c = c0 + NWP * t;
                    const double cf = c < ncols ? coef[c] : 0.0;
#pragma unroll
                    for (int h = 0; h < 2; ++h) s[h] = fma(xs[h][t], cf, s[h]);
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int rl = rc + 32 * h + lane;
                if (rl < RBMAX) stg[warp * RBMAX + rl] = s[h];
            }
        }
        __syncthreads();
        for (int rl = tid; rl < nr; rl += PNT) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < NWP; ++w) t += stg[w * RBMAX + rl];
            g_dyn[rl] = t;
        }
        __syncthreads();
    }
    // after a grid sync: dst[c] = sum_b part[b][off + c]  (fixed order: deterministic).
    // Warps take 4 columns at a time, lanes split the CTA partials; all loads of a lane
    // are issued before the sums (the partials live in L2: latency, not bandwidth, bound).
    __device__ void gather(double *dst, int ncols, int off)
    {
        const double *pp = curpart() + (size_t)off * G;
        constexpr int MAXB = 8;  // G <= 256 CTAs
        constexpr int CU = 4;
        for (int c0 = warp * CU; c0 < ncols; c0 += NWP * CU) {
            double v[CU][MAXB];
#pragma unroll
            for (int u = 0; u < CU; ++u)
#pragma unroll
                for (int q = 0; q < MAXB; ++q) {
                    const int b = lane + 32 * q;
                    v[u][q] = (b < G && c0 + u < ncols) ? __ldcg(pp + (size_t)(c0 + u) * G + b) : 0.0;
                }
#pragma unroll
            for (int u = 0; u < CU; ++u) {
                double t = 0.0;
#pragma unroll
                for (int q = 0; q < MAXB; ++q) t += v[u][q];
                t = warp_sum(t);
                if (lane == 0 && c0 + u < ncols) dst[c0 + u] = t;
            }
        }
        __syncthreads();
    }
    // Upper-triangular k x k mat-vec with the matrix in global memory (L2):
    //   !TR: out[i] = sum_{c >= i} M(i,c) v[c];   TR: out[c] = sum_{i <= c} M(i,c) v[i]
    // scale multiplies the result.  All warps; per-lane partials staged in smem.
    template <bool TR, class MF>
    __device__ void trimv(MF Mget, int m, const double *v, double *out, double scale = 1.0)
    {
        if (!TR) {
            // out[i] = sum_{c >= i} M(i, c) v[c], column-oriented: warps over columns, lanes over
            // rows, so every load is a contiguous column segment and all of a lane's loads are
            // independent; the 16 warp partials are added in a fixed order (deterministic)
            double *stg = g_dyn;  // NWP x m
            double acc[NBMAX / 32];
#pragma unroll
            for (int q = 0; q < NBMAX / 32; ++q) acc[q] = 0.0;
            for (int c = warp; c < m; c += NWP) {
                const double vc = v[c];
#pragma unroll
                for (int q = 0; q < NBMAX / 32; ++q) {
                    const int i = lane + 32 * q;
                    if (i <= c) acc[q] = fma(Mget(i, c), vc, acc[q]);
                }
            }
#pragma unroll
            for (int q = 0; q < NBMAX / 32; ++q) {
                const int i = lane + 32 * q;
                if (i < m) stg[warp * m + i] = acc[q];
            }
            __syncthreads();
            for (int o = tid; o < m; o += PNT) {
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < NWP; ++w) t += stg[w * m + o];
                out[o] = scale * t;
            }
            __syncthreads();
            return;
        }
        double *stg = g_dyn;  // m x 33
#pragma unroll 2
        for (int o = warp; o < m; o += NWP) {
            double s = 0.0;
            if (!TR) {
                for (int c = o + lane; c < m; c += 32) s += Mget(o, c) * v[c];
            } else {
                for (int i = lane; i <= o; i += 32) s += Mget(i, o) * v[i];
            }
            stg[o * 33 + lane] = s;
        }
        __syncthreads();
        for (int o = tid; o < m; o += PNT) {
            double t = 0.0;
#pragma unroll 8
            for (int l = 0; l < 32; ++l) t += stg[o * 33 + l];
            out[o] = scale * t;
        }
        __syncthreads();
    }
    // trimv with M in shared memory, packed upper triangle (column c at c(c+1)/2): four threads
    // per output (m <= 128 outputs per pass) each sum a strided quarter, combined by a fixed
    // xor-shuffle tree (deterministic).  ~300 cycles instead of several L2 round trips.
    template <bool TR>
    __device__ void trimv_sm(const double *Mp, int m, const double *v, double *out, double scale = 1.0)
    {
        constexpr int TPO = 4;
        for (int o0 = 0; o0 < m; o0 += PNT / TPO) {
            const int o = o0 + tid / TPO, part = tid % TPO;
            double s0 = 0.0, s1 = 0.0;
            if (o < m) {
                if (TR) {  // out[o] = sum_{i <= o} M(i, o) v[i]
                    const double *col = Mp + o * (o + 1) / 2;
                    int i = part;
                    for (; i + TPO <= o; i += 2 * TPO) {
                        s0 = fma(col[i], v[i], s0);
                        s1 = fma(col[i + TPO], v[i + TPO], s1);
                    }
                    if (i <= o) s0 = fma(col[i], v[i], s0);
                } else {   // out[o] = sum_{o <= c < m} M(o, c) v[c]
                    int c = o + part;
                    for (; c + TPO < m; c += 2 * TPO) {
                        s0 = fma(Mp[c * (c + 1) / 2 + o], v[c], s0);
                        s1 = fma(Mp[(c + TPO) * (c + TPO + 1) / 2 + o], v[c + TPO], s1);
                    }
                    if (c < m) s0 = fma(Mp[c * (c + 1) / 2 + o], v[c], s0);
                }
            }
            double sum = s0 + s1;
            sum += __shfl_xor_sync(0xffffffffu, sum, 1);
            sum += __shfl_xor_sync(0xffffffffu, sum, 2);
            if (part == 0 && o < m) out[o] = scale * sum;
        }
        __syncthreads();
    }
    __device__ double block_reduce_to_part(double v, int off)
    {
        double s = block_sum(v, g_sm.red);
        if (tid == 0) putpart(off, s);
        return s;
    }
};

// ---------------------------------------------------------------------------
// Flag-chained block back-substitution (see trsv_blocked below).
// 2^e as a double for |e| <= 1000 (exact; bit construction instead of ldexp's special cases)
__device__ __forceinline__ double pow2i(int e)
{
    e = e < -1000 ? -1000 : (e > 1000 ? 1000 : e);
    return __longlong_as_double((long long)(e + 1023) << 52);
}
// Flag-in-data ("LL") publication of the solve blocks: every double of y~_b travels as
// two 8-byte words (epoch << 32 | 32-bit half), and the block exponent as one more word.
// 8-byte accesses are single-copy atomic, so a reader that sees the current epoch in a
// word has that word's payload: no separate flag, no release fence, one L2 round trip.
__device__ __forceinline__ unsigned long long ld_volatile64(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile64(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Solve hand-over inside a 2-CTA cluster: the hi CTA stores y~_b into the lo CTA's shared
// memory and every storing thread arrives (release, cluster scope) on the lo CTA's mbarrier;
// the lo CTA waits on the phase (acquire).  One-way, ~DSMEM latency: no cluster barrier.
__device__ __forceinline__ void mbar_remote_arrive(unsigned long long *local_bar, unsigned rank)
{
    const unsigned la = (unsigned)__cvta_generic_to_shared(local_bar);
    unsigned ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned long long *bar, unsigned parity)
{
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done)
        asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, P;\n}\n"
                     : "=r"(done) : "r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void ll_put(unsigned long long *w, double x, unsigned epoch)
{
    // one 16-byte store; each 8-byte word is single-copy atomic and carries the epoch itself
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const unsigned long long e = (unsigned long long)epoch << 32;
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(w), "l"(e | (b & 0xffffffffull)), "l"(e | (b >> 32))
                 : "memory");
}
__device__ __forceinline__ double ll_get(const unsigned long long *w, unsigned epoch)
{
    unsigned long long lo, hi;
    while (true) {
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(w) : "memory");
        if ((unsigned)(lo >> 32) == epoch && (unsigned)(hi >> 32) == epoch) break;
#ifndef HT_POLL_NS
#define HT_POLL_NS 64
#endif
        if (HT_POLL_NS > 0) __nanosleep(HT_POLL_NS);  // back off: the pollers of all waiting CTAs share L2 with the chain
    }
    return __longlong_as_double((long long)((hi << 32) | (lo & 0xffffffffull)));
}
__device__ __forceinline__ int ll_get_exp(const unsigned long long *w, unsigned epoch)
{
    unsigned long long v;
    while (true) {
        v = ld_volatile64(w);
        if ((unsigned)(v >> 32) == epoch) break;
        if (HT_POLL_NS > 0) __nanosleep(HT_POLL_NS);
    }
    return (int)(unsigned)(v & 0xffffffffull);
}
// Packed layout of the pre-scaled block rows Bt = Dinv_b B(block b, blocks > b) (formed per
// panel by ht_panel_run): block row b is a TB x W_b column-major panel with ld TB (= ldbt),
// W_b = M - (b+1) TB columns, stored after the block rows above it -- so every TB x TB tile
// (b, c) is one contiguous 128 KB range (DRAM-friendly streaming in the solve).
__host__ __device__ __forceinline__ int64_t bt_row_offset(int64_t M, int64_t b)
{
    return (int64_t)TB * (b * M - (int64_t)TB * b * (b + 1) / 2);
}
// Stage block cb of the solution (w values) into ys[] and return its exponent (all threads).
__device__ __forceinline__ int fetch_block(Ctx &C, int cb, int w, unsigned epoch, double *ys)
{
    const int64_t c0 = C.p0 + (int64_t)cb * TB;
    if (C.tid < TB) ys[C.tid] = (C.tid < w) ? ll_get(C.a.yll + 2 * (c0 + C.tid), epoch) : 0.0;
    if (C.tid == TB) g_sm.ival[cb & 1] = ll_get_exp(C.a.yll_exp + cb, epoch);
    __syncthreads();
    return g_sm.ival[cb & 1];
}

// One 128 x 128 tile of the block row (column-major, ld ldx) held in registers by the
// CTA: thread (rp, grp) keeps rows 2rp, 2rp+1 of columns grp, grp+8, ..., loaded with
// 16-byte loads BEFORE the solution block it multiplies is waited for (the loads do not
// depend on it), so HBM latency is off the chain's critical path.
struct TileRegs {
    double2 x[16];
};
__device__ __forceinline__ void tile_load(TileRegs &t, const double *Xt, int64_t ldx, int w, int h, int tid)
{
    const int rp = tid & 63, grp = tid >> 6;  // 64 row pairs x 8 column groups
    const bool vec = ((ldx & 1) == 0) && ((((uintptr_t)Xt) & 15) == 0);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int l = grp + 8 * q;
        if (vec && l < w && 2 * rp + 1 < h) {
            t.x[q] = *reinterpret_cast<const double2 *>(Xt + (size_t)l * ldx + 2 * rp);
        } else {
            t.x[q].x = (l < w && 2 * rp < h) ? Xt[(size_t)l * ldx + 2 * rp] : 0.0;
            t.x[q].y = (l < w && 2 * rp + 1 < h) ? Xt[(size_t)l * ldx + 2 * rp + 1] : 0.0;
        }
    }
}
__device__ __forceinline__ void tile_fma(const TileRegs &t, const double *ys, int tid, double &a0, double &a1)
{
    const int grp = tid >> 6;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const double yv = ys[grp + 8 * q];
        a0 = fma(t.x[q].x, yv, a0);
        a1 = fma(t.x[q].y, yv, a1);
    }
}

// Block back-substitution  y~ = B(p0:n, p0:n)^{-1} rhs  (flag chain, 128-row blocks).
// rhs(r) = base(r) - U(r, 0:k) z2(0:k) - unew(r) z2(k).
// Block b is owned by CTA (Nb-1-b) mod G and published through the 64-bit word
// flag-in-data words (yll, yll_exp) with exponent e_b, where true y~_b = 2^e_b * vy_b.
// Safe blocks use the pre-scaled block rows  Bt_bc = Dinv_b B_bc  (c > b, formed per
// panel by ht_panel_run):  y~_b = Dinv_b rhs_b - sum_{c > b} Bt_bc y~_c, the terms
// accumulated as the y~_c arrive; the chain's critical path is the last term
// Bt_{b,b+1} y~_{b+1}, staged in shared memory.  Unsafe blocks (tiny pivots) use the
// original B and the overflow-safe sequential substitution.
template <class BaseF, class UnewF>
__device__ void trsv_blocked(Ctx &C, BaseF base, UnewF unew, int k, const double *z2, unsigned epoch, int64_t jcol)
{
    unsigned long long *tt = (C.a.ttrace && jcol == C.a.tcol && C.tid == 0) ? C.a.ttrace : nullptr;
    const PanelArgs &a = C.a;
    double *Dsm = g_dyn;             // TB x TB: Bt_{b,b+1} (safe) or D (unsafe)
    double *accg = g_dyn + TB * TB;  // 4 x TB (reused as 8 x 64 pairs)
    const int64_t n = C.n, p0 = C.p0, M = C.M;
    const int Nb = (int)((M + TB - 1) / TB);
    const int ri = C.tid & (TB - 1), grp = C.tid >> 7;  // 128 rows x 4 column groups
    // Blocks are paired from the bottom into super-blocks {hi = Nb-1-2s, lo = hi-1}, one
    // super-block per 2-CTA cluster: rank 0 solves hi, rank 1 solves lo, and hi's solution
    // reaches lo through distributed shared memory instead of a flag round trip through L2.
    cg::cluster_group cl = cg::this_cluster();
    const bool pair = cl.num_blocks() == 2;  // else (profiling launch) single CTAs, L2 hand-offs only
    const int per = pair ? 2 : 1;
    const int rank = pair ? (int)cl.block_rank() : 0, ncl = C.G / per, cid = C.bid / per;
    const int Nsb = (Nb + per - 1) / per;
    for (int sb = cid; sb < Nsb; sb += ncl) {
        const int b = Nb - 1 - per * sb - rank;  // hi (rank 0) or lo (rank 1)
        const bool paired_lo = pair && rank == 1;  // lo: y~_{b+1} comes from the partner
        if (b < 0) {  // odd Nb: the top super-block has no lo; its hi still hands over
            mbar_wait_parity(&g_sm.mbar, C.mbpar);
            C.mbpar ^= 1u;
            if (Nsb > ncl) cl.sync();
            continue;
        }
        const int64_t r0 = p0 + (int64_t)b * TB;
        const int h = (int)(n - r0 < TB ? n - r0 : TB);
        const bool safe = a.dsafe[b] != 0;
        const bool last = (b == Nb - 1);
        const int hn = last ? 0 : (int)(n - (r0 + TB) < TB ? n - (r0 + TB) : TB);  // rows of block b+1
        // off-diagonal tiles: B, or the packed Bt (a.ldbt = TB), addressed like B: tile (b, c)
        // = Bsrc + c0(c) * ldsrc + r0 with the base shifted so that tile (b, b+1) is block row b's start
        const double *Bsrc = safe ? a.Bt + bt_row_offset(M, b) - ((r0 + TB) * a.ldbt + r0) : a.B;
        const int64_t ldsrc = safe ? a.ldbt : a.ldb;
        // (1) rhs_b (all loads of a thread first)
        {
            const int64_t r = r0 + ri;
            double u = 0.0;
            if (ri < h) {
                double uv[8], zv[8];
                for (int c0 = grp; c0 < k; c0 += 32) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int c = c0 + 4 * q;
                        uv[q] = (c < k) ? a.U[(size_t)c * n + r] : 0.0;
                        zv[q] = (c < k) ? z2[c] : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) u = fma(uv[q], zv[q], u);
                }
            }
            accg[grp * TB + ri] = u;
            __syncthreads();
            if (C.tid < TB) {
                double rb = 0.0;
                if (C.tid < h) {
                    const int64_t rr = r0 + C.tid;
                    rb = base(rr) - ((accg[C.tid] + accg[TB + C.tid]) + (accg[2 * TB + C.tid] + accg[3 * TB + C.tid]))
                         - unew(rr) * z2[k];
                }
                g_sm.rhs[C.tid] = rb;
            }
            __syncthreads();
        }
        // (2) stage Bt_{b,b+1} (safe) or D (unsafe) in shared memory; c_b = Dinv_b rhs_b (safe)
        if (safe) {
            if (!last) {
                const double *src = Bsrc + (size_t)(r0 + TB) * a.ldbt + r0;
                for (int l0 = 0; l0 < TB; l0 += 32) {  // 32 columns per round, 8 loads per thread
                    double t[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int idx = C.tid + q * PNT, l = l0 + idx / TB, i = idx % TB;
                        t[q] = (l < hn && i < h) ? src[(size_t)l * a.ldbt + i] : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int idx = C.tid + q * PNT;
                        Dsm[(l0 + idx / TB) * TB + idx % TB] = t[q];
                    }
                }
            }
            const double *Di = a.Dinv + (size_t)b * TB * TB;
            double s = 0.0;
            double dv[8];
            for (int l0 = grp; l0 < TB; l0 += 32) {
#pragma unroll
                for (int q = 0; q < 8; ++q) dv[q] = Di[(l0 + 4 * q) * TB + ri];
#pragma unroll
                for (int q = 0; q < 8; ++q) s = fma(dv[q], g_sm.rhs[l0 + 4 * q], s);
            }
            accg[grp * TB + ri] = s;
            __syncthreads();
            if (C.tid < TB)
                g_sm.cbv[C.tid] = (accg[C.tid] + accg[TB + C.tid]) + (accg[2 * TB + C.tid] + accg[3 * TB + C.tid]);
            __syncthreads();
        } else {
            for (int idx = C.tid; idx < TB * TB; idx += PNT) {
                int i = idx & (TB - 1), j = idx >> 7;
                Dsm[idx] = (i < h && j < h && i <= j) ? a.B[(size_t)(r0 + j) * a.ldb + r0 + i] : 0.0;
            }
        }
        // (3) off-diagonal tiles c > b+1 (safe) or c > b (unsafe), as their solutions arrive
        double acc0 = 0.0, acc1 = 0.0;
        int Eacc = 0;
        const int cstop = safe ? b + 1 : b;
        double *ys = accg + 4 * TB;  // staged solution block (TB doubles)
        for (int cb = Nb - 1; cb > cstop; --cb) {
            const int64_t c0 = p0 + (int64_t)cb * TB;
            const int w = (int)(n - c0 < TB ? n - c0 : TB);
            TileRegs tr;
            tile_load(tr, Bsrc + (size_t)c0 * ldsrc + r0, ldsrc, w, h, C.tid);  // independent of y~_cb
            const int ecb = fetch_block(C, cb, w, epoch, ys);
            if (ecb > Eacc) {
                acc0 *= pow2i(Eacc - ecb);
                acc1 *= pow2i(Eacc - ecb);
                Eacc = ecb;
            }
            double t0 = 0.0, t1 = 0.0;
            tile_fma(tr, ys, C.tid, t0, t1);
            const double sc = pow2i(ecb - Eacc);
            acc0 = fma(t0, sc, acc0);
            acc1 = fma(t1, sc, acc1);
            __syncthreads();  // ys is reused by the next tile
        }
        if (tt) tt[8 * b + 0] = gtime();
        int e = Eacc;
        double xv = 0.0;  // this thread's entry of the block (tid < TB), exponent e
        const int rp = C.tid & 63, g8 = C.tid >> 6;
        if (safe) {
            // (4) critical path: y~_b = c_b 2^(-E) - [acc 2^(Eacc-E) + Bt_{b,b+1} y~_{b+1} 2^(e1-E)]:
            // the tile moves from shared memory into registers before the wait, so after the
            // hand-over the hop is 32 FMA + one 8-way fold (the off-diagonal sums ride along)
            if (!last) {
                TileRegs ct;  // rows 2rp, 2rp+1; columns g8 + 8q
#pragma unroll
                for (int q = 0; q < 16; ++q) ct.x[q] = *reinterpret_cast<const double2 *>(Dsm + (g8 + 8 * q) * TB + 2 * rp);
                const double *yb1;
                int e1;
                if (paired_lo) {
                    mbar_wait_parity(&g_sm.mbar, C.mbpar);  // partner wrote y~_{b+1}, exponent
                    yb1 = g_sm.yrecv;
                    e1 = g_sm.erecv;
                } else {
                    e1 = fetch_block(C, b + 1, hn, epoch, g_sm.rhs);
                    yb1 = g_sm.rhs;
                }
                if (tt) tt[8 * b + 1] = gtime() + (yb1[0] != yb1[0] ? 1 : 0);  // depends on the staged data
                double t0 = 0.0, t1 = 0.0;
                tile_fma(ct, yb1, C.tid, t0, t1);
                const int E = max(e1, Eacc);
                const double sa_ = pow2i(Eacc - E), sb_ = pow2i(e1 - E);
                acc0 = fma(t0, sb_, acc0 * sa_);
                acc1 = fma(t1, sb_, acc1 * sa_);
                e = E;
            }
            accg[g8 * TB + 2 * rp] = acc0;  // fold the 8 column groups: rows 2rp, 2rp+1
            accg[g8 * TB + 2 * rp + 1] = acc1;
            __syncthreads();
            if (tt) tt[8 * b + 3] = gtime() + (accg[0] != accg[0] ? 1 : 0);
            if (C.tid < TB) {
                double s8 = 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q) s8 += accg[q * TB + C.tid];
                xv = g_sm.cbv[C.tid] * pow2i(-e) - s8;
            }
            // (5) post-hoc power-of-two rescale, only if some entry of the block is too large
            const bool big = (C.tid < h) && !(fabs(xv) <= BIG);
            int ex = 0;
            if (__syncthreads_or(big)) {
                double mx = (C.tid < h) ? fabs(xv) : 0.0;
                mx = warp_max(mx);
                if (C.tid < TB && C.lane == 0) g_sm.red[C.warp] = mx;
                __syncthreads();
                mx = fmax(fmax(g_sm.red[0], g_sm.red[1]), fmax(g_sm.red[2], g_sm.red[3]));
                if (!(mx <= BIG)) frexp(mx, &ex);
                if (!isfinite(mx)) ex = 0;
            }
            if (ex) xv = ldexp(xv, -ex);
            e += ex;
            if (pair && !paired_lo && C.tid < TB) {
                // hand y~_b to the lo partner's shared memory FIRST (before the global stores)
                PanelSmem *peer = cl.map_shared_rank(&g_sm, 1);
                peer->yrecv[C.tid] = (C.tid < h) ? xv : 0.0;
                if (C.tid == 0) peer->erecv = e;
                mbar_remote_arrive(&g_sm.mbar, 1);
            }
            if (C.tid < h) {
                a.vy[r0 + C.tid] = xv;
                ll_put(a.yll + 2 * (r0 + C.tid), xv, epoch);
            }
        } else {
            accg[g8 * TB + 2 * rp] = acc0;  // fold the 8 column groups: rows 2rp, 2rp+1
            accg[g8 * TB + 2 * rp + 1] = acc1;
            __syncthreads();
            double s8 = 0.0;
            if (C.tid < TB) {
#pragma unroll
                for (int q = 0; q < 8; ++q) s8 += accg[q * TB + C.tid];
            }
            __syncthreads();
            if (C.tid < TB) g_sm.rhs[C.tid] = (C.tid < h) ? ldexp(g_sm.rhs[C.tid], -Eacc) - s8 : 0.0;
            __syncthreads();
            if (C.warp == 0) {
                // overflow-safe sequential back-substitution (unsafe block, e.g. config 4)
                const int l = C.lane;
                double v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = g_sm.rhs[l + 32 * q];
                for (int c = h - 1; c >= 0; --c) {
                    const int own = c & 31, hq = c >> 5;
                    double mine = v[0];
                    if (hq == 1) mine = v[1];
                    if (hq == 2) mine = v[2];
                    if (hq == 3) mine = v[3];
                    const double dcc = Dsm[c * TB + c];
                    double xc = __shfl_sync(0xffffffffu, mine, own) / dcc;
                    if (!(fabs(xc) <= BIG)) {
                        int exx;
                        frexp(xc, &exx);
#pragma unroll
                        for (int q = 0; q < 4; ++q) v[q] = ldexp(v[q], -exx);
                        e += exx;
                        mine = v[0];
                        if (hq == 1) mine = v[1];
                        if (hq == 2) mine = v[2];
                        if (hq == 3) mine = v[3];
                        xc = __shfl_sync(0xffffffffu, mine, own) / dcc;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int row = l + 32 * q;
                        if (row == c) v[q] = xc;
                        else if (row < c) v[q] -= Dsm[c * TB + row] * xc;
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (l + 32 * q < h) {
                        a.vy[r0 + l + 32 * q] = v[q];
                        g_sm.rhs[l + 32 * q] = v[q];
                        ll_put(a.yll + 2 * (r0 + l + 32 * q), v[q], epoch);
                    }
                if (l == 0) g_sm.ival[3] = e;
            }
            __syncthreads();
            e = g_sm.ival[3];
            if (C.tid < TB) xv = (C.tid < h) ? g_sm.rhs[C.tid] : 0.0;
            if (pair && !paired_lo && C.tid < TB) {  // unsafe hi block: hand y~_b over
                PanelSmem *peer = cl.map_shared_rank(&g_sm, 1);
                peer->yrecv[C.tid] = (C.tid < h) ? xv : 0.0;
                if (C.tid == 0) peer->erecv = e;
                mbar_remote_arrive(&g_sm.mbar, 1);
            }
        }
        // the block exponent: its word carries the epoch like the value words (no ordering with them)
        if (C.tid == 0) {
            a.bexp[b] = e;
            st_volatile64(a.yll_exp + b, ((unsigned long long)epoch << 32) | (unsigned)e);
            if (tt) tt[8 * b + 2] = gtime();
        }
        if (paired_lo) {
            // every phase of the mbarrier completes once per super-block (the hi partner always
            // hands over); a lo block that did not wait on it still consumes the phase
            if (!(safe && !last)) mbar_wait_parity(&g_sm.mbar, C.mbpar);
            C.mbpar ^= 1u;
        }
        // yrecv is rewritten only by the next super-block of this cluster: a cluster barrier keeps
        // the lo CTA's reads of this one ahead of it (not needed while n <= TB * G)
        if (pair && Nsb > ncl) cl.sync();
        else __syncthreads();
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// 256-row flag-chained solve on 4-CTA clusters (trsv4).  Same recurrence as trsv_blocked,
//   y~_b = Dinv4_b rhs_b - sum_{c > b} Bt_bc y~_c,   Bt_bc = Dinv4_b B_bc   (packed, ld T4),
// with blocks of T4 = 256 rows: half as many hops on the chain's critical path.  Cluster
// rank q owns the 64-column slice q of every tile of its block row (T4 x 64 doubles in
// registers, 32 per thread) and consumes only slice q of each y~_c; its 256-row partial sums
// (and its slice of Dinv4_b rhs_b) reach rank 0 in one bulk copy over distributed shared
// memory, and rank 0 forms and publishes y~_b (one exponent per block, as trsv_blocked).
// Used for a panel only when every 256-row diagonal block is safe (ht_panel_run).
__host__ __device__ __forceinline__ int64_t bt4_row_offset(int64_t M, int64_t b)
{
    return (int64_t)T4 * (b * M - (int64_t)T4 * b * (b + 1) / 2);
}
struct Tile4 {
    double2 x[16];  // rows 2rp, 2rp+1 x columns 16 grp + u of the slice
};
__device__ __forceinline__ void tile4_load(Tile4 &t, const double *X, int w, int h, int tid)
{
    const int rp = tid & 127, grp = tid >> 7;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const int c = 16 * grp + u;
        if (c < w && 2 * rp + 1 < h) {
            t.x[u] = *reinterpret_cast<const double2 *>(X + (size_t)c * T4 + 2 * rp);
        } else {
            t.x[u].x = (c < w && 2 * rp < h) ? X[(size_t)c * T4 + 2 * rp] : 0.0;
            t.x[u].y = 0.0;
        }
    }
}
__device__ __forceinline__ void tile4_fma(const Tile4 &t, const double *ys, int tid, double &a0, double &a1)
{
    const int grp = tid >> 7;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const double yv = ys[16 * grp + u];
        a0 = fma(t.x[u].x, yv, a0);
        a1 = fma(t.x[u].y, yv, a1);
    }
}
// slice q (w values) of the published solution block cb (256-row blocks) and its exponent
__device__ __forceinline__ int fetch4(Ctx &C, int cb, int q, int w, unsigned epoch, double *ys)
{
    const int64_t c0 = C.p0 + (int64_t)cb * T4 + 64 * q;
    if (C.tid < 64) ys[C.tid] = (C.tid < w) ? ll_get(C.a.yll + 2 * (c0 + C.tid), epoch) : 0.0;
    if (C.tid == 64) g_sm.ival[cb & 1] = ll_get_exp(C.a.yll_exp + cb, epoch);
    __syncthreads();
    return g_sm.ival[cb & 1];
}
template <class BaseF, class UnewF>
__device__ void trsv4(Ctx &C, BaseF base, UnewF unew, int k, const double *z2, unsigned epoch)
{
    const PanelArgs &a = C.a;
    const int64_t n = C.n, p0 = C.p0, M = C.M;
    const int Nb = (int)((M + T4 - 1) / T4);
    cg::cluster_group cl = cg::this_cluster();
    const int q = (int)cl.block_rank(), ncl = C.G / C4, cid = C.bid / C4;
    const int rp = C.tid & 127, grp = C.tid >> 7;
    constexpr int SZ = 2 * T4 + 8;  // message: 256 partial sums, 256 slice sums of Dinv4 rhs, exponent
    double *ys = g_dyn;             // [64]
    double *rs = ys + 64;           // [64] rhs slice
    double *pa = rs + 64;           // [4][T4] partial sums of the column groups
    double *pc = pa + 4 * T4;       // [4][T4]
    double *snd = pc + 4 * T4;      // [SZ] message to rank 0
    double *rcv = snd + SZ;         // [3][SZ] messages at rank 0
    for (int sb = cid; sb < Nb; sb += ncl) {
        const int b = Nb - 1 - sb;
        const int64_t r0 = p0 + (int64_t)b * T4;
        const int h = (int)(n - r0 < T4 ? n - r0 : T4);
        const bool last = (b == Nb - 1);
        const int hq = h - 64 * q < 0 ? 0 : (h - 64 * q > 64 ? 64 : h - 64 * q);  // rows of slice q
        // (1) slice q of rhs_b, then its share of Dinv4_b rhs_b (independent of the chain)
        {
            const int row = C.tid >> 3, part = C.tid & 7;
            const int64_t r = r0 + 64 * q + row;
            double u = 0.0;
            if (row < hq)
                for (int c = part; c < k; c += 8) u = fma(a.U[(size_t)c * n + r], z2[c], u);
            u += __shfl_xor_sync(0xffffffffu, u, 1);
            u += __shfl_xor_sync(0xffffffffu, u, 2);
            u += __shfl_xor_sync(0xffffffffu, u, 4);
            if (part == 0) rs[row] = (row < hq) ? base(r) - u - unew(r) * z2[k] : 0.0;
            __syncthreads();
        }
        double c0 = 0.0, c1 = 0.0;
        {
            Tile4 dt;
            tile4_load(dt, a.Dinv4 + (size_t)b * T4 * T4 + (size_t)(64 * q) * T4, hq, h, C.tid);
            tile4_fma(dt, rs, C.tid, c0, c1);
        }
        // (2) off-diagonal tiles c > b+1, as their solution slices arrive
        double acc0 = 0.0, acc1 = 0.0;
        int Eacc = 0;
        const double *rowp = a.Bt + bt4_row_offset(M, b);  // columns from p0 + T4 (b+1), ld T4
        for (int cb = Nb - 1; cb > b + 1; --cb) {
            const int64_t cw0 = (int64_t)T4 * cb + 64 * q;  // first column of the slice (relative to p0)
            const int w = (int)(M - cw0 < 0 ? 0 : (M - cw0 > 64 ? 64 : M - cw0));
            Tile4 tr;
            tile4_load(tr, rowp + (size_t)(cw0 - (int64_t)T4 * (b + 1)) * T4, w, h, C.tid);
            const int ecb = fetch4(C, cb, q, w, epoch, ys);
            if (ecb > Eacc) {
                acc0 *= pow2i(Eacc - ecb);
                acc1 *= pow2i(Eacc - ecb);
                Eacc = ecb;
            }
            double t0 = 0.0, t1 = 0.0;
            tile4_fma(tr, ys, C.tid, t0, t1);
            const double sc = pow2i(ecb - Eacc);
            acc0 = fma(t0, sc, acc0);
            acc1 = fma(t1, sc, acc1);
            __syncthreads();  // ys is reused
        }
        int E = Eacc;
        if (!last) {  // (3) the critical tile (b, b+1): loaded before the wait for y~_{b+1}
            const int64_t cw0 = (int64_t)T4 * (b + 1) + 64 * q;
            const int w = (int)(M - cw0 < 0 ? 0 : (M - cw0 > 64 ? 64 : M - cw0));
            Tile4 ct;
            tile4_load(ct, rowp + (size_t)(64 * q) * T4, w, h, C.tid);
            const int e1 = fetch4(C, b + 1, q, w, epoch, ys);
            double t0 = 0.0, t1 = 0.0;
            tile4_fma(ct, ys, C.tid, t0, t1);
            E = max(e1, Eacc);
            const double sa_ = pow2i(Eacc - E), sb_ = pow2i(e1 - E);
            acc0 = fma(t0, sb_, acc0 * sa_);
            acc1 = fma(t1, sb_, acc1 * sa_);
        }
        // (4) fold the 4 column groups; ranks 1-3 send their 256-row sums to rank 0
        pa[grp * T4 + 2 * rp] = acc0;
        pa[grp * T4 + 2 * rp + 1] = acc1;
        pc[grp * T4 + 2 * rp] = c0;
        pc[grp * T4 + 2 * rp + 1] = c1;
        __syncthreads();
        double sa = 0.0, sc = 0.0;
        if (C.tid < T4) {
            sa = (pa[C.tid] + pa[T4 + C.tid]) + (pa[2 * T4 + C.tid] + pa[3 * T4 + C.tid]);
            sc = (pc[C.tid] + pc[T4 + C.tid]) + (pc[2 * T4 + C.tid] + pc[3 * T4 + C.tid]);
            if (q != 0) {
                snd[C.tid] = sa;
                snd[T4 + C.tid] = sc;
            }
        }
        if (q != 0) {
            if (C.tid == 0) snd[2 * T4] = (double)E;
            if (C.tid < T4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // writers: generic -> bulk copy
            __syncthreads();
            if (C.tid == 0) {
                unsigned dst, mbr;
                const unsigned src = (unsigned)__cvta_generic_to_shared(snd);
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst)
                             : "r"((unsigned)__cvta_generic_to_shared(rcv + (q - 1) * SZ)), "r"(0));
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(mbr)
                             : "r"((unsigned)__cvta_generic_to_shared(&g_sm.mbar4)), "r"(0));
                // relaxed: rank 0 needs only the copied bytes (complete_tx), not this thread's other writes
                asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(mbr),
                             "r"(SZ * 8) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(dst), "r"(src), "r"(SZ * 8), "r"(mbr) : "memory");
            }
        } else {
            // (5) rank 0: combine, rescale if needed, publish y~_b.  The messages are bulk copies into
            // this CTA's shared memory counted on its own mbarrier: a CTA-scope wait suffices
            {
                const unsigned ma = (unsigned)__cvta_generic_to_shared(&g_sm.mbar4);
                unsigned done = 0;
                while (!done)
                    asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
                                 : "=r"(done) : "r"(ma), "r"(C.mb4par) : "memory");
            }
            C.mb4par ^= 1u;
            int ei[3];
            int Eall = E;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                ei[i] = (int)rcv[i * SZ + 2 * T4];
                Eall = max(Eall, ei[i]);
            }
            double xv = 0.0;
            if (C.tid < T4) {
                double s = sa * pow2i(E - Eall), c = sc;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    s = fma(rcv[i * SZ + C.tid], pow2i(ei[i] - Eall), s);
                    c += rcv[i * SZ + T4 + C.tid];
                }
                xv = c * pow2i(-Eall) - s;
            }
            int e = Eall;
            const bool big = (C.tid < h) && !(fabs(xv) <= BIG);
            int ex = 0;
            if (__syncthreads_or(big)) {
                double mx = (C.tid < h) ? fabs(xv) : 0.0;
                mx = warp_max(mx);
                if (C.lane == 0) g_sm.red[C.warp] = mx;
                __syncthreads();
                mx = 0.0;
                for (int w = 0; w < NWP; ++w) mx = fmax(mx, g_sm.red[w]);
                if (!(mx <= BIG)) frexp(mx, &ex);
                if (!isfinite(mx)) ex = 0;
            }
            if (ex) xv = ldexp(xv, -ex);
            e += ex;
            if (C.tid == 0) st_volatile64(a.yll_exp + b, ((unsigned long long)epoch << 32) | (unsigned)e);
            if (C.tid < h) ll_put(a.yll + 2 * (r0 + C.tid), xv, epoch);  // the chain's hand-over first
            if (C.tid < h) a.vy[r0 + C.tid] = xv;
            if (C.tid == 0) a.bexp[b] = e;
        }
        // the messages' buffers are reused by the next block of this cluster
        cl.sync();
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// 256-row flag-chained solve with the rows of a block split over four CTAs (trsv4r).
// Same recurrence as trsv4,  y~_b = Dinv4_b rhs_b - sum_{c > b} Bt_bc y~_c  (Bt_bc = Dinv4_b B_bc),
// but because Dinv4_b is the inverse of the whole 256 x 256 diagonal block, every ROW of y~_b
// depends only on the blocks below it: the four 64-row slices (b, q) of a block are independent
// work units.  Unit (b, q) holds rows 64q.. of the critical tile Bt_{b,b+1} in registers (64 x 256,
// 32 doubles per thread), waits for all of y~_{b+1} (four published slices), folds its eight
// column groups in shared memory and publishes its 64 rows with their own exponent -- no
// cluster, no distributed-shared-memory combine step on the chain (a hop is one L2 hand-over
// plus one register mat-vec).  Units u = 4 (Nb-1-b) + q go to CTA u mod G in increasing u; a
// unit only waits on lower units, so the chain cannot deadlock.  Exponent words and bexp are
// per 64-row slice (C.tbs = 64).
__device__ __forceinline__ void tile64_load(double (&t)[32], const double *X, int w, int h, int tid)
{
    const int rr = 32 * ((tid >> 5) & 1) + (tid & 31), grp = tid >> 6;  // row of the slice, 8 column groups
    const double *x = X + (size_t)(32 * grp) * T4 + rr;
    if (rr < h && 32 * grp + 32 <= w) {  // full: unpredicated loads at immediate offsets (few registers)
#pragma unroll
        for (int u = 0; u < 32; ++u) t[u] = __ldcs(x + (size_t)u * T4);  // streamed once
    } else {
#pragma unroll
        for (int u = 0; u < 32; ++u) t[u] = (32 * grp + u < w && rr < h) ? __ldcs(x + (size_t)u * T4) : 0.0;
    }
}
__device__ __forceinline__ double tile64_dot(const double (&t)[32], const double *ys, int tid)
{
    const double *y = ys + 32 * (tid >> 6);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int u = 0; u < 32; u += 4) {
        s0 = fma(t[u], y[u], s0);
        s1 = fma(t[u + 1], y[u + 1], s1);
        s2 = fma(t[u + 2], y[u + 2], s2);
        s3 = fma(t[u + 3], y[u + 3], s3);
    }
    return (s0 + s1) + (s2 + s3);
}
// part pf (columns 8 pf .. 8 pf + 7 of the thread's 32) of a 64 x 256 slice tile: the streamed
// tiles go through 8 registers at a time (the critical tile holds 32)
constexpr int TPART = 8;
__device__ __forceinline__ void tile64_load_part(double (&t)[TPART], const double *X, int w, int h, int tid, int pf)
{
    const int rr = 32 * ((tid >> 5) & 1) + (tid & 31), grp = tid >> 6, c0 = 32 * grp + TPART * pf;
    const double *x = X + (size_t)c0 * T4 + rr;
    if (rr < h && c0 + TPART <= w) {
#pragma unroll
        for (int u = 0; u < TPART; ++u) t[u] = __ldcs(x + (size_t)u * T4);
    } else {
#pragma unroll
        for (int u = 0; u < TPART; ++u) t[u] = (c0 + u < w && rr < h) ? __ldcs(x + (size_t)u * T4) : 0.0;
    }
}
__device__ __forceinline__ double tile64_dot_part(const double (&t)[TPART], const double *ys, int tid, int pf)
{
    const double *y = ys + 32 * (tid >> 6) + TPART * pf;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int u = 0; u < TPART; u += 2) {
        s0 = fma(t[u], y[u], s0);
        s1 = fma(t[u + 1], y[u + 1], s1);
    }
    return s0 + s1;
}
// all hc rows of the published block cb into ys[], the four slice exponents into g_sm.es4
__device__ __forceinline__ void fetch4r(const PanelArgs &a, int64_t p0, int cb, int hc, unsigned epoch, double *ys)
{
    const int64_t c0 = p0 + (int64_t)cb * T4;
    const int tid = threadIdx.x;
    if (tid < T4) ys[tid] = (tid < hc) ? ll_get(a.yll + 2 * (c0 + tid), epoch) : 0.0;
    else if (tid < T4 + 4) {
        const int q = tid - T4;
        g_sm.es4[q] = (64 * q < hc) ? ll_get_exp(a.yll_exp + 4 * cb + q, epoch) : 0;
    }
    __syncthreads();
}
// The right-hand side of a solve, rhs(r) = base(r) - U(r, 0:k) z2(0:k) - unew(r) z2(k), in scalar
// form (the solve is a separate, non-inlined function so that its critical tile owns the
// registers):  base(r) = bvec ? bvec[r] : (r == jb ? 1 : 0);
//              unew(r) = ucol ? ucol[r] : (r < j1 ? 0 : (r == j1 ? 1 : ux[r] * uscal)).
struct RhsSpec {
    const double *bvec, *ucol, *ux;
    int64_t jb, j1;
    double uscal;
    __device__ __forceinline__ double base(int64_t r) const { return bvec ? __ldcg(bvec + r) : (r == jb ? 1.0 : 0.0); }
    __device__ __forceinline__ double unew(int64_t r) const
    {
        return ucol ? __ldcg(ucol + r) : (r < j1 ? 0.0 : (r == j1 ? 1.0 : __ldcg(ux + r) * uscal));
    }
};
__device__ __noinline__ void trsv4r(const PanelArgs &a, const RhsSpec rs, int k, const double *z2, unsigned epoch,
                                    int64_t jcol)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, G = gridDim.x, bid = blockIdx.x;
    unsigned long long *tt = (a.ttrace && jcol == a.tcol && tid == 0) ? a.ttrace : nullptr;  // HT_TRACE_COL
    const int64_t n = a.n, p0 = a.s0 + 1, M = n - p0;
    const int Nb = (int)((M + T4 - 1) / T4);
    const int grp = tid >> 6, rr = 32 * ((tid >> 5) & 1) + lane;
    double *ys = g_dyn;           // [T4] fetched y~_c
    double *rhs = ys + T4;        // [T4] rhs_b
    double *pw = rhs + T4;        // [NWP][T4] rhs partials / [3][8][64] fold
    for (int u = bid; u < 4 * Nb; u += G) {
        const int sb = u >> 2, q = u & 3, b = Nb - 1 - sb;
        const int64_t rb0 = p0 + (int64_t)b * T4;
        const int hb = (int)(n - rb0 < T4 ? n - rb0 : T4);
        const int h = hb - 64 * q < 0 ? 0 : (hb - 64 * q > 64 ? 64 : hb - 64 * q);
        if (h <= 0) continue;  // no rows: nothing to publish, consumers skip the slice
        const int64_t r0 = rb0 + 64 * q;
        unsigned long long *tu = tt ? tt + 8 * (size_t)(4 * b + q) : nullptr;
        if (tu) tu[4] = gtime();
        const double *rowp = a.Bt + bt4_row_offset(M, b) + 64 * q;  // columns from p0 + T4 (b+1), ld T4
        const int wcrit = (b + 1 < Nb) ? (int)(M - (int64_t)T4 * (b + 1) < T4 ? M - (int64_t)T4 * (b + 1) : T4) : 0;
        // (1) rhs_b = base - U z2 - unew z2(k) over the hb rows of block b: warps over columns,
        //     lanes over rows, 4 columns x 8 row chunks of loads per batch
        {
            double acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = 0.0;
            for (int c0 = warp; c0 < k; c0 += NWP * 2) {
                double uv[2][8];
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const int c = c0 + NWP * t;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int r = 32 * j + lane;
                        uv[t][j] = (c < k && r < hb) ? a.U[(size_t)c * n + rb0 + r] : 0.0;
                    }
                }
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const int c = c0 + NWP * t;
                    const double zc = c < k ? z2[c] : 0.0;
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j] = fma(uv[t][j], zc, acc[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) pw[warp * T4 + 32 * j + lane] = acc[j];
            __syncthreads();
            if (tid < T4) {
                double s = 0.0;
#pragma unroll
                for (int w = 0; w < NWP; ++w) s += pw[w * T4 + tid];
                const int64_t r = rb0 + tid;
                rhs[tid] = (tid < hb) ? rs.base(r) - s - rs.unew(r) * z2[k] : 0.0;
            }
            __syncthreads();
        }
        // (2) this slice's rows of Dinv4_b rhs_b (half tiles: the critical tile holds 32 registers)
        double cd = 0.0;
#pragma unroll 1
        for (int pf = 0; pf < 32 / TPART; ++pf) {
            double t[TPART];
            tile64_load_part(t, a.Dinv4 + (size_t)b * T4 * T4 + 64 * q, hb, h, tid, pf);
            cd += tile64_dot_part(t, rhs, tid, pf);
            asm volatile("" ::: "memory");
        }
        // (3) off-diagonal tiles c > b+1 as their solutions arrive (exponent per column group)
        double acc = 0.0;
        int E = 0;
        for (int cb = Nb - 1; cb > b + 1; --cb) {
            const int wc = (int)(M - (int64_t)T4 * cb < T4 ? M - (int64_t)T4 * cb : T4);
            double t[32];  // the whole slice tile in flight (per-SM streaming bandwidth)
            tile64_load(t, rowp + (size_t)T4 * (cb - b - 1) * T4, wc, h, tid);
            fetch4r(a, p0, cb, wc, epoch, ys);
            const int ec = g_sm.es4[grp >> 1];
            const double tc = tile64_dot(t, ys, tid);
            if (ec > E) {
                acc *= pow2i(E - ec);
                E = ec;
            }
            acc = fma(tc, pow2i(ec - E), acc);
            __syncthreads();  // ys is reused
        }
        if (tu) tu[0] = gtime();
        // (4) the critical tile (b, b+1): loaded after the streamed tiles (registers), before the
        // wait for y~_{b+1}
        if (b + 1 < Nb) {
            double tcrit[32];
            tile64_load(tcrit, rowp, wcrit, h, tid);
            fetch4r(a, p0, b + 1, wcrit, epoch, ys);
            if (tu) tu[1] = gtime();
            const int ec = g_sm.es4[grp >> 1];
            const double tc = tile64_dot(tcrit, ys, tid);
            if (ec > E) {
                acc *= pow2i(E - ec);
                E = ec;
            }
            acc = fma(tc, pow2i(ec - E), acc);
            if (tu) tu[5] = gtime() + (acc != acc);
        }
        // (5) fold the eight column groups: y~ = 2^Eall (cd 2^-Eall - sum acc 2^(E - Eall))
        double *fa = pw, *fc = pw + 8 * 64;
        int *fe = reinterpret_cast<int *>(pw + 16 * 64);
        fa[grp * 64 + rr] = acc;
        fc[grp * 64 + rr] = cd;
        fe[grp * 64 + rr] = E;
        __syncthreads();
        if (tu) tu[6] = gtime();
        double xv = 0.0;
        int e = 0;
        if (tid < 64) {
            int Eall = 0;
#pragma unroll
            for (int g = 0; g < 8; ++g) Eall = max(Eall, fe[g * 64 + tid]);
            double sa = 0.0, sc = 0.0;
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                sa = fma(fa[g * 64 + tid], pow2i(fe[g * 64 + tid] - Eall), sa);
                sc += fc[g * 64 + tid];
            }
            xv = sc * pow2i(-Eall) - sa;
            e = Eall;
        }
        if (tu) tu[3] = gtime();
        // (6) overflow guard (reading R-Z8): a power-of-two rescale of the slice
        const bool big = (tid < h) && !(fabs(xv) <= BIG);
        int ex = 0;
        if (__syncthreads_or(big)) {
            double mx = (tid < h) ? fabs(xv) : 0.0;
            mx = warp_max(mx);
            if (lane == 0) g_sm.red[warp] = mx;
            __syncthreads();
            mx = fmax(g_sm.red[0], g_sm.red[1]);
            if (!(mx <= BIG)) frexp(mx, &ex);
            if (!isfinite(mx)) ex = 0;
        }
        if (tu) tu[7] = gtime();
        // (7) publish: the rows (the chain's hand-over) first, then the slice exponent
        if (tid < h) {
            if (ex) xv = ldexp(xv, -ex);
            ll_put(a.yll + 2 * (r0 + tid), xv, epoch);
            a.vy[r0 + tid] = xv;
        }
        if (tid == 0) {
            st_volatile64(a.yll_exp + 4 * b + q, ((unsigned long long)epoch << 32) | (unsigned)(e + ex));
            a.bexp[4 * b + q] = e + ex;
            if (tu) tu[2] = gtime();
        }
        __syncthreads();
    }
    __syncthreads();
}

// After a completed solve (grid synced): Emax over all blocks.
__device__ int trsv_emax(Ctx &C)
{
    const int Nb = (int)((C.M + C.tbs - 1) / C.tbs);
    int e = INT_MIN;
    for (int b = C.tid; b < Nb; b += PNT) e = max(e, __ldcg(&C.a.bexp[b]));  // all loads in parallel
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e = max(e, __shfl_xor_sync(0xffffffffu, e, o));
    if (C.lane == 0) g_sm.ival[C.warp & 3] = INT_MIN;
    __syncthreads();
    if (C.lane == 0) atomicMax(&g_sm.ival[0], e);
    __syncthreads();
    const int r = g_sm.ival[0];
    __syncthreads();
    return r;
}

// Row-slab sweep  out(r) = sum_{c in [cbeg, n)} X(r,c) vec(c)  over rows [r0, r1)
// (TRI: only c >= r): lanes over 32-row chunks, warps over columns, 4 independent
// accumulators so that every warp keeps 4 column loads in flight.
template <bool TRI, class VecF>
__device__ void slab_sweep(Ctx &C, const double *X, int64_t ldx, int64_t r0, int64_t r1, int64_t cfirst, VecF vec,
                           double *out)
{
    double *stg = g_dyn;  // NWP x 64
    const int64_t n = C.n;
    for (int64_t rc = r0; rc < r1; rc += 64) {
        const int64_t rowA = rc + C.lane, rowB = rc + 32 + C.lane;
        const bool okA = rowA < r1, okB = rowB < r1;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        if (okA) {
            const int64_t cb = TRI ? rc : cfirst;
            const double *xa = X + rowA;
            const double *xb = X + (okB ? rowB : rowA);
            int64_t c = cb + C.warp;
            for (; c + 3 * NWP < n; c += 4 * NWP) {
                double xa_[4], xb_[4], v_[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    xa_[q] = xa[(size_t)(c + q * NWP) * ldx];
                    xb_[q] = xb[(size_t)(c + q * NWP) * ldx];
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) v_[q] = vec(c + q * NWP);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (TRI) {
                        if (rowA > c + q * NWP) xa_[q] = 0.0;
                        if (rowB > c + q * NWP) xb_[q] = 0.0;
                    }
                    if (q & 1) {
                        a1 += xa_[q] * v_[q];
                        b1 += xb_[q] * v_[q];
                    } else {
                        a0 += xa_[q] * v_[q];
                        b0 += xb_[q] * v_[q];
                    }
                }
            }
            for (; c < n; c += NWP) {
                const double v0 = vec(c);
                double xa0 = xa[(size_t)c * ldx], xb0 = xb[(size_t)c * ldx];
                if (TRI) {
                    if (rowA > c) xa0 = 0.0;
                    if (rowB > c) xb0 = 0.0;
                }
                a0 += xa0 * v0;
                b0 += xb0 * v0;
            }
        }
        stg[C.warp * 64 + C.lane] = a0 + a1;
        stg[C.warp * 64 + 32 + C.lane] = okB ? b0 + b1 : 0.0;
        __syncthreads();
        if (C.tid < 64 && rc + C.tid < r1) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < NWP; ++w) t += stg[w * 64 + C.tid];
            out[rc + C.tid] = t;
        }
        __syncthreads();
    }
}

// Tiled mat-vec  y = X(r_beg:r_end, c_beg:c_end) * vf  (TRI: only entries with c >= r,
// i.e. an upper-triangular X), HBM-bound.  The matrix is cut into 256 x 256 items that
// are dealt round-robin to the CTAs; inside an item every warp streams 16 columns with
// 16-byte loads over all 256 rows (16 independent loads in flight per lane), so each
// SM keeps ~128 KB of loads outstanding.  Item partial sums go to ypart[cc][r]
// (cc = column chunk) and are added in a fixed order by tiled_sum2() after a grid sync;
// the items of both mat-vecs are handed out dynamically (tiled_matvec2)
// (deterministic).
constexpr int TRT = 256, TCW = 256;
struct TileGeom {
    int64_t r_al, r_end, c_beg, c_end;
    int nrb, ncc;
    bool tri;
    __device__ TileGeom(int64_t rb_, int64_t re_, int64_t cb_, int64_t ce_, bool t)
        : r_al(rb_ & ~(int64_t)1), r_end(re_), c_beg(cb_), c_end(ce_), tri(t)
    {
        nrb = (int)((r_end - r_al + TRT - 1) / TRT);
        ncc = (int)((c_end - c_beg + TCW - 1) / TCW);
    }
    // first column chunk that meets row block rb (TRI), else 0
    __device__ int cc_min(int rb) const
    {
        if (!tri) return 0;
        const int64_t d = r_al + (int64_t)TRT * rb - c_beg;
        return d <= 0 ? 0 : (int)(d / TCW);
    }
    __device__ int items() const
    {
        if (!tri) return nrb * ncc;
        int t = 0;
        for (int rb = 0; rb < nrb; ++rb) t += ncc - cc_min(rb);
        return t;
    }
    __device__ void item(int i, int &rb, int &cc) const
    {
        if (!tri) { rb = i / ncc; cc = i % ncc; return; }
        for (rb = 0; rb < nrb; ++rb) {
            const int m = ncc - cc_min(rb);
            if (i < m) { cc = cc_min(rb) + i; return; }
            i -= m;
        }
    }
};

// One 256 x 256 item of a fused-sweep mat-vec (see tiled_matvec2).
template <class VF>
__device__ __forceinline__ void sweep_item(Ctx &C, const TileGeom &tg, const double *X, int64_t ldx, VF vf, double *yp,
                                           int it, bool cs)
{
    double *red = g_dyn;               // [NWP][TRT]
    double *vs = g_dyn + NWP * TRT;    // [TCW]
    const bool vec = (ldx % 2) == 0;
        int rb, cc;
        tg.item(it, rb, cc);
        const int64_t r0 = tg.r_al + (int64_t)TRT * rb, c0 = tg.c_beg + (int64_t)TCW * cc;
        __syncthreads();
        if (C.tid < TCW) {
            const int64_t c = c0 + C.tid;
            vs[C.tid] = (c < tg.c_end) ? vf(c) : 0.0;
        }
        __syncthreads();
        double acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0;
        const int cw0 = C.warp * (TCW / NWP);  // 16 columns per warp
        const bool diag = tg.tri && (r0 + TRT - 1 > c0);
        const bool full = (r0 + TRT <= tg.r_end);
        if (vec && full && diag) {
            // triangular item: vector loads, entries below the diagonal masked out
#pragma unroll 1
            for (int u0 = 0; u0 < TCW / NWP; u0 += 2) {
                double2 xv[2][4];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int64_t c = c0 + cw0 + u0 + u;
                    const double2 *col = reinterpret_cast<const double2 *>(X + (size_t)(c < tg.c_end ? c : c0) * ldx + r0);
#pragma unroll
                    for (int i = 0; i < 4; ++i) xv[u][i] = cs ? __ldcs(col + C.lane + 32 * i) : col[C.lane + 32 * i];
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const double v = vs[cw0 + u0 + u];
                    const int kk = (int)(c0 - r0) + cw0 + u0 + u - 2 * C.lane;  // c - r(i=0,h=0)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        acc[2 * i] = fma(64 * i > kk ? 0.0 : xv[u][i].x, v, acc[2 * i]);
                        acc[2 * i + 1] = fma(64 * i + 1 > kk ? 0.0 : xv[u][i].y, v, acc[2 * i + 1]);
                    }
                }
            }
        } else if (vec && full) {
#pragma unroll 1
            for (int u0 = 0; u0 < TCW / NWP; u0 += 4) {
                double2 xv[4][4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t c = c0 + cw0 + u0 + u;
                    const double2 *col = reinterpret_cast<const double2 *>(X + (size_t)(c < tg.c_end ? c : c0) * ldx + r0);
#pragma unroll
                    for (int i = 0; i < 4; ++i) xv[u][i] = cs ? __ldcs(col + C.lane + 32 * i) : col[C.lane + 32 * i];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double v = vs[cw0 + u0 + u];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        acc[2 * i] = fma(xv[u][i].x, v, acc[2 * i]);
                        acc[2 * i + 1] = fma(xv[u][i].y, v, acc[2 * i + 1]);
                    }
                }
            }
        } else {
#pragma unroll 1
            for (int u0 = 0; u0 < TCW / NWP; u0 += 2) {
                double xv[2][8];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int64_t c = c0 + cw0 + u0 + u;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int64_t r = r0 + 2 * C.lane + 64 * i + h;
                            const bool ok = c < tg.c_end && r < tg.r_end && (!tg.tri || c >= r);
                            xv[u][2 * i + h] = ok ? X[(size_t)c * ldx + r] : 0.0;
                        }
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const double v = vs[cw0 + u0 + u];
#pragma unroll
                    for (int q = 0; q < 8; ++q) acc[q] = fma(xv[u][q], v, acc[q]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            red[C.warp * TRT + 2 * C.lane + 64 * i] = acc[2 * i];
            red[C.warp * TRT + 2 * C.lane + 64 * i + 1] = acc[2 * i + 1];
        }
        __syncthreads();
        if (C.tid < TRT) {
            const int64_t r = r0 + C.tid;
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < NWP; ++w) t += red[w * TRT + C.tid];
            if (r < tg.r_end) yp[(size_t)cc * C.n + r] = t;
        }
}

// The fused sweep's two mat-vecs (A over A(s+1:n, j+1:n), B over the upper part of B) as one
// pool of 256 x 256 items handed out by an atomic counter: a CTA takes its next item as it
// finishes one (the next index is fetched while the current item streams), so the A/B split
// and the last round no longer leave SMs idle (static round-robin did).  Partial sums go to
// yp[cc][r] exactly as before: the result does not depend on which CTA took which item.
// ctr: this sweep's counter (zeroed before the sweep, see the panel loop).
template <class VF>
__device__ void tiled_matvec2(Ctx &C, const TileGeom &ta, const double *XA, int64_t lda_, double *ypA, const TileGeom &tb,
                              const double *XB, int64_t ldb_, double *ypB, VF vf, unsigned *ctr, int res)
{
    const int na = ta.items(), nt = na + tb.items();
    if (C.tid == 0) g_sm.ival[2] = (int)atomicAdd(ctr, 1u);
    __syncthreads();
    int it = g_sm.ival[2];
    while (it < nt) {
        unsigned nxt = 0;
        if (C.tid == 0) nxt = atomicAdd(ctr, 1u);  // in flight while this item streams
        // L2 residency (res >= 0): the first `res` items of the pool B-then-A keep the default
        // policy and stay in the L2 from one column's sweep to the next (their rows are fixed
        // for the panel, their columns move by one per step); all other items are read with the
        // evict-first hint, so the stream does not push the resident ones out.
        if (it < na) sweep_item(C, ta, XA, lda_, vf, ypA, it, res >= 0 && it >= res - (nt - na));
        else sweep_item(C, tb, XB, ldb_, vf, ypB, it - na, res >= 0 && it - na >= res);
        __syncthreads();  // every thread has read g_sm.ival[2]
        if (C.tid == 0) g_sm.ival[2] = (int)nxt;
        __syncthreads();
        it = g_sm.ival[2];
    }
    __syncthreads();
}

// Both fused-sweep row sums of the own rows: f(rl, sum of A's item partials, sum of B's).
// Eight threads per row split the column chunks (all their loads issued at once) and combine
// by a fixed xor-shuffle tree (deterministic); 64 rows per pass.
template <class F>
__device__ __forceinline__ void tiled_sum2(const Ctx &C, const TileGeom &ta, const TileGeom &tb, const double *ya,
                                           const double *yb, F f)
{
    constexpr int SUB = 8, PER = 8;
    const int sub = C.tid & (SUB - 1);
    for (int rl0 = 0; rl0 < C.nr; rl0 += PNT / SUB) {
        const int rl = rl0 + C.tid / SUB;
        const bool ok = rl < C.nr;
        const int64_t r = C.rb0 + rl;
        const int ca = ok ? ta.cc_min((int)((r - ta.r_al) / TRT)) : 0;
        const int cb = ok ? tb.cc_min((int)((r - tb.r_al) / TRT)) : 0;
        double sa = 0.0, sb = 0.0;
        const int nccm = ta.ncc > tb.ncc ? ta.ncc : tb.ncc;
        for (int c0 = 0; c0 < nccm; c0 += SUB * PER) {  // one pass for n <= 16384
            double va[PER], vb[PER];
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int cc = c0 + sub + SUB * e;
                va[e] = (ok && cc >= ca && cc < ta.ncc) ? __ldcg(ya + (size_t)cc * C.n + r) : 0.0;
                vb[e] = (ok && cc >= cb && cc < tb.ncc) ? __ldcg(yb + (size_t)cc * C.n + r) : 0.0;
            }
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                sa += va[e];
                sb += vb[e];
            }
        }
#pragma unroll
        for (int o = 1; o < SUB; o <<= 1) {
            sa += __shfl_xor_sync(0xffffffffu, sa, o);
            sb += __shfl_xor_sync(0xffffffffu, sb, o);
        }
        if (ok && sub == 0) f(rl, sa, sb);
    }
}

__global__ void __launch_bounds__(PNT, 1) panel_kernel(const __grid_constant__ PanelArgs a)
{
    cg::grid_group grid = cg::this_grid();
    Ctx C(a);
    if (threadIdx.x == 0) {  // the solve's hand-over barrier: TB remote arrivals per phase
        const unsigned mb = (unsigned)__cvta_generic_to_shared(&g_sm.mbar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(TB) : "memory");
        const unsigned mb4 = (unsigned)__cvta_generic_to_shared(&g_sm.mbar4);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb4), "r"(C4 - 1) : "memory");  // trsv4 senders
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cg::this_cluster().sync();  // the partner's barrier is initialised before any remote arrive
    const int64_t n = a.n, s0 = a.s0, p0 = C.p0, lda = a.lda;
    double *A = a.A;
    double *U = a.U, *V = a.V, *Y = a.Y, *S = a.S, *T = a.T;
    const int nb = a.nb;
    // S, T cached in shared memory; re-derived from the launch parameters at every use (kept
    // out of registers: the solve's tile loop runs at the 128-register limit)
#define stc (a.solve4 && a.nb <= STC_NB)
#define Ssm (g_dyn + OFF_ST)
#define Tsm (g_dyn + OFF_ST + STC_SZ)
    auto Sg = [&](int i, int c) -> double { return stc ? Ssm[c * (c + 1) / 2 + i] : S[(size_t)c * nb + i]; };
    auto Tget = [&](int i, int c) -> double { return stc ? Tsm[c * (c + 1) / 2 + i] : T[(size_t)c * nb + i]; };
    unsigned epoch = a.epoch;
    int k = 0, failed = 0;
    int nsweep = 0;  // sweeps so far: sweep s uses counter a.sweep_ctr[s & 1]
    if (C.bid == 0 && C.tid == 0) a.sweep_ctr[0] = a.sweep_ctr[1] = 0u;  // grid barriers precede the first sweep
    long long ir_steps = 0, ir_cols = 0, rescales = 0;
    int ffi = 0;  // cursor into the forced-failure list
    const bool prof = a.ptime && C.bid == 0 && C.tid == 0;
    unsigned long long tp = 0ull;
    if (prof) {
        for (int i = 0; i < 16; ++i) g_sm.pt[i] = 0.0;
        tp = gtime();
    }
    auto mark = [&](int bin) {  // shared-memory accumulation: no global round trip per mark
        if (prof) {
            unsigned long long t = gtime();
            g_sm.pt[bin] += (double)(t - tp) * 1e-9;
            tp = t;
        }
    };
    while (k < a.kmax) {
        const int64_t j0 = s0 + k;
        const int ku = k + 1;  // U columns incl. the new u
        C.ph++;
        // ================= P1: update column j of A =========================
        for (int c = C.tid; c < k; c += PNT) g_sm.sv1[c] = (c == k - 1) ? 1.0 : V[(size_t)c * n + j0];
        __syncthreads();
        C.rowgemv(Y, n, k, g_sm.sv1);
        mark(8);
        for (int rl = C.tid; rl < C.nr; rl += PNT) {
            const int64_t r = C.rb0 + rl;
            double a0 = A[(size_t)j0 * lda + r];
            a.vsave[r] = a0;
            g_sm.vloc[rl] = a0 - g_dyn[rl];
        }
        __syncthreads();
        C.coltdot(U, n, k, 0);
        mark(9);
        grid.sync();
        mark(10);
        C.gather(g_sm.sv2, k, 0);
        __syncthreads();
        mark(11);
        if (stc) C.trimv_sm<true>(Ssm, k, g_sm.sv2, g_sm.sv3); else C.trimv<true>(Sg, k, g_sm.sv2, g_sm.sv3);  // sv3 = S^T t
        mark(12);
        C.rowgemv(U, n, k, g_sm.sv3);
        mark(13);
        C.ph++;
        {
            double ss = 0.0;
            for (int rl = C.tid; rl < C.nr; rl += PNT) {
                const int64_t r = C.rb0 + rl;
                double av = g_sm.vloc[rl] - g_dyn[rl];
                a.vx[r] = av;
                if (r <= j0) A[(size_t)j0 * lda + r] = av;  // rows s+1:j of the updated column
                if (r >= j0 + 2) ss += av * av;
                g_sm.vloc[rl] = (r >= j0 + 2) ? av : 0.0;     // a_tail for U^T a_tail
            }
            __syncthreads();
            C.coltdot(U, n, k, 1);
            C.block_reduce_to_part(ss, 0);
        }
        mark(14);
        grid.sync();
        mark(0);
        // ================= P2: left reflector (no barrier needed) ============
        double tau_u, scal_u, beta_u, alpha_u;
        {
            C.gather(g_sm.sv1, k + 1, 0);  // [||a_tail||^2, U^T a_tail]
            __syncthreads();
            const double ss = g_sm.sv1[0];
            alpha_u = __ldcg(&a.vx[j0 + 1]);
            tau_u = 0.0;
            scal_u = 0.0;
            beta_u = alpha_u;
            if (ss > 0.0) {
                double nrm = sqrt(alpha_u * alpha_u + ss);
                beta_u = alpha_u >= 0.0 ? -nrm : nrm;
                tau_u = (beta_u - alpha_u) / beta_u;
                scal_u = 1.0 / (alpha_u - beta_u);
            }
        }
        // U^T u = scal * U^T a_tail + U(j0+1, :)^T   (u(j0+1) = 1)
        for (int c = C.tid; c < k; c += PNT) g_sm.sv2[c] = scal_u * g_sm.sv1[1 + c] + U[(size_t)c * n + j0 + 1];
        __syncthreads();
        if (stc) C.trimv_sm<false>(Ssm, k, g_sm.sv2, g_sm.snew, -tau_u); else C.trimv<false>(Sg, k, g_sm.sv2, g_sm.snew, -tau_u);
        if (C.tid == 0) g_sm.snew[k] = tau_u;
        auto unew = [&](int64_t r) -> double {
            return (r < j0 + 1) ? 0.0 : (r == j0 + 1 ? 1.0 : __ldcg(&a.vx[r]) * scal_u);
        };
        for (int rl = C.tid; rl < C.nr; rl += PNT) {
            const int64_t r = C.rb0 + rl;
            U[(size_t)k * n + r] = unew(r);
            if (r == j0 + 1) A[(size_t)j0 * lda + r] = beta_u;
            else if (r >= j0 + 2) A[(size_t)j0 * lda + r] = 0.0;  // Set A(j+2:n, j) <- 0
        }
        __syncthreads();
        if (C.bid == 0)
            for (int i = C.tid; i <= k; i += PNT) S[(size_t)k * nb + i] = g_sm.snew[i];
        if (stc)
            for (int i = C.tid; i <= k; i += PNT) Ssm[k * (k + 1) / 2 + i] = g_sm.snew[i];
        auto Sget = [&](int i, int c) -> double { return c == k ? g_sm.snew[i] : Sg(i, c); };

        // ================= P3: factored solve ==================================
        for (int c = C.tid; c < ku; c += PNT) g_sm.sv1[c] = (c == k) ? 1.0 : U[(size_t)c * n + j0 + 1];
        __syncthreads();
        if (stc) C.trimv_sm<false>(Ssm, ku, g_sm.sv1, g_sm.sv3); else C.trimv<false>(Sget, ku, g_sm.sv1, g_sm.sv3);  // z2 = S_{k+1} w, w(c) = U(j0+1, c)
        ++epoch;
        if (a.solve4 == 2) trsv4r(a, RhsSpec{nullptr, nullptr, a.vx, j0 + 1, j0 + 1, scal_u}, k, g_sm.sv3, epoch, j0);
        else if (a.solve4) trsv4(C, [&](int64_t r) { return r == j0 + 1 ? 1.0 : 0.0; }, unew, k, g_sm.sv3, epoch);
        else trsv_blocked(C, [&](int64_t r) { return r == j0 + 1 ? 1.0 : 0.0; }, unew, k, g_sm.sv3, epoch, j0);
        grid.sync();
        mark(1);
        int emax = trsv_emax(C);
        if (emax > 0) ++rescales;
        C.ph++;
        for (int rl = C.tid; rl < C.nr; rl += PNT) {
            const int64_t r = C.rb0 + rl;
            int eb = __ldcg(&a.bexp[(r - p0) / C.tbs]);
            g_sm.vloc[rl] = ldexp(__ldcg(&a.vy[r]), eb - emax);
        }
        __syncthreads();
        C.coltdot(V, n, k, 0);
        grid.sync();
        C.gather(g_sm.sv1, k, 0);
        __syncthreads();
        if (stc) C.trimv_sm<true>(Tsm, k, g_sm.sv1, g_sm.sv2); else C.trimv<true>(Tget, k, g_sm.sv1, g_sm.sv2);  // T^T (V^T y~)
        C.rowgemv(V, n, k, g_sm.sv2);
        C.ph++;
        {
            double sx = 0.0, st = 0.0;
            for (int rl = C.tid; rl < C.nr; rl += PNT) {
                const int64_t r = C.rb0 + rl;
                double xv = 0.0;
                if (r >= j0 + 1) {
                    xv = g_sm.vloc[rl] - g_dyn[rl];
                    sx += xv * xv;
                    if (r >= j0 + 2) st += xv * xv;
                }
                a.vx[r] = xv;
                g_sm.vloc[rl] = xv;
            }
            __syncthreads();
            C.coltdot(V, n, k, 2);
            C.block_reduce_to_part(sx, 0);
            C.block_reduce_to_part(st, 1);
        }
        grid.sync();
        mark(2);
        double xnorm2 = 0.0, xtail2 = 0.0;
        C.gather(g_sm.sv1, 2, 0);
        __syncthreads();
        xnorm2 = g_sm.sv1[0];
        xtail2 = g_sm.sv1[1];
        __syncthreads();

        // ================= P4: residual + iterative refinement ================
        // One HBM sweep per solve serves both P4 and P5: with x known,
        //   A x over A(s+1:n, j+1:n)   -> P5's A v = A e_{j+1} + scal (A x - A e_{j+1} x_{j+1})
        //   B x over B(s+1:n, j+1:n)   -> the residual's B w = B x - (B V)(T V^T x)
        // where B V is kept column by column (B v = B e_{j+1} + scal (B x - B e_{j+1} x_{j+1})).
        // If IR corrects x, the sweep is redone for the new x (the A half is then speculative).
        bool accepted = (k == 0);  // k = 0: stable solve, no test (reading R-Z4)
        bool forced = false;
        while (ffi < a.n_force_fail && a.force_fail[ffi] < j0) ++ffi;
        if (ffi < a.n_force_fail && a.force_fail[ffi] == j0 && k > 0) forced = true;
        int ir = 0;
        bool this_col_ir = false;
        const TileGeom tga(p0, n, j0 + 1, n, false);  // A(s+1:n, j+1:n)
        const TileGeom tgb(p0, n, j0 + 1, n, true);   // B(s+1:n, j+1:n), upper part
        while (true) {
            C.gather(g_sm.svx, k, 2);  // V^T x
            __syncthreads();
            if (k > 0) { if (stc) C.trimv_sm<false>(Tsm, k, g_sm.svx, g_sm.sv2); else C.trimv<false>(Tget, k, g_sm.svx, g_sm.sv2); }  // z = T V^T x
            mark(6);
            if (C.bid == 0 && C.tid == 0) a.sweep_ctr[(nsweep + 1) & 1] = 0u;  // the next sweep's counter
            tiled_matvec2(C, tga, A, lda, a.ypart, tgb, a.B, a.ldb, a.ypartB,
                          [&](int64_t c) { return __ldcg(&a.vx[c]); }, a.sweep_ctr + (nsweep & 1), a.sweep_res);
            ++nsweep;
            grid.sync();
            mark(4);
            if (k > 0) C.rowgemv(a.BV, n, k, g_sm.sv2);  // (B V) z for own rows
            tiled_sum2(C, tga, tgb, a.ypart, a.ypartB, [&](int rl, double ax, double bx) {
                const int64_t r = C.rb0 + rl;
                a.vw[r] = ax;
                a.vbx[r] = bx;
                if (k > 0) {
                    const double w2 = bx - g_dyn[rl];  // w2 = B w
                    a.vw2[r] = w2;
                    g_sm.vloc[rl] = w2;
                }
            });
            if (accepted) break;  // k = 0
            __syncthreads();
            C.ph++;
            C.coltdot(U, n, ku, 0);  // partial U^T w2
            grid.sync();
            mark(7);
            // r = sigma e1 - ((I - U S^T U^T) w2)(j0+1:)
            C.gather(g_sm.sv1, ku, 0);
            __syncthreads();
            if (stc) C.trimv_sm<true>(Ssm, ku, g_sm.sv1, g_sm.sv2); else C.trimv<true>(Sget, ku, g_sm.sv1, g_sm.sv2);  // S_{k+1}^T t
            C.rowgemv(U, n, ku, g_sm.sv2);
            C.ph++;
            const double sigma = ldexp(1.0, -emax);
            {
                double sr = 0.0;
                for (int rl = C.tid; rl < C.nr; rl += PNT) {
                    const int64_t r = C.rb0 + rl;
                    double rv = 0.0;
                    if (r >= j0 + 1) {
                        rv = (r == j0 + 1 ? sigma : 0.0) - (__ldcg(&a.vw2[r]) - g_dyn[rl]);
                        sr += rv * rv;
                    }
                    a.vr[r] = rv;
                    g_sm.vloc[rl] = rv;
                }
                __syncthreads();
                C.coltdot(U, n, ku, 1);
                C.block_reduce_to_part(sr, 0);
            }
            grid.sync();
            C.gather(g_sm.sv1, 1, 0);
            __syncthreads();
            const double rn = sqrt(g_sm.sv1[0]), xn = sqrt(xnorm2);
            __syncthreads();
            if (a.dbg && C.bid == 0 && C.tid == 0 && ir < 12) a.dbg[j0 * 12 + ir] = rn / (a.tol * xn);
            if (!forced && rn <= a.tol * xn && isfinite(rn)) {
                accepted = true;
                break;
            }
            if (forced || ir >= a.max_ir) break;  // IR failed
            // ---- IR correction: solve B~22 c = r with the same factored solve ----
            ++ir;
            ++ir_steps;
            this_col_ir = true;
            C.gather(g_sm.sv1, ku, 1);  // U^T r_ext
            __syncthreads();
            if (stc) C.trimv_sm<false>(Ssm, ku, g_sm.sv1, g_sm.sv3); else C.trimv<false>(Sget, ku, g_sm.sv1, g_sm.sv3);  // S_{k+1} (U^T r)
            ++epoch;
            // (vx now holds x, so the new column of U is read back from U(:, k), written in P2)
            if (a.solve4 == 2)
                trsv4r(a, RhsSpec{a.vr, U + (size_t)k * n, nullptr, 0, 0, 0.0}, k, g_sm.sv3, epoch, -1);
            else if (a.solve4)
                trsv4(C, [&](int64_t r) { return __ldcg(&a.vr[r]); },
                      [&](int64_t r) { return __ldcg(&U[(size_t)k * n + r]); }, k, g_sm.sv3, epoch);
            else
                trsv_blocked(C, [&](int64_t r) { return __ldcg(&a.vr[r]); },
                             [&](int64_t r) { return __ldcg(&U[(size_t)k * n + r]); }, k, g_sm.sv3, epoch, -1);
            grid.sync();
            const int ec = trsv_emax(C);
            if (ec > 0) { ++rescales; break; }  // a rescaled correction counts as IR failure
            C.ph++;
            for (int rl = C.tid; rl < C.nr; rl += PNT) g_sm.vloc[rl] = __ldcg(&a.vy[C.rb0 + rl]);
            __syncthreads();
            C.coltdot(V, n, k, 0);
            grid.sync();
            C.gather(g_sm.sv1, k, 0);
            __syncthreads();
            if (stc) C.trimv_sm<true>(Tsm, k, g_sm.sv1, g_sm.sv2); else C.trimv<true>(Tget, k, g_sm.sv1, g_sm.sv2);
            C.rowgemv(V, n, k, g_sm.sv2);
            C.ph++;
            {
                double sx = 0.0, st = 0.0;
                for (int rl = C.tid; rl < C.nr; rl += PNT) {
                    const int64_t r = C.rb0 + rl;
                    double xv = 0.0;
                    if (r >= j0 + 1) {
                        xv = __ldcg(&a.vx[r]) + (g_sm.vloc[rl] - g_dyn[rl]);
                        sx += xv * xv;
                        if (r >= j0 + 2) st += xv * xv;
                    }
                    a.vx[r] = xv;
                    g_sm.vloc[rl] = xv;
                }
                __syncthreads();
                C.coltdot(V, n, k, 2);
                C.block_reduce_to_part(sx, 0);
                C.block_reduce_to_part(st, 1);
            }
            grid.sync();
            C.gather(g_sm.sv1, 2, 0);
            __syncthreads();
            xnorm2 = g_sm.sv1[0];
            xtail2 = g_sm.sv1[1];
            __syncthreads();
        }
        mark(3);
        if (this_col_ir) ++ir_cols;
        if (C.bid == 0 && C.tid == 0)
            a.irtrace[j0] = (accepted ? 0 : 1000) + (a.irtrace[j0] >= 1000 ? 1000 : 0) + ir;
        if (!accepted) {
            // undo the left reflector: restore column j of A (Algorithm 1)
            for (int rl = C.tid; rl < C.nr; rl += PNT) A[(size_t)j0 * lda + C.rb0 + rl] = a.vsave[C.rb0 + rl];
            failed = 1;
            break;
        }
        // ================= P5: right reflector, T, Y (no sweep, no grid barrier) ==========
        double gam, scal_v;
        const double x1 = __ldcg(&a.vx[j0 + 1]);
        {
            gam = 0.0;
            scal_v = 0.0;
            if (xtail2 > 0.0) {
                double nrm = sqrt(x1 * x1 + xtail2);
                double bet = x1 >= 0.0 ? -nrm : nrm;
                gam = (bet - x1) / bet;
                scal_v = 1.0 / (x1 - bet);
            }
        }
        // V^T v = V(j+1,:)^T + scal (V^T x - V(j+1,:)^T x_{j+1})   (v = [1; scal x(j+2:n)])
        for (int c = C.tid; c < k; c += PNT) {
            const double vj = V[(size_t)c * n + j0 + 1];
            g_sm.sv1[c] = vj + scal_v * (g_sm.svx[c] - vj * x1);
        }
        __syncthreads();
        if (C.bid == 0 || stc) {  // every CTA keeps its copy of T (all compute the new column)
            if (stc) C.trimv_sm<false>(Tsm, k, g_sm.sv1, g_sm.sv2, -gam); else C.trimv<false>(Tget, k, g_sm.sv1, g_sm.sv2, -gam);
            if (C.bid == 0) {
                for (int i = C.tid; i < k; i += PNT) T[(size_t)k * nb + i] = g_sm.sv2[i];
                if (C.tid == 0) T[(size_t)k * nb + k] = gam;
            }
            if (stc) {
                for (int i = C.tid; i < k; i += PNT) Tsm[k * (k + 1) / 2 + i] = g_sm.sv2[i];
                if (C.tid == 0) Tsm[k * (k + 1) / 2 + k] = gam;
            }
        }
        C.rowgemv(Y, n, k, g_sm.sv1);
        for (int rl = C.tid; rl < C.nr; rl += PNT) {
            const int64_t r = C.rb0 + rl;
            V[(size_t)k * n + r] = (r < j0 + 1) ? 0.0 : (r == j0 + 1 ? 1.0 : __ldcg(&a.vx[r]) * scal_v);
            const double acol = A[(size_t)(j0 + 1) * lda + r];
            const double av = acol + scal_v * (a.vw[r] - acol * x1);                 // A v
            const double bcol = (r <= j0 + 1) ? a.B[(size_t)(j0 + 1) * a.ldb + r] : 0.0;
            a.BV[(size_t)k * n + r] = bcol + scal_v * (a.vbx[r] - bcol * x1);        // B v
            Y[(size_t)k * n + r] = gam * (av - g_dyn[rl]);
        }
        ++k;
        __syncthreads();
        mark(5);
    }
#undef stc
#undef Ssm
#undef Tsm
    grid.sync();
    if (prof)
        for (int i = 0; i < 16; ++i) a.ptime[i] += g_sm.pt[i];
    if (C.bid == 0 && C.tid == 0) {
        a.out[0] = k;
        a.out[1] = failed;
        a.out[2] = ir_steps;
        a.out[3] = ir_cols;
        a.out[4] = rescales;
        a.out[5] = epoch;
    }
}

// Inverse of each TB x TB diagonal block of B(p0:n, p0:n) (column-major, ld TB) and a
// safety flag: finite, max|inv| <= 2^200, and max|inv| * max|D| <= 4e3 (well-conditioned, so the
// look-ahead block solve stays backward stable to ~4e3 u) (else the
// panel uses the overflow-safe sequential substitution for that block).
constexpr int IDT = 512;                    // inv_diag_kernel threads: 128 rows x 4 column groups
constexpr int TRI = TB * (TB + 1) / 2;      // packed upper triangle, P(i, j) = j (j + 1) / 2 + i
__global__ void __launch_bounds__(IDT) inv_diag_kernel(const double *B, int64_t ldb, int64_t p0, int64_t n,
                                                       double *Dinv, int *dsafe)
{
    // Column j of X = D^{-1} by back substitution on e_j (for l = j .. 0: x_l /= D_ll, then
    // x_i -= D_il x_l for i < l), all columns in lock step over l: D and X as packed upper
    // triangles in shared memory, thread (i, jg) owns row i of the columns j = jg mod 4 in the
    // updates, and the scaled row l of X goes through a shared row (two barriers per l).
    // Every x_i(j) sees the same operations in the same order as the column-by-column
    // substitution (bitwise the same inverse).
    extern __shared__ __align__(16) double X[];
    double *Dp = X, *Xp = X + TRI;
    __shared__ double rowl[TB];
    __shared__ double smax[2][IDT / 32];
    const int b = blockIdx.x, tid = threadIdx.x, i = tid % TB, jg = tid / TB;
    const int64_t r0 = p0 + (int64_t)b * TB;
    const int h = (int)(n - r0 < TB ? n - r0 : TB);
    const double *D = B + r0 + r0 * ldb;
    double dmax = 0.0;
    {
        constexpr int JU = TB / (IDT / TB);  // columns per thread: all loads before any store
        double dv[JU];
#pragma unroll
        for (int u = 0; u < JU; ++u) {
            const int j = jg + (IDT / TB) * u;
            dv[u] = (i <= j && j < h) ? D[(size_t)j * ldb + i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < JU; ++u) {
            const int j = jg + (IDT / TB) * u;
            if (i > j) continue;
            dmax = fmax(dmax, fabs(dv[u]));
            Dp[j * (j + 1) / 2 + i] = dv[u];
            Xp[j * (j + 1) / 2 + i] = (i == j && j < h) ? 1.0 : 0.0;
        }
    }
    __syncthreads();
    // per l: (a) row l of X is final up to its scaling: x_l(j) /= D_ll for all j in [l, h), one
    // column per thread (the divisions run in parallel), the scaled row also to rowl; (b) rank-1
    // update of the rows i < l with it.  Two barriers per l.
    for (int l = h - 1; l >= 0; --l) {
        const double dl = Dp[l * (l + 1) / 2 + l];
        for (int j = l + tid; j < h; j += IDT) {
            const double x = Xp[j * (j + 1) / 2 + l] / dl;
            Xp[j * (j + 1) / 2 + l] = x;
            rowl[j] = x;
        }
        __syncthreads();
        if (i < l) {
            const double dil = Dp[l * (l + 1) / 2 + i];
            int j = l + ((jg - l) % 4 + 4) % 4;
            for (; j + 12 < h; j += 16) {  // four columns per round: loads ahead of the stores
                double xl[4], xv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    xl[u] = rowl[j + 4 * u];
                    xv[u] = Xp[(j + 4 * u) * (j + 4 * u + 1) / 2 + i];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (xl[u] != 0.0) Xp[(j + 4 * u) * (j + 4 * u + 1) / 2 + i] = xv[u] - dil * xl[u];
            }
            for (; j < h; j += 4) {
                const double xl = rowl[j];
                if (xl != 0.0) Xp[j * (j + 1) / 2 + i] -= dil * xl;
            }
        }
        __syncthreads();
    }
    double imax = 0.0;
    bool fin = true;
    double *out = Dinv + (size_t)b * TB * TB;
    for (int j = jg; j < TB; j += IDT / TB) {
        const double v = (i <= j) ? Xp[j * (j + 1) / 2 + i] : 0.0;
        if (!isfinite(v)) fin = false;
        imax = fmax(imax, fabs(v));
        out[(size_t)j * TB + i] = v;
    }
    if (!fin) imax = INFINITY;
    double a1 = warp_max(imax), a2 = warp_max(dmax);
    if ((tid & 31) == 0) {
        smax[0][tid >> 5] = a1;
        smax[1][tid >> 5] = a2;
    }
    __syncthreads();
    if (tid == 0) {
        double im = 0.0, dm = 0.0;
        for (int w = 0; w < IDT / 32; ++w) {
            im = fmax(im, smax[0][w]);
            dm = fmax(dm, smax[1][w]);
        }
        dsafe[b] = (isfinite(im) && im <= 0x1p200 && im * dm <= 4e3) ? 1 : 0;
    }
}

// trsv4 set-up: Dinv4_b = [[Dinv_2b, X], [0, Dinv_2b+1]] (ld T4) with X = -Dinv_2b B_{2b,2b+1}
// Dinv_2b+1 formed by two GEMMs afterwards; this kernel writes the diagonal quadrants and zeros
// the rest (the lower-left quadrant doubles as the GEMMs' scratch and is zeroed again by
// inv4_safety_kernel).
constexpr int I4T = 1024, I4U = 16;  // inv4 kernels: threads, elements per thread and round
__global__ void __launch_bounds__(I4T) inv4_assemble_kernel(const double *__restrict__ Dinv, int Nb,
                                                            double *__restrict__ Dinv4)
{
    const int b4 = blockIdx.x, i0 = 2 * b4;
    double *D = Dinv4 + (size_t)b4 * T4 * T4;
    for (int base = 0; base < T4 * T4; base += I4T * I4U) {
        double v[I4U];
#pragma unroll
        for (int u = 0; u < I4U; ++u) {  // all loads of a round in flight
            const int idx = base + u * I4T + threadIdx.x, r = idx % T4, c = idx / T4;
            v[u] = 0.0;
            if (r < TB && c < TB) v[u] = Dinv[(size_t)i0 * TB * TB + (size_t)c * TB + r];
            else if (r >= TB && c >= TB && i0 + 1 < Nb) v[u] = Dinv[(size_t)(i0 + 1) * TB * TB + (size_t)(c - TB) * TB + (r - TB)];
        }
#pragma unroll
        for (int u = 0; u < I4U; ++u) D[base + u * I4T + threadIdx.x] = v[u];
    }
}
// Safety of each 256-row block (the criterion of inv_diag_kernel on the whole block) and the
// final zeroing of the scratch quadrant.
__global__ void __launch_bounds__(I4T) inv4_safety_kernel(const double *__restrict__ B, int64_t ldb, int64_t p0,
                                                          int64_t n, double *__restrict__ Dinv4, const int *dsafe, int Nb,
                                                          int *dsafe4)
{
    __shared__ double sm[2][I4T / 32];
    const int b4 = blockIdx.x, i0 = 2 * b4, tid = threadIdx.x;
    const int64_t r0 = p0 + (int64_t)b4 * T4;
    const int h = (int)(n - r0 < T4 ? n - r0 : T4);
    double *D = Dinv4 + (size_t)b4 * T4 * T4;
    double im = 0.0, dm = 0.0;
    bool fin = true;
    for (int base = 0; base < T4 * T4; base += I4T * I4U) {
        double v[I4U], bv[I4U];
#pragma unroll
        for (int u = 0; u < I4U; ++u) {  // all loads of a round in flight
            const int idx = base + u * I4T + tid, r = idx % T4, c = idx / T4;
            v[u] = (r >= TB && c < TB) ? 0.0 : D[idx];
            bv[u] = (r < h && c < h && r <= c) ? B[(size_t)(r0 + c) * ldb + r0 + r] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < I4U; ++u) {
            const int idx = base + u * I4T + tid, r = idx % T4, c = idx / T4;
            if (r >= TB && c < TB) D[idx] = 0.0;  // scratch quadrant
            else {
                if (!isfinite(v[u])) fin = false;
                im = fmax(im, fabs(v[u]));
            }
            dm = fmax(dm, fabs(bv[u]));
        }
    }
    if (!fin) im = INFINITY;
    im = warp_max(im);
    dm = warp_max(dm);
    if ((tid & 31) == 0) {
        sm[0][tid >> 5] = im;
        sm[1][tid >> 5] = dm;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0.0, d = 0.0;
        for (int w = 0; w < I4T / 32; ++w) {
            a = fmax(a, sm[0][w]);
            d = fmax(d, sm[1][w]);
        }
        const bool ok = dsafe[i0] && (i0 + 1 >= Nb || dsafe[i0 + 1]);
        dsafe4[b4] = (ok && isfinite(a) && a <= 0x1p200 && a * d <= 4e3) ? 1 : 0;
    }
}

}  // namespace

int ht_panel_max_blocks(int *nblocks_out)
{
    int dev = 0, nsm = 0, per = 0;
    HT_CUDA_TRY(cudaGetDevice(&dev));
    HT_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    HT_CUDA_TRY(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     DYN_DOUBLES * (int)sizeof(double)));
    HT_CUDA_TRY(cudaFuncSetAttribute(inv_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     2 * TRI * (int)sizeof(double)));
    HT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, panel_kernel, PNT,
                                                              DYN_DOUBLES * sizeof(double)));
    if (per < 1) return 4;
    *nblocks_out = nsm;
    return 0;
}

// L2 persisting window for `bytes` of panel workspace: sets the device's persisting carve-out
// once (min(bytes, 3/8 of L2, the device maximum)) and returns the window size and hit ratio.
// Off by default since the fused sweep reads with the evict-first hint (the workspace then stays
// in the L2 without a carve-out, and the absorption keeps the whole L2: cfg3 2.702 -> 2.690 s);
// HT_L2PERSIST=1 (development) enables it.
int ht_l2_persist_window(size_t bytes, size_t *win, float *hit)
{
    const bool off = getenv("HT_L2PERSIST") == nullptr;  // read per call (tests toggle it)
    *win = 0;
    *hit = 0.f;
    if (off) return 0;
    int dev = 0, l2 = 0, maxp = 0, maxw = 0;
    HT_CUDA_TRY(cudaGetDevice(&dev));
    HT_CUDA_TRY(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    HT_CUDA_TRY(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
    HT_CUDA_TRY(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev));
    if (maxp <= 0 || maxw <= 0) return 0;
    const size_t carve = std::min<size_t>({(size_t)l2 / 8 * 3, (size_t)maxp, bytes});
    static std::mutex mu;
    static size_t have[64] = {0};
    {
        std::lock_guard<std::mutex> lk(mu);
        if (have[dev & 63] < carve) {
            HT_CUDA_TRY(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
            have[dev & 63] = carve;
        }
    }
    *win = std::min<size_t>(bytes, (size_t)maxw);
    *hit = (float)std::min(1.0, (double)carve / (double)*win);
    return 0;
}

int ht_panel_run(cudaStream_t st, PanelArgs *a, int nblocks)
{
    const int64_t M = a->n - a->s0 - 1;
    const int Nb = (int)((M + TB - 1) / TB);
    inv_diag_kernel<<<Nb, IDT, 2 * TRI * sizeof(double), st>>>(a->B, a->ldb, a->s0 + 1, a->n, a->Dinv, a->dsafe);
    HT_CUDA_TRY(cudaGetLastError());
    // The 256-row solve on 4-CTA clusters (trsv4) when every 256-row diagonal block is safe
    // (decided on the host: one small copy per panel), else the 128-row paired solve.
    static const bool no4 = getenv("HT_NO_TRSV4") != nullptr;  // development: force the 128-row solve
    static const bool nocl = getenv("HT_PANEL_NOCLUSTER") != nullptr;
    const int Nb4 = (int)((M + T4 - 1) / T4);
    a->solve4 = 0;
    {
        // Fused sweep: a panel whose per-column stream (A block + B's upper part, ~1.5 M^2
        // doubles) exceeds the L2 keeps only a fixed part of it resident (ht_panel.cu
        // tiled_matvec2); HT_SWEEP_RES_MB sets that part (default 0: every item evict-first; < 0: no hints).
        const char *e = getenv("HT_SWEEP_RES_MB");
        const double mb = e ? atof(e) : 0.0;
        a->sweep_res = mb < 0 ? -1 : (int)(mb * 1e6 / (8.0 * 256 * 256));
    }
    int ncl4 = 0;
    const bool cl4 = getenv("HT_TRSV4_CLUSTER") != nullptr;  // read per panel (tests toggle it)
    bool use4 = false;  // the 256-row solve is possible (trsv4r needs no clusters; trsv4 needs 4-CTA ones)
    if (!no4 && Nb4 >= 2 && a->Dinv4 && !(cl4 && nocl)) use4 = true;
    if (use4 && cl4) {
        cudaLaunchConfig_t oc = {};
        oc.gridDim = dim3((unsigned)(nblocks & ~(C4 - 1)));
        oc.blockDim = dim3(PNT);
        oc.dynamicSmemBytes = DYN_DOUBLES * sizeof(double);
        cudaLaunchAttribute oat[1];
        oat[0].id = cudaLaunchAttributeClusterDimension;
        oat[0].val.clusterDim.x = C4;
        oat[0].val.clusterDim.y = 1;
        oat[0].val.clusterDim.z = 1;
        oc.attrs = oat;
        oc.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&ncl4, panel_kernel, &oc) != cudaSuccess) {
            cudaGetLastError();
            ncl4 = 0;
        }
        use4 = ncl4 >= 2;
    }
    if (use4) {
        inv4_assemble_kernel<<<Nb4, I4T, 0, st>>>(a->Dinv, Nb, a->Dinv4);
        HT_CUDA_TRY(cudaGetLastError());
        std::vector<GemmBatchItem> g1, g2;
        for (int b4 = 0; b4 < Nb4; ++b4) {
            const int i0 = 2 * b4;
            if (i0 + 1 >= Nb) continue;
            const int64_t r0 = a->s0 + 1 + (int64_t)i0 * TB, c0 = r0 + TB;
            const int w1 = (int)std::min<int64_t>(TB, a->n - c0);
            double *D = a->Dinv4 + (size_t)b4 * T4 * T4;
            // W = B_{i0,i0+1} Dinv_{i0+1} into the lower-left quadrant; X = -Dinv_{i0} W (upper right)
            g1.push_back(GemmBatchItem{a->B + r0 + c0 * a->ldb, a->Dinv + (size_t)(i0 + 1) * TB * TB, D + TB, a->ldb, TB, T4,
                                       TB, w1, w1, 1.0, 0.0, 0.0});
            g2.push_back(GemmBatchItem{a->Dinv + (size_t)i0 * TB * TB, D + TB, D + (size_t)TB * T4, TB, T4, T4, TB, w1, TB,
                                       -1.0, 0.0, 0.0});
        }
        if (!g1.empty()) {
            int rc = ht_gemm_multi(st, 'N', 'N', g1.data(), (int)g1.size());
            if (rc) return rc;
            rc = ht_gemm_multi(st, 'N', 'N', g2.data(), (int)g2.size());
            if (rc) return rc;
        }
        inv4_safety_kernel<<<Nb4, I4T, 0, st>>>(a->B, a->ldb, a->s0 + 1, a->n, a->Dinv4, a->dsafe, Nb, a->dsafe4);
        HT_CUDA_TRY(cudaGetLastError());
        HT_CUDA_TRY(cudaMemcpyAsync(a->h_dsafe4, a->dsafe4, Nb4 * sizeof(int), cudaMemcpyDeviceToHost, st));
        HT_CUDA_TRY(cudaStreamSynchronize(st));
        bool all = true;
        for (int b4 = 0; b4 < Nb4; ++b4) all = all && a->h_dsafe4[b4] != 0;
        // the row-split solve (trsv4r, default) needs no clusters; HT_TRSV4_CLUSTER=1 (development)
        // selects the 4-CTA cluster variant (trsv4)
        a->solve4 = all ? (cl4 ? 1 : 2) : 0;
    }
    if (a->solve4) {
        // Bt = Dinv4_b B(block b, blocks > b), block rows of T4 rows packed with ld T4
        std::vector<GemmBatchItem> it;
        for (int b4 = 0; b4 + 1 < Nb4; ++b4) {
            const int64_t r0 = a->s0 + 1 + (int64_t)b4 * T4, c0 = r0 + T4;
            const int w = (int)(a->n - c0);
            it.push_back(GemmBatchItem{a->Dinv4 + (size_t)b4 * T4 * T4, a->B + r0 + c0 * a->ldb, a->Bt + bt4_row_offset(M, b4),
                                       T4, a->ldb, T4, T4, w, T4, 1.0, 0.0, 0.0});
        }
        int rc = ht_gemm_multi(st, 'N', 'N', it.data(), (int)it.size());
        if (rc) return rc;
        for (const auto &x : it) g_ht_flops -= 2.0 * TB * (double)TB * x.N;  // the zero lower-left quadrant of Dinv4
    } else if (Nb > 1) {
        // Bt(block b, blocks > b) = Dinv_b * B(block b, blocks > b): pre-scaled block rows, packed
        // (bt_row_offset, ld TB: every TB x TB tile contiguous)
        a->ldbt = TB;
        std::vector<GemmBatchItem> it;
        for (int b = 0; b + 1 < Nb; ++b) {
            const int64_t r0 = a->s0 + 1 + (int64_t)b * TB, c0 = r0 + TB;
            const int w = (int)(a->n - c0);
            it.push_back(GemmBatchItem{a->Dinv + (size_t)b * TB * TB, a->B + r0 + c0 * a->ldb, a->Bt + bt_row_offset(M, b),
                                       TB, a->ldb, TB, TB, w, TB, 1.0, 0.0, 0.0});
        }
        int rc = ht_gemm_multi(st, 'N', 'N', it.data(), (int)it.size());
        if (rc) return rc;
    }
    a->ldbt = TB;
    // cooperative launch (grid barriers) in clusters of 2 CTAs (the solve hands blocks over
    // through distributed shared memory); the grid is even.  HT_PANEL_NOCLUSTER=1 (profiling
    // only: ncu cannot replay cooperative cluster launches) runs unpaired single CTAs.
    const int csz = a->solve4 == 1 ? C4 : 2;
    if (!nocl) {
        nblocks &= ~(csz - 1);
        if (a->solve4 == 1 && nblocks > C4 * ncl4) nblocks = C4 * ncl4;
        if (nblocks < csz) nblocks = csz;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nblocks);
    cfg.blockDim = dim3(PNT);
    cfg.dynamicSmemBytes = DYN_DOUBLES * sizeof(double);
    cfg.stream = st;
    cudaLaunchAttribute at[3];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = (unsigned)csz;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = nocl ? 1 : 2;
    // The panel's small arrays (U, V, Y, B V, S, T, n-vectors; one allocation) are re-read by
    // every column's latency-bound phases while the fused sweep streams ~0.5 GB of A and B per
    // column (and the side streams stream A, Q, Z): an L2-persisting access-policy window keeps
    // them on chip.  The persisting carve-out is sized once per device (at most 3/8 of L2).
    size_t win = 0;
    float hit = 0.f;
    if (a->hot && a->hot_bytes && ht_l2_persist_window(a->hot_bytes, &win, &hit) == 0 && win > 0) {
        at[cfg.numAttrs].id = cudaLaunchAttributeAccessPolicyWindow;
        at[cfg.numAttrs].val.accessPolicyWindow.base_ptr = a->hot;
        at[cfg.numAttrs].val.accessPolicyWindow.num_bytes = win;
        at[cfg.numAttrs].val.accessPolicyWindow.hitRatio = hit;
        at[cfg.numAttrs].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at[cfg.numAttrs].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.numAttrs++;
    }
    HT_CUDA_TRY(cudaLaunchKernelEx(&cfg, panel_kernel, *a));
    return 0;
}
