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
// Every phase boundary is a grid-wide barrier (cooperative launch); the
// triangular solve is a flag-chained block back-substitution with per-block
// power-of-two exponents (overflow-safe, reading R-Z8), so the IR loop and the
// fallback are decided on the device without host round trips.
#include <cooperative_groups.h>
#include "ht_common.cuh"
#include "ht_internal.h"

namespace cg = cooperative_groups;

namespace {

constexpr int PNT = 512;   // threads per CTA
constexpr int NWP = PNT / 32;
constexpr int TB = 64;     // triangular-solve block size
constexpr int NBMAX = 256; // max panel width supported
constexpr double BIG = 0x1p256;

struct __align__(16) PanelSmem {
    double sv1[NBMAX + 1];
    double sv2[NBMAX + 1];
    double sv3[NBMAX + 1];
    double snew[NBMAX + 1];  // new column of S
    double red[32];
    double accg[8][TB];
    double D[TB][TB + 1];    // diagonal block of B (trsv)
    double rhs[TB];
    int ival[4];
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct Ctx {
    const PanelArgs &a;
    PanelSmem &sm;
    int G, bid, tid, lane, warp;
    int64_t n, p0, M, rb0, rb1;
    double *part[2];
    int ph;
    __device__ Ctx(const PanelArgs &aa, PanelSmem &s) : a(aa), sm(s)
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
        rb1 = rb0 + RB < n ? rb0 + RB : n;
        if (rb0 > n) rb0 = n;
        part[0] = a.part;
        part[1] = a.part + (size_t)G * a.pw;
        ph = 0;
    }
    __device__ double *mypart() { return part[ph & 1] + (size_t)bid * a.pw; }
    __device__ double *curpart() { return part[ph & 1]; }
    // out[c] = sum_{r in [rb0,rb1)} X(r,c) * vec(r)   (c < ncols), into mypart()[off + c]
    template <class F>
    __device__ void rows_tdot(const double *X, int64_t ldx, int ncols, F vec, int off)
    {
        double *out = mypart() + off;
        for (int c = warp; c < ncols; c += NWP) {
            double s = 0.0;
            for (int64_t r = rb0 + lane; r < rb1; r += 32) s += X[(size_t)c * ldx + r] * vec(r);
            s = warp_sum(s);
            if (lane == 0) out[c] = s;
        }
    }
    // after a grid sync: dst[c] = sum_b part[b][off + c]  (fixed order: deterministic)
    __device__ void gather(double *dst, int ncols, int off)
    {
        const double *pp = curpart();
        for (int c = tid; c < ncols; c += PNT) {
            double s = 0.0;
            for (int b = 0; b < G; ++b) s += pp[(size_t)b * a.pw + off + c];
            dst[c] = s;
        }
    }
    __device__ double block_reduce_to_part(double v, int off)
    {
        double s = block_sum(v, sm.red);
        if (tid == 0) mypart()[off] = s;
        return s;
    }
};

// ---------------------------------------------------------------------------
// Overflow-safe block back-substitution  y~ = B(p0:n, p0:n)^{-1} rhs.
// Block b (TB rows, from the top) is owned by CTA (Nb-1-b) mod G and published
// through flags[b] = epoch with exponent bexp[b]: true y~ = 2^bexp[b] * vy.
// rhs(r) = base(r) - U(r, 0:ku) z2 is formed on the fly.
template <class BaseF>
__device__ void trsv_scaled(Ctx &C, BaseF base, int ku, const double *z2, unsigned epoch)
{
    const PanelArgs &a = C.a;
    PanelSmem &sm = C.sm;
    const int64_t n = C.n, p0 = C.p0, M = C.M;
    const int Nb = (int)((M + TB - 1) / TB);
    const int ri = C.tid & (TB - 1), grp = C.tid >> 6;  // 64 rows x 8 column groups
    for (int b = Nb - 1 - C.bid; b >= 0; b -= C.G) {
        const int64_t r0 = p0 + (int64_t)b * TB;
        const int h = (int)(n - r0 < TB ? n - r0 : TB);
        double acc = 0.0;
        int Eacc = 0;
        for (int cb = Nb - 1; cb > b; --cb) {
            const int64_t c0 = p0 + (int64_t)cb * TB;
            const int w = (int)(n - c0 < TB ? n - c0 : TB);
            if (C.tid == 0) {
                while (ld_acquire(&a.flags[cb]) != epoch) {
                }
                __threadfence();
                sm.ival[0] = __ldcg(&a.bexp[cb]);
            }
            __syncthreads();
            const int ecb = sm.ival[0];
            if (ecb > Eacc) {
                acc = ldexp(acc, Eacc - ecb);
                Eacc = ecb;
            }
            const double scl = ldexp(1.0, ecb - Eacc);
            if (ri < h) {
                const double *bp = a.B + (size_t)c0 * a.ldb + r0 + ri;
                double s = 0.0;
                for (int cc = grp; cc < w; cc += 8) s += bp[(size_t)cc * a.ldb] * __ldcg(&a.vy[c0 + cc]);
                acc += s * scl;
            }
            __syncthreads();
        }
        sm.accg[grp][ri] = acc;
        // stage the diagonal block
        for (int idx = C.tid; idx < TB * TB; idx += PNT) {
            int i = idx & (TB - 1), j = idx >> 6;
            sm.D[i][j] = (i < h && j < h && i <= j) ? a.B[(size_t)(r0 + j) * a.ldb + r0 + i] : 0.0;
        }
        __syncthreads();
        if (C.tid < TB) {
            double s = 0.0;
            for (int g = 0; g < 8; ++g) s += sm.accg[g][C.tid];
            double rv = 0.0;
            if (C.tid < h) {
                const int64_t r = r0 + C.tid;
                double u = 0.0;
                for (int c = 0; c < ku; ++c) u += a.U[(size_t)c * n + r] * z2[c];
                rv = ldexp(base(r) - u, -Eacc) - s;
            }
            sm.rhs[C.tid] = rv;
        }
        __syncthreads();
        if (C.warp == 0) {
            const int l = C.lane;
            double v0 = sm.rhs[l], v1 = sm.rhs[l + 32];
            int e = Eacc;
            for (int c = h - 1; c >= 0; --c) {
                const int own = c & 31, hi = c >> 5;
                double mine = hi ? v1 : v0;
                double xc = __shfl_sync(0xffffffffu, mine, own) / sm.D[c][c];
                if (!(fabs(xc) <= BIG)) {  // rescale everything by 2^-ex (exact)
                    int ex;
                    frexp(xc, &ex);
                    v0 = ldexp(v0, -ex);
                    v1 = ldexp(v1, -ex);
                    e += ex;
                    mine = hi ? v1 : v0;
                    xc = __shfl_sync(0xffffffffu, mine, own) / sm.D[c][c];
                }
                if (l == own) {
                    if (hi) v1 = xc; else v0 = xc;
                }
                if (l < c) v0 -= sm.D[l][c] * xc;
                if (l + 32 < c) v1 -= sm.D[l + 32][c] * xc;
            }
            if (l < h) a.vy[r0 + l] = v0;
            if (l + 32 < h) a.vy[r0 + l + 32] = v1;
            if (l == 0) a.bexp[b] = e;
            __threadfence();
            __syncwarp();
            if (l == 0) st_release(&a.flags[b], epoch);
        }
        __syncthreads();
    }
}

// After a completed trsv (grid synced): Emax over all blocks.
__device__ int trsv_emax(Ctx &C)
{
    const int Nb = (int)((C.M + TB - 1) / TB);
    int e = INT_MIN;
    for (int b = 0; b < Nb; ++b) e = max(e, __ldcg(&C.a.bexp[b]));
    return e;
}

__global__ void __launch_bounds__(PNT, 1) panel_kernel(PanelArgs a)
{
    cg::grid_group grid = cg::this_grid();
    __shared__ PanelSmem sm;
    Ctx C(a, sm);
    const int64_t n = a.n, s0 = a.s0, p0 = C.p0, lda = a.lda;
    double *A = a.A;
    double *U = a.U, *V = a.V, *Y = a.Y, *S = a.S, *T = a.T;
    const int nb = a.nb;
    unsigned epoch = a.epoch;
    int k = 0, failed = 0;
    long long ir_steps = 0, ir_cols = 0, rescales = 0;
    int ffi = 0;  // cursor into the forced-failure list

    while (k < a.kmax) {
        const int64_t j0 = s0 + k;
        const int ku = k + 1;  // U columns incl. the new u
        C.ph++;
        // ================= P1: update column j of A =========================
        for (int c = C.tid; c < k; c += PNT) sm.sv1[c] = (c == k - 1) ? 1.0 : V[(size_t)c * n + j0];
        __syncthreads();
        for (int64_t r = C.rb0 + C.tid; r < C.rb1; r += PNT) {
            double a0 = A[(size_t)j0 * lda + r];
            a.vsave[r] = a0;
            double s = 0.0;
            for (int c = 0; c < k; ++c) s += Y[(size_t)c * n + r] * sm.sv1[c];
            a.vx[r] = a0 - s;
        }
        __syncthreads();
        C.rows_tdot(U, n, k, [&](int64_t r) { return a.vx[r]; }, 0);
        grid.sync();
        C.gather(sm.sv2, k, 0);
        __syncthreads();
        for (int c = C.tid; c < k; c += PNT) {  // sv3 = S^T t
            double s = 0.0;
            for (int i = 0; i <= c; ++i) s += S[(size_t)c * nb + i] * sm.sv2[i];
            sm.sv3[c] = s;
        }
        __syncthreads();
        C.ph++;
        {
            double ss = 0.0;
            for (int64_t r = C.rb0 + C.tid; r < C.rb1; r += PNT) {
                double s = 0.0;
                for (int c = 0; c < k; ++c) s += U[(size_t)c * n + r] * sm.sv3[c];
                double av = a.vx[r] - s;
                a.vx[r] = av;
                if (r >= j0 + 2) ss += av * av;
            }
            C.block_reduce_to_part(ss, 0);
        }
        grid.sync();
        // ================= P2: left reflector ===============================
        double tau_u, scal_u, beta_u, alpha_u;
        {
            C.gather(sm.sv1, 1, 0);
            __syncthreads();
            const double ss = sm.sv1[0];
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
        __syncthreads();
        for (int64_t r = C.rb0 + C.tid; r < C.rb1; r += PNT) {
            double u = (r < j0 + 1) ? 0.0 : (r == j0 + 1 ? 1.0 : a.vx[r] * scal_u);
            U[(size_t)k * n + r] = u;
            if (r <= j0) A[(size_t)j0 * lda + r] = a.vx[r];  // rows s+1:j of the updated column (P1)
            else if (r == j0 + 1) A[(size_t)j0 * lda + r] = beta_u;
            else if (r >= j0 + 2) A[(size_t)j0 * lda + r] = 0.0;  // Set A(j+2:n, j) <- 0
        }
        C.ph++;
        C.rows_tdot(U, n, k, [&](int64_t r) {
            return (r < j0 + 1) ? 0.0 : (r == j0 + 1 ? 1.0 : a.vx[r] * scal_u);
        }, 0);
        grid.sync();
        C.gather(sm.sv2, k, 0);  // U^T u
        __syncthreads();
        for (int i = C.tid; i <= k; i += PNT) {
            double s = 0.0;
            if (i < k) {
                for (int l = i; l < k; ++l) s += S[(size_t)l * nb + i] * sm.sv2[l];
                s *= -tau_u;
            } else {
                s = tau_u;
            }
            sm.snew[i] = s;
        }
        __syncthreads();
        if (C.bid == 0)
            for (int i = C.tid; i <= k; i += PNT) S[(size_t)k * nb + i] = sm.snew[i];
        // S_{k+1}(i, c): c < k from global S, c == k from snew
        auto Sget = [&](int i, int c) -> double { return c == k ? sm.snew[i] : S[(size_t)c * nb + i]; };

        // ================= P3: solve, P4: residual + IR ======================
        // z2 = S_{k+1} w, w(c) = U(j0+1, c)
        for (int i = C.tid; i < ku; i += PNT) {
            double s = 0.0;
            for (int c = i; c < ku; ++c) {
                double wc = (c == k) ? 1.0 : U[(size_t)c * n + j0 + 1];
                s += Sget(i, c) * wc;
            }
            sm.sv3[i] = s;
        }
        __syncthreads();
        ++epoch;
        trsv_scaled(C, [&](int64_t r) { return r == j0 + 1 ? 1.0 : 0.0; }, ku, sm.sv3, epoch);
        grid.sync();
        int emax = trsv_emax(C);
        if (emax > 0) ++rescales;
        // normalise y~ and form V^T y~
        C.ph++;
        for (int64_t r = C.rb0 + C.tid; r < C.rb1; r += PNT) {
            int eb = __ldcg(&a.bexp[(r - p0) / TB]);
            a.vy[r] = ldexp(__ldcg(&a.vy[r]), eb - emax);
        }
        __syncthreads();
        C.rows_tdot(V, n, k, [&](int64_t r) { return a.vy[r]; }, 0);
        grid.sync();
        // x = (y~ - V T^T V^T y~)(j0+1:)
        C.gather(sm.sv1, k, 0);
        __syncthreads();
        for (int c = C.tid; c < k; c += PNT) {
            double s = 0.0;
            for (int i = 0; i <= c; ++i) s += T[(size_t)c * nb + i] * sm.sv1[i];
            sm.sv2[c] = s;
        }
        __syncthreads();
        C.ph++;
        {
            double sx = 0.0, st = 0.0;
            for (int64_t r = C.rb0 + C.tid; r < C.rb1; r += PNT) {
                double xv = 0.0;
                if (r >= j0 + 1) {
                    double s = 0.0;
                    for (int c = 0; c < k; ++c) s += V[(size_t)c * n + r] * sm.sv2[c];
                    xv = a.vy[r] - s;
                    sx += xv * xv;
                    if (r >= j0 + 2) st += xv * xv;
                }
                a.vx[r] = xv;
            }
            __syncthreads();
            C.rows_tdot(V, n, k, [&](int64_t r) { return a.vx[r]; }, 2);
            C.block_reduce_to_part(sx, 0);
            C.block_reduce_to_part(st, 1);
        }
        grid.sync();
        double xnorm2 = 0.0, xtail2 = 0.0;
        {
            C.gather(sm.sv1, 2, 0);
            __syncthreads();
            xnorm2 = sm.sv1[0];
            xtail2 = sm.sv1[1];
            __syncthreads();
        }
        bool accepted = (k == 0);  // k = 0: stable solve, no test (reading R-Z4)
        bool forced = false;
        while (ffi < a.n_force_fail && a.force_fail[ffi] < j0) ++ffi;
        if (ffi < a.n_force_fail && a.force_fail[ffi] == j0 && k > 0) forced = true;
        int ir = 0;
        bool this_col_ir = false;
        while (!accepted) {
            // ---- P4 residual: w = (I - V T V^T)[0; x] ----
            C.gather(sm.sv1, k, 2);  // V^T x (from the phase that produced x)
            __syncthreads();
            for (int i = C.tid; i < k; i += PNT) {  // sv2 = T t
                double s = 0.0;
                for (int c = i; c < k; ++c) s += T[(size_t)c * nb + i] * sm.sv1[c];
                sm.sv2[i] = s;
            }
            __syncthreads();
            for (int64_t r = C.rb0 + C.tid; r < C.rb1; r += PNT) {
                double s = 0.0;
                for (int c = 0; c < k; ++c) s += V[(size_t)c * n + r] * sm.sv2[c];
                a.vw[r] = a.vx[r] - s;
            }
            grid.sync();
            // ---- w2 = B w (area-balanced row slabs of the upper triangle) ----
            C.ph++;
            int64_t tr0, tr1;
            {
                double f0 = 1.0 - (double)C.bid / C.G, f1 = 1.0 - (double)(C.bid + 1) / C.G;
                tr0 = n - (int64_t)llround((double)C.M * sqrt(f0));
                tr1 = n - (int64_t)llround((double)C.M * sqrt(f1 > 0.0 ? f1 : 0.0));
                if (C.bid == 0) tr0 = p0;
                if (C.bid == C.G - 1) tr1 = n;
                if (tr0 < p0) tr0 = p0;
                if (tr1 > n) tr1 = n;
            }
            for (int64_t rc = tr0; rc < tr1; rc += 32) {
                const int64_t row = rc + C.lane;
                double s = 0.0;
                if (row < tr1)
                    for (int64_t c = rc + C.warp; c < n; c += NWP)
                        if (row <= c) s += a.B[(size_t)c * a.ldb + row] * a.vw[c];
                sm.accg[C.warp & 7][C.lane + 32 * (C.warp >> 3)] = s;
                __syncthreads();
                if (C.tid < 32 && rc + C.tid < tr1) {
                    double t2 = 0.0;
                    for (int g = 0; g < 8; ++g) t2 += sm.accg[g][C.tid] + sm.accg[g][C.tid + 32];
                    a.vw2[rc + C.tid] = t2;
                }
                __syncthreads();
            }
            // partial U^T w2 over [tr0, tr1)
            {
                double *out = C.mypart();
                for (int c = C.warp; c < ku; c += NWP) {
                    double s = 0.0;
                    for (int64_t r = tr0 + C.lane; r < tr1; r += 32) s += U[(size_t)c * n + r] * a.vw2[r];
                    s = warp_sum(s);
                    if (C.lane == 0) out[c] = s;
                }
            }
            grid.sync();
            // ---- r = sigma e1 - ((I - U S^T U^T) w2)(j0+1:) ----
            C.gather(sm.sv1, ku, 0);
            __syncthreads();
            for (int c = C.tid; c < ku; c += PNT) {  // sv2 = S^T t
                double s = 0.0;
                for (int i = 0; i <= c; ++i) s += Sget(i, c) * sm.sv1[i];
                sm.sv2[c] = s;
            }
            __syncthreads();
            C.ph++;
            const double sigma = ldexp(1.0, -emax);
            {
                double sr = 0.0;
                for (int64_t r = C.rb0 + C.tid; r < C.rb1; r += PNT) {
                    double rv = 0.0;
                    if (r >= j0 + 1) {
                        double s = 0.0;
                        for (int c = 0; c < ku; ++c) s += U[(size_t)c * n + r] * sm.sv2[c];
                        rv = (r == j0 + 1 ? sigma : 0.0) - (a.vw2[r] - s);
                        sr += rv * rv;
                    }
                    a.vr[r] = rv;
                }
                __syncthreads();
                C.rows_tdot(U, n, ku, [&](int64_t r) { return a.vr[r]; }, 1);
                C.block_reduce_to_part(sr, 0);
            }
            grid.sync();
            C.gather(sm.sv1, 1, 0);
            __syncthreads();
            const double rn = sqrt(sm.sv1[0]), xn = sqrt(xnorm2);
            __syncthreads();
            if (!forced && rn <= a.tol * xn && isfinite(rn)) {
                accepted = true;
                break;
            }
            if (forced || ir >= a.max_ir) break;  // IR failed
            // ---- IR correction: solve B~22 c = r with the same factored solve ----
            ++ir;
            ++ir_steps;
            this_col_ir = true;
            C.gather(sm.sv1, ku, 1);  // U^T r_ext
            __syncthreads();
            for (int i = C.tid; i < ku; i += PNT) {  // sv3 = S_{k+1} (U^T r)
                double s = 0.0;
                for (int c = i; c < ku; ++c) s += Sget(i, c) * sm.sv1[c];
                sm.sv3[i] = s;
            }
            __syncthreads();
            ++epoch;
            trsv_scaled(C, [&](int64_t r) { return __ldcg(&a.vr[r]); }, ku, sm.sv3, epoch);
            grid.sync();
            const int ec = trsv_emax(C);
            if (ec > 0) { ++rescales; break; }  // a rescaled correction counts as IR failure (C.8)
            C.ph++;
            for (int64_t r = C.rb0 + C.tid; r < C.rb1; r += PNT) {
                int eb = __ldcg(&a.bexp[(r - p0) / TB]);
                a.vy[r] = ldexp(__ldcg(&a.vy[r]), eb);
            }
            __syncthreads();
            C.rows_tdot(V, n, k, [&](int64_t r) { return a.vy[r]; }, 0);
            grid.sync();
            C.gather(sm.sv1, k, 0);
            __syncthreads();
            for (int c = C.tid; c < k; c += PNT) {
                double s = 0.0;
                for (int i = 0; i <= c; ++i) s += T[(size_t)c * nb + i] * sm.sv1[i];
                sm.sv2[c] = s;
            }
            __syncthreads();
            C.ph++;
            {
                double sx = 0.0, st = 0.0;
                for (int64_t r = C.rb0 + C.tid; r < C.rb1; r += PNT) {
                    double xv = 0.0;
                    if (r >= j0 + 1) {
                        double s = 0.0;
                        for (int c = 0; c < k; ++c) s += V[(size_t)c * n + r] * sm.sv2[c];
                        xv = a.vx[r] + (a.vy[r] - s);
                        sx += xv * xv;
                        if (r >= j0 + 2) st += xv * xv;
                    }
                    a.vx[r] = xv;
                }
                __syncthreads();
                C.rows_tdot(V, n, k, [&](int64_t r) { return a.vx[r]; }, 2);
                C.block_reduce_to_part(sx, 0);
                C.block_reduce_to_part(st, 1);
            }
            grid.sync();
            C.gather(sm.sv1, 2, 0);
            __syncthreads();
            xnorm2 = sm.sv1[0];
            xtail2 = sm.sv1[1];
            __syncthreads();
        }
        if (this_col_ir) ++ir_cols;
        if (C.bid == 0 && C.tid == 0) a.irtrace[j0] = (accepted ? 0 : 1000) + (a.irtrace[j0] >= 1000 ? 1000 : 0) + ir;
        if (!accepted) {
            // undo the left reflector: restore column j of A (Algorithm 1)
            for (int64_t r = C.rb0 + C.tid; r < C.rb1; r += PNT) A[(size_t)j0 * lda + r] = a.vsave[r];
            failed = 1;
            break;
        }
        // ================= P5: right reflector, T, Y ===========================
        double gam, scal_v;
        {
            const double alpha = __ldcg(&a.vx[j0 + 1]);
            gam = 0.0;
            scal_v = 0.0;
            if (xtail2 > 0.0) {
                double nrm = sqrt(alpha * alpha + xtail2);
                double bet = alpha >= 0.0 ? -nrm : nrm;
                gam = (bet - alpha) / bet;
                scal_v = 1.0 / (alpha - bet);
            }
        }
        auto vget = [&](int64_t r) -> double {
            return (r < j0 + 1) ? 0.0 : (r == j0 + 1 ? 1.0 : __ldcg(&a.vx[r]) * scal_v);
        };
        C.ph++;
        for (int64_t r = C.rb0 + C.tid; r < C.rb1; r += PNT) V[(size_t)k * n + r] = vget(r);
        C.rows_tdot(V, n, k, vget, 0);
        // A(p0:n, j0+1:n) v over own rows: lanes over rows, warps over columns
        for (int64_t rc = C.rb0; rc < C.rb1; rc += 32) {
            const int64_t row = rc + C.lane;
            double s = 0.0;
            if (row < C.rb1)
                for (int64_t c = j0 + 1 + C.warp; c < n; c += NWP) s += A[(size_t)c * lda + row] * vget(c);
            sm.accg[C.warp & 7][C.lane + 32 * (C.warp >> 3)] = s;
            __syncthreads();
            if (C.tid < 32 && rc + C.tid < C.rb1) {
                double t2 = 0.0;
                for (int g = 0; g < 8; ++g) t2 += sm.accg[g][C.tid] + sm.accg[g][C.tid + 32];
                a.vw2[rc + C.tid] = t2;
            }
            __syncthreads();
        }
        grid.sync();
        C.gather(sm.sv1, k, 0);  // z = V^T v
        __syncthreads();
        if (C.bid == 0)
            for (int i = C.tid; i <= k; i += PNT) {
                double s = 0.0;
                if (i < k) {
                    for (int l = i; l < k; ++l) s += T[(size_t)l * nb + i] * sm.sv1[l];
                    s *= -gam;
                } else {
                    s = gam;
                }
                T[(size_t)k * nb + i] = s;
            }
        for (int64_t r = C.rb0 + C.tid; r < C.rb1; r += PNT) {
            double s = 0.0;
            for (int c = 0; c < k; ++c) s += Y[(size_t)c * n + r] * sm.sv1[c];
            Y[(size_t)k * n + r] = gam * (a.vw2[r] - s);
        }
        ++k;
        __syncthreads();
    }
    grid.sync();
    if (C.bid == 0 && C.tid == 0) {
        a.out[0] = k;
        a.out[1] = failed;
        a.out[2] = ir_steps;
        a.out[3] = ir_cols;
        a.out[4] = rescales;
        a.out[5] = epoch;
    }
}

}  // namespace

int ht_panel_max_blocks(int *nblocks_out)
{
    int dev = 0, nsm = 0, per = 0;
    HT_CUDA_TRY(cudaGetDevice(&dev));
    HT_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    HT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, panel_kernel, PNT, 0));
    if (per < 1) return 4;
    *nblocks_out = nsm * (per > 1 ? 1 : per);
    return 0;
}

int ht_panel_run(cudaStream_t st, PanelArgs *a, int nblocks)
{
    void *args[] = {(void *)a};
    HT_CUDA_TRY(cudaLaunchCooperativeKernel((void *)panel_kernel, dim3(nblocks), dim3(PNT), args, 0, st));
    return 0;
}
