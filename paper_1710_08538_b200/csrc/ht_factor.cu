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
// with T formed here as well; the driver forms Qw explicitly and applies it.
//
// B200 design: one CTA of 512 threads per
// chain; the window is factored in 32-column panels (left-looking, DMMA), each
// panel in four 8-column leaves held in registers (lane = (column, row group)),
// so that one Householder column step is ~100 instructions per warp and ONE
// block barrier; a finished leaf updates the rest of its panel as a blocked (WY)
// update.
#include "ht_common.cuh"
#include "ht_internal.h"

namespace {

constexpr int PBW = 32;   // panel width (left-looking granularity)
constexpr int LW = 8;     // leaf width (columns factored one by one)
constexpr int NLF = PBW / LW;
constexpr int VRC = 256;  // rows per staged chunk of a previous panel's V
constexpr int LDX = 36;   // ld of the 32x32 X buffer (== 4 mod 16: conflict-free 64-bit B fragments)
constexpr int LDT = 36;   // == 4 mod 16: conflict-free 64-bit A fragments of T_i^T

// Optional phase profile (micro-benchmarks only): when non-null, thread 0 accumulates
// globaltimer nanoseconds per phase into g_fprof[phase].
__device__ unsigned long long *g_fprof = nullptr;
__device__ __forceinline__ unsigned long long fclock()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define FPROF(ph)                                                          \
    do {                                                                   \
        if (fprof && threadIdx.x == 0) {                                   \
            const unsigned long long _t = fclock();                        \
            fprof[ph] += _t - fprof_t;                                     \
            fprof_t = _t;                                                  \
        }                                                                  \
    } while (0)

__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Householder scalars of x = [alpha; tail], ||tail||^2 = ss > 0 (dlarfg convention, R-Z1):
// beta = -sign(alpha) ||x||, tau = (beta - alpha) / beta = 1 + |alpha| / ||x||,
// scal = 1 / (alpha - beta) = sign(alpha) / (||x|| tau)  (so that v = [1; tail * scal]).
// One rsqrt and one division by tau in [1, 2]: a short dependency chain on the column
// step's critical path.
__device__ __forceinline__ void house_scalars(double alpha, double ss, double &beta, double &tau, double &scal)
{
    const double N = fma(alpha, alpha, ss);
    const double r = rsqrt(N);  // 1 / ||x||
    const double nrm = N * r;
    beta = alpha >= 0.0 ? -nrm : nrm;
    tau = fma(fabs(alpha), r, 1.0);
    const double sc = r / tau;  // (measured: one IEEE division is ~40 cycles shorter than a float seed + 2 Newton steps)
    scal = alpha >= 0.0 ? sc : -sc;
}

// Column-step scalars of the wide layout (one out-of-line copy shared by the 32 unrolled
// steps: the unrolled loop otherwise misses in the instruction cache).  Sums the active
// warps' partial dot products in a fixed order, then forms the reflector of column jj.
struct StepScalars {
    double S, tau, scal, beta, myrow;
};
template <int FNW>
__device__ __forceinline__ StepScalars step_scalars(const double *part, const double *rowc, int buf, int bw, int rmax,
                                                 int rpt, int lane, int jj)
{
    double pr[FNW];
#pragma unroll
    for (int w = 0; w < FNW; ++w) pr[w] = (w >= bw && w * rpt <= rmax) ? part[(buf * FNW + w) * 32 + lane] : 0.0;
#pragma unroll
    for (int hh = FNW / 2; hh >= 1; hh >>= 1)  // tree sum (fixed order: deterministic)
#pragma unroll
        for (int w = 0; w < hh; ++w) pr[w] += pr[w + hh];
    StepScalars r;
    r.S = pr[0];
    const double ss = __shfl_sync(0xffffffffu, r.S, jj);  // squared tail norm
    const double alpha = rowc[buf * 32 + jj];
    r.myrow = rowc[buf * 32 + lane];
    r.tau = 0.0;
    r.scal = 0.0;
    r.beta = alpha;
    if (ss > 0.0) house_scalars(alpha, ss, r.beta, r.tau, r.scal);
    return r;
}

// Layout of one factor CTA.  Two register layouts of the 32-column panel:
//  * leaf layout (WIDE = false, 512 threads): a warp holds 4 row groups x 8 leaf columns,
//    RPT rows per thread and leaf, MAXP = 16 warps * 4 * RPT rows;
//  * wide layout (WIDE = true, 256 threads): lane = panel column, warp w holds rows
//    w*RPT .. w*RPT+RPT-1 of all 32 columns, MAXP = 8 * RPT rows (p <= 256).
template <int NT_, int RPT_, bool WIDE_>
struct FactorSmem {
    static constexpr int NT = NT_, NW = NT / 32, RPT = RPT_;
    static constexpr bool WIDE = WIDE_;
    static constexpr int MAXP = WIDE ? NW * RPT : NW * 4 * RPT;
    static constexpr int LDP = MAXP + 4;                       // == 4 mod 32
    static constexpr int RC = MAXP < VRC ? MAXP : VRC;
    static constexpr int LDV = RC + 4;                         // == 4 mod 32
    static constexpr int TPW = 16 / NW;                        // 8x8 tiles of a 32x32 product per warp
    static constexpr int VSZ = (WIDE || PBW * LDV > NW * LW * PBW) ? PBW * LDV : NW * LW * PBW;
    static constexpr int DOUBLES = PBW * LDP + VSZ + PBW * LDX + PBW * LDT + 2 * NW * PBW + 2 * PBW + PBW + 2 * 64 + 4 * LW +
                                   (WIDE ? 2 * MAXP : 0);
};

// Vs[c][rr] = V(r0 + rr, col0 + c) (view row order), rr < RC, zero beyond `rows`.
// All loads of a thread are issued before any store (memory-level parallelism).
template <class L>
__device__ __forceinline__ void stage_v(const FactorDesc &d, int col0, int r0, int rows, double *Vs)
{
    constexpr int PER = (PBW * L::RC + L::NT - 1) / L::NT;
    const int tid = threadIdx.x, p = d.p;
    double t[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) {
        const int idx = tid + e * L::NT;
        const int c = idx / L::RC, rr = idx % L::RC, r = r0 + rr;
        t[e] = (c < PBW && rr < rows) ? d.V[(int64_t)(col0 + c) * d.ldv + (d.rev ? p - 1 - r : r)] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < PER; ++e) {
        const int idx = tid + e * L::NT;
        const int c = idx / L::RC, rr = idx % L::RC;
        if (c < PBW) Vs[c * L::LDV + rr] = t[e];
    }
}

// X(32 x 32) = V_i(r_beg:p, :)^T * Ps(r_beg:p, :) by DMMA (K = rows), V_i = columns
// 32i..32i+31 of the window's V (view row order).  Warp w computes the 8x8 tiles
// t = w + NW*j (j < TPW), (tm, tn) = (t/4, t%4), and returns them in
// o[j] = X(8tm+g, 8tn+2t4 + {0,1}).
template <class L>
__device__ __forceinline__ void vt_times_panel(const FactorDesc &d, int i, int r_beg, int r_end, const double *Ps,
                                               double *Vs, double (&o)[L::TPW][2])
{
    constexpr int TPW = L::TPW, CH = 4;  // 4 independent DMMA chains per tile
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
    double x[TPW][CH][2];
#pragma unroll
    for (int j = 0; j < TPW; ++j)
#pragma unroll
        for (int u = 0; u < CH; ++u) x[j][u][0] = x[j][u][1] = 0.0;
    unsigned long long *fp = g_fprof;
    long long c_a = 0, c_b = 0;
    for (int r0 = r_beg; r0 < r_end; r0 += L::RC) {
        const int rows = min(L::RC, r_end - r0);
        __syncthreads();
        if (fp && tid == 0) c_a = clock64();
        stage_v<L>(d, i * PBW, r0, rows, Vs);
        __syncthreads();
        if (fp && tid == 0) c_b = clock64() + (Vs[0] != Vs[0] ? 1 : 0);
        const double *va[TPW], *pb[TPW];
#pragma unroll
        for (int j = 0; j < TPW; ++j) {
            const int t = warp + L::NW * j, tm = t >> 2, tn = t & 3;
            va[j] = Vs + (8 * tm + g) * L::LDV + t4;
            pb[j] = Ps + (8 * tn + g) * L::LDP + r0 + t4;
        }
        constexpr int KS = 4 * CH;
        int kk = 0;
        for (; kk + KS <= rows; kk += KS) {
#pragma unroll
            for (int u = 0; u < CH; ++u)
#pragma unroll
                for (int j = 0; j < TPW; ++j) dmma884(x[j][u][0], x[j][u][1], va[j][kk + 4 * u], pb[j][kk + 4 * u]);
        }
        for (; kk < rows; kk += 4)  // padded rows are 0
#pragma unroll
            for (int j = 0; j < TPW; ++j) dmma884(x[j][0][0], x[j][0][1], va[j][kk], pb[j][kk]);
    }
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int u = 0; u < CH; ++u) { a0 += x[j][u][0]; a1 += x[j][u][1]; }
        o[j][0] = a0;
        o[j][1] = a1;
    }
    if (fp && tid == 0) {
        const long long c_c = clock64() + (o[0][0] != o[0][0] ? 1 : 0);
        atomicAdd(&fp[24], (unsigned long long)(c_b - c_a));
        atomicAdd(&fp[25], (unsigned long long)(c_c - c_b));
        atomicAdd(&fp[26], 1ull);
    }
}

// Blocked, left-looking Householder QR of one p x q window view (p <= MAXP), PAPER.md
// sec. 2.1 reflectors (dlarfg convention, reading R-Z1) accumulated in compact WY form
// (eq. compactWY):
//   for each 32-column panel b:  P <- Q_{b-1}^T ... Q_0^T P     (Q_i = I - V_i T_i V_i^T, DMMA)
//     for each 8-column leaf:    column steps (one block reduction per column gives the
//                                tail norm and the leaf's dot products), then the leaf's
//                                8 reflectors update the rest of the panel (WY, T_leaf)
//   T_b from G = V_b^T V_b (DMMA) by the dlarft recurrence.
// Outputs: R (upper trapezoid, exact zeros below) back through the view, V in natural
// row order, tau, and the diagonal 32x32 blocks T_b of T:  Q = H_0 ... H_{q-1} =
// Q_0 Q_1 ...,  Q_b = I - V_b T_b V_b^T  (V_b = columns 32b..32b+31).  The off-diagonal
// blocks of T are never formed: every consumer applies Q panel block by panel block
// (ht_band_wy / ht_form_qhat, ht_chain.cu).  (The 512-thread leaf layout shares this code.)
// Wavefront mode for staircase chains whose windows are [new rows; R of the previous window]
// (R1: V2 top -> bottom, L1: U2 bottom -> top; sec. 3.3.1b, 3.3.2b).  Window i's column c
// holds R_{i-1}(0..c, c) in its bottom rows, and left-looking panel b of window i reads only
// R_{i-1}'s columns of panel b -- which window i-1 stores at the end of ITS panel b (later
// reflectors of window i-1 never touch them).  So panel b of window i may start as soon as
// (i-1, b) and (i, b-1) are done: a (windows + panels) wavefront instead of windows x panels.
// Persistent CTAs take windows in order from an atomic ticket (a CTA only ever waits on a
// lower ticket, which is already running: no deadlock) and publish "(i, b) stored" as an
// epoch-valued flag (release after a fence; the waiter acquires, then a block barrier).
struct WaveArgs {
    int *flags;      // [nd][WF_NB] epoch flags, null = sequential mode (one CTA, windows in order)
    int *ticket;     // zeroed before the launch
    int epoch;
};
constexpr int WF_NB = 8;  // panels per window (q <= 256)

__device__ __forceinline__ int ld_acquire_gpu(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int *p, int v)
{
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Up to four descriptors travel in the launch parameters (no host-to-device copy in the stream
// ahead of the kernel: one fewer operation per window on the critical stream).
struct FactorDescs4 {
    FactorDesc d[4];
};
template <class L>
__global__ void __launch_bounds__(L::NT, 1) factor_qr_kernel(const FactorDesc *descs, int nd, double *gscratch,
                                                             const WaveArgs wa, const __grid_constant__ FactorDescs4 inl)
{
    constexpr int FNT = L::NT, FNW = L::NW, RPT = L::RPT, TPW = L::TPW;
    constexpr bool WIDE = L::WIDE;
    extern __shared__ __align__(16) double fsm[];
    double *Ps = fsm;                         // [PBW][LDP]   panel, column-major
    double *Vs = Ps + PBW * L::LDP;           // [PBW][LDV]   staged V_i chunk / leaf partials
    double *Xs = Vs + L::VSZ;                 // [PBW][LDX]   X = T^T V^T P (row-major) / G_b
    double *Ts = Xs + PBW * LDX;              // [PBW][LDT]   T_i (left-looking) / leaf W
    double *part = Ts + PBW * LDT;            // [2][FNW][LW] (wide: [2][FNW][PBW])
    double *rowc = part + 2 * FNW * PBW;      // [2][LW]      (wide: [2][PBW])
    double *taus = rowc + 2 * PBW;            // [PBW]
    double *Zl = taus + PBW;                  // [LW][LW] leaf Z
    double *Tl = Zl + 64;                     // [LW][LW] leaf T
    double *coef = Tl + 64;                   // [2][2][LW] column-step update coefficients
    double *pivs = coef + 4 * LW;             // wide: [2][MAXP] pivot column (per-warp row slices)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int c8 = lane & 7, rq = lane >> 3;    // leaf column / row group of this lane
    const int rw0 = warp * 4 * RPT + rq * RPT;  // first of this thread's RPT rows
    unsigned long long *fprof = g_fprof;
    unsigned long long fprof_t = fprof ? fclock() : 0ull;

    __shared__ int s_ticket;
    auto next_window = [&](int cur) -> int {
        if (!wa.flags) return cur + 1;
        __syncthreads();
        if (tid == 0) s_ticket = atomicAdd(wa.ticket, 1);
        __syncthreads();
        return s_ticket;
    };
    for (int di = next_window(-1); di < nd; di = next_window(di)) {
        const FactorDesc d = descs ? descs[di] : inl.d[di];
        const int p = d.p, q = d.q;
        // rows >= dense + c + 1 of view column c are exactly zero (staircase windows)
        const int dense = (d.dense > 0 && d.dense < p) ? d.dense : p;
        const int64_t rs = d.rs, cs = d.cs;
        auto nat = [&](int r) -> int64_t { return d.rev ? (int64_t)(p - 1 - r) : (int64_t)r; };
        auto Tout = [&](int a, int c) -> double & { return d.T[(int64_t)c * d.ldt + a]; };
        const int nblk = (q + PBW - 1) / PBW;
        for (int b = 0; b < nblk; ++b) {
            const int c0 = b * PBW, nc = min(PBW, q - c0);
            if (wa.flags && di > 0) {  // wavefront: R_{i-1}'s columns of panel b are stored
                if (tid == 0)
                    while (ld_acquire_gpu(wa.flags + (size_t)(di - 1) * WF_NB + b) != wa.epoch) __nanosleep(64);
                __syncthreads();
            }
            // ---- load panel columns c0 .. c0+nc of the view (zero padding) ----
            {
                constexpr int PER = (PBW * L::LDP + FNT - 1) / FNT;
                const bool rowfast = (rs == 1 || rs == -1);  // contiguous along the view's rows
                double t[PER];
#pragma unroll
                for (int e = 0; e < PER; ++e) {
                    const int idx = tid + e * FNT;
                    const int j = rowfast ? idx / L::LDP : idx % PBW, r = rowfast ? idx % L::LDP : idx / PBW;
                    t[e] = (j < nc && r < p) ? __ldcg(d.W + ((int64_t)r * rs + (int64_t)(c0 + j) * cs)) : 0.0;
                }
#pragma unroll
                for (int e = 0; e < PER; ++e) {
                    const int idx = tid + e * FNT;
                    const int j = rowfast ? idx / L::LDP : idx % PBW, r = rowfast ? idx % L::LDP : idx / PBW;
                    if (j < PBW && r < L::LDP) Ps[j * L::LDP + r] = t[e];
                }
            }
            FPROF(0);
            // ---- left-looking: P <- (I - V_i T_i^T V_i^T) P for i < b ----
            for (int i = 0; i < b; ++i) {
                const int r_lo = i * PBW;  // V_i is zero above row r_lo
                __syncthreads();
                {
                    constexpr int E = PBW * PBW / FNT;  // elements per thread, all loads first
                    const int c = tid / PBW, a = tid % PBW;
                    double tv[E];
#pragma unroll
                    for (int e = 0; e < E; ++e) tv[e] = Tout(r_lo + a, r_lo + c + e * (FNT / PBW));
#pragma unroll
                    for (int e = 0; e < E; ++e) Ts[a * LDT + c + e * (FNT / PBW)] = tv[e];  // diagonal block T_i
                }
                const int r_hi = min(p, dense + r_lo + PBW);  // V_i is zero below this row
                double o[TPW][2];
                vt_times_panel<L>(d, i, r_lo, r_hi, Ps, Vs, o);
#pragma unroll
                for (int j = 0; j < TPW; ++j) {
                    const int t = warp + FNW * j, tm = t >> 2, tn = t & 3;
                    Xs[(8 * tm + g) * LDX + 8 * tn + 2 * t4] = o[j][0];
                    Xs[(8 * tm + g) * LDX + 8 * tn + 2 * t4 + 1] = o[j][1];
                }
                __syncthreads();
                FPROF(8);
                // X <- -T_i^T X  (T_i upper triangular, zero below the diagonal) on the tensor
                // pipe: X'(a, c) = sum_{l <= a} T(l, a) X(l, c), 16 8x8 tiles, K <= 32
                double xo[TPW][2];
#pragma unroll
                for (int j = 0; j < TPW; ++j) {
                    const int t = warp + FNW * j, tm = t >> 2, tn = t & 3;
                    double c0 = 0.0, c1 = 0.0;
#pragma unroll
                    for (int k = 0; k < PBW; k += 4)
                        if (k < 8 * tm + 8) dmma884(c0, c1, Ts[(k + t4) * LDT + 8 * tm + g], Xs[(k + t4) * LDX + 8 * tn + g]);
                    xo[j][0] = -c0;
                    xo[j][1] = -c1;
                }
                __syncthreads();
#pragma unroll
                for (int j = 0; j < TPW; ++j) {
                    const int t = warp + FNW * j, tm = t >> 2, tn = t & 3;
                    Xs[(8 * tm + g) * LDX + 8 * tn + 2 * t4] = xo[j][0];
                    Xs[(8 * tm + g) * LDX + 8 * tn + 2 * t4 + 1] = xo[j][1];
                }
                __syncthreads();
                FPROF(9);
                // P -= V_i X : per chunk, warp w owns row tiles w, w + FNW, ... x 4 column tiles
                for (int r0 = r_lo; r0 < r_hi; r0 += L::RC) {
                    const int rows = min(L::RC, r_hi - r0);
                    if (r_hi - r_lo > L::RC) {  // multi-chunk: Vs holds the last chunk -> re-stage
                        __syncthreads();
                        stage_v<L>(d, r_lo, r0, rows, Vs);
                        __syncthreads();
                    }
                    for (int tr = warp; 8 * tr < rows; tr += FNW) {
                        double acc[4][2];
#pragma unroll
                        for (int tn2 = 0; tn2 < 4; ++tn2) {
                            acc[tn2][0] = Ps[(8 * tn2 + 2 * t4) * L::LDP + r0 + 8 * tr + g];
                            acc[tn2][1] = Ps[(8 * tn2 + 2 * t4 + 1) * L::LDP + r0 + 8 * tr + g];
                        }
#pragma unroll
                        for (int kk = 0; kk < PBW; kk += 4) {
                            const double av = Vs[(kk + t4) * L::LDV + 8 * tr + g];
#pragma unroll
                            for (int tn2 = 0; tn2 < 4; ++tn2)
                                dmma884(acc[tn2][0], acc[tn2][1], av, Xs[(kk + t4) * LDX + 8 * tn2 + g]);
                        }
#pragma unroll
                        for (int tn2 = 0; tn2 < 4; ++tn2) {
                            Ps[(8 * tn2 + 2 * t4) * L::LDP + r0 + 8 * tr + g] = acc[tn2][0];
                            Ps[(8 * tn2 + 2 * t4 + 1) * L::LDP + r0 + 8 * tr + g] = acc[tn2][1];
                        }
                    }
                }
            }
            __syncthreads();
            FPROF(10);

            // R (upper trapezoid of the panel columns) and V go through Ps so that the global
            // stores are coalesced along the view's contiguous direction.
            auto store_R = [&]() {
                __syncthreads();
                if (rs == 1 || rs == -1) {  // contiguous along rows: lanes over rows
                    for (int j = warp; j < nc; j += FNW)
                        for (int r = lane; r < p; r += 32) d.W[(int64_t)r * rs + (int64_t)(c0 + j) * cs] = Ps[j * L::LDP + r];
                } else {                     // contiguous along columns: lanes over columns
                    for (int r = warp; r < p; r += FNW)
                        if (lane < nc) d.W[(int64_t)r * rs + (int64_t)(c0 + lane) * cs] = Ps[lane * L::LDP + r];
                }
                __syncthreads();
            };
            auto store_V = [&]() {
                __syncthreads();
                for (int j = warp; j < nc; j += FNW)
                    for (int r = lane; r < p; r += 32) d.V[(int64_t)(c0 + j) * d.ldv + nat(r)] = Ps[j * L::LDP + r];
            };
            if constexpr (WIDE) {
                // ---- wide layout: val[e] = P(w0 + e, c0 + lane), all 32 columns of the panel ----
                // One column step = every active warp: pivot column of its rows by shuffles,
                // partial dot products with all 32 columns -> part; ONE barrier; every active
                // warp sums the partials (same fixed order everywhere, so the scalars agree
                // bitwise), forms the reflector scalars and updates its own rows of all
                // later columns.  Rows above the diagonal row dr never change.
                const int w0 = warp * RPT;
                double val[RPT];
                {
                    const double2 *src = reinterpret_cast<const double2 *>(Ps + lane * L::LDP + w0);
#pragma unroll
                    for (int e = 0; e < RPT; e += 2) {
                        const double2 t = src[e / 2];
                        val[e] = t.x;
                        val[e + 1] = t.y;
                    }
                }
                // The pivot column of the next step goes through shared memory: its owner lane
                // stores the warp's rows, the warp reads them back as broadcasts (a 64-bit
                // shuffle per element would cost two SHFL per row and lane).  The warp owning
                // the next diagonal row writes zeros at rows <= that row, so the dot products and
                // updates need no per-element masks.
                // Column steps run in groups of 8 (unrolled: static register indices) inside a
                // rolled loop over the groups (the fully unrolled 32-step loop missed in the
                // instruction cache).  The warp owning a group's 8 diagonal rows keeps them in
                // val[0..7]: after the group they are final, go to Ps, and the warp shifts its
                // rows up by 8 (zeros enter at the bottom).  A warp that has shifted sh rows holds
                // row w0 + sh + e in val[e].
                int sh = 0;
                auto put_pivot = [&](int jn, int bn, int eon) {  // eon: local diagonal index, -1: not own
#ifdef HT_FACTOR_SHFL_PIVOT
                    return;
#endif
                    if (lane == jn) {
                        double2 *dst = reinterpret_cast<double2 *>(pivs + bn * L::MAXP + w0);
#pragma unroll
                        for (int e = 0; e < RPT; e += 2)
                            dst[e / 2] = make_double2(e > eon ? val[e] : 0.0, e + 1 > eon ? val[e + 1] : 0.0);
                    }
                    __syncwarp();
                };
                put_pivot(0, 0, warp == c0 / RPT ? 0 : -1);
#pragma unroll 1
                for (int g = 0; 8 * g < nc; ++g) {
                    const bool gown = warp == (c0 + 8 * g) / RPT;  // owns this group's diagonal rows
#pragma unroll
                    for (int jj8 = 0; jj8 < 8; ++jj8) {
                        const int jj = 8 * g + jj8;
                        if (jj >= nc) break;
                        const int buf = jj & 1;
                        const int dr = c0 + jj;           // diagonal row of column jj
                        const int bw = dr / RPT;          // warp holding row dr (in val[jj8])
                        const int rmax = dense + dr;      // last row that can be nonzero in column jj
                        const bool act = warp >= bw && warp * RPT <= rmax, own = gown;
                        double xr[RPT];
#ifdef HT_FACTOR_STEP_PROF
                        const bool cpw = fprof && lane == 0 && warp == FNW - 1;
                        long long ck0 = cpw ? clock64() : 0;
#endif
                        if (act) {
                            double sa[4] = {0.0, 0.0, 0.0, 0.0};
#ifdef HT_FACTOR_SHFL_PIVOT
                            // pivot column jj by shuffles from its lane (own warp: rows <= dr read as 0)
#pragma unroll
                            for (int e = 0; e < RPT; ++e) {
                                const double t = __shfl_sync(0xffffffffu, val[e], jj);
                                xr[e] = (own && e <= jj8) ? 0.0 : t;
                            }
#else
                            const double2 *src = reinterpret_cast<const double2 *>(pivs + buf * L::MAXP + w0);
#pragma unroll
                            for (int e = 0; e < RPT; e += 2) {
                                const double2 t = src[e / 2];
                                xr[e] = t.x;
                                xr[e + 1] = t.y;
                            }
#endif
#pragma unroll
                            for (int e = 0; e < RPT; ++e) sa[e & 3] = fma(xr[e], val[e], sa[e & 3]);  // xr = 0 at rows <= dr
                            part[(buf * FNW + warp) * PBW + lane] = (sa[0] + sa[1]) + (sa[2] + sa[3]);
                            if (own) rowc[buf * PBW + lane] = val[jj8];
                        }
#ifdef HT_FACTOR_STEP_PROF
                        long long ck1 = cpw ? clock64() + (int)(part[0] != part[0]) : 0;
#endif
                        __syncthreads();
#ifdef HT_FACTOR_STEP_PROF
                        long long ck2 = cpw ? clock64() : 0, ck3 = 0;
#endif
                        if (act) {
                            const StepScalars sc = step_scalars<FNW>(part, rowc, buf, bw, rmax, RPT, lane, jj);
#ifdef HT_FACTOR_STEP_PROF
                            if (cpw) ck3 = clock64() + (int)(sc.tau != sc.tau);
#endif
                            const double S = sc.S, myrow = sc.myrow, tau = sc.tau, scal = sc.scal, beta = sc.beta;
                            const double zc = myrow + scal * S;  // lanes < jj: v_lane^T v_jj = G_b(lane, jj)
                            const double wj = tau * zc;
                            if (own && lane < jj) Xs[jj * LDX + lane] = zc;
                            // rows > dr: column jj -> scal * x (its tail of v); later columns -= w_j v
                            const double mx = lane > jj ? -wj * scal : (lane == jj ? scal - 1.0 : 0.0);
#pragma unroll
                            for (int e = 0; e < RPT; ++e) val[e] = fma(mx, xr[e], val[e]);  // rows <= dr: xr = 0
                            if (own) {
                                val[jj8] = lane > jj ? val[jj8] - wj : (lane == jj ? beta : val[jj8]);
                                if (lane == jj) taus[jj] = tau;
                            }
                        }
#ifdef HT_FACTOR_STEP_PROF
                        long long ck4 = cpw ? clock64() + (int)(val[RPT - 1] != val[RPT - 1]) : 0;
#endif
                        // next step's pivot slices inside the group (a warp may become active)
                        if (jj8 < 7 && jj + 1 < nc && warp >= (dr + 1) / RPT && warp * RPT <= rmax + 1)
                            put_pivot(jj + 1, buf ^ 1, gown ? jj8 + 1 : -1);
#ifdef HT_FACTOR_STEP_PROF
                        if (cpw) {
                            const long long ck5 = clock64();
                            atomicAdd(&fprof[12], (unsigned long long)(ck1 - ck0));
                            atomicAdd(&fprof[13], (unsigned long long)(ck2 - ck1));
                            atomicAdd(&fprof[14], (unsigned long long)(ck3 - ck2));
                            atomicAdd(&fprof[15], (unsigned long long)(ck4 - ck3));
                            atomicAdd(&fprof[16], (unsigned long long)(ck5 - ck4));
                        }
#endif
                    }
                    if (gown) {  // this group's diagonal rows are final: to Ps, shift up by 8
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const int r = w0 + sh + e;
                            Ps[lane * L::LDP + r] = (r < p && lane < nc) ? val[e] : 0.0;
                        }
#pragma unroll
                        for (int e = 0; e + 8 < RPT; ++e) val[e] = val[e + 8];
#pragma unroll
                        for (int e = RPT - 8; e < RPT; ++e) val[e] = 0.0;
                        sh += 8;
                    }
                    const int jn = 8 * (g + 1);  // first column of the next group
                    if (jn < nc && warp >= (c0 + jn) / RPT && warp * RPT <= dense + c0 + jn)
                        put_pivot(jn, jn & 1, warp == (c0 + jn) / RPT ? 0 : -1);
                }
                FPROF(2);
                __syncthreads();
                {   // the rows still in registers (row w0 + sh + e in val[e]); R (view) and V (natural
                    // order) are both stored from Ps
#pragma unroll
                    for (int e = 0; e < RPT; ++e) {
                        const int r = w0 + sh + e;
                        if (e < RPT - sh) Ps[lane * L::LDP + r] = (r < p && lane < nc) ? val[e] : 0.0;
                    }
                }
                __syncthreads();
#ifdef HT_FACTOR_STEP_PROF
                FPROF(28);
#endif
                // R and V leave through Ps; every thread reads all its elements before its first
                // global store (the shared-memory latency is paid once per batch, not per element)
                constexpr int SB = 16, NPASS = (PBW * L::MAXP / FNT + SB - 1) / SB;  // elements per thread and pass
                const bool rowfast = rs == 1 || rs == -1;
                // R: rowfast -> lanes over rows (contiguous), else lanes over columns
#pragma unroll 1
                for (int ps = 0; ps < NPASS; ++ps) {
                    double t[SB];
#pragma unroll
                    for (int e = 0; e < SB; ++e) {
                        const int idx = tid + (ps * SB + e) * FNT;
                        const int j = rowfast ? idx / L::MAXP : idx % PBW, r = rowfast ? idx % L::MAXP : idx / PBW;
                        t[e] = (r <= c0 + j && j < PBW && r < L::MAXP) ? Ps[j * L::LDP + r] : 0.0;
                    }
#pragma unroll
                    for (int e = 0; e < SB; ++e) {
                        const int idx = tid + (ps * SB + e) * FNT;
                        const int j = rowfast ? idx / L::MAXP : idx % PBW, r = rowfast ? idx % L::MAXP : idx / PBW;
                        if (j < nc && r < p) d.W[(int64_t)r * rs + (int64_t)(c0 + j) * cs] = t[e];
                    }
                }
#ifdef HT_FACTOR_STEP_PROF
                FPROF(29);
#endif
#pragma unroll 1
                for (int ps = 0; ps < NPASS; ++ps) {  // V: unit diagonal, zeros above (and for tau = 0)
                    double t[SB];
#pragma unroll
                    for (int e = 0; e < SB; ++e) {
                        const int idx = tid + (ps * SB + e) * FNT, j = idx / L::MAXP, r = idx % L::MAXP, col = c0 + j;
                        t[e] = (r < col || j >= PBW) ? 0.0 : (r == col ? 1.0 : (taus[j] == 0.0 ? 0.0 : Ps[j * L::LDP + r]));
                    }
#pragma unroll
                    for (int e = 0; e < SB; ++e) {
                        const int idx = tid + (ps * SB + e) * FNT, j = idx / L::MAXP, r = idx % L::MAXP;
                        if (j < nc && r < p) d.V[(int64_t)(c0 + j) * d.ldv + nat(r)] = t[e];
                    }
                }
            } else {
            // ---- the panel in registers: val[l][e] = P(rw0 + e, 8l + c8) ----
            double val[NLF][RPT];
#pragma unroll
            for (int l = 0; l < NLF; ++l)
#pragma unroll
                for (int e = 0; e < RPT; ++e) val[l][e] = Ps[(LW * l + c8) * L::LDP + rw0 + e];
            int buf = 0;
#pragma unroll
            for (int lf = 0; lf < NLF; ++lf) {
                const int jbeg = LW * lf;
                if (jbeg >= nc) break;
                const int jend = min(nc, jbeg + LW);
                // -------- column steps inside the leaf --------
                // A (all warps): partial dot products of the pivot column with the leaf's
                //   columns over own rows -> part;  B (warp 0, lanes = columns): sums, the
                //   reflector scalars and per-column update coefficients -> coef;
                //   C (all warps): rank-1 update of own rows.  Two barriers per column.
                for (int jj = jbeg; jj < jend; ++jj) {
                    const bool cp = fprof && lane == 0 && (warp == 0 || warp == FNW - 1);
                    const int cpo = 12 + (warp == 0 ? 0 : 5);
                    long long ck0 = cp ? clock64() : 0;
                    const int jc = jj - jbeg;
                    const int dr = c0 + jj;                             // diagonal row of this column
                    const bool active = warp * 4 * RPT + 4 * RPT > dr;  // warp-uniform: rows >= dr here
                    const int src = (rq << 3) | jc;
                    double xr[RPT];
                    if (active) {
                        double sa[2] = {0.0, 0.0};
#pragma unroll
                        for (int e = 0; e < RPT; ++e) {
                            xr[e] = __shfl_sync(0xffffffffu, val[lf][e], src);
                            const double vm = (rw0 + e > dr) ? val[lf][e] : 0.0;
                            sa[e & 1] = fma(vm, xr[e], sa[e & 1]);
                        }
                        double s = sa[0] + sa[1];
                        s += __shfl_xor_sync(0xffffffffu, s, 8);
                        s += __shfl_xor_sync(0xffffffffu, s, 16);
                        if (rq == 0) part[(buf * FNW + warp) * LW + c8] = s;
                    } else if (rq == 0) {
                        part[(buf * FNW + warp) * LW + c8] = 0.0;
                    }
                    if (dr >= rw0 && dr < rw0 + RPT) {  // this thread holds row dr
#pragma unroll
                        for (int e = 0; e < RPT; ++e)
                            if (rw0 + e == dr) rowc[buf * LW + c8] = val[lf][e];
                    }
                    long long ck1 = cp ? clock64() : 0;
                    __syncthreads();
                    long long ck2 = cp ? clock64() : 0;
                    if (warp == 0) {
                        double pr[FNW];
#pragma unroll
                        for (int w = 0; w < FNW; ++w) pr[w] = part[(buf * FNW + w) * LW + c8];
#pragma unroll
                        for (int hh = FNW / 2; hh >= 1; hh >>= 1)  // tree sum (fixed order: deterministic)
#pragma unroll
                            for (int w = 0; w < hh; ++w) pr[w] += pr[w + hh];
                        const double S = pr[0];
                        const double ss = __shfl_sync(0xffffffffu, S, jc);  // lane jc: column jj
                        const double alpha = rowc[buf * LW + jc];
                        double tau = 0.0, scal = 0.0, beta = alpha;
                        if (ss > 0.0) house_scalars(alpha, ss, beta, tau, scal);
                        const double myrow = rowc[buf * LW + c8];
                        const double wj = tau * (myrow + scal * S);
                        if (lane < LW) {
                            // rows > dr: val += mx * x  (column jc: x = own value -> val = scal * x)
                            coef[(buf * 2) * LW + c8] = (c8 > jc) ? -wj * scal : (c8 == jc ? scal - 1.0 : 0.0);
                            coef[(buf * 2 + 1) * LW + c8] = (c8 > jc) ? -wj : beta;  // row dr
                            if (c8 < jc) Zl[c8 * LW + jc] = myrow + scal * S;  // Z(l, jj) = v_l^T v_jj
                            if (c8 == jc) taus[jj] = tau;
                        }
                    }
                    long long ck3 = cp ? clock64() : 0;
                    __syncthreads();
                    long long ck4 = cp ? clock64() : 0;
                    if (active) {
                        const double mx = coef[(buf * 2) * LW + c8];
#pragma unroll
                        for (int e = 0; e < RPT; ++e)
                            if (rw0 + e > dr) val[lf][e] = fma(mx, xr[e], val[lf][e]);
                        if (dr >= rw0 && dr < rw0 + RPT) {  // row dr: beta on the diagonal, -w_j to its right
                            const double c2 = coef[(buf * 2 + 1) * LW + c8];
#pragma unroll
                            for (int e = 0; e < RPT; ++e)
                                if (rw0 + e == dr) val[lf][e] = (c8 > jc) ? val[lf][e] + c2 : (c8 == jc ? c2 : val[lf][e]);
                        }
                    }
                    if (cp) {
                        long long ck5 = clock64();
                        atomicAdd(&fprof[cpo + 0], (unsigned long long)(ck1 - ck0));
                        atomicAdd(&fprof[cpo + 1], (unsigned long long)(ck2 - ck1));
                        atomicAdd(&fprof[cpo + 2], (unsigned long long)(ck3 - ck2));
                        atomicAdd(&fprof[cpo + 3], (unsigned long long)(ck4 - ck3));
                        atomicAdd(&fprof[cpo + 4], (unsigned long long)(ck5 - ck4));
                    }
                    buf ^= 1;
                }
                FPROF(2);
                // -------- blocked update of the later leaves of this panel --------
                if (jend < nc) {
                    __syncthreads();  // taus, Zl of the leaf complete
                    // leaf T (8x8): T(i,i) = tau_i, T(i,c) = -tau_c sum_{l=i}^{c-1} T(i,l) Z(l,c)
                    if (tid < LW) {
                        const int i = tid;
                        double trow[LW];
#pragma unroll
                        for (int c = 0; c < LW; ++c) {
                            double tv = 0.0;
                            if (c == i) tv = taus[jbeg + i];
                            else if (c > i) {
                                double sacc = 0.0;
#pragma unroll
                                for (int l = 0; l < c; ++l)
                                    if (l >= i) sacc += trow[l] * Zl[l * LW + c];
                                tv = -taus[jbeg + c] * sacc;
                            }
                            trow[c] = tv;
                        }
#pragma unroll
                        for (int c = 0; c < LW; ++c) Tl[i * LW + c] = trow[c];
                    }
                    // W(i, (l', c)) = sum_r v_i(r) P_l'(r, c) for the leaf's reflectors i
                    double *wpart = Vs;  // [FNW][LW][PBW]
#pragma unroll
                    for (int l2 = lf + 1; l2 < NLF; ++l2) {
                        double acc[LW];
#pragma unroll
                        for (int i = 0; i < LW; ++i) acc[i] = 0.0;
#pragma unroll
                        for (int i = 0; i < LW; ++i) {
                            const int di_ = c0 + jbeg + i;  // diagonal row of reflector i
#pragma unroll
                            for (int e = 0; e < RPT; ++e) {
                                const double vr = __shfl_sync(0xffffffffu, val[lf][e], (rq << 3) | i);
                                const int r = rw0 + e;
                                const double v = (r > di_) ? vr : (r == di_ ? 1.0 : 0.0);
                                acc[i] = fma(v, val[l2][e], acc[i]);
                            }
                        }
#pragma unroll
                        for (int i = 0; i < LW; ++i) {
                            acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 8);
                            acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 16);
                        }
                        if (rq == 0)
#pragma unroll
                            for (int i = 0; i < LW; ++i) wpart[(warp * LW + i) * PBW + LW * l2 + c8] = acc[i];
                    }
                    __syncthreads();
                    double *Wl = Ts;  // [LW][PBW]
                    if (tid < LW * PBW) {
                        const int i = tid / PBW, c = tid % PBW;
                        double pr[FNW];
#pragma unroll
                        for (int w = 0; w < FNW; ++w) pr[w] = (c >= LW * (lf + 1)) ? wpart[(w * LW + i) * PBW + c] : 0.0;
#pragma unroll
                        for (int hh = FNW / 2; hh >= 1; hh >>= 1)
#pragma unroll
                            for (int w = 0; w < hh; ++w) pr[w] += pr[w + hh];
                        Wl[i * PBW + c] = pr[0];
                    }
                    __syncthreads();
                    // W' = T_leaf^T W  (reflectors with jbeg + i >= jend have tau = 0 -> zero rows)
                    double wp = 0.0;
                    if (tid < LW * PBW) {
                        const int a = tid / PBW, c = tid % PBW;
                        for (int l = 0; l <= a; ++l) wp += Tl[l * LW + a] * Wl[l * PBW + c];
                    }
                    __syncthreads();
                    if (tid < LW * PBW) Wl[tid] = wp;
                    __syncthreads();
                    // P_l' -= V_leaf W'
#pragma unroll
                    for (int l2 = lf + 1; l2 < NLF; ++l2) {
                        double wv[LW];
#pragma unroll
                        for (int i = 0; i < LW; ++i) wv[i] = Wl[i * PBW + LW * l2 + c8];
#pragma unroll
                        for (int i = 0; i < LW; ++i) {
                            const int di_ = c0 + jbeg + i;
#pragma unroll
                            for (int e = 0; e < RPT; ++e) {
                                const double vr = __shfl_sync(0xffffffffu, val[lf][e], (rq << 3) | i);
                                const int r = rw0 + e;
                                const double v = (r > di_) ? vr : (r == di_ ? 1.0 : 0.0);
                                val[l2][e] = fma(-v, wv[i], val[l2][e]);
                            }
                        }
                    }
                    __syncthreads();
                }
                FPROF(3);
            }
            __syncthreads();
#pragma unroll
            for (int l = 0; l < NLF; ++l)
#pragma unroll
                for (int e = 0; e < RPT; ++e) {
                    const int r = rw0 + e, jl = LW * l + c8, col = c0 + jl;
                    Ps[jl * L::LDP + r] = (r <= col && r < p && jl < nc) ? val[l][e] : 0.0;
                }
            store_R();
#pragma unroll
            for (int l = 0; l < NLF; ++l)
#pragma unroll
                for (int e = 0; e < RPT; ++e) {
                    const int r = rw0 + e, jl = LW * l + c8, col = c0 + jl;
                    const double tv = taus[jl < nc ? jl : 0];
                    const double v = (jl >= nc || r < col) ? 0.0 : (r == col ? 1.0 : (tv == 0.0 ? 0.0 : val[l][e]));
                    Ps[jl * L::LDP + r] = (r < p) ? v : 0.0;
                }
            store_V();
            }
            if (tid < nc) d.tau[c0 + tid] = taus[tid];
            __threadfence_block();
            FPROF(4);
            // ---- G_b = V_b^T V_b (DMMA; the wide layout has it from the column steps) and
            //      T_b by the dlarft recurrence (row i per lane) ----
            __syncthreads();
            if constexpr (!WIDE)
#pragma unroll
            for (int j = 0; j < TPW; ++j) {
                const int t = warp + FNW * j, tm = t >> 2, tn = t & 3;
                const double *pa = Ps + (8 * tm + g) * L::LDP + t4, *pb = Ps + (8 * tn + g) * L::LDP + t4;
                double x[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
                int kk = c0;
                for (; kk + 16 <= p; kk += 16) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) dmma884(x[u][0], x[u][1], pa[kk + 4 * u], pb[kk + 4 * u]);
                }
                for (; kk < p; kk += 4) dmma884(x[0][0], x[0][1], pa[kk], pb[kk]);
                Xs[(8 * tm + g) * LDX + 8 * tn + 2 * t4] = (x[0][0] + x[1][0]) + (x[2][0] + x[3][0]);
                Xs[(8 * tm + g) * LDX + 8 * tn + 2 * t4 + 1] = (x[0][1] + x[1][1]) + (x[2][1] + x[3][1]);
            }
            __syncthreads();
            FPROF(11);
            if (fprof && tid == 0) atomicAdd(&fprof[27], (unsigned long long)(-clock64()));
            {
                // T_b by the dlarft forward recurrence
                //   T(i,i) = tau_i,  T(i,c) = -tau_c sum_{l<c} T(i,l) G(l,c)
                // Rows are independent: warp w takes rows w*RW .. w*RW+RW-1, the LPR lanes of a
                // row split its columns (lane cl: columns cl, cl+LPR, ...).  In right-looking
                // order, T(i,c) (computed by the owner lane of column c, then shuffled to the
                // row's lanes) is added into the sums of the later columns right away.
                constexpr int RW = PBW / FNW, LPR = 32 / RW, CPL = PBW / LPR;
                const int rr = lane / LPR, cl = lane % LPR, i = warp * RW + rr;
                double acc[CPL], tr[CPL];
#pragma unroll
                for (int u = 0; u < CPL; ++u) acc[u] = tr[u] = 0.0;
#pragma unroll
                for (int c = 0; c < PBW; ++c) {
                    const int uo = c / LPR, clo = c % LPR;
                    const double tc = taus[c < nc ? c : 0];
                    double tv = (c > i) ? -tc * acc[uo] : (c == i ? tc : 0.0);
                    tv = (c < nc && i < nc) ? tv : 0.0;
                    tv = __shfl_sync(0xffffffffu, tv, rr * LPR + clo);
                    if (cl == clo) tr[uo] = tv;
#pragma unroll
                    for (int u = 0; u < CPL; ++u) {
                        const int c2 = cl + LPR * u;
                        if (c2 > c) acc[u] = fma(tv, Xs[c2 * LDX + c], acc[u]);
                    }
                }
                if (fprof && tid == 0) {
                    const long long ckT = clock64() + (tr[0] != tr[0] ? 1 : 0);
                    atomicAdd(&fprof[27], (unsigned long long)ckT);
                }
                if (i < nc) {
                    // row i of T_b -> the diagonal block of the global T (columns c0..c0+nc)
#pragma unroll
                    for (int u = 0; u < CPL; ++u) {
                        const int c2 = cl + LPR * u;
                        if (c2 < nc) Tout(c0 + i, c0 + c2) = tr[u];
                    }
                }
            }
            __threadfence_block();
            __syncthreads();
            if (wa.flags && tid == 0) {  // publish: panel b's R columns (and V, T_b) are stored
                __threadfence();
                st_release_gpu(wa.flags + (size_t)di * WF_NB + b, wa.epoch);
            }
            FPROF(5);
        }
        // the next window of this launch may read what this one wrote (its R): a block barrier
        // orders global writes and reads inside the CTA; later kernels follow in stream order
        __syncthreads();
    }
}

template <class L>
int launch_factor(cudaStream_t st, const FactorDesc *d_descs, int nd, double *gscratch, const WaveArgs &wa, int grid,
                  const FactorDescs4 &inl)
{
    const int smem = L::DOUBLES * (int)sizeof(double);
    static std::mutex mu;
    static unsigned long long done = 0;
    const int rc = ht_once_per_device(mu, done, [smem] {
        HT_CUDA_TRY(cudaFuncSetAttribute(factor_qr_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        return 0;
    });
    if (rc) return rc;
    factor_qr_kernel<L><<<grid, L::NT, smem, st>>>(d_descs, nd, gscratch, wa, inl);
    HT_CUDA_TRY(cudaGetLastError());
    return 0;
}

using FWide128 = FactorSmem<256, 16, true>;   // p <= 128
using FWide256 = FactorSmem<256, 32, true>;   // p <= 256
using FLeaf512 = FactorSmem<512, 8, false>;   // p <= 512

}  // namespace

// Development profile of the factorization phases (HT_FPROF): dev = 32 zeroed counters or null.
int ht_factor_set_prof(unsigned long long *dev)
{
    HT_CUDA_TRY(cudaMemcpyToSymbol(g_fprof, &dev, sizeof(dev)));
    return 0;
}

int ht_factor_run(cudaStream_t st, const FactorDesc *d_descs, int nd, double *gscratch, int maxp, int *wave_flags,
                  int *wave_ticket, int wave_epoch, const FactorDesc *h_descs)
{
    if (nd <= 0) return 0;
    FactorDescs4 inl{};
    if (h_descs && nd <= 4) {  // by value: d_descs is not read
        for (int i = 0; i < nd; ++i) inl.d[i] = h_descs[i];
        d_descs = nullptr;
    }
    WaveArgs wa{nullptr, nullptr, 0};
    int grid = 1;
    if (wave_flags && nd > 1) {
        wa = WaveArgs{wave_flags, wave_ticket, wave_epoch};
        HT_CUDA_TRY(cudaMemsetAsync(wave_ticket, 0, sizeof(int), st));
        grid = nd < HT_WAVE_CTAS ? nd : HT_WAVE_CTAS;
    }
    if (maxp <= FWide128::MAXP) return launch_factor<FWide128>(st, d_descs, nd, gscratch, wa, grid, inl);
    if (maxp <= FWide256::MAXP) return launch_factor<FWide256>(st, d_descs, nd, gscratch, wa, grid, inl);
    if (maxp <= FLeaf512::MAXP) return launch_factor<FLeaf512>(st, d_descs, nd, gscratch, wa, grid, inl);
    return 4;  // HT_ENUMERIC: window taller than 512 rows (nb <= 256 guarantees p <= 512)
}
