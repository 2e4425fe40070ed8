// ht_driver.cu -- host driver of HouseHT (Algorithm 1) and the C ABI.
//
// The driver is the runtime around the kernels: it owns the device workspace,
// launches the persistent panel kernel (sec. 3.2), and sequences the
// absorption (sec. 3.3) as staircase window factorizations (ht_factor.cu) and
// FP64 tensor-core GEMMs (ht_gemm.cu).  All arithmetic on the data runs in
// those kernels; the host only computes indices and pointers.
//
// Readings of the paper:
//   R-Z9  after an IR failure the next panel restarts AT the failed column (text P:497).
//   R-Z10 reflectors pending at the end of the loop are absorbed.
//   R-Z11 when m = n-j <= 2k the absorption is done explicitly (two-sided compact
//         WY + one dense QR of the trailing m x m block of B).
//   Remark 4: first right window has kt rows, k < kt <= 2k, k | (m-kt);
//         restore chunks are aligned to the window boundaries.
#include <cuda.h>  // green-context types only (the entry points are fetched at run time)
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/ht.h"
#include "ht_common.cuh"
#include "ht_internal.h"

namespace {

#define TRY(x)                     \
    do {                           \
        int _rc = (x);             \
        if (_rc) return _rc;       \
    } while (0)

struct Work {
    int dev = -1;
    int64_t ncap = 0, nbcap = 0;
    int gmax = 0;
    cudaStream_t own_stream = nullptr;
    double *U = nullptr, *V = nullptr, *Y = nullptr, *S = nullptr, *T = nullptr;
    double *vec = nullptr, *part = nullptr;
    // U, V, Y, BV, S, T and the panel's n-vectors live in ONE allocation (`hot`, hot_bytes) so
    // that the panel launch can mark it L2-persisting (ht_panel_run): the fused sweep streams
    // the trailing A and B (~0.5 GB per column) and the side streams stream A, Q, Z, which
    // otherwise evict these small, reused arrays between columns (every access then pays HBM
    // latency on the panel's latency-bound phases).
    double *hot = nullptr;
    size_t hot_bytes = 0;
    // wavefront factorization of staircase chains (ht_factor_run): epoch flags + ticket
    int *wave_flags = nullptr, *wave_ticket = nullptr;
    bool green = false;  // sA, sQZ (and sA2, sQZ2: larger n) live in SM partitions (green contexts)
    cudaStream_t sA2 = nullptr, sQZ2 = nullptr;
    cudaStream_t side_a(int64_t n) const { return green && n >= 12288 ? sA2 : sA; }
    cudaStream_t side_qz(int64_t n) const { return green && n >= 12288 ? sQZ2 : sQZ; }
    int wave_epoch = 0;
    unsigned long long *yll = nullptr, *yll_exp = nullptr;
    int *bexp = nullptr;
    unsigned epoch = 0;
    int64_t *d_out = nullptr, *h_out = nullptr;
    double *d_scal = nullptr, *h_scal = nullptr;
    int *d_iflags = nullptr, *h_iflags = nullptr;
    double *VW = nullptr, *UW = nullptr;
    double *Vhat = nullptr, *tau = nullptr, *Gm = nullptr, *Tm = nullptr, *Wt = nullptr, *Qw = nullptr;
    double *tmp = nullptr, *W1 = nullptr, *W2 = nullptr, *UR = nullptr, *fscr = nullptr;
    // second window store for the U2 staircase (L1), factored on side_stream concurrently
    double *VhatL = nullptr, *QwL = nullptr, *TmL = nullptr, *tauL = nullptr, *WtL = nullptr, *fscrL = nullptr;
    cudaStream_t side_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // critical path (panel, B, factorization chains) on a high-priority stream; the A
    // and Q/Z window applies on two low-priority streams that overlap the chains
    cudaStream_t hp_stream = nullptr, sA = nullptr, sQZ = nullptr;
    // sB (high priority): Qhat formation and the full-height B updates of the R3/L3
    // windows; the critical stream only updates the band the next window reads
    cudaStream_t sB = nullptr;
    cudaEvent_t evF = nullptr, evE = nullptr;
    cudaEvent_t ev[12] = {};
    double *W1A = nullptr, *W2A = nullptr, *W1Q = nullptr, *W2Q = nullptr;
    // window stores of the R3 and L3 chains (their A/Z/Q applies run after the chain)
    double *VhatR = nullptr, *QwR = nullptr, *TmR = nullptr, *tauR = nullptr, *WtR = nullptr;
    double *VhatB = nullptr, *QwB = nullptr, *TmB = nullptr, *tauB = nullptr, *WtB = nullptr;
    int64_t *d_force = nullptr;
    int *d_irtrace = nullptr;
    double *Dinv = nullptr, *Bt = nullptr, *ypart = nullptr, *ypartB = nullptr, *BV = nullptr;
    int *dsafe = nullptr;
    double *Dinv4 = nullptr;                 // 256-row solve (trsv4): inverted 256 x 256 diagonal blocks
    int *dsafe4 = nullptr, *h_dsafe4 = nullptr;
    double *fro_part = nullptr;  // fixed-order partial sums of ||B||_F^2
    double *mgbuf = nullptr;     // packed all-gather staging (ht_reduce_mg)
    size_t mgcap = 0;
    cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;  // timing events of one call
    FactorDesc *d_fd = nullptr, *h_fd = nullptr;
    void *d_bd = nullptr, *h_bd = nullptr;  // band/Qhat-formation descriptors (one per factor descriptor)
    ChainWin *d_cw = nullptr, *h_cw = nullptr;
    int64_t ndesc = 0, ncw = 0, fd_cur = 0, ld_cur = 0, cw_cur = 0;
};

std::mutex g_mu[16];  // one per device: calls on different devices run concurrently
Work g_work[16];

// Device staging of the host entry points (ht_reduce / ht_reduce_host), kept per device
// between calls; its own lock (the call takes g_mu inside ht_reduce_ex).
struct HostStage {
    double *d[4] = {nullptr, nullptr, nullptr, nullptr};
    size_t bytes = 0;
    cudaStream_t st = nullptr;
};
std::mutex g_hmu[16];
HostStage g_hst[16];
void host_stage_free(HostStage &hs)
{
    for (auto &p : hs.d)
        if (p) { cudaFree(p); p = nullptr; }
    hs.bytes = 0;
}

// Per-kernel-class device time from CUDA events recorded on the launch stream.
// Classes: 0 panel, 1 DMMA GEMM, 2 factorizations (side streams), 3 other, 4 chained window
// applies, 5 absorb-right span and 6 absorb-left span (critical stream), 7 factorizations on
// the critical stream.
struct Timer {
    std::vector<cudaEvent_t> all, free_;
    struct Pend { int cls; cudaEvent_t a, b; };
    std::vector<Pend> pending;
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t launches = 0;
    int cls = 0;
    cudaEvent_t cur = nullptr;
    // class-4 launches run on several streams at once: their [begin, end] offsets from `base`
    // (the reduction's start event) give the time during which at least one of them runs
    cudaEvent_t base = nullptr;
    std::vector<std::pair<float, float>> iv4;
    double busy4()
    {
        std::sort(iv4.begin(), iv4.end());
        double tot = 0.0;
        float lo = 0.f, hi = 0.f;
        bool open = false;
        for (const auto &v : iv4) {
            if (open && v.first <= hi) { hi = std::max(hi, v.second); continue; }
            if (open) tot += (double)(hi - lo);
            lo = v.first; hi = v.second; open = true;
        }
        if (open) tot += (double)(hi - lo);
        return tot * 1e-3;
    }
    cudaEvent_t get()
    {
        if (free_.empty()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            all.push_back(e);
            return e;
        }
        cudaEvent_t e = free_.back();
        free_.pop_back();
        return e;
    }
    void begin(cudaStream_t st, int c, int nlaunch = 1)
    {
        cls = c;
        cur = get();
        cudaEventRecord(cur, st);
        launches += nlaunch;
    }
    void end(cudaStream_t st)
    {
        cudaEvent_t e = get();
        cudaEventRecord(e, st);
        pending.push_back({cls, cur, e});
        static const bool chk = getenv("HT_SYNC_CHECK") != nullptr;  // debugging: first failing launch
        if (chk) {
            const cudaError_t r = cudaStreamSynchronize(st);
            if (r != cudaSuccess) fprintf(stderr, "[ht sync] launch %lld (class %d) failed: %s\n", (long long)launches, cls, cudaGetErrorString(r));
        }
    }
    // an interval on `st` that is not a launch (phase spans): begin with span_begin, end with span_end
    cudaEvent_t span_begin(cudaStream_t st)
    {
        cudaEvent_t e = get();
        cudaEventRecord(e, st);
        return e;
    }
    void span_end(cudaStream_t st, int c, cudaEvent_t a)
    {
        cudaEvent_t e = get();
        cudaEventRecord(e, st);
        pending.push_back({c, a, e});
    }
    // Resolve the first `upto` pending intervals (their events must have completed); the
    // driver calls this after enqueueing the next absorption so that the host work of
    // reading events overlaps the device instead of delaying the next launches.
    void resolve(size_t upto = (size_t)-1)
    {
        upto = std::min(upto, pending.size());
        for (size_t i = 0; i < upto; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, pending[i].a, pending[i].b);
            acc[pending[i].cls] += ms * 1e-3;
            if (pending[i].cls == 4 && base) {
                float t0 = 0.f;
                cudaEventElapsedTime(&t0, base, pending[i].a);
                iv4.emplace_back(t0, t0 + ms);
            }
            free_.push_back(pending[i].a);
            free_.push_back(pending[i].b);
        }
        pending.erase(pending.begin(), pending.begin() + upto);
    }
    ~Timer()
    {
        for (auto e : all) cudaEventDestroy(e);
    }
};


// Side streams in an SM partition (green context, CUDA driver >= 12.4): the A/Q/Z window
// applies run only on `nsm` SMs, so the critical stream's single-CTA factorizations, band
// updates and sB's work always find free SMs (a factorization CTA needs a whole SM, and the
// side kernels' CTAs run for milliseconds).  Entry points come from cudaGetDriverEntryPoint, so
// the library has no link-time dependency on libcuda.  Returns false (caller keeps ordinary
// streams) if green contexts are unavailable.
static bool make_green_streams(int dev, int nsm, int priority, cudaStream_t *s1, cudaStream_t *s2)
{
    using GetRes = CUresult (*)(CUdevice, CUdevResource *, CUdevResourceType);
    using Split = CUresult (*)(CUdevResource *, unsigned *, const CUdevResource *, CUdevResource *, unsigned, unsigned);
    using GenDesc = CUresult (*)(CUdevResourceDesc *, CUdevResource *, unsigned);
    using Create = CUresult (*)(CUgreenCtx *, CUdevResourceDesc, CUdevice, unsigned);
    using SCreate = CUresult (*)(CUstream *, CUgreenCtx, unsigned, int);
    void *f[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    const char *names[5] = {"cuDeviceGetDevResource", "cuDevSmResourceSplitByCount", "cuDevResourceGenerateDesc",
                            "cuGreenCtxCreate", "cuGreenCtxStreamCreate"};
    for (int i = 0; i < 5; ++i) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint(names[i], &f[i], cudaEnableDefault, &q) != cudaSuccess || !f[i] ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return false;
        }
    }
    CUdevResource all, part, rem;
    unsigned ng = 1;
    CUdevResourceDesc desc;
    CUgreenCtx g;
    CUstream a, b;
    if (((GetRes)f[0])((CUdevice)dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return false;
    if (nsm <= 0 || (unsigned)nsm >= all.sm.smCount) return false;
    if (((Split)f[1])(&part, &ng, &all, &rem, 0, (unsigned)nsm) != CUDA_SUCCESS || ng < 1) return false;
    if (((GenDesc)f[2])(&desc, &part, 1) != CUDA_SUCCESS) return false;
    if (((Create)f[3])(&g, desc, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return false;
    if (((SCreate)f[4])(&a, g, CU_STREAM_NON_BLOCKING, priority) != CUDA_SUCCESS ||
        ((SCreate)f[4])(&b, g, CU_STREAM_NON_BLOCKING, priority) != CUDA_SUCCESS)
        return false;
    *s1 = (cudaStream_t)a;
    *s2 = (cudaStream_t)b;
    return true;
}

void work_free(Work &w)
{
    w.U = w.V = w.Y = w.S = w.T = w.vec = w.BV = nullptr;  // carved out of w.hot
    w.hot_bytes = 0;
    double **dp[] = {&w.hot, &w.part, &w.VW, &w.UW, &w.Vhat, &w.tau,
                     &w.Gm, &w.Tm, &w.Wt, &w.Qw, &w.tmp, &w.W1, &w.W2, &w.UR, &w.fscr, &w.d_scal,
                     &w.VhatL, &w.QwL, &w.TmL, &w.tauL, &w.WtL, &w.fscrL, &w.W1A, &w.W2A, &w.W1Q, &w.W2Q,
                     &w.VhatR, &w.QwR, &w.TmR, &w.tauR, &w.WtR, &w.VhatB, &w.QwB, &w.TmB, &w.tauB, &w.WtB};
    for (auto p : dp)
        if (*p) { cudaFree(*p); *p = nullptr; }
    if (w.wave_flags) cudaFree(w.wave_flags);
    if (w.wave_ticket) cudaFree(w.wave_ticket);
    w.wave_flags = w.wave_ticket = nullptr;
    if (w.yll) cudaFree(w.yll);
    if (w.yll_exp) cudaFree(w.yll_exp);
    w.yll = nullptr; w.yll_exp = nullptr;
    if (w.bexp) cudaFree(w.bexp);
    if (w.d_out) cudaFree(w.d_out);
    if (w.d_iflags) cudaFree(w.d_iflags);
    if (w.d_force) cudaFree(w.d_force);
    if (w.d_irtrace) cudaFree(w.d_irtrace);
    w.d_irtrace = nullptr;
    if (w.fro_part) cudaFree(w.fro_part);
    w.fro_part = nullptr;
    if (w.mgbuf) cudaFree(w.mgbuf);
    w.mgbuf = nullptr;
    w.mgcap = 0;
    if (w.Dinv) cudaFree(w.Dinv);
    if (w.Bt) cudaFree(w.Bt);
    w.Bt = nullptr;
    if (w.ypart) cudaFree(w.ypart);
    w.ypart = nullptr;
    if (w.ypartB) cudaFree(w.ypartB);
    w.ypartB = nullptr;
    if (w.dsafe) cudaFree(w.dsafe);
    w.Dinv = nullptr;
    w.dsafe = nullptr;
    if (w.Dinv4) cudaFree(w.Dinv4);
    if (w.dsafe4) cudaFree(w.dsafe4);
    if (w.h_dsafe4) cudaFreeHost(w.h_dsafe4);
    w.Dinv4 = nullptr;
    w.dsafe4 = w.h_dsafe4 = nullptr;
    if (w.d_fd) cudaFree(w.d_fd);
    if (w.h_out) cudaFreeHost(w.h_out);
    if (w.h_scal) cudaFreeHost(w.h_scal);
    if (w.h_iflags) cudaFreeHost(w.h_iflags);
    if (w.h_fd) cudaFreeHost(w.h_fd);
    if (w.d_cw) cudaFree(w.d_cw);
    if (w.h_cw) cudaFreeHost(w.h_cw);
    if (w.d_bd) cudaFree(w.d_bd);
    if (w.h_bd) cudaFreeHost(w.h_bd);
    w.d_bd = w.h_bd = nullptr;
    w.d_cw = nullptr; w.h_cw = nullptr;
    w.bexp = nullptr; w.d_out = nullptr; w.d_iflags = nullptr; w.d_force = nullptr;
    w.d_fd = nullptr; w.h_out = nullptr; w.h_scal = nullptr; w.h_iflags = nullptr;
    w.h_fd = nullptr;
    w.ncap = w.nbcap = 0;
}

int dalloc(double **p, size_t count)
{
    if (cudaMalloc((void **)p, std::max<size_t>(count, 1) * sizeof(double)) != cudaSuccess) return HT_ENOMEM;
    return 0;
}

int work_get(int dev, int64_t n, int64_t nb, Work **out)
{
    if (dev < 0 || dev >= 16) return HT_ECUDA;
    Work &w = g_work[dev];
    if (w.ncap >= n && w.nbcap >= nb && w.ncap > 0) {
        *out = &w;
        return 0;
    }
    work_free(w);
    w.dev = dev;
    if (!w.own_stream && cudaStreamCreateWithFlags(&w.own_stream, cudaStreamNonBlocking) != cudaSuccess)
        return HT_ECUDA;
    const int64_t N = std::max<int64_t>(n, 8), NB = std::max<int64_t>(nb, 1);
    TRY(ht_panel_max_blocks(&w.gmax));
    const size_t nnb = (size_t)N * NB, nb2 = (size_t)NB * NB;
    {
        auto r32 = [](size_t c) { return (c + 31) & ~(size_t)31; };  // 256-byte aligned pieces
        const size_t a = r32(nnb), b = r32(nb2), cnt = 4 * a + 2 * b + r32(8 * (size_t)N);
        TRY(dalloc(&w.hot, cnt));
        w.hot_bytes = cnt * sizeof(double);
        w.U = w.hot; w.V = w.U + a; w.Y = w.V + a; w.BV = w.Y + a;
        w.S = w.BV + a; w.T = w.S + b; w.vec = w.T + b;
    }
    TRY(dalloc(&w.part, 2 * (size_t)w.gmax * (NB + 8)));
    const size_t nblk = (size_t)(N / 64 + 4);
    if (cudaMalloc((void **)&w.yll, 2 * (size_t)N * sizeof(unsigned long long)) != cudaSuccess) return HT_ENOMEM;
    if (cudaMalloc((void **)&w.yll_exp, nblk * sizeof(unsigned long long)) != cudaSuccess) return HT_ENOMEM;
    cudaMemset(w.yll, 0, 2 * (size_t)N * sizeof(unsigned long long));
    cudaMemset(w.yll_exp, 0, nblk * sizeof(unsigned long long));
    if (cudaMalloc((void **)&w.bexp, nblk * sizeof(int)) != cudaSuccess) return HT_ENOMEM;
    w.epoch = 1;
    if (cudaMalloc((void **)&w.d_out, 8 * sizeof(int64_t)) != cudaSuccess) return HT_ENOMEM;
    if (cudaMallocHost((void **)&w.h_out, 8 * sizeof(int64_t)) != cudaSuccess) return HT_ENOMEM;
    TRY(dalloc(&w.d_scal, 8));
    if (cudaMallocHost((void **)&w.h_scal, 8 * sizeof(double)) != cudaSuccess) return HT_ENOMEM;
    if (cudaMalloc((void **)&w.d_iflags, 8 * sizeof(int)) != cudaSuccess) return HT_ENOMEM;
    if (cudaMallocHost((void **)&w.h_iflags, 8 * sizeof(int)) != cudaSuccess) return HT_ENOMEM;
    TRY(dalloc(&w.VW, nnb)); TRY(dalloc(&w.UW, nnb));
    TRY(dalloc(&w.Vhat, 2 * nnb + 4 * nb2));
    TRY(dalloc(&w.Wt, 2 * nnb + 4 * nb2));
    TRY(dalloc(&w.tau, (size_t)N + 2 * NB));
    TRY(dalloc(&w.Gm, nnb + 2 * nb2));
    TRY(dalloc(&w.Tm, nnb + 2 * nb2));
    TRY(dalloc(&w.Qw, 4 * nnb + 8 * nb2));
    TRY(dalloc(&w.W1, nnb + 4 * nb2)); TRY(dalloc(&w.W2, nnb + 4 * nb2));
    TRY(dalloc(&w.UR, 2 * nb2));
    TRY(dalloc(&w.fscr, 4 * nb2 + 16384 + 64));
    TRY(dalloc(&w.VhatL, 2 * nnb + 4 * nb2)); TRY(dalloc(&w.WtL, 2 * nnb + 4 * nb2));
    TRY(dalloc(&w.QwL, 4 * nnb + 8 * nb2)); TRY(dalloc(&w.TmL, nnb + 2 * nb2));
    TRY(dalloc(&w.tauL, (size_t)N + 2 * NB)); TRY(dalloc(&w.fscrL, 4 * nb2 + 16384 + 64));
    if (!w.side_stream && cudaStreamCreateWithFlags(&w.side_stream, cudaStreamNonBlocking) != cudaSuccess)
        return HT_ECUDA;
    if (!w.ev_fork && cudaEventCreateWithFlags(&w.ev_fork, cudaEventDisableTiming) != cudaSuccess) return HT_ECUDA;
    if (!w.ev_join && cudaEventCreateWithFlags(&w.ev_join, cudaEventDisableTiming) != cudaSuccess) return HT_ECUDA;
    TRY(dalloc(&w.W1A, nnb + 4 * nb2)); TRY(dalloc(&w.W2A, nnb + 4 * nb2));
    TRY(dalloc(&w.W1Q, nnb + 4 * nb2)); TRY(dalloc(&w.W2Q, nnb + 4 * nb2));
    TRY(dalloc(&w.VhatR, 2 * nnb + 4 * nb2)); TRY(dalloc(&w.WtR, 2 * nnb + 4 * nb2));
    TRY(dalloc(&w.QwR, 4 * nnb + 8 * nb2)); TRY(dalloc(&w.TmR, nnb + 2 * nb2)); TRY(dalloc(&w.tauR, (size_t)N + 2 * NB));
    TRY(dalloc(&w.VhatB, 2 * nnb + 4 * nb2)); TRY(dalloc(&w.WtB, 2 * nnb + 4 * nb2));
    TRY(dalloc(&w.QwB, 4 * nnb + 8 * nb2)); TRY(dalloc(&w.TmB, nnb + 2 * nb2)); TRY(dalloc(&w.tauB, (size_t)N + 2 * NB));
    if (!w.hp_stream) {
        int lo = 0, hi = 0;
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return HT_ECUDA;
        // side streams (A; Q and Z) on an SM partition (green context; HT_NO_GREEN=1 or no
        // green-context support: ordinary streams with capped grids).  Two partitions: 100 of
        // 148 SMs below n = 12288, 120 above (the side work grows as n^3, the critical chains as
        // n^2); HT_GREEN_SMS overrides both.
        const int gsm = getenv("HT_GREEN_SMS") ? atoi(getenv("HT_GREEN_SMS")) : 0;
        w.green = getenv("HT_NO_GREEN") == nullptr && make_green_streams(dev, gsm ? gsm : 100, lo, &w.sA, &w.sQZ) &&
                  make_green_streams(dev, gsm ? gsm : 120, lo, &w.sA2, &w.sQZ2);
        if (cudaStreamCreateWithPriority(&w.hp_stream, cudaStreamNonBlocking, hi) != cudaSuccess ||
            (!w.green && cudaStreamCreateWithPriority(&w.sA, cudaStreamNonBlocking, lo) != cudaSuccess) ||
            (!w.green && cudaStreamCreateWithPriority(&w.sQZ, cudaStreamNonBlocking, lo) != cudaSuccess) ||
            cudaStreamCreateWithPriority(&w.sB, cudaStreamNonBlocking, hi) != cudaSuccess)
            return HT_ECUDA;
        if (cudaEventCreateWithFlags(&w.evF, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&w.evE, cudaEventDisableTiming) != cudaSuccess)
            return HT_ECUDA;
        for (auto &e : w.ev)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return HT_ECUDA;
    }
    if (cudaMalloc((void **)&w.d_force, (size_t)N * sizeof(int64_t)) != cudaSuccess) return HT_ENOMEM;
    if (cudaMalloc((void **)&w.d_irtrace, (size_t)N * sizeof(int)) != cudaSuccess) return HT_ENOMEM;
    TRY(dalloc(&w.fro_part, (size_t)ht_fro_scratch_size()));
    if (!w.ev_t0 && (cudaEventCreate(&w.ev_t0) != cudaSuccess || cudaEventCreate(&w.ev_t1) != cudaSuccess))
        return HT_ECUDA;
    TRY(dalloc(&w.Dinv, (size_t)(N / 128 + 2) * 128 * 128));
    TRY(dalloc(&w.Bt, (size_t)N * (size_t)N));
    TRY(dalloc(&w.ypart, (size_t)(N / 256 + 2) * (size_t)N));
    TRY(dalloc(&w.ypartB, (size_t)(N / 256 + 2) * (size_t)N));
    if (cudaMalloc((void **)&w.dsafe, (size_t)(N / 128 + 2) * sizeof(int)) != cudaSuccess) return HT_ENOMEM;
    TRY(dalloc(&w.Dinv4, (size_t)(N / 256 + 2) * 256 * 256));
    if (cudaMalloc((void **)&w.dsafe4, (size_t)(N / 256 + 2) * sizeof(int)) != cudaSuccess) return HT_ENOMEM;
    if (cudaMallocHost((void **)&w.h_dsafe4, (size_t)(N / 256 + 2) * sizeof(int)) != cudaSuccess) return HT_ENOMEM;
    w.ndesc = 4 * (N + 16);
    if (cudaMalloc((void **)&w.wave_flags, (size_t)w.ndesc * 8 * sizeof(int)) != cudaSuccess) return HT_ENOMEM;
    if (cudaMalloc((void **)&w.wave_ticket, 8 * sizeof(int)) != cudaSuccess) return HT_ENOMEM;  // [0,1] wave tickets, [2,3] sweep counters
    cudaMemset(w.wave_flags, 0, (size_t)w.ndesc * 8 * sizeof(int));
    w.wave_epoch = 0;
    w.ncw = 16 * (N + 16);  // chain windows: each window list is issued per stream (B; A; Q/Z)
    if (cudaMalloc((void **)&w.d_fd, w.ndesc * sizeof(FactorDesc)) != cudaSuccess) return HT_ENOMEM;
    if (cudaMallocHost((void **)&w.h_fd, w.ndesc * sizeof(FactorDesc)) != cudaSuccess) return HT_ENOMEM;
    if (cudaMalloc(&w.d_bd, w.ndesc * ht_band_desc_size()) != cudaSuccess) return HT_ENOMEM;
    if (cudaMallocHost(&w.h_bd, w.ndesc * ht_band_desc_size()) != cudaSuccess) return HT_ENOMEM;
    if (cudaMalloc((void **)&w.d_cw, w.ncw * sizeof(ChainWin)) != cudaSuccess) return HT_ENOMEM;
    if (cudaMallocHost((void **)&w.h_cw, w.ncw * sizeof(ChainWin)) != cudaSuccess) return HT_ENOMEM;
    w.ncap = N;
    w.nbcap = NB;
    *out = &w;
    return 0;
}

// HT_NO_WAVE=1 (development): factor the R1/L1 staircase chains window by window (one CTA)
// instead of as a wavefront (ht_factor_run).
static bool no_wave() { return getenv("HT_NO_WAVE") != nullptr; }  // read per call (tests toggle it)

// Critical-stream phase profile (HT_PHASES=1, development only): the time between two
// consecutive marks on the high-priority stream is charged to the later mark's phase.
struct Phases {
    bool on = getenv("HT_PHASES") != nullptr;
    std::vector<cudaEvent_t> pool;
    std::vector<int> cls;
    double acc[16] = {0};
    double host[2] = {0, 0};  // host seconds: event resolution after the panel sync, absorption enqueue
    void mark(cudaStream_t st, int c)
    {
        if (!on) return;
        if (cls.size() == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        cudaEventRecord(pool[cls.size()], st);
        cls.push_back(c);
    }
    void resolve()  // every recorded mark has completed
    {
        if (!on || cls.empty()) return;
        for (size_t i = 1; i < cls.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, pool[i - 1], pool[i]);
            acc[cls[i]] += ms * 1e-3;
        }
        std::swap(pool[0], pool[cls.size() - 1]);
        cls.assign(1, 0);
    }
    void print()
    {
        if (!on) return;
        static const char *nm[16] = {"panel", "pre-R1", "R2 B+W", "R3 rest", "L1 wait", "L2", "L3 rest", "join",
                                     "factor", "form", "band", "sB wait", "", "", "", ""};
        fprintf(stderr, "[ht phases] critical stream (s):");
        for (int i = 0; i < 12; ++i) fprintf(stderr, " %s=%.3f", nm[i], acc[i]);
        fprintf(stderr, " | host: resolve=%.3f absorb-enqueue=%.3f\n", host[0], host[1]);
    }
    ~Phases()
    {
        for (auto e : pool) cudaEventDestroy(e);
    }
};

// One reduction in flight.
struct Run {
    Work *w;
    Timer tm;
    Phases ph;
    cudaStream_t st;
    int64_t n, nb;
    double *A, *B, *Q, *Z;
    int64_t lda, ldb, ldq, ldz;
    bool wq, wz;
    int64_t qz0 = 0, qz1 = 0;  // rows of Q and Z this call computes (multi-GPU row slabs)
    // Multi-GPU (ht_reduce_mg): P ranks, this is rank `me`; `comm` is the NCCL
    // communicator, or NULL = loopback (this call plays all P ranks on one device).  A's
    // right-hand applies (R2, R3, Remark 2) run on row slabs, its left-hand applies (L2, L3)
    // on column slabs of [J, n); one packed all-gather after each phase switches layouts.
    int P = 1, me = 0;
    void *comm = nullptr;
    int part_begin() const { return comm ? me : 0; }
    int part_end() const { return comm ? me + 1 : P; }
    int gather(cudaStream_t s, double *X, int64_t ldx, int64_t r0, int64_t r1, int64_t c0, int64_t c1, int by_cols)
    {
        if (P <= 1) return 0;
        tm.begin(s, 3);
        const int rc = ht_mg_allgather(s, comm, P, me, X, ldx, r0, r1, c0, c1, by_cols, w->mgbuf, w->mgcap);
        tm.end(s);
        return rc;
    }
    ht_report rep;
    double extra_flops = 0.0;
    double chain_flops = 0.0;
    int64_t chain_launches = 0;

    // ---------------- helpers --------------------------------------------
    int gemm_on(cudaStream_t s, char ta, char tb, int64_t M, int64_t N, int64_t K, double al, const double *Ap,
                int64_t la, const double *Bp, int64_t lb, double be, double *Cp, int64_t lc)
    {
        if (M <= 0 || N <= 0) return 0;
        tm.begin(s, 1);
        int rc = ht_gemm(s, ta, tb, M, N, K, al, Ap, la, Bp, lb, be, Cp, lc);
        tm.end(s);
        return rc;
    }
    int gemm(char ta, char tb, int64_t M, int64_t N, int64_t K, double al, const double *Ap, int64_t la,
             const double *Bp, int64_t lb, double be, double *Cp, int64_t lc)
    {
        return gemm_on(st, ta, tb, M, N, K, al, Ap, la, Bp, lb, be, Cp, lc);
    }
    // s waits for everything issued so far on `from`
    int dep(cudaStream_t s, cudaStream_t from, int slot)
    {
        HT_CUDA_TRY(cudaEventRecord(w->ev[slot], from));
        HT_CUDA_TRY(cudaStreamWaitEvent(s, w->ev[slot], 0));
        return 0;
    }
    int copy2d(int64_t rows, int64_t cols, const double *src, int64_t lds, double *dst, int64_t ldd)
    {
        if (rows <= 0 || cols <= 0) return 0;
        tm.begin(st, 3);
        int rc = ht_copy2d(st, rows, cols, src, lds, dst, ldd);
        tm.end(st);
        return rc;
    }
    int zero_lower(int64_t rows, int64_t cols, double *M, int64_t ld, int64_t off)
    {
        if (rows <= 0 || cols <= 0) return 0;
        tm.begin(st, 3);
        int rc = ht_zero_lower(st, rows, cols, M, ld, off);
        tm.end(st);
        return rc;
    }
    // X(rows, c0:c0+nc) <- X (I - Vp T Vp^T), Vp nc x k (ld ldv)
    int right_wy(double *X, int64_t ldx, int64_t rows, int64_t c0, int64_t nc, const double *Vp, int64_t ldv,
                 const double *Tp, int64_t ldt, int64_t k)
    {
        TRY(gemm('N', 'N', rows, k, nc, 1.0, X + c0 * ldx, ldx, Vp, ldv, 0.0, w->W1, n));
        TRY(gemm('N', 'N', rows, k, k, 1.0, w->W1, n, Tp, ldt, 0.0, w->W2, n));
        TRY(gemm('N', 'T', rows, nc, k, -1.0, w->W2, n, Vp, ldv, 1.0, X + c0 * ldx, ldx));
        return 0;
    }
    // X(r0:r0+nr, c0:c0+nc) <- (I - Up S^T Up^T) X   (the transposed left WY, eq. tildeB)
    int left_wy(double *X, int64_t ldx, int64_t r0, int64_t nr, int64_t c0, int64_t nc, const double *Up, int64_t ldu,
                const double *Sp, int64_t lds, int64_t k)
    {
        double *Xp = X + r0 + c0 * ldx;
        TRY(gemm('T', 'N', k, nc, nr, 1.0, Up, ldu, Xp, ldx, 0.0, w->W1, k));
        TRY(gemm('T', 'N', k, nc, k, 1.0, Sp, lds, w->W1, k, 0.0, w->W2, k));
        TRY(gemm('N', 'N', nr, nc, k, -1.0, Up, ldu, w->W2, k, 1.0, Xp, ldx));
        return 0;
    }

    // Window bookkeeping for one chain: packed offsets into a window store.
    struct Win {
        int p, q;
        size_t ov, oq, og, ot;
    };
    struct Store {  // V-hat, explicit Q-hat, T, tau, V T, factor scratch
        double *Vhat, *Qw, *Tm, *tau, *Wt, *fscr;
    };
    Store main_store() const { return Store{w->Vhat, w->Qw, w->Tm, w->tau, w->Wt, w->fscr}; }
    Store side_store() const { return Store{w->VhatL, w->QwL, w->TmL, w->tauL, w->WtL, w->fscrL}; }
    std::vector<Win> wins, winsL;
    void wins_reset() { wins.clear(); }
    static Win add_win(std::vector<Win> &ws, int p, int q)
    {
        Win x{p, q, 0, 0, 0, 0};
        if (!ws.empty()) {
            const Win &b = ws.back();
            x.ov = b.ov + (size_t)b.p * b.q;
            x.oq = b.oq + (((size_t)b.p * b.p + 1) & ~(size_t)1);  // 16-byte aligned Qhat (bulk-copy staging)
            x.og = b.og + (size_t)b.q * b.q;
            x.ot = b.ot + (size_t)b.q;
        }
        ws.push_back(x);
        return x;
    }
    Win add_win(int p, int q) { return add_win(wins, p, q); }

    // Factor the windows `ws` (descriptors `fds`, one per window) on stream `s` with the
    // window store `sto`, then form Qw = I - V T V^T for each (on `sf` if given: it waits
    // for the factorization through evF).
    // wave: the descriptors are one staircase chain ([new rows; R of the previous window]),
    // factored as a wavefront (ht_factor_run); the ticket is per store (main / side) so that
    // chains on different streams may run concurrently.
    int factor_and_form(const std::vector<FactorDesc> &fds, const std::vector<Win> &ws, const Store &sto,
                        cudaStream_t s, cudaStream_t sf = nullptr, bool wave = false)
    {
        const int nd = (int)fds.size();
        if (nd == 0) return 0;
        if (w->fd_cur + nd > w->ndesc) return HT_ENUMERIC;
        FactorDesc *hf = w->h_fd + w->fd_cur;
        int maxp = 0;
        for (int i = 0; i < nd; ++i) {
            const Win &x = ws[i];
            hf[i] = fds[i];
            hf[i].T = sto.Tm + x.og;  // q x q compact-WY T, formed inside the factor kernel
            hf[i].ldt = x.q;
            maxp = std::max(maxp, fds[i].p);
            extra_flops += 2.0 * x.q * (double)x.q * (x.p - x.q / 3.0) + x.q * (double)x.q * x.q / 3.0;
        }
        // more than four descriptors go through device memory (<= 4 travel in the launch parameters)
        const bool fbyval = nd <= 4;  // descriptors in the launch parameters (no copy ahead of the kernel)
        if (!fbyval) HT_CUDA_TRY(cudaMemcpyAsync(w->d_fd + w->fd_cur, hf, nd * sizeof(FactorDesc), cudaMemcpyHostToDevice, s));
        tm.begin(s, s == st ? 7 : 2);
        if (wave && nd > 1 && !no_wave()) {
            // flags are indexed by descriptor slot (fd_cur + i): distinct for concurrent chains
            const int ep = ++w->wave_epoch;
            TRY(ht_factor_run(s, w->d_fd + w->fd_cur, nd, sto.fscr, maxp, w->wave_flags + (size_t)w->fd_cur * 8,
                              w->wave_ticket + (sto.Vhat == w->Vhat ? 0 : 1), ep, fbyval ? hf : nullptr));
        } else {
            TRY(ht_factor_run(s, w->d_fd + w->fd_cur, nd, sto.fscr, maxp, nullptr, nullptr, 0, fbyval ? hf : nullptr));
        }
        tm.end(s);
        if (s == st) ph.mark(st, 8);
        if (sf) {
            HT_CUDA_TRY(cudaEventRecord(w->evF, s));
            HT_CUDA_TRY(cudaStreamWaitEvent(sf, w->evF, 0));
            s = sf;
        }
        // Qw = Q_0 Q_1 ... (panel blocks of the factorization, ht_form_qhat)
        std::vector<double *> qp(nd);
        std::vector<const double *> vp(nd), tp(nd);
        std::vector<int> pp(nd), qq(nd);
        for (int i = 0; i < nd; ++i) {
            const Win &x = ws[i];
            qp[i] = sto.Qw + x.oq;
            vp[i] = sto.Vhat + x.ov;
            tp[i] = sto.Tm + x.og;
            pp[i] = x.p;
            qq[i] = x.q;
        }
        tm.begin(s, 1);
        TRY(ht_form_qhat(s, nd, qp.data(), pp.data(), qq.data(), vp.data(), tp.data(),
                         (char *)w->d_bd + w->fd_cur * ht_band_desc_size(), (char *)w->h_bd + w->fd_cur * ht_band_desc_size()));
        tm.end(s);
        if (s == st) ph.mark(st, 9);
        w->fd_cur += nd;
        return 0;
    }
    int factor_and_form(const std::vector<FactorDesc> &fds, size_t i0)
    {
        std::vector<Win> ws(wins.begin() + i0, wins.begin() + i0 + fds.size());
        return factor_and_form(fds, ws, main_store(), st);
    }

    // Chained window applies (ht_chain.cu): every matrix in `mats` takes the windows of
    // `wl` in order; lo/hi of a window are indexed by the matrix position in `mats`.
    int chain(const std::vector<ChainMat> &mats, const std::vector<ChainWin> &wl) { return chain_on(st, mats, wl, 0); }
    int chain_on(cudaStream_t s, const std::vector<ChainMat> &mats, const std::vector<ChainWin> &wl, int maxgrid)
    {
        if (wl.empty() || mats.empty()) return 0;
        const int nw = (int)wl.size();
        if (w->cw_cur + nw > w->ncw) return HT_ENUMERIC;
        ChainWin *hc = w->h_cw + w->cw_cur;
        int pmax = 0;
        for (int i = 0; i < nw; ++i) {
            hc[i] = wl[i];
            pmax = std::max(pmax, wl[i].p);
            for (size_t m = 0; m < mats.size(); ++m) {
                const int64_t a = std::max(wl[i].lo[m], mats[m].s_begin), b = std::min(wl[i].hi[m], mats[m].s_end);
                if (b > a) {
                    const double f = 2.0 * (double)(b - a) * wl[i].p * (double)wl[i].p;
                    g_ht_flops += f;
                    chain_flops += f;
                }
            }
        }
        // (chain windows stay in device memory: passing them in the launch parameters made the side
        // streams faster at the critical stream's expense before the SM partition, and is neutral with it)
        HT_CUDA_TRY(cudaMemcpyAsync(w->d_cw + w->cw_cur, hc, nw * sizeof(ChainWin), cudaMemcpyHostToDevice, s));
        tm.begin(s, 4);
        ++chain_launches;
        int rc = ht_chain_apply(s, mats.data(), (int)mats.size(), w->d_cw + w->cw_cur, nw, pmax, maxgrid);
        tm.end(s);
        w->cw_cur += nw;
        return rc;
    }

    // ---------------- front end: Householder QR by staircase panels ---------------------
    // X(r0:n, c0:c0+c) <- R (upper trapezoidal, exact zeros below) in place, by panels of q <= nq
    // columns.  A panel (rows rt:n) is reduced bottom -> top by a staircase of window QRs,
    // exactly the chain structure of sec. 3.3.2b (eq. qrdecomposition): the first
    // window is the bottom kt rows (q < kt <= 2q, q | (m - kt), Remark 4), every next one is
    // [q new rows; R of the window below].  The window transforms are then applied from the
    // left to X's columns [c0+p+q, x_end) and to Y(rt:n, y_c0:y_c1), and from the right to
    // Q(:, rt:n) -- the panel's Q factor is exactly the product of its windows (Q <- Q W1 W2 ...).
    int qr_left(double *X, int64_t ldx, int64_t r0, int64_t c0, int64_t c, int64_t x_end, double *Y, int64_t ldy,
                int64_t y_c0, int64_t y_c1, int64_t nq)
    {
        const Store sto = main_store();
        for (int64_t p = 0; p < c; p += nq) {
            const int64_t rt = r0 + p, m = n - rt, q = std::min<int64_t>(nq, c - p);
            if (m <= 1 || q <= 0) break;
            const int64_t q1 = std::min<int64_t>(q, m);
            w->fd_cur = w->ld_cur = w->cw_cur = 0;
            wins_reset();
            std::vector<FactorDesc> fds;
            std::vector<int64_t> tops;
            auto window = [&](int64_t a, int64_t b, bool stair) {
                Win x = add_win((int)(b - a), (int)q1);
                FactorDesc fd{X + (rt + a) + (c0 + p) * ldx, 1, ldx, (int)(b - a), (int)q1, 0, sto.Vhat + x.ov, b - a,
                              sto.tau + x.ot};
                if (stair) fd.dense = (int)(b - a - q1);  // [q new rows; R of the window below]
                fds.push_back(fd);
                tops.push_back(a);
            };
            if (m <= 2 * q1) {
                window(0, m, false);
            } else {
                const int64_t rem = (m - q1) % q1, kt = q1 + (rem == 0 ? q1 : rem);
                window(m - kt, m, false);
                for (int64_t top = m - kt; top > 0; top -= q1) window(top - q1, top + q1, true);
            }
            TRY(factor_and_form(fds, 0));
            std::vector<ChainWin> wl;
            const int64_t xs = c0 + p + q1;
            for (size_t i = 0; i < fds.size(); ++i)
                wl.push_back(ChainWin{sto.Qw + wins[i].oq, rt + tops[i], wins[i].p, {xs, y_c0, qz0}, {x_end, y_c1, qz1}});
            std::vector<ChainMat> mats;
            mats.push_back(ChainMat{X, ldx, 1, xs, x_end});
            mats.push_back(ChainMat{Y, ldy, 1, y_c0, y_c1});
            if (wq) mats.push_back(ChainMat{Q, ldq, 0, qz0, qz1});
            TRY(chain(mats, wl));
            // the descriptors live in pinned host buffers read by the queued copies: drain before
            // the next panel rewrites them
            HT_CUDA_TRY(cudaStreamSynchronize(st));
        }
        return 0;
    }

    // Front end (ht_options.flags).  HT_FLAG_DEFLATE_ZERO_COLUMNS: sec. 3.5.1 --
    // zero columns of B first (Z0; Q0 = Z0 if B is diagonal), QR of A's first l columns, QR of
    // the trailing block of B; *s_begin = l.  HT_FLAG_GENERAL_B: QR of B (QZ step 1).
    int front_end(uint32_t flags, int64_t *s_begin)
    {
        *s_begin = 0;
        const int64_t nq = std::min<int64_t>(nb, 128);
        if (flags & HT_FLAG_DEFLATE_ZERO_COLUMNS) {
            int *zc = reinterpret_cast<int *>(w->d_irtrace);  // n ints of scratch (the IR trace is set later)
            TRY(ht_zero_columns(st, n, B, ldb, zc, w->d_iflags + 2));
            std::vector<int> hz(n);
            HT_CUDA_TRY(cudaMemcpyAsync(hz.data(), zc, n * sizeof(int), cudaMemcpyDeviceToHost, st));
            HT_CUDA_TRY(cudaMemcpyAsync(w->h_iflags + 2, w->d_iflags + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
            HT_CUDA_TRY(cudaStreamSynchronize(st));
            const bool diagonal = w->h_iflags[2] == 0;
            std::vector<int64_t> perm;  // zero columns first, stable (SPEC's determinism)
            for (int64_t j = 0; j < n; ++j)
                if (hz[j]) perm.push_back(j);
            const int64_t l = (int64_t)perm.size();
            for (int64_t j = 0; j < n; ++j)
                if (!hz[j]) perm.push_back(j);
            if (l > 0 && l < n) {
                int64_t *dp = w->d_force;  // n int64 of scratch (the forced-failure list is uploaded later)
                HT_CUDA_TRY(cudaMemcpyAsync(dp, perm.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
                double *tmp = w->Bt;       // n x n scratch (used by the panels only)
                const int64_t *pr = diagonal ? dp : nullptr;
                // A0 = Q0^T A Z0, B0 = Q0^T B Z0 (Q0 = Z0 for diagonal B): rows and columns gathered
                TRY(ht_permute(st, n, n, A, lda, tmp, n, pr, dp));
                TRY(ht_copy2d(st, n, n, tmp, n, A, lda));
                TRY(ht_permute(st, n, n, B, ldb, tmp, n, pr, dp));
                TRY(ht_copy2d(st, n, n, tmp, n, B, ldb));
                if (wz) TRY(ht_perm_matrix(st, n, Z, ldz, dp));
                if (wq && diagonal) TRY(ht_perm_matrix(st, n, Q, ldq, dp));
                HT_CUDA_TRY(cudaStreamSynchronize(st));  // dp is reused as the forced-failure list
                // A0(:, 1:l) = Q1 [A11; 0]: Q1^T on A's other columns and on B (its first l columns are 0)
                TRY(qr_left(A, lda, 0, 0, l, n, B, ldb, l, n, nq));
                // the trailing block B(l:n, l:n) back to triangular form; A(l:n, 1:l) = 0 stays 0
                TRY(qr_left(B, ldb, l, l, n - l, n, A, lda, l, n, nq));
                TRY(zero_lower(n - l, n - l, B + l + l * ldb, ldb, 0));
                TRY(zero_lower(n, l, A, lda, 0));  // A11 upper triangular, zeros below (exact)
                *s_begin = l;
            }
        }
        if ((flags & HT_FLAG_GENERAL_B) && *s_begin == 0) {
            TRY(qr_left(B, ldb, 0, 0, n, n, A, lda, 0, n, nq));  // B = Q0 R; A <- Q0^T A; Q <- Q0
            TRY(zero_lower(n, n, B, ldb, 0));
        }
        return 0;
    }

    // ---------------- absorption (sec. 3.3) ---------------------------------
    // Streams: st (high priority) carries the critical path -- the staircase factorization
    // chains and every update of B (the chains read B's band); sA applies the same window
    // transforms to A, sQZ to Z and Q (their rows/columns never feed a factorization), so
    // those big applies overlap the one-SM factorization chains.  Both are joined before
    // the next panel.  Per matrix the paper's order of operations is kept.
    // CTAs of an A or Q/Z chain apply on the low-priority streams (measured: 64 is best at
    // n = 8192 -- 56 leaves the side streams as the tail of each absorption, 72+ starves the
    // B stream; at n = 16384 the side work grows as n^3 against ~n^2 for the critical
    // factorization chains and 96 is best)
    int sb_grid() const  // CTAs of sB's full-height B updates (0: uncapped)
    {
        static const int env = getenv("HT_SB_GRID") ? atoi(getenv("HT_SB_GRID")) : 0;
        return env;
    }
    int side_grid() const  // CTAs of A's window applies while the critical chains run
    {
        static const int env = getenv("HT_SIDE_GRID") ? atoi(getenv("HT_SIDE_GRID")) : 0;
        if (env > 0) return env;
        if (w->green) return 0;  // the SM partition bounds them: full grids
        return n >= 12288 ? 96 : 56;
    }
    int side_grid_qz() const  // the same for Q and Z
    {
        static const int env = getenv("HT_SIDE_GRID_QZ") ? atoi(getenv("HT_SIDE_GRID_QZ")) : 0;
        return env > 0 ? env : side_grid();
    }
    int absorb(int64_t s0, int64_t k)
    {
        const int64_t p0 = s0 + 1, J = s0 + k, m = n - J - 1;
        double *U = w->U, *V = w->V, *Y = w->Y, *S = w->S, *T = w->T;
        const bool serial = getenv("HT_SERIAL") != nullptr;  // debug: everything on st
        const int BATCH = getenv("HT_BATCH") ? atoi(getenv("HT_BATCH")) : 4;  // windows per side-stream apply
        cudaStream_t sA = serial ? st : w->side_a(n), sQ = serial ? st : w->side_qz(n);
        w->fd_cur = w->ld_cur = w->cw_cur = 0;
        TRY(dep(sA, st, 0));
        TRY(dep(sQ, st, 0));
        // Remark 2: rows 0:p0 of Y, then the deferred update of the panel columns (A: sA);
        // row-separable, so each rank takes the rows of its A slab (all rows before the tail rule)
        const bool tail = m <= 2 * k;
        for (int q = tail ? 0 : part_begin(); q < (tail ? 1 : part_end()); ++q) {
            int64_t a0 = 0, a1 = n;
            if (!tail) ht_slab(0, n, P, q, &a0, &a1);
            a1 = std::min(a1, p0);
            if (a1 <= a0) continue;
            const int64_t h = a1 - a0;
            TRY(gemm_on(sA, 'N', 'N', h, k, n - p0, 1.0, A + a0 + p0 * lda, lda, V + p0, n, 0.0, w->W1A + a0, n));
            TRY(gemm_on(sA, 'N', 'N', h, k, k, 1.0, w->W1A + a0, n, T, nb, 0.0, Y + a0, n));
            if (J > p0) TRY(gemm_on(sA, 'N', 'T', h, J - p0, k, -1.0, Y + a0, n, V + p0, n, 1.0, A + a0 + p0 * lda, lda));
        }
        if (tail) {
            TRY(dep(st, sA, 1));
            TRY(dep(st, sQ, 2));
            return absorb_tail(s0, k);
        }

        // staircase step ks >= k (reading R-step): windows of 2 ks x k rows stepping
        // by ks.  The paper's ks = k keeps the same structure for any ks >= k (the rows between
        // the carried k x k triangle and the ks new rows are zero), and R3/L3 then restore
        // ks x 2ks blocks.  Tiny premature absorptions (k down to 1) would otherwise make
        // ~m/k windows per chain; ks = min(32, nb) bounds that to ~m/32.
        const int64_t kmin = std::min<int64_t>(32, nb);
        const int64_t ks = (k < kmin && m > 2 * kmin) ? kmin : k;
        // geometry (Remark 4): right boundaries rb = {0, kt-ks, kt, kt+ks, ..., m}
        const int64_t rem = (m - ks) % ks;
        const int64_t kt = ks + (rem == 0 ? ks : rem);
        const int r = (int)((m - kt) / ks + 1);
        std::vector<int64_t> rb(r + 2), lb(r + 2);
        rb[0] = 0;
        for (int t = 1; t <= r + 1; ++t) rb[t] = kt - ks + (int64_t)(t - 1) * ks;
        for (int t = 0; t <= r + 1; ++t) lb[t] = m - rb[r + 1 - t];
        const int64_t ldw = n;  // VW/UW leading dimension
        TRY(copy2d(m, k, V + J + 1, n, w->VW, ldw));
        TRY(copy2d(m, k, U + J + 1, n, w->UW, ldw));
        const int K = (int)k;
        cudaEvent_t span_r = tm.span_begin(st);

        // ===== L1: QR staircase of U2, bottom -> top (sec. 3.3.2b) =====
        // It depends only on U2, so it is factored on the side stream while R1-R3 run.
        winsL.clear();
        {
            std::vector<FactorDesc> fl;
            const Store sl = side_store();
            for (int i = 0; i < r; ++i) {
                const int64_t top = lb[r - 1 - i], bot = lb[r + 1 - i];
                const int p = (int)(bot - top);
                Win x = add_win(winsL, p, K);
                fl.push_back(FactorDesc{w->UW + top, 1, ldw, p, K, 0, sl.Vhat + x.ov, p, sl.tau + x.ot});
                if (i > 0) fl.back().dense = p - (int)ks;  // [ks new rows; R of the window below; 0]
            }
            HT_CUDA_TRY(cudaEventRecord(w->ev_fork, st));
            HT_CUDA_TRY(cudaStreamWaitEvent(w->side_stream, w->ev_fork, 0));
            TRY(factor_and_form(fl, winsL, sl, w->side_stream, nullptr, true));
            HT_CUDA_TRY(cudaEventRecord(w->ev_join, w->side_stream));
        }

        // ===== R1: QL staircase of V2, top -> bottom (sec. 3.3.1b) =====
        // + R2 on B, pipelined: st factors the windows one by one; sB forms each window's
        // Qhat and applies it to B at once (R2's chain order), so B's R2 update ends one
        // window apply after the last factorization instead of a whole chain later.
        // (Rows of the R2 chain are independent, so its critical time is the chain length,
        // not the number of rows: splitting rows off does not help.)
        // Small k (premature absorptions): many small windows, launch-bound -> one factor launch
        // for all windows and one chain launch on st instead.
        cudaStream_t sBq = serial ? st : w->sB;
        const bool pipelined = k >= 64;
        wins_reset();
        std::vector<ChainWin> wl;
        std::vector<FactorDesc> fds;
        ph.mark(st, 1);
        for (int i = 0; i < r; ++i) {
            const int p = (int)(rb[i + 2] - rb[i]);
            Win x = add_win(p, K);
            FactorDesc fd{w->VW + (rb[i + 2] - 1) + (int64_t)(K - 1) * ldw, -1, -ldw, p, K, 1, w->Vhat + x.ov, p,
                          w->tau + x.ot};
            if (i > 0) fd.dense = p - (int)ks;  // view: [ks new rows; L of the window above, reversed; 0]
            wl.push_back(ChainWin{w->Qw + x.oq, J + 1 + rb[i], x.p, {0, 0, 0}, {J + 1 + rb[i + 2], n, n}});
            if (pipelined && no_wave()) {
                TRY(factor_and_form(std::vector<FactorDesc>{fd}, std::vector<Win>{x}, main_store(), st, sBq));
                TRY(chain_on(sBq, {ChainMat{B, ldb, 0, 0, n}}, {wl.back()}, 0));
            } else {
                fds.push_back(fd);
            }
        }
        if (pipelined && !no_wave()) {
            // The R1 chain as wavefront launches on st in groups of windows; sB forms each
            // group's Qhat and applies the group to B (R2, chain order) while st factors the
            // next group.  (One launch for the whole chain would leave B's R2 chain -- whose
            // top slab passes every window -- exposed after it.)
            const int grp_env = getenv("HT_WAVE_GROUP") ? atoi(getenv("HT_WAVE_GROUP")) : 0;
            // groups of 16; the last group is kept short (its B chain is exposed after it)
            const int grp = grp_env > 0 ? grp_env : 16;
            const int tail = grp_env > 0 ? 0 : std::min(r, 6);
            for (int g0 = 0; g0 < r;) {
                const int g1 = (g0 < r - tail) ? std::min(r - tail, g0 + grp) : r;
                // a group's first window continues the chain: its input (the previous group's
                // last R) is complete in stream order, so it needs no flag
                std::vector<FactorDesc> fg(fds.begin() + g0, fds.begin() + g1);
                std::vector<Win> wg(wins.begin() + g0, wins.begin() + g1);
                std::vector<ChainWin> cg(wl.begin() + g0, wl.begin() + g1);
                TRY(factor_and_form(fg, wg, main_store(), st, sBq, true));
                TRY(chain_on(sBq, {ChainMat{B, ldb, 0, 0, n}}, cg, 0));
                g0 = g1;
            }
            TRY(dep(st, sBq, 11));
        } else if (pipelined) {
            TRY(dep(st, sBq, 11));  // B's R2 chain done, all R1 windows formed
        } else {
            TRY(factor_and_form(fds, 0));
            TRY(chain_on(st, {ChainMat{B, ldb, 0, 0, n}}, wl, 0));
        }
        // ===== R2: B, Z, A <- . * RV_1 ... RV_r (sec. 3.3.1c-e) =====
        // B above; A (sA) and Z (sQZ) take the whole chain after B's W-update.
        const double *L1 = w->VW + (m - k);  // L^_1 (k x k lower), ld ldw
        // W-updates: B on st (+ sB), Z on sQZ, A on sA
        struct WX { double *X; int64_t ld, rows; cudaStream_t s; double *W1, *W2; } wx[2] = {
            {B, ldb, n, st, w->W1, w->W2}, {wz ? Z + qz0 : nullptr, ldz, qz1 - qz0, sQ, w->W1Q, w->W2Q}};
        auto wupdate = [&](const WX &e) -> int {
            if (!e.X || e.rows <= 0) return 0;
            TRY(gemm_on(e.s, 'N', 'N', e.rows, k, k, 1.0, e.X + p0 * e.ld, e.ld, V + p0, n, 0.0, e.W1, n));
            TRY(gemm_on(e.s, 'N', 'N', e.rows, k, k, 1.0, e.X + (n - k) * e.ld, e.ld, L1, ldw, 1.0, e.W1, n));
            TRY(gemm_on(e.s, 'N', 'N', e.rows, k, k, 1.0, e.W1, n, T, nb, 0.0, e.W2, n));
            TRY(gemm_on(e.s, 'N', 'T', e.rows, k, k, -1.0, e.W2, n, V + p0, n, 1.0, e.X + p0 * e.ld, e.ld));
            TRY(gemm_on(e.s, 'N', 'T', e.rows, k, k, -1.0, e.W2, n, L1, ldw, 1.0, e.X + (n - k) * e.ld, e.ld));
            return 0;
        };
        TRY(wupdate(wx[0]));
        TRY(dep(sA, st, 3));  // R1 windows, L^_1 (in VW) ready; B's R2 issued first
        TRY(dep(sQ, st, 3));
        {
            std::vector<ChainWin> wa = wl;
            for (auto &x : wa) x.hi[0] = n;  // A: all rows
            for (int q = part_begin(); q < part_end(); ++q) {
                int64_t a0, a1;
                ht_slab(0, n, P, q, &a0, &a1);
                TRY(chain_on(sA, {ChainMat{A, lda, 0, a0, a1}}, wa, side_grid()));
            }
            if (wz) TRY(chain_on(sQ, {ChainMat{Z, ldz, 0, qz0, qz1}}, wa, side_grid_qz()));
        }
        TRY(wupdate(wx[1]));
        for (int q = part_begin(); q < part_end(); ++q) {
            int64_t a0, a1;
            ht_slab(0, n, P, q, &a0, &a1);
            if (a1 <= a0) continue;
            TRY(gemm_on(sA, 'N', 'T', a1 - a0, 1, k, -1.0, Y + a0, n, V + J, n, 1.0, A + a0 + J * lda, lda));
            TRY(gemm_on(sA, 'N', 'T', a1 - a0, k, k, -1.0, Y + a0, n, L1, ldw, 1.0, A + a0 + (n - k) * lda, lda));
        }
        ph.mark(st, 2);
        // ===== R3: RQ staircase restoring B, bottom -> top (sec. 3.3.1 second "e)") =====
        // Window t is factored on st; the next window (t-1) reads only the band of rows
        // [C0, R0) of its columns, which st updates straight from (V, T) (ht_band_wy).
        // sB forms Qhat and updates the rows above the band (their next reader is window
        // t-1's band update, which waits for it through evE -- a full factorization later);
        // A and Z take the windows in batches after sB has formed them.
        const Store sr{w->VhatR, w->QwR, w->TmR, w->tauR, w->WtR, w->fscr};
        TRY(dep(sBq, st, 9));  // B after R2
        auto flush_right = [&](std::vector<ChainWin> &ws) -> int {
            if (ws.empty()) return 0;
            TRY(dep(sA, sBq, 4));
            TRY(dep(sQ, sBq, 4));
            for (int q = part_begin(); q < part_end(); ++q) {
                int64_t a0, a1;
                ht_slab(0, n, P, q, &a0, &a1);
                TRY(chain_on(sA, {ChainMat{A, lda, 0, a0, a1}}, ws, side_grid()));
            }
            if (wz) TRY(chain_on(sQ, {ChainMat{Z, ldz, 0, qz0, qz1}}, ws, side_grid_qz()));
            ws.clear();
            return 0;
        };
        // L2's chain on B (the L1 windows from the left, bottom -> top) only touches rows the R3
        // chain (also bottom -> top) has finished, and left and right transforms commute, so
        // with k >= 64 each L2 window goes to B on the L1 side stream as soon as R3 has moved
        // above its rows (overlapping the rest of R3).
        std::vector<ChainWin> wlu;
        for (int i = 0; i < r; ++i) {
            const Win &x = winsL[i];
            const int64_t R0 = J + 1 + lb[r - 1 - i];
            wlu.push_back(ChainWin{w->QwL + x.oq, R0, x.p, {R0, 0, 0}, {n, n, n}});
        }
        cudaStream_t sLq = serial ? st : w->side_stream;
        int nl2 = 0;  // L2 windows issued
        auto issue_l2 = [&](int64_t row_final) -> int {  // rows >= row_final are final for R3
            if (!pipelined) return 0;
            bool waited = false;
            while (nl2 < r && wlu[nl2].o >= row_final) {
                if (!waited) {
                    TRY(dep(sLq, st, 11));
                    waited = true;
                }
                TRY(chain_on(sLq, {ChainMat{B, ldb, 1, J + 1, n}}, {wlu[nl2]}, 0));
                ++nl2;
            }
            return 0;
        };
        std::vector<Win> winsR;
        std::vector<ChainWin> wr;
        bool have_e = false;
        for (int t = r; t >= 0; --t) {
            int64_t R0, h, C0, wdt;
            if (t >= 1) {
                R0 = J + 1 + rb[t];
                h = rb[t + 1] - rb[t];
                C0 = J + 1 + rb[t - 1];
                wdt = rb[t + 1] - rb[t - 1];
            } else {
                R0 = J + 1;
                h = rb[1];
                C0 = J + 1;
                wdt = h;
            }
            if (wdt <= 1) continue;
            Win x = add_win(winsR, (int)wdt, (int)h);
            std::vector<FactorDesc> f1{FactorDesc{B + (R0 + h - 1) + (C0 + wdt - 1) * ldb, -ldb, -1, (int)wdt, (int)h,
                                                  1, sr.Vhat + x.ov, wdt, sr.tau + x.ot}};
            TRY(factor_and_form(f1, std::vector<Win>{x}, sr, st, sBq));
            // sB: rows [0, C0) of the window's columns
            const ChainWin cw{sr.Qw + x.oq, C0, (int)wdt, {0, 0, 0}, {C0, n, n}};
            if (C0 > 0) TRY(chain_on(sBq, {ChainMat{B, ldb, 0, 0, C0}}, {cw}, sb_grid()));
            // st: the band [C0, R0) after the previous window's sB update
            if (R0 > C0) {
                if (have_e) HT_CUDA_TRY(cudaStreamWaitEvent(st, w->evE, 0));
                ph.mark(st, 11);
                tm.begin(st, 4);
                TRY(ht_band_wy(st, B, ldb, 0, C0, R0 - C0, C0, (int)wdt, (int)h, sr.Vhat + x.ov, wdt, sr.Tm + x.og, h));
                tm.end(st);
                chain_flops += 4.0 * (double)(R0 - C0) * wdt * h;
            }
            if (sBq != st) {
                HT_CUDA_TRY(cudaEventRecord(w->evE, sBq));
                have_e = true;
            }
            ph.mark(st, 10);
            TRY(issue_l2(R0));
            wr.push_back(ChainWin{sr.Qw + x.oq, C0, (int)wdt, {0, 0, 0}, {n, n, n}});
            if ((int)wr.size() == BATCH || t == 0) TRY(flush_right(wr));  // A, Z take the windows in batches
        }
        TRY(issue_l2(J + 1));
        TRY(flush_right(wr));
        TRY(dep(st, sBq, 10));  // B complete
        ph.mark(st, 3);
        tm.span_end(st, 5, span_r);
        cudaEvent_t span_l = tm.span_begin(st);
        HT_CUDA_TRY(cudaStreamWaitEvent(st, w->ev_join, 0));  // join the L1 staircase
        ph.mark(st, 4);
        // ===== L2: spike, chain on B, A, Q, W-updates =====
        {  // the k x k spike U^T B has a long K: split-K with W2 (free until the next GEMM) as slices
            tm.begin(st, 1);
            TRY(ht_gemm_splitk(st, 'T', 'N', k, k, n - p0, 1.0, U + p0, n, B + p0 + p0 * ldb, ldb, 0.0, w->W1, nb, w->W2,
                               (int64_t)n * nb));
            tm.end(st);
        }
        TRY(gemm('T', 'N', k, k, k, 1.0, S, nb, w->W1, nb, 0.0, w->W2, nb));
        TRY(gemm('N', 'N', k, k, k, -1.0, U + p0, n, w->W2, nb, 1.0, B + p0 + p0 * ldb, ldb));
        TRY(zero_lower(n - p0, k, B + p0 + p0 * ldb, ldb, 0));
        if (pipelined) TRY(dep(st, sLq, 11));  // L2's B chain (issued during R3) done
        else TRY(chain_on(st, {ChainMat{B, ldb, 1, J + 1, n}}, wlu, 0));
        // UR = [U1; R~1]  (2k x k)
        const int64_t ldur = 2 * k;
        TRY(copy2d(k, k, U + p0, n, w->UR, ldur));
        TRY(copy2d(k, k, w->UW, ldw, w->UR + k, ldur));
        TRY(zero_lower(k, k, w->UR + k, ldur, 0));

        // layout switch of A: row slabs -> full rows [0, n) x columns [p0, n) on every rank
        TRY(gather(sA, A, lda, 0, n, p0, n, 0));
        TRY(dep(sA, st, 5));  // L1 windows and UR are ready
        TRY(dep(sQ, st, 5));
        {
            std::vector<ChainWin> wla = wlu;
            for (auto &x : wla) x.lo[0] = J;  // A: columns J..n (column slabs per rank)
            for (int q = part_begin(); q < part_end(); ++q) {
                int64_t c0, c1;
                ht_slab(J, n, P, q, &c0, &c1);
                TRY(chain_on(sA, {ChainMat{A, lda, 1, c0, c1}}, wla, side_grid()));
            }
            std::vector<ChainWin> wlq = wlu;
            for (auto &x : wlq) x.lo[0] = 0;
            if (wq) TRY(chain_on(sQ, {ChainMat{Q, ldq, 0, qz0, qz1}}, wlq, side_grid_qz()));
        }
        {
            // B(p0:p0+2k, J+1:n) (st) and A(p0:p0+2k, J:n) (sA):  X <- X - UR S^T (X^T UR)^T
            struct LX { double *X; int64_t ld, c0, c1; cudaStream_t s; double *W1, *W2; };
            std::vector<LX> lx{{B, ldb, J + 1, n, st, w->W1, w->W2}};
            for (int q = part_begin(); q < part_end(); ++q) {
                int64_t c0, c1;
                ht_slab(J, n, P, q, &c0, &c1);
                lx.push_back({A, lda, c0, c1, sA, w->W1A, w->W2A});
            }
            for (auto &e : lx) {
                const int64_t nc = e.c1 - e.c0;
                if (nc <= 0) continue;
                double *Xp = e.X + p0 + e.c0 * e.ld;
                TRY(gemm_on(e.s, 'T', 'N', nc, k, 2 * k, 1.0, Xp, e.ld, w->UR, ldur, 0.0, e.W1, n));
                TRY(gemm_on(e.s, 'N', 'N', nc, k, k, 1.0, e.W1, n, S, nb, 0.0, e.W2, n));
                TRY(gemm_on(e.s, 'N', 'T', 2 * k, nc, k, -1.0, w->UR, ldur, e.W2, n, 1.0, Xp, e.ld));
            }
            if (wq && qz1 > qz0) {  // Q(rows, p0:p0+2k) <- Q (I - UR S UR^T)   (sQZ)
                double *Xp = Q + qz0 + p0 * ldq;
                const int64_t nr = qz1 - qz0;
                TRY(gemm_on(sQ, 'N', 'N', nr, k, 2 * k, 1.0, Xp, ldq, w->UR, ldur, 0.0, w->W1Q, n));
                TRY(gemm_on(sQ, 'N', 'N', nr, k, k, 1.0, w->W1Q, n, S, nb, 0.0, w->W2Q, n));
                TRY(gemm_on(sQ, 'N', 'T', nr, 2 * k, k, -1.0, w->W2Q, n, w->UR, ldur, 1.0, Xp, ldq));
            }
        }
        ph.mark(st, 5);
        // ===== L3: QR staircase restoring B, top -> bottom (sec. 3.3.2f) =====
        // As R3 with columns: st updates the next window's columns [R0+q, R0+q+qn) from
        // (V, T), sB forms Qhat and updates the columns to their right.
        const Store sb{w->VhatB, w->QwB, w->TmB, w->tauB, w->WtB, w->fscr};
        TRY(dep(sBq, st, 9));
        auto flush_left = [&](std::vector<ChainWin> &ws, int grid) -> int {
            if (ws.empty()) return 0;
            TRY(dep(sA, sBq, 6));
            TRY(dep(sQ, sBq, 6));
            for (int q = part_begin(); q < part_end(); ++q) {
                int64_t c0, c1;
                ht_slab(J, n, P, q, &c0, &c1);
                TRY(chain_on(sA, {ChainMat{A, lda, 1, c0, c1}}, ws, grid));
            }
            if (wq) {
                std::vector<ChainWin> wq_ = ws;
                for (auto &x : wq_) x.lo[0] = 0;
                TRY(chain_on(sQ, {ChainMat{Q, ldq, 0, qz0, qz1}}, wq_, grid ? side_grid_qz() : 0));
            }
            ws.clear();
            return 0;
        };
        std::vector<Win> winsB;
        std::vector<ChainWin> wb;
        have_e = false;
        for (int t = 0; t <= r; ++t) {
            const int64_t R0 = J + 1 + lb[t];
            const int64_t q = lb[t + 1] - lb[t];
            const int64_t p = (t < r) ? lb[t + 2] - lb[t] : q;
            if (p <= 1) continue;
            const int64_t qn = (t < r) ? lb[t + 2] - lb[t + 1] : 0;  // columns of the next window
            Win x = add_win(winsB, (int)p, (int)q);
            std::vector<FactorDesc> f1{FactorDesc{B + R0 + R0 * ldb, 1, ldb, (int)p, (int)q, 0, sb.Vhat + x.ov, p,
                                                  sb.tau + x.ot}};
            TRY(factor_and_form(f1, std::vector<Win>{x}, sb, st, sBq));
            const int64_t c1 = R0 + q + qn;  // sB: columns [c1, n)
            if (c1 < n)
                TRY(chain_on(sBq, {ChainMat{B, ldb, 1, c1, n}}, {ChainWin{sb.Qw + x.oq, R0, (int)p, {c1, 0, 0}, {n, n, n}}}, sb_grid()));
            if (qn > 0) {
                if (have_e) HT_CUDA_TRY(cudaStreamWaitEvent(st, w->evE, 0));
                ph.mark(st, 11);
                tm.begin(st, 4);
                TRY(ht_band_wy(st, B, ldb, 1, R0 + q, qn, R0, (int)p, (int)q, sb.Vhat + x.ov, p, sb.Tm + x.og, q));
                tm.end(st);
                chain_flops += 4.0 * (double)qn * p * q;
            }
            if (sBq != st) {
                HT_CUDA_TRY(cudaEventRecord(w->evE, sBq));
                have_e = true;
            }
            ph.mark(st, 10);
            wb.push_back(ChainWin{sb.Qw + x.oq, R0, (int)p, {J, 0, 0}, {n, n, n}});
            if ((int)wb.size() == BATCH) TRY(flush_left(wb, side_grid()));
        }
        TRY(flush_left(wb, 0));  // the last batch: the critical stream is done, full grid
        // layout switch back: column slabs -> the full trailing block on every rank
        TRY(gather(sA, A, lda, p0, n, J, n, 1));
        TRY(dep(st, sBq, 10));
        ph.mark(st, 6);
        // join: the next panel reads A and B; U, V, S, T, Y, the window stores are reused
        TRY(dep(st, sA, 7));
        TRY(dep(st, sQ, 8));
        ph.mark(st, 7);
        tm.span_end(st, 6, span_l);
        return 0;
    }

    // Reading R-Z11: explicit absorption when m <= 2k.
    int absorb_tail(int64_t s0, int64_t k)
    {
        const int64_t p0 = s0 + 1, J = s0 + k, m = n - J - 1;
        double *U = w->U, *V = w->V, *Y = w->Y, *S = w->S, *T = w->T;
        // right: A(:, J:n) -= Y V(J:n,:)^T ; B, Z <- . (I - V T V^T)
        TRY(gemm('N', 'T', n, n - J, k, -1.0, Y, n, V + J, n, 1.0, A + J * lda, lda));
        TRY(right_wy(B, ldb, n, p0, n - p0, V + p0, n, T, nb, k));
        if (wz && qz1 > qz0) TRY(right_wy(Z + qz0, ldz, qz1 - qz0, p0, n - p0, V + p0, n, T, nb, k));
        // left: A(p0:n, J:n), B(p0:n, p0:n) <- (I - U S^T U^T) . ; Q <- Q (I - U S U^T)
        TRY(left_wy(A, lda, p0, n - p0, J, n - J, U + p0, n, S, nb, k));
        TRY(left_wy(B, ldb, p0, n - p0, p0, n - p0, U + p0, n, S, nb, k));
        TRY(zero_lower(n - p0, k, B + p0 + p0 * ldb, ldb, 0));  // Fact 3
        if (wq && qz1 > qz0) TRY(right_wy(Q + qz0, ldq, qz1 - qz0, p0, n - p0, U + p0, n, S, nb, k));
        if (m >= 2) {
            const int64_t R0 = J + 1;
            wins_reset();
            Win x = add_win((int)m, (int)m);
            std::vector<FactorDesc> f1{FactorDesc{B + R0 + R0 * ldb, 1, ldb, (int)m, (int)m, 0, w->Vhat + x.ov, m,
                                                  w->tau + x.ot}};
            TRY(factor_and_form(f1, 0));
            std::vector<ChainMat> mats{ChainMat{A, lda, 1, J, n}};
            if (wq) mats.push_back(ChainMat{Q, ldq, 0, qz0, qz1});
            TRY(chain(mats, {ChainWin{w->Qw + x.oq, R0, (int)m, {J, 0, 0}, {n, n, n}}}));
        }
        return 0;
    }
};

int validate(int64_t n, const double *A, int64_t lda, const double *B, int64_t ldb, const double *Q, int64_t ldq,
             const double *Z, int64_t ldz, int wantq, int wantz, const ht_options *opt)
{
    if (n < 0 || n > (int64_t)1 << 20) return HT_EARG_N;
    if (n > 0 && (!A || lda < n)) return HT_EARG_A;
    if (n > 0 && (!B || ldb < n)) return HT_EARG_B;
    if (n > 0 && wantq && (!Q || ldq < n)) return HT_EARG_Q;
    if (n > 0 && wantz && (!Z || ldz < n)) return HT_EARG_Z;
    if (wantq != 0 && wantq != 1) return HT_EARG_WANTQ;
    if (wantz != 0 && wantz != 1) return HT_EARG_WANTZ;
    if (opt && opt->nb > ((int64_t)1 << 20)) return HT_EARG_NB;
    if (opt && (opt->n_force_ir_fail < 0 || (opt->n_force_ir_fail > 0 && !opt->force_ir_fail))) return HT_EARG_OPT;
    if (opt && (opt->flags & ~(HT_FLAG_GENERAL_B | HT_FLAG_DEFLATE_ZERO_COLUMNS | HT_FLAG_SOLVE128))) return HT_EARG_OPT;
    if (opt && (opt->row_begin != 0 || opt->row_end != 0) &&
        (opt->row_begin < 0 || opt->row_end > n || opt->row_begin > opt->row_end))
        return HT_EARG_OPT;
    return 0;
}

// Algorithmic HBM bytes of one panel: per solve, the trailing B triangle
// once (the factored solve reads the packed Bt = Dinv B, the same element count) and one fused
// sweep over A(s+1:n, j+1:n) and the upper part of B(s+1:n, j+1:n) (P4's B w and P5's A v);
// every IR step repeats both.
double panel_elems_sweep(int64_t n, int64_t s0, int64_t i)
{
    const double M = (double)(n - s0 - 1), c = (double)(n - (s0 + i) - 1);
    return M * c + (double)i * c + c * (c + 1) / 2.0;  // A block + B rows s+1..j + B triangle
}
double panel_bytes(int64_t n, int64_t s0, int64_t k, int64_t ir_steps)
{
    const double M = (double)(n - s0 - 1);
    const double tri = M * (M + 1) / 2.0;
    double e = 0.0;
    for (int64_t i = 0; i < k; ++i) e += tri + panel_elems_sweep(n, s0, i);
    e += (double)ir_steps * (tri + panel_elems_sweep(n, s0, k / 2));
    return 8.0 * e;
}

double panel_flops(int64_t n, int64_t s0, int64_t k, int64_t ir_steps)
{
    const double M = (double)(n - s0 - 1);
    double f = 0.0;
    for (int64_t i = 0; i < k; ++i) {
        f += M * M + 2.0 * panel_elems_sweep(n, s0, i);  // factored solve (trsv) + fused sweep
        f += (4.0 * n + 22.0 * M) * (double)i;           // small WY terms
    }
    f += (double)ir_steps * (M * M + 2.0 * panel_elems_sweep(n, s0, k / 2));  // IR: solve + sweep
    return f;
}

}  // namespace

extern "C" {

const char *ht_strerror(int code)
{
    switch (code) {
    case HT_OK: return "ok";
    case HT_EARG_N: return "invalid n";
    case HT_EARG_A: return "invalid A / lda";
    case HT_EARG_B: return "invalid B / ldb, or B not upper triangular";
    case HT_EARG_Q: return "invalid Q / ldq";
    case HT_EARG_Z: return "invalid Z / ldz";
    case HT_EARG_OPT: return "invalid options";
    case HT_ENONFINITE: return "A or B contains Inf/NaN";
    case HT_ECUDA: return "CUDA error or no CUDA device";
    case HT_ENOMEM: return "device allocation failed";
    case HT_ENUMERIC: return "internal numerical guard";
    default: return "unknown error";
    }
}

int ht_version(void) { return 100; }

int ht_bench_chain_apply(int64_t rows, int p, int nwin, int left, int reps, double *seconds, double *flops)
{
    if (rows < 1 || p < 2 || p > 512 || nwin < 1) return HT_EARG_N;
    if (reps < 1) reps = 1;
    const int64_t half = p / 2, width = (int64_t)(nwin - 1) * half + p;
    double *X = nullptr, *Qw = nullptr;
    ChainWin *dw = nullptr;
    int rc = HT_OK;
    if (cudaMalloc((void **)&X, (size_t)rows * width * sizeof(double)) != cudaSuccess ||
        cudaMalloc((void **)&Qw, (size_t)p * p * sizeof(double)) != cudaSuccess ||
        cudaMalloc((void **)&dw, (size_t)nwin * sizeof(ChainWin)) != cudaSuccess)
        rc = HT_ENOMEM;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (rc == HT_OK) {
        std::vector<ChainWin> hw(nwin);
        for (int i = 0; i < nwin; ++i) hw[i] = ChainWin{Qw, (int64_t)i * half, p, {0, 0, 0}, {rows, rows, rows}};
        const int64_t ld = left ? width : rows;
        ChainMat m{X, ld, left, 0, rows};
        if (cudaMemset(X, 0, (size_t)rows * width * sizeof(double)) != cudaSuccess ||
            cudaMemset(Qw, 0, (size_t)p * p * sizeof(double)) != cudaSuccess ||
            cudaMemcpy(dw, hw.data(), nwin * sizeof(ChainWin), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
            rc = HT_ECUDA;
        float best = 1e30f;
        for (int it = 0; it <= reps && rc == HT_OK; ++it) {  // first launch: warm-up
            cudaEventRecord(e0, 0);
            rc = ht_chain_apply(0, &m, 1, dw, nwin, p, 0);
            cudaEventRecord(e1, 0);
            if (cudaEventSynchronize(e1) != cudaSuccess) rc = HT_ECUDA;
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it > 0 && ms < best) best = ms;
        }
        if (rc == HT_OK) {
            if (seconds) *seconds = best * 1e-3;
            if (flops) *flops = 2.0 * (double)rows * p * (double)p * nwin;
        }
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaFree(X);
    cudaFree(Qw);
    cudaFree(dw);
    return rc;
}

int ht_release_workspace(void)
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return HT_ECUDA;
    if (dev < 0 || dev >= 16) return HT_OK;
    {
        std::lock_guard<std::mutex> lk(g_hmu[dev]);
        host_stage_free(g_hst[dev]);
    }
    std::lock_guard<std::mutex> lk(g_mu[dev]);
    work_free(g_work[dev]);
    return HT_OK;
}

}  // extern "C"

namespace {

// Everything of one reduction after the caller's stream has forked into R.st.  Any error
// return leaves work queued on the library streams; ht_reduce_ex drains them.
int reduce_body(Run &R, const ht_options *opt)
{
    Work *w = R.w;
    cudaStream_t st = R.st;
    const int64_t n = R.n, nb = R.nb;
    double *dA = R.A, *dB = R.B, *dQ = R.Q, *dZ = R.Z;
    const int64_t ldda = R.lda, lddb = R.ldb, lddq = R.ldq, lddz = R.ldz;
    unsigned long long *d_max = reinterpret_cast<unsigned long long *>(w->d_scal + 4);

    // validation that needs the data: finite entries, B upper triangular (before any write);
    // the same pass finds max|A|, max|B| for the range scaling below
    TRY(ht_check_input(st, n, dA, ldda, dB, lddb, w->d_iflags, d_max));
    HT_CUDA_TRY(cudaMemcpyAsync(w->h_iflags, w->d_iflags, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    HT_CUDA_TRY(cudaMemcpyAsync(w->h_scal + 4, d_max, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    HT_CUDA_TRY(cudaStreamSynchronize(st));
    const uint32_t flags = opt ? opt->flags : 0u;
    if (w->h_iflags[0]) return HT_ENONFINITE;
    if (w->h_iflags[1] && !(flags & HT_FLAG_GENERAL_B)) return HT_EARG_B;
    // exact power-of-two range scaling (include/ht.h "Range"): squared norms of columns,
    // reflectors and ||B||_F stay finite and normal; no rounding is introduced, and the
    // result is bitwise that of the unscaled computation whenever no scaling is needed
    auto pick = [](double mx) -> double {
        if (!(mx > 0.0) || (mx >= 0x1p-100 && mx <= 0x1p100)) return 1.0;
        return ldexp(1.0, -ilogb(mx));
    };
    const double sa = pick(w->h_scal[4]), sb = pick(w->h_scal[5]);
    R.rep.scale_a = sa;
    R.rep.scale_b = sb;
    TRY(ht_scale(st, n, n, dA, ldda, sa));
    TRY(ht_scale(st, n, n, dB, lddb, sb));

    HT_CUDA_TRY(cudaEventRecord(w->ev_t0, st));
    R.tm.base = w->ev_t0;
    if (R.wq) TRY(ht_fill2d(st, n, n, dQ, lddq, 0.0, 1.0));
    if (R.wz) TRY(ht_fill2d(st, n, n, dZ, lddz, 0.0, 1.0));
    int64_t s_begin = 0;
    if (n > 2 && (flags & (HT_FLAG_GENERAL_B | HT_FLAG_DEFLATE_ZERO_COLUMNS))) {
        const auto f0 = std::chrono::steady_clock::now();
        TRY(R.front_end(flags, &s_begin));
        HT_CUDA_TRY(cudaStreamSynchronize(st));
        R.rep.t_front = std::chrono::duration<double>(std::chrono::steady_clock::now() - f0).count();
        R.rep.deflated_columns = s_begin;
    }
    int64_t ndesing = 0;
    if (n > 2) {
        TRY(ht_fro_norm_sq(st, n, n, dB, lddb, w->d_scal, w->fro_part));
        HT_CUDA_TRY(cudaMemcpyAsync(w->h_scal, w->d_scal, sizeof(double), cudaMemcpyDeviceToHost, st));
        HT_CUDA_TRY(cudaStreamSynchronize(st));
        const double nB = sqrt(w->h_scal[0]);
        const double tolf = (opt && opt->tol_factor > 0) ? opt->tol_factor : 2.0;
        const int max_ir = (opt && opt->max_ir > 0) ? opt->max_ir : 10;
        const uint64_t seed = opt ? opt->seed : 0;
        int nforce = 0;
        if (opt && opt->n_force_ir_fail > 0) {
            std::vector<int64_t> fl(opt->force_ir_fail, opt->force_ir_fail + opt->n_force_ir_fail);
            std::sort(fl.begin(), fl.end());
            nforce = (int)std::min<int64_t>((int64_t)fl.size(), w->ncap);
            HT_CUDA_TRY(cudaMemcpyAsync(w->d_force, fl.data(), nforce * sizeof(int64_t), cudaMemcpyHostToDevice, st));
            HT_CUDA_TRY(cudaStreamSynchronize(st));
        }
        HT_CUDA_TRY(cudaMemsetAsync(w->d_iflags, 0, sizeof(int), st));
        HT_CUDA_TRY(cudaMemsetAsync(w->d_irtrace, 0, (size_t)n * sizeof(int), st));
        // development switches (HT_DEBUG_IR, HT_PROFILE, HT_TRACE_COL, HT_FPROF): diagnostics
        // printed to stderr; they add instrumentation but never change the arithmetic
        struct DevBuf {
            void *p = nullptr;
            ~DevBuf() { if (p) cudaFree(p); }
        } dbg_buf, prof_buf, ttr_buf, fprof_buf;
        double *dbg = nullptr;
        const bool dbg_on = getenv("HT_DEBUG_IR") != nullptr;
        double *ptime = nullptr;
        const bool prof_on = getenv("HT_PROFILE") != nullptr;
        if (prof_on) {
            HT_CUDA_TRY(cudaMalloc(&prof_buf.p, 16 * sizeof(double)));
            ptime = (double *)prof_buf.p;
            HT_CUDA_TRY(cudaMemset(ptime, 0, 16 * sizeof(double)));
        }
        if (dbg_on) {
            HT_CUDA_TRY(cudaMalloc(&dbg_buf.p, (size_t)n * 12 * sizeof(double)));
            dbg = (double *)dbg_buf.p;
            HT_CUDA_TRY(cudaMemset(dbg, 0, (size_t)n * 12 * sizeof(double)));
        }
        unsigned long long *ttr = nullptr;
        const int64_t tcol = getenv("HT_TRACE_COL") ? atoll(getenv("HT_TRACE_COL")) : -1;
        if (tcol >= 0) {
            const size_t nt = (size_t)((n - 1 + 63) / 64 + 4) * 8;  // 64-row units (trsv4r) or 128-row blocks
            HT_CUDA_TRY(cudaMalloc(&ttr_buf.p, nt * sizeof(unsigned long long)));
            ttr = (unsigned long long *)ttr_buf.p;
            HT_CUDA_TRY(cudaMemset(ttr, 0, nt * sizeof(unsigned long long)));
        }
        unsigned long long *fprof = nullptr;
        if (getenv("HT_FPROF")) {
            HT_CUDA_TRY(cudaMalloc(&fprof_buf.p, 32 * sizeof(unsigned long long)));
            fprof = (unsigned long long *)fprof_buf.p;
            HT_CUDA_TRY(cudaMemset(fprof, 0, 32 * sizeof(unsigned long long)));
            TRY(ht_factor_set_prof(fprof));
        }
        int64_t s0 = s_begin;  // > 0 after the sec. 3.5.1 preprocessing: only the trailing pencil
        while (s0 <= n - 3) {
            const int64_t kmax = std::min<int64_t>(nb, n - 2 - s0);
            TRY(ht_desingularize(st, n, dB, lddb, s0 + 1, HT_U * nB, 2.0 * HT_U * nB, seed, s0, w->d_iflags));
            HT_CUDA_TRY(cudaMemsetAsync(w->S, 0, (size_t)nb * nb * sizeof(double), st));
            HT_CUDA_TRY(cudaMemsetAsync(w->T, 0, (size_t)nb * nb * sizeof(double), st));
            PanelArgs pa;
            memset(&pa, 0, sizeof(pa));
            pa.n = n; pa.lda = ldda; pa.ldb = lddb; pa.A = dA; pa.B = dB;
            pa.s0 = s0; pa.kmax = (int)kmax; pa.nb = (int)nb;
            pa.U = w->U; pa.V = w->V; pa.Y = w->Y; pa.S = w->S; pa.T = w->T;
            double *vv = w->vec;
            const int64_t N = w->ncap;
            pa.vsave = vv; pa.vrhs = vv + N; pa.vy = vv + 2 * N; pa.vx = vv + 3 * N;
            pa.vw = vv + 4 * N; pa.vw2 = vv + 5 * N; pa.vr = vv + 6 * N;
            pa.part = w->part; pa.pw = (int)nb + 8;
            pa.yll = w->yll; pa.yll_exp = w->yll_exp; pa.bexp = w->bexp; pa.epoch = w->epoch;
            pa.Dinv = w->Dinv; pa.Bt = w->Bt; pa.ldbt = n; pa.dsafe = w->dsafe; pa.ypart = w->ypart;
            pa.Dinv4 = (flags & HT_FLAG_SOLVE128) ? nullptr : w->Dinv4;  // null: 128-row solve only
            pa.dsafe4 = w->dsafe4; pa.h_dsafe4 = w->h_dsafe4;
            pa.ypartB = w->ypartB; pa.BV = w->BV; pa.vbx = vv + 7 * N;
            pa.hot = w->hot; pa.hot_bytes = w->hot_bytes;
            pa.sweep_ctr = reinterpret_cast<unsigned *>(w->wave_ticket + 2);
            pa.tol = tolf * HT_U * nB; pa.max_ir = max_ir;
            pa.force_fail = w->d_force; pa.n_force_fail = nforce;
            pa.out = w->d_out;
            pa.irtrace = w->d_irtrace;
            pa.dbg = dbg;
            pa.ttrace = ttr;
            pa.tcol = tcol;
            pa.ptime = ptime;
            const int64_t M = n - s0 - 1;
            int G = (int)std::min<int64_t>(w->gmax, std::max<int64_t>(1, (M + 31) / 32));
            R.ph.mark(st, 7);
            R.tm.begin(st, 0);
            TRY(ht_panel_run(st, &pa, G));
            R.tm.end(st);
            R.ph.mark(st, 0);
            HT_CUDA_TRY(cudaMemcpyAsync(w->h_out, w->d_out, 6 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            HT_CUDA_TRY(cudaStreamSynchronize(st));
            const auto h0 = std::chrono::steady_clock::now();
            const size_t done = R.tm.pending.size();  // complete: st has passed the joins of every stream
            R.ph.resolve();
            const auto h1 = std::chrono::steady_clock::now();
            const int64_t k = w->h_out[0];
            const int failed = (int)w->h_out[1];
            w->epoch = (unsigned)w->h_out[5] + 1;
            R.rep.panels++;
            R.rep.absorptions++;
            R.rep.ir_steps_total += w->h_out[2];
            R.rep.ir_extra_columns += w->h_out[3];
            R.rep.solve_rescales += w->h_out[4];
            if (failed) { R.rep.ir_failed_columns++; R.rep.premature_absorptions++; }
            R.extra_flops += panel_flops(n, s0, k, w->h_out[2]);
            R.rep.panel_bytes += panel_bytes(n, s0, k, w->h_out[2]);
            if (k <= 0) return HT_ENUMERIC;
            TRY(R.absorb(s0, k));
            R.tm.resolve(done);
            if (R.ph.on) {
                const auto h2 = std::chrono::steady_clock::now();
                R.ph.host[0] += std::chrono::duration<double>(h1 - h0).count();
                R.ph.host[1] += std::chrono::duration<double>(h2 - h1).count();
            }
            s0 += k;
            if (opt && opt->max_panels > 0 && R.rep.panels >= opt->max_panels) break;
        }
        HT_CUDA_TRY(cudaMemcpyAsync(w->h_iflags, w->d_iflags, sizeof(int), cudaMemcpyDeviceToHost, st));
        HT_CUDA_TRY(cudaStreamSynchronize(st));
        ndesing = w->h_iflags[0];
        if (prof_on) {
            double hp[16];
            HT_CUDA_TRY(cudaMemcpy(hp, ptime, sizeof(hp), cudaMemcpyDeviceToHost));
            const char *names[16] = {"P1.sync2", "P2+trsv", "P3 rest", "P4 r+IR", "P4 sweep", "P5", "P4 VTx,TVTx", "P4 sums+UTw2",
                                     "P1.Yv", "P1.UTa", "P1.sync1", "P1.gather", "P1.S^T", "P1.U(S^T)", "P1.tail", ""};
            fprintf(stderr, "[ht profile] panel phases (s):");
            for (int i = 0; i < 15; ++i) fprintf(stderr, " %s=%.4f", names[i], hp[i]);
            fprintf(stderr, "\n");
        }
        if (fprof) {
            HT_CUDA_TRY(cudaDeviceSynchronize());
            unsigned long long hp[32];
            HT_CUDA_TRY(cudaMemcpy(hp, fprof, sizeof(hp), cudaMemcpyDeviceToHost));
            fprintf(stderr, "[ht fprof] factor phases (s): load %.3f left[X %.3f TX %.3f upd %.3f] steps %.3f leafupd %.3f "
                            "write %.3f G %.3f T %.3f offT %.3f zero %.3f | vt calls %llu stage %.0f dmma %.0f cyc/call\n",
                    hp[0] * 1e-9, hp[8] * 1e-9, hp[9] * 1e-9, hp[10] * 1e-9, hp[2] * 1e-9, hp[3] * 1e-9, hp[4] * 1e-9,
                    hp[11] * 1e-9, hp[5] * 1e-9, hp[6] * 1e-9, hp[7] * 1e-9, hp[26], hp[24] / (double)(hp[26] ? hp[26] : 1),
                    hp[25] / (double)(hp[26] ? hp[26] : 1));
            TRY(ht_factor_set_prof(nullptr));
        }
        if (ttr) {
            const int nbk = (int)((n - 1 + 63) / 64) + 4;
            std::vector<unsigned long long> h((size_t)nbk * 8);
            HT_CUDA_TRY(cudaMemcpy(h.data(), ttr, h.size() * 8, cudaMemcpyDeviceToHost));
            unsigned long long t0 = ~0ull;
            for (auto v : h)
                if (v && v < t0) t0 = v;
            fprintf(stderr, "[ht trace] col %lld: block: start stage_done lastload lastfetch tiles_done wait_done matvec_done publish (us)\n", (long long)tcol);
            auto us = [&](unsigned long long v) { return v ? (v - t0) * 1e-3 : -1.0; };
            for (int b = nbk - 1; b >= 0; --b)
                if (h[8 * b + 2])
                    fprintf(stderr, "[ht trace] %3d: %8.2f %8.2f %8.2f %8.2f %8.2f %8.2f %8.2f %8.2f\n", b, us(h[8 * b + 4]), us(h[8 * b + 5]),
                            us(h[8 * b + 7]), us(h[8 * b + 6]), us(h[8 * b + 0]), us(h[8 * b + 1]), us(h[8 * b + 3]), us(h[8 * b + 2]));
        }
        if (dbg_on) {
            std::vector<double> hd((size_t)n * 12);
            HT_CUDA_TRY(cudaMemcpy(hd.data(), dbg, hd.size() * sizeof(double), cudaMemcpyDeviceToHost));
            for (int64_t j = 0; j < n; ++j) {
                if (hd[j * 12] == 0.0) continue;
                fprintf(stderr, "[ht dbg] col %lld:", (long long)j);
                for (int it = 0; it < 12 && hd[j * 12 + it] != 0.0; ++it) fprintf(stderr, " %.3g", hd[j * 12 + it]);
                fprintf(stderr, "\n");
            }
        }
        if (opt && opt->ir_trace) {
            std::vector<int> tr(n);
            HT_CUDA_TRY(cudaMemcpy(tr.data(), w->d_irtrace, n * sizeof(int), cudaMemcpyDeviceToHost));
            for (int64_t j = 0; j < n; ++j) opt->ir_trace[j] = tr[j];
        }
    }
    // exact structural zeros of H and T (Alg. 2 "Set ... <- 0"), undo the
    // range scaling, and check the result for non-finite entries -- one pass
    TRY(ht_finish(st, n, dA, ldda, dB, lddb, R.wq ? dQ : nullptr, lddq, R.wz ? dZ : nullptr, lddz, 1.0 / sa, 1.0 / sb,
                  (opt && opt->max_panels > 0) ? 1 : 0, w->d_iflags + 4));
    R.tm.launches++;
    HT_CUDA_TRY(cudaEventRecord(w->ev_t1, st));
    HT_CUDA_TRY(cudaMemcpyAsync(w->h_iflags + 4, w->d_iflags + 4, sizeof(int), cudaMemcpyDeviceToHost, st));
    HT_CUDA_TRY(cudaStreamSynchronize(st));
    R.tm.resolve();
    R.ph.mark(st, 7);
    HT_CUDA_TRY(cudaStreamSynchronize(st));
    R.ph.resolve();
    R.ph.print();
    R.rep.t_panel = R.tm.acc[0];
    R.rep.t_gemm = R.tm.acc[1];
    R.rep.t_factor = R.tm.acc[2] + R.tm.acc[7];
    R.rep.t_other = R.tm.acc[3];
    R.rep.t_chain = R.tm.acc[4];
    R.rep.t_chain_busy = R.tm.busy4();
    R.rep.t_absorb_right = R.tm.acc[5];
    R.rep.t_absorb_left = R.tm.acc[6];
    R.rep.t_factor_exposed = R.tm.acc[7];
    R.rep.flops_chain = R.chain_flops;
    R.rep.chain_launches = R.chain_launches;
    R.rep.launches = R.tm.launches;
    float ms = 0.f;
    HT_CUDA_TRY(cudaEventElapsedTime(&ms, w->ev_t0, w->ev_t1));
    HT_CUDA_TRY(cudaGetLastError());
    R.rep.seconds = ms * 1e-3;
    R.rep.flops_level3 = g_ht_flops;
    R.rep.flops = g_ht_flops + R.extra_flops;
    R.rep.desingularizations = ndesing;
    if (w->h_iflags[4]) return HT_ENUMERIC;
    return HT_OK;
}

// After an error: wait for every library stream so that no queued kernel keeps writing the
// caller's buffers or the workspace once we return (errors are ignored: a sticky CUDA error
// makes every call fail).
void drain(Work *w)
{
    cudaStream_t ss[] = {w->hp_stream, w->sA, w->sQZ, w->sB, w->side_stream, w->sA2, w->sQZ2};
    for (cudaStream_t s : ss)
        if (s) cudaStreamSynchronize(s);
}

// One reduction on the current device: the single-GPU entry point (P = 1) and one rank of
// the multi-GPU one (P > 1: rank `me` with NCCL `comm`, or every rank when comm is NULL).
int reduce_impl(int64_t n, double *dA, int64_t ldda, double *dB, int64_t lddb, double *dQ, int64_t lddq, double *dZ,
                int64_t lddz, int wantq, int wantz, const ht_options *opt, ht_report *rep, int P, int me, void *comm,
                int gather_qz)
{
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return HT_ECUDA;
    int dev = 0;
    HT_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 16) return HT_ECUDA;
    std::lock_guard<std::mutex> lk(g_mu[dev]);
    int64_t nb = (opt && opt->nb > 0) ? opt->nb : 128;
    nb = std::max<int64_t>(1, std::min<int64_t>({nb, 256, std::max<int64_t>(1, n - 2)}));
    Work *w = nullptr;
    TRY(work_get(dev, n, nb, &w));
    if (P > 1) {  // packed all-gather staging: P + 1 chunks of at most ceil(n / P) x n doubles
        const size_t need = (size_t)(P + 1) * (size_t)((n + P - 1) / P) * (size_t)n;
        if (w->mgcap < need) {
            if (w->mgbuf) cudaFree(w->mgbuf);
            w->mgbuf = nullptr;
            w->mgcap = 0;
            if (cudaMalloc((void **)&w->mgbuf, need * sizeof(double)) != cudaSuccess) return HT_ENOMEM;
            w->mgcap = need;
        }
    }
    Run R;
    memset(&R.rep, 0, sizeof(R.rep));
    R.w = w;
    // the caller's stream forks into the library's high-priority stream and joins it at the end
    // (NULL is the legacy default stream, exactly as in the CUDA runtime: work the caller
    //  queued there, e.g. the copies that produced A and B, is ordered before the reduction)
    const cudaStream_t user_st = opt ? (cudaStream_t)opt->stream : (cudaStream_t)0;
    R.st = w->hp_stream;
    HT_CUDA_TRY(cudaEventRecord(w->ev[9], user_st));
    HT_CUDA_TRY(cudaStreamWaitEvent(R.st, w->ev[9], 0));
    R.n = n; R.nb = nb;
    R.A = dA; R.B = dB; R.Q = dQ; R.Z = dZ;
    R.lda = ldda; R.ldb = lddb; R.ldq = lddq; R.ldz = lddz;
    R.wq = wantq != 0; R.wz = wantz != 0;
    R.P = P; R.me = me; R.comm = comm;
    R.qz0 = 0; R.qz1 = n;
    if (opt && (opt->row_begin != 0 || opt->row_end != 0)) { R.qz0 = opt->row_begin; R.qz1 = opt->row_end; }
    if (P > 1 && comm) ht_slab(0, n, P, me, &R.qz0, &R.qz1);  // Q, Z: this rank's row slab
    g_ht_flops = 0.0;
    int rc = reduce_body(R, opt);
    if (rc == HT_OK && P > 1 && gather_qz) {  // C6: every rank gets the full Q, Z (not in rep.seconds)
        if (R.wq) rc = R.gather(R.st, dQ, lddq, 0, n, 0, n, 0);
        if (rc == HT_OK && R.wz) rc = R.gather(R.st, dZ, lddz, 0, n, 0, n, 0);
        if (rc == HT_OK && cudaStreamSynchronize(R.st) != cudaSuccess) rc = HT_ECUDA;
    }
    if (rc != HT_OK) drain(w);
    // join: the caller's stream is ordered after everything the call queued
    if (cudaEventRecord(w->ev[10], R.st) == cudaSuccess) cudaStreamWaitEvent(user_st, w->ev[10], 0);
    if (rep && (rc == HT_OK || rc == HT_ENUMERIC)) *rep = R.rep;
    return rc;
}

}  // namespace

extern "C" {

int ht_reduce_ex(int64_t n, double *dA, int64_t ldda, double *dB, int64_t lddb, double *dQ, int64_t lddq, double *dZ,
                 int64_t lddz, int wantq, int wantz, const ht_options *opt, ht_report *rep)
{
    int rc = validate(n, dA, ldda, dB, lddb, dQ, lddq, dZ, lddz, wantq, wantz, opt);
    if (rc) return rc;
    if (n == 0) {
        if (rep) memset(rep, 0, sizeof(*rep));
        return HT_OK;
    }
    return reduce_impl(n, dA, ldda, dB, lddb, dQ, lddq, dZ, lddz, wantq, wantz, opt, rep, 1, 0, nullptr, 0);
}

int ht_reduce_mg(int64_t n, const ht_mg_layout *L, void *nccl_comm, int rank, int nranks, int wantq, int wantz,
                 const ht_options *opt, ht_report *rep)
{
    if (!L) return HT_EARG_OPT;
    int rc = validate(n, L->A, L->lda, L->B, L->ldb, L->Q, L->ldq, L->Z, L->ldz, wantq, wantz, opt);
    if (rc) return rc;
    if (nranks < 1 || (nccl_comm && (rank < 0 || rank >= nranks))) return HT_EARG_OPT;
    if (opt && (opt->row_begin != 0 || opt->row_end != 0)) return HT_EARG_OPT;  // the layout decides the slabs
    if (n == 0) {
        if (rep) memset(rep, 0, sizeof(*rep));
        return HT_OK;
    }
    if (nccl_comm && nranks > 1) {
        rc = ht_mg_check_comm(nccl_comm, rank, nranks);
        if (rc) return rc;
    }
    return reduce_impl(n, L->A, L->lda, L->B, L->ldb, L->Q, L->ldq, L->Z, L->ldz, wantq, wantz, opt, rep, nranks,
                       nccl_comm ? rank : 0, nranks > 1 ? nccl_comm : nullptr, L->gather_qz);
}

int ht_reduce_host(int64_t n, const double *A, const double *B, double *H, double *T, double *Q, double *Z,
                   int wantq, int wantz, int64_t nb)
{
    int rc = validate(n, A, n, B, n, Q, n, Z, n, wantq, wantz, nullptr);
    if (rc) return rc;
    if (n > 0 && !H) return HT_EARG_A;
    if (n > 0 && !T) return HT_EARG_B;
    if (n == 0) return HT_OK;
    int ndev = 0, dev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0 || cudaGetDevice(&dev) != cudaSuccess) return HT_ECUDA;
    if (dev < 0 || dev >= 16) return HT_ECUDA;
    const size_t bytes = (size_t)n * n * sizeof(double);
    std::lock_guard<std::mutex> lk(g_hmu[dev]);
    HostStage &hs = g_hst[dev];
    if (hs.bytes < bytes) {
        host_stage_free(hs);
        for (int i = 0; i < 4; ++i)
            if (cudaMalloc((void **)&hs.d[i], bytes) != cudaSuccess) {
                cudaGetLastError();
                host_stage_free(hs);
                return HT_ENOMEM;
            }
        hs.bytes = bytes;
    }
    if (!hs.st && cudaStreamCreateWithFlags(&hs.st, cudaStreamNonBlocking) != cudaSuccess) return HT_ECUDA;
    double **d = hs.d;
    if (cudaMemcpyAsync(d[0], A, bytes, cudaMemcpyHostToDevice, hs.st) != cudaSuccess ||
        cudaMemcpyAsync(d[1], B, bytes, cudaMemcpyHostToDevice, hs.st) != cudaSuccess) {
        cudaStreamSynchronize(hs.st);
        return HT_ECUDA;
    }
    ht_options opt;
    memset(&opt, 0, sizeof(opt));
    opt.nb = nb;
    opt.stream = hs.st;
    rc = ht_reduce_ex(n, d[0], n, d[1], n, wantq ? d[2] : nullptr, n, wantz ? d[3] : nullptr, n, wantq, wantz, &opt,
                      nullptr);
    if (rc == HT_OK) {
        if (cudaMemcpyAsync(H, d[0], bytes, cudaMemcpyDeviceToHost, hs.st) != cudaSuccess ||
            cudaMemcpyAsync(T, d[1], bytes, cudaMemcpyDeviceToHost, hs.st) != cudaSuccess ||
            (wantq && cudaMemcpyAsync(Q, d[2], bytes, cudaMemcpyDeviceToHost, hs.st) != cudaSuccess) ||
            (wantz && cudaMemcpyAsync(Z, d[3], bytes, cudaMemcpyDeviceToHost, hs.st) != cudaSuccess))
            rc = HT_ECUDA;
    }
    if (cudaStreamSynchronize(hs.st) != cudaSuccess && rc == HT_OK) rc = HT_ECUDA;
    return rc;
}

int ht_reduce(int64_t n, double *A, double *B, double *Q, double *Z, int wantq, int wantz, int64_t nb)
{
    return ht_reduce_host(n, A, B, A, B, Q, Z, wantq, wantz, nb);
}

}  // extern "C"
