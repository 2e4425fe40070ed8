/*
 * include/ht.h -- C ABI of the B200-native HouseHT library (libht_b200.so).
 *
 * Householder-based Hessenberg-triangular (HT) reduction of a real FP64 pencil
 * A - lambda*B with B upper triangular (Bujanovic, Karlsson, Kressner,
 * arXiv 1710.08538; PAPER.md).  The problem statement this ABI follows
 * (sec. 1): find orthogonal Q, Z such that
 *     H = Q^T A Z   is upper Hessenberg   and   T = Q^T B Z   is upper triangular,
 * with B "already reduced to triangular form" and Q, Z "initialized to
 * identity"; signature [H, T, Q, Z] = HouseHT(A, B) (Algorithm 1,
 * P:1219).  The method is Algorithm 1: panels of nb columns
 * reduced by left Householder reflectors and opposite (right) reflectors from
 * a solve with B (sec. 3.2), accumulated in compact WY form and absorbed into
 * A, B, Q, Z by staircase transformations (sec. 3.3).
 *
 * Conventions (all entry points):
 *   - FP64 (IEEE binary64), column-major storage.
 *   - On success A is overwritten by H (exact zeros below the first
 *     sub-diagonal) and B by T (exact zeros below the diagonal).
 *   - If wantq != 0, Q is OVERWRITTEN with the accumulated orthogonal factor
 *     (initialised internally to I; Q e1 = e1).  If wantq == 0, Q may be NULL
 *     and is never referenced.  Likewise Z / wantz.
 *   - nb <= 0 selects the default 128; otherwise nb is clamped to
 *     [1, min(256, max(1, n-2))].  nb changes speed, not the result beyond
 *     rounding (the HT form is unique up to signs for nonsingular B).
 *   - n = 0: nothing is touched, HT_OK.  n in {1, 2}: H = A, T = B, Q = Z = I.
 *   - Iterative-refinement failures are NOT errors: they trigger a premature
 *     absorption and are reported in ht_report.
 *
 * Error behaviour: arguments are validated before any write -- on a negative
 * return code every buffer is untouched.  Positive codes are runtime errors
 * after which buffer contents are unspecified (except HT_ENONFINITE and
 * HT_EARG_B, detected before any write).  On every return the library's
 * internal streams have finished all work of the call (nothing keeps writing the
 * caller's buffers), and the caller's stream is ordered after the call.
 *
 * Range: inputs are scaled by exact powers of two at entry when max|A| or max|B|
 * lies outside [2^-100, 2^100] (undone on H, T at exit; Q, Z are invariant), so
 * any finite pencil is accepted; a non-finite entry in the result is reported as
 * HT_ENUMERIC.
 *
 * Ownership: the caller owns A, B, Q, Z (host memory for ht_reduce, device
 * memory for ht_reduce_ex).  The library owns its device workspace (cached per
 * device, reused across calls) and keeps no caller pointer after returning.
 * Calls on the same device are serialised by an internal per-device mutex;
 * calls on different devices (e.g. one host thread per GPU) run concurrently.
 *
 * No CPU fallback exists: without a CUDA device every entry point returns
 * HT_ECUDA.
 */
#ifndef HT_B200_H
#define HT_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define HT_API __attribute__((visibility("default")))
#else
#define HT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
    HT_OK = 0,
    HT_EARG_N = -1,     /* n < 0 or too large                                  */
    HT_EARG_A = -2,     /* A == NULL (n > 0) or lda < n                         */
    HT_EARG_B = -3,     /* B == NULL, ldb < n, or B not upper triangular        */
    HT_EARG_Q = -4,     /* wantq and (Q == NULL or ldq < n)                     */
    HT_EARG_Z = -5,     /* wantz and (Z == NULL or ldz < n)                     */
    HT_EARG_WANTQ = -6, /* wantq not 0 or 1                                     */
    HT_EARG_WANTZ = -7, /* wantz not 0 or 1                                     */
    HT_EARG_NB = -8,    /* nb > 2^20 (absurd; nb <= 0 selects the default)      */
    HT_EARG_OPT = -9,   /* invalid ht_options                                   */
    HT_ENONFINITE = 1,  /* A or B holds Inf/NaN (detected before any write)     */
    HT_ECUDA = 2,       /* CUDA runtime error / no device                       */
    HT_ENOMEM = 3,      /* device allocation failed                             */
    HT_ENUMERIC = 4,    /* internal numerical guard tripped: a non-finite entry in H, T, Q or Z */
    HT_ENCCL = 5        /* NCCL error (ht_reduce_mg)                                            */
};

/* Options for ht_reduce_ex (zero-initialise, then set what you need). */
typedef struct {
    int64_t nb;            /* panel width; <= 0 -> 128                                   */
    int max_ir;            /* max IR corrections per column; <= 0 -> 10          */
    double tol_factor;     /* IR tolerance factor c in c*u*||B||_F; <= 0 -> 2    */
    uint64_t seed;         /* seed of the desingularisation draws rho            */
    void *stream;          /* cudaStream_t the reduction is ordered on (NULL: the legacy
                              default stream); the library forks its own streams from it */
    const int64_t *force_ir_fail; /* host array of 0-based columns whose solve is forced
                                     to fail IR (test hook for premature absorption)   */
    int64_t n_force_ir_fail;
    int32_t *ir_trace;     /* optional host array of length n: on return, the number of IR
                              corrections column j needed (+1000 if an earlier attempt at
                              column j failed and triggered a premature absorption)       */
    int64_t max_panels;    /* test hook: stop after this many panel+absorption steps (0 = all);
                              the output is then a partial reduction with A = Q^T A0 Z etc. */
    /* Multi-GPU row slab: unless both are 0, only rows [row_begin, row_end) of Q and Z
       are computed (Q and Z only receive right multiplications, so their rows are
       independent).  A, B (H, T) are computed in
       full on every caller.  Rows of Q, Z outside the slab are left unspecified.
       0, 0 = all rows.  Requires 0 <= row_begin <= row_end <= n, else HT_EARG_OPT. */
    int64_t row_begin;
    int64_t row_end;
    /* HT_FLAG_* below (0 = the plain reduction of a triangular B) */
    uint32_t flags;
} ht_options;

/* ht_options.flags */
/* QZ step 1 front end: B may be a general square matrix; the library
   first computes B = Q0 R (Householder QR by panels, each panel reduced by a staircase of
   2k x k window QRs as in sec. 3.3.2b), A <- Q0^T A, B <- R, and the returned Q includes Q0.
   (Q e1 = e1 then no longer holds.)  Without the flag B must be upper triangular. */
#define HT_FLAG_GENERAL_B 1u
/* Preprocessing of sec. 3.5.1: if B (upper triangular) has l > 0 exactly-zero
   columns, a permutation Z0 moves them first (Q0 = Z0 if B is diagonal, else I), a QR of
   the first l columns of Q0^T A Z0 gives A(:, 1:l) = [A11; 0], the trailing block of B is
   re-triangularised (QR), and only the trailing (n-l) x (n-l) pencil is reduced to HT form.
   The leading l x l part is already in generalised Schur form (T's first l columns are 0). */
#define HT_FLAG_DEFLATE_ZERO_COLUMNS 2u
/* Solve-path selection (verification): the panel's triangular solves (P3, IR corrections) run
   on 256-row blocks with 4-CTA clusters whenever every 256-row diagonal block of the panel's B
   is well conditioned, else on 128-row blocks with 2-CTA clusters.  This flag forces the
   128-row path for every panel; the result agrees to rounding (the same recurrence, blocked
   differently). */
#define HT_FLAG_SOLVE128 4u

/* Statistics of one reduction (the paper's Table 3/4 columns). */
typedef struct {
    double seconds;            /* wall time of the reduction (device events)           */
    double flops;              /* executed FP64 flops, instrumented      */
    double flops_level3;       /* part of `flops` executed by the DMMA GEMM            */
    int64_t panels;            /* panel reductions run                                  */
    int64_t absorptions;       /* absorptions (= panels)                                */
    int64_t premature_absorptions; /* absorptions triggered by an IR failure            */
    int64_t ir_steps_total;    /* IR correction solves                                  */
    int64_t ir_extra_columns;  /* columns that needed >= 1 IR correction               */
    int64_t ir_failed_columns; /* columns whose IR failed (premature absorption)        */
    int64_t desingularizations;/* zero pivots replaced by 2u*rho*||B||_F                */
    int64_t solve_rescales;    /* triangular solves that needed power-of-two rescaling  */
    double t_panel;            /* device seconds in panel kernels (CUDA events)         */
    double t_gemm;             /* device seconds in DMMA GEMM launches (excl. chains)   */
    double t_factor;           /* device seconds in window factorizations (+larft)      */
    double t_other;            /* device seconds in copies / fills / small kernels      */
    double panel_bytes;        /* algorithmic HBM bytes of the panel phase  */
    int64_t launches;          /* kernels launched by the library                       */
    double t_chain;            /* device seconds in chained window applies (sum over    */
                               /* launches; launches on concurrent streams overlap)     */
    double flops_chain;        /* FP64 flops executed by the chained window applies     */
    int64_t chain_launches;    /* chained window-apply launches                         */
    /* critical-stream phase times (device seconds, CUDA events on the library's high-
       priority stream): absorb-right = R1..R3 (sec. 3.3.1), absorb-left = L1..L3 (sec.
       3.3.2); factor_exposed = factorization launches on that stream (the staircase chains
       the critical path waits for)                                                      */
    double t_absorb_right;
    double t_absorb_left;
    double t_factor_exposed;
    /* exact power-of-two scalings applied at entry (and undone on H, T at exit) so that
       squared norms cannot overflow or underflow: A <- scale_a A, B <- scale_b B (1 = none;
       Q and Z are invariant under such scalings)                                       */
    double scale_a;
    double scale_b;
    int64_t deflated_columns;  /* l of HT_FLAG_DEFLATE_ZERO_COLUMNS (sec. 3.5.1)             */
    double t_front;            /* device seconds of the front end (GENERAL_B / DEFLATE)      */
    double t_chain_busy;       /* device seconds during which at least one chained window     */
                               /* apply was running (union of the launch intervals that       */
                               /* t_chain sums; the launches overlap on concurrent streams)   */
} ht_report;

/*
 * North-star entry point (host memory).  A, B, Q, Z are n x n, column-major
 * with leading dimension n.  Synchronous: copies to the device, reduces,
 * copies back.  Returns HT_OK or an error code above.  Same as
 * ht_reduce_host(n, A, B, A, B, Q, Z, wantq, wantz, nb).
 */
HT_API int ht_reduce(int64_t n, double *A, double *B, double *Q, double *Z, int wantq, int wantz, int64_t nb);

/*
 * Out-of-place host entry point (H = Q^T A Z, T = Q^T B Z).
 *   A, B   (in)  n x n column-major pencil, ld n; read only (not modified unless aliased).
 *   H, T   (out) n x n, ld n: the Hessenberg and triangular results; H may alias A and
 *                T may alias B (that is ht_reduce).
 *   Q, Z   (out) n x n, ld n, if wantq / wantz (else ignored, may be NULL).
 * Device staging buffers are kept per device between calls (freed by
 * ht_release_workspace).  Host buffers allocated as pinned memory (cudaHostAlloc /
 * cudaHostRegister) are copied by DMA on the library's stream at full link rate; pageable
 * buffers work too, at the driver's staged-copy rate.  Synchronous.  Errors as ht_reduce
 * (HT_EARG_* for NULL pointers or n < 0; on error H, T, Q, Z are unspecified).
 */
HT_API int ht_reduce_host(int64_t n, const double *A, const double *B, double *H, double *T, double *Q, double *Z,
                          int wantq, int wantz, int64_t nb);

/*
 * Device-memory entry point.  dA, dB, dQ, dZ are device pointers with leading
 * dimensions ldda.. >= n.  Runs on opt->stream (or the library stream) and
 * returns after the reduction completed on the device.  opt and rep may be
 * NULL.  rep (if given) is filled on return.
 */
HT_API int ht_reduce_ex(int64_t n, double *dA, int64_t ldda, double *dB, int64_t lddb, double *dQ, int64_t lddq,
                 double *dZ, int64_t lddz, int wantq, int wantz, const ht_options *opt, ht_report *rep);

/*
 * Multi-GPU entry point: one process per GPU of one node,
 * called collectively by every rank with its own device buffers.
 *   Layout: A, B are n x n on every rank with identical contents (replicated); on return
 *   every rank holds H and T.  The work is sharded: A's right-hand applies (R2, R3, the
 *   Remark-2 rows; sec. 3.3.1) run on row slabs, its left-hand applies (L2, L3;
 *   sec. 3.3.2) on column slabs, with one packed ncclAllGather after each phase (the
 *   layout switch); Q and Z only receive right multiplications (P:886, P:945, P:1157,
 *   P:1198), so each rank computes the row slab ht_mg_slab(0, n, nranks, rank) of them,
 *   all-gathered at the end when gather_qz != 0 (else the other rows are unspecified).
 *   The panel, B and the staircase factorizations are computed redundantly on every rank
 *   (bitwise identical: deterministic kernels, fixed-order reductions).
 *   nccl_comm: an ncclComm_t of nranks ranks whose rank `rank` is this process (see
 *   ht_nccl_comm_init), ordered on opt->stream.  nccl_comm == NULL is the LOOPBACK mode: the
 *   call plays all nranks ranks on the current device (slab launches + the pack/unpack of
 *   every all-gather without the network) -- a single-GPU test of the sharded path.
 *   opt->row_begin/row_end must be 0 (HT_EARG_OPT).  Errors as ht_reduce_ex, plus
 *   HT_ENCCL for NCCL failures and HT_EARG_OPT for a communicator that does not match
 *   (rank, nranks).
 */
typedef struct {
    double *A; int64_t lda;
    double *B; int64_t ldb;
    double *Q; int64_t ldq;
    double *Z; int64_t ldz;
    int gather_qz;
} ht_mg_layout;
HT_API int ht_reduce_mg(int64_t n, const ht_mg_layout *layout, void *nccl_comm, int rank, int nranks, int wantq,
                        int wantz, const ht_options *opt, ht_report *rep);

/* NCCL bootstrap for ht_reduce_mg (NCCL is loaded at run time from the process's
 * libnccl.so.2): rank 0 calls ht_nccl_unique_id (128 opaque bytes), sends them to every
 * rank (e.g. torch.distributed), and every rank calls ht_nccl_comm_init.  HT_ENCCL if
 * NCCL is unavailable or fails. */
HT_API int ht_nccl_unique_id(void *id128);
HT_API int ht_nccl_comm_init(void **comm, int nranks, const void *id128, int rank);
HT_API int ht_nccl_comm_destroy(void *comm);

/* The contiguous balanced partition used by ht_reduce_mg: part `part` of [begin, end) over
 * `parts` parts is [*lo, *hi) (sizes differ by at most 1, lower parts larger).  Host-only. */
HT_API int ht_mg_slab(int64_t begin, int64_t end, int parts, int part, int64_t *lo, int64_t *hi);

/* Human-readable text for a return code (static storage). */
HT_API const char *ht_strerror(int code);

/* Library version: major*10000 + minor*100 + patch. */
HT_API int ht_version(void);

/* Release the cached device workspace of the current device. Returns HT_OK.
 * Process-level state that persists (created once per device by the first call): the
 * library's streams (the A and Q/Z side streams live in two green-context SM partitions of
 * 100 and 120 SMs when the driver supports them).  The device's persisting-L2 limit
 * (cudaLimitPersistingL2CacheSize) is left alone unless the development switch HT_L2PERSIST=1
 * is set (then raised to at most 3/8 of L2 for the panel workspace). */
HT_API int ht_release_workspace(void);

/*
 * Measurement hook (bench.py's standalone roofline of the WY-apply kernel): times the
 * chained staircase-window apply alone on the current device -- one matrix of `rows`
 * slabs (rows for left = 0, columns for left = 1), a chain of `nwin` windows of width p
 * overlapping by p/2 (the shape of a first-absorption R2 update at n = rows, nb = p/2),
 * full grid, no concurrent work.  Device memory is allocated and freed inside; the data
 * are synthetic (values do not matter for timing).  On HT_OK, *seconds is the best of
 * `reps` launches (CUDA events) and *flops the algorithmic flops of one launch
 * (2 * rows * p^2 * nwin).  Errors: HT_EARG_N for rows < 1, p < 2, p > 512 or nwin < 1,
 * HT_ENOMEM, HT_ECUDA.
 */
HT_API int ht_bench_chain_apply(int64_t rows, int p, int nwin, int left, int reps, double *seconds, double *flops);

#ifdef __cplusplus
}
#endif

#endif /* HT_B200_H */
