// ht_internal.h -- internal (non-ABI) declarations of the B200 HouseHT library.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// One window of a staircase factorization: Householder QR of the strided view
// W(i,j) = W[i*rs + j*cs], i < p, j < q (p >= q).  R (upper trapezoid, exact
// zeros below) is written back through the view; the reflectors go to
// V(:, j) in natural row order (row rev ? p-1-i : i), tau to tau[j].
struct FactorDesc {
    double *W;
    int64_t rs, cs;
    int p, q;
    int rev;
    double *V;
    int64_t ldv;
    double *tau;
    double *T;     // q x q upper-triangular compact-WY factor of Q = H_0 H_1 ... H_{q-1}
    int64_t ldt;
    int dense;     // > 0: view rows >= dense + c + 1 of column c are exactly zero (staircase
                   // windows [k new rows; R of the previous window]); 0: no structure
};

// chained window applies (ht_chain.cu): per matrix, slab dimension s in [s_begin, s_end)
// (rows if !left, columns if left), window dimension c; element (s, c) is X[s + c*ld]
// (right apply, X <- X Qhat) or X[c + s*ld] (left apply, X <- Qhat^T X).
struct ChainMat {
    double *X;
    int64_t ld;
    int left;
    int64_t s_begin, s_end;
};
// one window: columns (rows) [o, o+p) <- . * Qw (p x p, stored ROW-major: Qw(k, c) at Qw[k p + c]);
// applied to slabs s in [lo[m], hi[m])
struct ChainWin {
    const double *Qw;
    int64_t o;
    int p;
    int64_t lo[3], hi[3];
};
// maxgrid > 0: at most that many CTAs (they loop over the slabs).  h_wins (optional): the same
// windows in host memory; with nw <= 4 they travel in the launch parameters (d_wins unread).
int ht_chain_apply(cudaStream_t st, const ChainMat *mats, int nm, const ChainWin *d_wins, int nw, int pmax,
                   int maxgrid = 0, const ChainWin *h_wins = nullptr);
// One window transform applied to a narrow band of slabs straight from its factors (no
// explicit Qhat): on the slab view S(s, c) (element X[s + c*ld] for a right apply,
// X[c + s*ld] for a left apply; s in [s0, s0+cnt), c in [0, p) offset by o)
//   S <- S Q_0 Q_1 ...,  Q_b = I - V_b T_b V_b^T  (32-column panel blocks of V, p x q,
// ld ldv, and the diagonal 32x32 blocks T_b of T, ld ldt), i.e. X <- X Qhat (right) or
// X <- Qhat^T X (left).  8 slabs per CTA.
int ht_band_wy(cudaStream_t st, double *X, int64_t ld, int left, int64_t s0, int64_t cnt, int64_t o, int p, int q,
               const double *V, int64_t ldv, const double *T, int64_t ldt);
// Explicit Qhat = Q_0 Q_1 ... (p x p, row-major) for nw windows (the same kernel on identity rows).
int ht_form_qhat(cudaStream_t st, int nw, double *const *Qw, const int *p, const int *q, const double *const *V,
                 const double *const *T, void *d_descs, void *h_descs);
size_t ht_band_desc_size();

// Window factorizations of `nd` descriptors.  wave_flags == null: one CTA, windows in order.
// Otherwise the descriptors form a staircase chain ([new rows; R of the previous window]) and
// are factored as a wavefront by HT_WAVE_CTAS persistent CTAs (ht_factor.cu): wave_flags holds
// nd x 8 ints (epoch-valued, never reset), wave_ticket one int (zeroed on `st` here).
constexpr int HT_WAVE_CTAS = 6;
// h_descs (optional): the same descriptors in host memory; with nd <= 4 they are passed in the
// launch parameters and d_descs is not read (no copy needed).
int ht_factor_run(cudaStream_t st, const FactorDesc *d_descs, int nd, double *gscratch, int maxp,
                  int *wave_flags = nullptr, int *wave_ticket = nullptr, int wave_epoch = 0,
                  const FactorDesc *h_descs = nullptr);
int ht_factor_set_prof(unsigned long long *dev);

// panel kernel (ht_panel.cu)
struct PanelArgs {
    int64_t n, lda, ldb;
    double *A;
    double *B;
    int64_t s0;    // first unreduced column (0-based)
    int kmax;      // max reflector pairs in this panel
    int nb;        // ld of S, T
    double *U, *V, *Y;  // n x nb, ld = n, absolute row index
    double *S, *T;      // nb x nb
    double *vsave, *vrhs, *vy, *vx, *vw, *vw2, *vr;  // n-vectors, absolute row index
    double *part;       // gridDim x PW partial sums
    int pw;
    unsigned long long *yll;     // trsv solution in flag-in-data words: 2 per double (epoch << 32 | half)
    unsigned long long *yll_exp; // per 128-row block: epoch << 32 | exponent
    double *Dinv;       // inverted 128x128 diagonal blocks of B(s+1:n, s+1:n)
    double *Bt;         // Dinv_b * B(block b, blocks > b): pre-scaled block rows
    int64_t ldbt;
    int *dsafe;         // per block: 1 = use Dinv, 0 = sequential scaled substitution
    // 256-row solve on 4-CTA clusters (ht_panel.cu trsv4), used for a panel when every 256-row
    // diagonal block is safe: Dinv4 = inverses of the 256 x 256 diagonal blocks (ld 256),
    // Bt = Dinv4_b B(block b, blocks > b) packed with ld 256; dsafe4 per 256-row block
    double *Dinv4;
    int *dsafe4, *h_dsafe4;  // device / pinned host
    int solve4;
    int sweep_res;      // fused sweep: items kept L2-resident (the rest is read evict-first); < 0: no hints
    int *bexp;          // trsv block exponents
    unsigned epoch;     // trsv flag epoch base
    double tol;         // 2 u ||B||_F
    int max_ir;         // 10
    const int64_t *force_fail;  // sorted list of columns whose IR is forced to fail (test hook)
    int n_force_fail;
    double *ptime;      // optional (HT_PROFILE): per-phase seconds, CTA 0 (globaltimer)
    double *dbg;        // optional (HT_DEBUG_IR): dbg[j*12 + it] = ||r||/(tol ||x||) per IR iteration
    int *irtrace;       // per-column IR count (+1000 after a failed attempt)
    unsigned long long *ttrace;  // optional (HT_TRACE_COL): per-block trsv timestamps of one column
    int64_t tcol;
    double *ypart;      // tiled mat-vec partial sums: [column chunk][row], ld = n (A x)
    double *ypartB;     // the same for B x
    double *BV;         // n x nb: B v_i of the panel's right reflectors (absolute row index)
    double *vbx;        // n-vector: B x of the current solve
    unsigned *sweep_ctr;  // [2] fused-sweep item counters (alternating sweeps)
    void *hot;          // U, V, Y, BV, S, T, n-vectors: one allocation, L2-persisting for the panel
    size_t hot_bytes;
    int64_t *out;       // [0]=k done, [1]=failed, [2]=ir steps, [3]=ir extra columns, [4]=rescales, [5]=epoch used
};
int ht_panel_run(cudaStream_t st, PanelArgs *a, int nblocks);
int ht_panel_max_blocks(int *nblocks_out);

// multi-GPU plumbing (ht_mg.cu)
#define TRY_HT(x)                  \
    do {                           \
        int _rc = (x);             \
        if (_rc) return _rc;       \
    } while (0)
void ht_slab(int64_t begin, int64_t end, int parts, int r, int64_t *lo, int64_t *hi);
int ht_mg_allgather(cudaStream_t st, void *comm, int P, int me, double *X, int64_t ldx, int64_t r_beg, int64_t r_end,
                    int64_t c_beg, int64_t c_end, int by_cols, double *buf, size_t buf_doubles);
int ht_mg_check_comm(void *comm, int rank, int nranks);

// misc kernels (ht_util.cu)
int ht_fro_norm_sq(cudaStream_t st, int64_t rows, int64_t cols, const double *M, int64_t ld, double *d_out,
                   double *d_part);  // d_part: ht_fro_scratch_size() doubles
int ht_fro_scratch_size();
int ht_check_input(cudaStream_t st, int64_t n, const double *A, int64_t lda, const double *B, int64_t ldb,
                   int *d_flags, unsigned long long *d_maxbits);
int ht_zero_columns(cudaStream_t st, int64_t n, const double *B, int64_t ldb, int *d_zc, int *d_flags);
int ht_permute(cudaStream_t st, int64_t rows, int64_t cols, const double *src, int64_t lds, double *dst, int64_t ldd,
               const int64_t *d_perm_r, const int64_t *d_perm_c);
int ht_perm_matrix(cudaStream_t st, int64_t n, double *M, int64_t ld, const int64_t *d_perm);
int ht_scale(cudaStream_t st, int64_t rows, int64_t cols, double *M, int64_t ld, double s);
int ht_finish(cudaStream_t st, int64_t n, double *A, int64_t lda, double *B, int64_t ldb, const double *Q, int64_t ldq,
              const double *Z, int64_t ldz, double sa, double sb, int partial, int *d_flag);
int ht_desingularize(cudaStream_t st, int64_t n, double *B, int64_t ldb, int64_t r0, double thresh, double repl,
                     uint64_t seed, int64_t key, int *d_count);
int ht_zero_lower(cudaStream_t st, int64_t rows, int64_t cols, double *M, int64_t ld, int64_t diag_offset);
