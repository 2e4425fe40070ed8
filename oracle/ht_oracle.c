/*
 * oracle/ht_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU implementations of the Hessenberg-
 * triangular (HT) reduction of a real pencil A - lambda*B with B upper
 * triangular (section 1).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_1710_08538_b200/csrc), and the CUDA path never calls it.
 *
 * All arithmetic is IEEE binary64.  Matrices are column-major, ld = n.
 * Indices below are 0-based; the paper is 1-based (paper j = our j + 1).
 *
 * Functions and the passages they follow:
 *   orc_house    Householder reflector, PAPER.md P:80-85 (sec. 2.1) with the
 *                GvL Alg. 5.1.1 construction named in Lemma 1; LAPACK
 *                dlarfg sign convention (reading R1).
 *   orc_givens   plane rotation [c s; -s c][f; g] = [r; 0] (GvL sec. 5.1.8).
 *   orc_ht_0     "Oracle-0": Algorithm 2 BasicHouseHT (App. A)
 *                verbatim: dense trailing B, solve B_{j+1:n,j+1:n} x = e1 by
 *                LU with partial pivoting (backward stable, eq. computedx
 *                P:2392-2395).  Theta(n^4): small n only.
 *   orc_ht_T     "Oracle-T": Algorithm 2 with the trailing B kept upper
 *                triangular.  Step "Solve" uses the sec. 3.2.1 formula
 *                x = B22^{-1}(e1 - beta*u*u1) with B22 the
 *                *triangular* trailing block (the left reflector is kept in
 *                factored form, exactly as the paper's k = 0 case), with
 *                desingularisation of zero pivots (Remark 1 P:135-139)
 *                and overflow-safe scaling (reading R-Z8).  After G_j, the
 *                trailing block equals R + a1 b1^T + a2 b2^T and is returned to
 *                triangular form by two Givens rank-1 QR updates (GvL 12.5.1),
 *                applied also to A and Q.  O(n^3).
 *   orc_ht_G     "Oracle-G": Moler-Stewart Givens HT reduction (the method the
 *                paper compares with, LAPACK DGGHRD; Moler & Stewart 1973).
 *                Brute-force reference for tiny n and the cfg-4 parity
 *                reference.
 *
 * Parity status of every function is recorded in DESIGN.md section "Oracle".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define IX(i, j, ld) ((size_t)(j) * (size_t)(ld) + (size_t)(i))

static const double ORC_U = 1.1102230246251565404e-16; /* unit roundoff 2^-53 */

/* ------------------------------------------------------------------------- */
/* Scaled 2-norm (no overflow for entries up to ~1e300).                      */
static double orc_nrm2(int64_t m, const double *x)
{
    double scale = 0.0, ssq = 1.0;
    for (int64_t i = 0; i < m; ++i) {
        double a = fabs(x[i]);
        if (a == 0.0) continue;
        if (scale < a) {
            ssq = 1.0 + ssq * (scale / a) * (scale / a);
            scale = a;
        } else {
            ssq += (a / scale) * (a / scale);
        }
    }
    return scale * sqrt(ssq);
}

/*
 * Householder reflector H = I - beta v v^T with H x = alpha e1.
 * On entry x[0..m-1]; on return x[0] = alpha, x[1..m-1] = v(1..m-1), v(0) = 1.
 * Returns beta.  beta = 0 (H = I) when the tail x[1..] is exactly zero
 * (dlarfg convention, reading R1).  alpha = -sign(x0)*||x||, sign(0) = +1.
 */
double orc_house(int64_t m, double *x)
{
    if (m <= 1) return 0.0;
    double xnorm = orc_nrm2(m - 1, x + 1);
    if (xnorm == 0.0) return 0.0;
    double a0 = x[0];
    double nrm = hypot(a0, xnorm);
    double alpha = (a0 >= 0.0) ? -nrm : nrm;
    double beta = (alpha - a0) / alpha;
    double scal = 1.0 / (a0 - alpha);
    for (int64_t i = 1; i < m; ++i) x[i] *= scal;
    x[0] = alpha;
    return beta;
}

/* Plane rotation: [c s; -s c] [f; g] = [r; 0]. */
void orc_givens(double f, double g, double *c, double *s, double *r)
{
    if (g == 0.0) { *c = 1.0; *s = 0.0; *r = f; return; }
    if (f == 0.0) { *c = 0.0; *s = 1.0; *r = g; return; }
    double rr = hypot(f, g);
    *c = f / rr;
    *s = g / rr;
    *r = rr;
}

/* Counter-based normal draw for the desingularisation rho (reading R-Z7):
 * splitmix64 of (seed, column, row, counter) -> two uniforms -> Box-Muller. */
static uint64_t orc_mix(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
double orc_rho(uint64_t seed, int64_t col, int64_t row, uint32_t ctr)
{
    uint64_t h = orc_mix(seed ^ orc_mix((uint64_t)col * 0x100000001B3ULL ^ orc_mix((uint64_t)row + ((uint64_t)ctr << 40))));
    uint64_t h2 = orc_mix(h);
    double u1 = ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    double u2 = ((double)(h2 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925 * u2);
}

static double orc_fro(int64_t n, const double *M)
{
    return orc_nrm2(n * n, M);
}

static void orc_eye(int64_t n, double *M)
{
    memset(M, 0, sizeof(double) * (size_t)n * (size_t)n);
    for (int64_t i = 0; i < n; ++i) M[IX(i, i, n)] = 1.0;
}

/* C(r0:r0+m, c0:c1) <- (I - beta v v^T) C(...), v length m (v[0] = 1). */
static void orc_refl_left(int64_t n, double *C, int64_t r0, int64_t m, int64_t c0, int64_t c1,
                          const double *v, double beta)
{
    if (beta == 0.0) return;
#pragma omp parallel for schedule(static) if ((c1 - c0) * m > 65536)
    for (int64_t c = c0; c < c1; ++c) {
        double *col = C + IX(r0, c, n);
        double w = 0.0;
        for (int64_t i = 0; i < m; ++i) w += v[i] * col[i];
        w *= beta;
        for (int64_t i = 0; i < m; ++i) col[i] -= w * v[i];
    }
}

/* C(r0:r1, c0:c0+m) <- C(...) (I - beta v v^T). */
static void orc_refl_right(int64_t n, double *C, int64_t r0, int64_t r1, int64_t c0, int64_t m,
                           const double *v, double beta)
{
    if (beta == 0.0 || r1 <= r0) return;
    int64_t rows = r1 - r0;
    double *w = (double *)calloc((size_t)rows, sizeof(double));
    /* w = C v */
    for (int64_t i = 0; i < m; ++i) {
        const double *col = C + IX(r0, c0 + i, n);
        double vi = v[i];
        for (int64_t r = 0; r < rows; ++r) w[r] += col[r] * vi;
    }
#pragma omp parallel for schedule(static) if (rows * m > 65536)
    for (int64_t i = 0; i < m; ++i) {
        double *col = C + IX(r0, c0 + i, n);
        double f = beta * v[i];
        for (int64_t r = 0; r < rows; ++r) col[r] -= f * w[r];
    }
    free(w);
}

/* ------------------------------------------------------------------------- */
/* Oracle-G: Moler-Stewart Givens HT reduction (LAPACK DGGHRD).        */
int orc_ht_G(int64_t n, double *A, double *B, double *Q, double *Z)
{
    if (n < 0) return -1;
    orc_eye(n, Q);
    orc_eye(n, Z);
    for (int64_t j = 0; j + 2 < n; ++j) {
        for (int64_t i = n - 1; i >= j + 2; --i) {
            double c, s, r;
            /* row rotation (i-1, i) zeroes A(i, j) */
            orc_givens(A[IX(i - 1, j, n)], A[IX(i, j, n)], &c, &s, &r);
            A[IX(i - 1, j, n)] = r;
            A[IX(i, j, n)] = 0.0;
            for (int64_t col = j + 1; col < n; ++col) {
                double x = A[IX(i - 1, col, n)], y = A[IX(i, col, n)];
                A[IX(i - 1, col, n)] = c * x + s * y;
                A[IX(i, col, n)] = -s * x + c * y;
            }
            for (int64_t col = i - 1; col < n; ++col) {
                double x = B[IX(i - 1, col, n)], y = B[IX(i, col, n)];
                B[IX(i - 1, col, n)] = c * x + s * y;
                B[IX(i, col, n)] = -s * x + c * y;
            }
            for (int64_t row = 0; row < n; ++row) {
                double x = Q[IX(row, i - 1, n)], y = Q[IX(row, i, n)];
                Q[IX(row, i - 1, n)] = c * x + s * y;
                Q[IX(row, i, n)] = -s * x + c * y;
            }
            /* column rotation (i-1, i) zeroes the fill B(i, i-1) */
            orc_givens(B[IX(i, i, n)], B[IX(i, i - 1, n)], &c, &s, &r);
            for (int64_t row = 0; row <= i; ++row) {
                double x = B[IX(row, i - 1, n)], y = B[IX(row, i, n)];
                B[IX(row, i, n)] = c * y + s * x;
                B[IX(row, i - 1, n)] = -s * y + c * x;
            }
            B[IX(i, i - 1, n)] = 0.0;
            for (int64_t row = 0; row < n; ++row) {
                double x = A[IX(row, i - 1, n)], y = A[IX(row, i, n)];
                A[IX(row, i, n)] = c * y + s * x;
                A[IX(row, i - 1, n)] = -s * y + c * x;
                x = Z[IX(row, i - 1, n)];
                y = Z[IX(row, i, n)];
                Z[IX(row, i, n)] = c * y + s * x;
                Z[IX(row, i - 1, n)] = -s * y + c * x;
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Oracle-0: Algorithm 2 (App. A) verbatim, dense LU solve.     */

/* Solve M x = e1 (M dense m x m, column-major, overwritten) by LU with partial
 * pivoting.  Returns 0, or 1 if an exact zero pivot is met. */
static int orc_lu_solve_e1(int64_t m, double *M, double *x)
{
    int64_t *piv = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    for (int64_t c = 0; c < m; ++c) {
        int64_t p = c;
        double best = fabs(M[IX(c, c, m)]);
        for (int64_t r = c + 1; r < m; ++r)
            if (fabs(M[IX(r, c, m)]) > best) { best = fabs(M[IX(r, c, m)]); p = r; }
        piv[c] = p;
        if (best == 0.0) { free(piv); return 1; }
        if (p != c)
            for (int64_t k = 0; k < m; ++k) {
                double t = M[IX(c, k, m)];
                M[IX(c, k, m)] = M[IX(p, k, m)];
                M[IX(p, k, m)] = t;
            }
        double d = M[IX(c, c, m)];
        for (int64_t r = c + 1; r < m; ++r) M[IX(r, c, m)] /= d;
        for (int64_t k = c + 1; k < m; ++k) {
            double f = M[IX(c, k, m)];
            if (f == 0.0) continue;
            for (int64_t r = c + 1; r < m; ++r) M[IX(r, k, m)] -= M[IX(r, c, m)] * f;
        }
    }
    for (int64_t i = 0; i < m; ++i) x[i] = (i == 0) ? 1.0 : 0.0;
    for (int64_t c = 0; c < m; ++c) { /* P (all interchanges, dgetrs order) */
        int64_t p = piv[c];
        if (p != c) { double t = x[c]; x[c] = x[p]; x[p] = t; }
    }
    for (int64_t c = 0; c < m; ++c) /* L^{-1} (unit lower) */
        for (int64_t r = c + 1; r < m; ++r) x[r] -= M[IX(r, c, m)] * x[c];
    for (int64_t c = m - 1; c >= 0; --c) { /* U^{-1} */
        x[c] /= M[IX(c, c, m)];
        for (int64_t r = 0; r < c; ++r) x[r] -= M[IX(r, c, m)] * x[c];
    }
    free(piv);
    return 0;
}

int orc_ht_0(int64_t n, double *A, double *B, double *Q, double *Z)
{
    if (n < 0) return -1;
    orc_eye(n, Q);
    orc_eye(n, Z);
    double *v = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *M = (double *)malloc(sizeof(double) * (size_t)(n * n + 1));
    int rc = 0;
    for (int64_t j = 0; j + 2 < n; ++j) {
        int64_t m = n - j - 1;
        /* F_j = I_j (+) House(A_{j+1:n, j});  A <- F A, B <- F B, Q <- Q F */
        for (int64_t i = 0; i < m; ++i) v[i] = A[IX(j + 1 + i, j, n)];
        double beta = orc_house(m, v);
        v[0] = 1.0;
        orc_refl_left(n, A, j + 1, m, 0, n, v, beta);
        orc_refl_left(n, B, j + 1, m, 0, n, v, beta);
        orc_refl_right(n, Q, 0, n, j + 1, m, v, beta);
        for (int64_t i = j + 2; i < n; ++i) A[IX(i, j, n)] = 0.0; /* Set A_{j+2:n,j} <- 0 */
        /* Solve B_{j+1:n,j+1:n} x = e1 */
        for (int64_t c = 0; c < m; ++c)
            for (int64_t r = 0; r < m; ++r) M[IX(r, c, m)] = B[IX(j + 1 + r, j + 1 + c, n)];
        if (orc_lu_solve_e1(m, M, v)) { rc = 1; break; }
        /* G_j = I_j (+) House(x);  A <- A G, B <- B G, Z <- Z G */
        double gamma = orc_house(m, v);
        v[0] = 1.0;
        orc_refl_right(n, A, 0, n, j + 1, m, v, gamma);
        orc_refl_right(n, B, 0, n, j + 1, m, v, gamma);
        orc_refl_right(n, Z, 0, n, j + 1, m, v, gamma);
        for (int64_t i = j + 2; i < n; ++i) B[IX(i, j + 1, n)] = 0.0; /* Set B_{j+2:n,j+1} <- 0 */
    }
    free(v);
    free(M);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* Oracle-T                                                                   */

/* Overflow-safe back substitution R x = 2^(-e) y for upper triangular R stored
 * at B(r0.., r0..) (reading R-Z8).  y is overwritten; x returned in x.  Scale
 * changes are exact powers of two; only the direction of x is used (Lemma 1). */
static void orc_trsv_scaled(int64_t n, const double *B, int64_t r0, int64_t m, double *y, double *x)
{
    const double BIG = 0x1p400;
    for (int64_t i = m - 1; i >= 0; --i) {
        const double *col = B + IX(r0, r0 + i, n);
        double xi = y[i] / col[i];
        if (!(fabs(xi) <= BIG)) {
            int e;
            frexp(xi, &e);
            double sc = ldexp(1.0, -e);
            for (int64_t l = 0; l <= i; ++l) y[l] *= sc;
            for (int64_t l = i + 1; l < m; ++l) x[l] *= sc;
            xi = y[i] / col[i];
        }
        x[i] = xi;
        if (xi != 0.0)
            for (int64_t l = 0; l < i; ++l) y[l] -= col[l] * xi;
    }
}

typedef struct { int64_t i; double c, s; } orc_rot; /* acts on local rows (i-1, i) */

/* Apply a list of row rotations (rows r0+i-1, r0+i) to C(., c0:c1), in order. */
static void orc_rows_rot(int64_t n, double *C, int64_t r0, int64_t c0, int64_t c1,
                         const orc_rot *rot, int64_t nr)
{
    if (nr == 0) return;
#pragma omp parallel for schedule(static) if ((c1 - c0) * nr > 32768)
    for (int64_t c = c0; c < c1; ++c) {
        double *col = C + IX(r0, c, n);
        for (int64_t t = 0; t < nr; ++t) {
            int64_t i = rot[t].i;
            double x = col[i - 1], y = col[i];
            col[i - 1] = rot[t].c * x + rot[t].s * y;
            col[i] = -rot[t].s * x + rot[t].c * y;
        }
    }
}

/* Apply the same rotations as column rotations (cols c0+i-1, c0+i) to Q(., .):
 * Q <- Q G^T, so the accumulated Q satisfies H = Q^T A Z. */
static void orc_cols_rot(int64_t n, double *Qm, int64_t c0, const orc_rot *rot, int64_t nr)
{
    if (nr == 0) return;
    const int64_t RB = 64;
#pragma omp parallel for schedule(static) if (n * nr > 32768)
    for (int64_t rb = 0; rb < n; rb += RB) {
        int64_t re = rb + RB < n ? rb + RB : n;
        for (int64_t t = 0; t < nr; ++t) {
            double *x = Qm + IX(0, c0 + rot[t].i - 1, n);
            double *y = Qm + IX(0, c0 + rot[t].i, n);
            double c = rot[t].c, s = rot[t].s;
            for (int64_t r = rb; r < re; ++r) {
                double xv = x[r], yv = y[r];
                x[r] = c * xv + s * yv;
                y[r] = -s * xv + c * yv;
            }
        }
    }
}

/* Rank-1 QR update (GvL 12.5.1): R + a b^T with R upper triangular (order mm,
 * stored at B(r0.., r0..)) is returned to triangular form by rotations
 * (phase 1: bottom-up on a; phase 2: top-down on the Hessenberg result).
 * Every rotation is also applied to the carried vector `carry` (if non-NULL),
 * to rows of A (cols ac0..n-1) and to columns of Q.  a is destroyed. */
static void orc_rank1_update(int64_t n, double *B, int64_t r0, int64_t mm, double *a, const double *b,
                             double *carry, double *A, int64_t ac0, double *Qm, orc_rot *rot)
{
    if (mm <= 0) return;
    int64_t nr = 0;
    /* phase 1: rotations (i-1, i), i = mm-1 .. 1, reduce a to a multiple of e1 */
    for (int64_t i = mm - 1; i >= 1; --i) {
        double c, s, r;
        orc_givens(a[i - 1], a[i], &c, &s, &r);
        a[i - 1] = r;
        a[i] = 0.0;
        rot[nr].i = i; rot[nr].c = c; rot[nr].s = s; ++nr;
    }
    /* apply to R column by column: column col has rows 0..col (+ fill row col+1) */
#pragma omp parallel for schedule(dynamic, 16) if (mm > 256)
    for (int64_t col = 0; col < mm; ++col) {
        double *cp = B + IX(r0, r0 + col, n);
        for (int64_t t = 0; t < nr; ++t) {
            int64_t i = rot[t].i;
            if (i - 1 > col) continue; /* both rows below the nonzero part */
            double x = cp[i - 1], y = (i <= col + 1) ? cp[i] : 0.0;
            cp[i - 1] = rot[t].c * x + rot[t].s * y;
            double yn = -rot[t].s * x + rot[t].c * y;
            if (i <= col + 1) cp[i] = yn;
        }
    }
    if (carry)
        for (int64_t t = 0; t < nr; ++t) {
            int64_t i = rot[t].i;
            double x = carry[i - 1], y = carry[i];
            carry[i - 1] = rot[t].c * x + rot[t].s * y;
            carry[i] = -rot[t].s * x + rot[t].c * y;
        }
    orc_rows_rot(n, A, r0, ac0, n, rot, nr);
    orc_cols_rot(n, Qm, r0, rot, nr);
    /* R <- R + a0 e1 b^T (upper Hessenberg stays upper Hessenberg) */
    for (int64_t col = 0; col < mm; ++col) B[IX(r0, r0 + col, n)] += a[0] * b[col];
    /* phase 2: rotations (i, i+1), i = 0 .. mm-2, zero the sub-diagonal */
    nr = 0;
    for (int64_t col = 0; col < mm; ++col) {
        double *cp = B + IX(r0, r0 + col, n);
        for (int64_t t = 0; t < nr; ++t) { /* rotations already found act on this column */
            int64_t i = rot[t].i; /* rows (i-1, i) */
            double x = cp[i - 1], y = cp[i];
            cp[i - 1] = rot[t].c * x + rot[t].s * y;
            cp[i] = -rot[t].s * x + rot[t].c * y;
        }
        if (col + 1 < mm) {
            double c, s, r;
            orc_givens(cp[col], cp[col + 1], &c, &s, &r);
            cp[col] = r;
            cp[col + 1] = 0.0;
            rot[nr].i = col + 1; rot[nr].c = c; rot[nr].s = s; ++nr;
        }
    }
    if (carry)
        for (int64_t t = 0; t < nr; ++t) {
            int64_t i = rot[t].i;
            double x = carry[i - 1], y = carry[i];
            carry[i - 1] = rot[t].c * x + rot[t].s * y;
            carry[i] = -rot[t].s * x + rot[t].c * y;
        }
    orc_rows_rot(n, A, r0, ac0, n, rot, nr);
    orc_cols_rot(n, Qm, r0, rot, nr);
}

/*
 * Oracle-T.  Processes columns j < jmax (jmax >= n-2 means the full
 * reduction; a smaller jmax is used only for the bounded cpu_baseline sample).
 * Returns 0.  *ndesing counts desingularised pivots.
 */
int orc_ht_T(int64_t n, double *A, double *B, double *Q, double *Z, uint64_t seed, int64_t jmax,
             int64_t *ndesing)
{
    if (n < 0) return -1;
    orc_eye(n, Q);
    orc_eye(n, Z);
    if (ndesing) *ndesing = 0;
    const double nB = orc_fro(n, B); /* ||B_0||_F, reading R-Z3 */
    double *u = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *x = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *y = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *Rtu = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *Rv = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *b1 = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *b2 = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *a2 = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    orc_rot *rot = (orc_rot *)malloc(sizeof(orc_rot) * (size_t)(n + 1));
    if (jmax > n - 2) jmax = n - 2;
    for (int64_t j = 0; j < jmax; ++j) {
        const int64_t m = n - j - 1, t0 = j + 1; /* trailing block rows/cols t0..n-1 */
        /* 1. left reflector F_j = House(A(j+1:n, j)) (Alg 2 step F_j) */
        for (int64_t i = 0; i < m; ++i) u[i] = A[IX(t0 + i, j, n)];
        const double beta = orc_house(m, u);
        A[IX(t0, j, n)] = u[0];
        for (int64_t i = 1; i < m; ++i) A[IX(t0 + i, j, n)] = 0.0; /* Set A_{j+2:n,j} <- 0 */
        u[0] = 1.0;
        orc_refl_left(n, A, t0, m, t0, n, u, beta);
        orc_refl_right(n, Q, 0, n, t0, m, u, beta);
        /* 2. desingularise zero pivots of R = B(t0:, t0:) (readings R-Z6/R-Z7) */
        for (int64_t i = 0; i < m; ++i) {
            double *d = B + IX(t0 + i, t0 + i, n);
            if (fabs(*d) < ORC_U * nB) {
                uint32_t ctr = 0;
                double rho;
                do { rho = orc_rho(seed, j, t0 + i, ctr++); } while (fabs(rho) < 0.5);
                *d = 2.0 * ORC_U * rho * nB;
                if (ndesing) ++*ndesing;
            }
        }
        /* 3. x = R^{-1} (e1 - beta u u_1)  (sec. 3.2.1) */
        for (int64_t i = 0; i < m; ++i) y[i] = -beta * u[i];
        y[0] += 1.0;
        orc_trsv_scaled(n, B, t0, m, y, x);
        /* 4. right reflector G_j = House(x) (Alg 2 step G_j) */
        const double gamma = orc_house(m, x);
        x[0] = 1.0; /* x now holds v */
        orc_refl_right(n, A, 0, n, t0, m, x, gamma);
        orc_refl_right(n, Z, 0, n, t0, m, x, gamma);
        orc_refl_right(n, B, 0, t0, t0, m, x, gamma); /* rows above the trailing block */
        /* trailing block: N = (I - beta u u^T) R (I - gamma v v^T) = R + u b1^T + z b2^T */
        for (int64_t c = 0; c < m; ++c) { /* Rtu = R^T u, column c: sum_{r<=c} R(r,c) u(r) */
            const double *col = B + IX(t0, t0 + c, n);
            double s = 0.0;
            for (int64_t r = 0; r <= c; ++r) s += col[r] * u[r];
            Rtu[c] = s;
        }
        for (int64_t r = 0; r < m; ++r) Rv[r] = 0.0; /* Rv = R v */
        for (int64_t c = 0; c < m; ++c) {
            const double *col = B + IX(t0, t0 + c, n);
            double vc = x[c];
            for (int64_t r = 0; r <= c; ++r) Rv[r] += col[r] * vc;
        }
        double utRv = 0.0;
        for (int64_t r = 0; r < m; ++r) utRv += u[r] * Rv[r];
        for (int64_t i = 0; i < m; ++i) {
            b1[i] = -beta * Rtu[i];
            a2[i] = Rv[i] - beta * u[i] * utRv; /* z */
            b2[i] = -gamma * x[i];
        }
        /* row 0 of N -> B(t0, t0:n); column 0 of N below the diagonal -> exact 0 */
        for (int64_t c = 0; c < m; ++c) B[IX(t0, t0 + c, n)] += u[0] * b1[c] + a2[0] * b2[c];
        for (int64_t r = 1; r < m; ++r) B[IX(t0 + r, t0, n)] = 0.0;
        /* 5. re-triangularise N(1:,1:) = R22 + u(1:) b1(1:)^T + z(1:) b2(1:)^T */
        if (m >= 2) {
            orc_rank1_update(n, B, t0 + 1, m - 1, u + 1, b1 + 1, a2 + 1, A, t0, Q, rot);
            orc_rank1_update(n, B, t0 + 1, m - 1, a2 + 1, b2 + 1, NULL, A, t0, Q, rot);
        }
        for (int64_t c = t0 + 1; c < n; ++c) /* structural zeros of the triangular result */
            for (int64_t r = c + 1; r < n; ++r) B[IX(r, c, n)] = 0.0;
    }
    free(u); free(x); free(y); free(Rtu); free(Rv); free(b1); free(b2); free(a2); free(rot);
    return 0;
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
