/*
 * phipm ORACLE — TEST INFRASTRUCTURE ONLY, NOT PRODUCT CODE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference)
 * may load this library.  It shares no code, header, table or helper with the CUDA product in
 * paper_0907_4631_b200/ and include/, and it never calls it.
 *
 * A plain, slow, single-threaded IEEE fp64 implementation of the phipm method of
 * J. Niesen and W. M. Wright, "Algorithm 919: A Krylov subspace algorithm for evaluating the
 * phi-functions appearing in exponential integrators" (arXiv:0907.4631), written from the paper.
 * "P:n" cites line n of PAPER.md, with the section/equation/algorithm it falls in; "Rn" names a
 * reading of an ambiguous passage, listed in DESIGN.md §3.
 *
 * Arithmetic conventions:
 *   - compiled with -O2 -ffp-contract=off (no fused multiply-add unless written as fma());
 *   - CSR rows are summed sequentially in ascending column order;
 *   - dot products / 2-norms over n use the compensated Dot2 algorithm (Ogita, Rump & Oishi
 *     2005: TwoProduct via fma + TwoSum), so the oracle's reductions are accurate to about
 *     eps*|result| + eps^2*sum|x_i y_i| independent of n;
 *   - the small dense exponential is the degree-13 Pade approximant with scaling and squaring
 *     (Sec. 3.1), evaluated with the odd/even split and an LU solve with partial
 *     pivoting, exactly as the algorithm states.
 *
 * Matrices are column-major.  Vectors of the Krylov basis are columns of V (leading dim n).
 *
 * Parity status of each function is stated in its comment: "pinned by ..." names the tests
 * that tie it to something other than itself.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENOMEM 2
#define ORC_ESTEP 4
#define ORC_ENONFINITE 5
#define ORC_ESINGULAR 6

static const double ORC_EPS = 2.220446049250313080847e-16; /* 2^-52 */

/* ------------------------------------------------------------------------------------------ */
/* Operators                                                                                   */
/* ------------------------------------------------------------------------------------------ */

/* Number of structural nonzeros of the 3/5/7-point stencil with zero Dirichlet boundary.
 * pinned by tests/test_oracle_operators.py (closed forms 3n-2, 5n-2(nx+ny), 7n-2(...)). */
int64_t orc_stencil_nnz(int dim, int nx, int ny, int nz)
{
    int64_t n = (int64_t)nx * ny * nz, nnz = 0;
    for (int64_t r = 0; r < n; r++) {
        int64_t i = r % nx, j = (r / nx) % ny, k = r / ((int64_t)nx * ny);
        nnz += 1;
        nnz += (i > 0) + (i < nx - 1);
        if (dim >= 2) nnz += (j > 0) + (j < ny - 1);
        if (dim >= 3) nnz += (k > 0) + (k < nz - 1);
    }
    return nnz;
}

/* CSR of the stencil operator: row r = i + nx*(j + ny*k); the entries of a row in ascending
 * column order are z-, y-, x-, centre, x+, y+, z+ (neighbours outside the grid are absent:
 * zero Dirichlet data).  c = {center, xm, xp, ym, yp, zm, zp}.
 * pinned by tests/test_oracle_operators.py (dense Kronecker-sum construction). */
void orc_csr_from_stencil(int dim, int nx, int ny, int nz, const double *c,
                          int32_t *row_ptr, int32_t *col, double *val)
{
    int64_t n = (int64_t)nx * ny * nz, e = 0, pl = (int64_t)nx * ny;
    for (int64_t r = 0; r < n; r++) {
        int64_t i = r % nx, j = (r / nx) % ny, k = r / pl;
        row_ptr[r] = (int32_t)e;
        if (dim >= 3 && k > 0)      { col[e] = (int32_t)(r - pl); val[e] = c[5]; e++; }
        if (dim >= 2 && j > 0)      { col[e] = (int32_t)(r - nx); val[e] = c[3]; e++; }
        if (i > 0)                  { col[e] = (int32_t)(r - 1);  val[e] = c[1]; e++; }
        col[e] = (int32_t)r; val[e] = c[0]; e++;
        if (i < nx - 1)             { col[e] = (int32_t)(r + 1);  val[e] = c[2]; e++; }
        if (dim >= 2 && j < ny - 1) { col[e] = (int32_t)(r + nx); val[e] = c[4]; e++; }
        if (dim >= 3 && k < nz - 1) { col[e] = (int32_t)(r + pl); val[e] = c[6]; e++; }
    }
    row_ptr[n] = (int32_t)e;
}

/* y = A x, each row summed sequentially in ascending column order (2 N_A flops).
 * pinned by tests/test_oracle_operators.py (scipy.sparse product). */
void orc_spmv(int64_t n, const int32_t *rp, const int32_t *col, const double *val,
              const double *x, double *y)
{
    for (int64_t i = 0; i < n; i++) {
        double s = 0.0;
        for (int32_t e = rp[i]; e < rp[i + 1]; e++) s = s + val[e] * x[col[e]];
        y[i] = s;
    }
}

/* ||A||_inf = max_i sum_j |a_ij|, rows summed in ascending column order (Eq. tau_0 input). */
double orc_inf_norm(int64_t n, const int32_t *rp, const double *val)
{
    double mx = 0.0;
    for (int64_t i = 0; i < n; i++) {
        double s = 0.0;
        for (int32_t e = rp[i]; e < rp[i + 1]; e++) s = s + fabs(val[e]);
        if (s > mx) mx = s;
    }
    return mx;
}

/* Compensated dot product Dot2 (TwoProduct with fma, TwoSum).  pinned by
 * tests/test_oracle_linalg.py (exact rational dot with fractions.Fraction). */
double orc_dot(int64_t n, const double *x, const double *y)
{
    double s = 0.0, c = 0.0;
    for (int64_t i = 0; i < n; i++) {
        double p = x[i] * y[i];
        double pe = fma(x[i], y[i], -p);          /* exact: x*y = p + pe */
        double t = s + p;
        double z = t - s;
        double se = (s - (t - z)) + (p - z);      /* exact: s + p = t + se */
        s = t;
        c = c + (pe + se);
    }
    return s + c;
}

double orc_norm2(int64_t n, const double *x) { return sqrt(orc_dot(n, x, x)); }

/* ------------------------------------------------------------------------------------------ */
/* Small dense linear algebra and the matrix exponential (Sec. 3.1, Eq. 8)          */
/* ------------------------------------------------------------------------------------------ */

/* C = A B, K x K column-major, plain triple loop. */
static void mm(int K, const double *A, const double *B, double *C)
{
    for (int j = 0; j < K; j++)
        for (int i = 0; i < K; i++) {
            double s = 0.0;
            for (int l = 0; l < K; l++) s = s + A[i + (size_t)l * K] * B[l + (size_t)j * K];
            C[i + (size_t)j * K] = s;
        }
}

/* Coefficients of the [13/13] diagonal Pade approximant to exp: p(z) = sum_j c_j z^j with
 * c_j = (26-j)! 13! / (26! j! (13-j)!)  (SPEC S:162 restating the standard formula; P:378
 * "degree-13 diagonal Pade approximant").  c_0 = 1; q(z) = p(-z).
 * Computed through the ratio c_{j+1}/c_j = (13-j)/((26-j)(j+1)).
 * pinned by tests/test_oracle_linalg.py (exact big-integer factorial formula). */
void orc_pade13_coeffs(double *c)
{
    c[0] = 1.0;
    for (int j = 0; j < 13; j++) c[j + 1] = c[j] * (double)(13 - j) / ((double)(26 - j) * (double)(j + 1));
}

/* ||A||_1 = max column abs sum. */
static double norm1(int K, const double *A)
{
    double mx = 0.0;
    for (int j = 0; j < K; j++) {
        double s = 0.0;
        for (int i = 0; i < K; i++) s = s + fabs(A[i + (size_t)j * K]);
        if (s > mx) mx = s;
    }
    return mx;
}

/* ceil_+(log2(x / 5.37)): the number of squarings (theta_13 = 5.37 as printed, R26;
 * ceil_+ = smallest nonnegative integer >= the argument, R37). */
int orc_expm_squarings(double norm)
{
    if (!(norm > 0.0)) return 0;
    double l = ceil(log2(norm / 5.37));
    return l > 0.0 ? (int)l : 0;
}

/* M(A) = 44/3 + 2 ceil_+(log2(||A||_1 / 5.37))  (Eq. 8). */
double orc_cost_M(double norm1_value) { return 44.0 / 3.0 + 2.0 * (double)orc_expm_squarings(norm1_value); }

/* E = exp(A), K x K, by Higham's degree-13 Pade scaling and squaring:
 *   s = ceil_+(log2(||A||_1/5.37)), A <- A/2^s,
 *   U = A [A6 (c13 A6 + c11 A4 + c9 A2) + c7 A6 + c5 A4 + c3 A2 + c1 I],
 *   V = A6 (c12 A6 + c10 A4 + c8 A2) + c6 A6 + c4 A4 + c2 A2 + c0 I,
 *   solve (V - U) X = (V + U)  (LU with partial pivoting), E = X^(2^s).
 * Returns ORC_ESINGULAR if a pivot is below 1e-300 in magnitude, ORC_ENONFINITE on NaN/Inf.
 * pinned by tests/test_oracle_linalg.py (identities, closed forms, scipy.linalg.expm). */
int orc_expm(int K, const double *Ain, double *E)
{
    if (K <= 0) return ORC_EINVAL;
    size_t KK = (size_t)K * K;
    double *A = malloc(KK * sizeof(double)), *A2 = malloc(KK * sizeof(double)),
           *A4 = malloc(KK * sizeof(double)), *A6 = malloc(KK * sizeof(double)),
           *T = malloc(KK * sizeof(double)), *U = malloc(KK * sizeof(double)),
           *V = malloc(KK * sizeof(double)), *P = malloc(KK * sizeof(double));
    int *piv = malloc((size_t)K * sizeof(int));
    int status = ORC_OK;
    if (!A || !A2 || !A4 || !A6 || !T || !U || !V || !P || !piv) { status = ORC_ENOMEM; goto out; }
    for (size_t e = 0; e < KK; e++) {
        if (!isfinite(Ain[e])) { status = ORC_ENONFINITE; goto out; }
    }
    double c[14];
    orc_pade13_coeffs(c);
    int s = orc_expm_squarings(norm1(K, Ain));
    double scale = ldexp(1.0, -s);
    for (size_t e = 0; e < KK; e++) A[e] = Ain[e] * scale;
    mm(K, A, A, A2);
    mm(K, A2, A2, A4);
    mm(K, A4, A2, A6);
    /* U */
    for (size_t e = 0; e < KK; e++) T[e] = c[13] * A6[e] + c[11] * A4[e] + c[9] * A2[e];
    mm(K, A6, T, P);
    for (size_t e = 0; e < KK; e++) P[e] = P[e] + c[7] * A6[e] + c[5] * A4[e] + c[3] * A2[e];
    for (int i = 0; i < K; i++) P[i + (size_t)i * K] += c[1];
    mm(K, A, P, U);
    /* V */
    for (size_t e = 0; e < KK; e++) T[e] = c[12] * A6[e] + c[10] * A4[e] + c[8] * A2[e];
    mm(K, A6, T, V);
    for (size_t e = 0; e < KK; e++) V[e] = V[e] + c[6] * A6[e] + c[4] * A4[e] + c[2] * A2[e];
    for (int i = 0; i < K; i++) V[i + (size_t)i * K] += c[0];
    /* (V - U) X = (V + U): Q in T, right-hand sides in P */
    for (size_t e = 0; e < KK; e++) { T[e] = V[e] - U[e]; P[e] = V[e] + U[e]; }
    /* LU with partial pivoting of T (Doolittle, in place) */
    for (int k = 0; k < K; k++) {
        int pr = k;
        double pm = fabs(T[k + (size_t)k * K]);
        for (int i = k + 1; i < K; i++)
            if (fabs(T[i + (size_t)k * K]) > pm) { pm = fabs(T[i + (size_t)k * K]); pr = i; }
        piv[k] = pr;
        if (!(pm >= 1e-300)) { status = ORC_ESINGULAR; goto out; }
        if (pr != k)
            for (int j = 0; j < K; j++) {
                double tmp = T[k + (size_t)j * K]; T[k + (size_t)j * K] = T[pr + (size_t)j * K]; T[pr + (size_t)j * K] = tmp;
            }
        for (int i = k + 1; i < K; i++) {
            double l = T[i + (size_t)k * K] / T[k + (size_t)k * K];
            T[i + (size_t)k * K] = l;
            for (int j = k + 1; j < K; j++) T[i + (size_t)j * K] = T[i + (size_t)j * K] - l * T[k + (size_t)j * K];
        }
    }
    /* apply the row interchanges to P, then forward (unit L) and back (U) substitution */
    for (int k = 0; k < K; k++)
        if (piv[k] != k)
            for (int j = 0; j < K; j++) {
                double tmp = P[k + (size_t)j * K]; P[k + (size_t)j * K] = P[piv[k] + (size_t)j * K]; P[piv[k] + (size_t)j * K] = tmp;
            }
    for (int j = 0; j < K; j++) {
        double *x = P + (size_t)j * K;
        for (int i = 0; i < K; i++) {
            double s2 = x[i];
            for (int l = 0; l < i; l++) s2 = s2 - T[i + (size_t)l * K] * x[l];
            x[i] = s2;
        }
        for (int i = K - 1; i >= 0; i--) {
            double s2 = x[i];
            for (int l = i + 1; l < K; l++) s2 = s2 - T[i + (size_t)l * K] * x[l];
            x[i] = s2 / T[i + (size_t)i * K];
        }
    }
    /* squaring */
    for (int q = 0; q < s; q++) {
        mm(K, P, P, T);
        memcpy(P, T, KK * sizeof(double));
    }
    for (size_t e = 0; e < KK; e++) {
        if (!isfinite(P[e])) { status = ORC_ENONFINITE; goto out; }
        E[e] = P[e];
    }
out:
    free(A); free(A2); free(A4); free(A6); free(T); free(U); free(V); free(P); free(piv);
    return status;
}

/* phi_p(tau H_mu) e1 and phi_{p+1}(tau H_mu) e1 from ONE exponential of the augmented matrix
 * (Eq. hathm P:368-377 with p+1 in place of p, as Sec. 3.2 P:451-453 says: "we only need to
 * exponentiate a matrix of size m+p+1"):
 *     Hhat = [[tau H, e1, 0], [0, 0, I_p], [0, 0, 0]],  K = mu + p + 1,
 * column mu+j (0-based) of exp(Hhat), top mu rows, is phi_{j+1}(tau H) e1 (R8: the Krylov
 * basis is that of A, tau enters only here).  p = 0: phi_0 is column 0 (R12).
 * H is mu x mu with leading dimension ldh.  Writes phip[0..mu-1], phip1[0..mu-1], and
 * *normH1 = ||H_mu||_1 (unscaled).
 * pinned by tests/test_oracle_phi.py (closed forms of Sec. 2, Taylor series). */
int orc_phi_pair(int mu, const double *H, int ldh, double tau, int p,
                 double *phip, double *phip1, double *normH1)
{
    if (mu < 1 || p < 0) return ORC_EINVAL;
    int K = mu + p + 1;
    double *Hh = calloc((size_t)K * K, sizeof(double)), *E = malloc((size_t)K * K * sizeof(double));
    if (!Hh || !E) { free(Hh); free(E); return ORC_ENOMEM; }
    double nh = 0.0;
    for (int j = 0; j < mu; j++) {
        double cs = 0.0;
        for (int i = 0; i < mu; i++) {
            Hh[i + (size_t)j * K] = tau * H[i + (size_t)j * ldh];
            cs = cs + fabs(H[i + (size_t)j * ldh]);
        }
        if (cs > nh) nh = cs;
    }
    Hh[0 + (size_t)mu * K] = 1.0;                            /* e1 in column mu */
    for (int i = 1; i <= p; i++) Hh[(mu + i - 1) + (size_t)(mu + i) * K] = 1.0;  /* I_p shifted */
    int st = orc_expm(K, Hh, E);
    if (st == ORC_OK) {
        int cp = (p == 0) ? 0 : mu + p - 1;
        int cp1 = mu + p;
        for (int i = 0; i < mu; i++) {
            phip[i] = E[i + (size_t)cp * K];
            phip1[i] = E[i + (size_t)cp1 * K];
        }
    }
    if (normH1) *normH1 = nh;
    free(Hh); free(E);
    return st;
}

/* ------------------------------------------------------------------------------------------ */
/* Krylov projection (Sec. 3.1, Algorithms 1 and 2)                                             */
/* ------------------------------------------------------------------------------------------ */

/* Breakdown threshold (R22): h_{j+1,j} <= n * eps * ||A||_inf. */
static int is_breakdown(int64_t n, double h, double normA) { return h <= (double)n * ORC_EPS * normA; }

/* Arnoldi iteration, Algorithm 1 verbatim: modified Gram-Schmidt.
 * Extends an existing basis v_0..v_k0 (columns of V, leading dim n; H (ldh >= m+1) column-major,
 * 0-based: h_{i,j} at H[i + j*ldh]) to m columns of H.  The caller sets v_0 = v/||v|| (line 1).
 * Returns the number k of valid columns of H (m, or the j+1 at which breakdown occurred);
 * *brk = 1 on breakdown (then v_k is not formed).
 * pinned by tests/test_oracle_krylov.py (Arnoldi relation, orthonormality, exactness at m=n). */
int orc_arnoldi(int64_t n, const int32_t *rp, const int32_t *col, const double *val, double normA,
                int k0, int m, double *V, double *H, int ldh, int *brk)
{
    double *w = malloc((size_t)n * sizeof(double));
    if (!w) return -ORC_ENOMEM;
    *brk = 0;
    for (int j = k0; j < m; j++) {
        orc_spmv(n, rp, col, val, V + (size_t)j * n, w);                       /* w = A v_j */
        for (int i = 0; i <= j; i++) {
            const double *vi = V + (size_t)i * n;
            double h = orc_dot(n, vi, w);                                      /* h_ij = v_i^T w */
            H[i + (size_t)j * ldh] = h;
            for (int64_t r = 0; r < n; r++) w[r] = w[r] - h * vi[r];           /* w = w - h_ij v_i */
        }
        double hn = orc_norm2(n, w);                                           /* h_{j+1,j} = ||w|| */
        H[(j + 1) + (size_t)j * ldh] = hn;
        if (is_breakdown(n, hn, normA)) { *brk = 1; free(w); return j + 1; }
        double *vn = V + (size_t)(j + 1) * n;
        for (int64_t r = 0; r < n; r++) vn[r] = w[r] / hn;                     /* v_{j+1} = w/h */
    }
    free(w);
    return m;
}

/* Lanczos iteration, Algorithm 2, 0-based.  Line 4's "t_{j,j-1} = ||w||;
 * t_{j-1,j} = ||w||" is read as t_{j+1,j} = t_{j,j+1} = ||w|| (R36: line 3 must use the
 * previous iteration's norm and line 5 divides by the current one; Trefethen & Bau Alg. 36.1).
 *   w = A v_j;  t_jj = v_j^T w;  w = w - t_{j,j-1} v_{j-1} - t_jj v_j;
 *   t_{j+1,j} = t_{j,j+1} = ||w||;  v_{j+1} = w / t_{j+1,j}.
 * T is stored in the Hessenberg array H.  Same extension/breakdown contract as orc_arnoldi.
 * pinned by tests/test_oracle_krylov.py (T equals Arnoldi H on symmetric A; Lanczos relation). */
int orc_lanczos(int64_t n, const int32_t *rp, const int32_t *col, const double *val, double normA,
                int k0, int m, double *V, double *H, int ldh, int *brk)
{
    double *w = malloc((size_t)n * sizeof(double));
    if (!w) return -ORC_ENOMEM;
    *brk = 0;
    for (int j = k0; j < m; j++) {
        const double *vj = V + (size_t)j * n;
        orc_spmv(n, rp, col, val, vj, w);                                      /* w = A v_j */
        double tjj = orc_dot(n, vj, w);                                        /* t_jj = v_j^T w */
        double tprev = (j > 0) ? H[j + (size_t)(j - 1) * ldh] : 0.0;           /* t_{j,j-1} (t_{1,0}=0) */
        const double *vprev = (j > 0) ? V + (size_t)(j - 1) * n : NULL;        /* v_0 = 0 */
        for (int64_t r = 0; r < n; r++) {
            double a = w[r];
            if (vprev) a = a - tprev * vprev[r];
            w[r] = a - tjj * vj[r];
        }
        H[j + (size_t)j * ldh] = tjj;
        if (j > 0) H[(j - 1) + (size_t)j * ldh] = tprev;                      /* symmetric T */
        double tn = orc_norm2(n, w);
        H[(j + 1) + (size_t)j * ldh] = tn;
        if (is_breakdown(n, tn, normA)) { *brk = 1; free(w); return j + 1; }
        double *vn = V + (size_t)(j + 1) * n;
        for (int64_t r = 0; r < n; r++) vn[r] = w[r] / tn;
    }
    free(w);
    return m;
}

/* ------------------------------------------------------------------------------------------ */
/* Step size and Krylov dimension control (Sec. 3.3-3.4, Eq. tau_0, Eqs. 2-7, Alg. 3-4)         */
/* ------------------------------------------------------------------------------------------ */

/* Eq. (tau_0): tau_0 = (10/||A||) (Tol ((mbar+1)/e)^(mbar+1) sqrt(2 pi (mbar+1))
 *                                            / (4 ||A|| ||b0||))^(1/mbar). */
double orc_tau0(double normA, double b_inf, double tol, double mbar)
{
    const double e = 2.718281828459045235360287;
    const double pi = 3.141592653589793238462643;
    double num = tol * pow((mbar + 1.0) / e, mbar + 1.0) * sqrt(2.0 * pi * (mbar + 1.0));
    double den = 4.0 * normA * b_inf;
    return (10.0 / normA) * pow(num / den, 1.0 / mbar);
}

/* Eq. (4): cost of one step.  M is Eq. (8)'s M(.) of the exponentiated matrix (R20). */
double orc_cost_C1(int m, int p, int64_t n, int64_t NA, int symmetric, double M)
{
    double mp = (double)(m + p), K = (double)(m + p + 1);
    if (symmetric) return mp * (double)NA + 3.0 * mp * (double)n + M * K * K * K;
    return mp * (double)NA + ((double)m * m + 3.0 * p + 2.0) * (double)n + M * K * K * K;
}

/* Eq. (5): C(tau, m) = ceil((t_end - t_k)/tau) C1(m). */
double orc_cost_C(double remaining, double tau, double C1) { return ceil(remaining / tau) * C1; }

/* Controller memory for Algorithm 4, within one step (R15). */
typedef struct {
    int rejected;        /* previous attempt in this step was rejected */
    int last_branch;     /* 1 = tau was changed ("tau was reduced"), 2 = m was changed (R14) */
    int q_have;          /* q-hat was computed by Eq. (6) in the previous attempt */
    double q;
    int k_have;          /* kappa-hat was computed by Eq. (7) in the previous attempt */
    double kappa;
    double tau_old, eps_old;
    int m_old;
} orc_mem;

/* One controller decision (Alg. 4 then Alg. 3's branch), exported for the pin tests.
 * in : tau, m (this attempt), eps, omega, normH1 = ||H_mu||_1, remaining = t_end - t_k,
 *      problem sizes; mem (updated in place).
 * out: tau_next, m_next, and *branch (1 tau / 2 m), *qhat, *khat.
 * Readings: R2 (tau clamp [tau/5, 2tau] and <= remaining), R3 (strict <, ties to m), R13 (Eq. 6
 * as printed unless eq6_variant), R18 (ceil, clamps, m_max), R19 (guards), R20 (costs on the
 * clamped candidates; M on max(tau ||H_mu||_1, 1)), R35 (a rejected attempt whose m-branch
 * cannot grow m takes the tau-branch). */
void orc_control(double tau, int m, double eps, double omega, double normH1, double remaining,
                 int p, int64_t n, int64_t NA, int symmetric, int m_max, int fixed_m, int eq6_variant,
                 int accepted, orc_mem *mem, double *tau_next, int *m_next, int *branch,
                 double *qhat, double *khat)
{
    const double gamma = 0.8;
    /* Algorithm 4: heuristic order q-hat (Eq. 6) */
    double q;
    int q_now = 0;
    if (mem->rejected && mem->last_branch == 1) {
        double a = log(tau / mem->tau_old), b = log(eps / mem->eps_old);
        q = eq6_variant ? (b / a - 1.0) : (a / b - 1.0);
        if (isfinite(q) && q + 1.0 > 0.0) q_now = 1;
        else q = (double)m / 4.0;
    } else if (mem->rejected && mem->q_have) {
        q = mem->q; q_now = 1;           /* "keep old value" */
    } else {
        q = (double)m / 4.0;
    }
    double tau_new = tau * pow(gamma / omega, 1.0 / (q + 1.0));      /* Eq. (2) */
    /* kappa-hat (Eq. 7) */
    double kap;
    int k_now = 0;
    if (mem->rejected && mem->last_branch == 2) {
        kap = pow(eps / mem->eps_old, 1.0 / (double)(mem->m_old - m));
        if (isfinite(kap) && kap > 1.0) k_now = 1;
        else kap = 2.0;
    } else if (mem->rejected && mem->k_have) {
        kap = mem->kappa; k_now = 1;
    } else {
        kap = 2.0;
    }
    double m_new_real = (double)m + log(omega / gamma) / log(kap);   /* Eq. (3) */
    /* clamps (Alg. 3, R2, R18) */
    double tau_c = tau_new;
    if (!(tau_c >= tau / 5.0)) tau_c = tau / 5.0;                    /* also catches NaN */
    if (tau_c > 2.0 * tau) tau_c = 2.0 * tau;
    if (tau_c > remaining) tau_c = remaining;
    int m_lo = (3 * m) / 4; if (m_lo < 1) m_lo = 1;
    int m_hi = (4 * m + 2) / 3;                                      /* ceil(4m/3) */
    if (m_hi > m_max) m_hi = m_max;
    if (m_lo > m_hi) m_lo = m_hi;
    int m_c;
    double mr = ceil(m_new_real);
    if (!(mr >= (double)m_lo)) m_c = m_lo;                           /* also catches NaN/-inf */
    else if (mr > (double)m_hi) m_c = m_hi;
    else m_c = (int)mr;
    /* Alg. 3 choice by Eq. (5) on the clamped candidates (R20) */
    double M_tau = orc_cost_M(fmax(tau_c * normH1, 1.0));
    double M_m = orc_cost_M(fmax(tau * normH1, 1.0));
    double C_tau = orc_cost_C(remaining, tau_c, orc_cost_C1(m, p, n, NA, symmetric, M_tau));
    double C_m = orc_cost_C(remaining, tau, orc_cost_C1(m_c, p, n, NA, symmetric, M_m));
    int br = (C_tau < C_m) ? 1 : 2;
    if (fixed_m) br = 1;                                             /* phip mode: tau only */
    if (!accepted && br == 2 && m_c == m) br = 1;                    /* R35 */
    *branch = br;
    *tau_next = (br == 1) ? tau_c : tau;
    *m_next = (br == 2) ? m_c : m;
    *qhat = q; *khat = kap;
    /* memory for the next attempt (R15): only used if this attempt is rejected */
    mem->q = q; mem->q_have = q_now;
    mem->kappa = kap; mem->k_have = k_now;
    if (!accepted) {
        mem->rejected = 1; mem->last_branch = br;
        mem->tau_old = tau; mem->eps_old = eps; mem->m_old = m;
    }
}

/* ------------------------------------------------------------------------------------------ */
/* The phipm solve (Algorithm 3)                                                     */
/* ------------------------------------------------------------------------------------------ */

/* stats[0..7]: nsteps, nreject, nspmv, nexpm, m_last, m_peak, (unused), (unused);
 * t_reached in *t_reached.  trace (optional, 10 doubles per attempt, up to max_trace attempts):
 * {t_k, tau, m, mu, omega, eps, accepted, branch, normH1, beta}. */
int orc_phipm(double t_end, int64_t n, const int32_t *rp, const int32_t *col, const double *val,
              int p, const double *u /* (p+1) x n, row k = u_k */, double tol,
              int m_init, int m_max, int symmetric, int fixed_m, int eq6_variant,
              double *w /* out, n */, int64_t *stats, double *t_reached,
              double *trace, int max_trace, int *n_trace)
{
    const double delta = 1.2;
    int ntr = 0;
    for (int i = 0; i < 8; i++) stats[i] = 0;
    if (n_trace) *n_trace = 0;
    *t_reached = 0.0;
    if (n <= 0 || p < 0 || !(tol > 0.0) || !(t_end >= 0.0) || m_init < 1 || m_max < m_init) return ORC_EINVAL;
    /* degenerate inputs (R7, R23) */
    int allzero = 1;
    for (int k = 0; k <= p && allzero; k++)
        for (int64_t r = 0; r < n; r++) if (u[(size_t)k * n + r] != 0.0) { allzero = 0; break; }
    if (allzero || t_end == 0.0) {
        for (int64_t r = 0; r < n; r++) w[r] = allzero ? 0.0 : u[r];
        *t_reached = t_end;
        return ORC_OK;
    }
    int64_t NA = rp[n] - rp[0];
    double normA = orc_inf_norm(n, rp, val);
    int mmax = m_max < n ? m_max : (int)n;
    int m = m_init < mmax ? m_init : mmax;
    /* initial step (Eq. tau_0, R6, R7) */
    double b_inf = 0.0;
    for (int k = 0; k <= p && b_inf == 0.0; k++)
        for (int64_t r = 0; r < n; r++) { double a = fabs(u[(size_t)k * n + r]); if (a > b_inf) b_inf = a; }
    double mbar = 0.5 * ((double)m_init + (double)mmax);
    double tau;
    if (normA == 0.0) tau = t_end;
    else { tau = orc_tau0(normA, b_inf, tol, mbar); if (!(tau <= t_end)) tau = t_end; }

    int ldh = mmax + 1;
    double *V = malloc((size_t)n * (mmax + 1) * sizeof(double));
    double *H = calloc((size_t)ldh * mmax, sizeof(double));
    double *W = malloc((size_t)n * (p + 1) * sizeof(double));      /* w_0..w_p */
    double *F = malloc((size_t)n * sizeof(double));
    double *uk = malloc((size_t)n * sizeof(double));
    double *phip = malloc((size_t)(mmax + 1) * sizeof(double)), *phip1 = malloc((size_t)(mmax + 1) * sizeof(double));
    int status = ORC_OK;
    if (!V || !H || !W || !F || !uk || !phip || !phip1) { status = ORC_ENOMEM; goto out; }
    memcpy(uk, u, (size_t)n * sizeof(double));
    double tk = 0.0;
    stats[5] = m;
    while (tk < t_end) {
        if (tau > t_end - tk) tau = t_end - tk;                      /* step 2(a) */
        /* Eq. (wrecurrence): w_0 = u_k, w_j = A w_{j-1} + sum_{l=0}^{p-j} t_k^l/l! b_{j+l} */
        memcpy(W, uk, (size_t)n * sizeof(double));
        for (int j = 1; j <= p; j++) {
            double *wj = W + (size_t)j * n;
            orc_spmv(n, rp, col, val, W + (size_t)(j - 1) * n, wj);
            stats[2]++;
            double coef = 1.0;                                       /* t_k^l / l! */
            for (int l = 0; l <= p - j; l++) {
                if (l > 0) coef = coef * tk / (double)l;
                const double *b = u + (size_t)(j + l) * n;
                for (int64_t r = 0; r < n; r++) wj[r] = wj[r] + coef * b[r];
            }
        }
        const double *wp = W + (size_t)p * n;
        double beta = orc_norm2(n, wp);
        if (!isfinite(beta)) { status = ORC_ENONFINITE; goto out; }
        int k = 0, brk = 0;                                          /* built basis size */
        if (beta > 0.0)
            for (int64_t r = 0; r < n; r++) V[r] = wp[r] / beta;     /* v_1 = v/||v|| */
        orc_mem mem;
        memset(&mem, 0, sizeof(mem));
        int attempts = 0;
        double tau_used;
        int mu = 0, m_used = m;
        double hcorr = 0.0, eps;
        for (;;) {
            attempts++;
            double normH1 = 0.0;
            if (beta == 0.0) {                                       /* R23: F = 0, eps = 0 */
                mu = 0; eps = 0.0;
            } else {
                if (k < m && !brk) {                                 /* extend k -> m (R17) */
                    int kk = symmetric ? orc_lanczos(n, rp, col, val, normA, k, m, V, H, ldh, &brk)
                                       : orc_arnoldi(n, rp, col, val, normA, k, m, V, H, ldh, &brk);
                    if (kk < 0) { status = -kk; goto out; }
                    stats[2] += kk - k;
                    k = kk;
                }
                mu = m < k ? m : k;
                int st = orc_phi_pair(mu, H, ldh, tau, p, phip, phip1, &normH1);
                stats[3]++;
                if (st != ORC_OK) { status = st; goto out; }
                /* Eq. (errest)/(phipapprox2) with A -> tau A (R9, R10): h = tau h_{mu+1,mu} */
                hcorr = (brk && mu == k) ? 0.0 : H[mu + (size_t)(mu - 1) * ldh];
                eps = pow(tau, (double)p) * beta * tau * fabs(hcorr * phip1[mu - 1]);
            }
            double omega = t_end * eps / (tau * tol);                /* Eq. (taunew) */
            if (!isfinite(omega)) { status = ORC_ENONFINITE; goto out; }
            int accepted = omega <= delta;                           /* R1 */
            double tau_next, qh, kh;
            int m_next, branch;
            orc_control(tau, m, eps, omega, normH1, t_end - tk, p, n, NA, symmetric, mmax, fixed_m,
                        eq6_variant, accepted, &mem, &tau_next, &m_next, &branch, &qh, &kh);
            if (trace && ntr < max_trace) {
                double *tr = trace + (size_t)ntr * 10;
                tr[0] = tk; tr[1] = tau; tr[2] = m; tr[3] = mu; tr[4] = omega; tr[5] = eps;
                tr[6] = accepted; tr[7] = branch; tr[8] = normH1; tr[9] = beta;
            }
            ntr++;
            tau_used = tau;
            m_used = m;
            if (m > (int)stats[5]) stats[5] = m;
            tau = tau_next;
            m = m_next;
            if (accepted) break;
            stats[1]++;
            if (attempts >= 100 || tau < 1e-15 * t_end) { status = ORC_ESTEP; goto out; }
        }
        /* F = beta V_mu phi_p e1 + beta tau h phi_{p+1}[mu] v_{mu+1} (Eq. phipapprox2, R9)
         * u_{k+1} = tau^p F + sum_{j<p} tau^j/j! w_j            (Eq. step) */
        for (int64_t r = 0; r < n; r++) F[r] = 0.0;
        if (mu > 0) {
            for (int i = 0; i < mu; i++) {
                double c = beta * phip[i];
                const double *vi = V + (size_t)i * n;
                for (int64_t r = 0; r < n; r++) F[r] = F[r] + c * vi[r];
            }
            if (hcorr != 0.0) {
                double c = beta * tau_used * hcorr * phip1[mu - 1];
                const double *vi = V + (size_t)mu * n;
                for (int64_t r = 0; r < n; r++) F[r] = F[r] + c * vi[r];
            }
        }
        double taup = pow(tau_used, (double)p);
        for (int64_t r = 0; r < n; r++) uk[r] = taup * F[r];
        double coef = 1.0;                                           /* tau^j / j! */
        for (int j = 0; j < p; j++) {
            if (j > 0) coef = coef * tau_used / (double)j;
            const double *wj = W + (size_t)j * n;
            for (int64_t r = 0; r < n; r++) uk[r] = uk[r] + coef * wj[r];
        }
        if (tau_used >= t_end - tk) tk = t_end; else tk = tk + tau_used;   /* R25 */
        stats[0]++;
        stats[4] = m_used;
        *t_reached = tk;
    }
    memcpy(w, uk, (size_t)n * sizeof(double));
out:
    if (n_trace) *n_trace = ntr;
    free(V); free(H); free(W); free(F); free(uk); free(phip); free(phip1);
    return status;
}
