/*
 * LSG-CPD FP64 CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  It shares no code, header, table or helper with the
 * CUDA product path (paper_2103_15039_b200/csrc); neither includes the other.
 *
 * Plain, slow, obviously-correct double precision evaluation of the paper's formulas.
 * Citations: P:<line> = /root/reference/PAPER.md line (LaTeX source of arXiv 2103.15039).
 *
 *   Eq. 1  p(x) = w p_o + (1-w) Σ_m π(m) p(x|m),  p_o = 1/V, π(m)=1/M
 *   Eq. 2  p(x|m) = c_m exp(-½ (x-y_m)ᵀ Σ_m⁻¹ (x-y_m)),  Σ_m⁻¹ = (α_m n_m n_mᵀ + I)/σ²
 *                      c_m = sqrt(det Σ_m⁻¹)/(2π)^{3/2} = sqrt(1+α_m)/(2πσ²)^{3/2}   (normalising constant)
 *   Eq. 5  P_mn = (1-w)π(m)p(x̂_n|m) / (w p_o + (1-w) Σ_m π(m) p(x̂_n|m)),  x̂_n = g_old(x_n)
 *
 * Reading (R1): consistent=1 uses the normalising c_m of Eq. 2; consistent=0 drops
 * the sqrt(1+α_m) factor as the matrix form of Eq. 9-10 does.
 *
 * Build (done by __graft_entry__.build() and tests/conftest.py):
 *   gcc -O2 -fopenmp -fPIC -shared -o oracle/liboracle.so oracle/lsgcpd_oracle.c -lm
 * No -ffast-math: IEEE semantics everywhere.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORA_REC 16

/*
 * Per-source-point E-step record (the sufficient statistics named by the north star):
 *   [0]      P_n      = Σ_m P_mn
 *   [1..3]   Σ_m P_mn y_m
 *   [4..9]   A_n      = Σ_m P_mn α_m n_m n_mᵀ       (xx, xy, xz, yy, yz, zz)
 *   [10..12] b_n      = Σ_m P_mn α_m (n_m·y_m) n_m
 *   [13]     D_n      = Σ_m P_mn d_mn,   d_mn = (x̂_n-y_m)ᵀ (α_m n_m n_mᵀ + I) (x̂_n-y_m) / σ²
 *   [14]     ln p(x̂_n)   (Eq. 1 with the Eq. 2 components; -Σ_n of it is the NLL of Eq. 4)
 *   [15]     P_o,n    = w p_o / p(x̂_n)   (outlier posterior; Σ_m P_mn + P_o,n = 1)
 *
 * The E step is evaluated per pair (m, n) exactly as Eq. 5 reads, in log space with the
 * usual max-subtraction (SPEC stabilisation; mathematically identical).  The max is taken in
 * a first pass over m, the sums in a second pass.
 */
void ora_estep(const double* Y, const double* Nrm, const double* alpha, int64_t M,
               const double* X, int64_t N, const double* R, const double* t,
               double sigma2, double w, double V, int consistent, double* rec, int nthreads)
{
    const double ln_mix = log((1.0 - w) / (double)M);                 /* ln((1-w) π(m)) */
    const double ln_gauss = -1.5 * log(2.0 * M_PI * sigma2);          /* ln (2πσ²)^{-3/2} */
    const double l_out = (w > 0.0) ? log(w / V) : -INFINITY;          /* ln(w p_o) */
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel
    {
        double* lbuf = (double*)malloc(sizeof(double) * (size_t)M);
        double* dbuf = (double*)malloc(sizeof(double) * (size_t)M);
#pragma omp for schedule(dynamic, 16)
        for (int64_t n = 0; n < N; ++n) {
            const double* x = X + 3 * n;
            double xh[3];
            for (int i = 0; i < 3; ++i)
                xh[i] = R[3 * i + 0] * x[0] + R[3 * i + 1] * x[1] + R[3 * i + 2] * x[2] + t[i];
            /* pass 1: log of the numerator of Eq. 5 for every component, and the max */
            double mu = l_out;
            for (int64_t m = 0; m < M; ++m) {
                const double* y = Y + 3 * m;
                const double* nm = Nrm + 3 * m;
                const double r0 = xh[0] - y[0], r1 = xh[1] - y[1], r2 = xh[2] - y[2];
                const double q = nm[0] * r0 + nm[1] * r1 + nm[2] * r2;
                const double d = (r0 * r0 + r1 * r1 + r2 * r2 + alpha[m] * q * q) / sigma2;
                const double ln_cm = ln_gauss + (consistent ? 0.5 * log(1.0 + alpha[m]) : 0.0);
                const double l = ln_mix + ln_cm - 0.5 * d;
                lbuf[m] = l;
                dbuf[m] = d;
                if (l > mu) mu = l;
            }
            /* pass 2: Z = Σ exp(l - μ) (including the outlier term) and the weighted sums */
            double Z = (w > 0.0) ? exp(l_out - mu) : 0.0;
            for (int64_t m = 0; m < M; ++m) Z += exp(lbuf[m] - mu);
            double acc[ORA_REC];
            memset(acc, 0, sizeof(acc));
            for (int64_t m = 0; m < M; ++m) {
                const double Pmn = exp(lbuf[m] - mu) / Z;
                const double* y = Y + 3 * m;
                const double* nm = Nrm + 3 * m;
                const double a = alpha[m];
                const double ny = nm[0] * y[0] + nm[1] * y[1] + nm[2] * y[2];
                acc[0] += Pmn;
                acc[1] += Pmn * y[0];
                acc[2] += Pmn * y[1];
                acc[3] += Pmn * y[2];
                acc[4] += Pmn * a * nm[0] * nm[0];
                acc[5] += Pmn * a * nm[0] * nm[1];
                acc[6] += Pmn * a * nm[0] * nm[2];
                acc[7] += Pmn * a * nm[1] * nm[1];
                acc[8] += Pmn * a * nm[1] * nm[2];
                acc[9] += Pmn * a * nm[2] * nm[2];
                acc[10] += Pmn * a * ny * nm[0];
                acc[11] += Pmn * a * ny * nm[1];
                acc[12] += Pmn * a * ny * nm[2];
                acc[13] += Pmn * dbuf[m];
            }
            acc[14] = mu + log(Z);                                        /* ln p(x̂_n) */
            acc[15] = (w > 0.0) ? exp(l_out - mu) / Z : 0.0;             /* P_o,n */
            memcpy(rec + ORA_REC * n, acc, sizeof(acc));
        }
        free(lbuf);
        free(dbuf);
    }
}

/*
 * Eq. 1 / Eq. 5 with the confidence-filtered model of Eq. 8: per-component prior
 * π(m) (prior[m], Σ_m π(m) = 1) and per-point outlier weight w_n (wn[n] ∈ [0, 1]):
 *   p(x̂_n) = w_n p_o + (1 - w_n) Σ_m π(m) p(x̂_n|m),
 *   P_mn   = (1 - w_n) π(m) p(x̂_n|m) / p(x̂_n),   P_o,n = w_n p_o / p(x̂_n).
 * With π(m) = 1/M and w_n = w it is ora_estep term for term.  w_n = 1 gives P_o,n = 1 exactly
 * (every component term is multiplied by 1 - w_n = 0).  Same record layout as ora_estep.
 */
void ora_estep_cf(const double* Y, const double* Nrm, const double* alpha, const double* prior, int64_t M,
                  const double* X, const double* wn, int64_t N, const double* R, const double* t,
                  double sigma2, double V, int consistent, double* rec, int nthreads)
{
    const double ln_gauss = -1.5 * log(2.0 * M_PI * sigma2);          /* ln (2πσ²)^{-3/2} */
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel
    {
        double* lbuf = (double*)malloc(sizeof(double) * (size_t)M);
        double* dbuf = (double*)malloc(sizeof(double) * (size_t)M);
#pragma omp for schedule(dynamic, 16)
        for (int64_t n = 0; n < N; ++n) {
            const double w = wn[n];
            const double l_out = (w > 0.0) ? log(w / V) : -INFINITY;      /* ln(w_n p_o) */
            const double ln_keep = (w < 1.0) ? log(1.0 - w) : -INFINITY;  /* ln(1 - w_n) */
            const double* x = X + 3 * n;
            double xh[3];
            for (int i = 0; i < 3; ++i)
                xh[i] = R[3 * i + 0] * x[0] + R[3 * i + 1] * x[1] + R[3 * i + 2] * x[2] + t[i];
            double mu = l_out;
            for (int64_t m = 0; m < M; ++m) {
                const double* y = Y + 3 * m;
                const double* nm = Nrm + 3 * m;
                const double r0 = xh[0] - y[0], r1 = xh[1] - y[1], r2 = xh[2] - y[2];
                const double q = nm[0] * r0 + nm[1] * r1 + nm[2] * r2;
                const double d = (r0 * r0 + r1 * r1 + r2 * r2 + alpha[m] * q * q) / sigma2;
                const double ln_cm = ln_gauss + (consistent ? 0.5 * log(1.0 + alpha[m]) : 0.0);
                const double l = ln_keep + log(prior[m]) + ln_cm - 0.5 * d;   /* ln((1-w_n) π(m) p(x̂|m)) */
                lbuf[m] = l;
                dbuf[m] = d;
                if (l > mu) mu = l;
            }
            double Z = (w > 0.0) ? exp(l_out - mu) : 0.0;
            for (int64_t m = 0; m < M; ++m) Z += exp(lbuf[m] - mu);
            double acc[ORA_REC];
            memset(acc, 0, sizeof(acc));
            for (int64_t m = 0; m < M; ++m) {
                const double Pmn = exp(lbuf[m] - mu) / Z;
                const double* y = Y + 3 * m;
                const double* nm = Nrm + 3 * m;
                const double a = alpha[m];
                const double ny = nm[0] * y[0] + nm[1] * y[1] + nm[2] * y[2];
                acc[0] += Pmn;
                acc[1] += Pmn * y[0];
                acc[2] += Pmn * y[1];
                acc[3] += Pmn * y[2];
                acc[4] += Pmn * a * nm[0] * nm[0];
                acc[5] += Pmn * a * nm[0] * nm[1];
                acc[6] += Pmn * a * nm[0] * nm[2];
                acc[7] += Pmn * a * nm[1] * nm[1];
                acc[8] += Pmn * a * nm[1] * nm[2];
                acc[9] += Pmn * a * nm[2] * nm[2];
                acc[10] += Pmn * a * ny * nm[0];
                acc[11] += Pmn * a * ny * nm[1];
                acc[12] += Pmn * a * ny * nm[2];
                acc[13] += Pmn * dbuf[m];
            }
            acc[14] = mu + log(Z);
            acc[15] = (w > 0.0) ? exp(l_out - mu) / Z : 0.0;
            memcpy(rec + ORA_REC * n, acc, sizeof(acc));
        }
        free(lbuf);
        free(dbuf);
    }
}

/*
 * Posterior matrix P (M×N, row-major P[m*N+n]) and outlier posterior (N) — tiny sizes only.
 * Same per-pair evaluation as ora_estep; used by the tests to compare element by element.
 */
void ora_posterior(const double* Y, const double* Nrm, const double* alpha, int64_t M,
                   const double* X, int64_t N, const double* R, const double* t,
                   double sigma2, double w, double V, int consistent, double* Pmat, double* Pout)
{
    const double ln_mix = log((1.0 - w) / (double)M);
    const double ln_gauss = -1.5 * log(2.0 * M_PI * sigma2);
    const double l_out = (w > 0.0) ? log(w / V) : -INFINITY;
    double* lbuf = (double*)malloc(sizeof(double) * (size_t)M);
    for (int64_t n = 0; n < N; ++n) {
        const double* x = X + 3 * n;
        double xh[3];
        for (int i = 0; i < 3; ++i)
            xh[i] = R[3 * i + 0] * x[0] + R[3 * i + 1] * x[1] + R[3 * i + 2] * x[2] + t[i];
        double mu = l_out;
        for (int64_t m = 0; m < M; ++m) {
            const double* y = Y + 3 * m;
            const double* nm = Nrm + 3 * m;
            const double r0 = xh[0] - y[0], r1 = xh[1] - y[1], r2 = xh[2] - y[2];
            const double q = nm[0] * r0 + nm[1] * r1 + nm[2] * r2;
            const double d = (r0 * r0 + r1 * r1 + r2 * r2 + alpha[m] * q * q) / sigma2;
            const double l = ln_mix + ln_gauss + (consistent ? 0.5 * log(1.0 + alpha[m]) : 0.0) - 0.5 * d;
            lbuf[m] = l;
            if (l > mu) mu = l;
        }
        double Z = (w > 0.0) ? exp(l_out - mu) : 0.0;
        for (int64_t m = 0; m < M; ++m) Z += exp(lbuf[m] - mu);
        for (int64_t m = 0; m < M; ++m) Pmat[m * N + n] = exp(lbuf[m] - mu) / Z;
        Pout[n] = (w > 0.0) ? exp(l_out - mu) / Z : 0.0;
    }
    free(lbuf);
}

/*
 * Exact k-nearest neighbours by brute force (SPEC spatial_index semantics):
 * each query's neighbourhood includes the point itself; ties in squared distance go to the
 * lower id.  queries == NULL means all M points.  idx is nq×k (int32).
 */
void ora_knn(const double* P, int64_t M, const int64_t* queries, int64_t nq, int k,
             int32_t* idx, double* dist2, int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    if (queries == NULL) nq = M;
#pragma omp parallel
    {
        double* bd = (double*)malloc(sizeof(double) * (size_t)(k + 1));
        int64_t* bi = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k + 1));
#pragma omp for schedule(dynamic, 64)
        for (int64_t qi = 0; qi < nq; ++qi) {
            const int64_t q = queries ? queries[qi] : qi;
            const double* p = P + 3 * q;
            int cnt = 0;
            for (int64_t j = 0; j < M; ++j) {
                const double dx = P[3 * j] - p[0], dy = P[3 * j + 1] - p[1], dz = P[3 * j + 2] - p[2];
                const double d = dx * dx + dy * dy + dz * dz;
                /* insertion into the sorted (d, id) list of length <= k */
                if (cnt == k && !(d < bd[k - 1] || (d == bd[k - 1] && j < bi[k - 1]))) continue;
                int pos = (cnt < k) ? cnt : k - 1;
                while (pos > 0 && (d < bd[pos - 1] || (d == bd[pos - 1] && j < bi[pos - 1]))) {
                    bd[pos] = bd[pos - 1];
                    bi[pos] = bi[pos - 1];
                    --pos;
                }
                bd[pos] = d;
                bi[pos] = j;
                if (cnt < k) ++cnt;
            }
            for (int i = 0; i < k; ++i) {
                idx[qi * k + i] = (int32_t)(i < cnt ? bi[i] : -1);
                if (dist2) dist2[qi * k + i] = i < cnt ? bd[i] : INFINITY;
            }
        }
        free(bd);
        free(bi);
    }
}

/* Σ_{m,n} ||x̂_n - y_m||² by the plain double loop (pins the closed form of σ²₀). */
double ora_sum_sq_pairs(const double* X, int64_t N, const double* Y, int64_t M, int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    double total = 0.0;
#pragma omp parallel for reduction(+ : total) schedule(static)
    for (int64_t n = 0; n < N; ++n) {
        double s = 0.0;
        for (int64_t m = 0; m < M; ++m) {
            const double dx = X[3 * n] - Y[3 * m], dy = X[3 * n + 1] - Y[3 * m + 1], dz = X[3 * n + 2] - Y[3 * m + 2];
            s += dx * dx + dy * dy + dz * dz;
        }
        total += s;
    }
    return total;
}

int ora_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
