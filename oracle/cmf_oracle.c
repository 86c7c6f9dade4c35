/*
 * cmf_oracle.c -- CPU restatement of the reference ALS half-iteration.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_1808_03843_b200/ links, loads or
 * calls this file.  It is imported by tests/ (as the checker), by
 * __graft_entry__.smoke() (as the checker) and by bench.py's cpu_baseline /
 * --impl reference leg (as the timed CPU port of the reference path).
 *
 * Pinned against golden vectors produced by the reference package itself
 * (tests/golden/make_golden.py imports /root/reference/pkg in this container
 * and writes .npz fixtures under tests/golden; tests/test_oracle.py checks bitwise where
 * the reference is bitwise deterministic and to 1e-12 where LAPACK is used).
 *
 * Each function names the reference lines it restates.  Build flags MUST keep
 * -ffp-contract=off: the reference (numba, fastmath=False) never fuses a
 * multiply into an add, and the Gram / CG loops below are bitwise equal to it
 * only when the compiler does not either.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
    return omp_get_max_threads();
#else
    (void)nthreads;
    return 1;
#endif
}

int oracle_max_threads(void) { return set_threads(0); }

/*
 * Gram assembly + right-hand side for rows [0, nrows) of a CSR/CSC view.
 * Restates gram.py:149-187 (_accumulate_row), :190-206 (_accumulate_chunk) and
 * :209-220 (_bias_chunk), as driven by assemble_side gram.py:236-314.
 *
 * Per packed entry (i, j<=i) the reference starts from base[k] and, for every
 * stored position p of the row in CSR order, applies
 *     scratch[i,j] = fl32( scratch[i,j] + fl32( fl32(w_p * theta_i) * theta_j ) )
 * (the tile/batch loops only reorder *different* entries, gram.py:16-18), then
 * adds float32(lam * n_u) (or float32(lam)) to the diagonal, gram.py:183-186.
 * The bias accumulates float64(w_p) * float64(theta_c) in CSR order and rounds
 * once to float32, gram.py:214-220.
 *
 * a_w == NULL means all-ones (gram.py:275-276); b_w == NULL skips the bias.
 * base == NULL means zeros (gram.py:269-270).  a_out is float32 (nrows x P);
 * the fp16 store is a separate pass (oracle_pack_half), as in gram.py:300-301.
 */
int oracle_assemble(const int64_t *indptr, const int32_t *indices,
                    const float *a_w, const float *b_w, int64_t nrows,
                    const float *theta, int f, double lam, int weighted,
                    const float *base, float *a_out, float *b_out,
                    int64_t *nu_out, int nthreads) {
    const int64_t P = (int64_t)f * (f + 1) / 2;
    set_threads(nthreads);
#pragma omp parallel
    {
        float *scaled = (float *)malloc(sizeof(float) * (size_t)f);
        double *acc = (double *)malloc(sizeof(double) * (size_t)f);
#pragma omp for schedule(dynamic, 16)
        for (int64_t u = 0; u < nrows; ++u) {
            float *A = a_out + u * P;
            const int64_t lo = indptr[u], hi = indptr[u + 1];
            for (int64_t k = 0; k < P; ++k) A[k] = base ? base[k] : 0.0f;
            for (int c = 0; c < f; ++c) acc[c] = 0.0;
            for (int64_t p = lo; p < hi; ++p) {
                const float *t = theta + (int64_t)indices[p] * f;
                const float w = a_w ? a_w[p] : 1.0f;
                for (int i = 0; i < f; ++i) scaled[i] = w * t[i];
                float *row = A;
                for (int i = 0; i < f; ++i) {
                    const float ci = scaled[i];
                    for (int j = 0; j <= i; ++j) {
                        const float prod = ci * t[j];
                        row[j] = row[j] + prod;
                    }
                    row += i + 1;
                }
                if (b_w) {
                    const double wb = (double)b_w[p];
                    for (int c = 0; c < f; ++c) {
                        const double prod = wb * (double)t[c];
                        acc[c] = acc[c] + prod;
                    }
                }
            }
            const int64_t n_u = hi - lo;
            const float reg = weighted ? (float)(lam * (double)n_u) : (float)lam;
            for (int i = 0; i < f; ++i) {
                float *d = A + (int64_t)i * (i + 1) / 2 + i;
                *d = *d + reg;
            }
            if (b_out)
                for (int c = 0; c < f; ++c) b_out[u * f + c] = (float)acc[c];
            if (nu_out) nu_out[u] = n_u;
        }
        free(scaled);
        free(acc);
    }
    return 0;
}

/*
 * float32 -> IEEE binary16, round to nearest even; restates the numpy cast in
 * gram.py:140 bit by bit.  Returns the number of finite inputs that became
 * infinite (gram.py:141-145 turns a non-zero count into NumericalError).
 */
static uint16_t f32_to_f16_rne(float x, int *overflow) {
    uint32_t u;
    memcpy(&u, &x, 4);
    const uint32_t sign = (u >> 16) & 0x8000u;
    const uint32_t absu = u & 0x7fffffffu;
    if (absu >= 0x7f800000u) {                       /* inf or nan */
        if (absu > 0x7f800000u) return (uint16_t)(sign | 0x7e00u | ((absu >> 13) & 0x3ffu));
        return (uint16_t)(sign | 0x7c00u);
    }
    const int32_t exp = (int32_t)(absu >> 23) - 127;
    if (exp > 15) { *overflow += 1; return (uint16_t)(sign | 0x7c00u); }
    if (exp >= -14) {                                /* normal half range */
        uint32_t mant = absu & 0x7fffffu;
        uint32_t h = ((uint32_t)(exp + 15) << 10) | (mant >> 13);
        const uint32_t rem = mant & 0x1fffu;
        if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h += 1u;  /* may carry into exponent */
        if ((h & 0x7fffu) >= 0x7c00u) *overflow += 1;
        return (uint16_t)(sign | h);
    }
    if (exp < -25) return (uint16_t)sign;              /* rounds to zero */
    /* subnormal half: value = mant_full * 2^(exp-23); quantum 2^-24 */
    const uint32_t mant_full = (absu & 0x7fffffu) | 0x800000u;
    const int shift = -exp - 1;                        /* 14 .. 24 */
    uint32_t h = mant_full >> shift;
    const uint32_t rem = mant_full & ((1u << shift) - 1u);
    const uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (h & 1u))) h += 1u;
    return (uint16_t)(sign | h);
}

int64_t oracle_pack_half(const float *in, uint16_t *out, int64_t n, int nthreads) {
    int64_t over = 0;
    set_threads(nthreads);
#pragma omp parallel for reduction(+ : over) schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        int o = 0;
        out[i] = f32_to_f16_rne(in[i], &o);
        over += o;
    }
    return over;
}

static double f16_to_f64(uint16_t h) {
    const int sign = (h >> 15) & 1;
    const int e = (h >> 10) & 0x1f;
    const int m = h & 0x3ff;
    double v;
    if (e == 0) v = ldexp((double)m, -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else v = ldexp((double)(m | 0x400), e - 25);
    return sign ? -v : v;
}

/*
 * Truncated CG on every system; restates solvers.py:70-80 (_symv),
 * :83-118 (_cg_system) and :121-145 (_cg_batch) operation for operation, in
 * float64 with no fused multiply-add.  a is packed lower, float32
 * (a_is_half == 0) or binary16 bits (a_is_half == 1), promoted element-wise.
 */
int oracle_cg_batch(const void *a, int a_is_half, const float *B, const float *X0,
                    const double *eps, int64_t nsys, int f, int f_s, float *out,
                    int64_t *iters, int64_t *broke, int nthreads) {
    const int64_t P = (int64_t)f * (f + 1) / 2;
    set_threads(nthreads);
#pragma omp parallel
    {
        double *sq = (double *)malloc(sizeof(double) * (size_t)f * f);
        double *vec = (double *)malloc(sizeof(double) * (size_t)f * 5);
#pragma omp for schedule(dynamic, 16)
        for (int64_t s = 0; s < nsys; ++s) {
            double *x = vec, *b = vec + f, *ap = vec + 2 * f, *r = vec + 3 * f, *p = vec + 4 * f;
            int64_t k = 0;
            for (int i = 0; i < f; ++i)
                for (int j = 0; j <= i; ++j, ++k) {
                    const double v = a_is_half ? f16_to_f64(((const uint16_t *)a)[s * P + k])
                                               : (double)((const float *)a)[s * P + k];
                    sq[i * f + j] = v;
                    sq[j * f + i] = v;
                }
            for (int i = 0; i < f; ++i) { x[i] = (double)X0[s * f + i]; b[i] = (double)B[s * f + i]; }
            /* _symv: y[i] += sq[j, i] * p[j], column sweep (solvers.py:74-80) */
#define SYMV(vin, yout)                                              \
    do {                                                             \
        for (int i_ = 0; i_ < f; ++i_) (yout)[i_] = 0.0;             \
        for (int j_ = 0; j_ < f; ++j_) {                             \
            const double c_ = (vin)[j_];                             \
            const double *row_ = sq + (int64_t)j_ * f;               \
            for (int i_ = 0; i_ < f; ++i_) {                         \
                const double t_ = row_[i_] * c_;                     \
                (yout)[i_] = (yout)[i_] + t_;                        \
            }                                                        \
        }                                                            \
    } while (0)
            SYMV(x, ap);
            for (int i = 0; i < f; ++i) r[i] = b[i] - ap[i];
            double rs_old = 0.0;
            for (int i = 0; i < f; ++i) { p[i] = r[i]; const double t = r[i] * r[i]; rs_old = rs_old + t; }
            int64_t it = 0, bd = 0;
            for (int step = 0; step < f_s; ++step) {
                SYMV(p, ap);
                double pap = 0.0;
                for (int i = 0; i < f; ++i) { const double t = p[i] * ap[i]; pap = pap + t; }
                if (pap <= 0.0) { bd = 1; break; }
                const double alpha = rs_old / pap;
                for (int i = 0; i < f; ++i) {
                    const double tx = alpha * p[i];
                    x[i] = x[i] + tx;
                    const double tr = alpha * ap[i];
                    r[i] = r[i] - tr;
                }
                double rs_new = 0.0;
                for (int i = 0; i < f; ++i) { const double t = r[i] * r[i]; rs_new = rs_new + t; }
                it += 1;
                if (rs_new == 0.0 || sqrt(rs_new) < eps[s]) break;
                const double beta = rs_new / rs_old;
                for (int i = 0; i < f; ++i) { const double t = beta * p[i]; p[i] = r[i] + t; }
                rs_old = rs_new;
            }
#undef SYMV
            for (int i = 0; i < f; ++i) out[s * f + i] = (float)x[i];
            iters[s] = it;
            broke[s] = bd;
        }
        free(sq);
        free(vec);
    }
    return 0;
}

/*
 * Exact solve: unpack to float64, lower Cholesky, two triangular solves;
 * restates solvers.py:148-164 (scipy cho_factor(lower=True) + cho_solve, i.e.
 * LAPACK dpotrf/dpotrs).  Unblocked column Cholesky: equal to LAPACK up to
 * float64 rounding (checked to 1e-12 in tests/test_oracle.py).  info[s] is 0
 * on success, k+1 if the k-th pivot is not positive (LAPACK convention); x is
 * left untouched for such systems.  Returns the number of failed systems.
 */
int64_t oracle_cholesky_batch(const float *a, const float *B, int64_t nsys, int f,
                              float *out, int32_t *info, int nthreads) {
    const int64_t P = (int64_t)f * (f + 1) / 2;
    int64_t nbad = 0;
    set_threads(nthreads);
#pragma omp parallel reduction(+ : nbad)
    {
        double *L = (double *)malloc(sizeof(double) * (size_t)f * f);
        double *y = (double *)malloc(sizeof(double) * (size_t)f);
#pragma omp for schedule(dynamic, 16)
        for (int64_t s = 0; s < nsys; ++s) {
            int64_t k = 0;
            for (int i = 0; i < f; ++i)
                for (int j = 0; j <= i; ++j, ++k) L[i * f + j] = (double)a[s * P + k];
            int bad = 0;
            for (int j = 0; j < f && !bad; ++j) {
                double d = L[j * f + j];
                for (int t = 0; t < j; ++t) d -= L[j * f + t] * L[j * f + t];
                if (!(d > 0.0)) { bad = j + 1; break; }
                d = sqrt(d);
                L[j * f + j] = d;
                for (int i = j + 1; i < f; ++i) {
                    double v = L[i * f + j];
                    for (int t = 0; t < j; ++t) v -= L[i * f + t] * L[j * f + t];
                    L[i * f + j] = v / d;
                }
            }
            info[s] = bad;
            if (bad) { nbad += 1; continue; }
            for (int i = 0; i < f; ++i) {          /* L y = b */
                double v = (double)B[s * f + i];
                for (int t = 0; t < i; ++t) v -= L[i * f + t] * y[t];
                y[i] = v / L[i * f + i];
            }
            for (int i = f - 1; i >= 0; --i) {     /* L^T x = y */
                double v = y[i];
                for (int t = i + 1; t < f; ++t) v -= L[t * f + i] * y[t];
                y[i] = v / L[i * f + i];
            }
            for (int i = 0; i < f; ++i) out[s * f + i] = (float)y[i];
        }
        free(L);
        free(y);
    }
    return nbad;
}
