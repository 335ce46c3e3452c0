/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.  Never linked into the product
 * (paper_1505_03410_b200/); only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Plain-C restatement of the reference's numba column kernels
 * (/root/reference/pkg/src/gapsafe/_kernels.py).  Every loop is strictly
 * sequential, left to right, with separate multiply and add roundings
 * (built with -ffp-contract=off, no -ffast-math), which is what the numba
 * code compiles to: SURVEY.md §2 records that a Python emulation of this
 * order matched numba bit-for-bit, and tests/test_oracle_kernels.py
 * re-checks these C versions against the numba kernels themselves.
 *
 * Index arrays are int64 (numpy np.flatnonzero / np.arange), CSC
 * indices/indptr are int32 (scipy canonical CSC), exactly as the reference
 * passes them.
 */
#include <stdint.h>

/* _kernels.py:14-24 tdot_dense.  X is Fortran-ordered (column j at X + j*ld). */
void oracle_tdot_dense(const double *X, int64_t n, int64_t ld, const double *v,
                       const int64_t *cols, int64_t k, double tail_scale,
                       double *out)
{
    for (int64_t i = 0; i < k; ++i) {
        const int64_t j = cols[i];
        const double *x = X + j * ld;
        double s = 0.0;
        for (int64_t r = 0; r < n; ++r)
            s += x[r] * v[r];
        if (tail_scale > 0.0)
            s += tail_scale * v[n + j];
        out[i] = s;
    }
}

/* _kernels.py:27-36 tdot_csc. */
void oracle_tdot_csc(const double *data, const int32_t *indices,
                     const int32_t *indptr, int64_t n_base, const double *v,
                     const int64_t *cols, int64_t k, double tail_scale,
                     double *out)
{
    for (int64_t i = 0; i < k; ++i) {
        const int64_t j = cols[i];
        double s = 0.0;
        for (int64_t q = indptr[j]; q < indptr[j + 1]; ++q)
            s += data[q] * v[indices[q]];
        if (tail_scale > 0.0)
            s += tail_scale * v[n_base + j];
        out[i] = s;
    }
}

/* _kernels.py:39-64 cd_pass_dense. */
void oracle_cd_pass_dense(const double *X, int64_t n, int64_t ld, double *beta,
                          double *rho, const int64_t *active, int64_t k,
                          double lam, const double *norms_sq, double tail_scale)
{
    for (int64_t i = 0; i < k; ++i) {
        const int64_t j = active[i];
        const double *x = X + j * ld;
        const double nsq = norms_sq[j];
        double g = 0.0;
        for (int64_t r = 0; r < n; ++r)
            g += x[r] * rho[r];
        if (tail_scale > 0.0)
            g += tail_scale * rho[n + j];
        const double z = beta[j] + g / nsq;
        const double u = lam / nsq;
        double nb;
        if (z > u)
            nb = z - u;
        else if (z < -u)
            nb = z + u;
        else
            nb = 0.0;
        const double d = nb - beta[j];
        if (d != 0.0) {
            beta[j] = nb;
            for (int64_t r = 0; r < n; ++r)
                rho[r] -= d * x[r];
            if (tail_scale > 0.0)
                rho[n + j] -= d * tail_scale;
        }
    }
}

/* _kernels.py:67-92 cd_pass_csc. */
void oracle_cd_pass_csc(const double *data, const int32_t *indices,
                        const int32_t *indptr, int64_t n_base, double *beta,
                        double *rho, const int64_t *active, int64_t k,
                        double lam, const double *norms_sq, double tail_scale)
{
    for (int64_t i = 0; i < k; ++i) {
        const int64_t j = active[i];
        const double nsq = norms_sq[j];
        double g = 0.0;
        for (int64_t q = indptr[j]; q < indptr[j + 1]; ++q)
            g += data[q] * rho[indices[q]];
        if (tail_scale > 0.0)
            g += tail_scale * rho[n_base + j];
        const double z = beta[j] + g / nsq;
        const double u = lam / nsq;
        double nb;
        if (z > u)
            nb = z - u;
        else if (z < -u)
            nb = z + u;
        else
            nb = 0.0;
        const double d = nb - beta[j];
        if (d != 0.0) {
            beta[j] = nb;
            for (int64_t q = indptr[j]; q < indptr[j + 1]; ++q)
                rho[indices[q]] -= d * data[q];
            if (tail_scale > 0.0)
                rho[n_base + j] -= d * tail_scale;
        }
    }
}
