/*
 * ks_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference kronschro hot path, used as the
 * parity checker for the CUDA product (paper_2311_18461_b200/libks.so) and as
 * the "port" CPU baseline in bench.py. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. The
 * product never links or calls it.
 *
 * Parity pin: the restatement is checked against the reference's own
 * sources compiled unmodified into oracle/_ref (oracle/build_ref.sh, Eigen
 * subset shim in oracle/eigen_shim) and against golden vectors generated
 * from that build (tests/golden/, tests/golden/make_golden.py).
 *
 * Every function follows the reference line by line (file:line relative to
 * /root/reference/proj), single-threaded, scalar kernels (src/kernels.cpp).
 * Complex arithmetic is C99 double _Complex, which GCC lowers like
 * std::complex<double> (same __muldc3/__divdc3 semantics, no FMA on x86-64).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double _Complex cplx;

/* ---------------- BLAS-1: src/kernels.cpp:10-34 (scalar backend) ---------- */
void ko_axpy_real(double a, const cplx* x, cplx* y, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] += a * x[i];
}
void ko_axpy(cplx a, const cplx* x, cplx* y, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] += a * x[i];
}
void ko_dotc(const cplx* x, const cplx* y, size_t n, double* re_out, double* im_out) {
    double re = 0.0, im = 0.0;
    for (size_t i = 0; i < n; ++i) {
        re += creal(x[i]) * creal(y[i]) + cimag(x[i]) * cimag(y[i]);
        im += creal(x[i]) * cimag(y[i]) - cimag(x[i]) * creal(y[i]);
    }
    *re_out = re;
    *im_out = im;
}
double ko_norm2sq(const cplx* x, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += creal(x[i]) * creal(x[i]) + cimag(x[i]) * cimag(x[i]);
    return s;
}

/* ---------------- tensor geometry: src/tensorops.cpp:24-29, :70-79 ---------- */
static void geom(const int* dims, int ndim, int axis, size_t* s, int* nm, size_t* outer) {
    size_t st = 1, tot = 1;
    for (int k = 0; k < ndim; ++k) tot *= (size_t)dims[k];
    for (int k = 0; k < axis; ++k) st *= (size_t)dims[k];
    *s = st;
    *nm = dims[axis];
    *outer = tot / (st * (size_t)dims[axis]);
}

/* banded entry, include/kronschro/banded.hpp:32-34, :91-94 */
static cplx band_get(const cplx* a, int n, int bw, int i, int j) {
    if (i < 0 || j < 0 || i >= n || j >= n || abs(i - j) > bw) return 0;
    return a[(size_t)(bw + i - j) + (size_t)j * (2 * bw + 1)];
}

/* BandedMatrix::matvec, banded.hpp:42-51 */
static void band_matvec(const cplx* a, int n, int bw, const cplx* x, cplx* y) {
    for (int i = 0; i < n; ++i) {
        cplx s = 0;
        const int j0 = i - bw > 0 ? i - bw : 0;
        const int j1 = i + bw < n - 1 ? i + bw : n - 1;
        for (int j = j0; j <= j1; ++j) s += a[(size_t)(bw + i - j) + (size_t)j * (2 * bw + 1)] * x[j];
        y[i] = s;
    }
}

/* mode_product(X, BandedMatrix<cplx>, axis): src/tensorops.cpp:89-123. Y must be zeroed. */
void ko_mode_product_band(const cplx* band, int bw, const cplx* X, cplx* Y, const int* dims,
                          int ndim, int axis) {
    size_t s, outer;
    int nm;
    geom(dims, ndim, axis, &s, &nm, &outer);
    const size_t total = s * (size_t)nm * outer;
    memset(Y, 0, total * sizeof(cplx));
    if (s == 1) {
        for (size_t o = 0; o < outer; ++o) band_matvec(band, nm, bw, X + o * nm, Y + o * nm);
        return;
    }
    const size_t slab = s * (size_t)nm;
    for (size_t o = 0; o < outer; ++o) {
        const cplx* xin = X + o * slab;
        cplx* yout = Y + o * slab;
        for (int r = 0; r < nm; ++r) {
            cplx* ycol = yout + (size_t)r * s;
            const int j0 = r - bw > 0 ? r - bw : 0;
            const int j1 = r + bw < nm - 1 ? r + bw : nm - 1;
            for (int j = j0; j <= j1; ++j) {
                const cplx a = band_get(band, nm, bw, r, j);
                if (a == 0) continue;
                const cplx* xcol = xin + (size_t)j * s;
                if (cimag(a) == 0.0) ko_axpy_real(creal(a), xcol, ycol, s);
                else ko_axpy(a, xcol, ycol, s);
            }
        }
    }
}

/* mode_product(X, Eigen::MatrixXd J, axis): src/tensorops.cpp:125-156.
 * J given column-major (rows x cols = l x nm); transposeJ uses J^T. */
void ko_mode_product_dense(const double* Jcm, int transposeJ, const cplx* X, cplx* Y,
                           const int* dims, int ndim, int axis) {
    size_t s, outer;
    int nm;
    geom(dims, ndim, axis, &s, &nm, &outer);
    const int l = nm; /* square */
#define JAT(r, j) (transposeJ ? Jcm[(size_t)(j) + (size_t)(r) * nm] : Jcm[(size_t)(r) + (size_t)(j) * nm])
    const size_t slab = s * (size_t)nm;
    memset(Y, 0, slab * outer * sizeof(cplx));
    for (size_t o = 0; o < outer; ++o) {
        const cplx* xin = X + o * slab;
        cplx* yout = Y + o * slab;
        if (s == 1) {
            for (int r = 0; r < l; ++r) {
                cplx acc = 0;
                for (int j = 0; j < nm; ++j) acc += JAT(r, j) * xin[j];
                yout[r] = acc;
            }
        } else {
            for (int r = 0; r < l; ++r) {
                cplx* ycol = yout + (size_t)r * s;
                for (int j = 0; j < nm; ++j) {
                    const double a = JAT(r, j);
                    if (a != 0.0) ko_axpy_real(a, xin + (size_t)j * s, ycol, s);
                }
            }
        }
    }
#undef JAT
}

/* ---------------- banded LU: src/eigensolve.cpp:77-140, :148-170 ---------- */
/* ab: ldab x n, ldab = 3p+1, a(i,j) at ab[kuf + i - j + j*ldab], kuf = 2p.  */
int ko_factor_banded(const cplx* H, int n, int p, cplx* ab, int* piv) {
    const int kl = p, ku0 = p, kuf = kl + ku0, ldab = 2 * kl + ku0 + 1;
#define A(i, j) ab[(size_t)(kuf + (i) - (j)) + (size_t)(j) * ldab]
    memset(ab, 0, (size_t)ldab * n * sizeof(cplx));
    for (int j = 0; j < n; ++j)
        for (int i = (j - ku0 > 0 ? j - ku0 : 0); i <= (j + kl < n - 1 ? j + kl : n - 1); ++i)
            A(i, j) = band_get(H, n, p, i, j);
    for (int k = 0; k < n; ++k) {
        const int imax = k + kl < n - 1 ? k + kl : n - 1;
        int pr = k;
        double best = cabs(A(k, k));
        for (int i = k + 1; i <= imax; ++i)
            if (cabs(A(i, k)) > best) {
                best = cabs(A(i, k));
                pr = i;
            }
        piv[k] = pr;
        if (best == 0.0) return 2; /* numerically singular pivot (:105-106) */
        const int jmax = k + kuf < n - 1 ? k + kuf : n - 1;
        if (pr != k)
            for (int j = k; j <= jmax; ++j) {
                const cplx t = A(k, j);
                A(k, j) = A(pr, j);
                A(pr, j) = t;
            }
        const cplx pivval = A(k, k);
        for (int i = k + 1; i <= imax; ++i) {
            const cplx m = A(i, k) / pivval;
            A(i, k) = m;
            if (m != 0)
                for (int j = k + 1; j <= jmax; ++j) A(i, j) -= m * A(k, j);
        }
    }
    return 0;
#undef A
}

void ko_solve_banded(const cplx* ab, const int* piv, int n, int p, cplx* x) {
    const int kl = p, kuf = 2 * p, ldab = kl + kuf + 1;
#define A(i, j) ab[(size_t)(kuf + (i) - (j)) + (size_t)(j) * ldab]
    for (int k = 0; k < n; ++k) {
        if (piv[k] != k) {
            const cplx t = x[k];
            x[k] = x[piv[k]];
            x[piv[k]] = t;
        }
        const int imax = k + kl < n - 1 ? k + kl : n - 1;
        for (int i = k + 1; i <= imax; ++i) x[i] -= A(i, k) * x[k];
    }
    for (int k = n - 1; k >= 0; --k) {
        x[k] /= A(k, k);
        const int imin = k - kuf > 0 ? k - kuf : 0;
        for (int i = imin; i < k; ++i) x[i] -= A(i, k) * x[k];
    }
#undef A
}

void ko_solve_banded_adjoint(const cplx* ab, const int* piv, int n, int p, cplx* x) {
    const int kl = p, kuf = 2 * p, ldab = kl + kuf + 1;
#define A(i, j) ab[(size_t)(kuf + (i) - (j)) + (size_t)(j) * ldab]
    for (int k = 0; k < n; ++k) {
        cplx s = x[k];
        const int imin = k - kuf > 0 ? k - kuf : 0;
        for (int i = imin; i < k; ++i) s -= conj(A(i, k)) * x[i];
        x[k] = s / conj(A(k, k));
    }
    for (int k = n - 1; k >= 0; --k) {
        const int imax = k + kl < n - 1 ? k + kl : n - 1;
        cplx s = x[k];
        for (int i = k + 1; i <= imax; ++i) s -= conj(A(i, k)) * x[i];
        x[k] = s;
        if (piv[k] != k) {
            const cplx t = x[k];
            x[k] = x[piv[k]];
            x[piv[k]] = t;
        }
    }
#undef A
}

/* ---------------- FD preconditioner: src/fdsolver.cpp ---------------------- */
typedef struct {
    int d, p, nt;
    int dims[4];
    size_t Ns, N;
    double* U[3];    /* column-major n_l x n_l */
    double* lambda;  /* composite, length Ns */
    cplx* ab;        /* Ns blocks, (3p+1) x nt each */
    int* piv;        /* Ns x nt */
} ko_fd;

/* W + W^H (fdsolver.cpp:95-103) and H(lam) (fdsolver.cpp:105-120); kind 1:
 * galerkin_fast_solver's H(lam) = Wt + nu*lam*Mt (fdsolver.cpp:177-191) */
static void build_block(const double* Lt, const double* Mt, const cplx* Wt, int nt, int p,
                        double nu, double lam, cplx* H, int kind) {
    const int ld = 2 * p + 1;
    memset(H, 0, (size_t)ld * nt * sizeof(cplx));
    for (int i = 0; i < nt; ++i)
        for (int j = (i - p > 0 ? i - p : 0); j <= (i + p < nt - 1 ? i + p : nt - 1); ++j) {
            const size_t ij = (size_t)(p + i - j) + (size_t)j * ld;
            if (kind == 1) {
                const cplx mt = Mt[ij];
                H[ij] = band_get(Wt, nt, p, i, j) + nu * lam * mt;
                continue;
            }
            const cplx wsym = band_get(Wt, nt, p, i, j) + conj(band_get(Wt, nt, p, j, i));
            const cplx lt = Lt[ij], mt = Mt[ij];
            H[ij] = lt + nu * nu * lam * lam * mt + nu * lam * wsym;
        }
}

static ko_fd* fd_create(int kind, int d, const int* dims, double nu, int p, const double* const* U,
                        const double* const* lam_axes, const double* Lt, const double* Mt,
                        const cplx* Wt, int* status);

/* FDPreconditioner(prob, u): spatial_eigenbasis (fdsolver.cpp:23-44) + FastDiagSolver ctor (:46-51) */
ko_fd* ko_fd_create(int d, const int* dims, double nu, int p, const double* const* U,
                    const double* const* lam_axes, const double* Lt, const double* Mt,
                    const cplx* Wt, int* status) {
    return fd_create(0, d, dims, nu, p, U, lam_axes, Lt, Mt, Wt, status);
}

/* galerkin_fast_solver(prob, u) (fdsolver.cpp:177-191) */
ko_fd* ko_fd_create_galerkin(int d, const int* dims, double nu, int p, const double* const* U,
                             const double* const* lam_axes, const double* Mt, const cplx* Wt,
                             int* status) {
    return fd_create(1, d, dims, nu, p, U, lam_axes, NULL, Mt, Wt, status);
}

static ko_fd* fd_create(int kind, int d, const int* dims, double nu, int p, const double* const* U,
                        const double* const* lam_axes, const double* Lt, const double* Mt,
                        const cplx* Wt, int* status) {
    ko_fd* f = (ko_fd*)calloc(1, sizeof(ko_fd));
    f->d = d;
    f->p = p;
    f->nt = dims[0];
    f->Ns = 1;
    for (int a = 0; a <= d; ++a) f->dims[a] = dims[a];
    for (int l = 1; l <= d; ++l) f->Ns *= (size_t)dims[l];
    f->N = f->Ns * (size_t)f->nt;
    for (int l = 0; l < d; ++l) {
        const size_t n = (size_t)dims[l + 1];
        f->U[l] = (double*)malloc(n * n * sizeof(double));
        memcpy(f->U[l], U[l], n * n * sizeof(double));
    }
    /* composite eigenvalues, axis 1 fastest (fdsolver.cpp:30-42) */
    f->lambda = (double*)malloc(f->Ns * sizeof(double));
    int idx[3] = {0, 0, 0};
    for (size_t i = 0; i < f->Ns; ++i) {
        double s = 0;
        for (int l = 0; l < d; ++l) s += lam_axes[l][idx[l]];
        f->lambda[i] = s;
        for (int l = 0; l < d; ++l) {
            if (++idx[l] < dims[l + 1]) break;
            idx[l] = 0;
        }
    }
    const int ldab = 3 * p + 1, nt = f->nt;
    f->ab = (cplx*)malloc(f->Ns * (size_t)ldab * nt * sizeof(cplx));
    f->piv = (int*)malloc(f->Ns * (size_t)nt * sizeof(int));
    cplx* H = (cplx*)malloc((size_t)(2 * p + 1) * nt * sizeof(cplx));
    *status = 0;
    for (size_t i = 0; i < f->Ns; ++i) {
        build_block(Lt, Mt, Wt, nt, p, nu, f->lambda[i], H, kind);
        if (ko_factor_banded(H, nt, p, f->ab + i * (size_t)ldab * nt, f->piv + i * (size_t)nt)) {
            *status = 2;
            break;
        }
    }
    free(H);
    return f;
}

void ko_fd_destroy(ko_fd* f) {
    if (!f) return;
    for (int l = 0; l < f->d; ++l) free(f->U[l]);
    free(f->lambda);
    free(f->ab);
    free(f->piv);
    free(f);
}

size_t ko_fd_vec_size(const ko_fd* f) { return f->N; }
const double* ko_fd_lambda(const ko_fd* f) { return f->lambda; }
const cplx* ko_fd_block_ab(const ko_fd* f, size_t i) { return f->ab + i * (size_t)(3 * f->p + 1) * f->nt; }
const int* ko_fd_block_piv(const ko_fd* f, size_t i) { return f->piv + i * (size_t)f->nt; }

/* FastDiagSolver::solve (fdsolver.cpp:53-63) / solve_adjoint (:65-75) */
static void fd_solve(const ko_fd* f, const cplx* r, cplx* y, int adjoint) {
    const int ndim = f->d + 1;
    cplx* X = (cplx*)malloc(f->N * sizeof(cplx));
    cplx* T = (cplx*)malloc(f->N * sizeof(cplx));
    memcpy(X, r, f->N * sizeof(cplx));
    /* to_eigen: axes 1..d with U^T (fdsolver.cpp:7-14) */
    for (int l = 0; l < f->d; ++l) {
        ko_mode_product_dense(f->U[l], 1, X, T, f->dims, ndim, l + 1);
        cplx* t = X; X = T; T = t;
    }
    const size_t nt = (size_t)f->nt, ldab = (size_t)(3 * f->p + 1);
    for (size_t i = 0; i < f->Ns; ++i) {
        if (adjoint) ko_solve_banded_adjoint(f->ab + i * ldab * nt, f->piv + i * nt, f->nt, f->p, X + i * nt);
        else ko_solve_banded(f->ab + i * ldab * nt, f->piv + i * nt, f->nt, f->p, X + i * nt);
    }
    /* from_eigen: axes 1..d with U (fdsolver.cpp:16-21) */
    for (int l = 0; l < f->d; ++l) {
        ko_mode_product_dense(f->U[l], 0, X, T, f->dims, ndim, l + 1);
        cplx* t = X; X = T; T = t;
    }
    memcpy(y, X, f->N * sizeof(cplx));
    free(X);
    free(T);
}
void ko_fd_apply(const ko_fd* f, const cplx* r, cplx* z) { fd_solve(f, r, z, 0); }
void ko_fd_apply_adjoint(const ko_fd* f, const cplx* r, cplx* z) { fd_solve(f, r, z, 1); }

/* ---------------- KroneckerOperator::apply: src/tensorops.cpp:236-254 ---------- */
/* terms: coeffs[t]; factors[t*ndim + k] (NULL = identity) with bandwidth bws[t*ndim + k] */
void ko_kron_apply(int ndim, const int* dims, int nterms, const cplx* coeffs,
                   const cplx* const* factors, const int* bws, const cplx* x, cplx* y) {
    size_t n = 1;
    for (int k = 0; k < ndim; ++k) n *= (size_t)dims[k];
    memset(y, 0, n * sizeof(cplx));
    cplx* in = (cplx*)malloc(n * sizeof(cplx));
    cplx* work = (cplx*)malloc(n * sizeof(cplx));
    for (int t = 0; t < nterms; ++t) {
        const cplx* src = x;
        for (int k = 0; k < ndim; ++k) {
            const cplx* F = factors[(size_t)t * ndim + k];
            if (!F) continue;
            memcpy(in, src, n * sizeof(cplx)); /* copy of the source (:245-247) */
            ko_mode_product_band(F, bws[(size_t)t * ndim + k], in, work, dims, ndim, k);
            src = work;
        }
        ko_axpy(coeffs[t], src, y, n); /* (:252) */
    }
    free(in);
    free(work);
}

/* ---------------- pcg: src/krylov.cpp:24-114 ------------------------------- */
typedef void (*ko_apply_fn)(void* ctx, const cplx* x, cplx* y);

/* returns 0 ok, 1 bad options. flags: bit0 converged, bit1 breakdown */
int ko_pcg(ko_apply_fn apply_a, void* actx, ko_apply_fn apply_p, void* pctx, const cplx* b,
           size_t n, double tol, int maxit, int strict, cplx* x_out, int* iterations,
           double* hist, int hist_cap, int* hist_len, int* flags) {
    if (!(tol > 0) || maxit < 0) return 1;
    *iterations = 0;
    *hist_len = 0;
    *flags = 0;
    memset(x_out, 0, n * sizeof(cplx));
    const double bnorm = sqrt(ko_norm2sq(b, n));
    if (bnorm == 0.0) {
        *flags = 1;
        return 0;
    }
    cplx* r = (cplx*)malloc(n * sizeof(cplx));
    cplx* z = (cplx*)malloc(n * sizeof(cplx));
    cplx* p = (cplx*)malloc(n * sizeof(cplx));
    cplx* q = (cplx*)malloc(n * sizeof(cplx));
    cplx* scratch = (cplx*)malloc(n * sizeof(cplx));
    cplx* x = x_out;
#define PRECOND(rr, zz) do { if (apply_p) apply_p(pctx, rr, zz); else memcpy(zz, rr, n * sizeof(cplx)); } while (0)
    memcpy(r, b, n * sizeof(cplx));
    PRECOND(r, z);
    memcpy(p, z, n * sizeof(cplx));
    double re, im;
    ko_dotc(r, z, n, &re, &im);
    double rho = re;
    int restarts = 0, hl = 0;
    for (int k = 0; k < maxit; ++k) {
        apply_a(actx, p, q);
        ko_dotc(p, q, n, &re, &im);
        const double curvature = re;
        if (curvature <= 0.0) {
            *flags |= 2;
            break;
        }
        const double alpha = rho / curvature;
        ko_axpy_real(alpha, p, x, n);
        ko_axpy_real(-alpha, q, r, n);
        ++*iterations;
        double relres = sqrt(ko_norm2sq(r, n)) / bnorm;
        if (strict) {
            apply_a(actx, x, scratch);
            ko_axpy_real(-1.0, b, scratch, n);
            relres = sqrt(ko_norm2sq(scratch, n)) / bnorm;
        }
        if (hl < hist_cap) hist[hl] = relres;
        ++hl;
        if (relres <= tol) {
            if (!strict) {
                apply_a(actx, x, scratch);
                ko_axpy_real(-1.0, b, scratch, n);
                const double tr = sqrt(ko_norm2sq(scratch, n)) / bnorm;
                if (hl - 1 < hist_cap) hist[hl - 1] = tr;
                if (tr > tol) {
                    if (++restarts > 2) break;
                    for (size_t i = 0; i < n; ++i) r[i] = -scratch[i];
                    PRECOND(r, z);
                    memcpy(p, z, n * sizeof(cplx));
                    ko_dotc(r, z, n, &re, &im);
                    rho = re;
                    continue;
                }
            }
            *flags |= 1;
            break;
        }
        PRECOND(r, z);
        ko_dotc(r, z, n, &re, &im);
        const double rho_new = re;
        const double beta = rho_new / rho;
        rho = rho_new;
        for (size_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
#undef PRECOND
    *hist_len = hl < hist_cap ? hl : hist_cap;
    free(r); free(z); free(p); free(q); free(scratch);
    return 0;
}

/* convenience callbacks for ctypes: operator handles as contexts */
typedef struct {
    int ndim;
    const int* dims;
    int nterms;
    const cplx* coeffs;
    const cplx* const* factors;
    const int* bws;
} ko_kron_ctx;

void ko_kron_cb(void* ctx, const cplx* x, cplx* y) {
    const ko_kron_ctx* k = (const ko_kron_ctx*)ctx;
    ko_kron_apply(k->ndim, k->dims, k->nterms, k->coeffs, k->factors, k->bws, x, y);
}
void ko_fd_cb(void* ctx, const cplx* x, cplx* y) { ko_fd_apply((const ko_fd*)ctx, x, y); }

/* seeded inputs shared by oracle and GPU: std::mt19937_64(seed), u = (g()>>11) * 2^-53,
 * re = 2u-1 then im = 2u-1 per entry in vec order. */
void ko_random_vec(uint64_t seed, cplx* v, size_t n) {
    /* MT19937-64 (Matsumoto & Nishimura), the generator behind std::mt19937_64 */
    uint64_t mt[312];
    int mti;
    mt[0] = seed;
    for (mti = 1; mti < 312; ++mti)
        mt[mti] = 6364136223846793005ULL * (mt[mti - 1] ^ (mt[mti - 1] >> 62)) + (uint64_t)mti;
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    for (size_t i = 0; i < 2 * n; ++i) {
        if (mti >= 312) {
            int k;
            uint64_t xx;
            for (k = 0; k < 312 - 156; ++k) {
                xx = (mt[k] & UM) | (mt[k + 1] & LM);
                mt[k] = mt[k + 156] ^ (xx >> 1) ^ mag01[(int)(xx & 1ULL)];
            }
            for (; k < 311; ++k) {
                xx = (mt[k] & UM) | (mt[k + 1] & LM);
                mt[k] = mt[k + (156 - 312)] ^ (xx >> 1) ^ mag01[(int)(xx & 1ULL)];
            }
            xx = (mt[311] & UM) | (mt[0] & LM);
            mt[311] = mt[155] ^ (xx >> 1) ^ mag01[(int)(xx & 1ULL)];
            mti = 0;
        }
        uint64_t y = mt[mti++];
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        y ^= (y >> 43);
        const double u = (double)(y >> 11) * (1.0 / 9007199254740992.0);
        double* d = (double*)v;
        d[i] = 2.0 * u - 1.0;
    }
}
