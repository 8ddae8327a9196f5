// ref_driver.cpp -- ORACLE TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the reference kronschro library, built from
// the reference's own unmodified sources (/root/reference/proj/src) by
// oracle/build_ref.sh into oracle/_ref/libkronschro_ref.so. Used by tests/,
// tests/golden/make_golden.py and bench.py's cpu_baseline / --impl reference
// legs. The product never links it.
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "kronschro/assembly.hpp"
#include "kronschro/experiments.hpp"
#include "kronschro/fdsolver.hpp"
#include "kronschro/kernels.hpp"
#include "kronschro/krylov.hpp"
#include "kronschro/problems.hpp"
#include "kronschro/tensorops.hpp"

using namespace kronschro;

namespace {
thread_local std::string g_err;

struct RefProblem {
    SpaceTimeProblem prob;
    UnivariateSet u;
    std::unique_ptr<FDPreconditioner> P;
    std::unique_ptr<KroneckerOperator> A;
    std::unique_ptr<FastDiagSolver> Gfd;       // galerkin_fast_solver (lazy)
    std::unique_ptr<KroneckerOperator> Gop;    // assemble_galerkin_operator (lazy)
    SpatialEigenbasis basis;
    explicit RefProblem(SpaceTimeProblem pr) : prob(std::move(pr)) {}
};

template <typename T> void band_out(const BandedMatrix<T>& b, T* out) {
    const int n = b.rows(), bw = b.bandwidth();
    std::memset(static_cast<void*>(out), 0, sizeof(T) * (size_t)(2 * bw + 1) * n);
    for (int j = 0; j < n; ++j)
        for (int i = std::max(0, j - bw); i <= std::min(n - 1, j + bw); ++i)
            out[(size_t)(bw + i - j) + (size_t)j * (2 * bw + 1)] = b(i, j);
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// kernels::force_backend("scalar"|"avx2"|"auto") (kernels.cpp:57-70)
int ref_force_backend(const char* name) {
    try {
        kernels::force_backend(name);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
const char* ref_active_backend() { return kernels::active().name; }

// SpaceTimeProblem::uniform + build_univariate + FDPreconditioner + assemble_system_operator
void* ref_problem_create(int d, int p, int n_el, int n_el_t, double T, double nu, int trial,
                         int with_fd) {
    try {
        auto r = new RefProblem(SpaceTimeProblem::uniform(
            d, p, n_el, n_el_t, T, nu,
            trial ? SpaceTimeProblem::TrialSpace::FinalCondition
                  : SpaceTimeProblem::TrialSpace::InitialCondition));
        r->u = build_univariate(r->prob);
        r->basis = spatial_eigenbasis(r->prob, r->u);
        if (with_fd) r->P = std::make_unique<FDPreconditioner>(r->prob, r->u);
        r->A = std::make_unique<KroneckerOperator>(assemble_system_operator(r->prob));
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_problem_destroy(void* h) { delete static_cast<RefProblem*>(h); }

void ref_dims(void* h, int* dims) {
    auto* r = static_cast<RefProblem*>(h);
    const auto v = r->prob.reduced_dims();
    for (size_t i = 0; i < v.size(); ++i) dims[i] = v[i];
}

void ref_time_bands(void* h, double* Lt, double* Mt, std::complex<double>* Wt) {
    auto* r = static_cast<RefProblem*>(h);
    band_out(r->u.Lt, Lt);
    band_out(r->u.Mt, Mt);
    band_out(r->u.Wt, Wt);
}

void ref_space_bands(void* h, int l, double* M, double* L, double* G, double* V) {
    auto* r = static_cast<RefProblem*>(h);
    band_out(r->u.M[l], M);
    band_out(r->u.L[l], L);
    band_out(r->u.G[l], G);
    band_out(r->u.V[l], V);
}

// SpatialEigenbasis axis l: U column-major, lambda ascending
void ref_eig(void* h, int l, double* U, double* lam) {
    auto* r = static_cast<RefProblem*>(h);
    const auto& e = r->basis.axes[l];
    for (Eigen::Index j = 0; j < e.U.cols(); ++j)
        for (Eigen::Index i = 0; i < e.U.rows(); ++i) U[i + j * e.U.rows()] = e.U(i, j);
    for (Eigen::Index i = 0; i < e.lambda.size(); ++i) lam[i] = e.lambda(i);
}

void ref_composite_lambda(void* h, double* out) {
    auto* r = static_cast<RefProblem*>(h);
    std::copy(r->basis.lambda.begin(), r->basis.lambda.end(), out);
}

int ref_fd_apply(void* h, const std::complex<double>* x, std::complex<double>* y) {
    auto* r = static_cast<RefProblem*>(h);
    if (!r->P) return 1;
    r->P->apply(x, y);
    return 0;
}

void ref_kron_apply(void* h, const std::complex<double>* x, std::complex<double>* y) {
    static_cast<RefProblem*>(h)->A->apply(x, y);
}

// factor_banded on H(lambda_i) built as make_fd_solver does (fdsolver.cpp:105-120)
int ref_fd_block(void* h, long i, std::complex<double>* ab, int* piv) {
    auto* r = static_cast<RefProblem*>(h);
    try {
        const double nu = r->prob.nu, lam = r->basis.lambda[i];
        const BandedMatrix<cplx> Lt = to_complex(r->u.Lt), Mt = to_complex(r->u.Mt);
        BandedMatrix<cplx> Wsym = r->u.Wt;
        const BandedMatrix<cplx> Wh = r->u.Wt.conjugate_transpose();
        for (int a = 0; a < Wsym.rows(); ++a)
            for (int b = std::max(0, a - Wsym.bandwidth());
                 b <= std::min(Wsym.cols() - 1, a + Wsym.bandwidth()); ++b)
                Wsym.ref(a, b) += Wh(a, b);
        BandedMatrix<cplx> H(Lt.rows(), Lt.bandwidth());
        for (int a = 0; a < H.rows(); ++a)
            for (int b = std::max(0, a - H.bandwidth()); b <= std::min(H.cols() - 1, a + H.bandwidth()); ++b)
                H.ref(a, b) = Lt(a, b) + nu * nu * lam * lam * Mt(a, b) + nu * lam * Wsym(a, b);
        const BandedFactorization F = factor_banded(H);
        std::copy(F.ab.begin(), F.ab.end(), ab);
        std::copy(F.piv.begin(), F.piv.end(), piv);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

// pcg (krylov.cpp:24-114) with A and (optionally) P
int ref_pcg(void* h, const std::complex<double>* b, double tol, int maxit, int strict, int use_p,
            std::complex<double>* x, int* iters, double* hist, int cap, int* hlen, int* flags,
            double* seconds) {
    auto* r = static_cast<RefProblem*>(h);
    try {
        const size_t n = r->A->vec_size();
        std::vector<cplx> bv(b, b + n);
        ApplyFn aa = [r](const cplx* xi, cplx* yo) { r->A->apply(xi, yo); };
        ApplyFn pp;
        if (use_p && r->P) pp = [r](const cplx* xi, cplx* yo) { r->P->apply(xi, yo); };
        PcgOptions o;
        o.tol = tol;
        o.maxit = maxit;
        o.strict_residual = strict != 0;
        const SolveReport rep = pcg(aa, pp, bv, o);
        std::copy(rep.x.begin(), rep.x.end(), x);
        *iters = rep.iterations;
        *hlen = 0;
        for (size_t k = 0; k < rep.res_history.size() && (int)k < cap; ++k) hist[(*hlen)++] = rep.res_history[k];
        *flags = (rep.converged ? 1 : 0) | (rep.breakdown ? 2 : 0);
        if (seconds) *seconds = rep.solve_seconds;
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    }
}

// dense oracles (size-capped, tensorops.cpp:277-301, fdsolver.cpp:135-175); column-major
int ref_kron_to_dense(void* h, std::complex<double>* out) {
    auto* r = static_cast<RefProblem*>(h);
    try {
        const Eigen::MatrixXcd D = r->A->to_dense();
        std::copy(D.data(), D.data() + D.size(), out);
        return 0;
    } catch (const std::length_error& e) {
        g_err = e.what();
        return 6;
    }
}
int ref_fd_to_dense(void* h, std::complex<double>* out) {
    auto* r = static_cast<RefProblem*>(h);
    try {
        const Eigen::MatrixXcd D = r->P->to_dense(r->prob);
        std::copy(D.data(), D.data() + D.size(), out);
        return 0;
    } catch (const std::length_error& e) {
        g_err = e.what();
        return 6;
    }
}

// galerkin_fast_solver(prob, u) solve / solve_adjoint (fdsolver.cpp:53-75,177-191)
int ref_galerkin_apply(void* h, const std::complex<double>* x, std::complex<double>* y, int adjoint) {
    auto* r = static_cast<RefProblem*>(h);
    try {
        if (!r->Gfd) r->Gfd = std::make_unique<FastDiagSolver>(galerkin_fast_solver(r->prob, r->u));
        if (adjoint) r->Gfd->solve_adjoint(x, y);
        else r->Gfd->solve(x, y);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

// assemble_galerkin_operator(prob).apply (assembly.cpp:273-286)
int ref_galerkin_kron_apply(void* h, const std::complex<double>* x, std::complex<double>* y) {
    auto* r = static_cast<RefProblem*>(h);
    try {
        if (!r->Gop) r->Gop = std::make_unique<KroneckerOperator>(assemble_galerkin_operator(r->prob));
        r->Gop->apply(x, y);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

// c2/c4 manufactured solution u = sin(pi x) sin(pi y) e^{-i 2 pi^2 t}, f = S u = (1+nu) d pi^2 u (4 pi^2 u at d=2, nu=1)
// (SURVEY G2), lifted with lift_nonhomogeneous (assembly.cpp:514-570)
int ref_sinsin_rhs(void* h, std::complex<double>* rhs, std::complex<double>* boundary) {
    auto* r = static_cast<RefProblem*>(h);
    const double pi = 3.14159265358979323846;
    SpaceTimeFn u = [pi](double t, std::span<const double> x) {
        double s = 1.0;
        for (double xi : x) s *= std::sin(pi * xi);
        return s * std::exp(cplx(0, -(double)x.size() * pi * pi * t));
    };
    const double nu = r->prob.nu;
    SpaceTimeFn f = [pi, u, nu](double t, std::span<const double> x) { // S u = i u_t - nu lap u
        return (1.0 + nu) * (double)x.size() * pi * pi * u(t, x);
    };
    const Lifting L = lift_nonhomogeneous(r->prob, u, f);
    std::copy(L.corrected_rhs.begin(), L.corrected_rhs.end(), rhs);
    if (boundary) std::copy(L.boundary_coeffs.begin(), L.boundary_coeffs.end(), boundary);
    return 0;
}

// manufactured solution by name: the reference's named problems (problems.cpp)
// or "sinsin" (c2/c4: u = prod sin(pi x_l) e^{-i d pi^2 t}, f = S u = (1+nu) d pi^2 u)
static ManufacturedSolution solution_by_name(const RefProblem* r, const std::string& name) {
    if (name != "sinsin") return find_problem(name);
    const double pi = 3.14159265358979323846;
    ManufacturedSolution s;
    s.name = "sinsin";
    s.d = r->prob.d;
    s.T = r->prob.T;
    s.nu = r->prob.nu;
    s.homogeneous = false;
    s.u = [pi](double t, std::span<const double> x) {
        double v = 1.0;
        for (double xi : x) v *= std::sin(pi * xi);
        return v * std::exp(cplx(0, -(double)x.size() * pi * pi * t));
    };
    auto u = s.u;
    const double nu = s.nu;
    s.f = [pi, u, nu](double t, std::span<const double> x) { // S u = i u_t - nu lap u
        return (1.0 + nu) * (double)x.size() * pi * pi * u(t, x);
    };
    return s;
}

// lift_nonhomogeneous (assembly.cpp:514-570) for a named solution: corrected rhs + boundary coefficients
int ref_lift_named(void* h, const char* name, std::complex<double>* rhs, std::complex<double>* boundary) {
    auto* r = static_cast<RefProblem*>(h);
    try {
        const ManufacturedSolution s = solution_by_name(r, name);
        const Lifting L = lift_nonhomogeneous(r->prob, s.u, s.f);
        std::copy(L.corrected_rhs.begin(), L.corrected_rhs.end(), rhs);
        std::copy(L.boundary_coeffs.begin(), L.boundary_coeffs.end(), boundary);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// assemble_rhs (assembly.cpp:390-404) of a named solution's f
int ref_assemble_rhs_named(void* h, const char* name, std::complex<double>* rhs) {
    auto* r = static_cast<RefProblem*>(h);
    try {
        const ManufacturedSolution s = solution_by_name(r, name);
        const std::vector<cplx> b = assemble_rhs(r->prob, s.f);
        std::copy(b.begin(), b.end(), rhs);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// assemble_ultraweak (assembly.cpp:572-640) for a named solution: f and u0 = u(0, .)
// (final-condition trial space; the reference throws otherwise)
int ref_ultraweak_named(void* h, const char* name, std::complex<double>* rhs) {
    auto* r = static_cast<RefProblem*>(h);
    try {
        const ManufacturedSolution s = solution_by_name(r, name);
        auto u = s.u;
        const SpaceFn u0 = [u](std::span<const double> x) { return u(0.0, x); };
        const auto [A, b] = assemble_ultraweak(r->prob, s.f, u0);
        std::copy(b.begin(), b.end(), rhs);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// error_norms (experiments.cpp:73-153) of full coefficients against a named solution
int ref_error_norms_named(void* h, const char* name, const std::complex<double>* full, double* l2, double* energy) {
    auto* r = static_cast<RefProblem*>(h);
    try {
        const ManufacturedSolution s = solution_by_name(r, name);
        const size_t n = CoeffTensor::total(r->prob.full_dims());
        const std::vector<cplx> c(full, full + n);
        const auto e = error_norms(r->prob, c, s);
        *l2 = e.first;
        *energy = e.second;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// extend_with_boundary (assembly.cpp:468-490)
int ref_extend(void* h, const std::complex<double>* reduced, const std::complex<double>* boundary,
               std::complex<double>* full) {
    auto* r = static_cast<RefProblem*>(h);
    const size_t nr = CoeffTensor::total(r->prob.reduced_dims()), nf = CoeffTensor::total(r->prob.full_dims());
    const std::vector<cplx> red(reduced, reduced + nr), bnd(boundary, boundary + nf);
    const std::vector<cplx> f = extend_with_boundary(r->prob, red, bnd);
    std::copy(f.begin(), f.end(), full);
    return 0;
}

// infsup_constant (experiments.cpp:185-232): method 0 = Galerkin, 1 = least squares
double ref_infsup(int method, int p, int n_el, double T, double nu) {
    try {
        return infsup_constant(method == 0 ? InfSupMethod::Galerkin : InfSupMethod::LeastSquares, p, n_el, T, nu);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

// RHS of a named manufactured problem (problems.cpp:find_problem) exactly as
// solve_problem builds it (experiments.cpp:34-42): assemble_rhs if
// homogeneous, else lift_nonhomogeneous.
int ref_named_rhs(void* h, const char* name, std::complex<double>* rhs) {
    auto* r = static_cast<RefProblem*>(h);
    try {
        const ManufacturedSolution s = find_problem(name);
        std::vector<cplx> b;
        if (s.homogeneous) b = assemble_rhs(r->prob, s.f);
        else b = lift_nonhomogeneous(r->prob, s.u, s.f).corrected_rhs;
        std::copy(b.begin(), b.end(), rhs);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

} // extern "C"
