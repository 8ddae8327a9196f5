// kronschro_gpu.hpp -- header-only C++ wrappers over the C-ABI (ks.h) with the
// reference's signatures, so a reference build can swap its hot-path objects
// for the B200 ones without touching the caller:
//
//   kronschro::FDPreconditioner::apply(const cplx* r, cplx* z) const   fdsolver.hpp:61
//   kronschro::KroneckerOperator::apply(const cplx* x, cplx* y) const  tensorops.hpp:76
//   kronschro::pcg(apply_a, apply_p, b, opts)                          krylov.hpp:37-38
//
// The wrappers take the reference's setup products as plain arrays (U_l,
// lambda_l column-major; bands in BandedMatrix layout), so this header does
// not depend on Eigen or on the reference headers. Error codes are rethrown
// as the std exceptions the reference throws.
#pragma once

#include <complex>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ks.h"

namespace kronschro_gpu {

using cplx = std::complex<double>;
static_assert(sizeof(cplx) == sizeof(ks_c64), "std::complex<double> must be interleaved (re, im)");

inline void check(int rc) {
    if (rc == KS_OK) return;
    const std::string msg = ks_last_error();
    switch (rc) {
    case KS_EINVAL: throw std::invalid_argument(msg);
    case KS_ELENGTH: throw std::length_error(msg);
    case KS_ENOMEM: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
    }
}

// FDPreconditioner (fdsolver.hpp:56-74). Construct from the reference's
// SpatialEigenbasis (U_l, lambda_l) and UnivariateSet time bands.
class FDPreconditioner {
  public:
    FDPreconditioner(const std::vector<int>& dims, double nu, int p_t,
                     const std::vector<const double*>& U, const std::vector<const double*>& lambda,
                     const double* Lt, const double* Mt, const cplx* Wt, int device = 0) {
        ks_fd* h = nullptr;
        check(ks_fd_create(static_cast<int>(dims.size()) - 1, dims.data(), nu, p_t, U.data(),
                           lambda.data(), Lt, Mt, reinterpret_cast<const ks_c64*>(Wt), device, &h));
        h_.reset(h);
    }
    // raw, unchecked-length apply on host pointers (the reference's signature)
    void apply(const cplx* r, cplx* z) const {
        check(ks_fd_apply(h_.get(), reinterpret_cast<const ks_c64*>(r), reinterpret_cast<ks_c64*>(z),
                          KS_MEM_HOST, nullptr));
    }
    // device-pointer apply (HBM-resident vectors)
    void apply_device(const cplx* r, cplx* z, void* stream = nullptr) const {
        check(ks_fd_apply(h_.get(), reinterpret_cast<const ks_c64*>(r), reinterpret_cast<ks_c64*>(z),
                          KS_MEM_DEVICE, stream));
    }
    std::vector<cplx> apply(const std::vector<cplx>& r) const {
        if (r.size() != vec_size()) throw std::invalid_argument("FastDiagSolver: vector length mismatch");
        std::vector<cplx> z(r.size());
        apply(r.data(), z.data());
        return z;
    }
    std::size_t vec_size() const { return ks_fd_vec_size(h_.get()); }
    ks_fd* handle() const { return h_.get(); }

  private:
    struct Del {
        void operator()(ks_fd* p) const { ks_fd_destroy(p); }
    };
    std::unique_ptr<ks_fd, Del> h_;
};

// KroneckerOperator (tensorops.hpp:57-87): terms are gathered with add_term
// and the device plan is built on first apply.
class KroneckerOperator {
  public:
    struct Factor {
        const cplx* data = nullptr; // BandedMatrix<cplx> storage, nullptr = identity
        int bw = 0;
    };
    explicit KroneckerOperator(std::vector<int> dims, int device = 0)
        : dims_(std::move(dims)), device_(device) {}

    void add_term(cplx coeff, std::vector<Factor> factors) {
        if (factors.size() != dims_.size()) throw std::invalid_argument("KroneckerOperator: wrong factor count");
        terms_.push_back({coeff, std::move(factors)});
        h_.reset();
    }
    void apply(const cplx* x, cplx* y) const {
        build();
        check(ks_kron_apply(h_.get(), reinterpret_cast<const ks_c64*>(x), reinterpret_cast<ks_c64*>(y),
                            KS_MEM_HOST, nullptr));
    }
    void apply_device(const cplx* x, cplx* y, void* stream = nullptr) const {
        build();
        check(ks_kron_apply(h_.get(), reinterpret_cast<const ks_c64*>(x), reinterpret_cast<ks_c64*>(y),
                            KS_MEM_DEVICE, stream));
    }
    std::size_t vec_size() const {
        std::size_t n = 1;
        for (int d : dims_) n *= static_cast<std::size_t>(d);
        return n;
    }
    ks_kron* handle() const {
        build();
        return h_.get();
    }

  private:
    struct Term {
        cplx coeff;
        std::vector<Factor> f;
    };
    void build() const {
        if (h_) return;
        std::vector<std::vector<const ks_c64*>> ptrs(terms_.size());
        std::vector<std::vector<int>> bws(terms_.size());
        std::vector<ks_term> kt(terms_.size());
        for (std::size_t t = 0; t < terms_.size(); ++t) {
            for (const Factor& f : terms_[t].f) {
                ptrs[t].push_back(reinterpret_cast<const ks_c64*>(f.data));
                bws[t].push_back(f.bw);
            }
            kt[t].coeff = {terms_[t].coeff.real(), terms_[t].coeff.imag()};
            kt[t].factors = ptrs[t].data();
            kt[t].bw = bws[t].data();
        }
        ks_kron* h = nullptr;
        check(ks_kron_create(static_cast<int>(dims_.size()), dims_.data(), static_cast<int>(kt.size()),
                             kt.data(), device_, &h));
        h_.reset(h);
    }
    struct Del {
        void operator()(ks_kron* p) const { ks_kron_destroy(p); }
    };
    std::vector<int> dims_;
    int device_;
    std::vector<Term> terms_;
    mutable std::unique_ptr<ks_kron, Del> h_;
};

struct PcgOptions {
    double tol = 1e-8;
    int maxit = 200;
    bool strict_residual = false;
};

struct SolveReport {
    std::vector<cplx> x;
    int iterations = 0;
    std::vector<double> res_history;
    bool converged = false;
    bool breakdown = false;
    double setup_seconds = 0, matvec_seconds = 0, precond_seconds = 0, solve_seconds = 0;
};

// pcg with the device-resident loop (krylov.cpp:24-114); P may be null.
inline SolveReport pcg(const KroneckerOperator& A, const FDPreconditioner* P,
                       const std::vector<cplx>& b, const PcgOptions& opts = {}) {
    SolveReport rep;
    rep.x.assign(b.size(), cplx(0));
    std::vector<double> hist(opts.maxit > 0 ? opts.maxit : 1);
    ks_pcg_opts o{opts.tol, opts.maxit, opts.strict_residual ? 1 : 0};
    ks_pcg_report r{};
    check(ks_pcg(A.handle(), P ? P->handle() : nullptr, reinterpret_cast<const ks_c64*>(b.data()),
                 reinterpret_cast<ks_c64*>(rep.x.data()), KS_MEM_HOST, &o, hist.data(),
                 static_cast<int>(hist.size()), &r));
    rep.iterations = r.iterations;
    rep.converged = r.converged != 0;
    rep.breakdown = r.breakdown != 0;
    rep.res_history.assign(hist.begin(), hist.begin() + r.hist_len);
    rep.matvec_seconds = r.matvec_seconds;
    rep.precond_seconds = r.precond_seconds;
    rep.solve_seconds = r.solve_seconds;
    return rep;
}

} // namespace kronschro_gpu
