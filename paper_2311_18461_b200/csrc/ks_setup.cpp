// Host setup: the small 1-D work that stays on the CPU.
//
// This is the product-side restatement of the setup the reference runs on
// the host and hands to the hot path (north_star: "shared with the
// reference"); when the reference itself is the caller it passes its own
// products through ks_fd_create / ks_kron_create instead.
//
//   open uniform knot vectors          bspline.cpp:48-60 (KnotVector::open_uniform)
//   span search                        bspline.cpp:69-85
//   basis values + derivatives         bspline.cpp:88-157 (here: the derivative
//                                      recursion D N_{i,q} = q/(u_{i+q}-u_i) D N_{i,q-1}
//                                      - q/(u_{i+q+1}-u_{i+1}) D N_{i+1,q-1})
//   Gauss-Legendre rule                bspline.cpp:159-208
//   univariate Galerkin matrices       assembly.cpp:24-76 (kinds M, L, G, V, W)
//   restrictions                       assembly.cpp:44-52, :146-160
//   generalized SPD eigenproblem       eigensolve.cpp:8-29 (Cholesky reduction +
//                                      cyclic Jacobi; ascending; sign fix: first
//                                      largest-|.| entry of each column positive)
//   system operator term list          assembly.cpp:202-251 (restricted case)
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ks.h"
#include "ks_quad_host.hpp"

namespace ks_host {

using cplx = std::complex<double>;

struct Knots {
    int p = 1;
    std::vector<double> u;
    int dim() const { return (int)u.size() - p - 1; }
};

Knots open_uniform(int p, int n_el, double a, double b) {
    if (p < 1 || n_el < 1 || !(a < b)) throw std::invalid_argument("open_uniform: invalid arguments");
    Knots k;
    k.p = p;
    for (int i = 0; i <= p; ++i) k.u.push_back(a);
    for (int i = 1; i < n_el; ++i) k.u.push_back(a + (b - a) * i / n_el);
    for (int i = 0; i <= p; ++i) k.u.push_back(b);
    return k;
}

int span_of(const Knots& k, double x) {
    const int m = k.dim();
    if (x >= k.u[m]) return m - 1;
    int lo = k.p, hi = m;
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (x < k.u[mid]) hi = mid;
        else lo = mid;
    }
    return lo;
}

// values of all degree-q functions nonzero at x, q = 0..p; tab[q][j] = N_{span-q+j, q}
// then derivatives of the degree-p functions by the recursion on q.
struct Basis {
    int first = 0;
    std::vector<std::vector<double>> d; // d[order][a], a = 0..p
};

Basis basis_at(const Knots& k, double x, int nder) {
    const int p = k.p, sp = span_of(k, x);
    const auto& u = k.u;
    std::vector<std::vector<double>> tab(p + 1);
    tab[0] = {1.0};
    for (int q = 1; q <= p; ++q) {
        tab[q].assign(q + 1, 0.0);
        for (int j = 0; j <= q; ++j) {
            const int i = sp - q + j; // N_{i,q} = w1 N_{i,q-1} + w2 N_{i+1,q-1}
            double v = 0.0;
            // N_{i,q-1} is tab[q-1][j-1] (index i - (sp-q+1))
            if (j - 1 >= 0) {
                const double den = u[i + q] - u[i];
                if (den != 0.0) v += (x - u[i]) / den * tab[q - 1][j - 1];
            }
            if (j <= q - 1) {
                const double den = u[i + q + 1] - u[i + 1];
                if (den != 0.0) v += (u[i + q + 1] - x) / den * tab[q - 1][j];
            }
            tab[q][j] = v;
        }
    }
    // D^r N_{i,q}(x) for i in the support window
    std::function<double(int, int, int)> der = [&](int r, int q, int i) -> double {
        if (r == 0) {
            const int j = i - (sp - q);
            return (j >= 0 && j <= q) ? tab[q][j] : 0.0;
        }
        if (q == 0) return 0.0;
        double v = 0.0;
        const double d1 = u[i + q] - u[i], d2 = u[i + q + 1] - u[i + 1];
        if (d1 != 0.0) v += q / d1 * der(r - 1, q - 1, i);
        if (d2 != 0.0) v -= q / d2 * der(r - 1, q - 1, i + 1);
        return v;
    };
    Basis b;
    b.first = sp - p;
    b.d.assign(nder + 1, std::vector<double>(p + 1, 0.0));
    for (int r = 0; r <= nder; ++r)
        for (int a = 0; a <= p; ++a) b.d[r][a] = der(r, p, sp - p + a);
    return b;
}

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    const double pi = 3.14159265358979323846;
    for (int i = 0; i < (n + 1) / 2; ++i) {
        double z = std::cos(pi * (i + 0.75) / (n + 0.5)), dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = 0.0;
            for (int j = 1; j <= n; ++j) { // P_j from P_{j-1}, P_{j-2}
                const double p2 = p1;
                p1 = p0;
                p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j;
            }
            dp = n * (z * p0 - p1) / (z * z - 1.0);
            const double dz = p0 / dp;
            z -= dz;
            if (std::fabs(dz) < 1e-15) break;
        }
        x[i] = -z;
        x[n - 1 - i] = z;
        w[i] = w[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
    }
    if (n % 2 == 1) x[n / 2] = 0.0;
}

// banded square matrix, BandedMatrix layout: (i,j) at bw + i - j + j*(2bw+1)
template <typename T> struct Band {
    int n = 0, bw = 0;
    std::vector<T> a;
    Band() = default;
    Band(int n_, int bw_) : n(n_), bw(bw_), a((size_t)(2 * bw_ + 1) * n_, T(0)) {}
    bool in(int i, int j) const { return i >= 0 && j >= 0 && i < n && j < n && std::abs(i - j) <= bw; }
    T get(int i, int j) const { return in(i, j) ? a[bw + i - j + (size_t)j * (2 * bw + 1)] : T(0); }
    T& at(int i, int j) { return a[bw + i - j + (size_t)j * (2 * bw + 1)]; }
    Band restricted(int r0, int r1) const {
        Band r(r1 - r0, bw);
        for (int i = r0; i < r1; ++i)
            for (int j = std::max(r0, i - bw); j <= std::min(r1 - 1, i + bw); ++j)
                r.at(i - r0, j - r0) = get(i, j);
        return r;
    }
};

enum Kind { Mass, Stiff, Second, Bilap, TimeDer };
enum Restr { None, DropFirst, DropLast, DropBoth };

Band<cplx> univariate(Kind kind, const Knots& k, Restr rs) {
    int ro = 0, co = 0;
    cplx scale(1, 0);
    switch (kind) {
    case Mass: break;
    case Stiff: ro = co = 1; break;
    case Second: ro = 2; break;
    case Bilap: ro = co = 2; break;
    case TimeDer: co = 1; scale = cplx(0, 1); break;
    }
    const int p = k.p, m = k.dim();
    if (std::max(ro, co) >= 2 && p < 2)
        throw std::invalid_argument("univariate_matrix: second derivatives require a C^1 space");
    Band<cplx> A(m, p);
    std::vector<double> gx, gw;
    gauss_legendre(p + 1, gx, gw);
    // elements = nonempty knot spans
    for (size_t e = 0; e + 1 < k.u.size(); ++e) {
        const double z0 = k.u[e], z1 = k.u[e + 1];
        if (!(z1 > z0)) continue;
        const double mid = 0.5 * (z0 + z1), half = 0.5 * (z1 - z0);
        for (int q = 0; q <= p; ++q) {
            const double x = mid + half * gx[q], w = half * gw[q];
            const Basis b = basis_at(k, x, std::max(ro, co));
            for (int a = 0; a <= p; ++a)
                for (int c = 0; c <= p; ++c)
                    A.at(b.first + a, b.first + c) += scale * (w * b.d[ro][a] * b.d[co][c]);
        }
    }
    switch (rs) {
    case None: return A;
    case DropFirst: return A.restricted(1, A.n);
    case DropLast: return A.restricted(0, A.n - 1);
    case DropBoth: return A.restricted(1, A.n - 1);
    }
    return A;
}

Band<double> real_part(const Band<cplx>& c) {
    Band<double> r(c.n, c.bw);
    for (size_t i = 0; i < c.a.size(); ++i) r.a[i] = c.a[i].real();
    return r;
}

// L u = lambda M u, both SPD dense n x n (row-major input), U column-major output
void gen_sym_eig(const Band<double>& Lb, const Band<double>& Mb, std::vector<double>& U,
                 std::vector<double>& lam) {
    const int n = Lb.n;
    std::vector<double> L((size_t)n * n), M((size_t)n * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            L[(size_t)i * n + j] = Lb.get(i, j);
            M[(size_t)i * n + j] = Mb.get(i, j);
        }
    // Cholesky M = C C^T (C lower, row-major)
    std::vector<double> C((size_t)n * n, 0.0);
    for (int j = 0; j < n; ++j) {
        double s = M[(size_t)j * n + j];
        for (int k = 0; k < j; ++k) s -= C[(size_t)j * n + k] * C[(size_t)j * n + k];
        if (!(s > 0)) throw std::runtime_error("generalized_sym_eig: M is not positive definite");
        const double cjj = std::sqrt(s);
        C[(size_t)j * n + j] = cjj;
        for (int i = j + 1; i < n; ++i) {
            double t = M[(size_t)i * n + j];
            for (int k = 0; k < j; ++k) t -= C[(size_t)i * n + k] * C[(size_t)j * n + k];
            C[(size_t)i * n + j] = t / cjj;
        }
    }
    // S = C^-1 L C^-T : W = C^-1 L (column by column), S = C^-1 W^T
    auto lower_solve = [&](std::vector<double>& B) { // B (n x n row-major) <- C^-1 B
        for (int c = 0; c < n; ++c)
            for (int i = 0; i < n; ++i) {
                double t = B[(size_t)i * n + c];
                for (int k = 0; k < i; ++k) t -= C[(size_t)i * n + k] * B[(size_t)k * n + c];
                B[(size_t)i * n + c] = t / C[(size_t)i * n + i];
            }
    };
    std::vector<double> S = L;
    lower_solve(S);
    std::vector<double> St((size_t)n * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) St[(size_t)i * n + j] = S[(size_t)j * n + i];
    lower_solve(St);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < i; ++j) {
            const double v = 0.5 * (St[(size_t)i * n + j] + St[(size_t)j * n + i]);
            St[(size_t)i * n + j] = St[(size_t)j * n + i] = v;
        }
    // cyclic Jacobi on St -> Q (row-major, columns = eigenvectors)
    std::vector<double> A = St, Q((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) Q[(size_t)i * n + i] = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int i = 0; i < n; ++i) {
            diag += A[(size_t)i * n + i] * A[(size_t)i * n + i];
            for (int j = i + 1; j < n; ++j) off += A[(size_t)i * n + j] * A[(size_t)i * n + j];
        }
        if (off <= 1e-32 * diag) break;
        for (int pp = 0; pp < n - 1; ++pp)
            for (int qq = pp + 1; qq < n; ++qq) {
                const double apq = A[(size_t)pp * n + qq];
                if (apq == 0.0) continue;
                const double app = A[(size_t)pp * n + pp], aqq = A[(size_t)qq * n + qq];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < n; ++k) { // columns pp, qq
                    const double akp = A[(size_t)k * n + pp], akq = A[(size_t)k * n + qq];
                    A[(size_t)k * n + pp] = c * akp - s * akq;
                    A[(size_t)k * n + qq] = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) { // rows pp, qq
                    const double apk = A[(size_t)pp * n + k], aqk = A[(size_t)qq * n + k];
                    A[(size_t)pp * n + k] = c * apk - s * aqk;
                    A[(size_t)qq * n + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    const double qkp = Q[(size_t)k * n + pp], qkq = Q[(size_t)k * n + qq];
                    Q[(size_t)k * n + pp] = c * qkp - s * qkq;
                    Q[(size_t)k * n + qq] = s * qkp + c * qkq;
                }
            }
    }
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        return A[(size_t)a * n + a] < A[(size_t)b * n + b];
    });
    lam.assign(n, 0.0);
    U.assign((size_t)n * n, 0.0);
    for (int c = 0; c < n; ++c) {
        const int e = order[c];
        lam[c] = A[(size_t)e * n + e];
        // u = C^-T q : back substitution with C^T (upper)
        std::vector<double> v(n);
        for (int i = 0; i < n; ++i) v[i] = Q[(size_t)i * n + e];
        for (int i = n - 1; i >= 0; --i) {
            double t = v[i];
            for (int k = i + 1; k < n; ++k) t -= C[(size_t)k * n + i] * v[k];
            v[i] = t / C[(size_t)i * n + i];
        }
        int imax = 0;
        for (int i = 1; i < n; ++i)
            if (std::fabs(v[i]) > std::fabs(v[imax])) imax = i;
        const double sg = v[imax] < 0 ? -1.0 : 1.0;
        for (int i = 0; i < n; ++i) U[(size_t)c * n + i] = sg * v[i];
    }
}

} // namespace ks_host

using namespace ks_host;

struct ks_setup {
    int d = 1, p = 1;
    double T = 1.0, nu = 1.0;
    int trial = 0;
    Knots tk;
    std::vector<Knots> sk;
    std::vector<int> dims; // reduced
    Band<double> Lt, Mt;
    Band<cplx> Wt;
    std::vector<Band<double>> M, L, G, V;
    std::vector<std::vector<double>> U, lam;
};

namespace ks {
void set_last_error(const std::string& msg);
}

extern "C" int ks_setup_create(int d, int p, int n_el, int n_el_time, double T, double nu,
                               int trial, ks_setup** out) {
    try {
        if (!out) throw std::invalid_argument("ks_setup_create: out is NULL");
        if (d < 1 || d > 3) throw std::invalid_argument("SpaceTimeProblem: d must be 1, 2 or 3");
        if (!(T > 0) || !(nu > 0)) throw std::invalid_argument("SpaceTimeProblem: T and nu must be positive");
        if (p < 2) throw std::invalid_argument("SpaceTimeProblem: spatial spaces must be C^1 with p_s >= 2");
        if (trial != 0 && trial != 1) throw std::invalid_argument("trial must be 0 or 1");
        auto s = new ks_setup();
        s->d = d;
        s->p = p;
        s->T = T;
        s->nu = nu;
        s->trial = trial;
        s->tk = open_uniform(p, n_el_time, 0.0, T);
        for (int l = 0; l < d; ++l) s->sk.push_back(open_uniform(p, n_el, 0.0, 1.0));
        const Restr rt = trial == 0 ? DropFirst : DropLast;
        s->Lt = real_part(univariate(Stiff, s->tk, rt));
        s->Mt = real_part(univariate(Mass, s->tk, rt));
        s->Wt = univariate(TimeDer, s->tk, rt);
        s->dims.push_back(s->tk.dim() - 1);
        for (int l = 0; l < d; ++l) {
            s->M.push_back(real_part(univariate(Mass, s->sk[l], DropBoth)));
            s->L.push_back(real_part(univariate(Stiff, s->sk[l], DropBoth)));
            s->G.push_back(real_part(univariate(Second, s->sk[l], DropBoth)));
            s->V.push_back(real_part(univariate(Bilap, s->sk[l], DropBoth)));
            s->dims.push_back(s->sk[l].dim() - 2);
            std::vector<double> U, lam;
            // identical axes share the decomposition
            if (l > 0 && s->sk[l].u == s->sk[0].u) {
                U = s->U[0];
                lam = s->lam[0];
            } else {
                gen_sym_eig(s->L[l], s->M[l], U, lam);
            }
            s->U.push_back(U);
            s->lam.push_back(lam);
        }
        *out = s;
        return KS_OK;
    } catch (std::invalid_argument& e) {
        ks::set_last_error(e.what());
        return KS_EINVAL;
    } catch (std::exception& e) {
        ks::set_last_error(e.what());
        return KS_ESINGULAR;
    }
}

extern "C" int ks_setup_dims(const ks_setup* s, int* d, int* dims, int* p) {
    if (!s) return KS_EINVAL;
    if (d) *d = s->d;
    if (p) *p = s->p;
    if (dims)
        for (int i = 0; i <= s->d; ++i) dims[i] = s->dims[i];
    return KS_OK;
}

extern "C" int ks_setup_time_bands(const ks_setup* s, double* Lt, double* Mt, ks_c64* Wt) {
    if (!s) return KS_EINVAL;
    if (Lt) std::memcpy(Lt, s->Lt.a.data(), s->Lt.a.size() * sizeof(double));
    if (Mt) std::memcpy(Mt, s->Mt.a.data(), s->Mt.a.size() * sizeof(double));
    if (Wt) std::memcpy(Wt, s->Wt.a.data(), s->Wt.a.size() * sizeof(ks_c64));
    return KS_OK;
}

extern "C" int ks_setup_space_bands(const ks_setup* s, int l, double* M, double* L, double* G,
                                    double* V) {
    if (!s || l < 0 || l >= s->d) return KS_EINVAL;
    const size_t n = s->M[l].a.size() * sizeof(double);
    if (M) std::memcpy(M, s->M[l].a.data(), n);
    if (L) std::memcpy(L, s->L[l].a.data(), n);
    if (G) std::memcpy(G, s->G[l].a.data(), n);
    if (V) std::memcpy(V, s->V[l].a.data(), n);
    return KS_OK;
}

extern "C" int ks_setup_eig(const ks_setup* s, int l, double* U, double* lambda) {
    if (!s || l < 0 || l >= s->d) return KS_EINVAL;
    if (U) std::memcpy(U, s->U[l].data(), s->U[l].size() * sizeof(double));
    if (lambda) std::memcpy(lambda, s->lam[l].data(), s->lam[l].size() * sizeof(double));
    return KS_OK;
}

extern "C" int ks_setup_create_fd(const ks_setup* s, int device, ks_fd** out) {
    if (!s) return KS_EINVAL;
    std::vector<const double*> U, lam;
    for (int l = 0; l < s->d; ++l) {
        U.push_back(s->U[l].data());
        lam.push_back(s->lam[l].data());
    }
    return ks_fd_create(s->d, s->dims.data(), s->nu, s->p, U.data(), lam.data(), s->Lt.a.data(),
                        s->Mt.a.data(), reinterpret_cast<const ks_c64*>(s->Wt.a.data()), device, out);
}

// galerkin_fast_solver (fdsolver.cpp:177-191): same eigenbasis, H = W + nu lam Mt
extern "C" int ks_setup_create_galerkin_fd(const ks_setup* s, int device, ks_fd** out) {
    if (!s) return KS_EINVAL;
    std::vector<const double*> U, lam;
    for (int l = 0; l < s->d; ++l) {
        U.push_back(s->U[l].data());
        lam.push_back(s->lam[l].data());
    }
    return ks_fd_create_galerkin(s->d, s->dims.data(), s->nu, s->p, U.data(), lam.data(), s->Mt.a.data(),
                                 reinterpret_cast<const ks_c64*>(s->Wt.a.data()), device, out);
}

static int create_system(const ks_setup* s, int device, int nranks, int rank, ks_kron** out, int kind);

// assemble_system (assembly.cpp:202-251), restricted (rs = DropBoth) branch
extern "C" int ks_setup_create_system(const ks_setup* s, int device, ks_kron** out) {
    return create_system(s, device, 0, 0, out, 0);
}
extern "C" int ks_setup_create_system_sharded(const ks_setup* s, int nranks, int rank, int device,
                                              ks_kron** out) {
    return create_system(s, device, nranks, rank, out, 0);
}
// assemble_galerkin_operator (assembly.cpp:273-286): 1 (W x M..) - nu sum_l (Mt x .. G_l^T ..)
extern "C" int ks_setup_create_galerkin_operator(const ks_setup* s, int device, ks_kron** out) {
    return create_system(s, device, 0, 0, out, 1);
}

static int create_system(const ks_setup* s, int device, int nranks, int rank, ks_kron** out, int kind) {
    if (!s) return KS_EINVAL;
    const int d = s->d, D = d + 1;
    const double nu = s->nu;
    auto cx = [](const Band<double>& b) {
        Band<cplx> c(b.n, b.bw);
        for (size_t i = 0; i < b.a.size(); ++i) c.a[i] = b.a[i];
        return c;
    };
    auto transpose = [](const Band<cplx>& b) {
        Band<cplx> t(b.n, b.bw);
        for (int i = 0; i < b.n; ++i)
            for (int j = std::max(0, i - b.bw); j <= std::min(b.n - 1, i + b.bw); ++j)
                t.at(j, i) = b.get(i, j);
        return t;
    };
    std::vector<Band<cplx>> store;
    store.reserve(4 + 6 * d);
    auto keep = [&](Band<cplx> b) -> const Band<cplx>* {
        store.push_back(std::move(b));
        return &store.back();
    };
    const Band<cplx>* Lt = keep(cx(s->Lt));
    const Band<cplx>* Mt = keep(cx(s->Mt));
    Band<cplx> ws = s->Wt; // W + W^H (fdsolver.cpp:95-103, assembly.cpp:178-182)
    for (int i = 0; i < ws.n; ++i)
        for (int j = std::max(0, i - ws.bw); j <= std::min(ws.n - 1, i + ws.bw); ++j)
            ws.at(i, j) += std::conj(s->Wt.get(j, i));
    const Band<cplx>* Wsym = keep(ws);
    std::vector<const Band<cplx>*> M(d), L(d), G(d), Gt(d), V(d);
    for (int l = 0; l < d; ++l) {
        M[l] = keep(cx(s->M[l]));
        L[l] = keep(cx(s->L[l]));
        G[l] = keep(cx(s->G[l]));
        Gt[l] = keep(transpose(*G[l]));
        V[l] = keep(cx(s->V[l]));
    }
    struct T {
        ks_c64 c;
        std::vector<const Band<cplx>*> f;
    };
    std::vector<T> terms;
    auto with_masses = [&](const Band<cplx>* tf) {
        std::vector<const Band<cplx>*> f(D);
        f[0] = tf;
        for (int l = 0; l < d; ++l) f[l + 1] = M[l];
        return f;
    };
    if (kind == 1) {
        const Band<cplx>* W = keep(s->Wt);
        terms.push_back({{1.0, 0.0}, with_masses(W)});
        for (int l = 0; l < d; ++l) {
            auto f = with_masses(Mt);
            f[l + 1] = Gt[l];
            terms.push_back({{-nu, 0.0}, f});
        }
    }
    if (kind == 0) terms.push_back({{1.0, 0.0}, with_masses(Lt)});
    for (int l = 0; l < d && kind == 0; ++l) {
        auto f = with_masses(Mt);
        f[l + 1] = V[l];
        terms.push_back({{nu * nu, 0.0}, f});
    }
    for (int l = 0; l < d && kind == 0; ++l)
        for (int m = 0; m < d; ++m) {
            if (l == m) continue;
            auto f = with_masses(Mt);
            f[l + 1] = G[l];
            f[m + 1] = Gt[m];
            terms.push_back({{nu * nu, 0.0}, f});
        }
    for (int l = 0; l < d && kind == 0; ++l) {
        auto f = with_masses(Wsym);
        f[l + 1] = L[l];
        terms.push_back({{nu, 0.0}, f});
    }
    std::vector<std::vector<const ks_c64*>> fp(terms.size());
    std::vector<std::vector<int>> bw(terms.size());
    std::vector<ks_term> kt(terms.size());
    for (size_t t = 0; t < terms.size(); ++t) {
        for (int a = 0; a < D; ++a) {
            fp[t].push_back(reinterpret_cast<const ks_c64*>(terms[t].f[a]->a.data()));
            bw[t].push_back(terms[t].f[a]->bw);
        }
        kt[t].coeff = terms[t].c;
        kt[t].factors = fp[t].data();
        kt[t].bw = bw[t].data();
    }
    if (nranks > 0)
        return ks_kronshard_create(D, s->dims.data(), (int)kt.size(), kt.data(), nranks, rank, device, out);
    return ks_kron_create(D, s->dims.data(), (int)kt.size(), kt.data(), device, out);
}

// ---------------------------------------------------------------------------
// quadrature / collocation data for the device RHS, lifting and error norms
// (ks_rhs.cu): element_quadrature(kv, p+1) (bspline.cpp:189-208),
// basis_eval_matrix (assembly.cpp:288-303), KnotVector::greville
// (bspline.cpp:77-86), the lifting's collocation factor (assembly.cpp:540-550)
// and the unrestricted univariate factors of assemble_system_operator_full
// (assembly.cpp:260-263)
// ---------------------------------------------------------------------------
namespace {
// factor_banded (eigensolve.cpp:77-121): kl = bw, ku_f = 2 bw, ldab = 3 bw + 1
void factor_band_host(const Band<cplx>& H, std::vector<cplx>& ab, std::vector<int>& piv) {
    const int n = H.n, p = H.bw, ldab = 3 * p + 1, kuf = 2 * p;
    ab.assign((size_t)ldab * n, cplx(0, 0));
    piv.assign(n, 0);
    auto A = [&](int r, int c) -> cplx& { return ab[(size_t)(kuf + r - c) + (size_t)c * ldab]; };
    for (int c = 0; c < n; ++c)
        for (int r = std::max(0, c - p); r <= std::min(n - 1, c + p); ++r) A(r, c) = H.get(r, c);
    for (int k = 0; k < n; ++k) {
        const int imax = std::min(k + p, n - 1);
        int pr = k;
        double best = std::abs(A(k, k));
        for (int r = k + 1; r <= imax; ++r)
            if (std::abs(A(r, k)) > best) {
                best = std::abs(A(r, k));
                pr = r;
            }
        piv[k] = pr;
        if (best == 0.0) throw std::runtime_error("factor_banded: singular collocation matrix");
        const int jmax = std::min(k + kuf, n - 1);
        if (pr != k)
            for (int c = k; c <= jmax; ++c) std::swap(A(k, c), A(pr, c));
        const cplx pv = A(k, k);
        for (int r = k + 1; r <= imax; ++r) {
            const cplx m = A(r, k) / pv;
            A(r, k) = m;
            if (m != cplx(0, 0))
                for (int c = k + 1; c <= jmax; ++c) A(r, c) -= m * A(k, c);
        }
    }
}

ks::QuadAxis quad_axis(const Knots& k) {
    ks::QuadAxis a;
    const int p = k.p;
    a.n = k.dim();
    a.npe = p + 1;
    std::vector<double> gx, gw;
    gauss_legendre(p + 1, gx, gw);
    for (size_t e = 0; e + 1 < k.u.size(); ++e) {
        const double z0 = k.u[e], z1 = k.u[e + 1];
        if (!(z1 > z0)) continue;
        const double mid = 0.5 * (z0 + z1), half = 0.5 * (z1 - z0);
        for (int q = 0; q <= p; ++q) {
            a.nodes.push_back(mid + half * gx[q]);
            a.weights.push_back(half * gw[q]);
        }
    }
    a.nq = (int)a.nodes.size();
    for (int o = 0; o < 3; ++o) a.E[o].assign((size_t)a.nq * (p + 1), 0.0);
    a.off.assign(a.nq, 0);
    for (int q = 0; q < a.nq; ++q) {
        const Basis b = basis_at(k, a.nodes[q], 2);
        a.off[q] = b.first;
        for (int o = 0; o < 3; ++o)
            for (int kk = 0; kk <= p; ++kk) a.E[o][(size_t)q * (p + 1) + kk] = b.d[o][kk];
    }
    a.greville.assign(a.n, 0.0);
    for (int i = 0; i < a.n; ++i) {
        double sm = 0.0;
        for (int kk = 1; kk <= p; ++kk) sm += k.u[i + kk];
        a.greville[i] = sm / p;
    }
    Band<cplx> C(a.n, p);
    for (int i = 0; i < a.n; ++i) {
        const Basis b = basis_at(k, a.greville[i], 0);
        for (int kk = 0; kk <= p; ++kk)
            if (C.in(i, b.first + kk)) C.at(i, b.first + kk) = b.d[0][kk];
    }
    factor_band_host(C, a.colloc_ab, a.colloc_piv);
    return a;
}
} // namespace

namespace ks {
QuadData setup_quad_data(const ks_setup* s) {
    if (!s) throw std::invalid_argument("ks_quad_create: NULL setup");
    QuadData q;
    q.d = s->d;
    q.p = s->p;
    q.trial = s->trial;
    q.nu = s->nu;
    q.red_dims = s->dims;
    q.full_dims.push_back(s->tk.dim());
    for (int l = 0; l < s->d; ++l) q.full_dims.push_back(s->sk[l].dim());
    q.axes.push_back(quad_axis(s->tk));
    for (int l = 0; l < s->d; ++l) q.axes.push_back(quad_axis(s->sk[l]));
    q.Lt = univariate(Stiff, s->tk, None).a;
    q.Mt = univariate(Mass, s->tk, None).a;
    q.Wt = univariate(TimeDer, s->tk, None).a;
    for (int l = 0; l < s->d; ++l) {
        q.M.push_back(univariate(Mass, s->sk[l], None).a);
        q.L.push_back(univariate(Stiff, s->sk[l], None).a);
        q.G.push_back(univariate(Second, s->sk[l], None).a);
        q.V.push_back(univariate(Bilap, s->sk[l], None).a);
    }
    return q;
}
} // namespace ks

extern "C" int ks_setup_full_dims(const ks_setup* s, int* dims) {
    if (!s || !dims) return KS_EINVAL;
    dims[0] = s->tk.dim();
    for (int l = 0; l < s->d; ++l) dims[l + 1] = s->sk[l].dim();
    return KS_OK;
}

// element_quadrature(kv, p+1) of axis `axis` (0 = time): nq nodes / weights
extern "C" int ks_setup_quad_rule(const ks_setup* s, int axis, int* nq, double* nodes, double* weights) {
    if (!s || !nq || axis < 0 || axis > s->d) return KS_EINVAL;
    const ks::QuadAxis a = quad_axis(axis == 0 ? s->tk : s->sk[axis - 1]);
    *nq = a.nq;
    if (nodes) std::copy(a.nodes.begin(), a.nodes.end(), nodes);
    if (weights) std::copy(a.weights.begin(), a.weights.end(), weights);
    return KS_OK;
}

// KnotVector::greville (bspline.cpp:77-86) of axis `axis`: n = full basis size
extern "C" int ks_setup_greville(const ks_setup* s, int axis, int* n, double* pts) {
    if (!s || !n || axis < 0 || axis > s->d) return KS_EINVAL;
    const Knots& k = axis == 0 ? s->tk : s->sk[axis - 1];
    *n = k.dim();
    if (pts)
        for (int i = 0; i < k.dim(); ++i) {
            double sm = 0.0;
            for (int kk = 1; kk <= k.p; ++kk) sm += k.u[i + kk];
            pts[i] = sm / k.p;
        }
    return KS_OK;
}

extern "C" int ks_setup_destroy(ks_setup* s) {
    delete s;
    return KS_OK;
}
