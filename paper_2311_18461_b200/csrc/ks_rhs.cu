// Right-hand side assembly, lifting and error norms on the device
// (SURVEY 8(f) rank 1): the sum-factorised quadrature machinery around the
// solve, with the same tensor contractions as the hot path.
//
// Reference:
//   assemble_rhs            assembly.cpp:390-404 (weighted_moments :338-388):
//                           moments int_Q f D^o(B_i) by mode_product_transpose
//                           (tensorops.cpp:158-217) with the sparse basis-
//                           evaluation matrices, chunked along the outermost
//                           axis, combined as -i mom_t - nu sum_l mom_l and
//                           restricted to the interior (:447-466)
//   lift_nonhomogeneous     assembly.cpp:514-570: Greville-grid collocation
//                           (mode_solve :492-512 with factor_banded), boundary
//                           coefficients (is_constrained :406-425), correction
//                           restrict(A_full g_h) with assemble_system_operator_full
//   extend_with_boundary    assembly.cpp:468-490
//   error_norms             experiments.cpp:73-153: the solution and its
//                           derivatives evaluated on the quadrature grid (mode
//                           products with the evaluation matrices, outermost
//                           axis first, chunk by chunk), L2 error and the
//                           residual of S u_h
//
// The caller evaluates f, u, g at the points (host or device samples); the
// contractions, solves, operator application and reductions run here.
#include "ks_internal.hpp"
#include "ks_quad_host.hpp"

#include <algorithm>
#include <complex>
#include <cstring>
#include <mutex>

using ks::DevBuf;
using cplx = std::complex<double>;

struct ks_quad {
    int device = 0;
    int d = 1, p = 1, trial = 0;
    double nu = 1.0;
    std::vector<int> full, red, nq;
    size_t Nfull = 0, Nred = 0, chunk_max = 0, work = 0;
    struct Axis {
        DevBuf E[3], off, qb, qe, w, ab, piv, nodes, grev;
    };
    std::vector<Axis> ax;
    std::vector<std::vector<double>> w_host;
    DevBuf mom[4];        // moment accumulators (full dims): time derivative, then d/dx_l^2
    DevBuf buf[4];        // work tensors
    DevBuf coeffs;        // full coefficients for the error norms
    DevBuf part;          // reduction partials
    ks_kron* Afull = nullptr;
    cudaStream_t stream = nullptr;
    std::mutex mu;
    ~ks_quad() {
        if (Afull) ks_kron_destroy(Afull);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace ks {
namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cdiv(double2 num, double2 den) { // libgcc __divdc3 (Smith)
    const double a = num.x, b = num.y, c = den.x, d = den.y;
    if (fabs(c) < fabs(d)) {
        const double r = c / d, dn = (c * r) + d;
        return make_double2(((a * r) + b) / dn, ((b * r) - a) / dn);
    }
    const double r = d / c, dn = (d * r) + c;
    return make_double2(((b * r) + a) / dn, (b - (a * r)) / dn);
}

// Fw = f * w with w = w_0[i0] * w_1[i1] * ... * w_d[r0 + i_d] (weighted_moments order)
__global__ void k_weight(const double2* __restrict__ f, double2* __restrict__ out, size_t n, int ndim, int4 dims,
                         const double* w0, const double* w1, const double* w2, const double* w3, int r0) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int dd[4] = {dims.x, dims.y, dims.z, dims.w};
    const double* ws[4] = {w0, w1, w2, w3};
    size_t t = i;
    double w = 1.0;
    for (int a = 0; a < ndim; ++a) {
        const int ia = (int)(t % (size_t)dd[a]);
        t /= (size_t)dd[a];
        const double wa = ws[a][(a == ndim - 1 ? r0 : 0) + ia];
        w = a == 0 ? wa : w * wa;
    }
    const double2 v = f[i];
    out[i] = make_double2(v.x * w, v.y * w);
}

// mode_product_transpose: Y[o][i][s] (+)= sum_{q in rows} E[q][i - off[q]] X[o][q - r0][s]
__global__ void k_mode_T(const double2* __restrict__ X, double2* __restrict__ Y, size_t s, int nin, int nout,
                         size_t outer, const double* __restrict__ E, const int* __restrict__ off,
                         const int* __restrict__ qb, const int* __restrict__ qe, int p, int r0, int acc) {
    const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t n = outer * (size_t)nout * s;
    if (idx >= n) return;
    const size_t q0 = idx % s, t = idx / s;
    const int i = (int)(t % (size_t)nout);
    const size_t o = t / (size_t)nout;
    const int a = max(qb[i], r0), b = min(qe[i], r0 + nin);
    double2 sum = make_double2(0.0, 0.0);
    for (int q = a; q < b; ++q) {
        const double e = E[(size_t)q * (p + 1) + (i - off[q])];
        const double2 x = X[(o * (size_t)nin + (q - r0)) * s + q0];
        sum.x += e * x.x;
        sum.y += e * x.y;
    }
    double2* y = Y + (o * (size_t)nout + i) * s + q0;
    if (acc) {
        const double2 v = *y;
        *y = make_double2(v.x + sum.x, v.y + sum.y);
    } else {
        *y = sum;
    }
}

// mode_product with an evaluation matrix: Y[o][q][s] = sum_k E[r0+q][k] X[o][off[r0+q]+k][s]
__global__ void k_mode_E(const double2* __restrict__ X, double2* __restrict__ Y, size_t s, int nin, int nout,
                         size_t outer, const double* __restrict__ E, const int* __restrict__ off, int p, int r0) {
    const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t n = outer * (size_t)nout * s;
    if (idx >= n) return;
    const size_t q0 = idx % s, t = idx / s;
    const int q = (int)(t % (size_t)nout);
    const size_t o = t / (size_t)nout;
    const int g = r0 + q, f = off[g];
    double2 sum = make_double2(0.0, 0.0);
    for (int k = 0; k <= p; ++k) {
        if (f + k >= nin) break;
        const double e = E[(size_t)g * (p + 1) + k];
        const double2 x = X[(o * (size_t)nin + (f + k)) * s + q0];
        sum.x += e * x.x;
        sum.y += e * x.y;
    }
    Y[(o * (size_t)nout + q) * s + q0] = sum;
}

// mode_solve with one banded LU factor per axis (solve_banded, eigensolve.cpp:123-140)
__global__ void k_mode_solve(double2* __restrict__ X, size_t s, int n, size_t outer, const double2* __restrict__ ab,
                             const int* __restrict__ piv, int p) {
    const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= outer * s) return;
    const size_t q0 = idx % s, o = idx / s;
    double2* x = X + o * (size_t)n * s + q0;
    const int ldab = 3 * p + 1, kuf = 2 * p;
    auto A = [&](int r, int c) { return ab[(size_t)(kuf + r - c) + (size_t)c * ldab]; };
    for (int k = 0; k < n; ++k) {
        const int pr = piv[k];
        if (pr != k) {
            const double2 t = x[(size_t)k * s];
            x[(size_t)k * s] = x[(size_t)pr * s];
            x[(size_t)pr * s] = t;
        }
        const double2 xk = x[(size_t)k * s];
        for (int r = k + 1; r <= min(k + p, n - 1); ++r) x[(size_t)r * s] = csub(x[(size_t)r * s], cmul(A(r, k), xk));
    }
    for (int k = n - 1; k >= 0; --k) {
        const double2 xk = cdiv(x[(size_t)k * s], A(k, k));
        x[(size_t)k * s] = xk;
        for (int r = max(0, k - kuf); r < k; ++r) x[(size_t)r * s] = csub(x[(size_t)r * s], cmul(A(r, k), xk));
    }
}

// full index of reduced element i (reduced_to_full, assembly.cpp:430-436)
__device__ __forceinline__ size_t red_to_full(size_t i, int ndim, const int* rd, const int* fd, int trial) {
    size_t f = 0, stride = 1;
    for (int a = 0; a < ndim; ++a) {
        const int ia = (int)(i % (size_t)rd[a]);
        i /= (size_t)rd[a];
        const int fa = ia + (a == 0 ? (trial == 0 ? 1 : 0) : 1);
        f += stride * (size_t)fa;
        stride *= (size_t)fd[a];
    }
    return f;
}

struct Dims4 {
    int v[4];
};

// out = (0,-1) mom_t + sum_l (-nu) mom_l, restricted to the interior (assemble_rhs)
__global__ void k_rhs_combine(const double2* __restrict__ mt, const double2* __restrict__ m1,
                              const double2* __restrict__ m2, const double2* __restrict__ m3, double2* __restrict__ out,
                              size_t nred, int ndim, Dims4 rd, Dims4 fd, int trial, double nu) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= nred) return;
    const size_t f = red_to_full(i, ndim, rd.v, fd.v, trial);
    // full = 0; axpy((0,-1), mom_t); axpy(-nu, mom_l) for l = 1..d
    double2 v = make_double2(0.0, 0.0);
    const double2 a = mt[f];
    v = make_double2(v.x + (0.0 * a.x - (-1.0) * a.y), v.y + (0.0 * a.y + (-1.0) * a.x));
    const double2* ml[3] = {m1, m2, m3};
    for (int l = 0; l < ndim - 1; ++l) {
        const double2 b = ml[l][f];
        v = make_double2(v.x + (-nu) * b.x, v.y + (-nu) * b.y);
    }
    out[i] = v;
}

__global__ void k_restrict(const double2* __restrict__ full, double2* __restrict__ red, size_t nred, int ndim, Dims4 rd,
                           Dims4 fd, int trial, int subtract) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= nred) return;
    const double2 v = full[red_to_full(i, ndim, rd.v, fd.v, trial)];
    if (subtract) {
        const double2 r = red[i];
        red[i] = make_double2(r.x + (-1.0) * v.x, r.y + (-1.0) * v.y); // axpy(-1, corr, rhs)
    } else {
        red[i] = v;
    }
}

__global__ void k_extend(const double2* __restrict__ red, double2* __restrict__ full, size_t nred, int ndim, Dims4 rd,
                         Dims4 fd, int trial) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= nred) return;
    full[red_to_full(i, ndim, rd.v, fd.v, trial)] = red[i];
}

// keep constrained (boundary / initial or final) coefficients, zero the rest
__global__ void k_boundary_mask(double2* __restrict__ c, size_t n, int ndim, Dims4 fd, int trial) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    size_t t = i;
    bool con = false;
    for (int a = 0; a < ndim; ++a) {
        const int ia = (int)(t % (size_t)fd.v[a]);
        t /= (size_t)fd.v[a];
        if (a == 0) con |= trial == 0 ? ia == 0 : ia == fd.v[0] - 1;
        else con |= ia == 0 || ia == fd.v[a] - 1;
    }
    if (!con) c[i] = make_double2(0.0, 0.0);
}

// su = i Ut (first) / su -= nu Uxx
__global__ void k_su(double2* __restrict__ su, const double2* __restrict__ u, size_t n, double nu, int first) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double2 v = u[i];
    if (first) {
        su[i] = make_double2(0.0 * v.x - 1.0 * v.y, 0.0 * v.y + 1.0 * v.x); // cplx(0,1) * Ut
    } else {
        const double2 s = su[i];
        su[i] = make_double2(s.x - nu * v.x, s.y - nu * v.y);
    }
}

// block partials of sum w |a - b|^2 over the chunk grid
__global__ void k_wnorm(const double2* __restrict__ a, const double2* __restrict__ b, size_t n, int ndim, int4 dims,
                        const double* w0, const double* w1, const double* w2, const double* w3, int r0,
                        double* __restrict__ part) {
    __shared__ double sh[256];
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    double v = 0.0;
    if (i < n) {
        const int dd[4] = {dims.x, dims.y, dims.z, dims.w};
        const double* ws[4] = {w0, w1, w2, w3};
        size_t t = i;
        double w = 1.0;
        for (int x = 0; x < ndim; ++x) {
            const int ia = (int)(t % (size_t)dd[x]);
            t /= (size_t)dd[x];
            const double wa = ws[x][(x == ndim - 1 ? r0 : 0) + ia];
            w = x == 0 ? wa : w * wa;
        }
        const double2 e = make_double2(a[i].x - b[i].x, a[i].y - b[i].y);
        v = w * (e.x * e.x + e.y * e.y);
    }
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st) sh[threadIdx.x] += sh[threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// built-in manufactured solutions sampled on a tensor grid (axis 0 = time fastest):
// 0 "sinsin": u = prod sin(pi x_l) e^{-i d pi^2 t}, f = (1 + nu) d pi^2 u
// 1 "traveling_wave_2d" (problems.cpp:95-117)
__global__ void k_sample(int which, int what, size_t n, int ndim, int4 dims, const double* c0, const double* c1,
                         const double* c2, const double* c3, int r0, double nu, double2* __restrict__ out) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int dd[4] = {dims.x, dims.y, dims.z, dims.w};
    const double* cs[4] = {c0, c1, c2, c3};
    double v[4] = {0, 0, 0, 0};
    size_t t = i;
    for (int a = 0; a < ndim; ++a) {
        const int ia = (int)(t % (size_t)dd[a]);
        t /= (size_t)dd[a];
        v[a] = cs[a][(a == ndim - 1 ? r0 : 0) + ia];
    }
    const double pi = 3.14159265358979323846;
    const int d = ndim - 1;
    double2 u;
    double2 fac = make_double2(1.0, 0.0);
    if (which == 0) {
        double sp = 1.0;
        for (int l = 1; l <= d; ++l) sp *= sin(pi * v[l]);
        double sn, cn;
        sincos(-(double)d * pi * pi * v[0], &sn, &cn);
        u = make_double2(sp * cn, sp * sn);
        fac = make_double2((1.0 + nu) * d * pi * pi, 0.0);
    } else {
        const double w = 0.2, iw2 = 1.0 / (w * w), a = pow(2.0 / (w * w), 0.25);
        const double r2 = v[1] * v[1] + v[2] * v[2];
        double sn, cn;
        sincos(-(r2 + v[0] * v[0]) * iw2, &sn, &cn);
        u = make_double2(a * cn, a * sn);
        fac = make_double2(4.0 * r2 * iw2 * iw2 + 2.0 * v[0] * iw2, 4.0 * iw2);
    }
    out[i] = what == 0 ? u : make_double2(u.x * fac.x - u.y * fac.y, u.x * fac.y + u.y * fac.x);
}

inline unsigned blocks(size_t n) { return (unsigned)((n + 255) / 256); }

size_t prod(const std::vector<int>& v) {
    size_t s = 1;
    for (int x : v) s *= (size_t)x;
    return s;
}

Dims4 d4(const std::vector<int>& v) {
    Dims4 r{{1, 1, 1, 1}};
    for (size_t i = 0; i < v.size() && i < 4; ++i) r.v[i] = v[i];
    return r;
}

// apply k_mode_T along axis a of a tensor with dims `dims` (axis a currently nin long)
void mode_T(ks_quad* q, const double2* X, double2* Y, std::vector<int>& dims, int a, int order, int r0, bool acc) {
    const int nin = dims[a], nout = q->full[a];
    size_t s = 1;
    for (int k = 0; k < a; ++k) s *= (size_t)dims[k];
    const size_t outer = prod(dims) / (s * (size_t)nin);
    auto& A = q->ax[a];
    k_mode_T<<<blocks(outer * (size_t)nout * s), 256, 0, q->stream>>>(
        X, Y, s, nin, nout, outer, A.E[order].as<double>(), A.off.as<int>(), A.qb.as<int>(), A.qe.as<int>(), q->p, r0,
        acc ? 1 : 0);
    check_launch("k_mode_T");
    dims[a] = nout;
}

void mode_E(ks_quad* q, const double2* X, double2* Y, std::vector<int>& dims, int a, int order, int r0, int nrows) {
    const int nin = dims[a];
    size_t s = 1;
    for (int k = 0; k < a; ++k) s *= (size_t)dims[k];
    const size_t outer = prod(dims) / (s * (size_t)nin);
    auto& A = q->ax[a];
    k_mode_E<<<blocks(outer * (size_t)nrows * s), 256, 0, q->stream>>>(X, Y, s, nin, nrows, outer,
                                                                         A.E[order].as<double>(), A.off.as<int>(),
                                                                         q->p, r0);
    check_launch("k_mode_E");
    dims[a] = nrows;
}

const double2* dev_in(ks_quad* q, const ks_c64* p, size_t n, int mem, DevBuf& stage) {
    if (mem == KS_MEM_DEVICE) return reinterpret_cast<const double2*>(p);
    if (stage.bytes < n * sizeof(double2)) stage.alloc(n * sizeof(double2));
    KS_CUDA(cudaMemcpyAsync(stage.p, p, n * sizeof(double2), cudaMemcpyHostToDevice, q->stream));
    return stage.as<double2>();
}

DevBuf& in_stage() {
    static thread_local DevBuf b;
    return b;
}
DevBuf& in_stage2() {
    static thread_local DevBuf b;
    return b;
}

void chunk_dims(ks_quad* q, int r0, int r1, std::vector<int>& dims) {
    dims.assign(q->nq.begin(), q->nq.end());
    dims[q->d] = r1 - r0;
}

} // namespace
} // namespace ks

using namespace ks;

#define API_BEGIN try {
#define API_END                                                                \
    }                                                                          \
    catch (const ks::Error& e) {                                               \
        ks::set_last_error(e.what());                                          \
        return e.code;                                                         \
    }                                                                          \
    catch (const std::exception& e) {                                          \
        ks::set_last_error(e.what());                                          \
        return KS_EINVAL;                                                      \
    }                                                                          \
    return KS_OK;

// moments of one chunk (device samples fd), accumulated into q->mom; no sync
static void rhs_chunk_dev(ks_quad* q, int r0, int r1, const double2* fd) {
    std::vector<int> dims;
    chunk_dims(q, r0, r1, dims);
    const size_t n = prod(dims);
    const int D = q->d + 1;
    int4 dm = make_int4(dims[0], D > 1 ? dims[1] : 1, D > 2 ? dims[2] : 1, D > 3 ? dims[3] : 1);
    const double* w[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int a = 0; a < D; ++a) w[a] = q->ax[a].w.as<double>();
    double2* Fw = q->buf[0].as<double2>();
    k_weight<<<blocks(n), 256, 0, q->stream>>>(fd, Fw, n, D, dm, w[0], w[1], w[2], w[3], r0);
    check_launch("k_weight");
    // order sets: time derivative, then second derivative on each spatial axis
    for (int st = 0; st <= q->d; ++st) {
        std::vector<int> cur = dims;
        const double2* src = Fw;
        int nb = 1;
        for (int a = 0; a < q->d; ++a) {
            const int order = a == 0 ? (st == 0 ? 1 : 0) : (st == a ? 2 : 0);
            double2* dst = q->buf[nb].as<double2>();
            mode_T(q, src, dst, cur, a, order, 0, false);
            src = dst;
            nb = nb == 1 ? 2 : 1;
        }
        const int a = q->d, order = a == 0 ? (st == 0 ? 1 : 0) : (st == a ? 2 : 0);
        mode_T(q, src, q->mom[st].as<double2>(), cur, a, order, r0, true);
    }
}

// built-in problem samples (what 0 = u, 1 = f) on quadrature rows [r0, r1) or the Greville grid; no sync
static void sample_dev(ks_quad* q, int which, int what, int grid, int r0, int r1, double2* out) {
    const int D = q->d + 1;
    std::vector<int> dims;
    const double* c[4] = {nullptr, nullptr, nullptr, nullptr};
    if (grid == 0) {
        chunk_dims(q, r0, r1, dims);
        for (int a = 0; a < D; ++a) c[a] = q->ax[a].nodes.as<double>();
    } else {
        dims = q->full;
        r0 = 0;
        for (int a = 0; a < D; ++a) c[a] = q->ax[a].grev.as<double>();
    }
    const size_t n = prod(dims);
    int4 dm = make_int4(dims[0], D > 1 ? dims[1] : 1, D > 2 ? dims[2] : 1, D > 3 ? dims[3] : 1);
    k_sample<<<blocks(n), 256, 0, q->stream>>>(which, what, n, D, dm, c[0], c[1], c[2], c[3], r0, q->nu, out);
    check_launch("k_sample");
}

static int problem_id(const ks_quad* q, const char* name) {
    if (std::strcmp(name, "sinsin") == 0) return 0;
    if (std::strcmp(name, "traveling_wave_2d") == 0 && q->d == 2) return 1;
    return -1;
}

extern "C" {

int ks_quad_create(const ks_setup* s, int device, ks_quad** out) {
    API_BEGIN
    KS_REQUIRE(s && out, KS_EINVAL, "ks_quad_create: NULL argument");
    ensure_device(device);
    const QuadData Q = setup_quad_data(s);
    std::unique_ptr<ks_quad> q(new ks_quad());
    q->device = device;
    q->d = Q.d;
    q->p = Q.p;
    q->trial = Q.trial;
    q->nu = Q.nu;
    q->full = Q.full_dims;
    q->red = Q.red_dims;
    q->Nfull = prod(q->full);
    q->Nred = prod(q->red);
    KS_CUDA(cudaStreamCreateWithFlags(&q->stream, cudaStreamNonBlocking));
    const int D = Q.d + 1;
    for (int a = 0; a < D; ++a) {
        const QuadAxis& A = Q.axes[a];
        q->nq.push_back(A.nq);
        q->ax.emplace_back();
        auto& X = q->ax.back();
        for (int o = 0; o < 3; ++o) {
            X.E[o].alloc(A.E[o].size() * sizeof(double));
            KS_CUDA(cudaMemcpy(X.E[o].p, A.E[o].data(), A.E[o].size() * sizeof(double), cudaMemcpyHostToDevice));
        }
        X.off.alloc(A.off.size() * sizeof(int));
        KS_CUDA(cudaMemcpy(X.off.p, A.off.data(), A.off.size() * sizeof(int), cudaMemcpyHostToDevice));
        // nodes q with off[q] <= i <= off[q] + p: a contiguous range per basis function
        std::vector<int> qb(A.n, A.nq), qe(A.n, 0);
        for (int g = 0; g < A.nq; ++g)
            for (int k = 0; k <= Q.p; ++k) {
                const int i = A.off[g] + k;
                if (i < A.n) {
                    qb[i] = std::min(qb[i], g);
                    qe[i] = std::max(qe[i], g + 1);
                }
            }
        for (int i = 0; i < A.n; ++i)
            if (qe[i] < qb[i]) qe[i] = qb[i];
        X.qb.alloc(A.n * sizeof(int));
        X.qe.alloc(A.n * sizeof(int));
        KS_CUDA(cudaMemcpy(X.qb.p, qb.data(), A.n * sizeof(int), cudaMemcpyHostToDevice));
        KS_CUDA(cudaMemcpy(X.qe.p, qe.data(), A.n * sizeof(int), cudaMemcpyHostToDevice));
        X.w.alloc(A.weights.size() * sizeof(double));
        KS_CUDA(cudaMemcpy(X.w.p, A.weights.data(), A.weights.size() * sizeof(double), cudaMemcpyHostToDevice));
        q->w_host.push_back(A.weights);
        X.nodes.alloc(A.nodes.size() * sizeof(double));
        KS_CUDA(cudaMemcpy(X.nodes.p, A.nodes.data(), A.nodes.size() * sizeof(double), cudaMemcpyHostToDevice));
        X.grev.alloc(A.greville.size() * sizeof(double));
        KS_CUDA(cudaMemcpy(X.grev.p, A.greville.data(), A.greville.size() * sizeof(double), cudaMemcpyHostToDevice));
        X.ab.alloc(A.colloc_ab.size() * sizeof(double2));
        KS_CUDA(cudaMemcpy(X.ab.p, A.colloc_ab.data(), A.colloc_ab.size() * sizeof(double2), cudaMemcpyHostToDevice));
        X.piv.alloc(A.colloc_piv.size() * sizeof(int));
        KS_CUDA(cudaMemcpy(X.piv.p, A.colloc_piv.data(), A.colloc_piv.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    // chunk = one element of the outermost axis (p+1 nodes)
    std::vector<int> cd(q->nq.begin(), q->nq.end());
    cd[Q.d] = Q.p + 1;
    q->chunk_max = prod(cd);
    q->work = std::max(q->chunk_max, q->Nfull);
    for (int k = 0; k < 4; ++k) q->buf[k].alloc(q->work * sizeof(double2));
    for (int k = 0; k <= Q.d; ++k) q->mom[k].alloc(q->Nfull * sizeof(double2));
    q->part.alloc(blocks(q->work) * sizeof(double));
    // assemble_system_operator_full (assembly.cpp:260-263): the unrestricted factors
    {
        const int d = Q.d, p = Q.p;
        auto transpose = [&](const std::vector<cplx>& b, int n) {
            std::vector<cplx> t(b.size(), cplx(0, 0));
            const int ld = 2 * p + 1;
            for (int j = 0; j < n; ++j)
                for (int i = std::max(0, j - p); i <= std::min(n - 1, j + p); ++i)
                    t[(size_t)(p + j - i) + (size_t)i * ld] = b[(size_t)(p + i - j) + (size_t)j * ld];
            return t;
        };
        std::vector<cplx> ws = Q.Wt; // W + W^H
        {
            const int n = Q.full_dims[0], ld = 2 * p + 1;
            for (int j = 0; j < n; ++j)
                for (int i = std::max(0, j - p); i <= std::min(n - 1, j + p); ++i)
                    ws[(size_t)(p + i - j) + (size_t)j * ld] =
                        Q.Wt[(size_t)(p + i - j) + (size_t)j * ld] + std::conj(Q.Wt[(size_t)(p + j - i) + (size_t)i * ld]);
        }
        std::vector<std::vector<cplx>> Gt(d);
        for (int l = 0; l < d; ++l) Gt[l] = transpose(Q.G[l], Q.full_dims[l + 1]);
        struct T {
            ks_c64 c;
            std::vector<const std::vector<cplx>*> f;
        };
        std::vector<T> terms;
        auto wm = [&](const std::vector<cplx>* tf) {
            std::vector<const std::vector<cplx>*> f(d + 1);
            f[0] = tf;
            for (int l = 0; l < d; ++l) f[l + 1] = &Q.M[l];
            return f;
        };
        terms.push_back({{1.0, 0.0}, wm(&Q.Lt)});
        for (int l = 0; l < d; ++l) {
            auto f = wm(&Q.Mt);
            f[l + 1] = &Q.V[l];
            terms.push_back({{Q.nu * Q.nu, 0.0}, f});
        }
        for (int l = 0; l < d; ++l)
            for (int m = 0; m < d; ++m) {
                if (l == m) continue;
                auto f = wm(&Q.Mt);
                f[l + 1] = &Q.G[l];
                f[m + 1] = &Gt[m];
                terms.push_back({{Q.nu * Q.nu, 0.0}, f});
            }
        // unrestricted coupling -nu [G^T x W^H + G x W] (assemble_system, rs == None branch,
        // assembly.cpp:226-240); on the Dirichlet space it collapses to nu L x (W + W^H)
        std::vector<cplx> Wh(Q.Wt.size(), cplx(0, 0));
        {
            const int n = Q.full_dims[0], ld = 2 * p + 1;
            for (int j = 0; j < n; ++j)
                for (int i = std::max(0, j - p); i <= std::min(n - 1, j + p); ++i)
                    Wh[(size_t)(p + i - j) + (size_t)j * ld] = std::conj(Q.Wt[(size_t)(p + j - i) + (size_t)i * ld]);
        }
        for (int l = 0; l < d; ++l) {
            auto f = wm(&Wh);
            f[l + 1] = &Gt[l];
            terms.push_back({{-Q.nu, 0.0}, f});
            f = wm(&Q.Wt);
            f[l + 1] = &Q.G[l];
            terms.push_back({{-Q.nu, 0.0}, f});
        }
        (void)ws;
        std::vector<std::vector<const ks_c64*>> fp(terms.size());
        std::vector<std::vector<int>> bw(terms.size());
        std::vector<ks_term> kt(terms.size());
        for (size_t t = 0; t < terms.size(); ++t) {
            for (int a = 0; a <= d; ++a) {
                fp[t].push_back(reinterpret_cast<const ks_c64*>(terms[t].f[a]->data()));
                bw[t].push_back(p);
            }
            kt[t].coeff = terms[t].c;
            kt[t].factors = fp[t].data();
            kt[t].bw = bw[t].data();
        }
        const int rc = ks_kron_create(d + 1, Q.full_dims.data(), (int)kt.size(), kt.data(), device, &q->Afull);
        KS_REQUIRE(rc == KS_OK, rc, "ks_quad_create: full-space operator");
    }
    *out = q.release();
    API_END
}

int ks_quad_destroy(ks_quad* q) {
    if (q) {
        cudaSetDevice(q->device);
        delete q;
    }
    return KS_OK;
}

int ks_quad_dims(const ks_quad* q, int* nq, int* chunk, int* full_dims) {
    API_BEGIN
    KS_REQUIRE(q, KS_EINVAL, "ks_quad_dims: NULL handle");
    for (int a = 0; a <= q->d; ++a) {
        if (nq) nq[a] = q->nq[a];
        if (full_dims) full_dims[a] = q->full[a];
    }
    if (chunk) *chunk = q->p + 1;
    API_END
}

int ks_quad_sample_named(ks_quad* q, const char* name, int what, int grid, int r0, int r1, ks_c64* out) {
    API_BEGIN
    KS_REQUIRE(q && name && out, KS_EINVAL, "ks_quad_sample_named: NULL argument");
    const int which = problem_id(q, name);
    KS_REQUIRE(which >= 0, KS_EINVAL, std::string("ks_quad_sample_named: unknown problem ") + name);
    KS_REQUIRE(grid != 0 || (r0 >= 0 && r1 > r0 && r1 <= q->nq[q->d]), KS_EINVAL, "ks_quad_sample_named: bad rows");
    std::lock_guard<std::mutex> lk(q->mu);
    ensure_device(q->device);
    sample_dev(q, which, what, grid, r0, r1, reinterpret_cast<double2*>(out));
    KS_CUDA(cudaStreamSynchronize(q->stream));
    API_END
}

int ks_quad_rhs_reset(ks_quad* q) {
    API_BEGIN
    KS_REQUIRE(q, KS_EINVAL, "ks_quad_rhs_reset: NULL handle");
    std::lock_guard<std::mutex> lk(q->mu);
    ensure_device(q->device);
    for (int k = 0; k <= q->d; ++k)
        KS_CUDA(cudaMemsetAsync(q->mom[k].p, 0, q->Nfull * sizeof(double2), q->stream));
    KS_CUDA(cudaStreamSynchronize(q->stream));
    API_END
}

int ks_quad_rhs_chunk(ks_quad* q, int r0, int r1, const ks_c64* f, int mem) {
    API_BEGIN
    KS_REQUIRE(q && f, KS_EINVAL, "ks_quad_rhs_chunk: NULL argument");
    KS_REQUIRE(r0 >= 0 && r1 > r0 && r1 <= q->nq[q->d] && r1 - r0 <= q->p + 1, KS_EINVAL,
               "ks_quad_rhs_chunk: rows must lie within one element of the outermost axis");
    std::lock_guard<std::mutex> lk(q->mu);
    ensure_device(q->device);
    std::vector<int> dims;
    chunk_dims(q, r0, r1, dims);
    const double2* fd = dev_in(q, f, prod(dims), mem, in_stage());
    rhs_chunk_dev(q, r0, r1, fd);
    KS_CUDA(cudaStreamSynchronize(q->stream));
    API_END
}

// assemble_rhs of a built-in problem's f, every chunk sampled and reduced on the device
int ks_quad_rhs_named(ks_quad* q, const char* name, ks_c64* rhs, int mem) {
    API_BEGIN
    KS_REQUIRE(q && name && rhs, KS_EINVAL, "ks_quad_rhs_named: NULL argument");
    const int which = problem_id(q, name);
    KS_REQUIRE(which >= 0, KS_EINVAL, std::string("ks_quad_rhs_named: unknown problem ") + name);
    std::lock_guard<std::mutex> lk(q->mu);
    ensure_device(q->device);
    for (int k = 0; k <= q->d; ++k) KS_CUDA(cudaMemsetAsync(q->mom[k].p, 0, q->Nfull * sizeof(double2), q->stream));
    const int last = q->nq[q->d];
    for (int r0 = 0; r0 < last; r0 += q->p + 1) {
        const int r1 = std::min(last, r0 + q->p + 1);
        sample_dev(q, which, 1, 0, r0, r1, q->buf[3].as<double2>());
        rhs_chunk_dev(q, r0, r1, q->buf[3].as<double2>());
    }
    double2* out = mem == KS_MEM_DEVICE ? reinterpret_cast<double2*>(rhs) : q->buf[0].as<double2>();
    const int D = q->d + 1;
    k_rhs_combine<<<blocks(q->Nred), 256, 0, q->stream>>>(
        q->mom[0].as<double2>(), q->d >= 1 ? q->mom[1].as<double2>() : nullptr,
        q->d >= 2 ? q->mom[2].as<double2>() : nullptr, q->d >= 3 ? q->mom[3].as<double2>() : nullptr, out, q->Nred, D,
        d4(q->red), d4(q->full), q->trial, q->nu);
    check_launch("k_rhs_combine");
    if (mem != KS_MEM_DEVICE)
        KS_CUDA(cudaMemcpyAsync(rhs, out, q->Nred * sizeof(double2), cudaMemcpyDeviceToHost, q->stream));
    KS_CUDA(cudaStreamSynchronize(q->stream));
    API_END
}

int ks_quad_rhs_finish(ks_quad* q, ks_c64* rhs, int mem) {
    API_BEGIN
    KS_REQUIRE(q && rhs, KS_EINVAL, "ks_quad_rhs_finish: NULL argument");
    std::lock_guard<std::mutex> lk(q->mu);
    ensure_device(q->device);
    double2* out = mem == KS_MEM_DEVICE ? reinterpret_cast<double2*>(rhs) : q->buf[3].as<double2>();
    const int D = q->d + 1;
    k_rhs_combine<<<blocks(q->Nred), 256, 0, q->stream>>>(
        q->mom[0].as<double2>(), q->d >= 1 ? q->mom[1].as<double2>() : nullptr,
        q->d >= 2 ? q->mom[2].as<double2>() : nullptr, q->d >= 3 ? q->mom[3].as<double2>() : nullptr, out, q->Nred, D,
        d4(q->red), d4(q->full), q->trial, q->nu);
    check_launch("k_rhs_combine");
    if (mem != KS_MEM_DEVICE)
        KS_CUDA(cudaMemcpyAsync(rhs, out, q->Nred * sizeof(double2), cudaMemcpyDeviceToHost, q->stream));
    KS_CUDA(cudaStreamSynchronize(q->stream));
    API_END
}

// interior of the spatial moments (full spatial dims fd -> reduced rd, axes 0..d-1)
// added into the reduced space-time rhs at time index 0: rhs[js * nt] += i * bt0 * mom[js]
__global__ void k_add_initial(const double2* __restrict__ mom, double2* __restrict__ rhs, size_t ns, int d, int4 rd,
                              int4 fd, int nt, double bt0) {
    const size_t js = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (js >= ns) return;
    const int r[3] = {rd.x, rd.y, rd.z}, f[3] = {fd.x, fd.y, fd.z};
    size_t t = js, full = 0, stride = 1;
    for (int a = 0; a < d; ++a) {
        const int ia = (int)(t % (size_t)r[a]);
        t /= (size_t)r[a];
        full += (size_t)(ia + 1) * stride; // drop the boundary index 0 on every spatial axis
        stride *= (size_t)f[a];
    }
    const double2 m = mom[full];
    double2 v = rhs[js * (size_t)nt];
    // cplx(0, 1) * bt0[0] * mom: (0 + i) * bt0 = (0, bt0); times mom
    const double2 c = make_double2(0.0 * bt0, 1.0 * bt0);
    v.x += c.x * m.x - c.y * m.y;
    v.y += c.x * m.y + c.y * m.x;
    rhs[js * (size_t)nt] = v;
}

int ks_quad_lift(ks_quad* q, const ks_c64* g_grev, int mem, ks_c64* boundary, ks_c64* correction) {
    API_BEGIN
    KS_REQUIRE(q && g_grev && boundary && correction, KS_EINVAL, "ks_quad_lift: NULL argument");
    std::lock_guard<std::mutex> lk(q->mu);
    ensure_device(q->device);
    double2* C = q->buf[0].as<double2>();
    const double2* g = dev_in(q, g_grev, q->Nfull, mem, in_stage());
    KS_CUDA(cudaMemcpyAsync(C, g, q->Nfull * sizeof(double2), cudaMemcpyDeviceToDevice, q->stream));
    const int D = q->d + 1;
    for (int a = 0; a < D; ++a) { // mode_solve along each axis (assembly.cpp:552-554)
        const int n = q->full[a];
        size_t s = 1;
        for (int k = 0; k < a; ++k) s *= (size_t)q->full[k];
        const size_t outer = q->Nfull / (s * (size_t)n);
        k_mode_solve<<<blocks(outer * s), 256, 0, q->stream>>>(C, s, n, outer, q->ax[a].ab.as<double2>(),
                                                                q->ax[a].piv.as<int>(), q->p);
        check_launch("k_mode_solve");
    }
    k_boundary_mask<<<blocks(q->Nfull), 256, 0, q->stream>>>(C, q->Nfull, D, d4(q->full), q->trial);
    check_launch("k_boundary_mask");
    double2* AC = q->buf[1].as<double2>();
    {
        const int rc = ks_kron_apply(q->Afull, reinterpret_cast<const ks_c64*>(C), reinterpret_cast<ks_c64*>(AC),
                                     KS_MEM_DEVICE, q->stream);
        KS_REQUIRE(rc == KS_OK, rc, "ks_quad_lift: full-space operator apply");
    }
    double2* corr = mem == KS_MEM_DEVICE ? reinterpret_cast<double2*>(correction) : q->buf[2].as<double2>();
    k_restrict<<<blocks(q->Nred), 256, 0, q->stream>>>(AC, corr, q->Nred, D, d4(q->red), d4(q->full), q->trial, 0);
    check_launch("k_restrict");
    if (mem == KS_MEM_DEVICE) {
        KS_CUDA(cudaMemcpyAsync(boundary, C, q->Nfull * sizeof(double2), cudaMemcpyDeviceToDevice, q->stream));
    } else {
        KS_CUDA(cudaMemcpyAsync(boundary, C, q->Nfull * sizeof(double2), cudaMemcpyDeviceToHost, q->stream));
        KS_CUDA(cudaMemcpyAsync(correction, corr, q->Nred * sizeof(double2), cudaMemcpyDeviceToHost, q->stream));
    }
    KS_CUDA(cudaStreamSynchronize(q->stream));
    API_END
}

// assemble_ultraweak's initial-datum term (assembly.cpp:580-637): rhs += i (u0, B_jt(0) phi_js)
int ks_quad_initial_term(ks_quad* q, const ks_c64* u0, int mem, ks_c64* rhs, int rhs_mem) {
    API_BEGIN
    KS_REQUIRE(q && u0 && rhs, KS_EINVAL, "ks_quad_initial_term: NULL argument");
    KS_REQUIRE(q->trial == 1, KS_EINVAL, "assemble_ultraweak: problem must use the final-condition space");
    std::lock_guard<std::mutex> lk(q->mu);
    ensure_device(q->device);
    const int d = q->d;
    // spatial quadrature samples: weights (reference order: w *= w_l for l = 0..d-1), then
    // mode_product_transpose with each spatial evaluation matrix (order 0)
    std::vector<int> dims(q->nq.begin() + 1, q->nq.end());
    size_t n = 1, nfull = 1, nmax = 1;
    for (int l = 0; l < d; ++l) {
        n *= (size_t)dims[l];
        nfull *= (size_t)q->full[l + 1];
    }
    {
        size_t cur = n;
        std::vector<int> dd = dims;
        for (int l = 0; l < d; ++l) {
            cur = cur / (size_t)dd[l] * (size_t)q->full[l + 1];
            dd[l] = q->full[l + 1];
            nmax = std::max(nmax, cur);
        }
        nmax = std::max(nmax, n);
    }
    DevBuf b0(nmax * sizeof(double2)), b1(nmax * sizeof(double2)), stage;
    const double2* src = dev_in(q, u0, n, mem, stage);
    int4 dm = make_int4(dims[0], d > 1 ? dims[1] : 1, d > 2 ? dims[2] : 1, 1);
    const double* w[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int l = 0; l < d; ++l) w[l] = q->ax[l + 1].w.as<double>();
    k_weight<<<blocks(n), 256, 0, q->stream>>>(src, b0.as<double2>(), n, d, dm, w[0], w[1], w[2], w[3], 0);
    check_launch("k_weight");
    double2* bufs[2] = {b0.as<double2>(), b1.as<double2>()};
    int cb = 0;
    for (int l = 0; l < d; ++l) {
        const int nin = dims[l], nout = q->full[l + 1];
        size_t sl = 1;
        for (int k = 0; k < l; ++k) sl *= (size_t)dims[k];
        size_t tot = 1;
        for (int k = 0; k < d; ++k) tot *= (size_t)dims[k];
        const size_t outer = tot / (sl * (size_t)nin);
        auto& A = q->ax[l + 1];
        k_mode_T<<<blocks(outer * (size_t)nout * sl), 256, 0, q->stream>>>(
            bufs[cb], bufs[cb ^ 1], sl, nin, nout, outer, A.E[0].as<double>(), A.off.as<int>(), A.qb.as<int>(),
            A.qe.as<int>(), q->p, 0, 0);
        check_launch("k_mode_T");
        dims[l] = nout;
        cb ^= 1;
    }
    // add into the reduced rhs (final-condition space: time index 0 is kept, and
    // on open knots only B_0 is nonzero at t = 0, with value 1)
    const int nt = q->red[0];
    size_t ns = 1;
    for (int l = 0; l < d; ++l) ns *= (size_t)q->red[l + 1];
    double2* out;
    DevBuf ostage;
    if (rhs_mem == KS_MEM_DEVICE) {
        out = reinterpret_cast<double2*>(rhs);
    } else {
        ostage.alloc(q->Nred * sizeof(double2));
        KS_CUDA(cudaMemcpyAsync(ostage.p, rhs, q->Nred * sizeof(double2), cudaMemcpyHostToDevice, q->stream));
        out = ostage.as<double2>();
    }
    const int4 rd = make_int4(q->red[1], d > 1 ? q->red[2] : 1, d > 2 ? q->red[3] : 1, 1);
    const int4 fd = make_int4(q->full[1], d > 1 ? q->full[2] : 1, d > 2 ? q->full[3] : 1, 1);
    k_add_initial<<<blocks(ns), 256, 0, q->stream>>>(bufs[cb], out, ns, d, rd, fd, nt, 1.0);
    check_launch("k_add_initial");
    if (rhs_mem != KS_MEM_DEVICE)
        KS_CUDA(cudaMemcpyAsync(rhs, out, q->Nred * sizeof(double2), cudaMemcpyDeviceToHost, q->stream));
    KS_CUDA(cudaStreamSynchronize(q->stream));
    (void)nfull;
    API_END
}

int ks_quad_extend(ks_quad* q, const ks_c64* reduced, const ks_c64* boundary, int mem, ks_c64* full) {
    API_BEGIN
    KS_REQUIRE(q && reduced && full, KS_EINVAL, "ks_quad_extend: NULL argument");
    std::lock_guard<std::mutex> lk(q->mu);
    ensure_device(q->device);
    double2* F = mem == KS_MEM_DEVICE ? reinterpret_cast<double2*>(full) : q->buf[0].as<double2>();
    if (boundary) {
        const double2* b = dev_in(q, boundary, q->Nfull, mem, in_stage2());
        KS_CUDA(cudaMemcpyAsync(F, b, q->Nfull * sizeof(double2), cudaMemcpyDeviceToDevice, q->stream));
    } else {
        KS_CUDA(cudaMemsetAsync(F, 0, q->Nfull * sizeof(double2), q->stream));
    }
    const double2* r = dev_in(q, reduced, q->Nred, mem, in_stage());
    k_extend<<<blocks(q->Nred), 256, 0, q->stream>>>(r, F, q->Nred, q->d + 1, d4(q->red), d4(q->full), q->trial);
    check_launch("k_extend");
    if (mem != KS_MEM_DEVICE)
        KS_CUDA(cudaMemcpyAsync(full, F, q->Nfull * sizeof(double2), cudaMemcpyDeviceToHost, q->stream));
    KS_CUDA(cudaStreamSynchronize(q->stream));
    API_END
}

int ks_quad_error_set(ks_quad* q, const ks_c64* full_coeffs, int mem) {
    API_BEGIN
    KS_REQUIRE(q && full_coeffs, KS_EINVAL, "ks_quad_error_set: NULL argument");
    std::lock_guard<std::mutex> lk(q->mu);
    ensure_device(q->device);
    if (!q->coeffs.p) q->coeffs.alloc(q->Nfull * sizeof(double2));
    KS_CUDA(cudaMemcpyAsync(q->coeffs.p, full_coeffs, q->Nfull * sizeof(double2),
                            mem == KS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, q->stream));
    KS_CUDA(cudaStreamSynchronize(q->stream));
    API_END
}

int ks_quad_error_chunk(ks_quad* q, int r0, int r1, const ks_c64* u, const ks_c64* f, int mem, double* l2sq,
                        double* ressq) {
    API_BEGIN
    KS_REQUIRE(q && u && f && l2sq && ressq, KS_EINVAL, "ks_quad_error_chunk: NULL argument");
    KS_REQUIRE(q->coeffs.p, KS_EINVAL, "ks_quad_error_chunk: call ks_quad_error_set first");
    KS_REQUIRE(r0 >= 0 && r1 > r0 && r1 <= q->nq[q->d] && r1 - r0 <= q->p + 1, KS_EINVAL,
               "ks_quad_error_chunk: rows must lie within one element of the outermost axis");
    std::lock_guard<std::mutex> lk(q->mu);
    ensure_device(q->device);
    std::vector<int> cdims;
    chunk_dims(q, r0, r1, cdims);
    const size_t n = prod(cdims);
    const int D = q->d + 1;
    const double2* ud = dev_in(q, u, n, mem, in_stage());
    const double2* fd = dev_in(q, f, n, mem, in_stage2());
    // evaluate the coefficients with derivative orders (last axis first, eval_chunk)
    auto eval = [&](const std::vector<int>& orders, double2* out) {
        std::vector<int> cur = q->full;
        const double2* src = q->coeffs.as<double2>();
        double2* bufs[2] = {q->buf[0].as<double2>(), q->buf[1].as<double2>()};
        int nb = 0;
        const int last = q->d;
        double2* dst = last == 0 ? out : bufs[nb];
        mode_E(q, src, dst, cur, last, orders[last], r0, r1 - r0);
        src = dst;
        nb ^= 1;
        for (int a = 0; a < last; ++a) {
            dst = a == last - 1 ? out : bufs[nb];
            mode_E(q, src, dst, cur, a, orders[a], 0, q->nq[a]);
            src = dst;
            nb ^= 1;
        }
    };
    int4 dm = make_int4(cdims[0], D > 1 ? cdims[1] : 1, D > 2 ? cdims[2] : 1, D > 3 ? cdims[3] : 1);
    const double* w[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int a = 0; a < D; ++a) w[a] = q->ax[a].w.as<double>();
    const unsigned nbk = blocks(n);
    std::vector<double> part(nbk);
    auto wsum = [&](const double2* a, const double2* b) {
        k_wnorm<<<nbk, 256, 0, q->stream>>>(a, b, n, D, dm, w[0], w[1], w[2], w[3], r0, q->part.as<double>());
        check_launch("k_wnorm");
        KS_CUDA(cudaMemcpyAsync(part.data(), q->part.p, nbk * sizeof(double), cudaMemcpyDeviceToHost, q->stream));
        KS_CUDA(cudaStreamSynchronize(q->stream));
        double s = 0.0;
        for (double v : part) s += v;
        return s;
    };
    double2* U = q->buf[2].as<double2>();
    double2* SU = q->buf[3].as<double2>();
    std::vector<int> o(D, 0);
    eval(o, U); // U0
    const double l2 = wsum(ud, U);
    o.assign(D, 0);
    o[0] = 1;
    eval(o, U); // Ut
    k_su<<<nbk, 256, 0, q->stream>>>(SU, U, n, q->nu, 1);
    check_launch("k_su");
    for (int l = 0; l < q->d; ++l) {
        o.assign(D, 0);
        o[l + 1] = 2;
        eval(o, U);
        k_su<<<nbk, 256, 0, q->stream>>>(SU, U, n, q->nu, 0);
        check_launch("k_su");
    }
    const double res = wsum(fd, SU);
    *l2sq = l2;
    *ressq = res;
    API_END
}

} // extern "C"
