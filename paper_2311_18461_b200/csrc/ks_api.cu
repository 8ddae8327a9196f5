// C-ABI implementation (include/ks.h): FD preconditioner, Kronecker operator,
// device-resident PCG, BLAS-1 entry points, device plumbing and timing.
#include "ks_internal.hpp"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <mutex>

namespace ks {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string t_last_error;
void set_last_error(const std::string& msg) { t_last_error = msg; }

void ensure_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw Error(KS_ECUDA, "no CUDA device available (libks has no CPU fallback)");
    KS_REQUIRE(device >= 0 && device < n, KS_EINVAL, "device index out of range");
    KS_CUDA(cudaSetDevice(device));
}

int transform_engine();

void smem_optin(const void* func, int bytes) {
    static std::mutex m;
    static std::vector<std::pair<int, const void*>> done; // (device, function) pairs opted in
    int dev = 0;
    KS_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(m);
        for (auto& e : done)
            if (e.first == dev && e.second == func) return;
    }
    // always the maximum: launches of one function may need different sizes
    (void)bytes;
    KS_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    std::lock_guard<std::mutex> lk(m);
    done.emplace_back(dev, func);
}

int device_sms() {
    static std::mutex m;
    static std::vector<int> sms; // by device index, 0 = unknown
    int dev = 0;
    KS_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(m);
    if ((int)sms.size() <= dev) sms.resize(dev + 1, 0);
    if (!sms[dev]) KS_CUDA(cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev));
    return sms[dev];
}

// kron engine (ks_kron.cu)
struct KronPlan;
KronPlan* kron_plan(const std::vector<int>& dims,
                                    const std::vector<std::vector<double2>>& bands,
                                    const std::vector<int>& band_n, const std::vector<int>& band_bw,
                                    const std::vector<double2>& coeffs,
                                    const std::vector<std::vector<int>>& fids);
void kron_apply(KronPlan& P, const double2* x, double2* y, cudaStream_t st,
                std::vector<void*>& host_ptrs);
void kron_plan_info(const KronPlan& P, int* npasses, int* nnodes, int* nproducts);
int kron_plan_engine(const KronPlan& P);
bool kron_has_table(const KronPlan& P, const void* x, const void* y); // 0 level passes, 1 fused pass pairs, 2 axis 3 + fused t/1/2
void kron_plan_free(KronPlan* p);
void kron_plan_set_shard(KronPlan& P, int rows, int in_off, int band_off);
struct KronPlanDeleter {
    void operator()(KronPlan* p) const { kron_plan_free(p); }
};

} // namespace ks

using namespace ks;

#define API_BEGIN try {
#define API_END                                                                \
    }                                                                          \
    catch (const ks::Error& e) {                                               \
        ks::set_last_error(e.what());                                          \
        return e.code;                                                         \
    }                                                                          \
    catch (const std::bad_alloc&) {                                            \
        ks::set_last_error("host allocation failed");                          \
        return KS_ENOMEM;                                                      \
    }                                                                          \
    catch (const std::exception& e) {                                          \
        ks::set_last_error(e.what());                                          \
        return KS_EINVAL;                                                      \
    }                                                                          \
    return KS_OK;

// ---------------------------------------------------------------------------
// handles
// ---------------------------------------------------------------------------
struct ks_fd {
    int device = 0;
    int d = 0, p = 0;
    double nu = 1.0;
    std::vector<int> dims;
    size_t N = 0, Ns = 0;
    std::vector<DevBuf> At_fwd, At_inv, lam;
    std::vector<FoldAxis> fold;   // per axis; fold[l].n == 0: dense transform
    std::vector<std::vector<double>> lam_host;
    std::vector<int> fiber_block; // host copy of the block map (empty = identity)
    bool tm1 = false;             // time-major hand-off on axis 1 (pair mode, folded axis 1)
    bool posall = false;          // tm1 with position-ordered rows on axes 2..d (ks_xform.cu transforms)
    bool axis1 = false;           // fused axis-1 stage (ks_fdaxis1.cu): transform + solves + transform
    DevBuf A1, order1, grp1;      // its matrix, slab order and per-slab block group
    int n1b = 0;                  // blocks per group (n1 rounded up to even)
    int kind = 0;                 // 0: least-squares blocks, 1: Galerkin blocks (galerkin_fast_solver)
    DevBuf Lt, Mt, Wsym;          // Wsym: W + W^H (least squares) or W itself (Galerkin)
    FdBlocks blocks;
    DevBuf s0, s1, io;
    cudaStream_t stream = nullptr;
    // asynchronous host-pointer applies (caller stream given): H2D, compute and
    // D2H on three streams, kNSlot staging buffers, so consecutive applies
    // overlap their copies in both directions with each other and with the
    // compute. Three slots let the H2D of apply i+2 start while apply i's D2H
    // still drains (two slots serialise H2D(i+2) behind D2H(i)).
    static constexpr int kNSlot = 3;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    DevBuf pio[kNSlot];
    cudaEvent_t ev_in[kNSlot] = {}, ev_comp[kNSlot] = {}, ev_out[kNSlot] = {};
    int slot = 0;
    // ordering across streams: every apply's device work waits for the previous
    // apply's (the scratch s0/s1/io and the staging slots are per handle, whatever
    // stream the caller picks), and records `done` when it has been enqueued
    cudaEvent_t done = nullptr, ev_user = nullptr;
    std::mutex mu;
    ~ks_fd() {
        if (done) cudaEventDestroy(done);
        if (ev_user) cudaEventDestroy(ev_user);
        for (int k = 0; k < kNSlot; ++k) {
            if (ev_in[k]) cudaEventDestroy(ev_in[k]);
            if (ev_comp[k]) cudaEventDestroy(ev_comp[k]);
            if (ev_out[k]) cudaEventDestroy(ev_out[k]);
        }
        if (h2d) cudaStreamDestroy(h2d);
        if (d2h) cudaStreamDestroy(d2h);
        if (stream) cudaStreamDestroy(stream);
    }
};

struct ks_kron {
    int device = 0;
    std::vector<int> dims;
    size_t N = 0;
    // sharded outermost axis: owned planes [lo, hi), haloed input [ext_lo, ext_hi)
    bool sharded = false;
    long long lo = 0, hi = 0, ext_lo = 0, ext_hi = 0;
    size_t plane = 0;
    int nranks = 1, rank = 0, bwd = 0; // sharded: the split and the halo width on the outermost axis
    DevBuf ext;                         // ks_kronshard_apply_comm: the haloed input
    std::unique_ptr<KronPlan, KronPlanDeleter> plan;
    DevBuf io_x, io_y;
    DevBuf pcg[6];                 // ks_pcg work vectors (x, r, z, p, q, scratch), kept across solves
    std::unique_ptr<Reducer> pcg_red[5]; // ks_pcg reducers (pinned host words), kept across solves
    std::vector<void*> hptrs;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr; // see ks_fd::done
    std::mutex mu;
    ~ks_kron() {
        if (done) cudaEventDestroy(done);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace {

inline cudaStream_t pick(void* user, cudaStream_t own) {
    return user ? static_cast<cudaStream_t>(user) : own;
}

// Per-launch timing of an FD apply: start/stop event pairs and the kind of
// each launch (0 spatial transform, 1 fused axis-1 stage, 2 block solves).
struct FdTimes {
    std::vector<cudaEvent_t> ev;
    std::vector<int> kind;
    template <class F> void run(int k, cudaStream_t st, F&& body) {
        cudaEvent_t a, b;
        KS_CUDA(cudaEventCreate(&a));
        KS_CUDA(cudaEventCreate(&b));
        KS_CUDA(cudaEventRecord(a, st));
        body();
        KS_CUDA(cudaEventRecord(b, st));
        ev.push_back(a);
        ev.push_back(b);
        kind.push_back(k);
    }
    ~FdTimes() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};

// FD apply on device pointers (Algorithm 1 steps 2-4; fdsolver.cpp:53-63).
// ev (optional): events around every kernel launch, by kind.
void fd_apply_dev(ks_fd* f, const double2* r, double2* z, bool adjoint, cudaStream_t st, FdTimes* ev) {
    const int d = f->d;
    const double* cur = reinterpret_cast<const double*>(r);
    double* bufs[2] = {f->s0.as<double>(), f->s1.as<double>()};
    int nb = 0;
    auto gemm = [&](const DevBuf& At, int l, const double* in, double* out, int layout) {
        const int n = f->dims[l];
        size_t stride = 1;
        for (int k = 0; k < l; ++k) stride *= (size_t)f->dims[k];
        const size_t outer = f->N / (stride * (size_t)n);
        const FoldAxis& F = f->fold[l - 1];
        const bool inv = &At == &f->At_inv[l - 1];
        auto launch = [&]() {
            if (F.n) launch_mode_gemm_fold(F, inv, in, out, stride, outer, st, layout, f->dims[0]);
            else launch_mode_gemm(At.as<double>(), n, in, out, stride, outer, st, layout, f->dims[0]);
        };
        if (ev) ev->run(0, st, launch);
        else launch();
    };
    // (posall: axes 2..d on the bulk-copy fed transform, eigen rows by position)
    // mode: 0 natural, 1 / 2 the axis-1 time-major hand-off (forward / inverse)
    auto std_gemm = [&](int l, bool inv, const double* in, double* out, int mode = 0) {
        if (!f->posall) return gemm(inv ? f->At_inv[l - 1] : f->At_fwd[l - 1], l, in, out, mode == 0 ? 0 : mode + 2);
        size_t stride = 1;
        for (int k = 0; k < l; ++k) stride *= (size_t)f->dims[k];
        const size_t outer = f->N / (stride * (size_t)f->dims[l]);
        auto launch = [&]() { launch_xfold(f->fold[l - 1], inv, in, out, stride, outer, st, mode); };
        if (ev) ev->run(0, st, launch);
        else launch();
    };
    if (f->axis1) {
        // forward axes d..2, then axis 1 + block solves + inverse axis 1 in one
        // kernel per slab, then inverse axes 2..d (the order of
        // mode products on distinct axes only changes rounding)
        for (int l = d; l >= 2; --l) {
            double* out = bufs[nb];
            nb ^= 1;
            std_gemm(l, false, cur, out);
            cur = out;
        }
        double* mid = d == 1 ? reinterpret_cast<double*>(z) : const_cast<double*>(cur); // in place
        auto launch = [&]() {
            launch_fd_axis1(f->fold[0], f->A1.as<double>(), f->dims[0], (long long)(f->Ns / (size_t)f->dims[1]),
                            f->order1.as<int>(), f->grp1.as<int>(), f->n1b, f->blocks, cur, mid, st);
        };
        if (ev) ev->run(1, st, launch);
        else launch();
        cur = mid;
        for (int l = 2; l <= d; ++l) {
            double* out = l == d ? reinterpret_cast<double*>(z) : bufs[nb];
            if (l != d) nb ^= 1;
            std_gemm(l, true, cur, out);
            cur = out;
        }
        return;
    }
    if (f->tm1) {
        // pair mode with a folded axis 1: forward axes d..1, the axis-1 transform
        // writes the position-ordered time-major layout; solves; inverse axis 1
        // first (reads the time-major layout), then 2..d
        for (int l = d; l >= 1; --l) {
            double* out = bufs[nb];
            nb ^= 1;
            std_gemm(l, false, cur, out, l == 1 ? 1 : 0);
            cur = out;
        }
        auto solve = [&]() {
            launch_fd_solve(f->blocks, reinterpret_cast<double2*>(const_cast<double*>(cur)), adjoint, st);
        };
        if (ev) ev->run(2, st, solve);
        else solve();
        for (int l = 1; l <= d; ++l) {
            double* out = l == d ? reinterpret_cast<double*>(z) : bufs[nb];
            if (l != d) nb ^= 1;
            std_gemm(l, true, cur, out, l == 1 ? 2 : 0);
            cur = out;
        }
        return;
    }
    // to_eigen: axes 1..d with U_l^T (fdsolver.cpp:7-14). The last one (the
    // outermost axis d) writes the time-major layout T[t][fiber] so that the
    // block solves read and write coalesced.
    for (int l = 1; l <= d; ++l) {
        double* out = bufs[nb];
        nb ^= 1;
        gemm(f->At_fwd[l - 1], l, cur, out, l == d ? 1 : 0);
        cur = out;
    }
    // N_s block solves (fdsolver.cpp:58-60), time-major
    auto solve = [&]() { launch_fd_solve(f->blocks, reinterpret_cast<double2*>(const_cast<double*>(cur)), adjoint, st); };
    if (ev) ev->run(2, st, solve);
    else solve();
    // from_eigen with U_l (fdsolver.cpp:16-21): axis d first (it consumes the
    // time-major layout), then axes 1..d-1. Mode products on distinct axes
    // commute, so only the rounding order differs.
    for (int k = 0; k < d; ++k) {
        const int l = k == 0 ? d : k;
        double* out = (k == d - 1) ? reinterpret_cast<double*>(z) : bufs[nb];
        if (k != d - 1) nb ^= 1;
        gemm(f->At_inv[l - 1], l, cur, out, k == 0 ? 2 : 0);
        cur = out;
    }
}

void fd_apply_any(ks_fd* f, const ks_c64* r, ks_c64* z, int mem, void* stream, bool adjoint) {
    KS_REQUIRE(f, KS_EINVAL, "ks_fd_apply: NULL handle");
    KS_REQUIRE(r && z, KS_EINVAL, "ks_fd_apply: NULL vector");
    std::lock_guard<std::mutex> lk(f->mu);
    ensure_device(f->device);
    cudaStream_t st = pick(stream, f->stream);
    const size_t bytes = f->N * sizeof(double2);
    if (mem == KS_MEM_DEVICE) {
        KS_CUDA(cudaStreamWaitEvent(st, f->done, 0));
        fd_apply_dev(f, reinterpret_cast<const double2*>(r), reinterpret_cast<double2*>(z), adjoint,
                     st, nullptr);
        KS_CUDA(cudaEventRecord(f->done, st));
        // no caller stream: behave like the reference's blocking call
        if (!stream) KS_CUDA(cudaStreamSynchronize(st));
    } else if (stream) {
        // pipelined: slot k's H2D waits until slot k's previous D2H has drained
        // its staging buffer (r is read from host memory as soon as the call is
        // made, like the reference's synchronous call reads it); the compute
        // waits for the handle's previous apply (shared scratch); the D2H into z
        // waits until the caller's stream reaches this call (earlier work there
        // may still read z); the caller's stream then waits for the D2H. Making
        // the H2D wait on the caller's stream as well would serialise every H2D
        // behind the previous apply's D2H (that stream waits on it).
        if (!f->h2d) {
            KS_CUDA(cudaStreamCreateWithFlags(&f->h2d, cudaStreamNonBlocking));
            KS_CUDA(cudaStreamCreateWithFlags(&f->d2h, cudaStreamNonBlocking));
            for (int k = 0; k < ks_fd::kNSlot; ++k) {
                KS_CUDA(cudaEventCreateWithFlags(&f->ev_in[k], cudaEventDisableTiming));
                KS_CUDA(cudaEventCreateWithFlags(&f->ev_comp[k], cudaEventDisableTiming));
                KS_CUDA(cudaEventCreateWithFlags(&f->ev_out[k], cudaEventDisableTiming));
                KS_CUDA(cudaEventRecord(f->ev_out[k], f->d2h));
                f->pio[k].alloc(bytes);
            }
        }
        const int k = f->slot;
        f->slot = (f->slot + 1) % ks_fd::kNSlot;
        cudaStream_t us = static_cast<cudaStream_t>(stream);
        double2* buf = f->pio[k].as<double2>();
        KS_CUDA(cudaEventRecord(f->ev_user, us));
        KS_CUDA(cudaStreamWaitEvent(f->h2d, f->ev_out[k], 0));
        KS_CUDA(cudaMemcpyAsync(buf, r, bytes, cudaMemcpyHostToDevice, f->h2d));
        KS_CUDA(cudaEventRecord(f->ev_in[k], f->h2d));
        KS_CUDA(cudaStreamWaitEvent(f->stream, f->ev_in[k], 0));
        KS_CUDA(cudaStreamWaitEvent(f->stream, f->done, 0));
        fd_apply_dev(f, buf, buf, adjoint, f->stream, nullptr);
        KS_CUDA(cudaEventRecord(f->done, f->stream));
        KS_CUDA(cudaEventRecord(f->ev_comp[k], f->stream));
        KS_CUDA(cudaStreamWaitEvent(f->d2h, f->ev_comp[k], 0));
        KS_CUDA(cudaStreamWaitEvent(f->d2h, f->ev_user, 0));
        KS_CUDA(cudaMemcpyAsync(z, buf, bytes, cudaMemcpyDeviceToHost, f->d2h));
        KS_CUDA(cudaEventRecord(f->ev_out[k], f->d2h));
        KS_CUDA(cudaStreamWaitEvent(us, f->ev_out[k], 0));
    } else {
        if (!f->io.p) f->io.alloc(bytes);
        KS_CUDA(cudaStreamWaitEvent(st, f->done, 0));
        KS_CUDA(cudaMemcpyAsync(f->io.p, r, bytes, cudaMemcpyHostToDevice, st));
        fd_apply_dev(f, f->io.as<double2>(), f->io.as<double2>(), adjoint, st, nullptr);
        KS_CUDA(cudaMemcpyAsync(z, f->io.p, bytes, cudaMemcpyDeviceToHost, st));
        KS_CUDA(cudaEventRecord(f->done, st));
        KS_CUDA(cudaStreamSynchronize(st));
    }
}

void kron_apply_any(ks_kron* k, const ks_c64* x, ks_c64* y, int mem, void* stream) {
    KS_REQUIRE(k, KS_EINVAL, "ks_kron_apply: NULL handle");
    KS_REQUIRE(x && y, KS_EINVAL, "ks_kron_apply: NULL vector");
    std::lock_guard<std::mutex> lk(k->mu);
    ensure_device(k->device);
    cudaStream_t st = pick(stream, k->stream);
    const size_t bytes = k->N * sizeof(double2);
    // the plan's intermediates and pointer tables are per handle: order this
    // apply after the previous one whatever stream either ran on
    KS_CUDA(cudaStreamWaitEvent(st, k->done, 0));
    if (mem == KS_MEM_DEVICE) {
        KS_REQUIRE(x != y, KS_EINVAL, "ks_kron_apply: x and y must not alias");
        kron_apply(*k->plan, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y), st,
                   k->hptrs);
        KS_CUDA(cudaEventRecord(k->done, st));
        if (!stream) KS_CUDA(cudaStreamSynchronize(st));
    } else {
        if (!k->io_x.p) {
            k->io_x.alloc(bytes);
            k->io_y.alloc(bytes);
        }
        KS_CUDA(cudaMemcpyAsync(k->io_x.p, x, bytes, cudaMemcpyHostToDevice, st));
        kron_apply(*k->plan, k->io_x.as<double2>(), k->io_y.as<double2>(), st, k->hptrs);
        KS_CUDA(cudaMemcpyAsync(y, k->io_y.p, bytes, cudaMemcpyDeviceToHost, st));
        KS_CUDA(cudaEventRecord(k->done, st));
        KS_CUDA(cudaStreamSynchronize(st));
    }
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    KS_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

} // namespace

extern "C" {

const char* ks_last_error(void) { return t_last_error.c_str(); }
int ks_version(void) { return 1; }
int ks_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}
uint64_t ks_launch_count(void) { return g_launches.load(); }
void ks_launch_count_reset(void) { g_launches.store(0); }

// ---------------------------------------------------------------------------
// FD preconditioner
// ---------------------------------------------------------------------------
} // extern "C"

// FDPreconditioner / galerkin_fast_solver construction (kind 0 / 1)
static void fd_create_impl(int kind, int d, const int* dims, double nu, int p_t, const double* const* U,
                           const double* const* lambda, const double* Lt, const double* Mt, const ks_c64* Wt,
                           int device, ks_fd** out) {
    KS_REQUIRE(out && dims && U && lambda && (Lt || kind == 1) && Mt && Wt, KS_EINVAL,
               "ks_fd_create: NULL argument");
    KS_REQUIRE(d >= 1 && d <= 3, KS_EINVAL, "ks_fd_create: d must be 1, 2 or 3");
    KS_REQUIRE(nu > 0, KS_EINVAL, "ks_fd_create: nu must be positive");
    KS_REQUIRE(p_t >= 1 && p_t <= 8, KS_EINVAL, "ks_fd_create: time degree must be 1..8");
    for (int a = 0; a <= d; ++a) KS_REQUIRE(dims[a] >= 1, KS_EINVAL, "CoeffTensor: dims must be positive");
    for (int l = 0; l < d; ++l) KS_REQUIRE(U[l] && lambda[l], KS_EINVAL, "ks_fd_create: NULL U/lambda");
    // (axes up to 160 keep the folded halves of the eigenvector matrix resident in
    // shared memory -- every BASELINE config: n <= 132; longer axes run the dense
    // panel kernel, ks_transform.cu)
    ensure_device(device);
    std::unique_ptr<ks_fd> f(new ks_fd());
    f->device = device;
    f->d = d;
    f->p = p_t;
    f->nu = nu;
    f->dims.assign(dims, dims + d + 1);
    f->Ns = 1;
    for (int l = 1; l <= d; ++l) f->Ns *= (size_t)dims[l];
    f->N = f->Ns * (size_t)dims[0];
    KS_CUDA(cudaStreamCreateWithFlags(&f->stream, cudaStreamNonBlocking));
    KS_CUDA(cudaEventCreateWithFlags(&f->done, cudaEventDisableTiming));
    KS_CUDA(cudaEventCreateWithFlags(&f->ev_user, cudaEventDisableTiming));
    for (int l = 0; l < d; ++l) {
        const int n = dims[l + 1];
        for (int i = 0; i < n; ++i)
            KS_REQUIRE(lambda[l][i] > 0, KS_EINVAL, "ks_fd_create: eigenvalues must be positive");
        std::vector<double> af((size_t)n * n), ai((size_t)n * n);
        // kernel wants At[j*n + r] = A[r][j]
        // forward A = U^T: A[r][j] = U(j,r) = U[j + r*n]
        // inverse A = U:   A[r][j] = U(r,j) = U[r + j*n]
        for (int j = 0; j < n; ++j)
            for (int r = 0; r < n; ++r) {
                af[(size_t)j * n + r] = U[l][j + (size_t)r * n];
                ai[(size_t)j * n + r] = U[l][r + (size_t)j * n];
            }
        f->At_fwd.emplace_back(af.size() * sizeof(double));
        f->At_inv.emplace_back(ai.size() * sizeof(double));
        KS_CUDA(cudaMemcpy(f->At_fwd.back().p, af.data(), af.size() * sizeof(double), cudaMemcpyHostToDevice));
        KS_CUDA(cudaMemcpy(f->At_inv.back().p, ai.data(), ai.size() * sizeof(double), cudaMemcpyHostToDevice));
        // even/odd fold (uniform meshes): symmetrised eigenvectors, deviation
        // <= 1e-9 of the column max (measured effect on an FD application
        // ~1e-13 relative at c3 sizes)
        f->fold.emplace_back();
        fold_axis_build(U[l], lambda[l], n, 1e-9, f->fold.back());
        f->lam.emplace_back(n * sizeof(double));
        KS_CUDA(cudaMemcpy(f->lam.back().p, lambda[l], n * sizeof(double), cudaMemcpyHostToDevice));
        f->lam_host.emplace_back(lambda[l], lambda[l] + n);
    }
    const int nt = dims[0], ld = 2 * p_t + 1;
    // W + W^H (fdsolver.cpp:95-103)
    std::vector<double2> ws((size_t)ld * nt, make_double2(0, 0));
    auto wget = [&](int i, int j) -> double2 {
        if (i < 0 || j < 0 || i >= nt || j >= nt || std::abs(i - j) > p_t) return make_double2(0, 0);
        const ks_c64 v = Wt[p_t + i - j + (size_t)j * ld];
        return make_double2(v.re, v.im);
    };
    f->kind = kind;
    for (int i = 0; i < nt; ++i)
        for (int j = std::max(0, i - p_t); j <= std::min(nt - 1, i + p_t); ++j) {
            const double2 a = wget(i, j), b = wget(j, i);
            ws[p_t + i - j + (size_t)j * ld] = kind == 1 ? a : make_double2(a.x + b.x, a.y - b.y);
        }
    f->Lt.alloc((size_t)ld * nt * sizeof(double));
    f->Mt.alloc((size_t)ld * nt * sizeof(double));
    f->Wsym.alloc(ws.size() * sizeof(double2));
    if (Lt) KS_CUDA(cudaMemcpy(f->Lt.p, Lt, (size_t)ld * nt * sizeof(double), cudaMemcpyHostToDevice));
    else KS_CUDA(cudaMemset(f->Lt.p, 0, (size_t)ld * nt * sizeof(double)));
    KS_CUDA(cudaMemcpy(f->Mt.p, Mt, (size_t)ld * nt * sizeof(double), cudaMemcpyHostToDevice));
    KS_CUDA(cudaMemcpy(f->Wsym.p, ws.data(), ws.size() * sizeof(double2), cudaMemcpyHostToDevice));
    // factored blocks (fdsolver.cpp:46-51): one per composite eigenvalue, or one
    // per distinct eigenvalue when all axes carry identical 1-D spectra.
    FdBlocks& B = f->blocks;
    B.nt = nt;
    B.p = p_t;
    B.ldab = 3 * p_t + 1;
    B.ns = f->Ns;
    bool dedup = d >= 2;
    for (int l = 1; l < d && dedup; ++l)
        dedup = dims[l + 1] == dims[1] &&
                std::memcmp(lambda[l], lambda[0], sizeof(double) * dims[1]) == 0;
    if (const char* e = std::getenv("KS_FD_DEDUP")) dedup = dedup && std::strcmp(e, "0") != 0;
    // d = 2: the permutation map makes the solves gather their factor rows (a warp of consecutive fibers
    // reads scattered blocks); one block per fiber in layout order reads them coalesced -- c4 FD 0.24 ->
    // 0.21 ms at p = 2, 0.41 -> 0.32 ms at p = 6 -- for twice the factor bytes, so only while those stay
    // small (KS_FD_DEDUP=1 keeps the deduplicated blocks)
    if (d == 2 && dedup) {
        const double row_bytes = kind == 0 ? 16.0 * p_t + 8.0 : (3.0 * p_t + 1.0) * 16.0 + 1.0;
        const char* e = std::getenv("KS_FD_DEDUP");
        if (!(e && std::strcmp(e, "1") == 0) && (double)f->Ns * dims[0] * row_bytes <= 4e9) dedup = false;
    }
    std::vector<double> lam_blk;
    f->fiber_block.clear();
    auto ref_sum = [&](const int* idx) { // fdsolver.cpp:33-35 order
        double sum = 0;
        for (int l = 0; l < d; ++l) sum += lambda[l][idx[l]];
        return sum;
    };
    int idx[3] = {0, 0, 0};
    // pair mode (default for d = 3 with identical axes 2, 3; KS_FD_PAIR=0 off):
    // coalesced two-fiber solves, half the blocks of the plain layout
    bool pair = d == 3 && dims[2] == dims[3] &&
                std::memcmp(lambda[1], lambda[2], sizeof(double) * dims[2]) == 0;
    if (const char* e = std::getenv("KS_FD_PAIR")) pair = pair && std::strcmp(e, "0") != 0;
    // time-major hand-off on axis 1 (pair mode with a folded axis 1): forward
    // transforms run axes d..1, the last one writes
    // T[t][pos(i1) + n1*(i2 + n2*i3)] with the even eigen-indices of axis 1 at
    // positions 0..hc-1 and the odd ones after them (FoldAxis::perm), so both
    // time-major transforms move whole 1 KB rows; the blocks are numbered by
    // position.
    // d = 2 (c2, c4): the same position-ordered plan without pair mode -- both axes on the bulk-copy fed
    // transform (ks_xform.cu), the axis-1 transform hands the time-major layout to the ring solves; the
    // block map / block order below follow the positions (KS_FD_XFOLD=0: round-1 transforms, natural order)
    bool pos2d = d == 2;
    for (int l = 0; l < d && pos2d; ++l)
        pos2d = f->fold[l].n > 0 && (int)f->fold[l].perm.size() == dims[l + 1] && xfold_supported(f->fold[l]);
    if (const char* e = std::getenv("KS_FD_XFOLD")) pos2d = pos2d && std::strcmp(e, "0") != 0;
    // (small problems -- c2: 67 column tiles per transform -- stay on the round-1 kernels: the persistent
    // bulk-copy fed transform measured 3 us slower per launch there, c2 FD 49 -> 55 us)
    // (KS_FD_XFOLD=1 keeps the position-ordered plan at any size: tests)
    const char* xf_env = std::getenv("KS_FD_XFOLD");
    if (pos2d && !(xf_env && std::strcmp(xf_env, "1") == 0) &&
        f->N / ((size_t)std::max(dims[1], dims[2]) * 64) < (size_t)device_sms())
        pos2d = false;
    const bool tm1 = (pair && f->fold[0].n > 0 && (int)f->fold[0].perm.size() == dims[1]) || pos2d;
    f->tm1 = tm1;
    // tm1 with every spatial axis folded: the transforms on axes 2..d keep their
    // eigen rows by position too (ks_xform.cu), so the pair blocks are keyed by
    // (position 2, position 3); needs identical position maps on axes 2 and 3
    bool posall = tm1 && d == 3 && xfold_supported(f->fold[0]);
    for (int l = 1; l < d && posall; ++l)
        posall = f->fold[l].n > 0 && (int)f->fold[l].perm.size() == dims[l + 1] && xfold_supported(f->fold[l]);
    posall = posall && f->fold[1].perm == f->fold[2].perm;
    if (const char* e = std::getenv("KS_FD_XFOLD")) posall = posall && std::strcmp(e, "0") != 0;
    posall = posall || pos2d;
    f->posall = posall;
    // position <-> eigen-index of the axes of a pos2d plan
    std::vector<int> q1, q2, ip1, ip2;
    if (pos2d) {
        q1 = f->fold[0].perm;
        q2 = f->fold[1].perm;
        ip1.resize(q1.size());
        ip2.resize(q2.size());
        for (size_t q = 0; q < q1.size(); ++q) ip1[q1[q]] = (int)q;
        for (size_t q = 0; q < q2.size(); ++q) ip2[q2[q]] = (int)q;
    }
    // fused axis-1 stage (least-squares blocks, folded axis 1, slab fits shared
    // memory; KS_FD_AXIS1=0 keeps the separate transform / solve / transform):
    // blocks numbered by axis-1 position within per-slab groups of n1b.
    // c3: 438 us against 509 us for the three kernels it replaces
    bool ax1 = kind == 0 && f->fold[0].n > 0 && (int)f->fold[0].perm.size() == dims[1] &&
               fd_axis1_supported(dims[1], nt, p_t);
    if (const char* e = std::getenv("KS_FD_AXIS1")) ax1 = ax1 && std::strcmp(e, "0") != 0;
    std::vector<int> grp1;
    if (pair) {
        const int n1 = dims[1], n2 = dims[2];
        // position -> eigen-index of axis 1 (identity unless tm1), and its inverse
        std::vector<int> perm1(n1), pos1(n1);
        for (int p = 0; p < n1; ++p) perm1[p] = tm1 ? f->fold[0].perm[p] : p;
        for (int p = 0; p < n1; ++p) pos1[perm1[p]] = p;
        std::vector<int2> prs;
        std::vector<int> pidx((size_t)n2 * n2);
        for (int i3 = 0; i3 < n2; ++i3)
            for (int i2 = 0; i2 <= i3; ++i2) {
                pidx[(size_t)i2 * n2 + i3] = pidx[(size_t)i3 * n2 + i2] = (int)prs.size();
                prs.push_back(make_int2(i2, i3));
            }
        const int nbg = ax1 ? (n1 + 1) / 2 * 2 : n1; // blocks per pair group
        // position -> eigen-index on axes 2, 3 (identity unless posall), and inverse
        std::vector<int> perm2(n2), pos2(n2);
        for (int q = 0; q < n2; ++q) perm2[q] = posall ? f->fold[1].perm[q] : q;
        for (int q = 0; q < n2; ++q) pos2[perm2[q]] = q;
        lam_blk.resize((size_t)nbg * prs.size());
        for (size_t pp = 0; pp < prs.size(); ++pp)
            for (int p1 = 0; p1 < nbg; ++p1) {
                // (a padding block repeats the group's last eigenvalue; never solved)
                const int id[3] = {perm1[std::min(p1, n1 - 1)], perm2[prs[pp].x], perm2[prs[pp].y]};
                lam_blk[(size_t)p1 + (size_t)nbg * pp] = ref_sum(id);
            }
        if (ax1) {
            grp1.resize(f->Ns / n1);
            for (size_t o = 0; o < grp1.size(); ++o)
                grp1[o] = pidx[(o % n2) * n2 + o / n2];
        }
        // host map by natural fiber index (ks_fd_block); device map by layout
        // position (time-major adjoint solves; natural order unless tm1)
        f->fiber_block.resize(f->Ns);
        std::vector<int> fb_dev(f->Ns);
        for (size_t i = 0; i < f->Ns; ++i) {
            const int i1 = (int)(i % n1), i2 = (int)((i / n1) % n2), i3 = (int)(i / ((size_t)n1 * n2));
            f->fiber_block[i] = pos1[i1] + nbg * pidx[(size_t)pos2[i2] * n2 + pos2[i3]];
            const int pb = nbg * pidx[(size_t)i2 * n2 + i3];
            fb_dev[i] = i1 + pb;
        }
        B.fiber_block.alloc(f->Ns * sizeof(int)); // adjoint / non-time-major solves
        KS_CUDA(cudaMemcpy(B.fiber_block.p, fb_dev.data(), f->Ns * sizeof(int), cudaMemcpyHostToDevice));
        B.pair_n1 = n1;
        B.pair_n2 = n2;
        B.pairs.alloc(prs.size() * sizeof(int2));
        KS_CUDA(cudaMemcpy(B.pairs.p, prs.data(), prs.size() * sizeof(int2), cudaMemcpyHostToDevice));
    } else if (ax1) {
        // one group of n1b position-ordered blocks per slab (no permutation dedup:
        // a slab's blocks must be consecutive)
        const int n1 = dims[1], nbg = (n1 + 1) / 2 * 2;
        const size_t nslab = f->Ns / (size_t)n1;
        std::vector<int> perm1(f->fold[0].perm), pos1(n1);
        for (int p = 0; p < n1; ++p) pos1[perm1[p]] = p;
        lam_blk.resize((size_t)nbg * nslab);
        grp1.resize(nslab);
        for (size_t o = 0; o < nslab; ++o) {
            int id[3] = {0, 0, 0};
            size_t rest = o;
            for (int l = 1; l < d; ++l) {
                id[l] = (int)(rest % (size_t)dims[l + 1]);
                rest /= (size_t)dims[l + 1];
            }
            if (pos2d) id[1] = q2[id[1]]; // slab o sits at position o of axis 2
            for (int p1 = 0; p1 < nbg; ++p1) {
                id[0] = perm1[std::min(p1, n1 - 1)];
                lam_blk[(size_t)p1 + (size_t)nbg * o] = ref_sum(id);
            }
            grp1[o] = (int)o;
        }
        f->fiber_block.resize(f->Ns);
        for (size_t i = 0; i < f->Ns; ++i) {
            const size_t o = i / (size_t)n1;
            f->fiber_block[i] = pos1[i % (size_t)n1] + nbg * (int)(pos2d ? (size_t)ip2[o] : o);
        }
    } else if (!dedup) {
        lam_blk.resize(f->Ns);
        if (pos2d) {
            // blocks in layout (position) order; the host map answers by natural fiber index
            const size_t n1 = (size_t)dims[1];
            f->fiber_block.resize(f->Ns);
            for (size_t i = 0; i < f->Ns; ++i) {
                const int id[3] = {q1[i % n1], q2[i / n1], 0};
                lam_blk[i] = ref_sum(id);
                f->fiber_block[(size_t)id[0] + n1 * (size_t)id[1]] = (int)i;
            }
        } else
        for (size_t i = 0; i < f->Ns; ++i) {
            lam_blk[i] = ref_sum(idx);
            for (int l = 0; l < d; ++l) {
                if (++idx[l] < dims[l + 1]) break;
                idx[l] = 0;
            }
        }
    } else {
        const size_t n = (size_t)dims[1];
        std::vector<int> id_of(f->Ns, -1);
        f->fiber_block.resize(f->Ns);
        // blocks are numbered by the spatial index of their sorted multi-index
        for (size_t i = 0; i < f->Ns; ++i) {
            bool sorted = true;
            for (int l = 1; l < d; ++l) sorted &= idx[l - 1] <= idx[l];
            if (sorted) {
                id_of[i] = (int)lam_blk.size();
                lam_blk.push_back(ref_sum(idx));
            }
            int srt[3] = {idx[0], idx[1], idx[2]};
            std::sort(srt, srt + d);
            size_t key = 0;
            for (int l = d - 1; l >= 0; --l) key = key * n + (size_t)srt[l];
            f->fiber_block[i] = key; // resolved below (key <= i)
            for (int l = 0; l < d; ++l) {
                if (++idx[l] < dims[l + 1]) break;
                idx[l] = 0;
            }
        }
        for (size_t i = 0; i < f->Ns; ++i) f->fiber_block[i] = id_of[f->fiber_block[i]];
        // device map by layout position (natural order unless pos2d)
        std::vector<int> fb_dev(f->fiber_block);
        if (pos2d)
            for (size_t i = 0; i < f->Ns; ++i)
                fb_dev[i] = f->fiber_block[(size_t)q1[i % n] + n * (size_t)q2[i / n]];
        B.fiber_block.alloc(f->Ns * sizeof(int));
        KS_CUDA(cudaMemcpy(B.fiber_block.p, fb_dev.data(), f->Ns * sizeof(int), cudaMemcpyHostToDevice));
    }
    B.nblk = lam_blk.size();
    B.lam_blk.alloc(B.nblk * sizeof(double));
    KS_CUDA(cudaMemcpy(B.lam_blk.p, lam_blk.data(), B.nblk * sizeof(double), cudaMemcpyHostToDevice));
    B.kind = kind;
    if (ax1) B.gsz = (size_t)((dims[1] + 1) / 2 * 2); // one factor group per slab group
    fd_blocks_alloc(B);
    launch_fd_factor(B, nu, f->Lt.as<double>(), f->Mt.as<double>(), f->Wsym.as<double2>(), f->stream);
    if (ax1) {
        const int n1 = dims[1];
        const size_t nslab = f->Ns / (size_t)n1;
        std::vector<double> Am;
        fd_axis1_matrix(f->fold[0], nt, p_t, Am);
        f->A1.alloc(Am.size() * sizeof(double));
        KS_CUDA(cudaMemcpy(f->A1.p, Am.data(), Am.size() * sizeof(double), cudaMemcpyHostToDevice));
        // slabs sharing their blocks (pair mode: (i2, i3) and (i3, i2)) run as
        // neighbouring work items, so the second factor read hits L2
        std::vector<int> order;
        order.reserve(nslab);
        if (pair) {
            const int n2 = dims[2];
            for (int i3 = 0; i3 < n2; ++i3)
                for (int i2 = 0; i2 <= i3; ++i2) {
                    order.push_back(i2 + n2 * i3);
                    if (i2 != i3) order.push_back(i3 + n2 * i2);
                }
        } else {
            for (size_t o = 0; o < nslab; ++o) order.push_back((int)o);
        }
        f->order1.alloc(order.size() * sizeof(int));
        KS_CUDA(cudaMemcpy(f->order1.p, order.data(), order.size() * sizeof(int), cudaMemcpyHostToDevice));
        f->grp1.alloc(grp1.size() * sizeof(int));
        KS_CUDA(cudaMemcpy(f->grp1.p, grp1.data(), grp1.size() * sizeof(int), cudaMemcpyHostToDevice));
        f->n1b = (n1 + 1) / 2 * 2;
        f->axis1 = true;
    }
    f->s0.alloc(f->N * sizeof(double2));
    f->s1.alloc(f->N * sizeof(double2));
    KS_CUDA(cudaStreamSynchronize(f->stream));
    *out = f.release();
}

extern "C" {

int ks_fd_create(int d, const int* dims, double nu, int p_t, const double* const* U,
                 const double* const* lambda, const double* Lt, const double* Mt, const ks_c64* Wt,
                 int device, ks_fd** out) {
    API_BEGIN
    KS_REQUIRE(Lt, KS_EINVAL, "ks_fd_create: NULL argument");
    fd_create_impl(0, d, dims, nu, p_t, U, lambda, Lt, Mt, Wt, device, out);
    API_END
}

int ks_fd_create_galerkin(int d, const int* dims, double nu, int p_t, const double* const* U,
                          const double* const* lambda, const double* Mt, const ks_c64* Wt, int device,
                          ks_fd** out) {
    API_BEGIN
    fd_create_impl(1, d, dims, nu, p_t, U, lambda, nullptr, Mt, Wt, device, out);
    API_END
}

int ks_fd_apply(ks_fd* fd, const ks_c64* r, ks_c64* z, int mem, void* stream) {
    API_BEGIN
    fd_apply_any(fd, r, z, mem, stream, false);
    API_END
}

int ks_fd_apply_adjoint(ks_fd* fd, const ks_c64* r, ks_c64* z, int mem, void* stream) {
    API_BEGIN
    fd_apply_any(fd, r, z, mem, stream, true);
    API_END
}

size_t ks_fd_vec_size(const ks_fd* fd) { return fd ? fd->N : 0; }

int ks_fd_eigenvalues(const ks_fd* fd, double* out) {
    API_BEGIN
    KS_REQUIRE(fd && out, KS_EINVAL, "ks_fd_eigenvalues: NULL argument");
    std::vector<int> idx(fd->d, 0);
    for (size_t i = 0; i < fd->Ns; ++i) {
        double s = 0;
        for (int l = 0; l < fd->d; ++l) s += fd->lam_host[l][idx[l]];
        out[i] = s;
        for (int l = 0; l < fd->d; ++l) {
            if (++idx[l] < fd->dims[l + 1]) break;
            idx[l] = 0;
        }
    }
    API_END
}

int ks_fd_block(const ks_fd* fd, size_t i, ks_c64* ab, int* piv) {
    API_BEGIN
    KS_REQUIRE(fd && ab && piv, KS_EINVAL, "ks_fd_block: NULL argument");
    KS_REQUIRE(i < fd->Ns, KS_EINVAL, "ks_fd_block: index out of range");
    ensure_device(fd->device);
    const size_t b = fd->fiber_block.empty() ? i : (size_t)fd->fiber_block[i];
    fd_block_to_host(fd->blocks, b, ab, piv);
    API_END
}

int ks_fd_info(const ks_fd* fd, int* folded_axes, size_t* blocks) {
    API_BEGIN
    KS_REQUIRE(fd, KS_EINVAL, "ks_fd_info: NULL handle");
    int m = 0;
    for (size_t l = 0; l < fd->fold.size(); ++l)
        if (fd->fold[l].n) m |= 1 << l;
    if (fd->tm1) m |= 1 << 17;
    if (fd->axis1) m |= 1 << 19;
    if (fd->blocks.kind == 0 || fd->blocks.nopiv) m |= 1 << 18; // kind 0: L D L^H, never pivots
    if (folded_axes) *folded_axes = m;
    if (blocks) *blocks = fd->blocks.nblk;
    API_END
}

int ks_fd_destroy(ks_fd* fd) {
    if (fd) {
        cudaSetDevice(fd->device);
        delete fd;
    }
    return KS_OK;
}

// ---------------------------------------------------------------------------
// Kronecker operator
// ---------------------------------------------------------------------------
static void kron_create_impl(int ndim, const int* dims, int nterms, const ks_term* terms, int device,
                             int nranks, int rank, ks_kron** out) {
    KS_REQUIRE(out && dims && ndim >= 1, KS_EINVAL, "ks_kron_create: bad arguments");
    KS_REQUIRE(nterms >= 0 && (nterms == 0 || terms), KS_EINVAL, "ks_kron_create: bad term list");
    for (int a = 0; a < ndim; ++a) KS_REQUIRE(dims[a] >= 1, KS_EINVAL, "CoeffTensor: dims must be positive");
    // factor dedup by content (shared prefixes need equal factors to share ids)
    const bool merge = [] {
        const char* e = std::getenv("KS_KRON_MERGE");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    std::vector<std::vector<double2>> bands;
    std::vector<int> bn, bbw;
    std::vector<double2> coeffs;
    std::vector<std::vector<int>> fids;
    for (int t = 0; t < nterms; ++t) {
        KS_REQUIRE(terms[t].factors, KS_EINVAL, "KroneckerOperator: wrong factor count");
        std::vector<int> ids(ndim, -1);
        double sign = 1.0;
        for (int a = 0; a < ndim; ++a) {
            const ks_c64* f = terms[t].factors[a];
            if (!f) continue;
            KS_REQUIRE(terms[t].bw, KS_EINVAL, "KroneckerOperator: missing bandwidths");
            const int bw = terms[t].bw[a];
            KS_REQUIRE(bw >= 0, KS_EINVAL, "BandedMatrix: invalid dimensions");
            const int n = dims[a];
            std::vector<double2> b((size_t)(2 * bw + 1) * n);
            for (size_t i = 0; i < b.size(); ++i) b[i] = make_double2(f[i].re, f[i].im);
            int id = -1;
            for (size_t e = 0; e < bands.size(); ++e)
                if (bn[e] == n && bbw[e] == bw &&
                    std::memcmp(bands[e].data(), b.data(), b.size() * sizeof(double2)) == 0) {
                    id = (int)e;
                    break;
                }
            // Equal up to sign and rounding (max-norm 1e-12 relative): the C^1
            // Dirichlet spaces have G = -L, so the cross terms' G_l, G_m^T are
            // one factor with L (test_assembly.cpp:39-48) --
            // fewer distinct factors, a smaller plan. KS_KRON_MERGE=0 keeps
            // them apart (exact-content deduplication only).
            if (id < 0 && merge) {
                double mx = 0.0;
                for (const double2& v : b) mx = std::max(mx, std::max(std::fabs(v.x), std::fabs(v.y)));
                for (size_t e = 0; e < bands.size() && id < 0 && mx > 0.0; ++e) {
                    if (bn[e] != n || bbw[e] != bw) continue;
                    for (double sg : {1.0, -1.0}) {
                        double dev = 0.0;
                        for (size_t i = 0; i < b.size() && dev <= 1e-12 * mx; ++i)
                            dev = std::max(dev, std::max(std::fabs(b[i].x - sg * bands[e][i].x),
                                                         std::fabs(b[i].y - sg * bands[e][i].y)));
                        if (dev <= 1e-12 * mx) {
                            id = (int)e;
                            sign *= sg;
                            break;
                        }
                    }
                }
            }
            if (id < 0) {
                id = (int)bands.size();
                bands.push_back(std::move(b));
                bn.push_back(n);
                bbw.push_back(bw);
            }
            ids[a] = id;
        }
        coeffs.push_back(make_double2(sign * terms[t].coeff.re, sign * terms[t].coeff.im));
        fids.push_back(ids);
    }
    ensure_device(device);
    std::unique_ptr<ks_kron> k(new ks_kron());
    k->device = device;
    k->dims.assign(dims, dims + ndim);
    std::vector<int> pdims = k->dims;
    if (nranks > 0) {
        // outermost axis split in slabs (same split as ks_shard_plan); halo = widest band on it
        const int D = ndim - 1;
        const long long nd = dims[D];
        KS_REQUIRE(nranks <= nd && rank >= 0 && rank < nranks, KS_EINVAL, "bad rank / nranks");
        const long long base = nd / nranks, rem = nd % nranks;
        k->lo = rank * base + std::min<long long>(rank, rem);
        k->hi = k->lo + base + (rank < rem ? 1 : 0);
        int bwd = 0;
        for (auto& t : fids)
            if (t[D] >= 0) bwd = std::max(bwd, bbw[t[D]]);
        KS_REQUIRE(nranks == 1 || k->hi - k->lo >= bwd, KS_EINVAL,
                   "sharded matvec: slab thinner than the band (halo would span ranks)");
        k->ext_lo = std::max<long long>(k->lo - bwd, 0);
        k->ext_hi = std::min<long long>(k->hi + bwd, nd);
        k->nranks = nranks;
        k->rank = rank;
        k->bwd = bwd;
        k->plane = 1;
        for (int a = 0; a < D; ++a) k->plane *= (size_t)dims[a];
        pdims[D] = (int)(k->ext_hi - k->ext_lo);
        k->sharded = true;
    }
    k->N = 1;
    for (int a = 0; a < ndim; ++a) k->N *= (size_t)(k->sharded && a == ndim - 1 ? k->hi - k->lo : dims[a]);
    KS_CUDA(cudaStreamCreateWithFlags(&k->stream, cudaStreamNonBlocking));
    KS_CUDA(cudaEventCreateWithFlags(&k->done, cudaEventDisableTiming));
    k->plan.reset(kron_plan(pdims, bands, bn, bbw, coeffs, fids));
    if (k->sharded && bbw.size() && pdims.back() != (int)(k->hi - k->lo))
        kron_plan_set_shard(*k->plan, (int)(k->hi - k->lo), (int)(k->lo - k->ext_lo), (int)k->lo);
    else if (k->sharded)
        kron_plan_set_shard(*k->plan, (int)(k->hi - k->lo), 0, (int)k->lo);
    *out = k.release();
}

int ks_kron_create(int ndim, const int* dims, int nterms, const ks_term* terms, int device,
                   ks_kron** out) {
    API_BEGIN
    kron_create_impl(ndim, dims, nterms, terms, device, 0, 0, out);
    API_END
}

int ks_kronshard_create(int ndim, const int* dims, int nterms, const ks_term* terms, int nranks,
                        int rank, int device, ks_kron** out) {
    API_BEGIN
    KS_REQUIRE(nranks >= 1, KS_EINVAL, "ks_kronshard_create: nranks >= 1");
    kron_create_impl(ndim, dims, nterms, terms, device, nranks, rank, out);
    API_END
}

// host-only slab + halo extents (same split as kron_create_impl)
int ks_kronshard_plan(long long nd, int bw, int nranks, int rank, long long* lo, long long* hi,
                      long long* ext_lo, long long* ext_hi) {
    API_BEGIN
    KS_REQUIRE(nranks >= 1 && nranks <= nd && rank >= 0 && rank < nranks && bw >= 0, KS_EINVAL,
               "ks_kronshard_plan: bad arguments");
    const long long base = nd / nranks, rem = nd % nranks;
    const long long l = rank * base + std::min<long long>(rank, rem);
    const long long h = l + base + (rank < rem ? 1 : 0);
    KS_REQUIRE(nranks == 1 || h - l >= bw, KS_EINVAL, "sharded matvec: slab thinner than the band");
    if (lo) *lo = l;
    if (hi) *hi = h;
    if (ext_lo) *ext_lo = std::max<long long>(l - bw, 0);
    if (ext_hi) *ext_hi = std::min<long long>(h + bw, nd);
    API_END
}

int ks_kronshard_sizes(const ks_kron* k, long long* lo, long long* hi, long long* ext_lo,
                       long long* ext_hi, size_t* plane) {
    API_BEGIN
    KS_REQUIRE(k && k->sharded, KS_EINVAL, "ks_kronshard_sizes: not a sharded operator");
    if (lo) *lo = k->lo;
    if (hi) *hi = k->hi;
    if (ext_lo) *ext_lo = k->ext_lo;
    if (ext_hi) *ext_hi = k->ext_hi;
    if (plane) *plane = k->plane;
    API_END
}

// y_slab = (K x)[slab] from the haloed input x_ext = x[ext_lo .. ext_hi) (device pointers)
int ks_kronshard_apply(ks_kron* k, const ks_c64* x_ext, ks_c64* y_slab, void* stream) {
    API_BEGIN
    KS_REQUIRE(k && k->sharded && x_ext && y_slab, KS_EINVAL, "ks_kronshard_apply: bad arguments");
    std::lock_guard<std::mutex> lk(k->mu);
    ensure_device(k->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : k->stream;
    KS_CUDA(cudaStreamWaitEvent(st, k->done, 0));
    kron_apply(*k->plan, reinterpret_cast<const double2*>(x_ext), reinterpret_cast<double2*>(y_slab), st,
               k->hptrs);
    KS_CUDA(cudaEventRecord(k->done, st));
    if (!stream) KS_CUDA(cudaStreamSynchronize(st));
    API_END
}

} // extern "C"

namespace ks {
// halo exchange with the neighbouring ranks into k->ext, then the local apply
void kronshard_apply_comm(ks_kron* k, ks_comm* c, const double2* x, double2* y, cudaStream_t st) {
    KS_REQUIRE(k->sharded, KS_EINVAL, "ks_kronshard_apply_comm: not a sharded operator");
    KS_REQUIRE(comm_size(c) == k->nranks && comm_rank(c) == k->rank, KS_EINVAL,
               "ks_kronshard_apply_comm: communicator does not match the shard");
    const size_t pl = k->plane, next = (size_t)(k->ext_hi - k->ext_lo) * pl;
    if (k->ext.bytes < next * sizeof(double2)) k->ext.alloc(next * sizeof(double2));
    double2* e = k->ext.as<double2>();
    const long long nd = k->dims.back();
    KS_CUDA(cudaMemcpyAsync(e + (size_t)(k->lo - k->ext_lo) * pl, x, (size_t)(k->hi - k->lo) * pl * sizeof(double2),
                            cudaMemcpyDeviceToDevice, st));
    comm_group_start();
    if (k->rank > 0) { // left neighbour: its right halo = my first planes; my left halo = its last
        long long l_lo, l_hi, l_elo, l_ehi;
        if (ks_kronshard_plan(nd, k->bwd, k->nranks, k->rank - 1, &l_lo, &l_hi, &l_elo, &l_ehi) != KS_OK)
            throw Error(KS_EINVAL, ks_last_error());
        comm_send(x, 2 * (size_t)(l_ehi - l_hi) * pl, k->rank - 1, c, st);
        comm_recv(e, 2 * (size_t)(k->lo - k->ext_lo) * pl, k->rank - 1, c, st);
    }
    if (k->rank + 1 < k->nranks) { // right neighbour
        long long r_lo, r_hi, r_elo, r_ehi;
        if (ks_kronshard_plan(nd, k->bwd, k->nranks, k->rank + 1, &r_lo, &r_hi, &r_elo, &r_ehi) != KS_OK)
            throw Error(KS_EINVAL, ks_last_error());
        comm_send(x + (size_t)(r_elo - k->lo) * pl, 2 * (size_t)(k->hi - r_elo) * pl, k->rank + 1, c, st);
        comm_recv(e + (size_t)(k->hi - k->ext_lo) * pl, 2 * (size_t)(k->ext_hi - k->hi) * pl, k->rank + 1, c, st);
    }
    comm_group_end();
    kron_apply(*k->plan, e, y, st, k->hptrs);
}
} // namespace ks

extern "C" {

int ks_kronshard_apply_comm(ks_kron* k, ks_comm* comm, const ks_c64* x_slab, ks_c64* y_slab, void* stream) {
    API_BEGIN
    KS_REQUIRE(k && comm && x_slab && y_slab, KS_EINVAL, "ks_kronshard_apply_comm: NULL argument");
    std::lock_guard<std::mutex> lk(k->mu);
    ensure_device(k->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : k->stream;
    KS_CUDA(cudaStreamWaitEvent(st, k->done, 0));
    kronshard_apply_comm(k, comm, reinterpret_cast<const double2*>(x_slab), reinterpret_cast<double2*>(y_slab), st);
    KS_CUDA(cudaEventRecord(k->done, st));
    if (!stream) KS_CUDA(cudaStreamSynchronize(st));
    API_END
}

int ks_kron_apply(ks_kron* k, const ks_c64* x, ks_c64* y, int mem, void* stream) {
    API_BEGIN
    kron_apply_any(k, x, y, mem, stream);
    API_END
}

size_t ks_kron_vec_size(const ks_kron* k) { return k ? k->N : 0; }

int ks_kron_plan_info(const ks_kron* k, int* npasses, int* nnodes, int* nproducts) {
    API_BEGIN
    KS_REQUIRE(k, KS_EINVAL, "NULL handle");
    kron_plan_info(*k->plan, npasses, nnodes, nproducts);
    API_END
}

int ks_kron_engine(const ks_kron* k, int* engine) {
    API_BEGIN
    KS_REQUIRE(k && engine, KS_EINVAL, "ks_kron_engine: bad arguments");
    *engine = kron_plan_engine(*k->plan);
    API_END
}

int ks_kron_destroy(ks_kron* k) {
    if (k) {
        cudaSetDevice(k->device);
        delete k;
    }
    return KS_OK;
}

// ---------------------------------------------------------------------------
// PCG (krylov.cpp:24-114)
// ---------------------------------------------------------------------------
} // extern "C"

// pcg body shared by ks_pcg (one GPU: A, P) and ks_pcg_sharded (this rank's
// slabs: sharded A, Ps, communicator; dots all-reduced on the device)
static void pcg_impl(ks_kron* A, ks_fd* P, ks_fdshard* Ps, ks_comm* comm, const ks_c64* b, ks_c64* x, int mem,
                     const ks_pcg_opts* opts, double* res_hist, int hist_cap, ks_pcg_report* report) {
    KS_REQUIRE(A && b && x && opts && report, KS_EINVAL, "ks_pcg: NULL argument");
    KS_REQUIRE(opts->tol > 0 && opts->maxit >= 0, KS_EINVAL, "pcg: bad options");
    KS_REQUIRE(!P || P->N == A->N, KS_EINVAL, "pcg: operator sizes differ");
    KS_REQUIRE(!P || P->device == A->device, KS_EINVAL, "pcg: operators on different devices");
    KS_REQUIRE(!Ps || (fdshard_slab_n(Ps) == A->N && fdshard_device(Ps) == A->device), KS_EINVAL,
               "pcg: sharded operators differ in slab or device");
    KS_REQUIRE(!comm || A->sharded, KS_EINVAL, "pcg_sharded: the operator is not sharded");
    // device scalars summed over the ranks (in place, stream-ordered)
    auto allreduce = [&](Reducer& rd) {
        if (comm) comm_allreduce_sum(rd.result.as<double>(), 1, comm, A->stream);
    };
    std::lock_guard<std::mutex> lka(A->mu);
    std::unique_ptr<std::lock_guard<std::mutex>> lkp;
    if (P) lkp.reset(new std::lock_guard<std::mutex>(P->mu));
    ensure_device(A->device);
    std::memset(report, 0, sizeof(*report));
    cudaStream_t st = A->stream;
    // after any apply still in flight on either handle (other streams)
    KS_CUDA(cudaStreamWaitEvent(st, A->done, 0));
    if (P) KS_CUDA(cudaStreamWaitEvent(st, P->done, 0));
    const size_t n = A->N, bytes = n * sizeof(double2);
    const auto t_start = std::chrono::steady_clock::now();

    // work vectors live in the operator handle: a solve allocates nothing after the first
    for (auto& w : A->pcg)
        if (w.bytes < bytes) w.alloc(bytes);
    DevBuf bb;
    DevBuf &xv = A->pcg[0], &r = A->pcg[1], &z = A->pcg[2], &p = A->pcg[3], &q = A->pcg[4],
           &scratch = A->pcg[5];
    const double2* bd;
    if (mem == KS_MEM_DEVICE) {
        bd = reinterpret_cast<const double2*>(b);
    } else {
        bb.alloc(bytes);
        KS_CUDA(cudaMemcpyAsync(bb.p, b, bytes, cudaMemcpyHostToDevice, st));
        bd = bb.as<double2>();
    }
    KS_CUDA(cudaMemsetAsync(xv.p, 0, bytes, st));
    // Scalars stay on the device: alpha and beta are formed by the update
    // kernels from the reducers' results, so an iteration has one host round
    // trip (curvature + ||r||^2, read together for the breakdown and
    // convergence tests). Operator timers: event pairs, summed at the end.
    for (auto& rp : A->pcg_red)
        if (!rp) rp.reset(new Reducer());
    Reducer &red = *A->pcg_red[0], &red_c = *A->pcg_red[1], &red_u = *A->pcg_red[2];
    Reducer &rho_old = *A->pcg_red[3], &rho_new = *A->pcg_red[4]; // rho_old <- rho_new after each p update
    std::vector<cudaEvent_t> evs;
    struct EvGuard {
        std::vector<cudaEvent_t>& v;
        ~EvGuard() {
            for (auto e : v) cudaEventDestroy(e);
        }
    } evg{evs};
    std::vector<std::pair<int, int>> mv_ev, pc_ev; // indices into evs
    auto ev_pair = [&](std::vector<std::pair<int, int>>& dst, auto&& body) {
        cudaEvent_t a, b2;
        KS_CUDA(cudaEventCreate(&a));
        evs.push_back(a);
        KS_CUDA(cudaEventCreate(&b2));
        evs.push_back(b2);
        KS_CUDA(cudaEventRecord(a, st));
        body();
        KS_CUDA(cudaEventRecord(b2, st));
        dst.push_back({(int)evs.size() - 2, (int)evs.size() - 1});
    };
    auto mv = [&](const double2* in, double2* outv) {
        if (comm) kronshard_apply_comm(A, comm, in, outv, st);
        else kron_apply(*A->plan, in, outv, st, A->hptrs);
    };
    auto pc = [&](const double2* rin, double2* zout) {
        if (Ps) fdshard_apply_comm(Ps, comm, rin, zout, st);
        else if (P) fd_apply_dev(P, rin, zout, false, st, nullptr);
        else KS_CUDA(cudaMemcpyAsync(zout, rin, bytes, cudaMemcpyDeviceToDevice, st));
    };
    auto matvec = [&](const double2* in, double2* outv) { ev_pair(mv_ev, [&]() { mv(in, outv); }); };
    auto precond = [&](const double2* rin, double2* zout) {
        if (P || Ps) ev_pair(pc_ev, [&]() { pc(rin, zout); });
        else pc(rin, zout);
    };
    // The two halves of an iteration, replayed as CUDA graphs after their first
    // (eager) run, which does the allocations, first-apply tuning and pointer
    // tables: phase A = q = A p, curvature, update of x and r, both scalars to
    // the host; phase B = z = P r, rho', p = z + (rho'/rho) p, rho <- rho'.
    // Opt-in (KS_PCG_GRAPH=1): a graph launch replaces ~10-20 kernel launches,
    // but measured c2 (279 K DOF) 2.43 vs 2.53 ms for 9 iterations, c3 20.9 vs
    // 21.1 ms, and the capture costs ~2.6 ms per solve -- the iterations are
    // bound by their kernels, not by launches. The matvec / precond timers
    // cover their whole phase (operator + fused BLAS-1).
    const bool graphs_ok = [] {
        const char* e = std::getenv("KS_PCG_GRAPH");
        return e && std::strcmp(e, "1") == 0;
    }();
    struct Graphs {
        cudaGraphExec_t g[2] = {nullptr, nullptr};
        void reset() {
            for (auto& e : g)
                if (e) {
                    cudaGraphExecDestroy(e);
                    e = nullptr;
                }
        }
        ~Graphs() { reset(); }
    } graphs;
    bool use_graph = graphs_ok && !comm, seen[2] = {false, false};
    // Deferred solution update: phase A updates only r, and x += alpha_k p_k
    // rides along the p update of phase B (which reads p_k anyway) -- or runs
    // alone before a true residual and at exit. Same arithmetic on the same
    // operands: bit-identical iterates, 48 B per element less vector traffic per
    // iteration. In strict mode x is needed every iteration, so it is updated
    // right after phase A.
    bool pending = false; // x += alpha_k p_k not yet applied
    auto apply_x = [&]() {
        if (!pending) return;
        launch_x_update_dev(rho_old.result.as<double>(), red_c.result.as<double>(), p.as<double2>(), xv.as<double2>(),
                            n, st);
        pending = false;
    };
    auto phase_a = [&]() {
        mv(p.as<double2>(), q.as<double2>());
        launch_dotc(red_c, p.as<double2>(), q.as<double2>(), n, st); // curvature Re <p, Ap>
        allreduce(red_c);
        launch_cg_update_r_dev(red_u, rho_old.result.as<double>(), red_c.result.as<double>(), q.as<double2>(),
                               r.as<double2>(), n, st);
        allreduce(red_u);
        KS_CUDA(cudaMemcpyAsync(red_c.host, red_c.result.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        KS_CUDA(cudaMemcpyAsync(red_u.host, red_u.result.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    };
    auto phase_b = [&]() {
        // z = P r and rho' = Re <r, z>
        pc(r.as<double2>(), z.as<double2>());
        launch_dotc(rho_new, r.as<double2>(), z.as<double2>(), n, st); // rho' = Re <r, z>
        allreduce(rho_new);
        if (pending) { // (the caller clears pending: a replayed graph does not run this body)
            launch_xpby_x_dev(z.as<double2>(), rho_new.result.as<double>(), rho_old.result.as<double>(),
                              red_c.result.as<double>(), p.as<double2>(), xv.as<double2>(), n, st);
        } else {
            launch_xpby_dev(z.as<double2>(), rho_new.result.as<double>(), rho_old.result.as<double>(),
                            p.as<double2>(), n, st);
        }
        KS_CUDA(cudaMemcpyAsync(rho_old.result.p, rho_new.result.p, sizeof(double), cudaMemcpyDeviceToDevice, st));
    };
    auto run_phase = [&](int which, auto&& body, std::vector<std::pair<int, int>>& tim) {
        if (use_graph && seen[which] && !graphs.g[which]) {
            cudaGraph_t gr = nullptr;
            bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                try {
                    body();
                } catch (const Error&) {
                    ok = false;
                }
                ok = cudaStreamEndCapture(st, &gr) == cudaSuccess && ok;
                ok = ok && cudaGraphInstantiate(&graphs.g[which], gr, 0) == cudaSuccess;
                if (gr) cudaGraphDestroy(gr);
            }
            if (!ok) { // capture not possible here: stay eager for this solve
                cudaGetLastError();
                graphs.reset();
                use_graph = false;
            }
        }
        if (graphs.g[which]) ev_pair(tim, [&]() { KS_CUDA(cudaGraphLaunch(graphs.g[which], st)); });
        else ev_pair(tim, [&]() { body(); });
        seen[which] = true;
    };
    auto norm2 = [&](const double2* a) {
        launch_norm2sq(red, a, n, st);
        allreduce(red);
        fetch(red, st, 1);
        return red.host[0];
    };
    auto finish_out = [&]() {
        KS_CUDA(cudaMemcpyAsync(x, xv.p, bytes,
                                mem == KS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                st));
        KS_CUDA(cudaEventRecord(A->done, st));
        if (P) KS_CUDA(cudaEventRecord(P->done, st));
        KS_CUDA(cudaStreamSynchronize(st));
        double t_mv = 0, t_pc = 0;
        for (auto& e : mv_ev) t_mv += elapsed(evs[e.first], evs[e.second]) * 1e-3;
        for (auto& e : pc_ev) t_pc += elapsed(evs[e.first], evs[e.second]) * 1e-3;
        report->matvec_seconds = t_mv;
        report->precond_seconds = t_pc;
        report->solve_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    };
    int hist_len = 0;
    auto push_hist = [&](double v) {
        if (res_hist && hist_len < hist_cap) res_hist[hist_len] = v;
        ++hist_len;
    };
    auto set_last_hist = [&](double v) {
        if (res_hist && hist_len - 1 < hist_cap && hist_len > 0) res_hist[hist_len - 1] = v;
    };

    const double bnorm = std::sqrt(norm2(bd));
    if (bnorm == 0.0) {
        report->converged = 1;
        finish_out();
        return;
    }
    auto true_relres = [&]() {
        // a new pointer table may evict the captured phases' tables: recapture later
        if (!kron_has_table(*A->plan, xv.p, scratch.p)) graphs.reset(), seen[0] = seen[1] = false;
        matvec(xv.as<double2>(), scratch.as<double2>());
        launch_axpy_real(-1.0, bd, scratch.as<double2>(), n, st); // Ax - b
        return std::sqrt(norm2(scratch.as<double2>())) / bnorm;
    };
    KS_CUDA(cudaMemcpyAsync(r.p, bd, bytes, cudaMemcpyDeviceToDevice, st));
    precond(r.as<double2>(), z.as<double2>());
    KS_CUDA(cudaMemcpyAsync(p.p, z.p, bytes, cudaMemcpyDeviceToDevice, st));
    launch_dotc(rho_old, r.as<double2>(), z.as<double2>(), n, st); // rho = Re <r, z>
    allreduce(rho_old);
    int restarts = 0;
    for (int k = 0; k < opts->maxit; ++k) {
        run_phase(0, phase_a, mv_ev);
        KS_CUDA(cudaStreamSynchronize(st));
        if (red_c.host[0] <= 0.0) { // x, r untouched by the update kernel
            report->breakdown = 1;
            break;
        }
        report->iterations++;
        pending = true;
        double relres = std::sqrt(red_u.host[0]) / bnorm;
        if (opts->strict_residual) {
            apply_x();
            relres = true_relres();
        }
        push_hist(relres);
        if (relres <= opts->tol) {
            if (!opts->strict_residual) {
                apply_x();
                const double tr = true_relres();
                set_last_hist(tr);
                if (tr > opts->tol) {
                    if (++restarts > 2) break;
                    launch_neg_copy(scratch.as<double2>(), r.as<double2>(), n, st);
                    precond(r.as<double2>(), z.as<double2>());
                    KS_CUDA(cudaMemcpyAsync(p.p, z.p, bytes, cudaMemcpyDeviceToDevice, st));
                    launch_dotc(rho_old, r.as<double2>(), z.as<double2>(), n, st);
                    allreduce(rho_old);
                    continue;
                }
            }
            report->converged = 1;
            break;
        }
        run_phase(1, phase_b, pc_ev);
        pending = false;
    }
    apply_x(); // maxit reached with the last update pending
    report->restarts = restarts;
    report->hist_len = hist_len < hist_cap ? hist_len : hist_cap;
    if (!res_hist) report->hist_len = 0;
    finish_out();
}

extern "C" {

int ks_pcg(ks_kron* A, ks_fd* P, const ks_c64* b, ks_c64* x, int mem, const ks_pcg_opts* opts,
           double* res_hist, int hist_cap, ks_pcg_report* report) {
    API_BEGIN
    KS_REQUIRE(!A || !A->sharded, KS_EINVAL, "ks_pcg: sharded operator (use ks_pcg_sharded)");
    pcg_impl(A, P, nullptr, nullptr, b, x, mem, opts, res_hist, hist_cap, report);
    API_END
}

int ks_pcg_sharded(ks_kron* A, ks_fdshard* P, ks_comm* comm, const ks_c64* b_slab, ks_c64* x_slab, int mem,
                   const ks_pcg_opts* opts, double* res_hist, int hist_cap, ks_pcg_report* report) {
    API_BEGIN
    KS_REQUIRE(comm, KS_EINVAL, "ks_pcg_sharded: NULL communicator");
    pcg_impl(A, nullptr, P, comm, b_slab, x_slab, mem, opts, res_hist, hist_cap, report);
    API_END
}


// ---------------------------------------------------------------------------
// BLAS-1 on device vectors
// ---------------------------------------------------------------------------
int ks_axpy_real(double a, const ks_c64* x, ks_c64* y, size_t n, void* stream) {
    API_BEGIN
    launch_axpy_real(a, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y), n,
                     static_cast<cudaStream_t>(stream));
    KS_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    API_END
}
int ks_axpy(ks_c64 a, const ks_c64* x, ks_c64* y, size_t n, void* stream) {
    API_BEGIN
    launch_axpy(make_double2(a.re, a.im), reinterpret_cast<const double2*>(x),
                reinterpret_cast<double2*>(y), n, static_cast<cudaStream_t>(stream));
    KS_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    API_END
}
int ks_dotc(const ks_c64* x, const ks_c64* y, size_t n, ks_c64* out, void* stream) {
    API_BEGIN
    KS_REQUIRE(out, KS_EINVAL, "ks_dotc: NULL out");
    Reducer red;
    launch_dotc(red, reinterpret_cast<const double2*>(x), reinterpret_cast<const double2*>(y), n,
                static_cast<cudaStream_t>(stream));
    fetch(red, static_cast<cudaStream_t>(stream), 2);
    out->re = red.host[0];
    out->im = red.host[1];
    API_END
}
int ks_norm2sq(const ks_c64* x, size_t n, double* out, void* stream) {
    API_BEGIN
    KS_REQUIRE(out, KS_EINVAL, "ks_norm2sq: NULL out");
    Reducer red;
    launch_norm2sq(red, reinterpret_cast<const double2*>(x), n, static_cast<cudaStream_t>(stream));
    fetch(red, static_cast<cudaStream_t>(stream), 1);
    *out = red.host[0];
    API_END
}

// PCG building blocks on device vectors (for the sharded PCG, dist.py)
int ks_cg_update(double alpha, const ks_c64* p, const ks_c64* q, ks_c64* x, ks_c64* r, size_t n,
                 double* rr, void* stream) {
    API_BEGIN
    KS_REQUIRE(rr, KS_EINVAL, "ks_cg_update: NULL rr");
    Reducer red;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    launch_cg_update(red, alpha, reinterpret_cast<const double2*>(p), reinterpret_cast<const double2*>(q),
                     reinterpret_cast<double2*>(x), reinterpret_cast<double2*>(r), n, st);
    fetch(red, st, 1);
    *rr = red.host[0];
    API_END
}
int ks_xpby(const ks_c64* z, double beta, ks_c64* p, size_t n, void* stream) {
    API_BEGIN
    launch_xpby(reinterpret_cast<const double2*>(z), beta, reinterpret_cast<double2*>(p), n,
                static_cast<cudaStream_t>(stream));
    KS_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    API_END
}

// ---------------------------------------------------------------------------
// plumbing
// ---------------------------------------------------------------------------
int ks_set_device(int device) {
    API_BEGIN
    ensure_device(device);
    API_END
}
int ks_malloc(void** ptr, size_t bytes) {
    API_BEGIN
    KS_REQUIRE(ptr, KS_EINVAL, "ks_malloc: NULL");
    KS_CUDA(cudaMalloc(ptr, bytes));
    API_END
}
int ks_free(void* ptr) {
    API_BEGIN
    KS_CUDA(cudaFree(ptr));
    API_END
}
int ks_memcpy(void* dst, const void* src, size_t bytes, int kind) {
    API_BEGIN
    const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                                       : (kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
    KS_CUDA(cudaMemcpy(dst, src, bytes, k));
    API_END
}
int ks_host_alloc(void** ptr, size_t bytes) {
    API_BEGIN
    KS_CUDA(cudaMallocHost(ptr, bytes));
    API_END
}
int ks_host_free(void* ptr) {
    API_BEGIN
    KS_CUDA(cudaFreeHost(ptr));
    API_END
}
int ks_stream_create(void** stream) {
    API_BEGIN
    KS_REQUIRE(stream, KS_EINVAL, "ks_stream_create: NULL argument");
    cudaStream_t st;
    KS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    *stream = st;
    API_END
}
int ks_stream_destroy(void* stream) {
    API_BEGIN
    if (stream) KS_CUDA(cudaStreamDestroy(static_cast<cudaStream_t>(stream)));
    API_END
}
int ks_stream_synchronize(void* stream) {
    API_BEGIN
    KS_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    API_END
}
int ks_synchronize(void) {
    API_BEGIN
    KS_CUDA(cudaDeviceSynchronize());
    API_END
}

static DevBuf& flush_buf() {
    static DevBuf b;
    return b;
}
int ks_flush_l2(size_t bytes) {
    API_BEGIN
    DevBuf& b = flush_buf();
    if (b.bytes < bytes) b.alloc(bytes);
    launch_fill_bytes(b.p, bytes, nullptr);
    API_END
}

int ks_fd_time(ks_fd* fd, const ks_c64* r, ks_c64* z, int iters, int flush, double* ms_out,
               double* ms_kernel) {
    double kinds[3] = {0, 0, 0};
    int nl[3] = {0, 0, 0};
    const int rc = ks_fd_profile(fd, r, z, iters, flush, ms_out, kinds, nl);
    if (rc == KS_OK && ms_kernel) *ms_kernel = kinds[0];
    return rc;
}

int ks_fd_profile(ks_fd* fd, const ks_c64* r, ks_c64* z, int iters, int flush, double* ms_out, double* ms_kind,
                  int* launches_kind) {
    API_BEGIN
    KS_REQUIRE(fd && r && z && iters > 0, KS_EINVAL, "ks_fd_time: bad arguments");
    std::lock_guard<std::mutex> lk(fd->mu);
    ensure_device(fd->device);
    cudaStream_t st = fd->stream;
    KS_CUDA(cudaStreamWaitEvent(st, fd->done, 0));
    DevBuf& fb = flush_buf();
    const size_t fbytes = (size_t)256 << 20;
    if (flush && fb.bytes < fbytes) fb.alloc(fbytes);
    cudaEvent_t a, b;
    KS_CUDA(cudaEventCreate(&a));
    KS_CUDA(cudaEventCreate(&b));
    double tot = 0, ker[3] = {0, 0, 0};
    int nl[3] = {0, 0, 0};
    for (int it = 0; it < iters; ++it) {
        if (flush) launch_fill_bytes(fb.p, fbytes, st);
        FdTimes ev;
        KS_CUDA(cudaEventRecord(a, st));
        fd_apply_dev(fd, reinterpret_cast<const double2*>(r), reinterpret_cast<double2*>(z), false, st, &ev);
        KS_CUDA(cudaEventRecord(b, st));
        KS_CUDA(cudaEventSynchronize(b));
        tot += elapsed(a, b);
        for (size_t e = 0; e < ev.kind.size(); ++e) {
            ker[ev.kind[e]] += elapsed(ev.ev[2 * e], ev.ev[2 * e + 1]);
            if (it == 0) ++nl[ev.kind[e]];
        }
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    KS_CUDA(cudaEventRecord(fd->done, st));
    if (ms_out) *ms_out = tot / iters;
    for (int k = 0; k < 3; ++k) {
        if (ms_kind) ms_kind[k] = ker[k] / iters;
        if (launches_kind) launches_kind[k] = nl[k];
    }
    API_END
}

int ks_fd_latency(ks_fd* fd, const ks_c64* r, ks_c64* z, int iters, int graph, double* ms_out) {
    API_BEGIN
    KS_REQUIRE(fd && r && z && iters > 0 && ms_out, KS_EINVAL, "ks_fd_latency: bad arguments");
    std::lock_guard<std::mutex> lk(fd->mu);
    ensure_device(fd->device);
    cudaStream_t st = fd->stream;
    KS_CUDA(cudaStreamWaitEvent(st, fd->done, 0));
    const double2* rd = reinterpret_cast<const double2*>(r);
    double2* zd = reinterpret_cast<double2*>(z);
    fd_apply_dev(fd, rd, zd, false, st, nullptr); // warm-up (lazy module loading)
    cudaGraphExec_t ge = nullptr;
    if (graph) {
        cudaGraph_t g = nullptr;
        KS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
            fd_apply_dev(fd, rd, zd, false, st, nullptr);
        } catch (...) {
            cudaStreamEndCapture(st, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        KS_CUDA(cudaStreamEndCapture(st, &g));
        const cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
        cudaGraphDestroy(g);
        KS_CUDA(e);
        KS_CUDA(cudaGraphLaunch(ge, st)); // warm-up replay
    }
    cudaEvent_t a, b;
    KS_CUDA(cudaEventCreate(&a));
    KS_CUDA(cudaEventCreate(&b));
    KS_CUDA(cudaEventRecord(a, st));
    for (int it = 0; it < iters; ++it) {
        if (ge) KS_CUDA(cudaGraphLaunch(ge, st));
        else fd_apply_dev(fd, rd, zd, false, st, nullptr);
    }
    KS_CUDA(cudaEventRecord(b, st));
    KS_CUDA(cudaEventSynchronize(b));
    *ms_out = elapsed(a, b) / iters;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (ge) cudaGraphExecDestroy(ge);
    KS_CUDA(cudaEventRecord(fd->done, st));
    API_END
}

int ks_kron_time(ks_kron* k, const ks_c64* x, ks_c64* y, int iters, int flush, double* ms_out) {
    API_BEGIN
    KS_REQUIRE(k && x && y && iters > 0, KS_EINVAL, "ks_kron_time: bad arguments");
    std::lock_guard<std::mutex> lk(k->mu);
    ensure_device(k->device);
    cudaStream_t st = k->stream;
    KS_CUDA(cudaStreamWaitEvent(st, k->done, 0));
    DevBuf& fb = flush_buf();
    const size_t fbytes = (size_t)256 << 20;
    if (flush && fb.bytes < fbytes) fb.alloc(fbytes);
    cudaEvent_t a, b;
    KS_CUDA(cudaEventCreate(&a));
    KS_CUDA(cudaEventCreate(&b));
    double tot = 0;
    for (int it = 0; it < iters; ++it) {
        if (flush) launch_fill_bytes(fb.p, fbytes, st);
        KS_CUDA(cudaEventRecord(a, st));
        kron_apply(*k->plan, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y), st,
                   k->hptrs);
        KS_CUDA(cudaEventRecord(b, st));
        KS_CUDA(cudaEventSynchronize(b));
        tot += elapsed(a, b);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (ms_out) *ms_out = tot / iters;
    API_END
}

int ks_fp64_peak(double* tflops) {
    API_BEGIN
    KS_REQUIRE(tflops, KS_EINVAL, "ks_fp64_peak: NULL");
    int dev = 0;
    KS_CUDA(cudaGetDevice(&dev));
    ensure_device(dev);
    fp64_peak_bench(tflops);
    API_END
}

int ks_transform_engine(void) { return transform_engine(); }

} // extern "C"
