// BLAS-1 and PCG vector kernels on complex FP64 device vectors.
//
// Mirrors the reference backend table kernels::Backend
// (include/kronschro/kernels.hpp:13-23; scalar definitions src/kernels.cpp:10-34):
//   axpy_real: y += a x (real a)      axpy: y += a x (complex a)
//   dotc: sum conj(x_i) y_i           norm2sq: sum |x_i|^2
// and fuses the PCG updates of src/krylov.cpp:73-78 and :109-110.
//
// Reductions are deterministic: a fixed grid of Reducer::kBlocks blocks each
// reduces a fixed strided subset (grid-stride, fixed tree inside the block),
// and the last block to finish sums the per-block partials in index order.
// No floating-point atomics: the same input gives the same bits every call.
// These kernels are HBM-bound (16-48 B per element, no reuse); they use
// 128-bit loads of one complex per thread per step.
#include "ks_internal.hpp"

namespace ks {

namespace {

constexpr int kB = Reducer::kBlocks;
constexpr int kT = Reducer::kThreads;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// reduce up to 3 values per thread over the block; thread 0 returns the sums
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*sh)[kT / 32]) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double s = warp_sum(v[k]);
        if (lane == 0) sh[k][w] = s;
    }
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = lane < kT / 32 ? sh[k][lane] : 0.0;
            v[k] = warp_sum(s);
        }
    }
}

// Last-block finalisation: partial[b*NV + k] written by every block; the block
// that observes counter == gridDim-1 sums them in index order.
template <int NV>
__device__ __forceinline__ void finish(double (&v)[NV], double* partial, unsigned* counter,
                                       double* result) {
    __shared__ double sh[NV][kT / 32];
    __shared__ bool last;
    block_sum<NV>(v, sh);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) partial[blockIdx.x * NV + k] = v[k];
        __threadfence();
        unsigned t = atomicAdd(counter, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // fixed-order sum of partials: thread t takes blocks t, t+kT, ...
    double acc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kT) {
#pragma unroll
        for (int k = 0; k < NV; ++k) acc[k] += ((volatile double*)partial)[b * NV + k];
    }
    __syncthreads();
    block_sum<NV>(acc, sh);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) result[k] = acc[k];
        *counter = 0u; // re-arm for the next launch on this stream
    }
}

__global__ void __launch_bounds__(kT) k_dotc(const double2* __restrict__ x,
                                             const double2* __restrict__ y, size_t n,
                                             double* partial, unsigned* counter, double* result) {
    double v[2] = {0.0, 0.0};
    for (size_t i = blockIdx.x * (size_t)kT + threadIdx.x; i < n; i += (size_t)gridDim.x * kT) {
        const double2 a = __ldg(x + i), b = __ldg(y + i);
        v[0] += a.x * b.x + a.y * b.y;
        v[1] += a.x * b.y - a.y * b.x;
    }
    finish<2>(v, partial, counter, result);
}

__global__ void __launch_bounds__(kT) k_norm2sq(const double2* __restrict__ x, size_t n,
                                                double* partial, unsigned* counter,
                                                double* result) {
    double v[1] = {0.0};
    for (size_t i = blockIdx.x * (size_t)kT + threadIdx.x; i < n; i += (size_t)gridDim.x * kT) {
        const double2 a = __ldg(x + i);
        v[0] += a.x * a.x + a.y * a.y;
    }
    finish<1>(v, partial, counter, result);
}

__global__ void __launch_bounds__(kT) k_cg_update(double alpha, const double2* __restrict__ p,
                                                  const double2* __restrict__ q,
                                                  double2* __restrict__ x, double2* __restrict__ r,
                                                  size_t n, double* partial, unsigned* counter,
                                                  double* result) {
    double v[1] = {0.0};
    for (size_t i = blockIdx.x * (size_t)kT + threadIdx.x; i < n; i += (size_t)gridDim.x * kT) {
        const double2 pi = __ldg(p + i), qi = __ldg(q + i);
        double2 xi = x[i], ri = r[i];
        xi.x += alpha * pi.x;
        xi.y += alpha * pi.y;
        ri.x += -alpha * qi.x;
        ri.y += -alpha * qi.y;
        x[i] = xi;
        r[i] = ri;
        v[0] += ri.x * ri.x + ri.y * ri.y;
    }
    finish<1>(v, partial, counter, result);
}

// Device-scalar variant: alpha = rho / curv read from the reducers' results
// (same double division as krylov.cpp:73); curv <= 0 (breakdown,
// krylov.cpp:68-72) leaves x and r untouched so the host can stop exactly
// where the reference does.
__global__ void __launch_bounds__(kT) k_cg_update_dev(const double* __restrict__ rho, const double* __restrict__ curv,
                                                      const double2* __restrict__ p, const double2* __restrict__ q,
                                                      double2* __restrict__ x, double2* __restrict__ r, size_t n,
                                                      double* partial, unsigned* counter, double* result) {
    const double c = *curv;
    const bool live = c > 0.0;
    const double alpha = live ? *rho / c : 0.0;
    double v[1] = {0.0};
    for (size_t i = blockIdx.x * (size_t)kT + threadIdx.x; i < n; i += (size_t)gridDim.x * kT) {
        double2 ri = r[i];
        if (live) {
            const double2 pi = __ldg(p + i), qi = __ldg(q + i);
            double2 xi = x[i];
            xi.x += alpha * pi.x;
            xi.y += alpha * pi.y;
            ri.x += -alpha * qi.x;
            ri.y += -alpha * qi.y;
            x[i] = xi;
            r[i] = ri;
        }
        v[0] += ri.x * ri.x + ri.y * ri.y;
    }
    finish<1>(v, partial, counter, result);
}

// Deferred-x variant: the same r update and ||r||^2, x left for the p update
// (x += alpha p_k is applied by k_xpby_x_dev, which reads p_k anyway, or by
// k_x_update_dev before a true residual / at exit): 48 instead of 96 B per
// element here, +32 B there -- the iterates are bit-identical.
__global__ void __launch_bounds__(kT) k_cg_update_r_dev(const double* __restrict__ rho, const double* __restrict__ curv,
                                                        const double2* __restrict__ q, double2* __restrict__ r, size_t n,
                                                        double* partial, unsigned* counter, double* result) {
    const double c = *curv;
    const bool live = c > 0.0;
    const double alpha = live ? *rho / c : 0.0;
    double v[1] = {0.0};
    for (size_t i = blockIdx.x * (size_t)kT + threadIdx.x; i < n; i += (size_t)gridDim.x * kT) {
        double2 ri = r[i];
        if (live) {
            const double2 qi = __ldg(q + i);
            ri.x += -alpha * qi.x;
            ri.y += -alpha * qi.y;
            r[i] = ri;
        }
        v[0] += ri.x * ri.x + ri.y * ri.y;
    }
    finish<1>(v, partial, counter, result);
}

// x += alpha_k p_k (alpha_k = rho_old / curv, krylov.cpp:73-75) and
// p = z + (rho_new / rho_old) p_k (krylov.cpp:105-110) in one pass
__global__ void k_xpby_x_dev(const double2* __restrict__ z, const double* __restrict__ rho_new,
                             const double* __restrict__ rho_old, const double* __restrict__ curv,
                             double2* __restrict__ p, double2* __restrict__ x, size_t n) {
    const double beta = *rho_new / *rho_old, alpha = *rho_old / *curv;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const double2 zi = __ldg(z + i);
        double2 pi = p[i], xi = x[i];
        xi.x += alpha * pi.x;
        xi.y += alpha * pi.y;
        pi.x = zi.x + beta * pi.x;
        pi.y = zi.y + beta * pi.y;
        x[i] = xi;
        p[i] = pi;
    }
}

__global__ void k_x_update_dev(const double* __restrict__ rho, const double* __restrict__ curv,
                               const double2* __restrict__ p, double2* __restrict__ x, size_t n) {
    const double alpha = *rho / *curv;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const double2 pi = __ldg(p + i);
        double2 xi = x[i];
        xi.x += alpha * pi.x;
        xi.y += alpha * pi.y;
        x[i] = xi;
    }
}

// p = z + (rho_new / rho_old) p  (krylov.cpp:105-110), beta formed on the device
__global__ void k_xpby_dev(const double2* __restrict__ z, const double* __restrict__ rho_new,
                           const double* __restrict__ rho_old, double2* __restrict__ p, size_t n) {
    const double beta = *rho_new / *rho_old;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const double2 zi = __ldg(z + i);
        double2 pi = p[i];
        pi.x = zi.x + beta * pi.x;
        pi.y = zi.y + beta * pi.y;
        p[i] = pi;
    }
}

__global__ void k_xpby(const double2* __restrict__ z, double beta, double2* __restrict__ p,
                       size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const double2 zi = __ldg(z + i);
        double2 pi = p[i];
        pi.x = zi.x + beta * pi.x;
        pi.y = zi.y + beta * pi.y;
        p[i] = pi;
    }
}

__global__ void k_axpy_real(double a, const double2* __restrict__ x, double2* __restrict__ y,
                            size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const double2 xi = __ldg(x + i);
        double2 yi = y[i];
        yi.x += a * xi.x;
        yi.y += a * xi.y;
        y[i] = yi;
    }
}

__global__ void k_axpy(double2 a, const double2* __restrict__ x, double2* __restrict__ y,
                       size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const double2 xi = __ldg(x + i);
        double2 yi = y[i];
        yi.x += a.x * xi.x - a.y * xi.y;
        yi.y += a.x * xi.y + a.y * xi.x;
        y[i] = yi;
    }
}

__global__ void k_neg_copy(const double2* __restrict__ x, double2* __restrict__ y, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const double2 xi = __ldg(x + i);
        y[i] = make_double2(-xi.x, -xi.y);
    }
}

__global__ void k_fill(uint4* p, size_t n16, unsigned v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16;
         i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(v, i, v ^ 0x5a5a5a5au, (unsigned)(i >> 7));
}

inline unsigned ew_blocks(size_t n) {
    size_t b = (n + 255) / 256;
    const size_t cap = 148 * 16;
    return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

} // namespace

Reducer::Reducer() : partial(kBlocks * 3 * sizeof(double)), counter(sizeof(unsigned)),
                     result(3 * sizeof(double)) {
    KS_CUDA(cudaMemset(counter.p, 0, sizeof(unsigned)));
    KS_CUDA(cudaMallocHost(&host, 3 * sizeof(double)));
}
Reducer::~Reducer() {
    if (host) cudaFreeHost(host);
}

void launch_dotc(Reducer& r, const double2* x, const double2* y, size_t n, cudaStream_t s) {
    k_dotc<<<kB, kT, 0, s>>>(x, y, n, r.partial.as<double>(), r.counter.as<unsigned>(),
                             r.result.as<double>());
    check_launch("k_dotc");
}
void launch_norm2sq(Reducer& r, const double2* x, size_t n, cudaStream_t s) {
    k_norm2sq<<<kB, kT, 0, s>>>(x, n, r.partial.as<double>(), r.counter.as<unsigned>(),
                                r.result.as<double>());
    check_launch("k_norm2sq");
}
void launch_cg_update(Reducer& red, double alpha, const double2* p, const double2* q,
                      double2* x, double2* r, size_t n, cudaStream_t s) {
    k_cg_update<<<kB, kT, 0, s>>>(alpha, p, q, x, r, n, red.partial.as<double>(),
                                  red.counter.as<unsigned>(), red.result.as<double>());
    check_launch("k_cg_update");
}
void launch_cg_update_dev(Reducer& red, const double* rho, const double* curv, const double2* p, const double2* q,
                          double2* x, double2* r, size_t n, cudaStream_t s) {
    k_cg_update_dev<<<kB, kT, 0, s>>>(rho, curv, p, q, x, r, n, red.partial.as<double>(), red.counter.as<unsigned>(),
                                      red.result.as<double>());
    check_launch("k_cg_update_dev");
}
void launch_cg_update_r_dev(Reducer& red, const double* rho, const double* curv, const double2* q, double2* r,
                            size_t n, cudaStream_t s) {
    k_cg_update_r_dev<<<kB, kT, 0, s>>>(rho, curv, q, r, n, red.partial.as<double>(), red.counter.as<unsigned>(),
                                        red.result.as<double>());
    check_launch("k_cg_update_r_dev");
}
void launch_xpby_x_dev(const double2* z, const double* rho_new, const double* rho_old, const double* curv,
                       double2* p, double2* x, size_t n, cudaStream_t s) {
    k_xpby_x_dev<<<ew_blocks(n), 256, 0, s>>>(z, rho_new, rho_old, curv, p, x, n);
    check_launch("k_xpby_x_dev");
}
void launch_x_update_dev(const double* rho, const double* curv, const double2* p, double2* x, size_t n,
                         cudaStream_t s) {
    k_x_update_dev<<<ew_blocks(n), 256, 0, s>>>(rho, curv, p, x, n);
    check_launch("k_x_update_dev");
}
void launch_xpby_dev(const double2* z, const double* rho_new, const double* rho_old, double2* p, size_t n,
                     cudaStream_t s) {
    k_xpby_dev<<<ew_blocks(n), 256, 0, s>>>(z, rho_new, rho_old, p, n);
    check_launch("k_xpby_dev");
}
void launch_xpby(const double2* z, double beta, double2* p, size_t n, cudaStream_t s) {
    k_xpby<<<ew_blocks(n), 256, 0, s>>>(z, beta, p, n);
    check_launch("k_xpby");
}
void launch_axpy_real(double a, const double2* x, double2* y, size_t n, cudaStream_t s) {
    k_axpy_real<<<ew_blocks(n), 256, 0, s>>>(a, x, y, n);
    check_launch("k_axpy_real");
}
void launch_axpy(double2 a, const double2* x, double2* y, size_t n, cudaStream_t s) {
    k_axpy<<<ew_blocks(n), 256, 0, s>>>(a, x, y, n);
    check_launch("k_axpy");
}
void launch_neg_copy(const double2* x, double2* y, size_t n, cudaStream_t s) {
    k_neg_copy<<<ew_blocks(n), 256, 0, s>>>(x, y, n);
    check_launch("k_neg_copy");
}
void launch_fill_bytes(void* p, size_t bytes, cudaStream_t s) {
    static unsigned salt = 1;
    k_fill<<<148 * 8, 256, 0, s>>>(static_cast<uint4*>(p), bytes / 16, salt++);
    check_launch("k_fill");
}
void fetch(Reducer& r, cudaStream_t s, int count) {
    KS_CUDA(cudaMemcpyAsync(r.host, r.result.p, count * sizeof(double), cudaMemcpyDeviceToHost, s));
    KS_CUDA(cudaStreamSynchronize(s));
}

} // namespace ks
