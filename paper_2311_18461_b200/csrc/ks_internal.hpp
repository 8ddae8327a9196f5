// Internal declarations shared by the libks translation units.
// Nothing here crosses the C-ABI (include/ks.h).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <array>
#include <vector>

#include "../../include/ks.h"

struct ks_comm;
struct ks_fdshard;

namespace ks {

// ---------------------------------------------------------------------------
// errors: one exception type carrying a ks_status; the API wrappers turn it
// into a return code + thread-local message.
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define KS_CUDA(expr)                                                          \
    do {                                                                       \
        cudaError_t e_ = (expr);                                               \
        if (e_ != cudaSuccess)                                                 \
            throw ::ks::Error(e_ == cudaErrorMemoryAllocation ? KS_ENOMEM      \
                                                              : KS_ECUDA,      \
                              std::string(#expr) + ": " +                      \
                                  cudaGetErrorString(e_));                     \
    } while (0)

#define KS_REQUIRE(cond, code, msg)                                            \
    do {                                                                       \
        if (!(cond))                                                           \
            throw ::ks::Error((code), (msg));                                  \
    } while (0)

// counts every kernel this library launches (ks_launch_count)
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
inline void check_launch(const char* what) {
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw Error(KS_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    explicit DevBuf(size_t b) { alloc(b); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t b) {
        release();
        if (b == 0) return;
        KS_CUDA(cudaMalloc(&p, b));
        bytes = b;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T> T* as() const { return static_cast<T*>(p); }
};

void ensure_device(int device);

// NCCL communicator (ks_comm.cu): grouped point-to-point in doubles, in-place sum
int comm_rank(const ks_comm* c);
int comm_size(const ks_comm* c);
void comm_group_start();
void comm_group_end();
void comm_send(const void* buf, size_t doubles, int peer, ks_comm* c, cudaStream_t st);
void comm_recv(void* buf, size_t doubles, int peer, ks_comm* c, cudaStream_t st);
void comm_allreduce_sum(double* buf, size_t count, ks_comm* c, cudaStream_t st);
// sharded FD apply over a communicator (ks_shard.cu), device pointers, stream-ordered
void fdshard_apply_comm(ks_fdshard* h, ks_comm* c, const double2* r_slab, double2* z_slab, cudaStream_t st);
size_t fdshard_slab_n(const ks_fdshard* h);
int fdshard_device(const ks_fdshard* h);
// Opt `func` into `bytes` of dynamic shared memory on the CURRENT device. The
// attribute is per device, so the cache is keyed by (device, function): a
// handle on a second GPU in the same process gets its own opt-in.
void smem_optin(const void* func, int bytes);
// SM count of the current device (cached per device)
int device_sms();

// ---------------------------------------------------------------------------
// reductions / BLAS-1 (ks_blas.cu). Deterministic: fixed grid, fixed tree.
// ---------------------------------------------------------------------------
struct Reducer {
    static constexpr int kBlocks = 592;   // 4 x 148 SMs
    static constexpr int kThreads = 256;
    DevBuf partial;   // kBlocks x 3 doubles
    DevBuf counter;   // unsigned int, last-block detection
    DevBuf result;    // 3 doubles
    double* host = nullptr; // pinned, 3 doubles
    Reducer();
    ~Reducer();
    Reducer(const Reducer&) = delete;
    Reducer& operator=(const Reducer&) = delete;
};

// device-side reductions; results land in r.result (device) and, after
// fetch(), in r.host.
void launch_dotc(Reducer& r, const double2* x, const double2* y, size_t n, cudaStream_t s);
void launch_norm2sq(Reducer& r, const double2* x, size_t n, cudaStream_t s);
// x += a p ; r -= a q ; result[0] = ||r||^2   (krylov.cpp:73-78)
void launch_cg_update(Reducer& red, double alpha, const double2* p, const double2* q,
                      double2* x, double2* r, size_t n, cudaStream_t s);
// device-scalar forms (no host round trip): alpha = *rho / *curv (no update
// when *curv <= 0), beta = *rho_new / *rho_old
void launch_cg_update_dev(Reducer& red, const double* rho, const double* curv, const double2* p, const double2* q,
                          double2* x, double2* r, size_t n, cudaStream_t s);
// deferred solution update (PCG): r -= alpha q and ||r||^2 only (x untouched) ...
void launch_cg_update_r_dev(Reducer& red, const double* rho, const double* curv, const double2* q, double2* r,
                            size_t n, cudaStream_t s);
// ... then x += alpha p_k fused into p = z + beta p_k (one pass over p), or alone
void launch_xpby_x_dev(const double2* z, const double* rho_new, const double* rho_old, const double* curv,
                       double2* p, double2* x, size_t n, cudaStream_t s);
void launch_x_update_dev(const double* rho, const double* curv, const double2* p, double2* x, size_t n,
                         cudaStream_t s);
void launch_xpby_dev(const double2* z, const double* rho_new, const double* rho_old, double2* p, size_t n,
                     cudaStream_t s);
// p = z + beta p   (krylov.cpp:109-110)
void launch_xpby(const double2* z, double beta, double2* p, size_t n, cudaStream_t s);
// y = a*x + y (real a)
void launch_axpy_real(double a, const double2* x, double2* y, size_t n, cudaStream_t s);
void launch_axpy(double2 a, const double2* x, double2* y, size_t n, cudaStream_t s);
// y = -x
void launch_neg_copy(const double2* x, double2* y, size_t n, cudaStream_t s);
void fetch(Reducer& r, cudaStream_t s, int count);
void launch_fill_bytes(void* p, size_t bytes, cudaStream_t s);

// ---------------------------------------------------------------------------
// dense mode product with a real n x n matrix (ks_transform.cu)
//   Y[o][r][q] = sum_j A[r][j] X[o][j][q],  q over 2*s doubles
// At is A stored k-major: At[j*n + r] = A[r][j].
// ---------------------------------------------------------------------------
// layout: 0 natural in/out; 1 natural in -> time-major out T[t][i];
//         2 time-major in -> natural out (1/2 need outer == 1; nt = time extent);
//         3 / 4: the same hand-off on axis 1 (folded axes only, rows stored by
//         position: FoldAxis::perm)
// rows_in / rows_out (optional, device arrays of n pointers): row j of the input
// / output is at rows_*[j] + column offset (rows on other GPUs, peer memory)
void launch_mode_gemm(const double* At, int n, const double* X, double* Y,
                      size_t s_complex, size_t outer, cudaStream_t st, int layout = 0, int nt = 0,
                      const double* const* rows_in = nullptr, double* const* rows_out = nullptr);

// folded (even/odd) transform of one axis whose eigenvectors are all even or
// odd to relative tolerance tol (centro-symmetric pencils): two half-size
// GEMMs instead of one (ks_transform.cu)
struct FoldAxis {
    int n = 0, hc = 0, th = 0; // hc = ceil(n/2) even eigenvectors; tile height 16*th >= hc
    int kst = 0;               // stored k rows of each half matrix (zero padded)
    DevBuf fwd, inv;           // [2][Kp][16*th] symmetrised half matrices (even, odd), k-major
    DevBuf rmap;               // int [2][16*th]: even eigen-indices, odd eigen-indices
    DevBuf rpos;               // int [2][16*th]: positions 0..hc-1, hc..n-1 (axis-1 time-major rows)
    std::vector<int> perm;     // eigen-index stored at position p of the axis-1 time-major layout
};
// U column-major (U[j + r*n] = U(j, r)); false (F untouched) if not foldable
// or KS_FD_FOLD=0
// lam: the axis eigenvalues (near-degenerate pairs are re-combined into even/odd)
bool fold_axis_build(const double* U, const double* lam, int n, double tol, FoldAxis& F);
void launch_mode_gemm_fold(const FoldAxis& F, bool inverse, const double* X, double* Y,
                           size_t s_complex, size_t outer, cudaStream_t st, int layout = 0, int nt = 0,
                           const double* const* rows_in = nullptr, double* const* rows_out = nullptr);

// ---------------------------------------------------------------------------
// plan-specialised fused level passes (ks_kron_jit.cu, NVRTC at plan creation)
// ---------------------------------------------------------------------------
// NVRTC for sm_100a, cached by source (ks_kron_jit.cu)
cudaKernel_t nvrtc_kernel(const std::string& src, const char* name, size_t max_smem);
struct JitContrib {
    int in, out, factor, coeff; // coeff = index into the coefficient table
};
struct KronJitPair;
// fused passes over tensors [n_outer][n_b][n_a][s_a] (axis a then axis b);
// null when the shape is unsupported or KS_KRON_JIT=0
KronJitPair* kron_jit_build(int nin, int nmid, int nout, int bw, const std::vector<JitContrib>& a,
                            const std::vector<JitContrib>& b, const std::vector<int>& freal,
                            const std::vector<double2>& coeffs, long long s_a, int n_a, int n_b, long long n_outer,
                            int tmax_default = 384, int dmax = 4);
// row-blocked variant for s_a > 1 (lanes across the inner columns, R rows of axis a
// per thread, band entries as literals); hrb = host copy of the band table
// rb[f][nmax][2 bw + 1]; null when the factors are not Toeplitz away from the boundary
KronJitPair* kron_jitb_build(int nin, int nmid, int nout, int bw, const std::vector<JitContrib>& a,
                             const std::vector<JitContrib>& b, const std::vector<int>& freal,
                             const std::vector<double2>& coeffs, long long s_a, int n_a, int n_b, long long n_outer,
                             const double2* hrb, int nmax, int R, bool align4 = false, bool shift = false);
// line variant for s_a = 1 (thread per point of C whole lines, planes as tensor-map boxes)
KronJitPair* kron_jitt_build(int nin, int nmid, int nout, int bw, const std::vector<JitContrib>& a,
                             const std::vector<JitContrib>& b, const std::vector<int>& freal,
                             const std::vector<double2>& coeffs, int n_a, int n_b, long long n_outer,
                             const double2* hrb, int nmax, int RB, int RA, int RR, int NWARP, int minb, int NAS);
struct KronJitPass;
KronJitPass* kron_jitc_build(int nin, int nout, int bw, const std::vector<JitContrib>& c, const std::vector<int>& freal,
                             const std::vector<double2>& coeffs, long long s_a, int n_a, long long n_outer,
                             const double2* hrb, int nmax, int RR);
void kron_jitc_launch(const KronJitPass& J, void* const* hin, void* const* hout, cudaStream_t st);
void kron_jitc_free(KronJitPass* p);
const char* kron_jit_tag(const KronJitPair& J);
std::vector<std::array<int, 6>> kron_jitt_candidates(int bw, int n_a, int n_b, int na_prod, int nb_prod, int nmid, int nout,
                                                     int keep);
bool kron_jit_same_shape(const KronJitPair& A, const KronJitPair& B);
int kron_jit_blocked_rows(const KronJitPair& J); // rows per thread of the row-blocked variant, -(lines per CTA) of the line variant, 0 for thread-per-point
bool kron_jit_launch(const KronJitPair& J, const double2* const* ip, double2* const* op, void* const* hin,
                     void* const* hout, const double2* rb, int nmax, cudaStream_t st);
void kron_jit_free(KronJitPair* p);
bool kron_jit_runs(const KronJitPair& J); // the grid fills the GPU (else the passes run separately)
struct KronJitDeleter {
    void operator()(KronJitPair* p) const { kron_jit_free(p); }
};

// ---------------------------------------------------------------------------
// banded block factor / solve (ks_fdsolve.cu)
// ---------------------------------------------------------------------------
struct FdBlocks {
    int nt = 0, p = 0, ldab = 0;
    size_t ns = 0;      // fibers (= N_s)
    size_t nblk = 0;    // factored blocks (N_s, or fewer when deduplicated)
    int kind = 0;       // 0: H = Lt + nu^2 lam^2 Mt + nu lam (W + W^H), HPD -> L D L^H;
                        // 1 (Galerkin): H = W + nu lam Mt -> partial-pivot LU
    // kind 0, group-blocked: blocks b = G * gsz + bl, and for step k
    //   dinv[(G*nt + k)*gsz + bl] = 1/d_k,  v[((G*nt + k)*p + j-1)*gsz + bl] = u(k,k+j)/d_k
    // one group (gsz = nblk, the default) is the plain block-interleaved layout; the
    // fused axis-1 stage uses one group per slab, so a chunk of steps of a slab's
    // fibers is one contiguous run (a single bulk copy)
    DevBuf dinv, v;
    size_t gsz = 0;
    // kind 1, block-interleaved band ab[(k*ldab + e)*nblk + b], pivot offsets piv[k*nblk + b]
    DevBuf ab, piv;
    DevBuf wpiv;        // uint8 per 32 consecutive blocks: some block pivoted (kind 1 pair solve)
    bool nopiv = false; // kind 1: no block pivoted at all
    DevBuf flag;        // int: bit 0 singular / not HPD, bit 1 some row interchange
    DevBuf lam_blk;     // double [nblk] composite eigenvalue of each block
    DevBuf fiber_block; // int [ns] block of each fiber (empty = identity)
    // pair mode (d = 3, axes 2 and 3 identical): block b = i1 + n1 * pidx over
    // pairs (i2 <= i3), solved for fibers (i1, i2, i3) and (i1, i3, i2) together
    int pair_n1 = 0, pair_n2 = 0;
    DevBuf pairs;       // int2 [npairs] (i2, i3)
    // the time bands the blocks were built from (owned by the handle; kept for
    // ks_fd_block's on-demand LU of one kind-0 block)
    double nu = 1.0;
    const double *Lt = nullptr, *Mt = nullptr;
    const double2* Wsym = nullptr;
};
// allocate the factor storage of B.nblk blocks for B.kind
void fd_blocks_alloc(FdBlocks& B);
// the reference's LU of block b (factor_banded layout, eigensolve.hpp:36-42) on the host
void fd_block_to_host(const FdBlocks& B, size_t b, ks_c64* ab, int* piv);
// time bands on device: Lt, Mt real (2p+1)xnt, Wsym complex
void launch_fd_factor(FdBlocks& B, double nu, const double* Lt, const double* Mt,
                      const double2* Wsym, cudaStream_t st);
// block solves on the time-major layout X = T[t][fiber] (stride ns between time steps)
void launch_fd_solve(const FdBlocks& B, double2* X, bool adjoint, cudaStream_t st);

// folded transform on the natural layout with POSITION-ordered eigen rows (even
// eigenvectors first), bulk-copy fed (ks_xform.cu)
bool xfold_supported(const FoldAxis& F);
// mode 0: natural in / out; 1 (axis 1, forward): time-major out T[t][pos + n1*o];
// 2 (axis 1, inverse): time-major in (s_complex = n_t, outer = N_s / n1)
void launch_xfold(const FoldAxis& F, bool inverse, const double* X, double* Y, size_t s_complex, size_t outer,
                  cudaStream_t st, int mode = 0);

// fused axis-1 stage (ks_fdaxis1.cu): forward folded axis-1 transform, L D L^H
// block solves, inverse transform, per (t, i1) slab in shared memory
bool fd_axis1_supported(int n1, int nt, int p);
// the folded axis's se / so halves in the kernel's layout (host array)
void fd_axis1_matrix(const FoldAxis& F, int nt, int p, std::vector<double>& out);
// X, Y natural layout (may alias); slab order[s] is processed by work item s;
// the block of the fiber at axis-1 position m of slab o is m + n1b * grp[o]
// (n1b = n1 rounded up to even: 16 B aligned factor rows for the L2 prefetch)
void launch_fd_axis1(const FoldAxis& F, const double* A, int nt, long long nslab, const int* order,
                     const int* grp, int n1b, const FdBlocks& B, const double* X, double* Y, cudaStream_t st);

// ---------------------------------------------------------------------------
// level-pass Kronecker engine (ks_kron.cu)
// ---------------------------------------------------------------------------
void fp64_peak_bench(double* tflops);

} // namespace ks
