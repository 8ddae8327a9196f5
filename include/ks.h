/*
 * ks.h — C-ABI of the B200 (sm_100a) hot path of the space-time least-squares
 * isogeometric Schroedinger solver (arXiv 2311.18461, reference "kronschro").
 *
 * This is the drop-in boundary. Every entry point replaces one reference C++
 * interface; the reference file:line it stands in for is cited beside it
 * (paths relative to the reference's proj/ directory). Only plain pointers,
 * sizes and POD structs cross it: no torch or C++ types.
 *
 * Conventions shared with the reference:
 *   - complex FP64 is interleaved (re, im): ks_c64 is layout-compatible with
 *     std::complex<double> (include/kronschro/tensorops.hpp:15, kernels_avx2.cpp:10);
 *   - tensors are linearised with axis 0 (time) fastest:
 *     vec index = i_0 + n_0*(i_1 + n_1*(i_2 + ...)) (include/kronschro/tensorops.hpp:15-16);
 *   - banded matrices use the LAPACK-style layout of BandedMatrix<T>: entry
 *     (i,j), |i-j| <= bw, lives at data[bw + i - j + j*(2*bw+1)]
 *     (include/kronschro/banded.hpp:11-13, :91-94);
 *   - dense eigenvector matrices U_l are column-major n_l x n_l, as Eigen's
 *     MatrixXd (include/kronschro/eigensolve.hpp:16-19).
 *
 * Errors: every int-returning call returns KS_OK or a KS_E* code and leaves a
 * thread-local message in ks_last_error(). The C++ wrappers in
 * kronschro_gpu.hpp rethrow the std exception the reference throws
 * (invalid_argument / runtime_error / length_error).
 *
 * There is no CPU fallback: without a CUDA device every compute call returns
 * KS_ECUDA.
 */
#ifndef KS_H_
#define KS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } ks_c64;

enum ks_status {
    KS_OK = 0,
    KS_EINVAL = 1,     /* std::invalid_argument in the reference */
    KS_ESINGULAR = 2,  /* std::runtime_error("factor_banded: numerically singular pivot"), eigensolve.cpp:105-106 */
    KS_ECUDA = 3,      /* CUDA runtime failure / no device */
    KS_ENOMEM = 4,     /* device allocation failed */
    KS_ENCCL = 5,      /* collective failure (multi-GPU) */
    KS_ELENGTH = 6     /* std::length_error (dense caps), tensorops.cpp:279, fdsolver.cpp:138-139 */
};

/* Where the vectors passed to an apply/solve call live. HOST means the call
 * copies in and out (the reference-facing parity path); DEVICE means the
 * pointers are device pointers on the handle's device (the HBM-resident path). */
enum ks_mem { KS_MEM_HOST = 0, KS_MEM_DEVICE = 1 };

const char* ks_last_error(void);
int ks_version(void);
/* Number of visible CUDA devices (0 on a CPU-only host; never throws). */
int ks_device_count(void);

/* ---------------------------------------------------------------------------
 * Fast-diagonalisation preconditioner (Algorithm 1)
 *
 * Replaces  FDPreconditioner(const SpaceTimeProblem&, const UnivariateSet&)
 *           (include/kronschro/fdsolver.hpp:58, src/fdsolver.cpp:124-126)
 * The host keeps the reference's setup: build_univariate (assembly.cpp:146-160)
 * and spatial_eigenbasis/generalized_sym_eig (fdsolver.cpp:23-44,
 * eigensolve.cpp:8-29) produce the inputs below; the N_s block factorisations
 * (fdsolver.cpp:46-51, eigensolve.cpp:77-121) run on the GPU inside create.
 *
 *   d        number of spatial axes (1..3)
 *   dims     d+1 ints: (n_t, n_1, ..., n_d) = SpaceTimeProblem::reduced_dims()
 *   nu       the problem's nu (> 0)
 *   p_t      time bandwidth (= time degree) of Lt, Mt, Wt
 *   U        d pointers, U[l] column-major n_{l+1} x n_{l+1} (M-orthonormal eigenvectors)
 *   lambda   d pointers, lambda[l] of length n_{l+1} (ascending eigenvalues)
 *   Lt, Mt   real time bands, (2*p_t+1) x n_t, BandedMatrix<double> layout
 *   Wt       complex time band (not yet symmetrised), same layout
 * The composite eigenvalues lambda_i = sum_l lambda_l[i_l] (fdsolver.cpp:30-42)
 * and the blocks H_i = Lt + nu^2 lambda_i^2 Mt + nu lambda_i (Wt + Wt^H)
 * (fdsolver.cpp:95-120) are formed on the device.
 * ------------------------------------------------------------------------- */
typedef struct ks_fd ks_fd;

/* Limits: d <= 3, p_t <= 8. Spatial axes up to 160 entries run the folded
 * transforms with U_l resident in shared memory; longer axes (no limit, as in
 * tensorops.cpp:125-156) run a dense panel kernel. */
int ks_fd_create(int d, const int* dims, double nu, int p_t,
                 const double* const* U, const double* const* lambda,
                 const double* Lt, const double* Mt, const ks_c64* Wt,
                 int device, ks_fd** out);
/* z = P^-1 r. Replaces FDPreconditioner::apply(const cplx* r, cplx* z) const
 * (fdsolver.hpp:61 -> FastDiagSolver::solve, fdsolver.cpp:53-63). r and z may
 * alias. stream is a cudaStream_t (NULL = the handle's own stream, blocking).
 * KS_MEM_HOST with a non-NULL stream is asynchronous: the H2D copy, the apply
 * and the D2H copy are queued on the handle's copy/compute streams (three
 * staging buffers, so consecutive applies overlap their transfers). r is read
 * from host memory as soon as the call is made (it must hold its values then,
 * as for the reference's synchronous call); the D2H into z waits until
 * `stream` reaches the call, and z is valid once `stream` is synchronised;
 * r and z must stay untouched (and should be pinned) until then.
 * Applies on one handle are ordered on the device whatever streams they use
 * (the handle's scratch is shared), and a host mutex serialises the calls. */
int ks_fd_apply(ks_fd* fd, const ks_c64* r, ks_c64* z, int mem, void* stream);
/* Same as apply but with the adjoint block solves (FastDiagSolver::solve_adjoint,
 * fdsolver.cpp:65-75, eigensolve.cpp:148-170). */
int ks_fd_apply_adjoint(ks_fd* fd, const ks_c64* r, ks_c64* z, int mem, void* stream);
size_t ks_fd_vec_size(const ks_fd* fd);                 /* fdsolver.hpp:63 */
/* Composite eigenvalues in spatial vec order (fdsolver.hpp:64-66); out has N_s entries. */
int ks_fd_eigenvalues(const ks_fd* fd, double* out);
/* Copy the device-factored block of spatial eigen-index i back to the host in
 * the BandedFactorization layout (eigensolve.hpp:36-42): ab is (3p+1) x n_t
 * complex with ldab = 3p+1, piv has n_t ints. For parity tests. */
int ks_fd_block(const ks_fd* fd, size_t i, ks_c64* ab, int* piv);
/* galerkin_fast_solver(prob, u) (fdsolver.hpp:76-79, fdsolver.cpp:177-191): the
 * same spatial eigenbasis with blocks H_i = Wt + nu lambda_i Mt -- the exact
 * inverse of the Galerkin matrix M_s x W_t - nu sum_l (..G_l^T..) x M_t.
 * Applied with ks_fd_apply (FastDiagSolver::solve) and ks_fd_apply_adjoint
 * (FastDiagSolver::solve_adjoint, fdsolver.cpp:65-75). */
int ks_fd_create_galerkin(int d, const int* dims, double nu, int p_t,
                          const double* const* U, const double* const* lambda,
                          const double* Mt, const ks_c64* Wt, int device, ks_fd** out);
/* Execution plan of a handle (no reference counterpart; diagnostics):
 * folded_axes bit l-1 set = axis l uses the even/odd folded transform
 * (centro-symmetric pencil); blocks = factored time blocks
 * (N_s, or fewer with permutation deduplication); bit 16 set = axes 1 and 2
 * run as one fused folded-transform pass (ks_fold12.cu). Either pointer may
 * be NULL. */
int ks_fd_info(const ks_fd* fd, int* folded_axes, size_t* blocks);
int ks_fd_destroy(ks_fd* fd);

/* ---------------------------------------------------------------------------
 * Kronecker-sum operator (include/kronschro/tensorops.hpp:57-87)
 *
 * Replaces KroneckerOperator(dims) + add_term(coeff, factors) (tensorops.cpp:219-234).
 * A term is coeff * (F_D x ... x F_1 x F_0); factor k acts on tensor axis k;
 * a NULL factor is the identity. Factors are complex square bands of size
 * dims[k] and bandwidth bw[k] (BandedMatrix<cplx> layout).
 * ------------------------------------------------------------------------- */
typedef struct {
    ks_c64 coeff;
    const ks_c64* const* factors; /* ndim pointers, NULL = identity */
    const int* bw;                /* ndim bandwidths (ignored for NULL factors) */
} ks_term;

typedef struct ks_kron ks_kron;

int ks_kron_create(int ndim, const int* dims, int nterms, const ks_term* terms,
                   int device, ks_kron** out);
/* y = K x (tensorops.cpp:236-254). x and y must not alias. */
int ks_kron_apply(ks_kron* k, const ks_c64* x, ks_c64* y, int mem, void* stream);
size_t ks_kron_vec_size(const ks_kron* k);
/* Planner diagnostics: number of fused level passes and intermediate tensors. */
int ks_kron_plan_info(const ks_kron* k, int* npasses, int* nnodes, int* nproducts);
/* Which kernels apply runs (diagnostics): 0 = one launch per level pass,
 * 1 = NVRTC fused pass pairs, 2 = d = 3 two-launch path (axis-3 pass, then
 * axes t/1/2 fused; ks_kron3.cu). */
int ks_kron_engine(const ks_kron* k, int* engine);
int ks_kron_destroy(ks_kron* k);

/* ---------------------------------------------------------------------------
 * Preconditioned CG (include/kronschro/krylov.hpp:11-38, src/krylov.cpp:24-114)
 * Device-resident loop with the reference's control flow: zero initial guess,
 * b = 0 -> converged in 0 iterations, breakdown on Re<p,Ap> <= 0, recurrence
 * residual confirmed by a true residual at exit with <= 2 restarts, strict mode.
 * ------------------------------------------------------------------------- */
typedef struct {
    double tol;           /* PcgOptions::tol (default 1e-8) */
    int maxit;            /* PcgOptions::maxit (default 200) */
    int strict_residual;  /* PcgOptions::strict_residual */
} ks_pcg_opts;

typedef struct {
    int iterations;
    int converged;
    int breakdown;
    int restarts;
    int hist_len;          /* entries written to res_hist (<= hist_cap) */
    double matvec_seconds; /* device time (CUDA events) per component */
    double precond_seconds;
    double solve_seconds;
} ks_pcg_report;

/* P may be NULL (unpreconditioned, krylov.hpp:36). b and x are host or device
 * per mem. res_hist (host, may be NULL) receives up to hist_cap relative
 * residuals, one per iteration (SolveReport::res_history). */
int ks_pcg(ks_kron* A, ks_fd* P, const ks_c64* b, ks_c64* x, int mem,
           const ks_pcg_opts* opts, double* res_hist, int hist_cap,
           ks_pcg_report* report);

/* ---------------------------------------------------------------------------
 * BLAS-1 (include/kronschro/kernels.hpp:13-48) on device vectors. Reductions
 * are deterministic (fixed two-stage tree, no atomics).
 * ------------------------------------------------------------------------- */
int ks_axpy_real(double a, const ks_c64* x, ks_c64* y, size_t n, void* stream);
int ks_axpy(ks_c64 a, const ks_c64* x, ks_c64* y, size_t n, void* stream);
int ks_dotc(const ks_c64* x, const ks_c64* y, size_t n, ks_c64* out, void* stream);
int ks_norm2sq(const ks_c64* x, size_t n, double* out, void* stream);

/* ---------------------------------------------------------------------------
 * Device memory / timing helpers (plumbing for the bench and tests)
 * ------------------------------------------------------------------------- */
int ks_set_device(int device);
int ks_malloc(void** ptr, size_t bytes);
int ks_free(void* ptr);
/* kind: 0 = host->device, 1 = device->host, 2 = device->device */
int ks_memcpy(void* dst, const void* src, size_t bytes, int kind);
int ks_host_alloc(void** ptr, size_t bytes); /* pinned host memory */
int ks_host_free(void* ptr);
int ks_synchronize(void);
/* streams for asynchronous applies (cudaStream_t behind a void*) */
int ks_stream_create(void** stream);
int ks_stream_destroy(void* stream);
int ks_stream_synchronize(void* stream);
/* Overwrite `bytes` of a device scratch buffer (L2 flush between timed runs). */
int ks_flush_l2(size_t bytes);
/* Time `iters` back-to-back launches of the FD apply / Kron apply on device
 * pointers with CUDA events on the handle's stream; optional per-iteration
 * L2 flush. ms_out receives the average ms per call and ms_kernel the
 * average device time per call of the spatial transform launches. */
int ks_fd_time(ks_fd* fd, const ks_c64* r, ks_c64* z, int iters, int flush,
               double* ms_out, double* ms_kernel);
int ks_kron_time(ks_kron* k, const ks_c64* x, ks_c64* y, int iters, int flush,
                 double* ms_out);
/* The same as ks_fd_time with the device time split by kernel kind (CUDA events
 * around every launch): ms_kind[0] spatial transforms, [1] the fused axis-1
 * stage, [2] block solves (ms per apply, 3 entries); launches_kind = launches
 * of each kind per apply. */
int ks_fd_profile(ks_fd* fd, const ks_c64* r, ks_c64* z, int iters, int flush, double* ms_out,
                  double* ms_kind, int* launches_kind);
/* Latency of the FD apply (device pointers): `iters` applies back to back on
 * the handle's stream between two CUDA events, either launched eagerly or as
 * replays of one CUDA graph holding a whole apply (graph = 1); ms_out = the
 * average per apply. For the latency-bound small configs (c1, c2). */
int ks_fd_latency(ks_fd* fd, const ks_c64* r, ks_c64* z, int iters, int graph, double* ms_out);
/* Measured FP64 FMA peak (TFLOP/s) of this device, from a DFMA microbenchmark. */
int ks_fp64_peak(double* tflops);
/* Both FP64 peaks: CUDA-core DFMA and tensor-core DMMA (mma.sync m8n8k4 f64). */
int ks_fp64_peaks(double* dfma_tflops, double* dmma_tflops);
/* Combined FP64 throughput with half the warps on DMMA and half on DFMA. */
int ks_fp64_peak_mixed(double* tflops);
/* FP64 tensor-core throughput with the sm_90+ mma.sync m16n8k16 shape. */
int ks_fp64_peak_mma16(double* tflops);
/* Streaming HBM throughput (GB/s) of a kernel that reads `nin` and writes `nout`
 * complex vectors of n entries -- the traffic mixes of the matvec passes (1 in /
 * 3 out, 3 in / 1 out at d = 3), which bound the two-pass matvec. */
int ks_bw_fan(int nin, int nout, size_t n, double* gbs);
/* DMMA (m8n8k4) throughput with `ctas_per_sm` CTAs of `threads` threads per SM. */
int ks_fp64_dmma_occupancy(int ctas_per_sm, int threads, double* tflops);
/* Which engine the spatial transforms use: 0 = DFMA, 1 = DMMA (env KS_GEMM). */
int ks_transform_engine(void);
/* Number of kernels the library launched since the last reset. */
uint64_t ks_launch_count(void);
void ks_launch_count_reset(void);

/* ---------------------------------------------------------------------------
 * Slab-sharded FD preconditioner (multi-GPU); one rank per GPU.
 * Axis d (outermost spatial) is split in contiguous slabs, so every rank owns
 * a contiguous chunk of each vector. The caller runs two all-to-alls
 * (counts from ks_shard_plan, in complex elements; the way back swaps the
 * send/recv roles):
 *   forward(r_slab -> send) ; all_to_all(send -> work) ; middle(work) ;
 *   all_to_all(work -> back) ; backward(back -> z_slab)
 * ks_shard_plan is host-only (no device needed).
 * ------------------------------------------------------------------------- */
typedef struct ks_fdshard ks_fdshard;

int ks_shard_plan(int d, const int* dims, int nranks, int rank, long long* slab_lo,
                  long long* slab_hi, long long* send_counts, long long* send_displs,
                  long long* recv_counts, long long* recv_displs);
int ks_fdshard_create(int d, const int* dims, double nu, int p_t,
                      const double* const* U, const double* const* lambda,
                      const double* Lt, const double* Mt, const ks_c64* Wt,
                      int nranks, int rank, int device, ks_fdshard** out);
/* complex elements of the local slab and of the re-sharded work tensor */
int ks_fdshard_sizes(const ks_fdshard* h, size_t* slab_n, size_t* work_n);
int ks_fdshard_forward(ks_fdshard* h, const ks_c64* r_slab, ks_c64* sendbuf, void* stream);
int ks_fdshard_middle(ks_fdshard* h, ks_c64* work, void* stream);
int ks_fdshard_backward(ks_fdshard* h, const ks_c64* recvbuf, ks_c64* z_slab, void* stream);
/* Peer-memory transport (no all-to-all): phase 1 writes the slab (n_t, N', m)
 * after the axis 1..d-1 transforms into an exported buffer; set_peers gives
 * every rank's exported phase-1 slab and output slab (device pointers valid in
 * this process: own, peer-enabled or CUDA-IPC-opened); the middle phase's
 * axis-d transform then reads its rows straight from the owners' slabs and
 * its inverse writes them straight into the owners' output slabs over
 * NVLink; phase 3 applies the inverse axis 1..d-1 transforms to the rank's
 * output slab. The caller puts a barrier across ranks between the phases. */
int ks_fdshard_forward_slab(ks_fdshard* h, const ks_c64* r_local, ks_c64* slab_out, void* stream);
int ks_fdshard_set_peers(ks_fdshard* h, const ks_c64* const* peer_in, ks_c64* const* peer_out);
int ks_fdshard_middle_peer(ks_fdshard* h, void* stream);
int ks_fdshard_backward_slab(ks_fdshard* h, const ks_c64* slab_in, ks_c64* z_local, void* stream);
/* CUDA IPC handles (64 bytes) for exporting device buffers to other processes */
int ks_ipc_get_handle(const void* dptr, void* handle);
int ks_ipc_open(const void* handle, void** dptr);
int ks_ipc_close(void* dptr);
int ks_fdshard_destroy(ks_fdshard* h);

/* ---------------------------------------------------------------------------
 * NCCL behind the C-ABI (one rank per GPU, one process per rank). Rank 0 calls
 * ks_comm_unique_id and hands the 128 bytes to the other ranks (any channel);
 * every rank then calls ks_comm_create (ncclCommInitRank). libnccl.so.2 is
 * opened at run time; failures return KS_ENCCL.
 * ------------------------------------------------------------------------- */
#define KS_COMM_ID_BYTES 128
typedef struct ks_comm ks_comm;
int ks_comm_unique_id(void* id /* KS_COMM_ID_BYTES */);
int ks_comm_create(int nranks, int rank, const void* id, int device, ks_comm** out);
int ks_comm_destroy(ks_comm* comm);
/* z_slab = P^-1 r_slab for this rank's slab (device pointers): the three phases
 * above with both all-to-alls as grouped ncclSend / ncclRecv (uneven slabs
 * included), stream-ordered on `stream` (NULL: the handle's stream, blocking).
 * The communicator's rank / size must match the shard plan. */
int ks_fdshard_apply(ks_fdshard* h, ks_comm* comm, const ks_c64* r_slab, ks_c64* z_slab, void* stream);

/* Sharded Kronecker operator: same slabs of the outermost axis; the input is
 * the slab plus a halo of bw planes on each side (bw = widest band on that
 * axis; the caller exchanges the halos with the neighbouring ranks):
 * x_ext = x[ext_lo .. ext_hi) planes, y_slab = (K x)[lo .. hi). Destroy with
 * ks_kron_destroy. */
int ks_kronshard_create(int ndim, const int* dims, int nterms, const ks_term* terms,
                        int nranks, int rank, int device, ks_kron** out);
int ks_kronshard_plan(long long nd, int bw, int nranks, int rank, long long* lo, long long* hi,
                      long long* ext_lo, long long* ext_hi); /* host-only */
int ks_kronshard_sizes(const ks_kron* k, long long* lo, long long* hi, long long* ext_lo,
                       long long* ext_hi, size_t* plane_elems);
int ks_kronshard_apply(ks_kron* k, const ks_c64* x_ext, ks_c64* y_slab, void* stream);
/* y_slab = (K x)[slab] from this rank's slab x_slab: the bw-plane halos are
 * exchanged with the neighbouring ranks (grouped ncclSend / ncclRecv) into the
 * handle's extended buffer, then the local apply. Device pointers. */
int ks_kronshard_apply_comm(ks_kron* k, ks_comm* comm, const ks_c64* x_slab, ks_c64* y_slab, void* stream);
/* Slab-sharded pcg (krylov.cpp:24-114): every rank calls it with its slabs of
 * b and x (device or host pointers, `mem`); A from ks_kronshard_create /
 * ks_setup_create_system_sharded, P from ks_fdshard_create (or NULL), both for
 * this rank. Same control flow and device-resident scalars as ks_pcg; the dots
 * are ncclAllReduce'd on the device, one host round trip per iteration. The
 * residual history and flags are identical on every rank. */
int ks_pcg_sharded(ks_kron* A, ks_fdshard* P, ks_comm* comm, const ks_c64* b_slab, ks_c64* x_slab, int mem,
                   const ks_pcg_opts* opts, double* res_hist, int hist_cap, ks_pcg_report* report);
/* PCG building blocks on device vectors (sharded PCG): x += a p, r -= a q,
 * *rr = local ||r||^2; and p = z + beta p. Both synchronise the stream. */
int ks_cg_update(double alpha, const ks_c64* p, const ks_c64* q, ks_c64* x, ks_c64* r, size_t n,
                 double* rr, void* stream);
int ks_xpby(const ks_c64* z, double beta, ks_c64* p, size_t n, void* stream);

/* ---------------------------------------------------------------------------
 * Host setup (product-side mirror of the reference's shared setup; used when
 * no reference process hands over its own setup products)
 *   SpaceTimeProblem::uniform  (assembly.cpp:110-117)
 *   build_univariate           (assembly.cpp:146-160)
 *   generalized_sym_eig        (eigensolve.cpp:8-29)
 *   assemble_system_operator   (assembly.cpp:202-257)
 * ------------------------------------------------------------------------- */
typedef struct ks_setup ks_setup;

/* trial: 0 = initial-condition space (time drops first), 1 = final-condition. */
int ks_setup_create(int d, int p, int n_el, int n_el_time, double T, double nu,
                    int trial, ks_setup** out);
int ks_setup_dims(const ks_setup* s, int* d, int* dims /* d+1 */, int* p);
/* Copy the time bands (Lt, Mt real; Wt complex), each (2p+1) x n_t. */
int ks_setup_time_bands(const ks_setup* s, double* Lt, double* Mt, ks_c64* Wt);
/* Spatial axis l (0-based): M, L, G, V real bands (2p+1) x n_l (any may be NULL). */
int ks_setup_space_bands(const ks_setup* s, int l, double* M, double* L,
                         double* G, double* V);
/* Eigenpairs of (L_l, M_l): U column-major n_l x n_l, lambda ascending. */
int ks_setup_eig(const ks_setup* s, int l, double* U, double* lambda);
int ks_setup_create_fd(const ks_setup* s, int device, ks_fd** out);
/* The system operator A as the reference's term list (assembly.cpp:202-251). */
int ks_setup_create_system(const ks_setup* s, int device, ks_kron** out);
/* galerkin_fast_solver(prob, u) on this setup (fdsolver.cpp:177-191) */
int ks_setup_create_galerkin_fd(const ks_setup* s, int device, ks_fd** out);
/* assemble_galerkin_operator(prob) (assembly.cpp:273-286) */
int ks_setup_create_galerkin_operator(const ks_setup* s, int device, ks_kron** out);
/* The same operator sharded over nranks (ks_kronshard_*). */
int ks_setup_create_system_sharded(const ks_setup* s, int nranks, int rank, int device,
                                   ks_kron** out);
/* unrestricted (full) tensor dims (SpaceTimeProblem::full_dims, assembly.hpp:51) */
int ks_setup_full_dims(const ks_setup* s, int* dims /* d+1 */);
/* element_quadrature(kv, p+1) of axis `axis` (0 = time; bspline.cpp:189-208):
 * *nq nodes; nodes / weights may be NULL to query the size */
int ks_setup_quad_rule(const ks_setup* s, int axis, int* nq, double* nodes, double* weights);
/* KnotVector::greville (bspline.cpp:77-86) of axis `axis`: *n = full basis size */
int ks_setup_greville(const ks_setup* s, int axis, int* n, double* pts);
int ks_setup_destroy(ks_setup* s);

/* ---------------------------------------------------------------------------
 * Right-hand side, lifting and error norms on the device.
 * The caller samples f / u / g at the points; the sum-factorised quadrature
 * contractions, collocation solves, full-space operator and reductions run on
 * the GPU. Quadrature grid: axis a has nq[a] nodes (ks_setup_quad_rule order),
 * axis 0 (time) fastest; the outermost axis is processed in chunks of rows
 * [r0, r1) inside one element (at most p+1 rows), as the reference does.
 * ------------------------------------------------------------------------- */
typedef struct ks_quad ks_quad;
int ks_quad_create(const ks_setup* s, int device, ks_quad** out);
int ks_quad_destroy(ks_quad* q);
int ks_quad_dims(const ks_quad* q, int* nq /* d+1 */, int* chunk, int* full_dims /* d+1 */);
/* assemble_rhs(prob, f) (assembly.cpp:390-404): reset, accumulate the moments
 * of f chunk by chunk (f: raw samples on the chunk grid), then combine and
 * restrict to the reduced space */
/* built-in manufactured solutions ("sinsin": SURVEY 8(d) c2/c4; "traveling_wave_2d":
 * problems.cpp:95-117) sampled on the device: what 0 = u, 1 = f = S u; grid 0 =
 * quadrature rows [r0, r1) of the outermost axis, grid 1 = the full Greville grid.
 * out is a device buffer. */
int ks_quad_sample_named(ks_quad* q, const char* name, int what, int grid, int r0, int r1, ks_c64* out);
int ks_quad_rhs_reset(ks_quad* q);
/* assemble_rhs of a built-in problem's f with every chunk sampled on the device */
int ks_quad_rhs_named(ks_quad* q, const char* name, ks_c64* rhs, int mem);
int ks_quad_rhs_chunk(ks_quad* q, int r0, int r1, const ks_c64* f, int mem);
int ks_quad_rhs_finish(ks_quad* q, ks_c64* rhs /* reduced */, int mem);
/* lift_nonhomogeneous (assembly.cpp:514-570): g sampled on the full Greville
 * grid -> boundary coefficients (full dims; zero on free indices) and the
 * correction restrict(A_full g_h); corrected_rhs = assemble_rhs(f) - correction */
int ks_quad_lift(ks_quad* q, const ks_c64* g_greville, int mem, ks_c64* boundary, ks_c64* correction);
/* extend_with_boundary (assembly.cpp:468-490); boundary may be NULL (zeros) */
int ks_quad_extend(ks_quad* q, const ks_c64* reduced, const ks_c64* boundary, int mem, ks_c64* full);
/* assemble_ultraweak's initial-datum term (assembly.cpp:572-640): rhs += i (u0, B_jt(0) phi_js)
 * for the final-condition trial space (KS_EINVAL otherwise, as the reference's
 * invalid_argument). u0: samples of the initial datum on the spatial quadrature
 * grid (axis 1 fastest, ks_setup_quad_rule nodes), `mem`; rhs: the reduced load
 * vector of f (ks_quad_rhs_*), updated in place, `rhs_mem`. The system operator
 * of the ultraweak pair is the least-squares one (ks_setup_create_system). */
int ks_quad_initial_term(ks_quad* q, const ks_c64* u0, int mem, ks_c64* rhs, int rhs_mem);
/* error_norms (experiments.cpp:73-153): set the full coefficients, then per
 * chunk return sum w |u - u_h|^2 and sum w |f - S u_h|^2 (S u = i u_t - nu lap u);
 * L2 = sqrt(sum l2sq), energy = sqrt(sum l2sq + sum ressq) */
int ks_quad_error_set(ks_quad* q, const ks_c64* full_coeffs, int mem);
int ks_quad_error_chunk(ks_quad* q, int r0, int r1, const ks_c64* u, const ks_c64* f, int mem,
                        double* l2sq, double* ressq);

#ifdef __cplusplus
}
#endif

#endif /* KS_H_ */
