// Slab-sharded FD preconditioner: one rank per GPU, the
// outermost spatial axis d split in contiguous slabs, so every rank owns a
// contiguous chunk of each vector in the reference's vec order.
//
// apply (the caller runs the two all-to-alls, e.g. NCCL via torch.distributed):
//   forward : transforms U_l^T on axes 1..d-1 of the local slab (n_t, N', m_p)
//             (N' = n_1*...*n_{d-1}), then pack block (t, rest in R_q, slab_p)
//             for every destination q into the send buffer (one 2-D copy each)
//   all-to-all #1
//   middle  : the received tensor is (n_t, |R_q|, n_d) in natural order (slabs
//             arrive in rank order and axis d is outermost): transform axis d
//             (time-major out), block solves on the local fibers, inverse
//             transform axis d (time-major in) -- the result, (n_t, |R_q|, n_d),
//             is already the send buffer of the way back (contiguous per slab)
//   all-to-all #2
//   backward: unpack block (t, R_q, slab_p) from every source into the slab,
//             inverse transforms U_l on axes 1..d-1
// Mode products on distinct axes commute, so this equals the
// single-GPU apply up to rounding. Only the ranks' own blocks are factored.
#include "ks_internal.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>

namespace ks {

namespace {

struct Range {
    long long lo, hi;
    long long n() const { return hi - lo; }
};

Range split(long long n, int parts, int k) {
    const long long base = n / parts, rem = n % parts;
    const long long lo = k * base + std::min<long long>(k, rem);
    return {lo, lo + base + (k < rem ? 1 : 0)};
}

struct Plan {
    int d = 0, nranks = 1, rank = 0, nt = 0;
    std::vector<int> dims;
    long long Np = 1;  // prod of spatial dims before axis d
    long long nd = 1;  // extent of axis d
    std::vector<Range> slab, rest; // per rank
    // complex-element counts/displacements of the two exchanges (from this rank's view)
    std::vector<long long> send1, sdisp1, recv1, rdisp1;
};

Plan make_plan(int d, const int* dims, int nranks, int rank) {
    KS_REQUIRE(d >= 2, KS_EINVAL, "sharded FD needs d >= 2 (axis d is split; axes 1..d-1 are re-sharded)");
    KS_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, KS_EINVAL, "bad rank / nranks");
    Plan P;
    P.d = d;
    P.nranks = nranks;
    P.rank = rank;
    P.dims.assign(dims, dims + d + 1);
    P.nt = dims[0];
    for (int l = 1; l < d; ++l) P.Np *= dims[l];
    P.nd = dims[d];
    KS_REQUIRE(P.nd >= nranks && P.Np >= nranks, KS_EINVAL, "more ranks than slabs");
    for (int k = 0; k < nranks; ++k) {
        P.slab.push_back(split(P.nd, nranks, k));
        P.rest.push_back(split(P.Np, nranks, k));
    }
    const long long nt = P.nt;
    long long sd = 0, rd = 0;
    for (int q = 0; q < nranks; ++q) {
        // send: block (t, R_q, slab_rank); recv: block (t, R_rank, slab_q)
        const long long s = nt * P.rest[q].n() * P.slab[rank].n();
        const long long r = nt * P.rest[rank].n() * P.slab[q].n();
        P.send1.push_back(s);
        P.sdisp1.push_back(sd);
        P.recv1.push_back(r);
        P.rdisp1.push_back(rd);
        sd += s;
        rd += r;
    }
    return P;
}

} // namespace

} // namespace ks

using namespace ks;

struct ks_fdshard {
    Plan plan;
    int device = 0;
    ks_fd* local_fd = nullptr;       // transforms on axes 1..d-1 only (dims of the slab)
    std::vector<DevBuf> At_fwd, At_inv; // per axis 1..d
    std::vector<FoldAxis> fold;         // per axis; n == 0: dense transform
    DevBuf rows_in, rows_out;           // peer transport: axis-d row pointer tables (n_d each)
    FdBlocks blocks;                 // blocks of this rank's fibers
    DevBuf Lt, Mt, Wsym;
    DevBuf s0, s1, work2;
    DevBuf csend, cwork, cback;      // ks_fdshard_apply (NCCL) exchange buffers
    cudaStream_t stream = nullptr;
    std::mutex mu;
    ~ks_fdshard() {
        if (stream) cudaStreamDestroy(stream);
    }
};


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

extern "C" {

int ks_shard_plan(int d, const int* dims, int nranks, int rank, long long* slab_lo,
                  long long* slab_hi, long long* send_counts, long long* send_displs,
                  long long* recv_counts, long long* recv_displs) {
    API_BEGIN
    KS_REQUIRE(dims, KS_EINVAL, "ks_shard_plan: NULL dims");
    const Plan P = make_plan(d, dims, nranks, rank);
    if (slab_lo) *slab_lo = P.slab[rank].lo;
    if (slab_hi) *slab_hi = P.slab[rank].hi;
    for (int q = 0; q < nranks; ++q) {
        if (send_counts) send_counts[q] = P.send1[q];
        if (send_displs) send_displs[q] = P.sdisp1[q];
        if (recv_counts) recv_counts[q] = P.recv1[q];
        if (recv_displs) recv_displs[q] = P.rdisp1[q];
    }
    API_END
}

} // extern "C"

namespace ks {
size_t fdshard_slab_n(const ks_fdshard* h) {
    const Plan& P = h->plan;
    return (size_t)P.nt * P.Np * P.slab[P.rank].n();
}
int fdshard_device(const ks_fdshard* h) { return h->device; }
void fdshard_apply_comm(ks_fdshard* h, ks_comm* c, const double2* r, double2* z, cudaStream_t st) {
    const Plan& P = h->plan;
    KS_REQUIRE(comm_size(c) == P.nranks && comm_rank(c) == P.rank, KS_EINVAL,
               "ks_fdshard_apply: communicator does not match the shard plan");
    const size_t slab_n = fdshard_slab_n(h), work_n = (size_t)P.nt * P.rest[P.rank].n() * P.nd;
    if (h->csend.bytes < slab_n * sizeof(double2)) h->csend.alloc(slab_n * sizeof(double2));
    if (h->cback.bytes < slab_n * sizeof(double2)) h->cback.alloc(slab_n * sizeof(double2));
    if (h->cwork.bytes < work_n * sizeof(double2)) h->cwork.alloc(work_n * sizeof(double2));
    auto ok = [](int rc) {
        if (rc != KS_OK) throw Error(rc, ks_last_error());
    };
    double2* sb = h->csend.as<double2>();
    double2* wb = h->cwork.as<double2>();
    double2* bb = h->cback.as<double2>();
    ok(ks_fdshard_forward(h, reinterpret_cast<const ks_c64*>(r), reinterpret_cast<ks_c64*>(sb), st));
    // all-to-all: block q of the send buffer to rank q, block q of the work tensor from rank q
    comm_group_start();
    for (int q = 0; q < P.nranks; ++q) {
        comm_send(sb + P.sdisp1[q], 2 * (size_t)P.send1[q], q, c, st);
        comm_recv(wb + P.rdisp1[q], 2 * (size_t)P.recv1[q], q, c, st);
    }
    comm_group_end();
    ok(ks_fdshard_middle(h, reinterpret_cast<ks_c64*>(wb), st));
    comm_group_start(); // and back
    for (int q = 0; q < P.nranks; ++q) {
        comm_send(wb + P.rdisp1[q], 2 * (size_t)P.recv1[q], q, c, st);
        comm_recv(bb + P.sdisp1[q], 2 * (size_t)P.send1[q], q, c, st);
    }
    comm_group_end();
    ok(ks_fdshard_backward(h, reinterpret_cast<const ks_c64*>(bb), reinterpret_cast<ks_c64*>(z), st));
}
} // namespace ks

extern "C" {

namespace {
// transform of axis l (1-based): folded when the axis' eigenvectors are even/odd
void shard_gemm(const ks_fdshard* h, int l, bool inv, const double* X, double* Y, size_t s, size_t outer,
                cudaStream_t st, int layout, int nt, const double* const* rin = nullptr,
                double* const* rout = nullptr) {
    const FoldAxis& F = h->fold[l - 1];
    if (F.n) launch_mode_gemm_fold(F, inv, X, Y, s, outer, st, layout, nt, rin, rout);
    else launch_mode_gemm((inv ? h->At_inv : h->At_fwd)[l - 1].as<double>(), h->plan.dims[l], X, Y, s, outer, st,
                          layout, nt, rin, rout);
}
} // namespace

int ks_fdshard_create(int d, const int* dims, double nu, int p_t, const double* const* U,
                      const double* const* lambda, const double* Lt, const double* Mt,
                      const ks_c64* Wt, int nranks, int rank, int device, ks_fdshard** out) {
    API_BEGIN
    KS_REQUIRE(out && dims && U && lambda && Lt && Mt && Wt, KS_EINVAL, "ks_fdshard_create: NULL argument");
    KS_REQUIRE(nu > 0 && p_t >= 1 && p_t <= 8, KS_EINVAL, "ks_fdshard_create: bad nu / p_t");
    ensure_device(device);
    std::unique_ptr<ks_fdshard> h(new ks_fdshard());
    h->plan = make_plan(d, dims, nranks, rank);
    h->device = device;
    const Plan& P = h->plan;
    KS_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    for (int l = 0; l < d; ++l) {
        const int n = dims[l + 1];
        std::vector<double> af((size_t)n * n), ai((size_t)n * n);
        for (int j = 0; j < n; ++j)
            for (int r = 0; r < n; ++r) {
                af[(size_t)j * n + r] = U[l][j + (size_t)r * n];
                ai[(size_t)j * n + r] = U[l][r + (size_t)j * n];
            }
        h->At_fwd.emplace_back(af.size() * sizeof(double));
        h->At_inv.emplace_back(ai.size() * sizeof(double));
        KS_CUDA(cudaMemcpy(h->At_fwd.back().p, af.data(), af.size() * sizeof(double), cudaMemcpyHostToDevice));
        KS_CUDA(cudaMemcpy(h->At_inv.back().p, ai.data(), ai.size() * sizeof(double), cudaMemcpyHostToDevice));
        h->fold.emplace_back();
        fold_axis_build(U[l], lambda[l], n, 1e-9, h->fold.back());
    }
    // W + W^H and the time bands
    const int nt = dims[0], ld = 2 * p_t + 1;
    std::vector<double2> ws((size_t)ld * nt, make_double2(0, 0));
    auto wget = [&](int i, int j) -> double2 {
        if (i < 0 || j < 0 || i >= nt || j >= nt || std::abs(i - j) > p_t) return make_double2(0, 0);
        const ks_c64 v = Wt[p_t + i - j + (size_t)j * ld];
        return make_double2(v.re, v.im);
    };
    for (int i = 0; i < nt; ++i)
        for (int j = std::max(0, i - p_t); j <= std::min(nt - 1, i + p_t); ++j) {
            const double2 a = wget(i, j), b = wget(j, i);
            ws[p_t + i - j + (size_t)j * ld] = make_double2(a.x + b.x, a.y - b.y);
        }
    h->Lt.alloc((size_t)ld * nt * sizeof(double));
    h->Mt.alloc((size_t)ld * nt * sizeof(double));
    h->Wsym.alloc(ws.size() * sizeof(double2));
    KS_CUDA(cudaMemcpy(h->Lt.p, Lt, (size_t)ld * nt * sizeof(double), cudaMemcpyHostToDevice));
    KS_CUDA(cudaMemcpy(h->Mt.p, Mt, (size_t)ld * nt * sizeof(double), cudaMemcpyHostToDevice));
    KS_CUDA(cudaMemcpy(h->Wsym.p, ws.data(), ws.size() * sizeof(double2), cudaMemcpyHostToDevice));

    // this rank's fibers after the re-shard: rest in R_rank (all of axes 1..d-1
    // flattened), all i_d; local fiber f = rl + |R| * i_d. Blocks: one per
    // distinct composite eigenvalue among them (sorted multi-index when the
    // axes' spectra are identical, as in ks_fd_create).
    const Range R = P.rest[rank];
    const size_t nf = (size_t)R.n() * (size_t)P.nd;
    bool dedup = true;
    for (int l = 1; l < d && dedup; ++l)
        dedup = dims[l + 1] == dims[1] &&
                std::memcmp(lambda[l], lambda[0], sizeof(double) * dims[1]) == 0;
    if (const char* e = std::getenv("KS_FD_DEDUP")) dedup = dedup && std::strcmp(e, "0") != 0;
    std::map<std::vector<int>, int> id_of;
    std::vector<double> lam_blk;
    std::vector<int> fblk(nf);
    std::vector<int> idx(d);
    for (size_t f = 0; f < nf; ++f) {
        const long long rl = (long long)(f % (size_t)R.n()), id = (long long)(f / (size_t)R.n());
        long long rest = R.lo + rl;
        for (int l = 0; l < d - 1; ++l) {
            idx[l] = (int)(rest % dims[l + 1]);
            rest /= dims[l + 1];
        }
        idx[d - 1] = (int)id;
        std::vector<int> key = idx;
        if (dedup) std::sort(key.begin(), key.end());
        auto it = id_of.find(key);
        if (it == id_of.end()) {
            double s = 0; // reference summation order of the (sorted) multi-index
            for (int l = 0; l < d; ++l) s += lambda[l][key[l]];
            it = id_of.emplace(key, (int)lam_blk.size()).first;
            lam_blk.push_back(s);
        }
        fblk[f] = it->second;
    }
    FdBlocks& B = h->blocks;
    B.nt = nt;
    B.p = p_t;
    B.ldab = 3 * p_t + 1;
    B.ns = nf;
    B.nblk = lam_blk.size();
    B.lam_blk.alloc(B.nblk * sizeof(double));
    KS_CUDA(cudaMemcpy(B.lam_blk.p, lam_blk.data(), B.nblk * sizeof(double), cudaMemcpyHostToDevice));
    B.fiber_block.alloc(nf * sizeof(int));
    KS_CUDA(cudaMemcpy(B.fiber_block.p, fblk.data(), nf * sizeof(int), cudaMemcpyHostToDevice));
    fd_blocks_alloc(B);
    launch_fd_factor(B, nu, h->Lt.as<double>(), h->Mt.as<double>(), h->Wsym.as<double2>(), h->stream);
    // scratch: slab-sized for phases 1/3, rest-sized for phase 2
    const size_t slab_n = (size_t)nt * P.Np * P.slab[rank].n();
    const size_t work_n = (size_t)nt * R.n() * P.nd;
    h->s0.alloc(std::max(slab_n, work_n) * sizeof(double2));
    h->s1.alloc(std::max(slab_n, work_n) * sizeof(double2));
    KS_CUDA(cudaStreamSynchronize(h->stream));
    *out = h.release();
    API_END
}

int ks_fdshard_sizes(const ks_fdshard* h, size_t* slab_n, size_t* work_n) {
    API_BEGIN
    KS_REQUIRE(h, KS_EINVAL, "NULL handle");
    const Plan& P = h->plan;
    if (slab_n) *slab_n = (size_t)P.nt * P.Np * P.slab[P.rank].n();
    if (work_n) *work_n = (size_t)P.nt * P.rest[P.rank].n() * P.nd;
    API_END
}

// phase 1: r_local (slab, natural) -> sendbuf (blocks per destination, rank order)
int ks_fdshard_forward(ks_fdshard* h, const ks_c64* r_local, ks_c64* sendbuf, void* stream) {
    API_BEGIN
    KS_REQUIRE(h && r_local && sendbuf, KS_EINVAL, "ks_fdshard_forward: NULL argument");
    std::lock_guard<std::mutex> lk(h->mu);
    ensure_device(h->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
    const Plan& P = h->plan;
    const int d = P.d;
    const long long m = P.slab[P.rank].n();
    // local dims (n_t, n_1..n_{d-1}, m): transforms on axes 1..d-1
    const double* cur = reinterpret_cast<const double*>(r_local);
    double* bufs[2] = {h->s0.as<double>(), h->s1.as<double>()};
    int nb = 0;
    const size_t N = (size_t)P.nt * P.Np * m;
    for (int l = 1; l < d; ++l) {
        size_t stride = 1;
        for (int k = 0; k < l; ++k) stride *= (size_t)P.dims[k];
        const size_t outer = N / (stride * (size_t)P.dims[l]);
        shard_gemm(h, l, false, cur, bufs[nb], stride, outer, st, 0, 0);
        cur = bufs[nb];
        nb ^= 1;
    }
    // pack: for destination q, rows j = 0..m-1 of width nt*|R_q| at column nt*R_q.lo
    const size_t row = (size_t)P.nt * P.Np * sizeof(double2);
    for (int q = 0; q < P.nranks; ++q) {
        const size_t w = (size_t)P.nt * P.rest[q].n() * sizeof(double2);
        const char* src = reinterpret_cast<const char*>(cur) + (size_t)P.nt * P.rest[q].lo * sizeof(double2);
        char* dst = reinterpret_cast<char*>(sendbuf) + (size_t)P.sdisp1[q] * sizeof(double2);
        if (w && m) KS_CUDA(cudaMemcpy2DAsync(dst, w, src, row, w, (size_t)m, cudaMemcpyDeviceToDevice, st));
    }
    if (!stream) KS_CUDA(cudaStreamSynchronize(st));
    API_END
}

// phase 2 (in place on the re-sharded tensor (n_t, |R|, n_d)):
// axis-d transform -> block solves -> inverse axis-d transform
int ks_fdshard_middle(ks_fdshard* h, ks_c64* work, void* stream) {
    API_BEGIN
    KS_REQUIRE(h && work, KS_EINVAL, "ks_fdshard_middle: NULL argument");
    std::lock_guard<std::mutex> lk(h->mu);
    ensure_device(h->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
    const Plan& P = h->plan;
    const size_t s = (size_t)P.nt * P.rest[P.rank].n();
    double* tmp = h->s0.as<double>();
    shard_gemm(h, P.d, false, reinterpret_cast<double*>(work), tmp, s, 1, st, 1, P.nt);
    launch_fd_solve(h->blocks, reinterpret_cast<double2*>(tmp), false, st);
    shard_gemm(h, P.d, true, tmp, reinterpret_cast<double*>(work), s, 1, st, 2, P.nt);
    if (!stream) KS_CUDA(cudaStreamSynchronize(st));
    API_END
}

// phase 3: recvbuf (blocks (t, R_q, slab_rank) from every q, rank order) -> z_local
int ks_fdshard_backward(ks_fdshard* h, const ks_c64* recvbuf, ks_c64* z_local, void* stream) {
    API_BEGIN
    KS_REQUIRE(h && recvbuf && z_local, KS_EINVAL, "ks_fdshard_backward: NULL argument");
    std::lock_guard<std::mutex> lk(h->mu);
    ensure_device(h->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
    const Plan& P = h->plan;
    const int d = P.d;
    const long long m = P.slab[P.rank].n();
    double* slab = h->s1.as<double>();
    const size_t row = (size_t)P.nt * P.Np * sizeof(double2);
    for (int q = 0; q < P.nranks; ++q) {
        const size_t w = (size_t)P.nt * P.rest[q].n() * sizeof(double2);
        const char* src = reinterpret_cast<const char*>(recvbuf) + (size_t)P.sdisp1[q] * sizeof(double2);
        char* dst = reinterpret_cast<char*>(slab) + (size_t)P.nt * P.rest[q].lo * sizeof(double2);
        if (w && m) KS_CUDA(cudaMemcpy2DAsync(dst, row, src, w, w, (size_t)m, cudaMemcpyDeviceToDevice, st));
    }
    const size_t N = (size_t)P.nt * P.Np * m;
    const double* cur = slab;
    double* bufs[2] = {h->s0.as<double>(), h->s1.as<double>()};
    int nb = 0;
    for (int l = 1; l < d; ++l) {
        size_t stride = 1;
        for (int k = 0; k < l; ++k) stride *= (size_t)P.dims[k];
        const size_t outer = N / (stride * (size_t)P.dims[l]);
        double* out = (l == d - 1) ? reinterpret_cast<double*>(z_local) : bufs[nb];
        shard_gemm(h, l, true, cur, out, stride, outer, st, 0, 0);
        cur = out;
        nb ^= 1;
    }
    if (!stream) KS_CUDA(cudaStreamSynchronize(st));
    API_END
}

// ---------------------------------------------------------------------------
// Peer-memory transport (no all-to-all): every rank exports its phase-1 slab
// and its output slab (CUDA IPC or, for virtual ranks, plain pointers); the
// axis-d transform of the middle phase gathers its K rows straight from the
// owners' slabs and the inverse transform scatters its rows straight into the
// owners' output slabs, so the exchange rides on the transform's own tile
// loads and stores over NVLink, tile by tile. The caller separates the three
// phases with a barrier across ranks (all slabs written before they are read).
// ---------------------------------------------------------------------------

// phase 1 (peer): local transforms on axes 1..d-1 into the exported slab (n_t, N', m)
int ks_fdshard_forward_slab(ks_fdshard* h, const ks_c64* r_local, ks_c64* slab_out, void* stream) {
    API_BEGIN
    KS_REQUIRE(h && r_local && slab_out, KS_EINVAL, "ks_fdshard_forward_slab: NULL argument");
    std::lock_guard<std::mutex> lk(h->mu);
    ensure_device(h->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
    const Plan& P = h->plan;
    const int d = P.d;
    const long long m = P.slab[P.rank].n();
    const double* cur = reinterpret_cast<const double*>(r_local);
    double* bufs[2] = {h->s0.as<double>(), h->s1.as<double>()};
    int nb = 0;
    const size_t N = (size_t)P.nt * P.Np * m;
    for (int l = 1; l < d; ++l) {
        size_t stride = 1;
        for (int k = 0; k < l; ++k) stride *= (size_t)P.dims[k];
        const size_t outer = N / (stride * (size_t)P.dims[l]);
        double* out = l == d - 1 ? reinterpret_cast<double*>(slab_out) : bufs[nb];
        shard_gemm(h, l, false, cur, out, stride, outer, st, 0, 0);
        cur = out;
        nb ^= 1;
    }
    if (!stream) KS_CUDA(cudaStreamSynchronize(st));
    API_END
}

// peers: phase-1 slabs (in) and output slabs (out) of every rank, device
// pointers valid in this process; builds the axis-d row tables of this rank
int ks_fdshard_set_peers(ks_fdshard* h, const ks_c64* const* peer_in, ks_c64* const* peer_out) {
    API_BEGIN
    KS_REQUIRE(h && peer_in && peer_out, KS_EINVAL, "ks_fdshard_set_peers: NULL argument");
    std::lock_guard<std::mutex> lk(h->mu);
    ensure_device(h->device);
    const Plan& P = h->plan;
    const Range R = P.rest[P.rank];
    std::vector<const double*> rin(P.nd);
    std::vector<double*> rout(P.nd);
    for (int q = 0; q < P.nranks; ++q)
        for (long long j = P.slab[q].lo; j < P.slab[q].hi; ++j) {
            // row j of axis d, columns (t, rest in R): slab_q + ((j - lo_q) N' + R.lo) n_t complex
            const size_t off = 2 * ((size_t)(j - P.slab[q].lo) * P.nt * P.Np + (size_t)P.nt * R.lo);
            rin[j] = reinterpret_cast<const double*>(peer_in[q]) + off;
            rout[j] = reinterpret_cast<double*>(peer_out[q]) + off;
        }
    h->rows_in.alloc(P.nd * sizeof(double*));
    h->rows_out.alloc(P.nd * sizeof(double*));
    KS_CUDA(cudaMemcpy(h->rows_in.p, rin.data(), P.nd * sizeof(double*), cudaMemcpyHostToDevice));
    KS_CUDA(cudaMemcpy(h->rows_out.p, rout.data(), P.nd * sizeof(double*), cudaMemcpyHostToDevice));
    API_END
}

// phase 2 (peer): axis-d transform gathering rows from the peers' slabs ->
// block solves -> inverse transform scattering rows into the peers' output slabs
int ks_fdshard_middle_peer(ks_fdshard* h, void* stream) {
    API_BEGIN
    KS_REQUIRE(h && h->rows_in.p, KS_EINVAL, "ks_fdshard_middle_peer: call ks_fdshard_set_peers first");
    std::lock_guard<std::mutex> lk(h->mu);
    ensure_device(h->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
    const Plan& P = h->plan;
    const size_t s = (size_t)P.nt * P.rest[P.rank].n();
    double* tmp = h->s0.as<double>();
    auto rin = static_cast<const double* const*>(h->rows_in.p);
    auto rout = static_cast<double* const*>(h->rows_out.p);
    shard_gemm(h, P.d, false, h->s1.as<double>() /* dummy, rows come from rin */, tmp, s, 1, st, 1, P.nt, rin, nullptr);
    launch_fd_solve(h->blocks, reinterpret_cast<double2*>(tmp), false, st);
    shard_gemm(h, P.d, true, tmp, nullptr, s, 1, st, 2, P.nt, nullptr, rout);
    if (!stream) KS_CUDA(cudaStreamSynchronize(st));
    API_END
}

// phase 3 (peer): inverse transforms on axes 1..d-1 of this rank's output slab
int ks_fdshard_backward_slab(ks_fdshard* h, const ks_c64* slab_in, ks_c64* z_local, void* stream) {
    API_BEGIN
    KS_REQUIRE(h && slab_in && z_local, KS_EINVAL, "ks_fdshard_backward_slab: NULL argument");
    std::lock_guard<std::mutex> lk(h->mu);
    ensure_device(h->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
    const Plan& P = h->plan;
    const int d = P.d;
    const long long m = P.slab[P.rank].n();
    const size_t N = (size_t)P.nt * P.Np * m;
    const double* cur = reinterpret_cast<const double*>(slab_in);
    double* bufs[2] = {h->s0.as<double>(), h->s1.as<double>()};
    int nb = 0;
    for (int l = 1; l < d; ++l) {
        size_t stride = 1;
        for (int k = 0; k < l; ++k) stride *= (size_t)P.dims[k];
        const size_t outer = N / (stride * (size_t)P.dims[l]);
        double* out = (l == d - 1) ? reinterpret_cast<double*>(z_local) : bufs[nb];
        shard_gemm(h, l, true, cur, out, stride, outer, st, 0, 0);
        cur = out;
        nb ^= 1;
    }
    if (!stream) KS_CUDA(cudaStreamSynchronize(st));
    API_END
}

// CUDA IPC plumbing for the peer transport across processes
int ks_ipc_get_handle(const void* dptr, void* handle /* 64 bytes */) {
    API_BEGIN
    KS_REQUIRE(dptr && handle, KS_EINVAL, "ks_ipc_get_handle: NULL argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t hd;
    KS_CUDA(cudaIpcGetMemHandle(&hd, const_cast<void*>(dptr)));
    std::memcpy(handle, &hd, sizeof(hd));
    API_END
}
int ks_ipc_open(const void* handle, void** dptr) {
    API_BEGIN
    KS_REQUIRE(handle && dptr, KS_EINVAL, "ks_ipc_open: NULL argument");
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, handle, sizeof(hd));
    KS_CUDA(cudaIpcOpenMemHandle(dptr, hd, cudaIpcMemLazyEnablePeerAccess));
    API_END
}
int ks_ipc_close(void* dptr) {
    API_BEGIN
    KS_CUDA(cudaIpcCloseMemHandle(dptr));
    API_END
}

int ks_fdshard_apply(ks_fdshard* h, ks_comm* comm, const ks_c64* r_slab, ks_c64* z_slab, void* stream) {
    API_BEGIN
    KS_REQUIRE(h && comm && r_slab && z_slab, KS_EINVAL, "ks_fdshard_apply: NULL argument");
    ensure_device(h->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
    fdshard_apply_comm(h, comm, reinterpret_cast<const double2*>(r_slab), reinterpret_cast<double2*>(z_slab), st);
    if (!stream) KS_CUDA(cudaStreamSynchronize(st));
    API_END
}

int ks_fdshard_destroy(ks_fdshard* h) {
    if (h) {
        cudaSetDevice(h->device);
        delete h;
    }
    return KS_OK;
}

} // extern "C"
