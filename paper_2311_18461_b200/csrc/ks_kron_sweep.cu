// Level pass kernel for the Kronecker-sum matvec (plan: ks_kron.cu).
//
// One thread per output position (o, r, q), consecutive threads on
// consecutive q (coalesced for every axis; along the fiber for the time
// axis). For each input node the 2*BW+1 band neighbours along the pass axis
// are loaded once into registers and reused by every contribution of that
// input (contributions grouped by input on the host); the NOUT outputs
// accumulate in registers through a uniform switch (static indices) and are
// written once. Neighbour rows are shared between threads through L1/L2, so
// HBM sees each input element about once. Band rows are pre-expanded
// row-major: rb[f][r][t] = F(r, r - BW + t).
//
// (Designs measured and dropped on B200, see profiles/: a per-column
// sliding-window sweep and a shared-memory column tile both moved exactly the
// algorithmic bytes but ran at 12-17% occupancy, 2-4x slower.)
#include "ks_internal.hpp"

#include <algorithm>
#include <cstdlib>

namespace ks {

struct SweepEntry {
    int out;    // output node
    int factor; // -1 = identity
    double2 coeff;
};
struct RingCon {  // ring sweep: one contribution, grouped by output node
    int in, factor;
    double2 coeff;
};

namespace {

constexpr int kTileThreads = 256;

// one thread per output position (o, r, q); consecutive threads = consecutive q
template <int NOUT, int BW>
__global__ void __launch_bounds__(kTileThreads) k_kron_elem(
    const double2* const* __restrict__ in_ptrs, int n_in, double2* const* __restrict__ out_ptrs,
    const int* __restrict__ in_begin, const SweepEntry* __restrict__ entries,
    const double2* __restrict__ rb, const int* __restrict__ freal, size_t N, size_t s, int n,
    int nmax, size_t nqt, int n_in_rows, int in_off, int band_off) {
    // n = output rows of the pass axis; the input has n_in_rows rows and output
    // row r reads input rows r + in_off - BW .. r + in_off + BW with band row
    // band_off + r (sharded outermost axis: haloed slab in, owned planes out)
    constexpr int TAPS = 2 * BW + 1;
    size_t idx, q, o;
    int r;
    if (nqt == 0) { // natural order: q fastest, then r
        idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
        if (idx >= N) return;
        q = idx % s;
        const size_t t = idx / s;
        r = (int)(t % (size_t)n);
        o = t / (size_t)n;
    } else {        // long strides: CTA = (o, q-tile, r), r fastest across CTAs so the
                    // +-BW neighbour rows of a q-tile are still in L2
        const size_t b = blockIdx.x;
        r = (int)(b % (size_t)n);
        const size_t rest = b / (size_t)n;
        const size_t qt = rest % nqt;
        o = rest / nqt;
        q = qt * blockDim.x + threadIdx.x;
        if (q >= s) return;
        idx = (o * (size_t)n + r) * s + q;
    }
    const size_t base = o * (size_t)n_in_rows * s + q;
    const double2 Z = make_double2(0.0, 0.0);
    double2 acc[NOUT];
#pragma unroll
    for (int a = 0; a < NOUT; ++a) acc[a] = Z;
    for (int j = 0; j < n_in; ++j) {
        const double2* __restrict__ in = in_ptrs[j] + base;
        double2 w[TAPS];
#pragma unroll
        for (int tp = 0; tp < TAPS; ++tp) {
            const int rr = r + in_off - BW + tp;
            w[tp] = (rr >= 0 && rr < n_in_rows) ? __ldg(in + (size_t)rr * s) : Z;
        }
        const int eb = __ldg(in_begin + j), ee = __ldg(in_begin + j + 1);
        for (int e = eb; e < ee; ++e) {
            const int ef = __ldg(&entries[e].factor), eo = __ldg(&entries[e].out);
            const double2 c = __ldg(&entries[e].coeff);
            double vr, vi;
            if (ef < 0) {
                vr = w[BW].x;
                vi = w[BW].y;
            } else {
                const double2* band = rb + ((size_t)ef * nmax + band_off + r) * TAPS;
                vr = 0.0;
                vi = 0.0;
                if (__ldg(freal + ef)) {
#pragma unroll
                    for (int tp = 0; tp < TAPS; ++tp) {
                        const double a = __ldg(&band[tp].x);
                        vr = fma(a, w[tp].x, vr);
                        vi = fma(a, w[tp].y, vi);
                    }
                } else {
#pragma unroll
                    for (int tp = 0; tp < TAPS; ++tp) {
                        const double2 a = __ldg(&band[tp]);
                        vr = fma(a.x, w[tp].x, fma(-a.y, w[tp].y, vr));
                        vi = fma(a.x, w[tp].y, fma(a.y, w[tp].x, vi));
                    }
                }
            }
            switch (eo) {
#define KS_ACC(OO)                                                                 \
    case OO:                                                                       \
        if (OO < NOUT) {                                                           \
            double2& A = acc[OO < NOUT ? OO : 0];                                  \
            A.x = fma(c.x, vr, fma(-c.y, vi, A.x));                                \
            A.y = fma(c.x, vi, fma(c.y, vr, A.y));                                 \
        }                                                                          \
        break;
                KS_ACC(0) KS_ACC(1) KS_ACC(2) KS_ACC(3) KS_ACC(4) KS_ACC(5) KS_ACC(6) KS_ACC(7)
#undef KS_ACC
            }
        }
    }
#pragma unroll
    for (int a = 0; a < NOUT; ++a) out_ptrs[a][idx] = acc[a];
}

// ---------------------------------------------------------------------------
// Tile kernel: a CTA owns kTQ = 8 consecutive columns (o, q) and the FULL axis
// (rows r = 0..n-1, RPT per thread, 32 row groups), so banded products are
// local. Input nodes are staged in shared memory one after another through a
// two-buffer cp.async pipeline (input j+1 loads while input j is consumed);
// rows are padded with BW zero rows so the tap loops have no branches.
// ---------------------------------------------------------------------------
constexpr int kTQ = 8, kRG = 32;

__device__ __forceinline__ void cpa16(void* dst, const void* src, bool v) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(v ? 16 : 0));
}

constexpr int kStg = 4; // ring stages over (column tile, input) work items

template <int NOUT, int BW, int RPT>
__global__ void __launch_bounds__(kTileThreads) k_kron_tile2(
    const double2* const* __restrict__ in_ptrs, int n_in, double2* const* __restrict__ out_ptrs,
    const int* __restrict__ in_begin, const SweepEntry* __restrict__ entries,
    const double2* __restrict__ rb, const int* __restrict__ freal, size_t ncols, size_t s, int n,
    int nmax, int n_in_rows, int in_off, int band_off) {
    // persistent: CTA b owns column tiles b, b + grid, ...; work item w = (tile, input j)
    constexpr int TAPS = 2 * BW + 1, PITCH = kTQ + 1;
    extern __shared__ __align__(16) double2 tl[]; // [kStg][n_in_rows + 2BW][PITCH]
    const int rows_p = n_in_rows + 2 * BW;
    const size_t stage_sz = (size_t)rows_p * PITCH;
    const int tid = threadIdx.x, cc = tid % kTQ, rg = tid / kTQ;
    const size_t ntiles = (ncols + kTQ - 1) / kTQ;
    const double2 Z = make_double2(0.0, 0.0);
    for (int e = tid; e < BW * PITCH; e += kTileThreads) // zero halo rows of every stage
        for (int b = 0; b < kStg; ++b) {
            tl[b * stage_sz + e] = Z;
            tl[b * stage_sz + (n_in_rows + BW) * PITCH + e] = Z;
        }
    const long long my_tiles =
        ntiles > blockIdx.x ? (long long)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
    const long long nwork = my_tiles * n_in;
    // issue side: column base of the item's tile (recomputed when the tile changes)
    long long ibase_tile = -1;
    long long ibase = 0;
    int incol = 0;
    auto issue = [&](long long w) {
        if (w < nwork) {
            const long long ti = w / n_in;
            const int j = (int)(w - ti * n_in);
            const size_t c0 = (size_t)(blockIdx.x + ti * gridDim.x) * kTQ;
            const int ncol = (int)min((size_t)kTQ, ncols - c0);
            double2* t = tl + (size_t)(w % kStg) * stage_sz + BW * PITCH;
            const double2* __restrict__ in = in_ptrs[j];
            const int tot = n_in_rows * kTQ;
            if (s == 1) {
                const double2* src0 = in + c0 * (size_t)n_in_rows; // fibers contiguous
                for (int e = tid; e < tot; e += kTileThreads) {
                    const int c = e / n_in_rows, r = e - c * n_in_rows;
                    const bool v = c < ncol;
                    cpa16(t + r * PITCH + c, v ? (const void*)(src0 + e) : (const void*)in, v);
                }
            } else {
                if (ibase_tile != ti) { // this thread's column (tid & 7 fixed for all e)
                    const size_t cm = c0 + (tid & (kTQ - 1));
                    const size_t oo = cm / s, qq = cm - oo * s;
                    ibase = (long long)(oo * (size_t)n_in_rows * s + qq);
                    incol = (int)(tid & (kTQ - 1)) < ncol;
                    ibase_tile = ti;
                }
                for (int e = tid; e < tot; e += kTileThreads) {
                    const int r = e >> 3, c = e & (kTQ - 1);
                    cpa16(t + r * PITCH + c, incol ? (const void*)(in + ibase + (size_t)r * s) : (const void*)in,
                          incol != 0);
                }
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    double2 acc[NOUT][RPT];
#pragma unroll
    for (int a = 0; a < NOUT; ++a)
#pragma unroll
        for (int k = 0; k < RPT; ++k) acc[a][k] = Z;
    __syncthreads(); // halos visible before any stage is consumed
#pragma unroll
    for (int q = 0; q < kStg - 1; ++q) issue(q);
    for (long long w = 0; w < nwork; ++w) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kStg - 2));
        __syncthreads();
        issue(w + kStg - 1);
        const long long ti = w / n_in;
        const int j = (int)(w - ti * n_in);
        const double2* t = tl + (size_t)(w % kStg) * stage_sz + cc;
        const int eb = in_begin[j], ee = in_begin[j + 1];
        for (int e = eb; e < ee; ++e) {
            const SweepEntry en = entries[e];
            double2 v[RPT];
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                const int r = rg + k * kRG;
                v[k] = Z;
                if (r < n) {
                    const double2* wv = t + (r + in_off) * PITCH;
                    if (en.factor < 0) {
                        v[k] = wv[BW * PITCH];
                    } else {
                        const double2* band = rb + ((size_t)en.factor * nmax + band_off + r) * TAPS;
                        double vr = 0.0, vi = 0.0;
                        if (freal[en.factor]) {
#pragma unroll
                            for (int tp = 0; tp < TAPS; ++tp) {
                                const double a = __ldg(&band[tp].x);
                                const double2 x = wv[tp * PITCH];
                                vr = fma(a, x.x, vr);
                                vi = fma(a, x.y, vi);
                            }
                        } else {
#pragma unroll
                            for (int tp = 0; tp < TAPS; ++tp) {
                                const double2 a = __ldg(&band[tp]);
                                const double2 x = wv[tp * PITCH];
                                vr = fma(a.x, x.x, fma(-a.y, x.y, vr));
                                vi = fma(a.x, x.y, fma(a.y, x.x, vi));
                            }
                        }
                        v[k] = make_double2(vr, vi);
                    }
                }
            }
            const double cr = en.coeff.x, ci = en.coeff.y;
            switch (en.out) {
#define KS_ACC(OO)                                                                 \
    case OO:                                                                       \
        if (OO < NOUT) {                                                           \
            _Pragma("unroll") for (int k = 0; k < RPT; ++k) {                      \
                double2& A = acc[OO < NOUT ? OO : 0][k];                           \
                A.x = fma(cr, v[k].x, fma(-ci, v[k].y, A.x));                      \
                A.y = fma(cr, v[k].y, fma(ci, v[k].x, A.y));                       \
            }                                                                      \
        }                                                                          \
        break;
                KS_ACC(0) KS_ACC(1) KS_ACC(2) KS_ACC(3) KS_ACC(4) KS_ACC(5) KS_ACC(6) KS_ACC(7)
#undef KS_ACC
            }
        }
        if (j == n_in - 1) { // tile complete: store and reset
            const size_t c0 = (size_t)(blockIdx.x + ti * gridDim.x) * kTQ;
            const int ncol = (int)min((size_t)kTQ, ncols - c0);
            if (cc < ncol) {
                const size_t cme = c0 + cc;
                const size_t o = cme / s, q = cme - o * s;
                const size_t base = o * (size_t)n * s + q;
#pragma unroll
                for (int a = 0; a < NOUT; ++a) {
                    double2* __restrict__ out = out_ptrs[a];
#pragma unroll
                    for (int k = 0; k < RPT; ++k) {
                        const int r = rg + k * kRG;
                        if (r < n) out[base + (size_t)r * s] = acc[a][k];
                    }
                }
            }
#pragma unroll
            for (int a = 0; a < NOUT; ++a)
#pragma unroll
                for (int k = 0; k < RPT; ++k) acc[a][k] = Z;
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
}

template <int NOUT, int BW>
bool launch_tile2(int rpt, unsigned grid, size_t sm, cudaStream_t st, const double2* const* ip, int nin,
                  double2* const* op, const int* ib, const SweepEntry* en, const double2* rb,
                  const int* fr, size_t ncols, size_t s, int n, int nmax, int nir, int ioff, int boff) {
#define KS_T2(R)                                                                                        \
    case R: {                                                                                           \
        static bool attr = false;                                                                       \
        if (!attr) {                                                                                    \
            KS_CUDA(cudaFuncSetAttribute(k_kron_tile2<NOUT, BW, R>,                                     \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));     \
            attr = true;                                                                                \
        }                                                                                               \
        k_kron_tile2<NOUT, BW, R><<<grid, kTileThreads, sm, st>>>(ip, nin, op, ib, en, rb, fr, ncols, s, \
                                                                  n, nmax, nir, ioff, boff);            \
        return true;                                                                                    \
    }
    switch (rpt) {
        KS_T2(1) KS_T2(2) KS_T2(3) KS_T2(4) KS_T2(5)
    }
#undef KS_T2
    return false;
}

// ---------------------------------------------------------------------------
// Ring sweep (spatial axes, s > 1): a CTA owns 32 consecutive columns (o, q)
// and walks the pass axis r = 0..n-1 once. Every input row enters a
// shared-memory ring (RW = 2BW+1+kPre rows per input node) exactly once via
// cp.async, kPre rows ahead, so L2 and HBM see each input element once (the
// element kernel re-fetches each element 2BW+1 times through L2 on long
// strides). Warp g computes output node g for the 32 columns: its
// contributions are warp-uniform (staged in shared memory), band
// coefficients are broadcast loads, the ring reads are conflict-free, and
// the output row is one coalesced 512 B store. One barrier per row.
// ---------------------------------------------------------------------------
constexpr int kRC = 32, kPre = 4, kMaxCon = 12;

template <int BW>
__global__ void __launch_bounds__(256) k_kron_ring(
    const double2* const* __restrict__ in_ptrs, int n_in, double2* const* __restrict__ out_ptrs,
    int n_out, const int* __restrict__ out_begin, const RingCon* __restrict__ cons,
    const double2* __restrict__ rb, const int* __restrict__ freal, size_t ncols, size_t s, int n,
    int nmax, int n_in_rows, int in_off, int band_off) {
    constexpr int TAPS = 2 * BW + 1, RW = TAPS + kPre;
    extern __shared__ __align__(16) double2 ring[]; // [n_in][RW][kRC]
    __shared__ RingCon scon[8][kMaxCon];
    __shared__ int sncon[8];
    __shared__ long long scol[kRC];         // input offset of each column (row 0); -1 = invalid
    __shared__ const double2* sin[8];
    const int tid = threadIdx.x, lane = tid & 31, g = tid >> 5;
    const size_t c0 = (size_t)blockIdx.x * kRC;
    if (tid < kRC) {
        const size_t cmc = c0 + tid;
        if (cmc < ncols) {
            const size_t oo = cmc / s, qq = cmc - oo * s;
            scol[tid] = (long long)(oo * (size_t)n_in_rows * s + qq);
        } else {
            scol[tid] = -1;
        }
    }
    if (tid < n_in && tid < 8) sin[tid] = in_ptrs[tid];
    if (tid < 8) sncon[tid] = tid < n_out ? out_begin[tid + 1] - out_begin[tid] : 0;
    for (int e = tid; e < 8 * kMaxCon; e += 256) {
        const int o = e / kMaxCon, k = e - o * kMaxCon;
        if (o < n_out && out_begin[o] + k < out_begin[o + 1]) scon[o][k] = cons[out_begin[o] + k];
    }
    // this lane's column (input geometry for loads, output geometry for stores)
    const size_t cm = c0 + lane;
    const bool cv = cm < ncols;
    size_t ibase = 0, obase = 0;
    if (cv) {
        const size_t oo = cm / s, qq = cm - oo * s;
        ibase = oo * (size_t)n_in_rows * s + qq;
        obase = oo * (size_t)n * s + qq;
    }
    // row x of input j lands in slot x % RW; loads: thread t handles (j, lane) pairs
    auto issue = [&](int x) { // input rows x (padded coordinate: x - BW is the true row)
        const int row = x - BW + in_off; // input row index
        const bool rv = row >= 0 && row < n_in_rows;
        for (int e = tid; e < n_in * kRC; e += 256) {
            const int j = e >> 5, c = e & (kRC - 1);
            double2* dst = ring + ((size_t)j * RW + (x % RW)) * kRC + c;
            const long long cb = scol[c];
            const bool v = rv && cb >= 0;
            const double2* src = sin[j];
            if (v) src += cb + (long long)row * (long long)s;
            const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(v ? 16 : 0));
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    __syncthreads(); // scol / sin / contributions visible
    // prologue: padded rows 0 .. TAPS-2 + kPre (true rows -BW .. BW-1+kPre)
    for (int x = 0; x < TAPS - 1 + kPre; ++x) issue(x);
    __syncthreads();
    const int nc = g < n_out ? sncon[g] : 0;
    for (int r = 0; r < n; ++r) {
        issue(r + TAPS - 1 + kPre); // keeps kPre rows in flight
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kPre));
        __syncthreads();
        if (g < n_out) {
            double ar = 0.0, ai = 0.0;
            for (int k = 0; k < nc; ++k) {
                const RingCon cn = scon[g][k];
                const double2* rj = ring + (size_t)cn.in * RW * kRC + lane;
                double vr, vi;
                if (cn.factor < 0) {
                    const double2 x = rj[((r + BW) % RW) * kRC];
                    vr = x.x;
                    vi = x.y;
                } else {
                    const double2* band = rb + ((size_t)cn.factor * nmax + band_off + r) * TAPS;
                    vr = 0.0;
                    vi = 0.0;
                    if (__ldg(freal + cn.factor)) {
#pragma unroll
                        for (int tp = 0; tp < TAPS; ++tp) {
                            const double a = __ldg(&band[tp].x);
                            const double2 x = rj[((r + tp) % RW) * kRC];
                            vr = fma(a, x.x, vr);
                            vi = fma(a, x.y, vi);
                        }
                    } else {
#pragma unroll
                        for (int tp = 0; tp < TAPS; ++tp) {
                            const double2 a = __ldg(&band[tp]);
                            const double2 x = rj[((r + tp) % RW) * kRC];
                            vr = fma(a.x, x.x, fma(-a.y, x.y, vr));
                            vi = fma(a.x, x.y, fma(a.y, x.x, vi));
                        }
                    }
                }
                ar = fma(cn.coeff.x, vr, fma(-cn.coeff.y, vi, ar));
                ai = fma(cn.coeff.x, vi, fma(cn.coeff.y, vr, ai));
            }
            if (cv) out_ptrs[g][obase + (size_t)r * s] = make_double2(ar, ai);
        }
        __syncthreads(); // slot (r % RW) is refilled by the next issue
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
}

template <int NOUT>
void launch_bw(int bw, unsigned grid, cudaStream_t st, const double2* const* ip, int nin,
               double2* const* op, const int* ib, const SweepEntry* en, const double2* rb,
               const int* fr, size_t N, size_t s, int n, int nmax, size_t nqt, int nir, int ioff,
               int boff) {
    switch (bw) {
    case 1: k_kron_elem<NOUT, 1><<<grid, kTileThreads, 0, st>>>(ip, nin, op, ib, en, rb, fr, N, s, n, nmax, nqt, nir, ioff, boff); break;
    case 2: k_kron_elem<NOUT, 2><<<grid, kTileThreads, 0, st>>>(ip, nin, op, ib, en, rb, fr, N, s, n, nmax, nqt, nir, ioff, boff); break;
    case 3: k_kron_elem<NOUT, 3><<<grid, kTileThreads, 0, st>>>(ip, nin, op, ib, en, rb, fr, N, s, n, nmax, nqt, nir, ioff, boff); break;
    default: k_kron_elem<NOUT, 4><<<grid, kTileThreads, 0, st>>>(ip, nin, op, ib, en, rb, fr, N, s, n, nmax, nqt, nir, ioff, boff); break;
    }
}

} // namespace

// returns false when the level's shape is outside the instantiated range
bool launch_colsweep(int nin, int nout, int bw, const double2* const* ip, double2* const* op,
                     const int* in_begin, const SweepEntry* entries, const double2* rb,
                     const int* freal, size_t ncols, size_t s, int n, int nmax, cudaStream_t st,
                     int nir, int ioff, int boff, const int* ring_begin, const RingCon* ring_cons) {
    if (nir <= 0) nir = n;
    if (nout < 1 || nout > 8 || bw < 1 || bw > 4) return false;
    // ring sweep: opt-in (KS_KRON_RING=1). Exact DRAM bytes but shared-memory
    // bandwidth bound (each tap re-read from the ring per contribution):
    // 5.69 ms vs 3.64 ms for the element kernel at c3 (profiles/round1_summary.md)
    if (s > 1 && ring_cons && nin >= 1 && std::getenv("KS_KRON_RING")) {
        const int RW = 2 * bw + 1 + kPre;
        const size_t sm = (size_t)nin * RW * kRC * sizeof(double2);
        if (sm <= 200 * 1024) {
            const unsigned grid = (unsigned)((ncols + kRC - 1) / kRC);
#define KS_RING(B)                                                                                    \
    case B: {                                                                                         \
        static bool attr = false;                                                                     \
        if (!attr) {                                                                                  \
            KS_CUDA(cudaFuncSetAttribute(k_kron_ring<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         200 * 1024));                                                \
            attr = true;                                                                              \
        }                                                                                             \
        k_kron_ring<B><<<grid, 256, sm, st>>>(ip, nin, op, nout, ring_begin, ring_cons, rb, freal,  \
                                              ncols, s, n, nmax, nir, ioff, boff);                    \
        break;                                                                                        \
    }
            switch (bw) { KS_RING(1) KS_RING(2) KS_RING(3) KS_RING(4) }
#undef KS_RING
            check_launch("k_kron_ring");
            return true;
        }
    }
    const int rpt = (n + kRG - 1) / kRG;
    // opt-in: measured 3.70 ms vs 3.64 ms for the element kernel at c3
    if (rpt <= 5 && std::getenv("KS_KRON_TILE")) {
        const size_t sm = (size_t)kStg * (nir + 2 * bw) * (kTQ + 1) * sizeof(double2);
        static int sms = 0;
        if (!sms) {
            int dev = 0;
            KS_CUDA(cudaGetDevice(&dev));
            KS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        }
        const size_t ntl = (ncols + kTQ - 1) / kTQ;
        const unsigned g = (unsigned)std::min<size_t>(ntl, (size_t)sms * 4);
        bool ok = false;
#define KS_T2B(NO)                                                                               \
    case NO:                                                                                     \
        switch (bw) {                                                                            \
        case 1: ok = launch_tile2<NO, 1>(rpt, g, sm, st, ip, nin, op, in_begin, entries, rb, freal, ncols, s, n, nmax, nir, ioff, boff); break; \
        case 2: ok = launch_tile2<NO, 2>(rpt, g, sm, st, ip, nin, op, in_begin, entries, rb, freal, ncols, s, n, nmax, nir, ioff, boff); break; \
        case 3: ok = launch_tile2<NO, 3>(rpt, g, sm, st, ip, nin, op, in_begin, entries, rb, freal, ncols, s, n, nmax, nir, ioff, boff); break; \
        default: ok = launch_tile2<NO, 4>(rpt, g, sm, st, ip, nin, op, in_begin, entries, rb, freal, ncols, s, n, nmax, nir, ioff, boff); break; \
        }                                                                                        \
        break;
        switch (nout) { KS_T2B(1) KS_T2B(2) KS_T2B(3) KS_T2B(4) KS_T2B(5) KS_T2B(6) KS_T2B(7) KS_T2B(8) }
#undef KS_T2B
        if (ok) {
            check_launch("k_kron_tile2");
            return true;
        }
    }
    const size_t N = ncols * (size_t)n;
    size_t nqt = 0;
    unsigned grid = (unsigned)((N + kTileThreads - 1) / kTileThreads);
    if (s >= 4 * kTileThreads) {
        nqt = (s + kTileThreads - 1) / kTileThreads;
        const size_t outer = ncols / s;
        grid = (unsigned)(outer * nqt * (size_t)n);
    }
    switch (nout) {
    case 1: launch_bw<1>(bw, grid, st, ip, nin, op, in_begin, entries, rb, freal, N, s, n, nmax, nqt, nir, ioff, boff); break;
    case 2: launch_bw<2>(bw, grid, st, ip, nin, op, in_begin, entries, rb, freal, N, s, n, nmax, nqt, nir, ioff, boff); break;
    case 3: launch_bw<3>(bw, grid, st, ip, nin, op, in_begin, entries, rb, freal, N, s, n, nmax, nqt, nir, ioff, boff); break;
    case 4: launch_bw<4>(bw, grid, st, ip, nin, op, in_begin, entries, rb, freal, N, s, n, nmax, nqt, nir, ioff, boff); break;
    case 5: launch_bw<5>(bw, grid, st, ip, nin, op, in_begin, entries, rb, freal, N, s, n, nmax, nqt, nir, ioff, boff); break;
    case 6: launch_bw<6>(bw, grid, st, ip, nin, op, in_begin, entries, rb, freal, N, s, n, nmax, nqt, nir, ioff, boff); break;
    case 7: launch_bw<7>(bw, grid, st, ip, nin, op, in_begin, entries, rb, freal, N, s, n, nmax, nqt, nir, ioff, boff); break;
    case 8: launch_bw<8>(bw, grid, st, ip, nin, op, in_begin, entries, rb, freal, N, s, n, nmax, nqt, nir, ioff, boff); break;
    }
    check_launch("k_kron_elem");
    return true;
}

} // namespace ks
