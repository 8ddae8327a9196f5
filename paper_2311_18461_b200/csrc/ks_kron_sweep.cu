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
