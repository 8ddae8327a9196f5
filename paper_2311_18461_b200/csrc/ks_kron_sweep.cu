// Level pass "column sweep" for the Kronecker-sum matvec (see ks_kron.cu for
// the level-pass plan). One thread owns one column (o, q) of the pass axis
// and walks its rows r = 0..n-1 once, keeping a (2*BW+1)-row sliding window of
// every input node in registers: each input element is loaded from HBM
// exactly once, each output element is written once, and consecutive
// threads own consecutive q, so every load and store of a warp is one
// contiguous segment. Used for the spatial axes (stride s > 1); the
// contiguous time axis keeps the row-chunk kernel in ks_kron.cu.
//
// The per-row work is the level's contribution list grouped by input node
// (entries[in_begin[ii] .. in_begin[ii+1])): for each entry the band row
// F(r, r-BW..r+BW) (pre-expanded row-major, rb[f][r][dj]) is applied to the
// window of input ii and added, times the entry's coefficient, into output
// `out`. NIN/NOUT/BW are template parameters so every register index is
// static; the output is selected by a uniform switch.
#include "ks_internal.hpp"

namespace ks {

struct SweepEntry {
    int out;    // output node
    int factor; // -1 = identity
    double2 coeff;
};

namespace {

template <int NIN, int NOUT, int BW>
__global__ void __launch_bounds__(128) k_kron_colsweep(
    const double2* const* __restrict__ in_ptrs, double2* const* __restrict__ out_ptrs,
    const int* __restrict__ in_begin, const SweepEntry* __restrict__ entries,
    const double2* __restrict__ rb, const int* __restrict__ freal, size_t ncols, size_t s, int n,
    int nmax) {
    constexpr int TAPS = 2 * BW + 1;
    const size_t col = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (col >= ncols) return;
    const size_t o = col / s, q = col - o * s;
    const size_t base = o * (size_t)n * s + q;
    const double2 Z = make_double2(0.0, 0.0);

    const double2* ip[NIN];
#pragma unroll
    for (int ii = 0; ii < NIN; ++ii) ip[ii] = in_ptrs[ii] + base;
    double2* op[NOUT];
#pragma unroll
    for (int oo = 0; oo < NOUT; ++oo) op[oo] = out_ptrs[oo] + base;

    // window rows r-BW .. r+BW; w[ii][t] = in_ii[r - BW + t]
    double2 w[NIN][TAPS];
#pragma unroll
    for (int ii = 0; ii < NIN; ++ii) {
#pragma unroll
        for (int t = 0; t < TAPS; ++t) {
            const int rr = t - BW; // r = 0
            w[ii][t] = (rr >= 0 && rr < n) ? __ldg(ip[ii] + (size_t)rr * s) : Z;
        }
    }
    for (int r = 0; r < n; ++r) {
        double2 acc[NOUT];
#pragma unroll
        for (int oo = 0; oo < NOUT; ++oo) acc[oo] = Z;
        // prefetch the row entering the window next (r + BW + 1)
        double2 nxt[NIN];
        const int rn = r + BW + 1;
#pragma unroll
        for (int ii = 0; ii < NIN; ++ii) nxt[ii] = rn < n ? __ldg(ip[ii] + (size_t)rn * s) : Z;
#pragma unroll
        for (int ii = 0; ii < NIN; ++ii) {
            const int eb = __ldg(in_begin + ii), ee = __ldg(in_begin + ii + 1);
            for (int e = eb; e < ee; ++e) {
                const int eo = __ldg(&entries[e].out), ef = __ldg(&entries[e].factor);
                const double2 c = __ldg(&entries[e].coeff);
                double vr, vi;
                if (ef < 0) {
                    vr = w[ii][BW].x;
                    vi = w[ii][BW].y;
                } else {
                    const double2* band = rb + ((size_t)ef * nmax + r) * TAPS;
                    vr = 0.0;
                    vi = 0.0;
                    if (__ldg(freal + ef)) {
#pragma unroll
                        for (int t = 0; t < TAPS; ++t) {
                            const double a = __ldg(&band[t].x);
                            vr = fma(a, w[ii][t].x, vr);
                            vi = fma(a, w[ii][t].y, vi);
                        }
                    } else {
#pragma unroll
                        for (int t = 0; t < TAPS; ++t) {
                            const double2 a = __ldg(&band[t]);
                            vr = fma(a.x, w[ii][t].x, fma(-a.y, w[ii][t].y, vr));
                            vi = fma(a.x, w[ii][t].y, fma(a.y, w[ii][t].x, vi));
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
        for (int oo = 0; oo < NOUT; ++oo) op[oo][(size_t)r * s] = acc[oo];
#pragma unroll
        for (int ii = 0; ii < NIN; ++ii) {
#pragma unroll
            for (int t = 0; t < TAPS - 1; ++t) w[ii][t] = w[ii][t + 1];
            w[ii][TAPS - 1] = nxt[ii];
        }
    }
}

template <int NIN, int NOUT>
bool launch_bw(int bw, unsigned grid, cudaStream_t st, const double2* const* ip, double2* const* op,
               const int* ib, const SweepEntry* en, const double2* rb, const int* fr, size_t ncols,
               size_t s, int n, int nmax) {
    switch (bw) {
    case 1: k_kron_colsweep<NIN, NOUT, 1><<<grid, 128, 0, st>>>(ip, op, ib, en, rb, fr, ncols, s, n, nmax); return true;
    case 2: k_kron_colsweep<NIN, NOUT, 2><<<grid, 128, 0, st>>>(ip, op, ib, en, rb, fr, ncols, s, n, nmax); return true;
    case 3: k_kron_colsweep<NIN, NOUT, 3><<<grid, 128, 0, st>>>(ip, op, ib, en, rb, fr, ncols, s, n, nmax); return true;
    case 4: k_kron_colsweep<NIN, NOUT, 4><<<grid, 128, 0, st>>>(ip, op, ib, en, rb, fr, ncols, s, n, nmax); return true;
    default: return false;
    }
}

template <int NIN>
bool launch_out(int nout, int bw, unsigned grid, cudaStream_t st, const double2* const* ip,
                double2* const* op, const int* ib, const SweepEntry* en, const double2* rb,
                const int* fr, size_t ncols, size_t s, int n, int nmax) {
    switch (nout) {
    case 1: return launch_bw<NIN, 1>(bw, grid, st, ip, op, ib, en, rb, fr, ncols, s, n, nmax);
    case 2: return launch_bw<NIN, 2>(bw, grid, st, ip, op, ib, en, rb, fr, ncols, s, n, nmax);
    case 3: return launch_bw<NIN, 3>(bw, grid, st, ip, op, ib, en, rb, fr, ncols, s, n, nmax);
    case 4: return launch_bw<NIN, 4>(bw, grid, st, ip, op, ib, en, rb, fr, ncols, s, n, nmax);
    case 5: return launch_bw<NIN, 5>(bw, grid, st, ip, op, ib, en, rb, fr, ncols, s, n, nmax);
    case 6: return launch_bw<NIN, 6>(bw, grid, st, ip, op, ib, en, rb, fr, ncols, s, n, nmax);
    case 7: return launch_bw<NIN, 7>(bw, grid, st, ip, op, ib, en, rb, fr, ncols, s, n, nmax);
    case 8: return launch_bw<NIN, 8>(bw, grid, st, ip, op, ib, en, rb, fr, ncols, s, n, nmax);
    default: return false;
    }
}

} // namespace

// returns false when the level's shape is outside the instantiated range
bool launch_colsweep(int nin, int nout, int bw, const double2* const* ip, double2* const* op,
                     const int* in_begin, const SweepEntry* entries, const double2* rb,
                     const int* freal, size_t ncols, size_t s, int n, int nmax, cudaStream_t st) {
    const unsigned grid = (unsigned)((ncols + 127) / 128);
    bool ok = false;
    switch (nin) {
    case 1: ok = launch_out<1>(nout, bw, grid, st, ip, op, in_begin, entries, rb, freal, ncols, s, n, nmax); break;
    case 2: ok = launch_out<2>(nout, bw, grid, st, ip, op, in_begin, entries, rb, freal, ncols, s, n, nmax); break;
    case 3: ok = launch_out<3>(nout, bw, grid, st, ip, op, in_begin, entries, rb, freal, ncols, s, n, nmax); break;
    case 4: ok = launch_out<4>(nout, bw, grid, st, ip, op, in_begin, entries, rb, freal, ncols, s, n, nmax); break;
    case 5: ok = launch_out<5>(nout, bw, grid, st, ip, op, in_begin, entries, rb, freal, ncols, s, n, nmax); break;
    case 6: ok = launch_out<6>(nout, bw, grid, st, ip, op, in_begin, entries, rb, freal, ncols, s, n, nmax); break;
    case 7: ok = launch_out<7>(nout, bw, grid, st, ip, op, in_begin, entries, rb, freal, ncols, s, n, nmax); break;
    case 8: ok = launch_out<8>(nout, bw, grid, st, ip, op, in_begin, entries, rb, freal, ncols, s, n, nmax); break;
    default: ok = false;
    }
    if (ok) check_launch("k_kron_colsweep");
    return ok;
}

} // namespace ks
