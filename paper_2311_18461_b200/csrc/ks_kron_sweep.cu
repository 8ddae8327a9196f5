// Level pass kernel for the Kronecker-sum matvec (plan: ks_kron.cu).
//
// A CTA owns TQ consecutive columns (o, q) of the pass axis and their FULL
// extent r = 0..n-1, so every banded product is local. Input nodes are staged
// through shared memory one at a time (rows padded with BW zero rows at both
// ends, so the band loops have no edge branches); loads are coalesced along q
// for the spatial axes (s > 1) and along r for the contiguous time axis
// (s = 1). Each thread owns one column and RPT rows (r = rg + k*RG) and keeps
// NOUT x RPT complex accumulators in registers; the level's contributions are
// grouped by input node on the host (entries[in_begin[j] .. in_begin[j+1]]),
// and the output slot is chosen by a uniform switch so all register indices
// are static. Each input element is read from HBM once per pass and each
// output element written once. Band rows are pre-expanded row-major:
// rb[f][r][t] = F(r, r - BW + t).
#include "ks_internal.hpp"

namespace ks {

struct SweepEntry {
    int out;    // output node
    int factor; // -1 = identity
    double2 coeff;
};

namespace {

constexpr int kTileThreads = 256;
constexpr int kRPT = 5;

template <int NOUT, int BW>
__global__ void __launch_bounds__(kTileThreads, (NOUT <= 3 ? 2 : 1)) k_kron_tile(
    const double2* const* __restrict__ in_ptrs, int n_in, double2* const* __restrict__ out_ptrs,
    const int* __restrict__ in_begin, const SweepEntry* __restrict__ entries,
    const double2* __restrict__ rb, const int* __restrict__ freal, size_t ncols, size_t s, int n,
    int nmax, int TQ) {
    constexpr int TAPS = 2 * BW + 1;
    extern __shared__ double2 tile[]; // [n + 2BW][TQ + 1]
    const int tid = threadIdx.x;
    const int pitch = TQ + 1;
    const int RG = kTileThreads / TQ; // row groups
    const int cc = tid % TQ, rg = tid / TQ;
    const size_t c0 = (size_t)blockIdx.x * TQ;
    const int ncol = (int)min((size_t)TQ, ncols - c0);
    const double2 Z = make_double2(0.0, 0.0);

    // zero halo rows once (never overwritten)
    for (int e = tid; e < BW * pitch; e += kTileThreads) {
        tile[e] = Z;
        tile[(n + BW) * pitch + e] = Z;
    }

    double2 acc[NOUT][kRPT];
#pragma unroll
    for (int a = 0; a < NOUT; ++a)
#pragma unroll
        for (int k = 0; k < kRPT; ++k) acc[a][k] = Z;

    for (int j = 0; j < n_in; ++j) {
        const double2* __restrict__ in = in_ptrs[j];
        __syncthreads();
        const int tot = n * TQ;
        if (s == 1) {
            for (int e = tid; e < tot; e += kTileThreads) {
                const int c = e / n, r = e - c * n;
                tile[(r + BW) * pitch + c] = c < ncol ? __ldg(in + (c0 + c) * (size_t)n + r) : Z;
            }
        } else {
            for (int e = tid; e < tot; e += kTileThreads) {
                const int r = e / TQ, c = e - r * TQ;
                double2 v = Z;
                if (c < ncol) {
                    const size_t cm = c0 + c;
                    const size_t oo = cm / s, qq = cm - oo * s;
                    v = __ldg(in + oo * (size_t)n * s + (size_t)r * s + qq);
                }
                tile[(r + BW) * pitch + c] = v;
            }
        }
        __syncthreads();
        const int eb = in_begin[j], ee = in_begin[j + 1];
        for (int e = eb; e < ee; ++e) {
            const SweepEntry en = entries[e];
            const bool real = en.factor >= 0 && freal[en.factor];
            double2 v[kRPT];
#pragma unroll
            for (int k = 0; k < kRPT; ++k) {
                const int r = rg + k * RG;
                v[k] = Z;
                if (r < n) {
                    const double2* t0 = tile + r * pitch + cc; // row r - BW (padded)
                    if (en.factor < 0) {
                        v[k] = t0[BW * pitch];
                    } else {
                        const double2* band = rb + ((size_t)en.factor * nmax + r) * TAPS;
                        double vr = 0.0, vi = 0.0;
                        if (real) {
#pragma unroll
                            for (int t = 0; t < TAPS; ++t) {
                                const double a = __ldg(&band[t].x);
                                const double2 x = t0[t * pitch];
                                vr = fma(a, x.x, vr);
                                vi = fma(a, x.y, vi);
                            }
                        } else {
#pragma unroll
                            for (int t = 0; t < TAPS; ++t) {
                                const double2 a = __ldg(&band[t]);
                                const double2 x = t0[t * pitch];
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
            _Pragma("unroll") for (int k = 0; k < kRPT; ++k) {                     \
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
    }
    if (cc >= ncol) return;
    const size_t cme = c0 + cc;
    const size_t o = cme / s, q = cme - o * s;
    const size_t base = o * (size_t)n * s + q;
#pragma unroll
    for (int a = 0; a < NOUT; ++a) {
        double2* __restrict__ out = out_ptrs[a];
#pragma unroll
        for (int k = 0; k < kRPT; ++k) {
            const int r = rg + k * RG;
            if (r < n) out[base + (size_t)r * s] = acc[a][k];
        }
    }
}

template <int NOUT>
void launch_bw(int bw, unsigned grid, size_t sm, cudaStream_t st, const double2* const* ip, int nin,
               double2* const* op, const int* ib, const SweepEntry* en, const double2* rb,
               const int* fr, size_t ncols, size_t s, int n, int nmax, int TQ) {
    switch (bw) {
    case 1: k_kron_tile<NOUT, 1><<<grid, kTileThreads, sm, st>>>(ip, nin, op, ib, en, rb, fr, ncols, s, n, nmax, TQ); break;
    case 2: k_kron_tile<NOUT, 2><<<grid, kTileThreads, sm, st>>>(ip, nin, op, ib, en, rb, fr, ncols, s, n, nmax, TQ); break;
    case 3: k_kron_tile<NOUT, 3><<<grid, kTileThreads, sm, st>>>(ip, nin, op, ib, en, rb, fr, ncols, s, n, nmax, TQ); break;
    default: k_kron_tile<NOUT, 4><<<grid, kTileThreads, sm, st>>>(ip, nin, op, ib, en, rb, fr, ncols, s, n, nmax, TQ); break;
    }
}

} // namespace

// returns false when the level's shape is outside the instantiated range
bool launch_colsweep(int nin, int nout, int bw, const double2* const* ip, double2* const* op,
                     const int* in_begin, const SweepEntry* entries, const double2* rb,
                     const int* freal, size_t ncols, size_t s, int n, int nmax, cudaStream_t st) {
    if (nout < 1 || nout > 8 || bw < 1 || bw > 4) return false;
    int TQ = 16;
    while (TQ > 1 && (n + kTileThreads / TQ - 1) / (kTileThreads / TQ) > kRPT) TQ /= 2;
    if ((n + kTileThreads / TQ - 1) / (kTileThreads / TQ) > kRPT) return false;
    const size_t sm = (size_t)(n + 2 * bw) * (TQ + 1) * sizeof(double2);
    if (sm > 200 * 1024) return false;
    const unsigned grid = (unsigned)((ncols + TQ - 1) / TQ);
    switch (nout) {
    case 1: launch_bw<1>(bw, grid, sm, st, ip, nin, op, in_begin, entries, rb, freal, ncols, s, n, nmax, TQ); break;
    case 2: launch_bw<2>(bw, grid, sm, st, ip, nin, op, in_begin, entries, rb, freal, ncols, s, n, nmax, TQ); break;
    case 3: launch_bw<3>(bw, grid, sm, st, ip, nin, op, in_begin, entries, rb, freal, ncols, s, n, nmax, TQ); break;
    case 4: launch_bw<4>(bw, grid, sm, st, ip, nin, op, in_begin, entries, rb, freal, ncols, s, n, nmax, TQ); break;
    case 5: launch_bw<5>(bw, grid, sm, st, ip, nin, op, in_begin, entries, rb, freal, ncols, s, n, nmax, TQ); break;
    case 6: launch_bw<6>(bw, grid, sm, st, ip, nin, op, in_begin, entries, rb, freal, ncols, s, n, nmax, TQ); break;
    case 7: launch_bw<7>(bw, grid, sm, st, ip, nin, op, in_begin, entries, rb, freal, ncols, s, n, nmax, TQ); break;
    case 8: launch_bw<8>(bw, grid, sm, st, ip, nin, op, in_begin, entries, rb, freal, ncols, s, n, nmax, TQ); break;
    }
    check_launch("k_kron_tile");
    return true;
}

} // namespace ks
