// Per-spatial-eigenvalue time blocks of the FD preconditioner: build,
// factor (partial-pivot banded LU) and solve, one time fiber per thread.
//
// Reference:
//   composite eigenvalue   lambda_i = sum_l lambda_l[i_l], axis 1 fastest
//                          (src/fdsolver.cpp:30-42)
//   block                  H_i = Lt + nu^2 lambda_i^2 Mt + nu lambda_i (W + W^H)
//                          (src/fdsolver.cpp:95-120; exact expression :115-116)
//   factor                 factor_banded (src/eigensolve.cpp:77-121):
//                          kl = p, ku_f = 2p, ldab = 3p+1, pivot = first argmax |a(i,k)|
//                          over i in [k, k+kl], singular if max == 0, row swap over
//                          [k, k+ku_f], multipliers stored in place
//   solve                  solve_banded (src/eigensolve.cpp:123-140)
//   adjoint solve          solve_banded_adjoint (src/eigensolve.cpp:148-170)
//
// Device layout (fd_band_index, ks_internal.hpp): per-block records by
// default -- band column k of block b is ab[(b*nt + k)*rec + e], e < ldab,
// with the pivot offset piv[k]-k stored as a double in slot ldab -- so one
// fiber's step reads one contiguous 128 B record (p = 2) whichever block its
// fiber maps to (with deduplication a warp's 32 fibers hit scattered blocks;
// the earlier block-interleaved layout ab[(k*ldab + e)*nblk + b] wasted half of
// every 32 B sector there and is kept as KS_FD_REC=0).
//
// Block deduplication: when all spatial axes carry the
// same 1-D eigenvalues (uniform identical meshes, every BASELINE config), the
// composite eigenvalue is symmetric under permutations of (i_1..i_d), so only
// the sorted multi-indices a <= b <= c are factored (45,760 instead of
// 262,144 blocks at c3) and fiber i reads block fiber_block[i]. Block lambda is
// summed in the reference's order for the sorted index; a permuted fiber's own
// reference sum can differ from it by one ulp (rounding only). The solve keeps the (p+1)-wide
// forward and (2p+1)-wide backward elimination windows in registers
// (compile-time p), so each tensor entry is read and written once per sweep.
//
// Complex arithmetic follows the reference's std::complex<double> operations:
// products (ac-bd, ad+bc), Smith-style division as in libgcc's __divdc3, and
// |z| = hypot(re, im) for the pivot search.
#include "ks_internal.hpp"

#include <cstdlib>
#include <cstring>

namespace ks {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconjmul(double2 a, double2 b) { // conj(a) * b
    return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
    return make_double2(a.x - b.x, a.y - b.y);
}
// (a + ib) / (c + id), Smith's algorithm as in libgcc __divdc3
__device__ __forceinline__ double2 cdiv(double2 num, double2 den) {
    const double a = num.x, b = num.y, c = den.x, d = den.y;
    double x, y;
    if (fabs(c) < fabs(d)) {
        const double ratio = c / d;
        const double denom = (c * ratio) + d;
        x = ((a * ratio) + b) / denom;
        y = ((b * ratio) - a) / denom;
    } else {
        const double ratio = d / c;
        const double denom = (d * ratio) + c;
        x = ((b * ratio) + a) / denom;
        y = (b - (a * ratio)) / denom;
    }
    return make_double2(x, y);
}
__device__ __forceinline__ double cabs_(double2 a) { return hypot(a.x, a.y); }

// ---------------------------------------------------------------------------
// factor: one thread per fiber; builds H(lambda_i) into the interleaved band
// and eliminates in place.
// ---------------------------------------------------------------------------
__global__ void k_fd_factor(double2* __restrict__ ab, unsigned char* __restrict__ piv,
                            int* __restrict__ flag, unsigned char* __restrict__ wpiv,
                            unsigned char* __restrict__ bpiv, size_t ns, int nt, int p,
                            const double* __restrict__ lam_blk, double nu,
                            const double* __restrict__ Lt, const double* __restrict__ Mt,
                            const double2* __restrict__ Wsym, int rec, int fused_nd, long long fused_np,
                            int kind) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= ns) return; // here ns = number of factored blocks
    const int ldab = 3 * p + 1, kuf = 2 * p, bwld = 2 * p + 1;
    const BandIndex bx = fd_band_index(i, nt, ldab, ns, rec, fused_nd, fused_np);
    const size_t base = bx.fb, estr = bx.fe, kstr = bx.fk;
    // composite eigenvalue lambda_i = sum_l lambda_l[i_l], formed on the host in
    // the reference's summation order (fdsolver.cpp:30-42)
    const double lam = lam_blk[i];
    auto A = [&](int r, int c) -> double2& {
        return ab[base + (size_t)c * kstr + (size_t)(kuf + r - c) * estr];
    };
    // fill: zero band, then H(r, c) for |r - c| <= p
    for (int c = 0; c < nt; ++c)
        for (int e = 0; e < (rec > 0 ? rec : ldab); ++e)
            ab[base + (size_t)c * kstr + (size_t)e * estr] = make_double2(0.0, 0.0);
    const double s2 = nu * nu * lam * lam; // nu*nu*lam*lam (left to right)
    const double s1 = nu * lam;
    for (int c = 0; c < nt; ++c) {
        const int r0 = c - p < 0 ? 0 : c - p, r1 = c + p > nt - 1 ? nt - 1 : c + p;
        for (int r = r0; r <= r1; ++r) {
            const int bi = p + r - c + c * bwld;
            const double2 w = Wsym[bi];
            double re, im;
            if (kind == 1) {
                // galerkin_fast_solver (fdsolver.cpp:177-191): Wt(i,j) + nu*lam*Mt(i,j)
                re = __dadd_rn(w.x, __dmul_rn(s1, Mt[bi]));
                im = __dadd_rn(w.y, __dmul_rn(s1, 0.0));
            } else {
                // Lt(i,j) + nu*nu*lam*lam*Mt(i,j) + nu*lam*Wsym(i,j), complex
                re = __dadd_rn(Lt[bi], __dmul_rn(s2, Mt[bi]));
                im = 0.0; // Lt, Mt have zero imaginary parts (to_complex)
                re = __dadd_rn(re, __dmul_rn(s1, w.x));
                im = __dadd_rn(im, __dmul_rn(s1, w.y));
            }
            A(r, c) = make_double2(re, im);
        }
    }
    // partial-pivot banded LU (eigensolve.cpp:93-119)
    bool swapped = false; // any row interchange: flag bit 1 (the solves then read the fill-in rows)
    struct SwapFlag {
        bool& s;
        int* f;
        unsigned char* w;
        unsigned char* bp;
        size_t i;
        __device__ ~SwapFlag() {
            if (s) {
                atomicOr(f, 2);
                w[i >> 5] = 1; // every writer stores 1
            }
            bp[i] = s ? 1 : 0;
        }
    } swap_flag{swapped, flag, wpiv, bpiv, i};
    for (int k = 0; k < nt; ++k) {
        const int imax = k + p < nt - 1 ? k + p : nt - 1;
        int pr = k;
        double best = cabs_(A(k, k));
        for (int r = k + 1; r <= imax; ++r) {
            const double v = cabs_(A(r, k));
            if (v > best) {
                best = v;
                pr = r;
            }
        }
        if (rec > 0) ab[base + (size_t)k * kstr + ldab] = make_double2((double)(pr - k), 0.0);
        else piv[bx.pb + (size_t)k * bx.pk] = (unsigned char)(pr - k);
        if (best == 0.0) {
            atomicOr(flag, 1);
            return;
        }
        swapped |= pr != k;
        const int jmax = k + kuf < nt - 1 ? k + kuf : nt - 1;
        if (pr != k)
            for (int c = k; c <= jmax; ++c) {
                const double2 t = A(k, c);
                A(k, c) = A(pr, c);
                A(pr, c) = t;
            }
        const double2 pivval = A(k, k);
        for (int r = k + 1; r <= imax; ++r) {
            const double2 m = cdiv(A(r, k), pivval);
            A(r, k) = m;
            if (m.x != 0.0 || m.y != 0.0)
                for (int c = k + 1; c <= jmax; ++c) A(r, c) = csub(A(r, c), cmul(m, A(k, c)));
        }
    }
}

// ---------------------------------------------------------------------------
// solve: x <- H_i^{-1} x on fiber i (contiguous nt complex at X + i*nt)
// ---------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(128) k_fd_solve(const double2* __restrict__ ab,
                                                  const unsigned char* __restrict__ piv,
                                                  double2* __restrict__ X, size_t ns, int nt,
                                                  size_t nblk, const int* __restrict__ fblk,
                                                  int tmajor, int rec, int fnd, long long fnp, int pfd) {
    const size_t f = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (f >= ns) return;
    constexpr int ldab = 3 * P + 1, kuf = 2 * P;
    // fiber f: contiguous (X[f][t]) or time-major (X[t][f], coalesced across threads)
    double2* x0 = tmajor ? X + f : X + f * (size_t)nt;
    const size_t xs = tmajor ? ns : 1;
    struct XA {
        double2* p;
        size_t s;
        __device__ double2& operator[](int k) const { return p[(size_t)k * s]; }
    } x{x0, xs};
    const size_t i = fblk ? (size_t)__ldg(fblk + f) : f; // factored block of this fiber
    const BandIndex bx = fd_band_index(i, nt, ldab, nblk, rec, fnd, fnp);
    auto band = [&](int k, int e) -> double2 { return __ldg(ab + bx.fb + (size_t)k * bx.fk + (size_t)e * bx.fe); };
    auto pivot = [&](int k) -> int {
        return rec > 0 ? (int)__ldg(&ab[bx.fb + (size_t)k * bx.fk + ldab].x) : (int)piv[bx.pb + (size_t)k * bx.pk];
    };
    // Each step's band row, pivot and the x entry entering the window are
    // loaded one step ahead into registers (the loads of step k+1 are in
    // flight while step k computes), and pfd > 0 adds an L2 prefetch of step
    // k+pfd (no registers).
    auto pf = [&](const void* a) { asm volatile("prefetch.global.L2 [%0];" ::"l"(a)); };
    // forward: L with row interchanges (eigensolve.cpp:127-133); w[m] = x[k+m]
    double2 w[P + 1];
#pragma unroll
    for (int m = 0; m <= P; ++m) w[m] = m < nt ? x[m] : make_double2(0.0, 0.0);
    double2 lb[P], xn;
    int po_n;
    auto load_f = [&](int k) {
#pragma unroll
        for (int m = 1; m <= P; ++m) lb[m - 1] = (k + m < nt) ? band(k, kuf + m) : make_double2(0.0, 0.0);
        po_n = pivot(k);
        xn = (k + P + 1 < nt) ? x[k + P + 1] : make_double2(0.0, 0.0);
    };
    load_f(0);
    for (int k = 0; k < nt; ++k) {
        double2 l[P];
#pragma unroll
        for (int m = 0; m < P; ++m) l[m] = lb[m];
        const int po = po_n;
        const double2 xin = xn;
        if (k + 1 < nt) load_f(k + 1);
        if (pfd > 0 && k + pfd < nt) {
            const int kp = k + pfd;
            pf(ab + bx.fb + (size_t)kp * bx.fk + (size_t)(kuf + 1) * bx.fe);
            if (rec == 0) pf(piv + bx.pb + (size_t)kp * bx.pk);
            if (kp + P + 1 < nt) pf(&x[kp + P + 1]);
        }
#pragma unroll
        for (int m = 1; m <= P; ++m)
            if (po == m) {
                const double2 t = w[0];
                w[0] = w[m];
                w[m] = t;
            }
#pragma unroll
        for (int m = 1; m <= P; ++m)
            if (k + m < nt) w[m] = csub(w[m], cmul(l[m - 1], w[0]));
        x[k] = w[0];
#pragma unroll
        for (int m = 0; m < P; ++m) w[m] = w[m + 1];
        w[P] = xin;
    }
    // backward: U, column oriented (eigensolve.cpp:134-139); u[j] = x[k-j]
    double2 u[2 * P + 1];
#pragma unroll
    for (int j = 0; j <= 2 * P; ++j) u[j] = (nt - 1 - j >= 0) ? x[nt - 1 - j] : make_double2(0.0, 0.0);
    double2 ub[2 * P + 1];
    auto load_b = [&](int k) {
#pragma unroll
        for (int j = 0; j <= 2 * P; ++j) ub[j] = (k - j >= 0) ? band(k, kuf - j) : make_double2(0.0, 0.0);
        xn = (k - 2 * P - 1 >= 0) ? x[k - 2 * P - 1] : make_double2(0.0, 0.0);
    };
    load_b(nt - 1);
    for (int k = nt - 1; k >= 0; --k) {
        double2 ucol[2 * P + 1];
#pragma unroll
        for (int j = 0; j <= 2 * P; ++j) ucol[j] = ub[j];
        const double2 xin = xn;
        if (k > 0) load_b(k - 1);
        if (pfd > 0 && k - pfd >= 0) {
            const int kp = k - pfd;
            pf(ab + bx.fb + (size_t)kp * bx.fk);
            if (kp - 2 * P - 1 >= 0) pf(&x[kp - 2 * P - 1]);
        }
        u[0] = cdiv(u[0], ucol[0]);
#pragma unroll
        for (int j = 1; j <= 2 * P; ++j)
            if (k - j >= 0) u[j] = csub(u[j], cmul(ucol[j], u[0]));
        x[k] = u[0];
#pragma unroll
        for (int j = 0; j < 2 * P; ++j) u[j] = u[j + 1];
        u[2 * P] = xin;
    }
}

// adjoint: H_i^{-H} x (eigensolve.cpp:148-170)
template <int P>
__global__ void __launch_bounds__(128) k_fd_solve_adj(const double2* __restrict__ ab,
                                                      const unsigned char* __restrict__ piv,
                                                      double2* __restrict__ X, size_t ns, int nt,
                                                      size_t nblk, const int* __restrict__ fblk,
                                                  int tmajor, int rec, int fnd, long long fnp) {
    const size_t f = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (f >= ns) return;
    constexpr int ldab = 3 * P + 1, kuf = 2 * P;
    // fiber f: contiguous (X[f][t]) or time-major (X[t][f], coalesced across threads)
    double2* x0 = tmajor ? X + f : X + f * (size_t)nt;
    const size_t xs = tmajor ? ns : 1;
    struct XA {
        double2* p;
        size_t s;
        __device__ double2& operator[](int k) const { return p[(size_t)k * s]; }
    } x{x0, xs};
    const size_t i = fblk ? (size_t)__ldg(fblk + f) : f;
    const BandIndex bx = fd_band_index(i, nt, ldab, nblk, rec, fnd, fnp);
    auto band = [&](int k, int e) -> double2 { return __ldg(ab + bx.fb + (size_t)k * bx.fk + (size_t)e * bx.fe); };
    auto pivot = [&](int k) -> int {
        return rec > 0 ? (int)__ldg(&ab[bx.fb + (size_t)k * bx.fk + ldab].x) : (int)piv[bx.pb + (size_t)k * bx.pk];
    };
    // U^H z = y, forward; h[j] = x[k - 2P + j] (finalised values)
    double2 h[2 * P];
#pragma unroll
    for (int j = 0; j < 2 * P; ++j) h[j] = make_double2(0.0, 0.0);
    for (int k = 0; k < nt; ++k) {
        double2 s = x[k];
#pragma unroll
        for (int j = 0; j < 2 * P; ++j) {
            const int r = k - 2 * P + j; // row index i, ascending
            if (r >= 0) s = csub(s, cconjmul(band(k, kuf + r - k), h[j]));
        }
        const double2 dk = band(k, kuf);
        s = cdiv(s, make_double2(dk.x, -dk.y));
        x[k] = s;
#pragma unroll
        for (int j = 0; j < 2 * P - 1; ++j) h[j] = h[j + 1];
        h[2 * P - 1] = s;
    }
    // L^H w = z with swaps in reverse; g[m] = x[k+m]
    double2 g[P + 1];
#pragma unroll
    for (int m = 0; m <= P; ++m) {
        const int r = nt - 1 + m;
        g[m] = r < nt ? x[r] : make_double2(0.0, 0.0);
    }
    for (int k = nt - 1; k >= 0; --k) {
        double2 s = g[0];
#pragma unroll
        for (int m = 1; m <= P; ++m)
            if (k + m < nt) s = csub(s, cconjmul(band(k, kuf + m), g[m]));
        g[0] = s;
        const int po = pivot(k);
#pragma unroll
        for (int m = 1; m <= P; ++m)
            if (po == m) {
                const double2 t = g[0];
                g[0] = g[m];
                g[m] = t;
            }
        if (k + P < nt) x[k + P] = g[P];
#pragma unroll
        for (int m = P; m > 0; --m) g[m] = g[m - 1];
        g[0] = k - 1 >= 0 ? x[k - 1] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int m = 1; m <= P; ++m)
        if (m - 1 < nt) x[m - 1] = g[m];
}

// ---------------------------------------------------------------------------
// ring solve (time-major fibers): the same sweeps as k_fd_solve, but each
// thread streams its band entries, pivot words and incoming x entries through
// a private D-step cp.async ring in shared memory ([slot][entry][thread], so a
// warp's 16 B accesses are contiguous), keeping D-1 steps of loads in flight
// without holding them in registers. Threads never share slots, so no
// barriers: cp.async.wait_group orders each thread's own copies.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cpa16(void* sdst, const void* g, bool v) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(g), "r"(v ? 16 : 0));
}
__device__ __forceinline__ void cpa4(void* sdst, const void* g, bool v) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(g), "r"(v ? 4 : 0));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// NP: this warp's fibers' blocks did not pivot (see k_fd_solve_pair)
template <int P, int D, int TB, bool NP>
__device__ __forceinline__ void fd_ring_body(const double2* __restrict__ ab, const unsigned char* __restrict__ piv,
                                             double2* __restrict__ X, size_t ns, int nt, size_t nblk,
                                             const int* __restrict__ fblk, int rec, int fnd, long long fnp,
                                             double2* ring, size_t f) {
    constexpr int ldab = 3 * P + 1, kuf = 2 * P, NE = 2 * P + 2;
    unsigned* pr = reinterpret_cast<unsigned*>(ring + (size_t)D * NE * TB);
    const int t = threadIdx.x;
    double2* x = X + f; // x[k * ns]
    const size_t i = fblk ? (size_t)__ldg(fblk + f) : f;
    const BandIndex bx = fd_band_index(i, nt, ldab, nblk, rec, fnd, fnp);
    auto slot = [&](int k, int e) -> double2* { return ring + ((size_t)((k % D) * NE + e) * TB + t); };
    auto baddr = [&](int k, int e) -> const double2* { return ab + bx.fb + (size_t)k * bx.fk + (size_t)e * bx.fe; };
    // pivot of step k: byte (or record slot) -> 4 B word in the ring
    auto issue_f = [&](int k) {
        if (k < nt) {
#pragma unroll
            for (int m = 1; m <= P; ++m) cpa16(slot(k, m - 1), k + m < nt ? baddr(k, kuf + m) : ab, k + m < nt);
            cpa16(slot(k, P), k + P + 1 < nt ? x + (size_t)(k + P + 1) * ns : X, k + P + 1 < nt);
            if (NP) {
            } else if (rec > 0) {
                cpa16(slot(k, P + 1), baddr(k, ldab), true);
            } else {
                const size_t o = bx.pb + (size_t)k * bx.pk;
                cpa4(pr + (k % D) * TB + t, piv + (o & ~(size_t)3), true);
            }
        }
        cpa_commit();
    };
    auto pivot_of = [&](int k) -> int {
        if (NP) return 0;
        if (rec > 0) return (int)slot(k, P + 1)->x;
        const size_t o = bx.pb + (size_t)k * bx.pk;
        return (int)((pr[(k % D) * TB + t] >> (8 * (unsigned)(o & 3))) & 0xffu);
    };
    // forward: L with row interchanges (eigensolve.cpp:127-133); w[m] = x[k+m]
    double2 w[P + 1];
#pragma unroll
    for (int m = 0; m <= P; ++m) w[m] = m < nt ? x[(size_t)m * ns] : make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < D - 1; ++k) issue_f(k);
    for (int k = 0; k < nt; ++k) {
        cpa_wait<D - 2>();
        issue_f(k + D - 1);
        const int po = pivot_of(k);
#pragma unroll
        for (int m = 1; m <= P; ++m)
            if (po == m) {
                const double2 tt = w[0];
                w[0] = w[m];
                w[m] = tt;
            }
#pragma unroll
        for (int m = 1; m <= P; ++m)
            if (k + m < nt) w[m] = csub(w[m], cmul(*slot(k, m - 1), w[0]));
        x[(size_t)k * ns] = w[0];
        const double2 xin = *slot(k, P);
#pragma unroll
        for (int m = 0; m < P; ++m) w[m] = w[m + 1];
        w[P] = xin;
    }
    cpa_wait<0>();
    // backward: U, column oriented (eigensolve.cpp:134-139); u[j] = x[k-j]
    auto issue_b = [&](int k) {
        if (k >= 0) {
#pragma unroll
            for (int j = 0; j <= (NP ? P : 2 * P); ++j) cpa16(slot(k, j), k - j >= 0 ? baddr(k, kuf - j) : ab, k - j >= 0);
            const int kx = k - 2 * P - 1;
            cpa16(slot(k, 2 * P + 1), kx >= 0 ? x + (size_t)kx * ns : X, kx >= 0);
        }
        cpa_commit();
    };
    double2 u[2 * P + 1];
#pragma unroll
    for (int j = 0; j <= 2 * P; ++j) u[j] = (nt - 1 - j >= 0) ? x[(size_t)(nt - 1 - j) * ns] : make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < D - 1; ++q) issue_b(nt - 1 - q);
    for (int k = nt - 1; k >= 0; --k) {
        cpa_wait<D - 2>();
        issue_b(k - (D - 1));
        // slot index of step k: use (nt-1-k) so the ring advances monotonically
        { // reciprocal conj(d)/|d|^2: one division on the step's latency chain instead of Smith's three
            const double2 dg = *slot(k, 0);
            const double sc = 1.0 / fma(dg.x, dg.x, dg.y * dg.y);
            u[0] = cmul(u[0], make_double2(dg.x * sc, -dg.y * sc));
        }
#pragma unroll
        for (int j = 1; j <= (NP ? P : 2 * P); ++j)
            if (k - j >= 0) u[j] = csub(u[j], cmul(*slot(k, j), u[0]));
        x[(size_t)k * ns] = u[0];
        const double2 xin = *slot(k, 2 * P + 1);
#pragma unroll
        for (int j = 0; j < 2 * P; ++j) u[j] = u[j + 1];
        u[2 * P] = xin;
    }
}

// wpivf[f / 32] != 0: one of the 32 fibers' blocks pivoted (built after the
// factorisation); null: full band everywhere
template <int P, int D, int TB = 128>
__global__ void __launch_bounds__(TB) k_fd_solve_ring(const double2* __restrict__ ab,
                                                       const unsigned char* __restrict__ piv,
                                                       double2* __restrict__ X, size_t ns, int nt, size_t nblk,
                                                       const int* __restrict__ fblk, int rec, int fnd,
                                                       long long fnp, const unsigned char* __restrict__ wpivf) {
    extern __shared__ __align__(16) double2 ring[]; // [D][NE][TB], then int [D][TB]
    const size_t f = blockIdx.x * (size_t)TB + threadIdx.x;
    if (f >= ns) return;
    if (wpivf && __ldg(wpivf + (f >> 5)) == 0)
        fd_ring_body<P, D, TB, true>(ab, piv, X, ns, nt, nblk, fblk, rec, fnd, fnp, ring, f);
    else
        fd_ring_body<P, D, TB, false>(ab, piv, X, ns, nt, nblk, fblk, rec, fnd, fnp, ring, f);
}

// per-fiber-group pivot flags for the ring solve from the per-block flags
__global__ void k_fiber_piv(const unsigned char* __restrict__ bpiv, const int* __restrict__ fblk, size_t ns,
                            unsigned char* __restrict__ wpivf) {
    const size_t f = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (f >= ns) return;
    const size_t i = fblk ? (size_t)fblk[f] : f;
    if (bpiv[i]) wpivf[f >> 5] = 1;
}

// ---------------------------------------------------------------------------
// pair solve (d = 3, axes 2 and 3 identical): block b = i1 + n1 * pidx(i2 <= i3)
// serves the fibers (i1, i2, i3) and (i1, i3, i2), which one thread solves
// together (two right-hand sides, one factor read). Consecutive threads take
// consecutive i1, so band reads (block-interleaved layout) and both fibers'
// time-major x accesses coalesce. Loads go through the per-thread cp.async ring
// as in k_fd_solve_ring.
// ---------------------------------------------------------------------------
#ifndef KS_PAIR_RECIP
#define KS_PAIR_RECIP 1
#endif
// NP: no block pivoted (FdBlocks::nopiv): pivot offsets not read, and the
// backward sweep reads U's p+1 rows instead of the 2p+1 of the fill-in band --
// the skipped entries are exact zeros, so the result is bit-identical
template <int P, int D, bool NP>
__device__ __forceinline__ void fd_pair_body(const double2* __restrict__ ab, const unsigned char* __restrict__ piv,
                                             double2* __restrict__ X, size_t ns, int nt, size_t nblk, int n1, int n2,
                                             const int2* __restrict__ pairs, double2* ring, size_t b) {
    constexpr int kuf = 2 * P, NE = 2 * P + 3;
    unsigned* pr = reinterpret_cast<unsigned*>(ring + (size_t)D * NE * 128);
    const int t = threadIdx.x;
    const int i1 = (int)(b % (size_t)n1);
    const int2 q = __ldg(pairs + b / (size_t)n1);
    const bool hb = q.x != q.y;
    double2* xa = X + (size_t)i1 + (size_t)n1 * ((size_t)q.x + (size_t)n2 * q.y);
    double2* xb = X + (size_t)i1 + (size_t)n1 * ((size_t)q.y + (size_t)n2 * q.x);
    auto slot = [&](int k, int e) -> double2* { return ring + ((size_t)((k % D) * NE + e) * 128 + t); };
    auto baddr = [&](int k, int e) -> const double2* { return ab + b + ((size_t)k * (3 * P + 1) + e) * nblk; };
    auto issue_f = [&](int k) {
        if (k < nt) {
#pragma unroll
            for (int m = 1; m <= P; ++m) cpa16(slot(k, m - 1), k + m < nt ? baddr(k, kuf + m) : ab, k + m < nt);
            const int kx = k + P + 1;
            cpa16(slot(k, P), kx < nt ? xa + (size_t)kx * ns : X, kx < nt);
            cpa16(slot(k, P + 1), kx < nt && hb ? xb + (size_t)kx * ns : X, kx < nt && hb);
            if (!NP) {
                const size_t o = (size_t)k * nblk + b;
                cpa4(pr + (k % D) * 128 + t, piv + (o & ~(size_t)3), true);
            }
        }
        cpa_commit();
    };
    // forward: L with row interchanges (eigensolve.cpp:127-133)
    double2 wa[P + 1], wb[P + 1];
#pragma unroll
    for (int m = 0; m <= P; ++m) {
        wa[m] = m < nt ? xa[(size_t)m * ns] : make_double2(0.0, 0.0);
        wb[m] = m < nt && hb ? xb[(size_t)m * ns] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int k = 0; k < D - 1; ++k) issue_f(k);
    for (int k = 0; k < nt; ++k) {
        cpa_wait<D - 2>();
        issue_f(k + D - 1);
        const size_t o = (size_t)k * nblk + b;
        const int po = NP ? 0 : (int)((pr[(k % D) * 128 + t] >> (8 * (unsigned)(o & 3))) & 0xffu);
#pragma unroll
        for (int m = 1; m <= P; ++m)
            if (po == m) {
                double2 tt = wa[0];
                wa[0] = wa[m];
                wa[m] = tt;
                tt = wb[0];
                wb[0] = wb[m];
                wb[m] = tt;
            }
#pragma unroll
        for (int m = 1; m <= P; ++m)
            if (k + m < nt) {
                const double2 l = *slot(k, m - 1);
                wa[m] = csub(wa[m], cmul(l, wa[0]));
                wb[m] = csub(wb[m], cmul(l, wb[0]));
            }
        xa[(size_t)k * ns] = wa[0];
        if (hb) xb[(size_t)k * ns] = wb[0];
        const double2 ina = *slot(k, P), inb = *slot(k, P + 1);
#pragma unroll
        for (int m = 0; m < P; ++m) {
            wa[m] = wa[m + 1];
            wb[m] = wb[m + 1];
        }
        wa[P] = ina;
        wb[P] = inb;
    }
    cpa_wait<0>();
    // backward: U, column oriented (eigensolve.cpp:134-139)
    auto issue_b = [&](int k) {
        if (k >= 0) {
#pragma unroll
            for (int j = 0; j <= (NP ? P : 2 * P); ++j) cpa16(slot(k, j), k - j >= 0 ? baddr(k, kuf - j) : ab, k - j >= 0);
            const int kx = k - 2 * P - 1;
            cpa16(slot(k, 2 * P + 1), kx >= 0 ? xa + (size_t)kx * ns : X, kx >= 0);
            cpa16(slot(k, 2 * P + 2), kx >= 0 && hb ? xb + (size_t)kx * ns : X, kx >= 0 && hb);
        }
        cpa_commit();
    };
    double2 ua[2 * P + 1], ub[2 * P + 1];
#pragma unroll
    for (int j = 0; j <= 2 * P; ++j) {
        const bool v = nt - 1 - j >= 0;
        ua[j] = v ? xa[(size_t)(nt - 1 - j) * ns] : make_double2(0.0, 0.0);
        ub[j] = v && hb ? xb[(size_t)(nt - 1 - j) * ns] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int qq = 0; qq < D - 1; ++qq) issue_b(nt - 1 - qq);
    for (int k = nt - 1; k >= 0; --k) {
        cpa_wait<D - 2>();
        issue_b(k - (D - 1));
        const double2 dg = *slot(k, 0);
        if (KS_PAIR_RECIP) { // one reciprocal for both fibers (rounding-level change)
            const double sc = 1.0 / fma(dg.x, dg.x, dg.y * dg.y);
            const double2 rd = make_double2(dg.x * sc, -dg.y * sc);
            ua[0] = cmul(ua[0], rd);
            ub[0] = cmul(ub[0], rd);
        } else {
            ua[0] = cdiv(ua[0], dg);
            ub[0] = cdiv(ub[0], dg);
        }
#pragma unroll
        for (int j = 1; j <= (NP ? P : 2 * P); ++j)
            if (k - j >= 0) {
                const double2 uu = *slot(k, j);
                ua[j] = csub(ua[j], cmul(uu, ua[0]));
                ub[j] = csub(ub[j], cmul(uu, ub[0]));
            }
        xa[(size_t)k * ns] = ua[0];
        if (hb) xb[(size_t)k * ns] = ub[0];
        const double2 ina = *slot(k, 2 * P + 1), inb = *slot(k, 2 * P + 2);
#pragma unroll
        for (int j = 0; j < 2 * P; ++j) {
            ua[j] = ua[j + 1];
            ub[j] = ub[j + 1];
        }
        ua[2 * P] = ina;
        ub[2 * P] = inb;
    }
}

// Warp-uniform choice per group of 32 blocks: wpiv[b / 32] != 0 when one of
// them pivoted (factor kernel). Only the smallest-eigenvalue blocks pivot
// (c3: the first ~0.01%), so nearly every warp takes the NP body. wpiv null:
// full band everywhere (KS_FD_NOPIV=0).
template <int P, int D>
__global__ void __launch_bounds__(128) k_fd_solve_pair(const double2* __restrict__ ab,
                                                       const unsigned char* __restrict__ piv,
                                                       double2* __restrict__ X, size_t ns, int nt, size_t nblk,
                                                       int n1, int n2, const int2* __restrict__ pairs,
                                                       const unsigned char* __restrict__ wpiv) {
    extern __shared__ __align__(16) double2 ring[]; // [D][NE][128], then unsigned [D][128]
    const size_t b = blockIdx.x * (size_t)128 + threadIdx.x;
    if (b >= nblk) return;
    if (wpiv && __ldg(wpiv + (b >> 5)) == 0)
        fd_pair_body<P, D, true>(ab, piv, X, ns, nt, nblk, n1, n2, pairs, ring, b);
    else
        fd_pair_body<P, D, false>(ab, piv, X, ns, nt, nblk, n1, n2, pairs, ring, b);
}

// ---------------------------------------------------------------------------
// Pair-mode solve on the NATURAL layout (t fastest: fiber i is the contiguous
// run X[i*nt .. i*nt + nt)), so the FD apply needs no time-major hand-off and
// its outermost-axis transforms run in the plain column mode (c3: 0.77 vs
// 0.85 ms for the six transforms). A CTA of T threads owns T consecutive
// blocks and their 2T fibers (pair mode: thread = block b = (i1, pair (i2,i3)),
// fibers (i1,i2,i3) and (i1,i3,i2)) and sweeps time in chunks of C steps:
// each chunk's fiber rows (2T segments of C*16 B), band entries (block-
// interleaved: T consecutive blocks = one contiguous run per entry) and the
// forward outputs move between HBM and shared memory CTA-wide with cp.async
// (double-buffered), while each thread runs the same register-window
// elimination as k_fd_solve_pair on its two fibers from shared memory.
// Forward (L, with the row interchanges) writes its outputs back to X; the
// backward sweep (U) reads them in reverse chunks. Same arithmetic, same
// order as k_fd_solve_pair (eigensolve.cpp:123-140).
// ---------------------------------------------------------------------------
template <int P, int C, int T>
__global__ void __launch_bounds__(T) k_fd_solve_nat(const double2* __restrict__ ab,
                                                    const unsigned char* __restrict__ piv,
                                                    double2* __restrict__ X, int nt, size_t nblk, int n1, int n2,
                                                    const int2* __restrict__ pairs) {
    constexpr int kuf = 2 * P, NF = 2 * T, CP = C + 1, NEB = 2 * P + 1;
    extern __shared__ __align__(16) double2 sm_nat[];
    double2* xin = sm_nat;                          // [2][NF][CP] chunk input rows
    double2* xout = xin + 2 * NF * CP;              // [2][NF][CP] chunk output rows
    double2* fac = xout + 2 * NF * CP;              // [2][C][NEB][T] band entries
    long long* fb = reinterpret_cast<long long*>(fac + 2 * C * NEB * T); // [NF] fiber offsets (-1: none)
    const int tid = threadIdx.x;
    const size_t b0 = (size_t)blockIdx.x * T;
    const size_t b = b0 + tid;
    const bool valid = b < nblk;
    {
        long long oa = -1, ob = -1;
        if (valid) {
            const int i1 = (int)(b % (size_t)n1);
            const int2 q = __ldg(pairs + b / (size_t)n1);
            oa = ((long long)i1 + (long long)n1 * ((long long)q.x + (long long)n2 * q.y)) * nt;
            if (q.x != q.y) ob = ((long long)i1 + (long long)n1 * ((long long)q.y + (long long)n2 * q.x)) * nt;
        }
        fb[tid] = oa;
        fb[T + tid] = ob;
    }
    __syncthreads();
    const bool hb = fb[T + tid] >= 0;
    const double2 Z = make_double2(0.0, 0.0);
    const int nb = (int)(nblk - b0 < (size_t)T ? nblk - b0 : (size_t)T);
    // chunk loads: rows [r0, r0 + C) of every fiber, entries (k0 + j, e(j)) of the T blocks
    auto load_rows = [&](double2* dst, int r0) {
        for (int e = tid; e < NF * C; e += T) {
            const int f = e / C, j = e - f * C, r = r0 + j;
            const long long o = fb[f];
            const bool v = o >= 0 && r >= 0 && r < nt;
            cpa16(dst + f * CP + j, v ? (const void*)(X + o + r) : (const void*)X, v);
        }
    };
    // forward entries: the P multipliers (k, kuf + 1 + m) of steps k0 .. k0 + C - 1
    auto load_fac = [&](double2* dst, int k0) {
        const bool vb = tid < nb;
#pragma unroll
        for (int j = 0; j < C; ++j)
#pragma unroll
            for (int m = 0; m < P; ++m) {
                const int k = k0 + j;
                const bool v = vb && k + 1 + m < nt;
                cpa16(dst + (j * NEB + m) * T + tid,
                      v ? (const void*)(ab + b0 + tid + ((size_t)k * (3 * P + 1) + kuf + 1 + m) * nblk) : (const void*)ab,
                      v);
            }
    };
    // backward entries: (k, kuf - m), m = 0 .. 2P, of steps k0 .. k0 + C - 1
    auto load_fac_b = [&](double2* dst, int k0) {
        const bool vb = tid < nb;
#pragma unroll
        for (int j = 0; j < C; ++j)
#pragma unroll
            for (int m = 0; m < NEB; ++m) {
                const int k = k0 + j;
                const bool v = vb && k >= 0 && k < nt && k - m >= 0;
                cpa16(dst + (j * NEB + m) * T + tid,
                      v ? (const void*)(ab + b0 + tid + ((size_t)k * (3 * P + 1) + kuf - m) * nblk) : (const void*)ab,
                      v);
            }
    };
    auto store_rows = [&](const double2* src, int r0) {
        for (int e = tid; e < NF * C; e += T) {
            const int f = e / C, j = e - f * C, r = r0 + j;
            const long long o = fb[f];
            if (o >= 0 && r >= 0 && r < nt) X[o + r] = src[f * CP + j];
        }
    };
    const int nch = (nt + C - 1) / C;
    // ---------------- forward: L with row interchanges (eigensolve.cpp:127-133)
    double2 wa[P + 1], wb[P + 1];
#pragma unroll
    for (int m = 0; m <= P; ++m) {
        wa[m] = valid && m < nt ? X[fb[tid] + m] : Z;
        wb[m] = hb && m < nt ? X[fb[T + tid] + m] : Z;
    }
    // chunk c: steps [cC, cC + C); new window rows cC + P + 1 + j
    load_rows(xin, P + 1);
    load_fac(fac, 0);
    cpa_commit();
    unsigned char pv[C], pvn[C];
#pragma unroll
    for (int j = 0; j < C; ++j) pv[j] = valid && j < nt ? __ldg(piv + (size_t)j * nblk + b) : 0;
    for (int c = 0; c < nch; ++c) {
        const int cb = c & 1;
        if (c + 1 < nch) {
            load_rows(xin + (cb ^ 1) * NF * CP, (c + 1) * C + P + 1);
            load_fac(fac + (cb ^ 1) * C * NEB * T, (c + 1) * C);
        }
        cpa_commit();
#pragma unroll
        for (int j = 0; j < C; ++j) {
            const int k = (c + 1) * C + j;
            pvn[j] = valid && k < nt ? __ldg(piv + (size_t)k * nblk + b) : 0;
        }
        cpa_wait<1>();
        __syncthreads();
        const double2* xi = xin + cb * NF * CP;
        double2* xo = xout + cb * NF * CP;
        const double2* fc = fac + cb * C * NEB * T;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            const int k = c * C + j;
            if (k < nt) {
                const int po = pv[j];
#pragma unroll
                for (int m = 1; m <= P; ++m)
                    if (po == m) {
                        double2 tt = wa[0];
                        wa[0] = wa[m];
                        wa[m] = tt;
                        tt = wb[0];
                        wb[0] = wb[m];
                        wb[m] = tt;
                    }
#pragma unroll
                for (int m = 1; m <= P; ++m)
                    if (k + m < nt) {
                        const double2 l = fc[(j * NEB + (m - 1)) * T + tid];
                        wa[m] = csub(wa[m], cmul(l, wa[0]));
                        wb[m] = csub(wb[m], cmul(l, wb[0]));
                    }
                xo[tid * CP + j] = wa[0];
                xo[(T + tid) * CP + j] = wb[0];
                const double2 ina = xi[tid * CP + j], inb = xi[(T + tid) * CP + j];
#pragma unroll
                for (int m = 0; m < P; ++m) {
                    wa[m] = wa[m + 1];
                    wb[m] = wb[m + 1];
                }
                wa[P] = ina;
                wb[P] = inb;
            }
        }
#pragma unroll
        for (int j = 0; j < C; ++j) pv[j] = pvn[j];
        __syncthreads();
        store_rows(xo, c * C);
    }
    cpa_wait<0>();
    __threadfence_block();
    __syncthreads();
    // ---------------- backward: U, column oriented (eigensolve.cpp:134-139)
    // chunk c: steps k = nt-1-cC-j; new window rows k - 2P - 1
    double2 ua[2 * P + 1], ub[2 * P + 1];
#pragma unroll
    for (int j = 0; j <= 2 * P; ++j) {
        const int r = nt - 1 - j;
        ua[j] = valid && r >= 0 ? X[fb[tid] + r] : Z;
        ub[j] = hb && r >= 0 ? X[fb[T + tid] + r] : Z;
    }
    // rows of chunk c (ascending in memory): [nt-1-cC-(C-1) - 2P - 1, nt-1-cC - 2P - 1]
    auto brow0 = [&](int c) { return nt - 1 - c * C - (C - 1) - 2 * P - 1; };
    auto bk0 = [&](int c) { return nt - 1 - c * C - (C - 1); }; // lowest step of chunk c
    load_rows(xin, brow0(0));
    load_fac_b(fac, bk0(0)); // slot j <-> step bk0 + j
    cpa_commit();
    for (int c = 0; c < nch; ++c) {
        const int cb = c & 1;
        if (c + 1 < nch) {
            load_rows(xin + (cb ^ 1) * NF * CP, brow0(c + 1));
            load_fac_b(fac + (cb ^ 1) * C * NEB * T, bk0(c + 1));
        }
        cpa_commit();
        cpa_wait<1>();
        __syncthreads();
        const double2* xi = xin + cb * NF * CP;
        double2* xo = xout + cb * NF * CP;
        const double2* fc = fac + cb * C * NEB * T;
        const int k0 = bk0(c);
#pragma unroll
        for (int jj = C - 1; jj >= 0; --jj) { // steps descending
            const int k = k0 + jj;
            if (k >= 0) {
                // one reciprocal of the pivot for both fibers: conj(d) / |d|^2
                // (1 division instead of Smith's 3 per quotient; differs from
                // the reference's __divdc3 by rounding only)
                const double2 dg = fc[(jj * NEB + 0) * T + tid];
                const double sc = 1.0 / fma(dg.x, dg.x, dg.y * dg.y);
                const double2 rd = make_double2(dg.x * sc, -dg.y * sc);
                ua[0] = cmul(ua[0], rd);
                ub[0] = cmul(ub[0], rd);
#pragma unroll
                for (int j = 1; j <= 2 * P; ++j)
                    if (k - j >= 0) {
                        const double2 uu = fc[(jj * NEB + j) * T + tid];
                        ua[j] = csub(ua[j], cmul(uu, ua[0]));
                        ub[j] = csub(ub[j], cmul(uu, ub[0]));
                    }
                xo[tid * CP + jj] = ua[0];
                xo[(T + tid) * CP + jj] = ub[0];
                // row k - 2P - 1 sits at chunk slot jj (chunk rows start at k0 - 2P - 1)
                const double2 ina = xi[tid * CP + jj], inb = xi[(T + tid) * CP + jj];
#pragma unroll
                for (int j = 0; j < 2 * P; ++j) {
                    ua[j] = ua[j + 1];
                    ub[j] = ub[j + 1];
                }
                ua[2 * P] = ina;
                ub[2 * P] = inb;
            }
        }
        __syncthreads();
        store_rows(xo, k0);
    }
}

template <int P>
void launch_solve_p(const FdBlocks& B, double2* X, bool adjoint, cudaStream_t st, int tm) {
    const unsigned grid = (unsigned)((B.ns + 127) / 128);
    if (adjoint) {
        k_fd_solve_adj<P><<<grid, 128, 0, st>>>(B.ab.as<double2>(), B.piv.as<unsigned char>(), X,
                                                B.ns, B.nt, B.nblk, B.fiber_block.as<int>(), tm, B.rec, B.fused_nd, B.fused_np);
        check_launch("k_fd_solve_adj");
    } else {
        static const int pfd = [] {
            const char* e = std::getenv("KS_FD_PFD");
            return e ? std::atoi(e) : 0;
        }();
        if (!tm && B.pair_n1 > 0 && B.rec == 0 && B.fused_nd == 0) {
            // natural layout (FD apply without the time-major hand-off)
            // C = 2 steps per chunk: 45 KB per CTA, five CTAs (10 warps) per SM
            // (C = 4: two CTAs per SM, latency bound at 0.88 ms)
            constexpr int C = 2, T = 64, NEB = 2 * P + 1;
            const size_t sm = (size_t)(4 * 2 * T * (C + 1) + 2 * C * NEB * T) * sizeof(double2) +
                              (size_t)2 * T * sizeof(long long);
            static bool attr = false;
            if (!attr) {
                KS_CUDA(cudaFuncSetAttribute(k_fd_solve_nat<P, C, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sm));
                attr = true;
            }
            const unsigned gn = (unsigned)((B.nblk + T - 1) / T);
            k_fd_solve_nat<P, C, T><<<gn, T, sm, st>>>(B.ab.as<double2>(), B.piv.as<unsigned char>(), X, B.nt, B.nblk,
                                                       B.pair_n1, B.pair_n2, B.pairs.as<int2>());
            check_launch("k_fd_solve_nat");
            return;
        }
        if (tm && B.pair_n1 > 0) {
            constexpr int NE = 2 * P + 3, D = 4;
            const size_t sm = (size_t)D * NE * 128 * sizeof(double2) + (size_t)D * 128 * sizeof(unsigned);
            static bool attr = false;
            if (!attr) {
                KS_CUDA(cudaFuncSetAttribute(k_fd_solve_pair<P, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sm));
                attr = true;
            }
            const unsigned gp = (unsigned)((B.nblk + 127) / 128);
            k_fd_solve_pair<P, D><<<gp, 128, sm, st>>>(B.ab.as<double2>(), B.piv.as<unsigned char>(), X, B.ns,
                                                       B.nt, B.nblk, B.pair_n1, B.pair_n2, B.pairs.as<int2>(),
                                                       B.nopiv_off ? nullptr : B.wpiv.as<unsigned char>());
            check_launch("k_fd_solve_pair");
            return;
        }
        static const int ring = [] {
            const char* e = std::getenv("KS_FD_RING");
            return e ? std::atoi(e) : 4;
        }();
        if (tm && (ring == 4 || ring == 8)) {
            constexpr int NE = 2 * P + 2;
            auto go = [&](auto kern, int D, int tb) {
                const size_t sm = (size_t)D * NE * tb * sizeof(double2) + (size_t)D * tb * sizeof(unsigned);
                KS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                const unsigned g = (unsigned)((B.ns + tb - 1) / tb);
                kern<<<g, tb, sm, st>>>(B.ab.as<double2>(), B.piv.as<unsigned char>(), X, B.ns, B.nt, B.nblk,
                                        B.fiber_block.as<int>(), B.rec, B.fused_nd, B.fused_np,
                                        B.nopiv_off ? nullptr : B.wpivf.as<unsigned char>());
            };
            // few fibers (c1, c2: < 2 x 148 CTAs of 128): one warp per CTA spreads
            // them over all SMs, and an 8-deep ring keeps more steps in flight
            static int sms = 0;
            if (!sms) {
                int dev = 0;
                KS_CUDA(cudaGetDevice(&dev));
                KS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            }
            if (grid < (unsigned)(2 * sms)) go(k_fd_solve_ring<P, 8, 32>, 8, 32);
            else if (ring == 8) go(k_fd_solve_ring<P, 8>, 8, 128);
            else go(k_fd_solve_ring<P, 4>, 4, 128);
            check_launch("k_fd_solve_ring");
            return;
        }
        k_fd_solve<P><<<grid, 128, 0, st>>>(B.ab.as<double2>(), B.piv.as<unsigned char>(), X,
                                            B.ns, B.nt, B.nblk, B.fiber_block.as<int>(), tm, B.rec, B.fused_nd,
                                            B.fused_np, pfd);
        check_launch("k_fd_solve");
    }
}

} // namespace

void fd_blocks_alloc(FdBlocks& B) {
    B.rec = 0;
    if (B.fused_nd == 0 && B.pair_n1 == 0) {
        // records are opt-in (KS_FD_REC=1): measured slower at c3 (0.84 vs 0.56 ms,
        // 2.3 GB vs 1.05 GB DRAM read -- the interleaved layout's sectors are shared
        // by neighbouring blocks that concurrently running fibers also read)
        if (const char* e = std::getenv("KS_FD_REC"))
            if (std::strcmp(e, "1") == 0) B.rec = B.ldab + 1;
    }
    const size_t per = B.rec > 0 ? (size_t)B.rec : (size_t)B.ldab;
    B.ab.alloc((size_t)B.nt * per * B.nblk * sizeof(double2));
    if (B.rec == 0) B.piv.alloc((size_t)B.nt * B.nblk + 4); // +4: 4 B cp.async words
    B.flag.alloc(sizeof(int));
    B.wpiv.alloc((B.nblk + 31) / 32 + 1);
    B.bpiv.alloc(B.nblk + 1);
    B.wpivf.alloc((B.ns + 31) / 32 + 1);
}

void fd_block_to_host(const FdBlocks& B, size_t b, ks_c64* ab, int* piv) {
    const BandIndex bx = fd_band_index(b, B.nt, B.ldab, B.nblk, B.rec, B.fused_nd, B.fused_np);
    for (int k = 0; k < B.nt; ++k) {
        for (int e = 0; e < B.ldab; ++e)
            KS_CUDA(cudaMemcpy(ab + (size_t)k * B.ldab + e, B.ab.as<double2>() + bx.fb + (size_t)k * bx.fk + (size_t)e * bx.fe,
                               sizeof(double2), cudaMemcpyDeviceToHost));
        if (B.rec > 0) {
            double2 v;
            KS_CUDA(cudaMemcpy(&v, B.ab.as<double2>() + bx.fb + (size_t)k * bx.fk + B.ldab, sizeof(v),
                               cudaMemcpyDeviceToHost));
            piv[k] = k + (int)v.x;
        } else {
            unsigned char po = 0;
            KS_CUDA(cudaMemcpy(&po, B.piv.as<unsigned char>() + bx.pb + (size_t)k * bx.pk, 1, cudaMemcpyDeviceToHost));
            piv[k] = k + po;
        }
    }
}

void launch_fd_factor(FdBlocks& B, double nu, const double* Lt, const double* Mt,
                      const double2* Wsym, cudaStream_t st) {
    KS_CUDA(cudaMemsetAsync(B.flag.p, 0, sizeof(int), st));
    KS_CUDA(cudaMemsetAsync(B.wpiv.p, 0, B.wpiv.bytes, st));
    const unsigned grid = (unsigned)((B.nblk + 127) / 128);
    k_fd_factor<<<grid, 128, 0, st>>>(B.ab.as<double2>(), B.piv.as<unsigned char>(),
                                      B.flag.as<int>(), B.wpiv.as<unsigned char>(), B.bpiv.as<unsigned char>(), B.nblk, B.nt, B.p, B.lam_blk.as<double>(), nu,
                                      Lt, Mt, Wsym, B.rec, B.fused_nd, B.fused_np, B.kind);
    check_launch("k_fd_factor");
    int h = 0;
    KS_CUDA(cudaMemcpyAsync(&h, B.flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    KS_CUDA(cudaStreamSynchronize(st));
    KS_REQUIRE((h & 1) == 0, KS_ESINGULAR, "factor_banded: numerically singular pivot");
    // no row interchange in any block: U has bandwidth p, the 2p-row fill-in
    // band stays exactly zero, and the pair solve skips it (and the pivots)
    B.nopiv = (h & 2) == 0;
    // fiber-group flags for the ring solve (fibers map to blocks through fiber_block)
    KS_CUDA(cudaMemsetAsync(B.wpivf.p, 0, B.wpivf.bytes, st));
    if (B.ns > 0) {
        k_fiber_piv<<<(unsigned)((B.ns + 255) / 256), 256, 0, st>>>(
            B.bpiv.as<unsigned char>(), B.fiber_block.bytes ? B.fiber_block.as<int>() : nullptr, B.ns,
            B.wpivf.as<unsigned char>());
        check_launch("k_fiber_piv");
        KS_CUDA(cudaStreamSynchronize(st));
    }
    B.nopiv_off = false;
    if (const char* e = std::getenv("KS_FD_NOPIV"))
        if (std::strcmp(e, "0") == 0) B.nopiv_off = true;
}

void launch_fd_solve(const FdBlocks& B, double2* X, bool adjoint, cudaStream_t st, bool time_major) {
    const int tm = time_major ? 1 : 0;
    switch (B.p) {
    case 1: launch_solve_p<1>(B, X, adjoint, st, tm); break;
    case 2: launch_solve_p<2>(B, X, adjoint, st, tm); break;
    case 3: launch_solve_p<3>(B, X, adjoint, st, tm); break;
    case 4: launch_solve_p<4>(B, X, adjoint, st, tm); break;
    case 5: launch_solve_p<5>(B, X, adjoint, st, tm); break;
    case 6: launch_solve_p<6>(B, X, adjoint, st, tm); break;
    case 7: launch_solve_p<7>(B, X, adjoint, st, tm); break;
    case 8: launch_solve_p<8>(B, X, adjoint, st, tm); break;
    default: throw Error(KS_EINVAL, "FD solve: time degree must be 1..8");
    }
}

} // namespace ks
