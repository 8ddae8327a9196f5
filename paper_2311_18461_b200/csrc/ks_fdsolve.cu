// Per-spatial-eigenvalue time blocks of the FD preconditioner: build, factor
// and solve, one time fiber per thread on the time-major layout T[t][fiber]
// (a warp's 32 fibers read and write 512 B contiguous runs at every step).
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
// Least-squares blocks (kind 0) are Hermitian positive definite by
// construction (Lt, Mt symmetric, W + W^H Hermitian, lambda > 0),
// so they are factored WITHOUT pivoting as H = L D L^H (banded, bandwidth p;
// Gaussian elimination is backward stable on HPD matrices, so this solves the
// same systems as the reference's partial-pivot LU to rounding, ~cond(H) eps).
// Stored per block and time step: 1/d_k (real) and the p normalised upper
// entries v_k,j = u(k, k+j) / d_k (complex) -- (16p + 8) bytes per row instead
// of the LU's (3p+1) * 16 + 1, and H^-1 = L^-H D^-1 L^-1 needs the same rows
// in both sweeps:
//   forward  y_k = x_k - sum_j conj(v_{k-j,j}) y_{k-j},  z_k = y_k / d_k
//   backward x_k = z_k - sum_j v_{k,j} x_{k+j}
// H^H = H, so the adjoint solve is the same solve. The Galerkin blocks
// (kind 1, H = W + nu lambda Mt, not Hermitian) keep the reference's
// partial-pivot LU, as do ks_fd_block's diagnostics (one block on demand).
//
// Block deduplication: when all spatial axes carry the
// same 1-D eigenvalues, the composite eigenvalue is symmetric under
// permutations of (i_1..i_d): pair mode (d = 3, axes 2 and 3 identical) keeps
// one block per (i1, {i2, i3}) and one thread solves both fibers with one
// factor read; otherwise fiber i reads block fiber_block[i].
//
// Loads go through a per-thread D-step cp.async ring in shared memory
// ([slot][entry][thread], so a warp's 16 B accesses are contiguous): D-1
// steps of factor and x loads in flight without holding registers, no
// barriers (each thread waits on its own groups).
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
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
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

// H(r, c) of block lambda, |r - c| <= p (fdsolver.cpp:115-116 expression order)
__device__ __forceinline__ double2 h_entry(int r, int c, int p, int kind, double s1, double s2,
                                           const double* __restrict__ Lt, const double* __restrict__ Mt,
                                           const double2* __restrict__ Wsym) {
    const int bi = p + r - c + c * (2 * p + 1);
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
    return make_double2(re, im);
}

// ---------------------------------------------------------------------------
// LU factor (kind 1, and kind-0 diagnostics): one thread per block, builds
// H(lambda) into the block-interleaved band ab[(k*ldab + e)*nblk + b] and runs
// factor_banded's partial-pivot elimination in place (eigensolve.cpp:93-119).
// ---------------------------------------------------------------------------
__global__ void k_fd_factor_lu(double2* __restrict__ ab, unsigned char* __restrict__ piv, int* __restrict__ flag,
                               unsigned char* __restrict__ wpiv, size_t nblk, int nt, int p,
                               const double* __restrict__ lam_blk, double nu, const double* __restrict__ Lt,
                               const double* __restrict__ Mt, const double2* __restrict__ Wsym, int kind) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= nblk) return;
    const int ldab = 3 * p + 1, kuf = 2 * p;
    const double lam = lam_blk[i];
    auto A = [&](int r, int c) -> double2& { return ab[((size_t)c * ldab + (size_t)(kuf + r - c)) * nblk + i]; };
    for (int c = 0; c < nt; ++c)
        for (int e = 0; e < ldab; ++e) ab[((size_t)c * ldab + e) * nblk + i] = make_double2(0.0, 0.0);
    const double s2 = nu * nu * lam * lam; // nu*nu*lam*lam (left to right)
    const double s1 = nu * lam;
    for (int c = 0; c < nt; ++c) {
        const int r0 = c - p < 0 ? 0 : c - p, r1 = c + p > nt - 1 ? nt - 1 : c + p;
        for (int r = r0; r <= r1; ++r) A(r, c) = h_entry(r, c, p, kind, s1, s2, Lt, Mt, Wsym);
    }
    bool swapped = false;
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
        piv[(size_t)k * nblk + i] = (unsigned char)(pr - k);
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
    if (swapped) {
        atomicOr(flag, 2);
        if (wpiv) wpiv[i >> 5] = 1; // every writer stores 1
    }
}

// ---------------------------------------------------------------------------
// L D L^H factor (kind 0): one thread per block, the (p+1) x (p+1) upper
// window of the partially eliminated block in registers. up[a][b] holds
// a(k+a, k+b), 0 <= a <= b <= P; without pivoting no fill leaves the band.
// ---------------------------------------------------------------------------
template <int P>
__global__ void k_fd_factor_ldl(double* __restrict__ dinv, double2* __restrict__ v, int* __restrict__ flag,
                                size_t nblk, size_t gsz, int nt, const double* __restrict__ lam_blk, double nu,
                                const double* __restrict__ Lt, const double* __restrict__ Mt,
                                const double2* __restrict__ Wsym) {
    const size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (b >= nblk) return;
    const size_t gb = b / gsz * (size_t)nt, bl = b % gsz; // group-blocked layout (FdBlocks::gsz)
    const double lam = lam_blk[b];
    const double s2 = nu * nu * lam * lam, s1 = nu * lam;
    const double2 Z = make_double2(0.0, 0.0);
    auto H = [&](int r, int c) -> double2 {
        return (r < nt && c < nt) ? h_entry(r, c, P, 0, s1, s2, Lt, Mt, Wsym) : Z;
    };
    double2 up[P + 1][P + 1];
#pragma unroll
    for (int a = 0; a <= P; ++a)
#pragma unroll
        for (int c = 0; c <= P; ++c) up[a][c] = c >= a ? H(a, c) : Z;
    for (int k = 0; k < nt; ++k) {
        const double dk = up[0][0].x;
        if (!(dk > 0.0)) { // not positive definite (cannot happen for lambda > 0)
            atomicOr(flag, 1);
            return;
        }
        const double di = 1.0 / dk;
        dinv[(gb + k) * gsz + bl] = di;
        double2 vv[P + 1];
#pragma unroll
        for (int j = 1; j <= P; ++j) {
            vv[j] = make_double2(up[0][j].x * di, up[0][j].y * di);
            v[((gb + k) * P + (j - 1)) * gsz + bl] = k + j < nt ? vv[j] : Z;
        }
        // a(k+a, k+c) -= l(k+a, k) u(k, k+c),  l(k+a, k) = conj(v_a)
#pragma unroll
        for (int a = 1; a <= P; ++a)
#pragma unroll
            for (int c = a; c <= P; ++c) up[a][c] = csub(up[a][c], cconjmul(vv[a], up[0][c]));
        // shift the window to step k+1; column k+1+P enters from H
#pragma unroll
        for (int a = 0; a < P; ++a)
#pragma unroll
            for (int c = a; c < P; ++c) up[a][c] = up[a + 1][c + 1];
#pragma unroll
        for (int a = 0; a <= P; ++a) up[a][P] = H(k + 1 + a, k + 1 + P);
    }
}

__device__ __forceinline__ void cpa16(void* sdst, const void* g, bool v) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(g), "r"(v ? 16 : 0));
}
__device__ __forceinline__ void cpa8(void* sdst, const void* g, bool v) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(g), "r"(v ? 8 : 0));
}
__device__ __forceinline__ void cpa4(void* sdst, const void* g, bool v) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(g), "r"(v ? 4 : 0));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---------------------------------------------------------------------------
// L D L^H solve of NF fibers sharing one block (NF = 2: pair mode, NF = 1:
// fiber map). x[f] points at step 0 of fiber f on the time-major layout
// (stride ns); null = absent (the diagonal pair i2 == i3).
// ---------------------------------------------------------------------------
template <int P, int D, int NF, int TB>
__device__ __forceinline__ void ldl_body(const double* __restrict__ dinv, const double2* __restrict__ v,
                                         double2* const (&x)[NF], size_t ns, int nt, size_t gsz, size_t b,
                                         double2* ring, double* dring) {
    const size_t gb = b / gsz * (size_t)nt, bl = b % gsz; // group-blocked layout (FdBlocks::gsz)
    constexpr int NE = P + NF;
    const int t = threadIdx.x;
    const double2 Z = make_double2(0.0, 0.0);
    auto slot = [&](int k, int e) -> double2* { return ring + ((size_t)((k % D) * NE + e) * TB + t); };
    auto vaddr = [&](int k, int j) -> const double2* { return v + ((gb + k) * P + j) * gsz + bl; };
    // forward: window w[f][m] = x[k+m] (pending updates applied), m = 0..P
    auto issue_f = [&](int k) {
        if (k < nt) {
#pragma unroll
            for (int j = 0; j < P; ++j) cpa16(slot(k, j), vaddr(k, j), k + 1 + j < nt);
            const int kx = k + P + 1;
#pragma unroll
            for (int f = 0; f < NF; ++f) cpa16(slot(k, P + f), kx < nt && x[f] ? x[f] + (size_t)kx * ns : v, kx < nt && x[f]);
            cpa8(dring + (k % D) * TB + t, dinv + (gb + k) * gsz + bl, true);
        }
        cpa_commit();
    };
    double2 w[NF][P + 1];
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int m = 0; m <= P; ++m) w[f][m] = m < nt && x[f] ? x[f][(size_t)m * ns] : Z;
#pragma unroll
    for (int k = 0; k < D - 1; ++k) issue_f(k);
    for (int k = 0; k < nt; ++k) {
        cpa_wait<D - 2>();
        issue_f(k + D - 1);
        const double di = dring[(k % D) * TB + t];
#pragma unroll
        for (int j = 1; j <= P; ++j) {
            const double2 l = *slot(k, j - 1); // zero past the end
#pragma unroll
            for (int f = 0; f < NF; ++f) w[f][j] = csub(w[f][j], cconjmul(l, w[f][0]));
        }
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            if (x[f]) x[f][(size_t)k * ns] = make_double2(w[f][0].x * di, w[f][0].y * di);
            const double2 in = *slot(k, P + f);
#pragma unroll
            for (int m = 0; m < P; ++m) w[f][m] = w[f][m + 1];
            w[f][P] = in;
        }
    }
    cpa_wait<0>();
    // backward: u[f][j] = x[k+j] (final), j = 1..P; z_k enters from the ring
    auto issue_b = [&](int k) {
        if (k >= 0) {
#pragma unroll
            for (int j = 0; j < P; ++j) cpa16(slot(k, j), vaddr(k, j), k + 1 + j < nt);
#pragma unroll
            for (int f = 0; f < NF; ++f) cpa16(slot(k, P + f), x[f] ? x[f] + (size_t)k * ns : v, x[f] != nullptr);
        }
        cpa_commit();
    };
    double2 u[NF][P + 1];
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int j = 0; j <= P; ++j) u[f][j] = Z;
#pragma unroll
    for (int q = 0; q < D - 1; ++q) issue_b(nt - 1 - q);
    for (int k = nt - 1; k >= 0; --k) {
        cpa_wait<D - 2>();
        issue_b(k - (D - 1));
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            double2 s = *slot(k, P + f);
#pragma unroll
            for (int j = 1; j <= P; ++j) s = csub(s, cmul(*slot(k, j - 1), u[f][j]));
            if (x[f]) x[f][(size_t)k * ns] = s;
#pragma unroll
            for (int j = P; j > 1; --j) u[f][j] = u[f][j - 1];
            u[f][1] = s;
        }
    }
}

// pair mode: block b = i1 + n1 * pidx(i2 <= i3) serves the fibers (i1, i2, i3)
// and (i1, i3, i2); consecutive threads take consecutive i1, so factor reads
// (block-interleaved) and both fibers' time-major accesses coalesce
template <int P, int D>
__global__ void __launch_bounds__(128) k_fd_ldl_pair(const double* __restrict__ dinv, const double2* __restrict__ v,
                                                      double2* __restrict__ X, size_t ns, int nt, size_t nblk, size_t gsz,
                                                      int n1, int n2, const int2* __restrict__ pairs) {
    extern __shared__ __align__(16) double2 ring[]; // [D][P+2][128], then double [D][128]
    const size_t b = blockIdx.x * (size_t)128 + threadIdx.x;
    if (b >= nblk) return;
    const int i1 = (int)(b % (size_t)n1);
    const int2 q = __ldg(pairs + b / (size_t)n1);
    double2* const x[2] = {X + (size_t)i1 + (size_t)n1 * ((size_t)q.x + (size_t)n2 * q.y),
                           q.x != q.y ? X + (size_t)i1 + (size_t)n1 * ((size_t)q.y + (size_t)n2 * q.x) : nullptr};
    ldl_body<P, D, 2, 128>(dinv, v, x, ns, nt, gsz, b, ring,
                           reinterpret_cast<double*>(ring + (size_t)D * (P + 2) * 128));
}

// fiber map: fiber f reads block fblk[f] (identity when null)
template <int P, int D, int TB>
__global__ void __launch_bounds__(TB) k_fd_ldl_ring(const double* __restrict__ dinv, const double2* __restrict__ v,
                                                     double2* __restrict__ X, size_t ns, int nt, size_t gsz,
                                                     const int* __restrict__ fblk) {
    extern __shared__ __align__(16) double2 ring[]; // [D][P+1][TB], then double [D][TB]
    const size_t f = blockIdx.x * (size_t)TB + threadIdx.x;
    if (f >= ns) return;
    const size_t b = fblk ? (size_t)__ldg(fblk + f) : f;
    double2* const x[1] = {X + f};
    ldl_body<P, D, 1, TB>(dinv, v, x, ns, nt, gsz, b, ring,
                          reinterpret_cast<double*>(ring + (size_t)D * (P + 1) * TB));
}

// ---------------------------------------------------------------------------
// LU solves (kind 1, Galerkin). NF fibers per block as above; NP: none of the
// warp's blocks pivoted, so the pivot bytes and the p fill-in rows of U
// (exact zeros) are not read -- bit-identical to the full band.
// ---------------------------------------------------------------------------
template <int P, int D, int NF, int TB, bool NP>
__device__ __forceinline__ void lu_body(const double2* __restrict__ ab, const unsigned char* __restrict__ piv,
                                        double2* const (&x)[NF], size_t ns, int nt, size_t nblk, size_t b,
                                        double2* ring) {
    constexpr int kuf = 2 * P, NE = 2 * P + 1 + NF;
    unsigned* pr = reinterpret_cast<unsigned*>(ring + (size_t)D * NE * TB);
    const int t = threadIdx.x;
    const double2 Z = make_double2(0.0, 0.0);
    auto slot = [&](int k, int e) -> double2* { return ring + ((size_t)((k % D) * NE + e) * TB + t); };
    auto baddr = [&](int k, int e) -> const double2* { return ab + b + ((size_t)k * (3 * P + 1) + e) * nblk; };
    auto issue_f = [&](int k) {
        if (k < nt) {
#pragma unroll
            for (int m = 1; m <= P; ++m) cpa16(slot(k, m - 1), k + m < nt ? baddr(k, kuf + m) : ab, k + m < nt);
            const int kx = k + P + 1;
#pragma unroll
            for (int f = 0; f < NF; ++f) cpa16(slot(k, P + f), kx < nt && x[f] ? x[f] + (size_t)kx * ns : ab, kx < nt && x[f]);
            if (!NP) {
                const size_t o = (size_t)k * nblk + b;
                cpa4(pr + (k % D) * TB + t, piv + (o & ~(size_t)3), true);
            }
        }
        cpa_commit();
    };
    // forward: L with row interchanges (eigensolve.cpp:127-133)
    double2 w[NF][P + 1];
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int m = 0; m <= P; ++m) w[f][m] = m < nt && x[f] ? x[f][(size_t)m * ns] : Z;
#pragma unroll
    for (int k = 0; k < D - 1; ++k) issue_f(k);
    for (int k = 0; k < nt; ++k) {
        cpa_wait<D - 2>();
        issue_f(k + D - 1);
        const size_t o = (size_t)k * nblk + b;
        const int po = NP ? 0 : (int)((pr[(k % D) * TB + t] >> (8 * (unsigned)(o & 3))) & 0xffu);
#pragma unroll
        for (int m = 1; m <= P; ++m)
            if (po == m)
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    const double2 tt = w[f][0];
                    w[f][0] = w[f][m];
                    w[f][m] = tt;
                }
#pragma unroll
        for (int m = 1; m <= P; ++m)
            if (k + m < nt) {
                const double2 l = *slot(k, m - 1);
#pragma unroll
                for (int f = 0; f < NF; ++f) w[f][m] = csub(w[f][m], cmul(l, w[f][0]));
            }
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            if (x[f]) x[f][(size_t)k * ns] = w[f][0];
            const double2 in = *slot(k, P + f);
#pragma unroll
            for (int m = 0; m < P; ++m) w[f][m] = w[f][m + 1];
            w[f][P] = in;
        }
    }
    cpa_wait<0>();
    // backward: U, column oriented (eigensolve.cpp:134-139)
    auto issue_b = [&](int k) {
        if (k >= 0) {
#pragma unroll
            for (int j = 0; j <= (NP ? P : 2 * P); ++j) cpa16(slot(k, j), k - j >= 0 ? baddr(k, kuf - j) : ab, k - j >= 0);
            const int kx = k - 2 * P - 1;
#pragma unroll
            for (int f = 0; f < NF; ++f)
                cpa16(slot(k, 2 * P + 1 + f), kx >= 0 && x[f] ? x[f] + (size_t)kx * ns : ab, kx >= 0 && x[f]);
        }
        cpa_commit();
    };
    double2 u[NF][2 * P + 1];
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int j = 0; j <= 2 * P; ++j) u[f][j] = nt - 1 - j >= 0 && x[f] ? x[f][(size_t)(nt - 1 - j) * ns] : Z;
#pragma unroll
    for (int q = 0; q < D - 1; ++q) issue_b(nt - 1 - q);
    for (int k = nt - 1; k >= 0; --k) {
        cpa_wait<D - 2>();
        issue_b(k - (D - 1));
        const double2 dg = *slot(k, 0);
#pragma unroll
        for (int f = 0; f < NF; ++f) u[f][0] = cdiv(u[f][0], dg);
#pragma unroll
        for (int j = 1; j <= (NP ? P : 2 * P); ++j)
            if (k - j >= 0) {
                const double2 uu = *slot(k, j);
#pragma unroll
                for (int f = 0; f < NF; ++f) u[f][j] = csub(u[f][j], cmul(uu, u[f][0]));
            }
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            if (x[f]) x[f][(size_t)k * ns] = u[f][0];
            const double2 in = *slot(k, 2 * P + 1 + f);
#pragma unroll
            for (int j = 0; j < 2 * P; ++j) u[f][j] = u[f][j + 1];
            u[f][2 * P] = in;
        }
    }
}

template <int P, int D>
__global__ void __launch_bounds__(128) k_fd_lu_pair(const double2* __restrict__ ab, const unsigned char* __restrict__ piv,
                                                     double2* __restrict__ X, size_t ns, int nt, size_t nblk, int n1,
                                                     int n2, const int2* __restrict__ pairs,
                                                     const unsigned char* __restrict__ wpiv) {
    extern __shared__ __align__(16) double2 ring[];
    const size_t b = blockIdx.x * (size_t)128 + threadIdx.x;
    if (b >= nblk) return;
    const int i1 = (int)(b % (size_t)n1);
    const int2 q = __ldg(pairs + b / (size_t)n1);
    double2* const x[2] = {X + (size_t)i1 + (size_t)n1 * ((size_t)q.x + (size_t)n2 * q.y),
                           q.x != q.y ? X + (size_t)i1 + (size_t)n1 * ((size_t)q.y + (size_t)n2 * q.x) : nullptr};
    if (__ldg(wpiv + (b >> 5)) == 0) lu_body<P, D, 2, 128, true>(ab, piv, x, ns, nt, nblk, b, ring);
    else lu_body<P, D, 2, 128, false>(ab, piv, x, ns, nt, nblk, b, ring);
}

template <int P, int D, int TB>
__global__ void __launch_bounds__(TB) k_fd_lu_ring(const double2* __restrict__ ab, const unsigned char* __restrict__ piv,
                                                    double2* __restrict__ X, size_t ns, int nt, size_t nblk,
                                                    const int* __restrict__ fblk) {
    extern __shared__ __align__(16) double2 ring[];
    const size_t f = blockIdx.x * (size_t)TB + threadIdx.x;
    if (f >= ns) return;
    const size_t b = fblk ? (size_t)__ldg(fblk + f) : f;
    double2* const x[1] = {X + f};
    lu_body<P, D, 1, TB, false>(ab, piv, x, ns, nt, nblk, b, ring);
}

// adjoint LU solve H^-H x (eigensolve.cpp:148-170), fiber map, time-major
template <int P>
__global__ void __launch_bounds__(128) k_fd_lu_adj(const double2* __restrict__ ab, const unsigned char* __restrict__ piv,
                                                    double2* __restrict__ X, size_t ns, int nt, size_t nblk,
                                                    const int* __restrict__ fblk) {
    const size_t f = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (f >= ns) return;
    constexpr int kuf = 2 * P;
    double2* const x0 = X + f;
    auto x = [&](int k) -> double2& { return x0[(size_t)k * ns]; };
    const size_t i = fblk ? (size_t)__ldg(fblk + f) : f;
    auto band = [&](int k, int e) -> double2 { return __ldg(ab + i + ((size_t)k * (3 * P + 1) + e) * nblk); };
    // U^H z = y, forward; h[j] = x[k - 2P + j] (finalised values)
    double2 h[2 * P];
#pragma unroll
    for (int j = 0; j < 2 * P; ++j) h[j] = make_double2(0.0, 0.0);
    for (int k = 0; k < nt; ++k) {
        double2 s = x(k);
#pragma unroll
        for (int j = 0; j < 2 * P; ++j) {
            const int r = k - 2 * P + j; // row index i, ascending
            if (r >= 0) s = csub(s, cconjmul(band(k, kuf + r - k), h[j]));
        }
        const double2 dk = band(k, kuf);
        s = cdiv(s, make_double2(dk.x, -dk.y));
        x(k) = s;
#pragma unroll
        for (int j = 0; j < 2 * P - 1; ++j) h[j] = h[j + 1];
        h[2 * P - 1] = s;
    }
    // L^H w = z with swaps in reverse; g[m] = x[k+m]
    double2 g[P + 1];
#pragma unroll
    for (int m = 0; m <= P; ++m) g[m] = nt - 1 + m < nt ? x(nt - 1 + m) : make_double2(0.0, 0.0);
    for (int k = nt - 1; k >= 0; --k) {
        double2 s = g[0];
#pragma unroll
        for (int m = 1; m <= P; ++m)
            if (k + m < nt) s = csub(s, cconjmul(band(k, kuf + m), g[m]));
        g[0] = s;
        const int po = piv[(size_t)k * nblk + i];
#pragma unroll
        for (int m = 1; m <= P; ++m)
            if (po == m) {
                const double2 t = g[0];
                g[0] = g[m];
                g[m] = t;
            }
        if (k + P < nt) x(k + P) = g[P];
#pragma unroll
        for (int m = P; m > 0; --m) g[m] = g[m - 1];
        g[0] = k - 1 >= 0 ? x(k - 1) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int m = 1; m <= P; ++m)
        if (m - 1 < nt) x(m - 1) = g[m];
}

template <int P>
void launch_solve_p(const FdBlocks& B, double2* X, bool adjoint, cudaStream_t st) {
    constexpr int D = 4;
    const bool pair = B.pair_n1 > 0;
    // few fibers (c1, c2: < 2 x 148 CTAs of 128): one warp per CTA spreads them
    // over all SMs
    const bool small = (B.ns + 127) / 128 < (size_t)(2 * device_sms());
    if (B.kind == 0) { // L D L^H: H^H = H, the adjoint is the same solve
        if (pair) {
            const size_t sm = (size_t)D * (P + 2) * 128 * sizeof(double2) + (size_t)D * 128 * sizeof(double);
            smem_optin((const void*)k_fd_ldl_pair<P, D>, (int)sm);
            k_fd_ldl_pair<P, D><<<(unsigned)((B.nblk + 127) / 128), 128, sm, st>>>(
                B.dinv.as<double>(), B.v.as<double2>(), X, B.ns, B.nt, B.nblk, B.gsz, B.pair_n1, B.pair_n2,
                B.pairs.as<int2>());
            check_launch("k_fd_ldl_pair");
            return;
        }
        auto go = [&](auto kern, int tb, int dr) {
            const size_t sm = (size_t)dr * (P + 1) * tb * sizeof(double2) + (size_t)dr * tb * sizeof(double);
            smem_optin((const void*)kern, (int)sm);
            kern<<<(unsigned)((B.ns + tb - 1) / tb), tb, sm, st>>>(B.dinv.as<double>(), B.v.as<double2>(), X, B.ns,
                                                                  B.nt, B.gsz, B.fiber_block.as<int>());
        };
        // few fibers (c1, c2): the sweeps are one latency chain per fiber, so a
        // 16-step ring keeps 15 steps of factor loads in flight per thread
        if (small) go(k_fd_ldl_ring<P, 16, 32>, 32, 16);
        else go(k_fd_ldl_ring<P, D, 128>, 128, D);
        check_launch("k_fd_ldl_ring");
        return;
    }
    if (adjoint) {
        k_fd_lu_adj<P><<<(unsigned)((B.ns + 127) / 128), 128, 0, st>>>(B.ab.as<double2>(), B.piv.as<unsigned char>(),
                                                                       X, B.ns, B.nt, B.nblk, B.fiber_block.as<int>());
        check_launch("k_fd_lu_adj");
        return;
    }
    if (pair) {
        constexpr int NE = 2 * P + 3;
        const size_t sm = (size_t)D * NE * 128 * sizeof(double2) + (size_t)D * 128 * sizeof(unsigned);
        smem_optin((const void*)k_fd_lu_pair<P, D>, (int)sm);
        k_fd_lu_pair<P, D><<<(unsigned)((B.nblk + 127) / 128), 128, sm, st>>>(
            B.ab.as<double2>(), B.piv.as<unsigned char>(), X, B.ns, B.nt, B.nblk, B.pair_n1, B.pair_n2,
            B.pairs.as<int2>(), B.wpiv.as<unsigned char>());
        check_launch("k_fd_lu_pair");
        return;
    }
    constexpr int NE = 2 * P + 2;
    auto go = [&](auto kern, int tb) {
        const size_t sm = (size_t)D * NE * tb * sizeof(double2) + (size_t)D * tb * sizeof(unsigned);
        smem_optin((const void*)kern, (int)sm);
        kern<<<(unsigned)((B.ns + tb - 1) / tb), tb, sm, st>>>(B.ab.as<double2>(), B.piv.as<unsigned char>(), X, B.ns,
                                                              B.nt, B.nblk, B.fiber_block.as<int>());
    };
    if (small) go(k_fd_lu_ring<P, D, 32>, 32);
    else go(k_fd_lu_ring<P, D, 128>, 128);
    check_launch("k_fd_lu_ring");
}

template <int P>
void launch_ldl_factor(FdBlocks& B, double nu, const double* Lt, const double* Mt, const double2* Wsym,
                       cudaStream_t st) {
    k_fd_factor_ldl<P><<<(unsigned)((B.nblk + 127) / 128), 128, 0, st>>>(
        B.dinv.as<double>(), B.v.as<double2>(), B.flag.as<int>(), B.nblk, B.gsz, B.nt, B.lam_blk.as<double>(), nu, Lt,
        Mt, Wsym);
    check_launch("k_fd_factor_ldl");
}

} // namespace

void fd_blocks_alloc(FdBlocks& B) {
    B.flag.alloc(sizeof(int));
    if (B.gsz == 0) B.gsz = B.nblk;
    KS_REQUIRE(B.nblk % B.gsz == 0, KS_EINVAL, "FD blocks: group size must divide the block count");
    if (B.kind == 0) {
        B.dinv.alloc((size_t)B.nt * B.nblk * sizeof(double));
        B.v.alloc((size_t)B.nt * B.p * B.nblk * sizeof(double2));
        return;
    }
    B.ab.alloc((size_t)B.nt * B.ldab * B.nblk * sizeof(double2));
    B.piv.alloc((size_t)B.nt * B.nblk + 4); // +4: 4 B cp.async words
    B.wpiv.alloc((B.nblk + 31) / 32 + 1);
}

void fd_block_to_host(const FdBlocks& B, size_t b, ks_c64* ab, int* piv) {
    // the reference's LU of this block (factor_banded layout, eigensolve.hpp:36-42):
    // stored for kind 1, refactored on demand from lambda for kind 0
    DevBuf tab, tpiv, tflag;
    const double2* src = B.ab.as<double2>();
    const unsigned char* psrc = B.piv.as<unsigned char>();
    size_t nb = B.nblk, bi = b;
    if (B.kind == 0) {
        tab.alloc((size_t)B.nt * B.ldab * sizeof(double2));
        tpiv.alloc((size_t)B.nt + 4);
        tflag.alloc(sizeof(int));
        KS_CUDA(cudaMemset(tflag.p, 0, sizeof(int)));
        k_fd_factor_lu<<<1, 1>>>(tab.as<double2>(), tpiv.as<unsigned char>(), tflag.as<int>(), nullptr, 1, B.nt, B.p,
                                 B.lam_blk.as<double>() + b, B.nu, B.Lt, B.Mt, B.Wsym, 0);
        check_launch("k_fd_factor_lu");
        KS_CUDA(cudaDeviceSynchronize());
        src = tab.as<double2>();
        psrc = tpiv.as<unsigned char>();
        nb = 1;
        bi = 0;
    }
    std::vector<double2> h((size_t)B.nt * B.ldab * nb);
    std::vector<unsigned char> hp((size_t)B.nt * nb);
    if (nb == 1) {
        KS_CUDA(cudaMemcpy(h.data(), src, h.size() * sizeof(double2), cudaMemcpyDeviceToHost));
        KS_CUDA(cudaMemcpy(hp.data(), psrc, hp.size(), cudaMemcpyDeviceToHost));
    }
    for (int k = 0; k < B.nt; ++k) {
        for (int e = 0; e < B.ldab; ++e) {
            double2 val;
            const size_t o = ((size_t)k * B.ldab + e) * nb + bi;
            if (nb == 1) val = h[o];
            else KS_CUDA(cudaMemcpy(&val, src + o, sizeof(val), cudaMemcpyDeviceToHost));
            ab[(size_t)k * B.ldab + e] = ks_c64{val.x, val.y};
        }
        unsigned char po = 0;
        if (nb == 1) po = hp[k];
        else KS_CUDA(cudaMemcpy(&po, psrc + (size_t)k * nb + bi, 1, cudaMemcpyDeviceToHost));
        piv[k] = k + po;
    }
}

void launch_fd_factor(FdBlocks& B, double nu, const double* Lt, const double* Mt, const double2* Wsym,
                      cudaStream_t st) {
    B.nu = nu;
    B.Lt = Lt;
    B.Mt = Mt;
    B.Wsym = Wsym;
    KS_CUDA(cudaMemsetAsync(B.flag.p, 0, sizeof(int), st));
    if (B.kind == 0) {
        switch (B.p) {
        case 1: launch_ldl_factor<1>(B, nu, Lt, Mt, Wsym, st); break;
        case 2: launch_ldl_factor<2>(B, nu, Lt, Mt, Wsym, st); break;
        case 3: launch_ldl_factor<3>(B, nu, Lt, Mt, Wsym, st); break;
        case 4: launch_ldl_factor<4>(B, nu, Lt, Mt, Wsym, st); break;
        case 5: launch_ldl_factor<5>(B, nu, Lt, Mt, Wsym, st); break;
        case 6: launch_ldl_factor<6>(B, nu, Lt, Mt, Wsym, st); break;
        case 7: launch_ldl_factor<7>(B, nu, Lt, Mt, Wsym, st); break;
        case 8: launch_ldl_factor<8>(B, nu, Lt, Mt, Wsym, st); break;
        default: throw Error(KS_EINVAL, "FD factor: time degree must be 1..8");
        }
        int h = 0;
        KS_CUDA(cudaMemcpyAsync(&h, B.flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        KS_CUDA(cudaStreamSynchronize(st));
        KS_REQUIRE(h == 0, KS_ESINGULAR, "FD factor: block not positive definite (numerically singular)");
        return;
    }
    KS_CUDA(cudaMemsetAsync(B.wpiv.p, 0, B.wpiv.bytes, st));
    k_fd_factor_lu<<<(unsigned)((B.nblk + 127) / 128), 128, 0, st>>>(
        B.ab.as<double2>(), B.piv.as<unsigned char>(), B.flag.as<int>(), B.wpiv.as<unsigned char>(), B.nblk, B.nt, B.p,
        B.lam_blk.as<double>(), nu, Lt, Mt, Wsym, B.kind);
    check_launch("k_fd_factor_lu");
    int h = 0;
    KS_CUDA(cudaMemcpyAsync(&h, B.flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    KS_CUDA(cudaStreamSynchronize(st));
    KS_REQUIRE((h & 1) == 0, KS_ESINGULAR, "factor_banded: numerically singular pivot");
    B.nopiv = (h & 2) == 0;
}

void launch_fd_solve(const FdBlocks& B, double2* X, bool adjoint, cudaStream_t st) {
    switch (B.p) {
    case 1: launch_solve_p<1>(B, X, adjoint, st); break;
    case 2: launch_solve_p<2>(B, X, adjoint, st); break;
    case 3: launch_solve_p<3>(B, X, adjoint, st); break;
    case 4: launch_solve_p<4>(B, X, adjoint, st); break;
    case 5: launch_solve_p<5>(B, X, adjoint, st); break;
    case 6: launch_solve_p<6>(B, X, adjoint, st); break;
    case 7: launch_solve_p<7>(B, X, adjoint, st); break;
    case 8: launch_solve_p<8>(B, X, adjoint, st); break;
    default: throw Error(KS_EINVAL, "FD solve: time degree must be 1..8");
    }
}

} // namespace ks
