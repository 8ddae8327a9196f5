// Fused pair of level passes for the Kronecker-sum matvec (plan: ks_kron.cu).
//
// The level plan applies the banded 1-D factors axis by axis; each pass reads
// its input level's tensors and writes the next level's (A at d = 3:
// 1 -> 3 -> 7 -> 5 -> 1 tensors, 32 x 16 B per DOF). This kernel runs two
// consecutive passes (axis a, then axis b = a + 1) in one sweep so the middle
// level never touches HBM:
//
//   * a CTA owns a block of points (q, i_a, o) -- all i_a of the axis-a lines
//     through nq inner columns q and no outer columns o -- and sweeps the
//     axis-b index i_b over its whole range;
//   * plane i_b of every input tensor streams through a D-deep cp.async ring in
//     shared memory (one 16 B element per thread per tensor, coalesced along
//     the contiguous index); the axis-a taps of a point are the neighbouring
//     threads' elements of the same plane;
//   * the middle-level values of the thread's point at plane i_b are formed in
//     registers (contributions grouped by input, as k_kron_elem) and pushed
//     into a (2BW+1)-row register window of output accumulators: mid plane i_b
//     contributes to output rows i_b-BW..i_b+BW through column i_b of the
//     axis-b factors; row i_b-BW is then complete and is stored.
//
// HBM traffic per fused pair: the input level once + the output level once
// (A at d = 3: passes (t, 1) read 1 and write 7 tensors, passes (2, 3) read 7
// and write 1 -> 16 x 16 B per DOF instead of 32).
//
// Reference: KroneckerOperator::apply (tensorops.cpp:236-254) / mode products
// (tensorops.cpp:89-123); the level plan restates the same sum of products in
// a factorised order.
#include "ks_internal.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace ks {

struct SweepEntry {
    int out;    // output node
    int factor; // -1 = identity
    double2 coeff;
};

namespace {

constexpr int kPairThreads = 256;

__device__ __forceinline__ void pcp16(void* sdst, const void* g, bool v) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(g), "r"(v ? 16 : 0));
}
__device__ __forceinline__ void pcommit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void pwait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// c * v (complex)
__device__ __forceinline__ void cfma(double2& acc, double2 c, double vr, double vi) {
    acc.x = fma(c.x, vr, fma(-c.y, vi, acc.x));
    acc.y = fma(c.x, vi, fma(c.y, vr, acc.y));
}

struct PairContrib { // axis-b contribution grouped by output (KronContrib layout)
    int in;
    int factor;
    double2 coeff;
};

// axis a: middle-level values of point (ia) at the plane held in `slot`
template <int BW, int NM>
__device__ __forceinline__ void pair_mid(double2 (&mid)[NM], const double2* slot, int n_in, int tid, int ia, int n_a,
                                         int nq, bool valid, const int* __restrict__ a_begin,
                                         const SweepEntry* __restrict__ a_ent, const double2* __restrict__ rb,
                                         const int* __restrict__ freal, int nmax) {
    constexpr int W = 2 * BW + 1;
    const double2 Z = make_double2(0.0, 0.0);
#pragma unroll
    for (int h = 0; h < NM; ++h) mid[h] = Z;
    for (int g = 0; g < n_in; ++g) {
        double2 w[W];
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int r = ia + k - BW;
            w[k] = (valid && r >= 0 && r < n_a) ? slot[g * kPairThreads + tid + (k - BW) * nq] : Z;
        }
        const int eb = __ldg(a_begin + g), ee = __ldg(a_begin + g + 1);
        for (int e = eb; e < ee; ++e) {
            const int ef = __ldg(&a_ent[e].factor), eo = __ldg(&a_ent[e].out);
            const double2 c = __ldg(&a_ent[e].coeff);
            double vr, vi;
            if (ef < 0) {
                vr = w[BW].x;
                vi = w[BW].y;
            } else {
                const double2* band = rb + ((size_t)ef * nmax + ia) * W;
                vr = 0.0;
                vi = 0.0;
                if (__ldg(freal + ef)) {
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        const double a = __ldg(&band[k].x);
                        vr = fma(a, w[k].x, vr);
                        vi = fma(a, w[k].y, vi);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        const double2 a = __ldg(&band[k]);
                        vr = fma(a.x, w[k].x, fma(-a.y, w[k].y, vr));
                        vi = fma(a.x, w[k].y, fma(a.y, w[k].x, vi));
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < NM; ++h)
                if (h == eo) cfma(mid[h], c, vr, vi);
        }
    }
}

// thread -> point (q, ia, o) of the CTA's block; base = element offset without i_b
struct PairGeom {
    long long base, s_b;
    int ia;
    bool valid;
};
__device__ __forceinline__ PairGeom pair_geom(long long s_a, int n_a, int n_b, long long n_outer, int nq, int no) {
    PairGeom G;
    const int tid = threadIdx.x;
    const long long nqb = (s_a + nq - 1) / nq;
    const long long q0 = (blockIdx.x % nqb) * nq, o0 = (blockIdx.x / nqb) * no;
    const int qq = tid % nq, rest = tid / nq;
    G.ia = rest % n_a;
    const int oo = rest / n_a;
    G.valid = oo < no && q0 + qq < s_a && o0 + oo < n_outer;
    G.s_b = s_a * n_a;
    G.base = G.valid ? (q0 + qq) + s_a * G.ia + G.s_b * (long long)n_b * (o0 + oo) : 0;
    return G;
}

__device__ __forceinline__ void pair_issue(double2* ring, const double2* const* in_ptrs, int n_in, int ib, int n_b,
                                           int D, const PairGeom& G) {
    if (ib < n_b) {
        double2* slot = ring + (size_t)(ib % D) * n_in * kPairThreads;
        for (int g = 0; g < n_in; ++g)
            pcp16(slot + g * kPairThreads + threadIdx.x,
                  G.valid ? (const void*)(in_ptrs[g] + G.base + G.s_b * ib) : (const void*)in_ptrs[0], G.valid);
    }
    pcommit();
}
__device__ __forceinline__ void pair_wait(int D) {
    if (D == 2) pwait<0>();
    else if (D == 3) pwait<1>();
    else pwait<2>();
}

// PUSH: mid plane ib is scattered into an output-row window acc[NOUT][W]
// (few outputs, up to 8 middle nodes)
template <int BW, int NOUT>
__global__ void __launch_bounds__(kPairThreads, (BW <= 2 ? 2 : 1)) k_kron_pair_push(
    const double2* const* __restrict__ in_ptrs, int n_in, double2* const* __restrict__ out_ptrs,
    const int* __restrict__ a_begin, const SweepEntry* __restrict__ a_ent,
    const int* __restrict__ b_begin, const SweepEntry* __restrict__ b_ent, int n_mid,
    const double2* __restrict__ rb, const int* __restrict__ freal, int nmax,
    long long s_a, int n_a, int n_b, long long n_outer, int nq, int no, int D) {
    constexpr int W = 2 * BW + 1;
    extern __shared__ __align__(16) double2 ring[]; // [D][n_in][kPairThreads]
    const int tid = threadIdx.x;
    const PairGeom G = pair_geom(s_a, n_a, n_b, n_outer, nq, no);
    const double2 Z = make_double2(0.0, 0.0);
    for (int k = 0; k < D - 1; ++k) pair_issue(ring, in_ptrs, n_in, k, n_b, D, G);
    double2 acc[NOUT][W]; // slot j <-> output row ib - BW + j
#pragma unroll
    for (int o = 0; o < NOUT; ++o)
#pragma unroll
        for (int j = 0; j < W; ++j) acc[o][j] = Z;
    for (int ib = 0; ib < n_b + BW; ++ib) {
        if (ib < n_b) {
            pair_wait(D);
            __syncthreads();
            pair_issue(ring, in_ptrs, n_in, ib + D - 1, n_b, D, G);
            double2 mid[8];
            pair_mid<BW, 8>(mid, ring + (size_t)(ib % D) * n_in * kPairThreads, n_in, tid, G.ia, n_a, nq, G.valid,
                            a_begin, a_ent, rb, freal, nmax);
            for (int h = 0; h < n_mid; ++h) {
                double2 m = mid[0];
#pragma unroll
                for (int hh = 1; hh < 8; ++hh)
                    if (hh == h) m = mid[hh];
                const int eb = __ldg(b_begin + h), ee = __ldg(b_begin + h + 1);
                for (int e = eb; e < ee; ++e) {
                    const int ef = __ldg(&b_ent[e].factor), eo = __ldg(&b_ent[e].out);
                    const double2 c = __ldg(&b_ent[e].coeff);
                    double2 cm;
                    cm.x = c.x * m.x - c.y * m.y;
                    cm.y = c.x * m.y + c.y * m.x;
                    const bool re = ef >= 0 && __ldg(freal + ef) != 0;
#pragma unroll
                    for (int j = 0; j < W; ++j) {
                        // F(r, ib) for output row r = ib + j - BW (column ib of the factor)
                        const int r = ib + j - BW;
                        double2 a;
                        if (ef < 0) a = make_double2(j == BW ? 1.0 : 0.0, 0.0);
                        else if (r >= 0 && r < n_b) a = __ldg(rb + ((size_t)ef * nmax + r) * W + (W - 1 - j));
                        else a = Z;
                        if (re) a.y = 0.0;
#pragma unroll
                        for (int o = 0; o < NOUT; ++o)
                            if (o == eo) {
                                acc[o][j].x = fma(a.x, cm.x, fma(-a.y, cm.y, acc[o][j].x));
                                acc[o][j].y = fma(a.x, cm.y, fma(a.y, cm.x, acc[o][j].y));
                            }
                    }
                }
            }
        }
        const int rd = ib - BW; // output row rd is complete
        if (rd >= 0 && G.valid) {
#pragma unroll
            for (int o = 0; o < NOUT; ++o) out_ptrs[o][G.base + G.s_b * rd] = acc[o][0];
        }
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
#pragma unroll
            for (int j = 0; j < W - 1; ++j) acc[o][j] = acc[o][j + 1];
            acc[o][W - 1] = Z;
        }
    }
    pwait<0>();
}

// PULL: a window of the last W middle planes per middle node (midw[NMID][W]);
// output row ib - BW is formed and stored node by node (many outputs, few
// middle nodes)
template <int BW, int NMID>
__global__ void __launch_bounds__(kPairThreads, (BW <= 2 ? 2 : 1)) k_kron_pair_pull(
    const double2* const* __restrict__ in_ptrs, int n_in, double2* const* __restrict__ out_ptrs, int n_out,
    const int* __restrict__ a_begin, const SweepEntry* __restrict__ a_ent,
    const int* __restrict__ b_obegin, const PairContrib* __restrict__ b_con,
    const double2* __restrict__ rb, const int* __restrict__ freal, int nmax,
    long long s_a, int n_a, int n_b, long long n_outer, int nq, int no, int D) {
    constexpr int W = 2 * BW + 1;
    extern __shared__ __align__(16) double2 ring[]; // [D][n_in][kPairThreads]
    const int tid = threadIdx.x;
    const PairGeom G = pair_geom(s_a, n_a, n_b, n_outer, nq, no);
    const double2 Z = make_double2(0.0, 0.0);
    for (int k = 0; k < D - 1; ++k) pair_issue(ring, in_ptrs, n_in, k, n_b, D, G);
    double2 midw[NMID][W]; // slot j <-> middle plane ib - 2BW + j
#pragma unroll
    for (int h = 0; h < NMID; ++h)
#pragma unroll
        for (int j = 0; j < W; ++j) midw[h][j] = Z;
    for (int ib = 0; ib < n_b + BW; ++ib) {
#pragma unroll
        for (int h = 0; h < NMID; ++h)
#pragma unroll
            for (int j = 0; j < W - 1; ++j) midw[h][j] = midw[h][j + 1];
        if (ib < n_b) {
            pair_wait(D);
            __syncthreads();
            pair_issue(ring, in_ptrs, n_in, ib + D - 1, n_b, D, G);
            double2 mid[NMID];
            pair_mid<BW, NMID>(mid, ring + (size_t)(ib % D) * n_in * kPairThreads, n_in, tid, G.ia, n_a, nq,
                               G.valid, a_begin, a_ent, rb, freal, nmax);
#pragma unroll
            for (int h = 0; h < NMID; ++h) midw[h][W - 1] = mid[h];
        } else {
#pragma unroll
            for (int h = 0; h < NMID; ++h) midw[h][W - 1] = Z;
        }
        const int rd = ib - BW; // output row rd uses middle planes rd-BW .. rd+BW = slots 0..W-1
        if (rd < 0) continue;
        for (int o = 0; o < n_out; ++o) {
            double2 acc = Z;
            const int cb = __ldg(b_obegin + o), ce = __ldg(b_obegin + o + 1);
            for (int e = cb; e < ce; ++e) {
                const int ef = __ldg(&b_con[e].factor), eh = __ldg(&b_con[e].in);
                const double2 c = __ldg(&b_con[e].coeff);
                double vr = 0.0, vi = 0.0;
                if (ef < 0) {
#pragma unroll
                    for (int h = 0; h < NMID; ++h)
                        if (h == eh) {
                            vr = midw[h][BW].x;
                            vi = midw[h][BW].y;
                        }
                } else {
                    // row rd of the factor: F(rd, rd - BW + j) = rb[ef][rd][j]
                    const double2* band = rb + ((size_t)ef * nmax + rd) * W;
                    const bool re = __ldg(freal + ef) != 0;
#pragma unroll
                    for (int j = 0; j < W; ++j) {
                        double2 a = __ldg(&band[j]);
                        if (re) a.y = 0.0;
#pragma unroll
                        for (int h = 0; h < NMID; ++h)
                            if (h == eh) {
                                vr = fma(a.x, midw[h][j].x, fma(-a.y, midw[h][j].y, vr));
                                vi = fma(a.x, midw[h][j].y, fma(a.y, midw[h][j].x, vi));
                            }
                    }
                }
                cfma(acc, c, vr, vi);
            }
            if (G.valid) out_ptrs[o][G.base + G.s_b * rd] = acc;
        }
    }
    pwait<0>();
}

} // namespace

// Fused passes (axis a = the pass axis of level k, axis b = a + 1) over tensors
// of shape [outer][n_b][n_a][s_a]. Axis-b contributions come grouped by input
// (b_begin/b_ent, push variant) and by output (b_obegin/b_con, pull variant).
// Returns false when the shape is outside the instantiated range (the caller
// then runs the two passes separately).
bool launch_kron_pair(int nin, int nmid, int nout, int bw, const double2* const* ip, double2* const* op,
                      const int* a_begin, const SweepEntry* a_ent, const int* b_begin, const SweepEntry* b_ent,
                      const int* b_obegin, const void* b_con, const double2* rb, const int* freal, int nmax,
                      long long s_a, int n_a, int n_b, long long n_outer, cudaStream_t st) {
    if (const char* e = std::getenv("KS_KRON_PAIR"))
        if (std::strcmp(e, "0") == 0) return false; // (the caller only tries this path when KS_KRON_PAIR is set)
    if (nin < 1 || nmid < 1 || nmid > 8 || nout < 1 || bw < 1 || bw > 4 || n_a > kPairThreads) return false;
    const bool pull = nmid <= 4 && nout > 2;
    if (!pull && nout > 2) return false;
    // point block: nq inner columns x n_a x no outer columns <= 256 threads,
    // the contiguous index fastest across threads
    int nq, no;
    if (s_a == 1) {
        nq = 1;
        no = kPairThreads / n_a;
    } else {
        nq = std::max(1, kPairThreads / n_a);
        if (nq > s_a) nq = (int)s_a;
        no = 1;
    }
    int D = 4; // ring depth: as deep as fits 2 CTAs/SM, at least 2
    auto smem = [&](int d) { return (size_t)d * nin * kPairThreads * sizeof(double2); };
    while (D > 2 && smem(D) > 110 * 1024) --D;
    if (smem(D) > 200 * 1024) return false;
    const size_t sm = smem(D);
    const long long nqb = (s_a + nq - 1) / nq, nob = (n_outer + no - 1) / no;
    const unsigned grid = (unsigned)(nqb * nob);
    auto go = [&](auto kern, auto... args) {
        static bool attr = false;
        if (!attr) {
            KS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            attr = true;
        }
        kern<<<grid, kPairThreads, sm, st>>>(args...);
    };
    const PairContrib* bc = static_cast<const PairContrib*>(b_con);
#define KS_PULL(B, M)                                                                                      \
    case M:                                                                                                \
        go(k_kron_pair_pull<B, M>, ip, nin, op, nout, a_begin, a_ent, b_obegin, bc, rb, freal, nmax, s_a,  \
           n_a, n_b, n_outer, nq, no, D);                                                                  \
        break;
#define KS_PUSH(B, NO)                                                                                     \
    case NO:                                                                                               \
        go(k_kron_pair_push<B, NO>, ip, nin, op, a_begin, a_ent, b_begin, b_ent, nmid, rb, freal, nmax,    \
           s_a, n_a, n_b, n_outer, nq, no, D);                                                             \
        break;
#define KS_BW(B)                                                                                           \
    case B:                                                                                                \
        if (pull) {                                                                                        \
            switch (nmid) { KS_PULL(B, 1) KS_PULL(B, 2) KS_PULL(B, 3) KS_PULL(B, 4) }                      \
        } else {                                                                                           \
            switch (nout) { KS_PUSH(B, 1) KS_PUSH(B, 2) }                                                  \
        }                                                                                                  \
        break;
    switch (bw) { KS_BW(1) KS_BW(2) KS_BW(3) KS_BW(4) }
#undef KS_BW
#undef KS_PUSH
#undef KS_PULL
    check_launch(pull ? "k_kron_pair_pull" : "k_kron_pair_push");
    return true;
}

} // namespace ks
