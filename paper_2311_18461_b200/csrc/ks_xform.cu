// Folded (even/odd) spatial transform on the natural layout, bulk-copy fed.
//
// Reference: mode_product(const CoeffTensor&, const Eigen::MatrixXd&, axis)
// (src/tensorops.cpp:125-156) with U_l^T (to_eigen, fdsolver.cpp:7-14) or U_l
// (from_eigen, :16-21). The tensor is X[o][j][q] (o over the axes after l, j
// over axis l, q over the s complex entries of the axes before l); the
// product is a real GEMM over 2 s interleaved-double columns per (o, j).
//
// Centro-symmetric pencils (uniform meshes) have even / odd eigenvectors, so
// with the symmetrised half columns s_e, s_o (FoldAxis, ks_transform.cu):
//   forward  Y[m]      = sum_j s_e[j][E_m] (X[j] + X[n-1-j])      positions m < hc
//            Y[hc + m] = sum_j s_o[j][O_m] (X[j] - X[n-1-j])      positions m < n - hc
//   inverse  e_j = sum_m s_e X[m],  o_j = sum_m s_o X[hc + m],
//            Y[j] = e_j + o_j,  Y[n-1-j] = e_j - o_j
// The eigen-space rows are stored by POSITION (even eigenvectors first), so
// both directions read and write contiguous row ranges.
//
// Structure (persistent CTAs, 8 or 16 warps):
//   * tiles = 64 consecutive flattened complex columns (may span slabs);
//   * warp 0 also streams a tile's rows in stages of 4*KS pair rows ("top"
//     rows j and "bottom" rows n-1-j, or the even / odd position blocks) with
//     one cp.async.bulk per row segment into a padded shared-memory ring
//     (pitch 132 doubles = 4 mod 16: conflict-free B fragments), full / empty
//     mbarriers per stage -- no per-thread address arithmetic on the load path;
//   * consumer warp w owns the tile's complex columns 8w..8w+7 (two 8-double
//     fragments) for all row blocks of BOTH halves: the fold is one add and one
//     subtract per loaded pair, the inverse unfold happens in registers, and
//     the epilogue stores straight from the accumulators (16 B per lane, each
//     warp instruction 8 rows x 64 B);
//   * the half matrices stay in shared memory for the whole kernel.
// FP64 tensor cores: mma.sync.aligned.m8n8k4.row.col.f64 (DMMA).
#include "ks_internal.hpp"

#include <algorithm>

namespace ks {

namespace {

constexpr int kTC = 64;                  // complex columns per tile
constexpr int kBP = 2 * kTC + 4;         // stage row pitch (doubles), 4 mod 16

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mwait(unsigned long long* b, unsigned parity) {
    unsigned ok = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok)
                     : "r"(su32(b)), "r"(parity)
                     : "memory");
    } while (!ok);
}

struct XArgs {
    const double* A; // [2][Kst][H] (k-major: element (k, row) at k*H + row), even then odd
    const double* X;
    double* Y;
    long long s, outer, Q, ntiles;
    long long Ns;    // MODE 1 / 2: spatial size of the time-major layout T[t][pos + n * o]
    int n, hc, Kst, H, K4, AP;
};
// MODE 0: natural in / out. MODE 1 (axis 1, forward): natural in, time-major
// out T[t][pos + n1 * o]. MODE 2 (axis 1, inverse): time-major in, natural out
// (rows are contiguous per column there, so the stages load with per-thread
// 16 B cp.async completing on the stage mbarrier instead of row bulk copies).

// NF 8-double column fragments per consumer warp: 2 (8 consumer warps) for
// short axes, 1 (16 warps) for long ones (HB > 5: 2 x HB x NF accumulators).
// The consumer warps also produce (a dedicated producer warp was measured
// slower: 9 warps at one CTA per SM, 136 vs 125 us at c3 and 236 vs 200 us at
// n = 66; two 9-warp CTAs per SM cap the registers at 96 and spill).
template <int NF> struct XCfg {
    static constexpr int kCons = 16 / NF;
    static constexpr int kThr = kCons * 32;
};
template <int HB, int KS, bool INV, bool ODD, int NF, int MODE>
__global__ void __launch_bounds__(XCfg<NF>::kThr, NF == 2 ? 2 : 1) k_xfold(XArgs a) {
    constexpr int kCons = XCfg<NF>::kCons, kXThr = XCfg<NF>::kThr;
    constexpr int SR = 8 * KS;   // stage rows: 4 KS top + 4 KS bottom
    constexpr int NST = KS == 2 ? 5 : 8;
    extern __shared__ __align__(16) double sm[];
    const int n = a.n, hc = a.hc, no = n - hc, AP = a.AP;
    const int nstg = (a.K4 + KS - 1) / KS; // stages per tile
    const int kpad = nstg * 4 * KS;
    double* As = sm;                                     // [2][kpad][AP]
    double* Bs = As + (size_t)2 * kpad * AP;             // [NST][SR][kBP]
    unsigned long long* full = reinterpret_cast<unsigned long long*>(Bs + (size_t)NST * SR * kBP);
    unsigned long long* empty = full + NST;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int e = tid; e < 2 * kpad * AP; e += kXThr) {
        const int g = e / (kpad * AP), r = e - g * kpad * AP, k = r / AP, m = r - k * AP;
        As[e] = (k < a.Kst && m < a.H) ? __ldg(a.A + ((size_t)g * a.Kst + k) * a.H + m) : 0.0;
    }
    for (int e = tid; e < NST * SR * kBP; e += kXThr) Bs[e] = 0.0; // rows never loaded stay finite
    if (tid == 0) {
        for (int q = 0; q < NST; ++q) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(full + q)),
                         "r"(MODE == 2 ? kXThr : SR)
                         : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(empty + q)), "r"(kCons) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long s = a.s;
    const int my_tiles = a.ntiles > (long long)blockIdx.x ? (int)((a.ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;

    // Producers: warps 0..PW-1, each issuing the bulk copies of RPW rows of a
    // stage (one cp.async.bulk per row segment: spreading the issue over warps
    // keeps the copies ahead of the DMMAs), NST-2 stages ahead of consumption,
    // across tiles. A slot is refilled only after every consumer warp has
    // released its previous stage. 32-bit column arithmetic (Q < 2^31).
    constexpr int PW = kCons < SR ? kCons : SR, RPW = SR / PW;
    int pit = 0, pg = 0, pst = 0; // next stage to produce: tile, stage in tile, slot
    unsigned plap = 0;
    unsigned pq0 = blockIdx.x * (unsigned)kTC;
    const unsigned su = (unsigned)s, Qu = (unsigned)a.Q;
    // MODE 2: every thread loads 16 B elements (row e % SR, column e / SR) of
    // the stage; its columns' (o, t) are fixed per tile
    constexpr int EPT = MODE == 2 ? SR * kTC / kXThr : 1;
    unsigned tin_off[EPT];
    bool tin_ok[EPT];
    int tin_tile = -1;
    auto produce_tin = [&]() {
        if (pit >= my_tiles) return;
        if (plap > 0) mwait(empty + pst, (plap - 1) & 1u);
        if (tin_tile != pit) {
#pragma unroll
            for (int j = 0; j < EPT; ++j) {
                const int col = (tid + kXThr * j) / SR;
                const unsigned q = pq0 + (unsigned)col;
                tin_ok[j] = q < Qu;
                const unsigned o = q / su, t = q - o * su;
                // T offset of (t, pos 0, o) in complex units (fits 32 bits: N < 2^31)
                tin_off[j] = tin_ok[j] ? (unsigned)((size_t)t * (size_t)a.Ns + (size_t)n * o) : 0u;
            }
            tin_tile = pit;
        }
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
            const int e = tid + kXThr * j, row = e % SR, col = e / SR;
            const int pos = row < 4 * KS ? pg * 4 * KS + row : hc + pg * 4 * KS + (row - 4 * KS);
            const bool v = tin_ok[j] && pos < n;
            const double* src = v ? a.X + 2 * ((size_t)tin_off[j] + pos) : a.X;
            const unsigned dst = su32(Bs + ((size_t)pst * SR + row) * kBP + 2 * col);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 16 : 0)
                         : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(full + pst)) : "memory");
        if (++pst == NST) pst = 0, ++plap;
        if (++pg == nstg) {
            pg = 0;
            ++pit;
            pq0 += gridDim.x * (unsigned)kTC;
        }
    };
    unsigned po = 0, pr = 0; // slab and offset of the tile's first column (per tile, not per stage)
    int ptile = -1;
    // With more consumer warps than stage rows (NPG > 1) the warps take turns:
    // group warp / PW produces every NPG-th stage, so no warp carries the whole
    // producer path (ncu at n = 130: the non-producing warps sat on `full`).
    constexpr int NPG = kCons / PW;
    int pcnt = 0;
    auto produce = [&]() {
        if (MODE == 2) return produce_tin();
        if (pit >= my_tiles) return;
        const bool mine = NPG == 1 || pcnt % NPG == warp / PW;
        ++pcnt;
        if (mine) {
            if (plap > 0) mwait(empty + pst, (plap - 1) & 1u);
            if (ptile != pit) {
                po = pq0 / su;
                pr = pq0 - po * su;
                ptile = pit;
            }
            const unsigned ncol = min((unsigned)kTC, Qu - pq0);
            const int i = (warp % PW) * RPW + lane; // stage row
            int row = -1;
            if (lane < RPW) {
                const int kr = pg * 4 * KS + (i % (4 * KS));
                if (!INV) row = i < 4 * KS ? kr : n - 1 - kr;
                else row = i < 4 * KS ? kr : hc + kr;
                if (row < 0 || row >= n) row = -1;
            }
            // every producing lane arrives for its own row (arrival count = SR): no
            // cross-lane reduction on the producers' path
            if (lane < RPW)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + pst)),
                             "r"(row >= 0 ? ncol * 16u : 0u)
                             : "memory");
            if (row >= 0) {
                // the tile's columns, split at slab boundaries
                double* dst = Bs + ((size_t)pst * SR + i) * kBP;
                unsigned o = po, r = pr, done = 0, len = min(ncol, su - r);
                while (done < ncol) {
                    const double* src = a.X + 2 * (((size_t)o * n + row) * s + r);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            su32(dst + 2 * done)),
                        "l"(src), "r"(len * 16u), "r"(su32(full + pst))
                        : "memory");
                    done += len;
                    ++o;
                    r = 0;
                    len = min(ncol - done, su);
                }
            }
        }
        if (++pst == NST) pst = 0, ++plap;
        if (++pg == nstg) {
            pg = 0;
            ++pit;
            pq0 += gridDim.x * (unsigned)kTC;
        }
    };
    // NST-2 stages ahead: a slot is refilled two stages after its consumption,
    // so the producers wait for the slowest warp of the stage before last, not
    // of the one just finished (which coupled all warps every stage)
    for (int q = 0; q < NST - 2; ++q) produce();
    // ===================== consumers (all warps) =====================
    const int ar = lane >> 2, ak = lane & 3;
    const int cw = 8 * NF * warp; // this warp's first double column in the tile
    const double* Ae = As;
    const double* Ao = As + (size_t)kpad * AP;
    int st = 0;
    unsigned lap = 0;
    // the next stage's `full` barrier is tested (non-blocking) before the current
    // stage's DMMAs and only waited on if that test failed: the ~100-cycle
    // barrier query overlaps the warp's own math
    auto mtest = [&](unsigned long long* b, unsigned parity) -> unsigned {
        unsigned ok;
        asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok)
                     : "r"(su32(b)), "r"(parity)
                     : "memory");
        return ok;
    };
    unsigned ready = my_tiles > 0 ? mtest(full, 0u) : 0u;
    for (int it = 0; it < my_tiles; ++it) {
        const long long q0 = ((long long)blockIdx.x + (long long)it * gridDim.x) * kTC;
        double ce[HB][NF][2], co[HB][NF][2];
#pragma unroll
        for (int r = 0; r < HB; ++r)
#pragma unroll
            for (int f = 0; f < NF; ++f) ce[r][f][0] = ce[r][f][1] = co[r][f][0] = co[r][f][1] = 0.0;
        for (int g = 0; g < nstg; ++g) {
            if (!ready) mwait(full + st, lap & 1u);
            const double* bs = Bs + (size_t)st * SR * kBP;
            {
                const int sn = st + 1 == NST ? 0 : st + 1;
                ready = mtest(full + sn, (sn == 0 ? lap + 1 : lap) & 1u);
            }
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) {
                const int kl = 4 * kk + ak;          // stage-local k row
                const int kg = g * 4 * KS + kl;      // global k
                double fe[HB], fo[HB];
#pragma unroll
                for (int r = 0; r < HB; ++r) {
                    fe[r] = Ae[(size_t)kg * AP + 8 * r + ar];
                    fo[r] = Ao[(size_t)kg * AP + 8 * r + ar];
                }
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    const int c = cw + 8 * f + ar;
                    const double t = bs[(size_t)kl * kBP + c];
                    double b = bs[(size_t)(4 * KS + kl) * kBP + c];
                    double be, bo;
                    if (!INV) {
                        if (ODD && kg == hc - 1) b = 0.0; // middle row of an odd axis has no mirror
                        be = t + b;
                        bo = t - b;
                    } else {
                        be = t;
                        bo = b;
                    }
#pragma unroll
                    for (int r = 0; r < HB; ++r) {
                        dmma(ce[r][f][0], ce[r][f][1], fe[r], be);
                        dmma(co[r][f][0], co[r][f][1], fo[r], bo);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + st)) : "memory");
            if (++st == NST) st = 0, ++lap;
            produce(); // the producing warps: their rows of the stage NST-2 ahead
        }
        // epilogue: complex column cc of the tile -> (slab o, offset r)
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const int cc = (cw >> 1) + 4 * f + ak;
            const unsigned q = (unsigned)q0 + (unsigned)cc;
            if (q >= (unsigned)a.Q) continue;
            const unsigned o = q / (unsigned)s, rr = q - o * (unsigned)s;
            if (MODE == 1) { // T[t = rr][pos + n * o]
                double* tb = a.Y + 2 * ((size_t)rr * (size_t)a.Ns + (size_t)n * o);
#pragma unroll
                for (int r = 0; r < HB; ++r) {
                    const int m = 8 * r + ar;
                    if (m < hc) __stcs(reinterpret_cast<double2*>(tb + 2 * m), make_double2(ce[r][f][0], ce[r][f][1]));
                    if (m < no)
                        __stcs(reinterpret_cast<double2*>(tb + 2 * (hc + m)), make_double2(co[r][f][0], co[r][f][1]));
                }
                continue;
            }
            double* yb = a.Y + 2 * ((size_t)o * n * s + rr);
#pragma unroll
            for (int r = 0; r < HB; ++r) {
                const int m = 8 * r + ar;
                if (!INV) {
                    if (m < hc)
                        __stcs(reinterpret_cast<double2*>(yb + 2 * (long long)m * s), make_double2(ce[r][f][0], ce[r][f][1]));
                    if (m < no)
                        __stcs(reinterpret_cast<double2*>(yb + 2 * (long long)(hc + m) * s),
                               make_double2(co[r][f][0], co[r][f][1]));
                } else if (m < hc) {
                    __stcs(reinterpret_cast<double2*>(yb + 2 * (long long)m * s),
                           make_double2(ce[r][f][0] + co[r][f][0], ce[r][f][1] + co[r][f][1]));
                    if (n - 1 - m != m)
                        __stcs(reinterpret_cast<double2*>(yb + 2 * (long long)(n - 1 - m) * s),
                               make_double2(ce[r][f][0] - co[r][f][0], ce[r][f][1] - co[r][f][1]));
                }
            }
        }
    }
}

template <int HB, int KS, bool INV, bool ODD, int MODE>
void launch_x(const XArgs& a, cudaStream_t st) {
    constexpr int NF = HB <= 5 ? 2 : 1, kXThr = XCfg<NF>::kThr;
    constexpr int SR = 8 * KS, NST = KS == 2 ? 5 : 8;
    const int nstg = (a.K4 + KS - 1) / KS, kpad = nstg * 4 * KS;
    const size_t sm = ((size_t)2 * kpad * a.AP + (size_t)NST * SR * kBP) * sizeof(double) + (size_t)2 * NST * 8;
    KS_REQUIRE(sm <= 227 * 1024, KS_EINVAL, "folded transform: axis too long");
    KS_REQUIRE(a.Q < (1LL << 31), KS_EINVAL, "folded transform: more than 2^31 columns");
    auto k = k_xfold<HB, KS, INV, ODD, NF, MODE>;
    smem_optin((const void*)k, (int)sm);
    const int per_sm = 2 * sm <= 227 * 1024 ? 2 : 1;
    const unsigned g = (unsigned)std::min<long long>(a.ntiles, (long long)device_sms() * per_sm);
    k<<<g, kXThr, sm, st>>>(a);
    check_launch("k_xfold");
}

template <int HB, bool INV, int MODE>
void launch_x_hb(const XArgs& a, cudaStream_t st) {
    // short axes: 8-row stages (two k4 steps); long ones: 4-row stages (less padding)
    const bool odd = a.n & 1;
    if (HB <= 4) {
        if (odd) launch_x<HB, 2, INV, true, MODE>(a, st);
        else launch_x<HB, 2, INV, false, MODE>(a, st);
    } else {
        if (odd) launch_x<HB, 1, INV, true, MODE>(a, st);
        else launch_x<HB, 1, INV, false, MODE>(a, st);
    }
}

} // namespace

bool xfold_supported(const FoldAxis& F) { return F.n >= 2 && (F.hc + 7) / 8 <= 10; }

void launch_xfold(const FoldAxis& F, bool inverse, const double* X, double* Y, size_t s_complex, size_t outer,
                  cudaStream_t st, int mode) {
    if (s_complex == 0 || outer == 0) return;
    XArgs a{};
    a.A = (inverse ? F.inv : F.fwd).as<double>();
    a.X = X;
    a.Y = Y;
    a.s = (long long)s_complex;
    a.outer = (long long)outer;
    a.Q = a.s * a.outer;
    a.ntiles = (a.Q + kTC - 1) / kTC;
    a.n = F.n;
    a.hc = F.hc;
    a.Kst = F.kst;
    a.H = 16 * F.th;
    a.K4 = (F.hc + 3) / 4;
    const int HB = (F.hc + 7) / 8;
    a.AP = 8 * HB + 4;
    while (a.AP % 16 != 4) ++a.AP;
    a.Ns = (long long)F.n * a.outer;
    KS_REQUIRE(mode == 0 || (mode == 1 && !inverse) || (mode == 2 && inverse), KS_EINVAL,
               "folded transform: time-major output is forward-only, input inverse-only");
#define KS_XB(V)                                                                 \
    case V:                                                                      \
        if (mode == 2) launch_x_hb<V, true, 2>(a, st);                           \
        else if (mode == 1) launch_x_hb<V, false, 1>(a, st);                     \
        else if (inverse) launch_x_hb<V, true, 0>(a, st);                        \
        else launch_x_hb<V, false, 0>(a, st);                                    \
        break;
    switch (HB) {
        KS_XB(1) KS_XB(2) KS_XB(3) KS_XB(4) KS_XB(5) KS_XB(6) KS_XB(7) KS_XB(8) KS_XB(9) KS_XB(10)
    default: throw Error(KS_EINVAL, "folded transform: axis too long");
    }
#undef KS_XB
}

} // namespace ks
