// Fused axis-1 stage of the FD apply: forward axis-1 transform, the block
// solves along time, inverse axis-1 transform -- one kernel, the (t, i1) slab
// never leaves shared memory.
//
// Reference: FastDiagSolver::solve (src/fdsolver.cpp:53-63) = to_eigen
// (mode products with U_l^T, :7-14), N_s banded solves on the time fibers
// (:58-60, eigensolve.cpp:123-140), from_eigen (U_l, :16-21). Mode products
// on distinct axes commute, so the apply runs the forward
// transforms on axes d..2 first, then this kernel, then the inverse ones on
// axes 2..d (ks_api.cu fd_apply_dev).
//
// Why: with the tensor laid out time fastest, the slab X[o] = (i1, t) for a
// fixed outer index o = (i2, .., id) is contiguous (c3: 64 x 65 complex =
// 66.5 KB). A separate axis-1 transform, a time-major block solve and the
// inverse transform move the tensor through HBM three times plus the
// factors; here the slab is read once and written once, and only the
// factors (L D L^H rows, ks_fdsolve.cu) stream through L2.
//
// Per slab (persistent CTAs, one per SM, warp-specialised pipeline below):
//   1. bulk-copy (cp.async.bulk + mbarrier) the n1 rows into shared memory
//      (rows padded to PD doubles, PD = 4 mod 16: conflict-free fragments);
//   2. folded forward transform on FP64 tensor cores (mma.m8n8k4 DMMA):
//      even warps Y[E] = se^T (X[j] + X[n1-1-j]), odd warps
//      Y[O] = so^T (X[j] - X[n1-1-j]); the results overwrite the slab by
//      position (even eigen-indices first, then odd);
//   3. one thread per fiber (position m): L D L^H forward / backward sweeps
//      along t in shared memory, factor rows through a 16-step per-thread
//      cp.async ring (the slab's blocks are consecutive -- position m of slab
//      o uses block m + n1b * grp[o] -- and are bulk-prefetched into L2 when
//      the slab load is issued, so the sweeps wait on L2, not HBM, latency);
//   4. folded inverse transform: even warps e_j = se X[E], odd warps
//      o_j = so X[O]; exchange through shared memory; Y[j] = e_j + o_j and
//      Y[n1-1-j] = e_j - o_j stored to HBM.
// Warp w: GEMM half g = w / 4 (even / odd), column group cq = w % 4 (8-double
// column blocks cq, cq+4, ...), all HB row blocks.
#include "ks_internal.hpp"

#include <algorithm>

namespace ks {

namespace {

constexpr int kNG = 9;            // GEMM warps (warps with (warp & 3) != 3)
// 12 warps (n1 <= 64: HB <= 4): 9 GEMM, solver warps 3 and 7, producer warp 11;
// 13 warps (HB = 5): solver warps 3, 7, 11, producer warp 12
constexpr int axis1_warps(int HB) { return HB >= 5 ? 13 : 12; }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

struct Axis1Args {
    const double* A;       // [2][SZ][AP] se / so, element (j, m) at j*AP + m, zero padded
    const double* X;       // natural layout, slab o at X + o * n1 * nt * 2
    double* Y;
    const int* order;      // slab processed by work item s (pairs of swapped slabs adjacent)
    const int* grp;        // blocks of slab o: b = m + n1b * grp[o] (position m, n1b >= n1 even)
    const double* dinv;    // L D L^H factors, block-interleaved (ks_fdsolve.cu)
    const double2* v;
    long long nblk;
    int nslab, n1, n1b, hc, nt, PD, AP, SZ, K4, CB;
    int nbuf, padr, asm_, ring; // slab buffers (2 or 3), zero rows after the slab, se / so in shared memory, factor ring slots
};

// Warp-specialised software pipeline, one CTA per SM, NB slab buffers (the
// plan uses 2; 3 would fit c3 only without the factor ring): at step t the
// solver warps sweep slab t in buffer t % NB while the 9 GEMM warps run the
// inverse transform + store of slab t-1, issue the load of slab t+NB-1 into
// the buffer that just became free, and forward-transform slab t+1; one named
// barrier per step. The DMMA work (the folded
// transforms) and the latency-bound sweeps (2 n_t dependent steps) overlap
// instead of alternating.
//
// GEMM warp w owns the 8-double column blocks w, w+9, w+18 of the slab and
// computes both halves (even and odd eigenvectors) for them: one fold
// (X[j] +- X[n1-1-j]) per loaded pair, the inverse unfold (e_j +- o_j) in
// registers, and no shared-memory traffic between warps. The half matrices
// se / so live in shared memory when they fit (ASM), else they come through L1.
//
// Solver thread m (position m) streams its factor rows from a D-slot ring in
// shared memory that one producer thread (a scheduler-3 warp without fibers)
// fills with bulk copies: the slab's blocks are consecutive (m + n1b * grp[o]),
// so step k of every fiber is one contiguous n1b-row run per factor array.
// Full / empty mbarriers per slot of 4 steps; the producer runs D-1 slots
// ahead, across sweeps and slabs, and bulk-prefetches the next slab's factor
// group into L2. (Reading the rows straight from global memory into registers
// one chunk ahead was measured slower, 0.58 vs 0.43 ms at c3: a 4-step lead
// does not cover the L2 latency and registers do not allow a longer one.) The
// recurrences are written so that only two dependent FMAs per step sit on the
// chain (the contribution of the newest value is applied last).
template <int HB, int NCB, int P, bool ODD, bool ASM>
__global__ void __launch_bounds__(32 * axis1_warps(HB), 1) k_fd_axis1(Axis1Args a) {
    extern __shared__ __align__(16) double sm[];
    const int n1 = a.n1, n1b = a.n1b, hc = a.hc, no = n1 - hc, nt = a.nt, PD = a.PD, AP = a.AP;
    constexpr int NB = 2;  // slab buffers
    constexpr int LG = 4;  // row groups of a slab load, one mbarrier each: the forward k loop starts on the first
    const size_t bufd = (size_t)(n1 + a.padr) * PD;                       // doubles per slab buffer
    double* S0 = sm;                                                      // [NB][n1 + padr][PD]
    double* Asm = S0 + (size_t)NB * bufd;                                 // [2][SZ][AP] (ASM)
    // factor ring: D slots of CK time steps, slot = [CK][P][n1b] v rows then [CK][n1b] 1/d
    constexpr int CK = 4;
    const int D = a.ring;
    const size_t slotd = (size_t)CK * n1b * (2 * P + 1);                  // doubles per slot
    double2* rv = reinterpret_cast<double2*>(Asm + (ASM ? (size_t)2 * a.SZ * AP : 0));
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(reinterpret_cast<double*>(rv) + (size_t)D * slotd); // [NB][LG]
    unsigned long long* full = bar + NB * LG;                             // [D]
    unsigned long long* empty = full + D;                                 // [D]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nsolve = 32 * ((n1 + 31) / 32);  // solver threads (whole warps)
    // Warp roles by scheduler: warps 3, 7, 11 (scheduler 3) run the sweeps, the
    // other nine the DMMA transforms -- the sweeps' dependent DFMA chains do not
    // queue behind 16-cycle DMMAs on a shared FP64 pipe (ncu: the solver warps
    // sat in math-pipe throttle and were the step's critical path), and nine
    // GEMM warps split the 17 column blocks of a c3 slab 2,2,..,1 instead of 3,2,..
    constexpr int NW = axis1_warps(HB);
    const bool producer = warp == NW - 1;
    const bool solver = !producer && (warp & 3) == 3;
    // GEMM and solver warps meet once per step (named barrier 2)
    auto step_bar = [&]() { asm volatile("bar.sync 2, %0;" ::"r"(32 * kNG + nsolve) : "memory"); };
    const int ar = lane >> 2, ak = lane & 3;
    const unsigned rowbytes = (unsigned)nt * 16u;
    const int nmine = a.nslab > (int)blockIdx.x ? (a.nslab - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    auto slab_of = [&](int t) -> long long { return a.order[blockIdx.x + (size_t)t * gridDim.x]; };

    for (int b = 0; b < NB; ++b)
        for (int e = tid; e < a.padr * PD; e += blockDim.x) S0[b * bufd + (size_t)n1 * PD + e] = 0.0; // padding rows (finite)
    if (ASM)
        for (int e = tid; e < 2 * a.SZ * AP; e += blockDim.x) Asm[e] = __ldg(a.A + e);
    if (tid == 0) {
        for (int q = 0; q < NB * LG; ++q)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + q)) : "memory");
        for (int q = 0; q < D; ++q) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full + q)) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(empty + q)), "r"(nsolve) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (nmine == 0) return;
    auto mwait = [&](unsigned long long* b, unsigned parity) {
        unsigned ok = 0;
        do {
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                         " selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok)
                         : "r"(su32(b)), "r"(parity)
                         : "memory");
        } while (!ok);
    };
    auto bulk = [&](void* dst, const void* src, unsigned bytes, unsigned long long* b) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(dst)),
                     "l"(src), "r"(bytes), "r"(su32(b))
                     : "memory");
    };

    if (producer) {
        // ---- producer: lane 0 fills the factor ring ----
        if (lane != 0) return;
        const size_t gsz = (size_t)n1b;
        const int nch = (nt + CK - 1) / CK;
        const int nuse = 2 * nch; // ring uses per slab: forward chunks 0..nch-1, then backward chunks nch-1..0
        auto prefetch_group = [&](int t) { // a slab's whole factor group into L2 (2 bulk prefetches)
            const size_t g0 = (size_t)a.grp[slab_of(t)] * (size_t)nt * gsz;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.v + g0 * P),
                         "r"((unsigned)(nt * P) * (unsigned)gsz * 16u)
                         : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.dinv + g0),
                         "r"((unsigned)nt * (unsigned)gsz * 8u)
                         : "memory");
        };
        int psl = 0, pwrap = 0;
        prefetch_group(0);
        for (int pt = 0; pt < nmine; ++pt) {
            if (pt + 1 < nmine) prefetch_group(pt + 1);
            const size_t pg = (size_t)a.grp[slab_of(pt)] * (size_t)nt; // group * nt
            for (int pu = 0; pu < nuse; ++pu) {
                if (pwrap > 0) mwait(empty + psl, (unsigned)((pwrap - 1) & 1)); // slot's previous use consumed
                const bool fwd = pu < nch;
                const int c = fwd ? pu : nuse - 1 - pu;
                const int k0 = c * CK, nk = min(CK, nt - k0);
                const unsigned vb = (unsigned)(nk * P) * (unsigned)gsz * 16u, db = (unsigned)nk * (unsigned)gsz * 8u;
                double2* dv = rv + (size_t)psl * (slotd / 2);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + psl)),
                             "r"(vb + (fwd ? db : 0u))
                             : "memory");
                bulk(dv, a.v + (pg + k0) * P * gsz, vb, full + psl);
                if (fwd)
                    bulk(reinterpret_cast<double*>(dv + (size_t)CK * P * gsz), a.dinv + (pg + k0) * gsz, db, full + psl);
                if (++psl == D) psl = 0, ++pwrap;
            }
        }
    } else if (!solver) {
        // =================== GEMM warps ===================
        const int w = warp - (warp >> 2); // 0..8
        unsigned phase = 0u; // bit b: parity of buffer b's next load completion
        const double* Ae = ASM ? Asm : a.A;
        const double* Ao = Ae + (size_t)a.SZ * AP;
        auto lda = [&](const double* p) -> double { return ASM ? *p : __ldg(p); };
        // k4 steps per row group: group g holds the rows j and n1-1-j of k4 in [g KG, (g+1) KG)
        const int KG = (a.K4 + LG - 1) / LG;
        auto issue_load = [&](int t) { // warp 0: slab t -> buffer t % NB, rows in consumption order
            if (w != 0 || t >= nmine) return;
            const int b = t % NB;
            double* Sx = S0 + (size_t)b * bufd;
            const double* Xs = a.X + (size_t)slab_of(t) * n1 * nt * 2;
            if (lane < LG) {
                const int j0 = min(4 * KG * lane, hc), j1 = min(4 * KG * (lane + 1), hc);
                int rows = 2 * (j1 - j0);
                if (ODD && j0 < hc && j1 == hc) --rows; // the middle row has no mirror
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + b * LG + lane)),
                             "r"(rowbytes * (unsigned)rows)
                             : "memory");
            }
            __syncwarp();
            for (int i = lane; i < n1; i += 32) {
                // pair index ii = 0, 1, 2, ..: rows 0, n1-1, 1, n1-2, ..
                const int j = i >> 1, row = (i & 1) ? n1 - 1 - j : j;
                if ((i & 1) && row == j) continue; // (odd n1: the middle row once)
                bulk(Sx + (size_t)row * PD, Xs + (size_t)row * nt * 2, rowbytes, bar + b * LG + j / (4 * KG));
            }
        };
        auto forward = [&](int t) {
            const int b = t % NB;
            double* Sx = S0 + (size_t)b * bufd;
            const unsigned par = (phase >> b) & 1u;
            phase ^= 1u << b;
            double ae_[HB][NCB][2], ao_[HB][NCB][2];
#pragma unroll
            for (int r = 0; r < HB; ++r)
#pragma unroll
                for (int i = 0; i < NCB; ++i) ae_[r][i][0] = ae_[r][i][1] = ao_[r][i][0] = ao_[r][i][1] = 0.0;
            for (int k4 = 0; k4 < a.K4; ++k4) {
                if (k4 % KG == 0) mwait(bar + b * LG + k4 / KG, par); // this row group has landed
                const int j = 4 * k4 + ak;
                double fe[HB], fo[HB];
#pragma unroll
                for (int r = 0; r < HB; ++r) {
                    fe[r] = lda(Ae + (size_t)j * AP + 8 * r + ar);
                    fo[r] = lda(Ao + (size_t)j * AP + 8 * r + ar);
                }
                const double* top = Sx + (size_t)j * PD;
                const double* bot = Sx + (size_t)max(n1 - 1 - j, 0) * PD; // (k padding: zero coefficients)
                const bool mid = ODD && j == hc - 1;
#pragma unroll
                for (int i = 0; i < NCB; ++i) {
                    const int cb = w + kNG * i;
                    if (cb < a.CB) {
                        const int c = 8 * cb + ar;
                        const double tv = top[c], bv = mid ? 0.0 : bot[c];
                        const double se = tv + bv, so = tv - bv;
#pragma unroll
                        for (int r = 0; r < HB; ++r) {
                            dmma(ae_[r][i][0], ae_[r][i][1], fe[r], se);
                            dmma(ao_[r][i][0], ao_[r][i][1], fo[r], so);
                        }
                    }
                }
            }
            __syncwarp(); // this warp's columns are read; write them back by position
#pragma unroll
            for (int r = 0; r < HB; ++r) {
                const int m = 8 * r + ar;
#pragma unroll
                for (int i = 0; i < NCB; ++i) {
                    const int cb = w + kNG * i, cc = 4 * cb + ak; // complex column
                    if (cb < a.CB && cc < nt) {
                        if (m < hc)
                            *reinterpret_cast<double2*>(Sx + (size_t)m * PD + 2 * cc) =
                                make_double2(ae_[r][i][0], ae_[r][i][1]);
                        if (m < no)
                            *reinterpret_cast<double2*>(Sx + (size_t)(hc + m) * PD + 2 * cc) =
                                make_double2(ao_[r][i][0], ao_[r][i][1]);
                    }
                }
            }
        };
        // inverse of slab t; then the load of slab `next` into the same buffer is
        // issued as soon as every GEMM warp has read it, before the stores
        auto inverse = [&](int t, int next) {
            double* Sx = S0 + (size_t)(t % NB) * bufd;
            double* Ys = a.Y + (size_t)slab_of(t) * n1 * nt * 2;
            double ee[HB][NCB][2], oo[HB][NCB][2];
#pragma unroll
            for (int r = 0; r < HB; ++r)
#pragma unroll
                for (int i = 0; i < NCB; ++i) ee[r][i][0] = ee[r][i][1] = oo[r][i][0] = oo[r][i][1] = 0.0;
            for (int k4 = 0; k4 < a.K4; ++k4) {
                const int mk = 4 * k4 + ak;
                double fe[HB], fo[HB];
#pragma unroll
                for (int r = 0; r < HB; ++r) {
                    fe[r] = lda(Ae + (size_t)(8 * r + ar) * AP + mk);
                    fo[r] = lda(Ao + (size_t)(8 * r + ar) * AP + mk);
                }
                const double* se = Sx + (size_t)mk * PD;
                const double* so = Sx + (size_t)(hc + mk) * PD;
#pragma unroll
                for (int i = 0; i < NCB; ++i) {
                    const int cb = w + kNG * i;
                    if (cb < a.CB) {
                        const int c = 8 * cb + ar;
                        const double be = se[c], bo = so[c];
#pragma unroll
                        for (int r = 0; r < HB; ++r) {
                            dmma(ee[r][i][0], ee[r][i][1], fe[r], be);
                            dmma(oo[r][i][0], oo[r][i][1], fo[r], bo);
                        }
                    }
                }
            }
            if (next < nmine) {
                asm volatile("bar.sync 1, %0;" ::"n"(32 * kNG) : "memory"); // all GEMM warps have read the buffer
                issue_load(next);
            }
#pragma unroll
            for (int r = 0; r < HB; ++r) {
                const int j = 8 * r + ar;
                if (j < hc) {
                    double2* d0 = reinterpret_cast<double2*>(Ys + (size_t)j * nt * 2);
                    double2* d1 = reinterpret_cast<double2*>(Ys + (size_t)(n1 - 1 - j) * nt * 2);
#pragma unroll
                    for (int i = 0; i < NCB; ++i) {
                        const int cb = w + kNG * i, cc = 4 * cb + ak;
                        if (cb < a.CB && cc < nt) {
                            __stcs(d0 + cc, make_double2(ee[r][i][0] + oo[r][i][0], ee[r][i][1] + oo[r][i][1]));
                            if (n1 - 1 - j != j)
                                __stcs(d1 + cc, make_double2(ee[r][i][0] - oo[r][i][0], ee[r][i][1] - oo[r][i][1]));
                        }
                    }
                }
            }
        };
        for (int t = 0; t < NB - 1; ++t) issue_load(t);
        forward(0);
        step_bar();
        for (int t = 0; t < nmine; ++t) {
            // buffer (t - 1) % NB is free once slab t-1 is transformed back
            if (t >= 1) inverse(t - 1, t + NB - 1);
            else issue_load(NB - 1);
            if (t + 1 < nmine) forward(t + 1);
            step_bar();
        }
        inverse(nmine - 1, nmine);
    } else {
        // =================== solver warps ===================
        const int m = 32 * (warp >> 2) + lane;
        const size_t gsz = (size_t)n1b; // factor group = the slab's n1b blocks (FdBlocks::gsz)
        const int nch = (nt + CK - 1) / CK;
        if (m >= nsolve) return; // (a warp with no fibers takes no part in the step barrier)
        const bool act = m < n1;
        int csl = 0;
        unsigned cph = 0; // consumer: slot, full-barrier parity
        const double2 Z = make_double2(0.0, 0.0);
        const int gm = (int)gsz;
        const double2* svm = rv + m; // this fiber's column of a ring slot
        for (int t = 0; t < nmine; ++t) {
            step_bar(); // slab t is in buffer t % NB (forward transform done)
            double2* row = reinterpret_cast<double2*>(S0 + (size_t)(t % NB) * bufd + (size_t)(act ? m : 0) * PD);
            // Static windows: xs[i] is position k0 + i of the chunk (i = 0..P carried
            // from the previous chunk, i = P+1..CK+P loaded), no per-step shifts.
            // L y = r, z = D^-1 y: xs[kk + j] -= conj(v_kk,j) xs[kk]; the chunk's factor
            // rows and incoming values go to registers first (independent loads), then
            // the sweep runs in registers with two dependent FMAs per step on the chain.
            double2 xs[CK + P + 1];
#pragma unroll
            for (int j = 0; j <= P; ++j) xs[j] = act && j < nt ? row[j] : Z;
            for (int c = 0; c < nch; ++c) {
                mwait(full + csl, cph);
                const double2* sv = svm + (size_t)csl * (slotd / 2);
                const double* sd = reinterpret_cast<const double*>(sv - m + (size_t)CK * P * gsz) + m;
                const int k0 = c * CK;
                if (act) {
                    double2 vr[CK][P];
                    double dr[CK];
                    if (k0 + CK + P < nt) { // full chunk, every incoming position inside the fiber
#pragma unroll
                        for (int kk = 0; kk < CK; ++kk) {
                            dr[kk] = sd[kk * gm];
#pragma unroll
                            for (int j = 0; j < P; ++j) vr[kk][j] = sv[(kk * P + j) * gm];
                            xs[P + 1 + kk] = row[k0 + P + 1 + kk];
                        }
                    } else {
                        const int nk = min(CK, nt - k0);
#pragma unroll
                        for (int kk = 0; kk < CK; ++kk) {
                            dr[kk] = kk < nk ? sd[kk * gm] : 0.0;
#pragma unroll
                            for (int j = 0; j < P; ++j) vr[kk][j] = kk < nk ? sv[(kk * P + j) * gm] : Z;
                            const int ki = k0 + P + 1 + kk;
                            xs[P + 1 + kk] = ki < nt ? row[ki] : Z;
                        }
                    }
#pragma unroll
                    for (int kk = 0; kk < CK; ++kk) {
                        const double2 w0 = xs[kk];
#pragma unroll
                        for (int j = 1; j <= P; ++j) {
                            const double2 v = vr[kk][j - 1];
                            xs[kk + j].x = fma(-v.y, w0.y, fma(-v.x, w0.x, xs[kk + j].x));
                            xs[kk + j].y = fma(v.y, w0.x, fma(-v.x, w0.y, xs[kk + j].y));
                        }
                        xs[kk] = make_double2(w0.x * dr[kk], w0.y * dr[kk]);
                    }
                    if (k0 + CK <= nt) {
#pragma unroll
                        for (int kk = 0; kk < CK; ++kk) row[k0 + kk] = xs[kk];
                    } else {
#pragma unroll
                        for (int kk = 0; kk < CK; ++kk)
                            if (k0 + kk < nt) row[k0 + kk] = xs[kk];
                    }
#pragma unroll
                    for (int j = 0; j <= P; ++j) xs[j] = xs[CK + j];
                }
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + csl)) : "memory");
                if (++csl == D) csl = 0, cph ^= 1u;
            }
            // L^H x = z: xb[kk] = z - sum_j v_kk,j xb[kk + j], the newest x applied last;
            // xb[CK..CK+P-1] carried from the chunk above
            double2 xb[CK + P];
#pragma unroll
            for (int j = 0; j < CK + P; ++j) xb[j] = Z;
            for (int c = nch - 1; c >= 0; --c) {
                mwait(full + csl, cph);
                const double2* sv = svm + (size_t)csl * (slotd / 2);
                const int k0 = c * CK;
                if (act) {
                    double2 vr[CK][P];
                    if (k0 + CK <= nt) {
#pragma unroll
                        for (int kk = 0; kk < CK; ++kk) {
                            xb[kk] = row[k0 + kk];
#pragma unroll
                            for (int j = 0; j < P; ++j) vr[kk][j] = sv[(kk * P + j) * gm];
                        }
                    } else { // (steps past n_t only in the last chunk: zero rows, zero values)
                        const int nk = nt - k0;
#pragma unroll
                        for (int kk = 0; kk < CK; ++kk) {
                            xb[kk] = kk < nk ? row[k0 + kk] : Z;
#pragma unroll
                            for (int j = 0; j < P; ++j) vr[kk][j] = kk < nk ? sv[(kk * P + j) * gm] : Z;
                        }
                    }
#pragma unroll
                    for (int kk = CK - 1; kk >= 0; --kk) {
                        double2 x = xb[kk];
#pragma unroll
                        for (int j = P; j >= 1; --j) {
                            const double2 v = vr[kk][j - 1], u = xb[kk + j];
                            x.x = fma(v.y, u.y, fma(-v.x, u.x, x.x));
                            x.y = fma(-v.y, u.x, fma(-v.x, u.y, x.y));
                        }
                        xb[kk] = x;
                    }
                    if (k0 + CK <= nt) {
#pragma unroll
                        for (int kk = 0; kk < CK; ++kk) row[k0 + kk] = xb[kk];
                    } else {
#pragma unroll
                        for (int kk = 0; kk < CK; ++kk)
                            if (k0 + kk < nt) row[k0 + kk] = xb[kk];
                    }
#pragma unroll
                    for (int j = P - 1; j >= 0; --j) xb[CK + j] = xb[j]; // (descending: the ranges overlap when P > CK)
                }
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + csl)) : "memory");
                if (++csl == D) csl = 0, cph ^= 1u;
            }
        }
        step_bar(); // matches the GEMM warps' last step barrier
    }
}

template <int HB, int NCB, int P, bool ODD>
void launch_axis1(const Axis1Args& a, size_t sm, cudaStream_t st) {
    const int grid = std::min(a.nslab, device_sms());
    const int thr = 32 * axis1_warps(HB);
    if (a.asm_) {
        auto k = k_fd_axis1<HB, NCB, P, ODD, true>;
        smem_optin((const void*)k, (int)sm);
        k<<<grid, thr, sm, st>>>(a);
    } else {
        auto k = k_fd_axis1<HB, NCB, P, ODD, false>;
        smem_optin((const void*)k, (int)sm);
        k<<<grid, thr, sm, st>>>(a);
    }
    check_launch("k_fd_axis1");
}

template <int HB, int NCB, bool ODD>
void launch_axis1_p(const Axis1Args& a, int p, size_t sm, cudaStream_t st) {
    switch (p) {
    case 1: launch_axis1<HB, NCB, 1, ODD>(a, sm, st); break;
    case 2: launch_axis1<HB, NCB, 2, ODD>(a, sm, st); break;
    case 3: launch_axis1<HB, NCB, 3, ODD>(a, sm, st); break;
    case 4: launch_axis1<HB, NCB, 4, ODD>(a, sm, st); break;
    case 5: launch_axis1<HB, NCB, 5, ODD>(a, sm, st); break;
    case 6: launch_axis1<HB, NCB, 6, ODD>(a, sm, st); break;
    default: throw Error(KS_EINVAL, "fused axis-1 FD stage: time degree 1..6");
    }
}

// Geometry and shared-memory plan: two slab buffers, the half matrices (when a
// ring of >= 4 slots still fits beside them, else they come through L1) and as
// many factor-ring slots as fit, up to 8 (c3: 144 + 18 + 6 x 10 KB).
struct Axis1Plan {
    int PD, AP, SZ, K4, HB, padr, nbuf, asm_, ring;
    size_t smem;
};
Axis1Plan axis1_plan(int n1, int nt, int p) {
    Axis1Plan q{};
    const int hc = (n1 + 1) / 2;
    q.HB = (hc + 7) / 8;
    q.K4 = (hc + 3) / 4;
    q.SZ = std::max(4 * q.K4, 8 * q.HB);
    q.AP = q.SZ;
    while (q.AP % 16 != 4) ++q.AP;
    q.PD = 2 * nt;
    while (q.PD % 16 != 4) ++q.PD;
    q.padr = std::max(0, hc + 4 * q.K4 - n1); // rows the k-padded loops read past the slab (kept zero)
    const size_t buf = (size_t)(n1 + q.padr) * q.PD * sizeof(double), am = (size_t)2 * q.SZ * q.AP * sizeof(double);
    // factor ring: slots of 4 steps x n1b blocks x (16 p + 8) B, at least 3, at most 8
    const int n1b = (n1 + 1) / 2 * 2;
    const size_t slot = (size_t)4 * n1b * (2 * p + 1) * sizeof(double);
    const size_t lim = 226 * 1024, bars = (size_t)(2 * 4 + 2 * 8) * 8; // slab row-group + ring barriers
    q.nbuf = 2;
    q.asm_ = 2 * buf + am + 4 * slot + bars <= lim;
    const size_t fixed = 2 * buf + (q.asm_ ? am : 0) + bars;
    q.ring = fixed + 3 * slot <= lim ? (int)std::min<size_t>(8, (lim - fixed) / slot) : 0;
    q.smem = fixed + (size_t)q.ring * slot;
    return q;
}

} // namespace

bool fd_axis1_supported(int n1, int nt, int p) {
    const Axis1Plan q = axis1_plan(n1, nt, p);
    const int CB = (2 * nt + 7) / 8;
    return n1 >= 2 && n1 <= 96 && q.HB >= 1 && q.HB <= 5 && (CB + kNG - 1) / kNG <= 3 && p >= 1 && p <= 6 &&
           q.ring >= 3 && q.smem <= 227 * 1024;
}

void launch_fd_axis1(const FoldAxis& F, const double* A, int nt, long long nslab, const int* order, const int* grp,
                     int n1b, const FdBlocks& B, const double* X, double* Y, cudaStream_t st) {
    Axis1Args a{};
    const Axis1Plan q = axis1_plan(F.n, nt, B.p);
    const int HB = q.HB;
    const size_t sm = q.smem;
    a.PD = q.PD, a.AP = q.AP, a.SZ = q.SZ, a.K4 = q.K4;
    a.nbuf = q.nbuf, a.padr = q.padr, a.asm_ = q.asm_, a.ring = q.ring;
    a.A = A;
    a.X = X;
    a.Y = Y;
    a.order = order;
    a.grp = grp;
    a.n1b = n1b;
    a.dinv = B.dinv.as<double>();
    a.v = B.v.as<double2>();
    a.nblk = (long long)B.nblk;
    a.nslab = (int)nslab;
    a.n1 = F.n;
    a.hc = F.hc;
    a.nt = nt;
    a.CB = (2 * nt + 7) / 8;
    const bool odd = F.n & 1;
    const int ncb = (a.CB + kNG - 1) / kNG;
#define KS_A1(HBV, NCBV)                                                                \
    if (HB == HBV && ncb <= NCBV) {                                                     \
        if (odd) launch_axis1_p<HBV, NCBV, true>(a, B.p, sm, st);                       \
        else launch_axis1_p<HBV, NCBV, false>(a, B.p, sm, st);                          \
        return;                                                                         \
    }
    KS_A1(1, 2) KS_A1(2, 2) KS_A1(3, 2) KS_A1(4, 2) KS_A1(5, 2)
    KS_A1(1, 3) KS_A1(2, 3) KS_A1(3, 3) KS_A1(4, 3) KS_A1(5, 3)
#undef KS_A1
    throw Error(KS_EINVAL, "fused axis-1 FD stage: unsupported shape");
}

// se / so of a folded axis in the kernel's layout: [2][SZ][AP], element (j, m)
void fd_axis1_matrix(const FoldAxis& F, int nt, int p, std::vector<double>& out) {
    const Axis1Plan q = axis1_plan(F.n, nt, p);
    const int AP = q.AP, SZ = q.SZ;
    const int H = 16 * F.th, Kp = F.kst;
    std::vector<double> fwd((size_t)2 * Kp * H);
    KS_CUDA(cudaMemcpy(fwd.data(), F.fwd.p, fwd.size() * sizeof(double), cudaMemcpyDeviceToHost));
    out.assign((size_t)2 * SZ * AP, 0.0);
    for (int g = 0; g < 2; ++g)
        for (int j = 0; j < SZ && j < Kp; ++j)
            for (int m = 0; m < SZ && m < H; ++m)
                out[((size_t)g * SZ + j) * AP + m] = fwd[((size_t)g * Kp + j) * H + m];
}

} // namespace ks
