// Dense spatial eigen-transform: the mode-l product of the complex FP64
// coefficient tensor with a dense real n x n matrix (U_l^T forward, U_l
// inverse).
//
// Reference: mode_product(const CoeffTensor&, const Eigen::MatrixXd&, axis)
// (src/tensorops.cpp:125-156), called from SpatialEigenbasis::to_eigen /
// from_eigen (src/fdsolver.cpp:7-21). The reference walks slabs and does
// one axpy of length s per (row, column) pair (:145-153).
//
// B200 formulation: with the tensor viewed as X[o][j][q] (o over the axes
// after l, j over axis l, q over 2*s interleaved doubles of the axes before
// l), the product is a real GEMM  Y(n x C) = A(n x n) * X(n x C)  over the
// flattened column index c = o*2s + q, C = outer*2s. Real x complex is exact
// in this view: the re and im parts are independent columns.
//
// Roofline: per complex DOF 4n flops (2n FMA) and 32 B compulsory (read X,
// write Y) -> n/8 flop/B, above the FP64 ridge (~5.7 flop/B at 37 TF /
// 6.5 TB/s) for every n >= 48: FP64-pipe bound. A stays in shared memory,
// X tiles stream through shared memory once (double-buffered), each output
// is written once.
//
// Engine: FP64 tensor cores, mma.sync.aligned.m8n8k4.row.col.f64 (DMMA), with
// the transform matrix resident in shared memory and X tiles streamed through
// a cp.async ring. (A DFMA CUDA-core engine over the same tiling measured
// slower -- c3 FD 3.13 vs 2.17 ms, operand-feed bound -- and was removed.)
#include "ks_internal.hpp"

#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <cmath>
#include <cstdio>
#include <vector>

namespace ks {

namespace {

constexpr int kThreads = 256; // 8 warps
constexpr int kBK = 16;       // k-chunk
constexpr int kBN = 128;      // columns (doubles) per CTA

// ---------------------------------------------------------------------------
// DMMA engine: FP64 mma.sync m8n8k4 (A row-major 8x4, B col-major 4x8).
// Fragment ownership (PTX ISA, mma.m8n8k4 .f64):
//   A: lane holds A[lane/4][lane%4]      B: lane holds B[lane%4][lane/4]
//   C: lane holds C[lane/4][2*(lane%4) + {0,1}]
// CTA tile: BM = 16*TM rows, kBN = 128 columns.
// Warps: wr = warp % 2 -> rows [wr*BM/2, +BM/2), wc = warp / 2 -> cols [wc*32, +32)
// Each warp: (BM/2/8) x 4 mma tiles.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// DMMA engine v2 (default): persistent CTAs, the whole n x n matrix resident in
// shared memory (loaded once per CTA), and a continuous S-stage cp.async ring
// over (column tile, k-chunk) work items, so the loads of the next tile are in
// flight while the current tile's DMMAs run. Same warp/fragment layout as
// k_mode_gemm_dmma. <=128 registers for TM <= 5 so two CTAs share an SM.
// ---------------------------------------------------------------------------
constexpr int kStages = 4;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    const int sz = valid ? 16 : 0; // src-size 0 -> zero fill
    // .cg: measured faster than .ca (c3 transforms 0.849 vs 0.886 ms) although
    // .ca removes the duplicate L2 sector reads of the misaligned rows
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Column maps: the GEMM's N dimension is a set of complex columns q (re/im =
// 2 adjacent doubles). MAP_STD walks the natural layout X[o][j][q']. For the
// outermost axis (outer = 1) the FD apply can instead hand the block solves a
// time-major layout T[t][i] (i = spatial index, axis 1 fastest): MAP_TOUT
// reads natural and writes time-major, MAP_TIN the reverse. Their column
// tiles are tbt (time) x tbr (lower spatial index) blocks of 64 columns, so
// both the natural side (consecutive t) and the time-major side (consecutive
// i) move 64-128 B segments.
//
// MAP_TOUT1 / MAP_TIN1 hand the time-major layout over on AXIS 1 instead
// (d = 3 pair-mode FD apply: forward axes d..2 natural, axis 1 last). Columns
// are enumerated as in MAP_STD (q = t + nt*o, o = the axes above 1), so the
// natural side moves whole 1 KB rows; on the time-major side a column's rows
// (i1) are contiguous: T[t][i1 + n1*o], row stride one complex (Np = 1).
enum { MAP_STD = 0, MAP_TOUT = 1, MAP_TIN = 2, MAP_TOUT1 = 3, MAP_TIN1 = 4 };
struct ColMap {
    int mode;
    int nt;            // time extent (T modes)
    int tbt, tbr;      // tile blocking (T modes), tbt * tbr = 64
    long long Q;       // complex columns
    long long s;       // complex stride of the axis in the natural layout
    long long Np;      // product of the spatial dims before the axis (T modes)
    long long Ns;      // spatial size (T modes)
    long long ntb;     // number of time blocks (T modes)
    long long ntiles;
    int tw = 64;       // complex columns per tile
    // optional row-pointer tables (device arrays of n pointers): row j of the
    // input / output lives at rin[j] + column offset instead of X + j*row stride
    // (the peer-memory sharded FD: rows of axis d on other GPUs)
    const double* const* rin = nullptr;
    double* const* rout = nullptr;
};
template <bool ROWS>
__device__ __forceinline__ const double* in_row(const ColMap& M, const double* X, long long col, int j,
                                               long long rs) {
    if (ROWS && M.rin) return M.rin[j] + col;
    return X + col + (long long)j * rs;
}
template <bool ROWS>
__device__ __forceinline__ double* out_row(const ColMap& M, double* Y, long long col, int r, long long rs) {
    if (ROWS && M.rout) return M.rout[r] + col;
    return Y + col + (long long)r * rs;
}

// offsets (doubles) and row strides of complex column j of tile tile
// per-tile state: one division per tile, none per column
struct TileBase {
    long long q0, o0, r0; // STD: first column, its slab o0 and offset r0 = q0 - o0*s
    long long tb, rb;     // T modes
};
__device__ __forceinline__ TileBase tile_base(const ColMap& M, long long tile) {
    TileBase b;
    if (M.mode == MAP_STD || M.mode >= MAP_TOUT1) {
        b.q0 = tile * M.tw;
        b.o0 = b.q0 / M.s;
        b.r0 = b.q0 - b.o0 * M.s;
        b.tb = b.rb = 0;
    } else {
        b.rb = tile / M.ntb;
        b.tb = tile - b.rb * M.ntb;
        b.q0 = b.o0 = b.r0 = 0;
    }
    return b;
}
__device__ __forceinline__ bool colmap(const ColMap& M, int n, const TileBase& B, int j,
                                       long long& in_off, long long& out_off) {
    if (M.mode == MAP_STD) {
        if (B.q0 + j >= M.Q) return false;
        long long o = B.o0, qq = B.r0 + j;
        while (qq >= M.s) { // s >= 1; a 64-column tile crosses at most ceil(64/s) slabs
            qq -= M.s;
            ++o;
        }
        in_off = out_off = 2 * (o * (long long)n * M.s + qq);
        return true;
    }
    if (M.mode >= MAP_TOUT1) { // STD columns, axis-1 time-major side
        if (B.q0 + j >= M.Q) return false;
        long long o = B.o0, qq = B.r0 + j;
        while (qq >= M.s) {
            qq -= M.s;
            ++o;
        }
        const long long nat = 2 * (o * (long long)n * M.s + qq), tm = 2 * (qq * M.Ns + (long long)n * o);
        in_off = M.mode == MAP_TIN1 ? tm : nat;
        out_off = M.mode == MAP_TOUT1 ? tm : nat;
        return true;
    }
    const long long tb = B.tb, rb = B.rb;
    // in-tile order: the time-major side's contiguous index fastest on the
    // store side (TOUT: spatial i fastest) / load side (TIN: t fastest); with
    // the m8n8k4 C fragment (4 consecutive columns per lane quad) both sides
    // then move >= 64 B contiguous segments
    const int jt = M.mode == MAP_TOUT ? j / M.tbr : j % M.tbt;
    const int jr = M.mode == MAP_TOUT ? j % M.tbr : j / M.tbt;
    const long long t = tb * M.tbt + jt, rest = rb * M.tbr + jr;
    if (t >= M.nt || rest >= M.Np) return false;
    const long long nat = 2 * (t + (long long)M.nt * rest);
    const long long tm = 2 * (t * M.Ns + rest);
    in_off = M.mode == MAP_TOUT ? nat : tm;
    out_off = M.mode == MAP_TOUT ? tm : nat;
    return true;
}

template <int TM, int STG = kStages, bool ROWS = false>
__global__ void __launch_bounds__(kThreads, (TM <= 5 ? 2 : 1))
k_mode_gemm_dmma2(const double* __restrict__ At, int n, const double* __restrict__ X,
                  double* __restrict__ Y, ColMap M) {
    constexpr int BM = 16 * TM;
    constexpr int MT = TM;
    constexpr int BMP = BM + 4; // == 4 (mod 16): conflict-free fragment loads
    constexpr int BNP = kBN + 4;
    extern __shared__ __align__(16) double smem[];
    const int nk = (n + kBK - 1) / kBK;
    double* As = smem;                          // [nk*kBK][BMP]
    double* Bs = smem + (size_t)nk * kBK * BMP; // [STG][kBK][BNP]
    const long long in_rs = (M.mode == MAP_TIN || M.mode == MAP_TIN1) ? 2 * M.Np : 2 * M.s;
    const long long out_rs = (M.mode == MAP_TOUT || M.mode == MAP_TOUT1) ? 2 * M.Np : 2 * M.s;
    const long long ntiles = M.ntiles;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wr = warp & 1, wc = warp >> 1;

    for (int e = tid; e < nk * kBK * BM; e += kThreads) {
        const int j = e / BM, r = e - j * BM;
        As[j * BMP + r] = (j < n && r < n) ? __ldg(At + (long long)j * n + r) : 0.0;
    }

    const int lcp = tid & 63, lrow0 = tid >> 6;
    const int my_tiles =
        ntiles > (long long)blockIdx.x ? (int)((ntiles - 1 - (long long)blockIdx.x) / gridDim.x + 1) : 0;
    const int nwork = my_tiles * nk;
    long long cur_tile = -1, cur_in = 0;
    bool cur_valid = false;

    auto issue = [&](int w) {
        if (w < nwork) {
            const int wt = w / nk;
            const long long tile = (long long)blockIdx.x + (long long)wt * gridDim.x;
            const int kc = w - wt * nk;
            if (tile != cur_tile) {
                long long dummy;
                cur_valid = colmap(M, n, tile_base(M, tile), lcp, cur_in, dummy);
                cur_tile = tile;
            }
            double* bs = Bs + (size_t)(w % STG) * kBK * BNP;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int jj = lrow0 + 4 * k, j = kc * kBK + jj;
                const bool v = cur_valid && j < n;
                cp_async16(bs + jj * BNP + 2 * lcp, v ? (const void*)in_row<ROWS>(M, X, cur_in, j, in_rs) : (const void*)X,
                           v);
            }
        }
        cp_async_commit();
    };

    double acc[MT][4][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int m = 0; m < 4; ++m) acc[i][m][0] = acc[i][m][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STG - 1; ++s) issue(s);

    const int r_warp = wr * (BM / 2), c_warp = wc * 32;
    const int ar = lane >> 2, ak = lane & 3;
    const int cr = lane >> 2;
    for (int w = 0; w < nwork; ++w) {
        cp_async_wait<STG - 2>();
        __syncthreads();
        issue(w + STG - 1);
        const int kc = w % nk;
        const double* bs = Bs + (size_t)(w % STG) * kBK * BNP;
        const double* as = As + (size_t)kc * kBK * BMP;
#pragma unroll
        for (int k4 = 0; k4 < kBK; k4 += 4) {
            double a[MT], b[4];
#pragma unroll
            for (int i = 0; i < MT; ++i) a[i] = as[(k4 + ak) * BMP + r_warp + i * 8 + ar];
#pragma unroll
            for (int m = 0; m < 4; ++m) b[m] = bs[(k4 + ak) * BNP + c_warp + m * 8 + ar];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int m = 0; m < 4; ++m) dmma_m8n8k4(acc[i][m][0], acc[i][m][1], a[i], b[m]);
        }
        if (kc == nk - 1) {
            const long long tile = (long long)blockIdx.x + (long long)(w / nk) * gridDim.x;
            const TileBase tbase = tile_base(M, tile);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int jcol = (c_warp >> 1) + m * 4 + (lane & 3); // complex column in tile
                long long io, oo;
                if (colmap(M, n, tbase, jcol, io, oo)) {
                    (void)0;
#pragma unroll
                    for (int i = 0; i < MT; ++i) {
                        const int r = r_warp + i * 8 + cr;
                        if (r < n)
                            *reinterpret_cast<double2*>(out_row<ROWS>(M, Y, oo, r, out_rs)) =
                                make_double2(acc[i][m][0], acc[i][m][1]);
                    }
                }
#pragma unroll
                for (int i = 0; i < MT; ++i) acc[i][m][0] = acc[i][m][1] = 0.0;
            }
        }
    }
    cp_async_wait<0>();
}

template <int TM>
void launch_tm(const double* At, int n, const double* X, double* Y, cudaStream_t st, const ColMap* map) {
    const int nk = (n + kBK - 1) / kBK;
    const size_t sm_a = (size_t)nk * kBK * (16 * TM + 4) * sizeof(double);
    const size_t sm_s = (size_t)kBK * (kBN + 4) * sizeof(double);
    // long axes (resident A large): fall back to a 2-stage ring
    const bool two = sm_a + kStages * sm_s > 227 * 1024;
    const size_t sm = sm_a + (two ? 2 : kStages) * sm_s;
    KS_REQUIRE(sm <= 227 * 1024, KS_EINVAL, "mode product: axis too long for the resident-A kernel");
    const int per_sm = (TM <= 5 && 2 * sm <= 227 * 1024) ? 2 : 1;
    ColMap M = *map;
    const unsigned g2 = (unsigned)std::min<long long>(M.ntiles, (long long)device_sms() * per_sm);
    if (M.rin || M.rout) { // peer-memory rows (sharded middle phase)
        if (two) {
            smem_optin((const void*)k_mode_gemm_dmma2<TM, 2, true>, (int)sm);
            k_mode_gemm_dmma2<TM, 2, true><<<g2, kThreads, sm, st>>>(At, n, X, Y, M);
        } else {
            smem_optin((const void*)k_mode_gemm_dmma2<TM, kStages, true>, (int)sm);
            k_mode_gemm_dmma2<TM, kStages, true><<<g2, kThreads, sm, st>>>(At, n, X, Y, M);
        }
    } else if (two) {
        smem_optin((const void*)k_mode_gemm_dmma2<TM, 2>, (int)sm);
        k_mode_gemm_dmma2<TM, 2><<<g2, kThreads, sm, st>>>(At, n, X, Y, M);
    } else {
        smem_optin((const void*)k_mode_gemm_dmma2<TM>, (int)sm);
        k_mode_gemm_dmma2<TM><<<g2, kThreads, sm, st>>>(At, n, X, Y, M);
    }
    check_launch("k_mode_gemm_dmma2");
}

// ---------------------------------------------------------------------------
// Panel variant for long axes (n > 160: the n x n matrix no longer fits shared
// memory): the output rows are processed in panels of 128, and the 16 x 128
// chunk of the matrix travels through the cp.async ring beside the X chunk
// (8-byte copies: a row of At starts at an odd double when n is odd). The X
// tile is re-read once per panel (from L2). Same fragment layout, column maps
// and layouts as k_mode_gemm_dmma2 with TM = 8. The reference has no length
// limit (tensorops.cpp:125-156); SPEC uses 1-D pencils up to 256 elements.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    const int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(sz));
}

template <int STG, bool ROWS>
__global__ void __launch_bounds__(kThreads, 1)
k_mode_gemm_panel(const double* __restrict__ At, int n, const double* __restrict__ X, double* __restrict__ Y, ColMap M) {
    constexpr int MT = 8, BM = 16 * MT;
    constexpr int BMP = BM + 4, BNP = kBN + 4;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;                           // [STG][kBK][BMP]
    double* Bs = smem + (size_t)STG * kBK * BMP; // [STG][kBK][BNP]
    const int nk = (n + kBK - 1) / kBK, np = (n + BM - 1) / BM;
    const long long in_rs = (M.mode == MAP_TIN || M.mode == MAP_TIN1) ? 2 * M.Np : 2 * M.s;
    const long long out_rs = (M.mode == MAP_TOUT || M.mode == MAP_TOUT1) ? 2 * M.Np : 2 * M.s;
    const long long ntiles = M.ntiles;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wr = warp & 1, wc = warp >> 1;
    const int lcp = tid & 63, lrow0 = tid >> 6;
    const int my_tiles =
        ntiles > (long long)blockIdx.x ? (int)((ntiles - 1 - (long long)blockIdx.x) / gridDim.x + 1) : 0;
    const long long nwork = (long long)my_tiles * np * nk;
    long long cur_tile = -1, cur_in = 0;
    bool cur_valid = false;

    auto issue = [&](long long w) {
        if (w < nwork) {
            const long long wt = w / ((long long)np * nk);
            const int rem = (int)(w - wt * np * nk), pnl = rem / nk, kc = rem - pnl * nk;
            const long long tile = (long long)blockIdx.x + wt * gridDim.x;
            if (tile != cur_tile) {
                long long dummy;
                cur_valid = colmap(M, n, tile_base(M, tile), lcp, cur_in, dummy);
                cur_tile = tile;
            }
            const int slot = (int)(w % STG);
            double* bs = Bs + (size_t)slot * kBK * BNP;
            double* as = As + (size_t)slot * kBK * BMP;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int jj = lrow0 + 4 * k, j = kc * kBK + jj;
                const bool v = cur_valid && j < n;
                cp_async16(bs + jj * BNP + 2 * lcp, v ? (const void*)in_row<ROWS>(M, X, cur_in, j, in_rs) : (const void*)X,
                           v);
            }
#pragma unroll
            for (int k = 0; k < (kBK * BM) / kThreads; ++k) {
                const int e = tid + k * kThreads, jj = e / BM, r = e - jj * BM;
                const int j = kc * kBK + jj, row = pnl * BM + r;
                const bool v = j < n && row < n;
                cp_async8(as + jj * BMP + r, v ? (const void*)(At + (long long)j * n + row) : (const void*)At, v);
            }
        }
        cp_async_commit();
    };

    double acc[MT][4][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int m = 0; m < 4; ++m) acc[i][m][0] = acc[i][m][1] = 0.0;
#pragma unroll
    for (int s = 0; s < STG - 1; ++s) issue(s);

    const int r_warp = wr * (BM / 2), c_warp = wc * 32;
    const int ar = lane >> 2, ak = lane & 3, cr = lane >> 2;
    int kc = 0, pnl = 0;
    long long wt = 0;
    for (long long w = 0; w < nwork; ++w) {
        cp_async_wait<STG - 2>();
        __syncthreads();
        issue(w + STG - 1);
        const int slot = (int)(w % STG);
        const double* bs = Bs + (size_t)slot * kBK * BNP;
        const double* as = As + (size_t)slot * kBK * BMP;
#pragma unroll
        for (int k4 = 0; k4 < kBK; k4 += 4) {
            double a[MT], b[4];
#pragma unroll
            for (int i = 0; i < MT; ++i) a[i] = as[(k4 + ak) * BMP + r_warp + i * 8 + ar];
#pragma unroll
            for (int m = 0; m < 4; ++m) b[m] = bs[(k4 + ak) * BNP + c_warp + m * 8 + ar];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int m = 0; m < 4; ++m) dmma_m8n8k4(acc[i][m][0], acc[i][m][1], a[i], b[m]);
        }
        if (kc == nk - 1) {
            const long long tile = (long long)blockIdx.x + wt * gridDim.x;
            const TileBase tbase = tile_base(M, tile);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int jcol = (c_warp >> 1) + m * 4 + (lane & 3); // complex column in tile
                long long io, oo;
                if (colmap(M, n, tbase, jcol, io, oo)) {
#pragma unroll
                    for (int i = 0; i < MT; ++i) {
                        const int r = pnl * BM + r_warp + i * 8 + cr;
                        if (r < n)
                            *reinterpret_cast<double2*>(out_row<ROWS>(M, Y, oo, r, out_rs)) =
                                make_double2(acc[i][m][0], acc[i][m][1]);
                    }
                }
#pragma unroll
                for (int i = 0; i < MT; ++i) acc[i][m][0] = acc[i][m][1] = 0.0;
            }
            kc = 0;
            if (++pnl == np) {
                pnl = 0;
                ++wt;
            }
        } else {
            ++kc;
        }
    }
    cp_async_wait<0>();
}

void launch_panel(const double* At, int n, const double* X, double* Y, cudaStream_t st, const ColMap* map) {
    constexpr int STG = 4;
    const size_t sm = (size_t)STG * kBK * ((16 * 8 + 4) + (kBN + 4)) * sizeof(double);
    ColMap M = *map;
    const unsigned g = (unsigned)std::min<long long>(M.ntiles, (long long)device_sms());
    if (M.rin || M.rout) {
        smem_optin((const void*)k_mode_gemm_panel<STG, true>, (int)sm);
        k_mode_gemm_panel<STG, true><<<g, kThreads, sm, st>>>(At, n, X, Y, M);
    } else {
        smem_optin((const void*)k_mode_gemm_panel<STG, false>, (int)sm);
        k_mode_gemm_panel<STG, false><<<g, kThreads, sm, st>>>(At, n, X, Y, M);
    }
    check_launch("k_mode_gemm_panel");
}

// ---------------------------------------------------------------------------
// Folded (even/odd) transform. On a uniform mesh the 1-D pencils are
// centro-symmetric (J K J = K, J M J = M, J the flip), so every eigenvector is
// even (u[n-1-j] = u[j]) or odd (u[n-1-j] = -u[j]); ceil(n/2) of them are even.
// With E / O the even / odd eigen-indices, s_e / s_o the symmetrised half
// columns (j < hc = ceil(n/2)):
//   forward  Y[E_m] = sum_j s_e[j][E_m] (X[j] + X[n-1-j])
//            Y[O_m] = sum_j s_o[j][O_m] (X[j] - X[n-1-j])
//   inverse  e_j = sum_m s_e[j][E_m] X[E_m],  o_j = sum_m s_o[j][O_m] X[O_m]
//            Y[j] = e_j + o_j,  Y[n-1-j] = e_j - o_j
// i.e. two (n/2 x n/2) GEMMs instead of one n x n: half the FP64 work, same
// HBM traffic. Stage chunk kc holds 16 rows: "top" rows 0-7 and "bottom" rows
// 8-15 (forward: X[j], X[n-1-j] for j = 8kc..8kc+7; inverse: X[E_m], X[O_m]),
// gathered by cp.async, so the fold is two FADDs per B fragment (forward) or
// nothing (inverse). Each warp owns the same (half-row, column) block of both
// GEMMs, so the inverse unfold happens in registers.
// Resident matrices: Af[2][kst][H] (k-major; [0] even, [1] odd, zero padded), staged as nkc*KC rows.
// ---------------------------------------------------------------------------
// RL: loader lanes along rows instead of columns (MAP_TIN1: a column's rows
// are contiguous on the time-major side, so a warp reads 2 x 256 B runs)
template <int TH, bool INV, int KC, int STG, int MINB, int BNC, bool ROWS = false, bool RL = false>
__global__ void __launch_bounds__(kThreads, MINB)
k_mode_gemm_fold(const double* __restrict__ Af, int Kst, const int* __restrict__ rmap, int n, int hc, int nkc,
                 const double* __restrict__ X, double* __restrict__ Y, ColMap M) {
    constexpr int H = 16 * TH;
    constexpr int MT = TH; // 8-row blocks per warp per GEMM (H/2 half-rows per warp)
    constexpr int BMP = H + 4;
    constexpr int BND = 2 * BNC;     // doubles per tile row
    constexpr int BNP = BND + 4;     // == 4 (mod 16): conflict-free fragment loads
    constexpr int NF = BND / 32;     // 8-column fragments per warp
    constexpr int RPP = kThreads / BNC; // smem rows per loader pass
    constexpr int SR = 2 * KC; // smem rows per stage: KC top + KC bottom
    static_assert(!RL || (kThreads % SR == 0 && BNC % (kThreads / SR) == 0 && BNC / (kThreads / SR) <= 32),
                  "row-lane loader geometry");
    // RL keeps a stage column-major, [complex column][row (SRP)][re, im]: a warp's
    // 32 rows of one column land contiguously (row-major staging would split every
    // 32 B sector over two smem rows and fetch it twice); SRP == 4 (mod 8) keeps
    // the B-fragment loads at two wavefronts
    constexpr int SRP = SR + 4;
    constexpr int STAGE_D = RL ? BNC * SRP * 2 : SR * BNP; // doubles per stage
    extern __shared__ __align__(16) double smem[];
    const int Kp = nkc * KC;
    double* Ae = smem;                        // [Kp][BMP]
    double* Ao = Ae + (size_t)Kp * BMP;       // [Kp][BMP]
    double* Bs = Ao + (size_t)Kp * BMP;       // [STG][SR][BNP]
    int* rE = reinterpret_cast<int*>(Bs + (size_t)STG * STAGE_D); // [H] even eigen-indices
    int* rO = rE + H;                                               // [H] odd eigen-indices
    const int no = n - hc;
    const long long in_rs = (M.mode == MAP_TIN || M.mode == MAP_TIN1) ? 2 * M.Np : 2 * M.s;
    const long long out_rs = (M.mode == MAP_TOUT || M.mode == MAP_TOUT1) ? 2 * M.Np : 2 * M.s;
    const long long ntiles = M.ntiles;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wr = warp & 1, wc = warp >> 1;

    for (int e = tid; e < Kp * H; e += kThreads) {
        const int k = e / H, r = e - k * H;
        const bool v = k < Kst;
        Ae[k * BMP + r] = v ? __ldg(Af + e) : 0.0;
        Ao[k * BMP + r] = v ? __ldg(Af + (size_t)Kst * H + e) : 0.0;
    }
    for (int e = tid; e < 2 * H; e += kThreads) rE[e] = __ldg(rmap + e);
    __syncthreads();

    const int lcp = tid % BNC, lrow0 = tid / BNC;
    const int my_tiles =
        ntiles > (long long)blockIdx.x ? (int)((ntiles - 1 - (long long)blockIdx.x) / gridDim.x + 1) : 0;
    const int nwork = my_tiles * nkc;
    long long cur_tile = -1, cur_in = 0;
    bool cur_valid = false;

    // RL loader state: the thread's row and the column offsets of its NPASS columns
    constexpr int CPP = kThreads / SR, NPASS = RL ? BNC / CPP : 1;
    long long rl_in[NPASS];
    unsigned rl_valid = 0;
    auto issue = [&](int w) {
        if (RL) {
            if (w < nwork) {
                const int wt = w / nkc;
                const long long tile = (long long)blockIdx.x + (long long)wt * gridDim.x;
                const int kc = w - wt * nkc;
                if (tile != cur_tile) {
                    const TileBase tb = tile_base(M, tile);
                    rl_valid = 0;
#pragma unroll
                    for (int c = 0; c < NPASS; ++c) {
                        long long dummy;
                        if (colmap(M, n, tb, tid / SR + CPP * c, rl_in[c], dummy)) rl_valid |= 1u << c;
                    }
                    cur_tile = tile;
                }
                double* bs = Bs + (size_t)(w % STG) * STAGE_D;
                const int jj = tid % SR;
                const int q = kc * KC + (jj % KC);
                int src;
                bool v;
                if (!INV) {
                    src = jj < KC ? q : n - 1 - q;
                    v = jj < KC ? q < hc : q < n - hc;
                } else {
                    v = jj < KC ? q < hc : q < no;
                    src = v ? (jj < KC ? rE[q] : rO[q]) : 0;
                }
#pragma unroll
                for (int c = 0; c < NPASS; ++c) {
                    const bool vc = v && ((rl_valid >> c) & 1u);
                    const int col = tid / SR + CPP * c;
                    cp_async16(bs + 2 * (col * SRP + jj), vc ? (const void*)in_row<ROWS>(M, X, rl_in[c], src, in_rs) : (const void*)X,
                               vc);
                }
            }
            cp_async_commit();
            return;
        }
        if (w < nwork) {
            const int wt = w / nkc;
            const long long tile = (long long)blockIdx.x + (long long)wt * gridDim.x;
            const int kc = w - wt * nkc;
            if (tile != cur_tile) {
                long long dummy;
                cur_valid = colmap(M, n, tile_base(M, tile), lcp, cur_in, dummy);
                cur_tile = tile;
            }
            double* bs = Bs + (size_t)(w % STG) * SR * BNP;
#pragma unroll
            for (int k = 0; k < SR / RPP; ++k) {
                const int jj = lrow0 + RPP * k; // smem row 0..SR-1
                const int q = kc * KC + (jj % KC);
                int src;
                bool v;
                if (!INV) {
                    src = jj < KC ? q : n - 1 - q;
                    v = jj < KC ? q < hc : q < n - hc; // odd n: the middle row has no mirror
                } else {
                    v = jj < KC ? q < hc : q < no;
                    src = v ? (jj < KC ? rE[q] : rO[q]) : 0;
                }
                v = v && cur_valid;
                cp_async16(bs + jj * BNP + 2 * lcp, v ? (const void*)in_row<ROWS>(M, X, cur_in, src, in_rs) : (const void*)X,
                           v);
            }
        }
        cp_async_commit();
    };

    double acc[2][MT][NF][2];
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int m = 0; m < NF; ++m) acc[g][i][m][0] = acc[g][i][m][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STG - 1; ++s) issue(s);

    const int r_warp = wr * (H / 2), c_warp = wc * (BND / 4);
    const int ar = lane >> 2, ak = lane & 3;
    const int cr = lane >> 2;
    for (int w = 0; w < nwork; ++w) {
        cp_async_wait<STG - 2>();
        __syncthreads();
        issue(w + STG - 1);
        const int kc = w % nkc;
        const double* bs = Bs + (size_t)(w % STG) * STAGE_D;
#pragma unroll
        for (int k4 = 0; k4 < KC; k4 += 4) {
            const int kr = kc * KC + k4 + ak;
            double ae[MT], ao[MT], be[NF], bo[NF];
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                ae[i] = Ae[kr * BMP + r_warp + i * 8 + ar];
                ao[i] = Ao[kr * BMP + r_warp + i * 8 + ar];
            }
#pragma unroll
            for (int m = 0; m < NF; ++m) {
                const int dc = c_warp + m * 8 + ar; // double column
                const double t = RL ? bs[2 * ((dc >> 1) * SRP + k4 + ak) + (dc & 1)] : bs[(k4 + ak) * BNP + dc];
                const double b = RL ? bs[2 * ((dc >> 1) * SRP + KC + k4 + ak) + (dc & 1)] : bs[(KC + k4 + ak) * BNP + dc];
                be[m] = INV ? t : t + b;
                bo[m] = INV ? b : t - b;
            }
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int m = 0; m < NF; ++m) {
                    dmma_m8n8k4(acc[0][i][m][0], acc[0][i][m][1], ae[i], be[m]);
                    dmma_m8n8k4(acc[1][i][m][0], acc[1][i][m][1], ao[i], bo[m]);
                }
        }
        if (kc == nkc - 1) {
            const long long tile = (long long)blockIdx.x + (long long)(w / nkc) * gridDim.x;
            const TileBase tbase = tile_base(M, tile);
#pragma unroll
            for (int m = 0; m < NF; ++m) {
                const int jcol = (c_warp >> 1) + m * 4 + (lane & 3);
                long long io, oo;
                if (colmap(M, n, tbase, jcol, io, oo)) {
#pragma unroll
                    for (int i = 0; i < MT; ++i) {
                        const int h = r_warp + i * 8 + cr;
                        const double2 e = make_double2(acc[0][i][m][0], acc[0][i][m][1]);
                        const double2 o = make_double2(acc[1][i][m][0], acc[1][i][m][1]);
                        if (!INV) {
                            if (h < hc) __stcs(reinterpret_cast<double2*>(out_row<ROWS>(M, Y, oo, rE[h], out_rs)), e);
                            if (h < no) __stcs(reinterpret_cast<double2*>(out_row<ROWS>(M, Y, oo, rO[h], out_rs)), o);
                        } else if (h < hc) {
                            const double2 v1 = make_double2(e.x + o.x, e.y + o.y);
                            __stcs(reinterpret_cast<double2*>(out_row<ROWS>(M, Y, oo, h, out_rs)), v1);
                            if (n - 1 - h != h) {
                                const double2 v2 = make_double2(e.x - o.x, e.y - o.y);
                                __stcs(reinterpret_cast<double2*>(out_row<ROWS>(M, Y, oo, n - 1 - h, out_rs)), v2);
                            }
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < MT; ++i)
                    acc[0][i][m][0] = acc[0][i][m][1] = acc[1][i][m][0] = acc[1][i][m][1] = 0.0;
            }
        }
    }
    cp_async_wait<0>();
}

// tile width (complex columns) of a column map; T modes block it as tbt x tbr
void set_tile_width(ColMap& M, int tw) {
    M.tw = tw;
    if (M.mode == MAP_STD || M.mode >= MAP_TOUT1) {
        M.ntiles = (M.Q + tw - 1) / tw;
    } else {
        M.tbr = M.Np >= 8 ? 8 : (M.Np >= 4 ? 4 : (M.Np >= 2 ? 2 : 1));
        M.tbt = tw / M.tbr;
        M.ntb = (M.nt + M.tbt - 1) / M.tbt;
        M.ntiles = M.ntb * ((M.Np + M.tbr - 1) / M.tbr);
    }
}

template <int TH, bool INV, int KC, int STG, int MINB, int BNC>
void launch_fold_cfg(const FoldAxis& F, const double* X, double* Y, ColMap M, cudaStream_t st) {
    constexpr int H = 16 * TH;
    const int nkc = (F.hc + KC - 1) / KC;
    const bool rl = M.mode == MAP_TIN1 && !M.rin && !M.rout; // column-major stages (row-lane loader)
    const size_t stage_d = rl ? (size_t)BNC * (2 * KC + 4) * 2 : (size_t)2 * KC * (2 * BNC + 4);
    const size_t sm = (size_t)2 * nkc * KC * (H + 4) * sizeof(double) + (size_t)2 * H * sizeof(int) +
                      (size_t)STG * stage_d * sizeof(double);
    KS_REQUIRE(sm <= 227 * 1024, KS_EINVAL, "folded mode product: axis too long");
    set_tile_width(M, BNC);
    const int per_sm = std::max(1, std::min(MINB, (int)((227 * 1024) / sm)));
    const unsigned g = (unsigned)std::min<long long>(M.ntiles, (long long)device_sms() * per_sm);
    const double* A = (INV ? F.inv : F.fwd).as<double>();
    if (M.rin || M.rout) { // peer-memory rows (sharded middle phase)
        auto k = k_mode_gemm_fold<TH, INV, KC, STG, MINB, BNC, true>;
        smem_optin((const void*)k, (int)sm);
        k<<<g, kThreads, sm, st>>>(A, F.kst, F.rmap.as<int>(), F.n, F.hc, nkc, X, Y, M);
    } else if (M.mode == MAP_TIN1 || M.mode == MAP_TOUT1) {
        // axis-1 time-major side: rows are stored by position (even eigen-indices
        // first, then odd), so the time-major row map is the position map
        const int* rm = F.rpos.as<int>();
        if (M.mode == MAP_TIN1) {
            auto k = k_mode_gemm_fold<TH, INV, KC, STG, MINB, BNC, false, true>;
            smem_optin((const void*)k, (int)sm);
            k<<<g, kThreads, sm, st>>>(A, F.kst, rm, F.n, F.hc, nkc, X, Y, M);
        } else {
            auto k = k_mode_gemm_fold<TH, INV, KC, STG, MINB, BNC>;
            smem_optin((const void*)k, (int)sm);
            k<<<g, kThreads, sm, st>>>(A, F.kst, rm, F.n, F.hc, nkc, X, Y, M);
        }
    } else {
        auto k = k_mode_gemm_fold<TH, INV, KC, STG, MINB, BNC>;
        smem_optin((const void*)k, (int)sm);
        k<<<g, kThreads, sm, st>>>(A, F.kst, F.rmap.as<int>(), F.n, F.hc, nkc, X, Y, M);
    }
    check_launch("k_mode_gemm_fold");
}

template <int TH, bool INV>
void launch_fold_th(const FoldAxis& F, const double* X, double* Y, const ColMap& M, cudaStream_t st) {
    if (TH <= 2) {
        // Variants measured at c3 (n = 64, six transforms per FD apply;
        // profiles/round1_part2_summary.md, round1_part5_summary.md):
        //   (KC 16, 2 stages, 2 CTA/SM, 64-column tiles)  0.847-0.864 ms   <- kept
        //   (KC  8, 4 stages, 2 CTA/SM)                   0.895 ms
        //   32-column tiles, 3-4 stages, 2-3 CTA/SM       0.867 ms
        //   1 CTA/SM, 3-4 stages                          1.08 ms
        //   smem-staged row-wise stores                   0.98-1.06 ms
        //   TMA bulk row loads + mbarrier                 0.862 ms
        return launch_fold_cfg<TH, INV, 16, 2, 2, 64>(F, X, Y, M, st);
    }
    // small problems (c1, c2: fewer 64-column tiles than SMs): 32-column tiles
    // give twice the CTAs
    if (M.mode == MAP_STD && !M.rin && !M.rout && (M.Q + 63) / 64 < device_sms()) {
        constexpr int Hs = 16 * TH;
        const int nkc8 = (F.hc + 7) / 8;
        const size_t sm32 = (size_t)2 * nkc8 * 8 * (Hs + 4) * sizeof(double) + (size_t)2 * Hs * sizeof(int) +
                            (size_t)4 * 16 * (64 + 4) * sizeof(double);
        if (sm32 <= 227 * 1024) return launch_fold_cfg<TH, INV, 8, 4, 1, 32>(F, X, Y, M, st);
    }
    // long axes: resident halves are large -> 1 CTA/SM; 2 stages when 4 do not fit
    constexpr int H = 16 * TH;
    const int nkc = (F.hc + 7) / 8;
    const size_t sm4 = (size_t)2 * nkc * 8 * (H + 4) * sizeof(double) + (size_t)2 * H * sizeof(int) +
                       (size_t)4 * 16 * (kBN + 4) * sizeof(double);
    if (sm4 <= 227 * 1024) return launch_fold_cfg<TH, INV, 8, 4, 1, 64>(F, X, Y, M, st);
    return launch_fold_cfg<TH, INV, 8, 2, 1, 64>(F, X, Y, M, st);
}

ColMap make_colmap(int n, size_t s_complex, size_t outer, int layout, int nt) {
    ColMap M{};
    M.mode = layout;
    M.s = (long long)s_complex;
    M.Q = (long long)s_complex * (long long)outer;
    if (layout == MAP_STD) {
        M.ntiles = (M.Q + 63) / 64;
    } else if (layout >= MAP_TOUT1) {
        KS_REQUIRE(nt > 0 && s_complex == (size_t)nt, KS_EINVAL, "axis-1 time-major transform needs axis 1");
        M.nt = nt;
        M.Np = 1;
        M.Ns = (long long)n * (long long)outer;
        M.ntiles = (M.Q + 63) / 64;
    } else {
        KS_REQUIRE(outer == 1 && nt > 0 && s_complex % (size_t)nt == 0, KS_EINVAL,
                   "time-major transform needs the outermost axis");
        M.nt = nt;
        M.Np = (long long)s_complex / nt;
        M.Ns = M.Np * n;
        M.tbr = M.Np >= 8 ? 8 : (M.Np >= 4 ? 4 : (M.Np >= 2 ? 2 : 1));
        M.tbt = 64 / M.tbr;
        M.ntb = (nt + M.tbt - 1) / M.tbt;
        M.ntiles = M.ntb * ((M.Np + M.tbr - 1) / M.tbr);
    }
    return M;
}

} // namespace

bool fold_axis_build(const double* U_in, const double* lam, int n, double tol, FoldAxis& F) {
    // U column-major: U(j, r) = U[j + r*n]
    if (n < 2 || n > 160) return false; // (long axes: the dense panel kernel)
    if (const char* e = std::getenv("KS_FD_FOLD"))
        if (std::strcmp(e, "0") == 0) return false;
    const int hc = (n + 1) / 2;
    std::vector<double> Uw(U_in, U_in + (size_t)n * n); // columns may be re-combined below
    const double* U = Uw.data();
    auto parity_dev = [&](int r, double& de, double& dd) {
        const double* u = U + (size_t)r * n;
        double mx = 0;
        de = dd = 0;
        for (int j = 0; j < n; ++j) {
            mx = std::max(mx, std::fabs(u[j]));
            de = std::max(de, std::fabs(u[j] - u[n - 1 - j]));
            dd = std::max(dd, std::fabs(u[j] + u[n - 1 - j]));
        }
        de /= mx;
        dd /= mx;
    };
    // Columns that are not even/odd to `tol`: (a) nearly so (<= 1e-6: the
    // eigensolver's error on a moderately close outlier pair; symmetrising such a
    // column moves an FD application by ~2e-14, tests/test_gpu_fold.py) -- symmetrised like the
    // rest; (b) mixed halves of a near-degenerate pair (relative gap <= 1e-10,
    // the outlier modes of p >= 3 splines) -- replaced by the even and the odd
    // combination of the pair (S c with |c| = 1, so still M-orthonormal). The
    // preconditioner then changes by the pair's eigenvalue gap (<= 1e-10
    // relative), and otherwise the axis stays dense.
    std::vector<int> mixed;
    for (int r = 0; r < n; ++r) {
        double de, dd;
        parity_dev(r, de, dd);
        if (!(std::isfinite(de) && std::isfinite(dd))) return false;
        if (std::min(de, dd) > 1e-6) mixed.push_back(r);
    }
    std::vector<bool> used(n, false);
    for (int a : mixed) {
        if (used[a]) continue;
        int b = -1;
        for (int c : mixed)
            if (c != a && !used[c] && (b < 0 || std::fabs(lam[c] - lam[a]) < std::fabs(lam[b] - lam[a]))) b = c;
        if (b < 0 || !(std::fabs(lam[b] - lam[a]) <= 1e-10 * std::fabs(lam[a]))) return false;
        used[a] = used[b] = true;
        // smallest right singular vectors of the odd / even parts of S = [u_a u_b]
        auto small_vec = [&](double sign, double c[2]) {
            double g00 = 0, g01 = 0, g11 = 0;
            const double* ua = U + (size_t)a * n;
            const double* ub = U + (size_t)b * n;
            for (int j = 0; j < n; ++j) {
                const double x = 0.5 * (ua[j] + sign * ua[n - 1 - j]), y = 0.5 * (ub[j] + sign * ub[n - 1 - j]);
                g00 += x * x;
                g01 += x * y;
                g11 += y * y;
            }
            // eigenvector of the smaller eigenvalue of [[g00 g01][g01 g11]]
            const double tr = g00 + g11, det = g00 * g11 - g01 * g01;
            const double lmin = 0.5 * tr - std::sqrt(std::max(0.0, 0.25 * tr * tr - det));
            double c0 = g01, c1 = lmin - g00;
            if (std::fabs(c0) + std::fabs(c1) < 1e-300) {
                c0 = lmin - g11;
                c1 = g01;
            }
            if (std::fabs(c0) + std::fabs(c1) < 1e-300) {
                c0 = 1.0;
                c1 = 0.0;
            }
            const double nr = std::sqrt(c0 * c0 + c1 * c1);
            c[0] = c0 / nr;
            c[1] = c1 / nr;
        };
        double ce[2], co[2];
        small_vec(-1.0, ce); // kills the odd part -> even combination
        small_vec(+1.0, co); // kills the even part -> odd combination
        std::vector<double> ve(n), vo(n);
        for (int j = 0; j < n; ++j) {
            const double ua = Uw[(size_t)a * n + j], ub = Uw[(size_t)b * n + j];
            ve[j] = ce[0] * ua + ce[1] * ub;
            vo[j] = co[0] * ua + co[1] * ub;
        }
        std::copy(ve.begin(), ve.end(), Uw.begin() + (size_t)a * n);
        std::copy(vo.begin(), vo.end(), Uw.begin() + (size_t)b * n);
    }
    std::vector<int> E, O;
    for (int r = 0; r < n; ++r) {
        double de, dd;
        parity_dev(r, de, dd);
        const double lim = std::max(tol, 1e-6);
        if (std::min(de, dd) > lim) return false;
        (de <= dd ? E : O).push_back(r);
    }
    if ((int)E.size() != hc) return false;
    const int th = (hc + 15) / 16;
    if (th > 5) return false;
    const int H = 16 * th, Kp = 16 * ((hc + 15) / 16); // stored k rows (multiple of 16)
    std::vector<double> fwd((size_t)2 * Kp * H, 0.0), inv((size_t)2 * Kp * H, 0.0);
    std::vector<int> rmap((size_t)2 * H, 0);
    const int no = n - hc;
    for (int m = 0; m < hc; ++m) rmap[m] = E[m];
    for (int m = 0; m < no; ++m) rmap[H + m] = O[m];
    for (int j = 0; j < hc; ++j) {
        const int jm = n - 1 - j;
        for (int m = 0; m < hc; ++m) { // even: s_e[j][E_m]
            const double* u = U + (size_t)E[m] * n;
            const double se = jm == j ? u[j] : 0.5 * (u[j] + u[jm]);
            fwd[(size_t)j * H + m] = se;        // forward: k = j, row = m
            inv[(size_t)m * H + j] = se;        // inverse: k = m, row = j
        }
        for (int m = 0; m < no; ++m) { // odd: s_o[j][O_m]
            const double* u = U + (size_t)O[m] * n;
            const double so = jm == j ? 0.0 : 0.5 * (u[j] - u[jm]);
            fwd[(size_t)Kp * H + (size_t)j * H + m] = so;
            inv[(size_t)Kp * H + (size_t)m * H + j] = so;
        }
    }
    F.n = n;
    F.hc = hc;
    F.th = th;
    F.kst = Kp;
    F.fwd.alloc(fwd.size() * sizeof(double));
    F.inv.alloc(inv.size() * sizeof(double));
    F.rmap.alloc(rmap.size() * sizeof(int));
    // position map of the axis-1 time-major layout: even eigenvectors at 0..hc-1, odd at hc..n-1
    std::vector<int> rpos((size_t)2 * H, 0);
    F.perm.assign(n, 0);
    for (int m = 0; m < hc; ++m) rpos[m] = m, F.perm[m] = E[m];
    for (int m = 0; m < no; ++m) rpos[H + m] = hc + m, F.perm[hc + m] = O[m];
    F.rpos.alloc(rpos.size() * sizeof(int));
    KS_CUDA(cudaMemcpy(F.rpos.p, rpos.data(), rpos.size() * sizeof(int), cudaMemcpyHostToDevice));
    KS_CUDA(cudaMemcpy(F.fwd.p, fwd.data(), fwd.size() * sizeof(double), cudaMemcpyHostToDevice));
    KS_CUDA(cudaMemcpy(F.inv.p, inv.data(), inv.size() * sizeof(double), cudaMemcpyHostToDevice));
    KS_CUDA(cudaMemcpy(F.rmap.p, rmap.data(), rmap.size() * sizeof(int), cudaMemcpyHostToDevice));
    return true;
}

void launch_mode_gemm_fold(const FoldAxis& F, bool inverse, const double* X, double* Y, size_t s_complex,
                           size_t outer, cudaStream_t st, int layout, int nt, const double* const* rows_in,
                           double* const* rows_out) {
    if (s_complex == 0 || outer == 0) return;
    ColMap M = make_colmap(F.n, s_complex, outer, layout, nt);
    M.rin = rows_in;
    M.rout = rows_out;
#define KS_FOLD_CASE(T)                                                                            \
    case T:                                                                                        \
        if (inverse) launch_fold_th<T, true>(F, X, Y, M, st);                                      \
        else launch_fold_th<T, false>(F, X, Y, M, st);                                             \
        break;
    switch (F.th) {
        KS_FOLD_CASE(1)
        KS_FOLD_CASE(2)
        KS_FOLD_CASE(3)
        KS_FOLD_CASE(4)
        KS_FOLD_CASE(5)
    default: throw Error(KS_EINVAL, "folded mode product: bad tile height");
    }
#undef KS_FOLD_CASE
}

int transform_engine() { return 2; } // DMMA (the only engine)

void launch_mode_gemm(const double* At, int n, const double* X, double* Y, size_t s_complex,
                      size_t outer, cudaStream_t st, int layout, int nt, const double* const* rows_in,
                      double* const* rows_out) {
    const long long W2 = 2 * (long long)s_complex;
    const long long C = W2 * (long long)outer;
    if (C == 0 || n == 0) return;
    if (layout != MAP_STD || rows_in || rows_out)
        KS_REQUIRE(layout == MAP_STD || (outer == 1 && nt > 0 && s_complex % (size_t)nt == 0), KS_EINVAL,
                   "time-major transform needs the outermost axis");
    ColMap M{};
    M.rin = rows_in;
    M.rout = rows_out;
    M.mode = layout;
    M.s = (long long)s_complex;
    M.Q = (long long)s_complex * (long long)outer;
    if (layout == MAP_STD) {
        M.ntiles = (M.Q + 63) / 64;
    } else {
        M.nt = nt;
        M.Np = (long long)s_complex / nt;
        M.Ns = M.Np * n;
        M.tbr = M.Np >= 8 ? 8 : (M.Np >= 4 ? 4 : (M.Np >= 2 ? 2 : 1));
        M.tbt = 64 / M.tbr;
        M.ntb = (nt + M.tbt - 1) / M.tbt;
        M.ntiles = M.ntb * ((M.Np + M.tbr - 1) / M.tbr);
    }
    const int tm = (n + 15) / 16;
    if (tm > 10) return launch_panel(At, n, X, Y, st, &M); // long axes: matrix panels streamed beside X
    switch (tm) {
    case 1: launch_tm<1>(At, n, X, Y, st, &M); break;
    case 2: launch_tm<2>(At, n, X, Y, st, &M); break;
    case 3: launch_tm<3>(At, n, X, Y, st, &M); break;
    case 4: launch_tm<4>(At, n, X, Y, st, &M); break;
    case 5: launch_tm<5>(At, n, X, Y, st, &M); break;
    case 6: launch_tm<6>(At, n, X, Y, st, &M); break;
    case 7: launch_tm<7>(At, n, X, Y, st, &M); break;
    case 8: launch_tm<8>(At, n, X, Y, st, &M); break;
    case 9: launch_tm<9>(At, n, X, Y, st, &M); break;
    case 10: launch_tm<10>(At, n, X, Y, st, &M); break;
    }
}

} // namespace ks
