// Fused folded transforms on spatial axes 1 and 2 (one HBM pass for two mode
// products of the FD apply, fdsolver.cpp:7-21 / tensorops.cpp:125-156).
//
// The FD apply's forward transform applies U_1^T on axis 1 and U_2^T on axis 2
// back to back (and the inverse U_1, U_2 back to back at the end). Run as two
// separate folded GEMMs (ks_transform.cu) each pass reads and writes the whole
// tensor (32 B/DOF each). Here one CTA owns a complete (axis-1 x axis-2) slab
// S[i2][i1] at one (t, outer) position -- n1*n2 complex = 64 KB at n = 64 --
// resident in shared memory:
//   load slab (cp.async, 16 B per element)
//   GEMM 1: folded even/odd product along i1, result written back into the slab
//   GEMM 2: folded even/odd product along i2, result stored straight to HBM
// so the pair costs one read and one write of the tensor. Both GEMMs are FP64
// DMMA (mma.m8n8k4.f64) with the same fragment layout as k_mode_gemm_fold and
// the same symmetrised half matrices (FoldAxis::fwd / inv, fold_axis_build).
//
// Slab layout: row = i2 slot, 2*i1slot + {re, im} within the row, pitch 2*N
// doubles, XOR-swizzled by (row & 3) so that the B fragments of both GEMMs
// (k along i1 for GEMM 1, k along i2 for GEMM 2) and the 16-byte epilogue
// writes are shared-memory-bank-conflict free. Forward: the slab is loaded in
// natural order and the eigen outputs kept in "half order" (even block, then
// odd block) until the final store maps them to their eigen-indices
// (FoldAxis::rmap). Inverse: the slab is loaded into half order and the
// unfold writes natural rows.
//
// Tiles are (t, outer) with t fastest, so concurrently running CTAs read the
// two 16-byte halves of the same 32-byte sectors (L2 merges them).
#include "ks_internal.hpp"

#include <cstdlib>
#include <cstring>

namespace ks {
namespace {

constexpr int kT12 = 256;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void* smem_dst, const void* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// XOR swizzle of a slab row: rows 4q..4q+3 -> 0, 8, 4, 12 (doubles)
__device__ __forceinline__ int swz(int row) { return (((row & 1) << 1) | ((row >> 1) & 1)) << 2; }

template <int N, bool INV>
__global__ void __launch_bounds__(kT12, 2)
k_fold12(const double* __restrict__ A1, const double* __restrict__ A2, int kst1, int kst2,
         const int* __restrict__ rmap1, const int* __restrict__ rmap2, const double* __restrict__ X,
         double* __restrict__ Y, int n0, long long ntiles) {
    constexpr int HC = N / 2;             // even (= odd) eigenvectors per axis
    constexpr int H = 16 * ((HC + 15) / 16); // stored rows of the half matrices
    constexpr int BMP = H + 4;            // == 4 (mod 16): conflict-free A fragments
    constexpr int P = 2 * N;              // slab row pitch (doubles)
    constexpr int MT = H / 16;            // 8-row blocks per warp (warp owns H/2 half-rows)
    constexpr int NF = P / 32;            // 8-column fragments per warp (4 warp columns)
    static_assert(N % 8 == 0 && P % 16 == 0, "k_fold12: N must be a multiple of 8");
    extern __shared__ __align__(16) double smem[];
    double* slab = smem;                     // [N][P]
    double* Ae1 = slab + (size_t)N * P;      // [HC][BMP] axis-1 even half, k-major
    double* Ao1 = Ae1 + HC * BMP;
    double* Ae2 = Ao1 + HC * BMP;
    double* Ao2 = Ae2 + HC * BMP;
    int* map1 = reinterpret_cast<int*>(Ao2 + HC * BMP); // [N] slot -> eigen index (fwd) / eigen index -> slot (inv)
    int* map2 = map1 + N;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wr = warp & 1, wc = warp >> 1;
    const int r_warp = wr * (H / 2), c_warp = wc * (P / 4);
    const int ar = lane >> 2, ak = lane & 3;

    for (int e = tid; e < HC * H; e += kT12) {
        const int k = e / H, r = e - k * H;
        Ae1[k * BMP + r] = __ldg(A1 + e);
        Ao1[k * BMP + r] = __ldg(A1 + (size_t)kst1 * H + e);
        Ae2[k * BMP + r] = __ldg(A2 + e);
        Ao2[k * BMP + r] = __ldg(A2 + (size_t)kst2 * H + e);
    }
    for (int s = tid; s < N; s += kT12) {
        const int e1 = s < HC ? __ldg(rmap1 + s) : __ldg(rmap1 + H + s - HC);
        const int e2 = s < HC ? __ldg(rmap2 + s) : __ldg(rmap2 + H + s - HC);
        if (!INV) {
            map1[s] = e1;
            map2[s] = e2;
        } else {
            map1[e1] = s;
            map2[e2] = s;
        }
    }
    __syncthreads();

    const long long col_stride = (long long)n0; // complex stride of axis 1
    auto tile_base = [&](long long tile) -> long long {
        const long long o = tile / n0, t = tile - o * n0;
        return t + (long long)n0 * N * N * o;
    };
    auto load = [&](long long tile) {
        const long long b = tile_base(tile);
        for (int e = tid; e < N * N; e += kT12) {
            const int i1 = e % N, i2 = e / N;
            const int s1 = INV ? map1[i1] : i1, s2 = INV ? map2[i2] : i2;
            cp16(slab + s2 * P + ((2 * s1) ^ swz(s2)), X + 2 * (b + col_stride * (i1 + (long long)N * i2)));
        }
        cp_commit();
    };

    long long tile = blockIdx.x;
    if (tile < ntiles) load(tile);
    for (; tile < ntiles; tile += gridDim.x) {
        cp_wait_all();
        __syncthreads();
        double acc[2][MT][NF][2];
        // ---------------- GEMM 1: along i1 (k = i1 slot), columns (i2, re/im)
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int m = 0; m < NF; ++m) acc[g][i][m][0] = acc[g][i][m][1] = 0.0;
#pragma unroll 2
        for (int k4 = 0; k4 < HC; k4 += 4) {
            const int kr = k4 + ak;
            double ae[MT], ao[MT], be[NF], bo[NF];
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                ae[i] = Ae1[kr * BMP + r_warp + i * 8 + ar];
                ao[i] = Ao1[kr * BMP + r_warp + i * 8 + ar];
            }
#pragma unroll
            for (int m = 0; m < NF; ++m) {
                const int col = c_warp + m * 8 + ar;
                const int row = col >> 1, cc = col & 1, sw = swz(row);
                const double* rp = slab + row * P;
                if (!INV) {
                    const double t = rp[(2 * kr + cc) ^ sw], b = rp[(2 * (N - 1 - kr) + cc) ^ sw];
                    be[m] = t + b;
                    bo[m] = t - b;
                } else {
                    be[m] = rp[(2 * kr + cc) ^ sw];
                    bo[m] = rp[(2 * (HC + kr) + cc) ^ sw];
                }
            }
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int m = 0; m < NF; ++m) {
                    dmma(acc[0][i][m][0], acc[0][i][m][1], ae[i], be[m]);
                    dmma(acc[1][i][m][0], acc[1][i][m][1], ao[i], bo[m]);
                }
        }
        __syncthreads(); // every warp done reading the slab
#pragma unroll
        for (int m = 0; m < NF; ++m) {
            const int q = (c_warp >> 1) + m * 4 + (lane & 3); // i2 slot (complex column)
            double* rp = slab + q * P;
            const int sw = swz(q);
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                const int h = r_warp + i * 8 + ar;
                if (h < HC) {
                    const double2 e = make_double2(acc[0][i][m][0], acc[0][i][m][1]);
                    const double2 o = make_double2(acc[1][i][m][0], acc[1][i][m][1]);
                    if (!INV) {
                        *reinterpret_cast<double2*>(rp + ((2 * h) ^ sw)) = e;
                        *reinterpret_cast<double2*>(rp + ((2 * (HC + h)) ^ sw)) = o;
                    } else {
                        *reinterpret_cast<double2*>(rp + ((2 * h) ^ sw)) = make_double2(e.x + o.x, e.y + o.y);
                        *reinterpret_cast<double2*>(rp + ((2 * (N - 1 - h)) ^ sw)) =
                            make_double2(e.x - o.x, e.y - o.y);
                    }
                }
            }
        }
        __syncthreads();
        // ---------------- GEMM 2: along i2 (k = i2 slot), columns (i1 slot, re/im)
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int m = 0; m < NF; ++m) acc[g][i][m][0] = acc[g][i][m][1] = 0.0;
#pragma unroll 2
        for (int k4 = 0; k4 < HC; k4 += 4) {
            const int kr = k4 + ak;
            double ae[MT], ao[MT], be[NF], bo[NF];
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                ae[i] = Ae2[kr * BMP + r_warp + i * 8 + ar];
                ao[i] = Ao2[kr * BMP + r_warp + i * 8 + ar];
            }
            const int rt = kr, rb = INV ? HC + kr : N - 1 - kr;
            const double* pt = slab + rt * P;
            const double* pb = slab + rb * P;
            const int st = swz(rt), sb = swz(rb);
#pragma unroll
            for (int m = 0; m < NF; ++m) {
                const int pos = c_warp + m * 8 + ar;
                const double t = pt[pos ^ st], b = pb[pos ^ sb];
                be[m] = INV ? t : t + b;
                bo[m] = INV ? b : t - b;
            }
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int m = 0; m < NF; ++m) {
                    dmma(acc[0][i][m][0], acc[0][i][m][1], ae[i], be[m]);
                    dmma(acc[1][i][m][0], acc[1][i][m][1], ao[i], bo[m]);
                }
        }
        __syncthreads(); // slab free: start the next tile's loads under this tile's stores
        const long long b = tile_base(tile);
        if (tile + gridDim.x < ntiles) load(tile + gridDim.x);
#pragma unroll
        for (int m = 0; m < NF; ++m) {
            const int q = (c_warp >> 1) + m * 4 + (lane & 3); // i1 slot
            const long long i1 = INV ? q : map1[q];
            double* yc = Y + 2 * (b + col_stride * i1);
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                const int h = r_warp + i * 8 + ar;
                if (h < HC) {
                    const double2 e = make_double2(acc[0][i][m][0], acc[0][i][m][1]);
                    const double2 o = make_double2(acc[1][i][m][0], acc[1][i][m][1]);
                    if (!INV) {
                        *reinterpret_cast<double2*>(yc + 2 * col_stride * N * map2[h]) = e;
                        *reinterpret_cast<double2*>(yc + 2 * col_stride * N * map2[HC + h]) = o;
                    } else {
                        *reinterpret_cast<double2*>(yc + 2 * col_stride * N * h) = make_double2(e.x + o.x, e.y + o.y);
                        *reinterpret_cast<double2*>(yc + 2 * col_stride * N * (N - 1 - h)) =
                            make_double2(e.x - o.x, e.y - o.y);
                    }
                }
            }
        }
    }
    cp_wait_all();
}

template <int N, bool INV>
void launch12(const FoldAxis& F1, const FoldAxis& F2, const double* X, double* Y, int n0, long long outer,
              cudaStream_t st) {
    constexpr int HC = N / 2, H = 16 * ((HC + 15) / 16), BMP = H + 4;
    const size_t sm = (size_t)N * 2 * N * sizeof(double) + (size_t)4 * HC * BMP * sizeof(double) +
                      (size_t)2 * N * sizeof(int);
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        KS_CUDA(cudaGetDevice(&dev));
        KS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        KS_CUDA(cudaFuncSetAttribute(k_fold12<N, INV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    }
    const long long ntiles = (long long)n0 * outer;
    const int per_sm = 2 * sm <= 227 * 1024 ? 2 : 1;
    const unsigned g = (unsigned)std::min<long long>(ntiles, (long long)sms * per_sm);
    const FoldAxis* f[2] = {&F1, &F2};
    const double* A1 = (INV ? f[0]->inv : f[0]->fwd).as<double>();
    const double* A2 = (INV ? f[1]->inv : f[1]->fwd).as<double>();
    k_fold12<N, INV><<<g, kT12, sm, st>>>(A1, A2, F1.kst, F2.kst, F1.rmap.as<int>(), F2.rmap.as<int>(), X, Y, n0,
                                         ntiles);
    check_launch("k_fold12");
}

} // namespace

bool fold12_supported(const FoldAxis& F1, const FoldAxis& F2) {
    // opt-in (KS_FD_FUSE12=1, read at handle creation). Measured at c3
    // (profiles/round1_part3_summary.md): 300-320 us per fused launch vs
    // 2 x 122-129 us for the two separate folded passes -- the slab kernel
    // loads/stores 16 B per element (t is the contiguous axis and a 64 KB slab
    // holds one t) and serialises load -> GEMM -> GEMM -> store per CTA; its
    // DMMA pipe is 40% active, i.e. the FP64 work of two axes alone (~128 us)
    // already exceeds one memory pass (~84 us).
    const char* e = std::getenv("KS_FD_FUSE12");
    if (!(e && std::strcmp(e, "1") == 0)) return false;
    if (!F1.n || !F2.n || F1.n != F2.n) return false;
    return F1.n == 64 || F1.n == 48 || F1.n == 32;
}

void launch_fold12(const FoldAxis& F1, const FoldAxis& F2, bool inverse, const double* X, double* Y, int n0,
                   long long outer, cudaStream_t st) {
    if (n0 == 0 || outer == 0) return;
#define KS_F12(NN)                                                                                 \
    case NN:                                                                                       \
        if (inverse) launch12<NN, true>(F1, F2, X, Y, n0, outer, st);                             \
        else launch12<NN, false>(F1, F2, X, Y, n0, outer, st);                                    \
        return;
    switch (F1.n) {
        KS_F12(64)
        KS_F12(48)
        KS_F12(32)
    default: throw Error(KS_EINVAL, "fused axis-1/2 transform: unsupported axis length");
    }
#undef KS_F12
}

} // namespace ks
