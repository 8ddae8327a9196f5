// Fused outermost-axis step of the FD apply: for each "rest column" rho
// (a fixed index of axes 1..d-1; rho < Np), the slab X[:, rho, :] of all n_t
// times and all n_d values of the outermost axis is loaded ONCE into shared
// memory, then
//   1. forward transform  Y = U_d^T X   (DMMA m8n8k4, result back to smem)
//   2. block solves       one thread per fiber (i_d, rho): the fiber is row
//                         i_d of the smem tile (time contiguous); factors are
//                         streamed from HBM in the per-column layout
//                         [rho][k][e][i_d] (coalesced), 8 steps ahead in
//                         register rings
//   3. inverse transform  Z = U_d Y, stored to HBM in natural layout.
// Versus the unfused path (time-major transform, separate solve kernel,
// time-major inverse transform) this removes four full-tensor HBM passes
// (2.2 GB at c3) and one launch; the tensor is read once and written once.
// Reference: fdsolver.cpp:7-21 (transforms), :58-60 + eigensolve.cpp:123-140
// (block solves). Mode products on distinct axes commute, so doing axis d last
// forward / first inverse changes only rounding.
//
// Shapes: n_d <= 96 (TM = 4 or 6 row tiles of 16), n_t <= 72 (2*n_t <= 144
// doubles = 18 n8 column tiles), p <= 8. Larger problems use the unfused path.
#include "ks_internal.hpp"

#include <algorithm>

namespace ks {

namespace {

__device__ __forceinline__ double2 cmul2(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 csub2(double2 a, double2 b) {
    return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double2 cdiv2(double2 num, double2 den) { // libgcc __divdc3 (Smith)
    const double a = num.x, b = num.y, c = den.x, d = den.y;
    double x, y;
    if (fabs(c) < fabs(d)) {
        const double ratio = c / d, denom = (c * ratio) + d;
        x = ((a * ratio) + b) / denom;
        y = ((b * ratio) - a) / denom;
    } else {
        const double ratio = d / c, denom = (d * ratio) + c;
        x = ((b * ratio) + a) / denom;
        y = (b - (a * ratio)) / denom;
    }
    return make_double2(x, y);
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void* dst, const void* src, bool v) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(v ? 16 : 0));
}

constexpr int kThr = 256;   // 8 warps: 4 row groups x 2 column halves
constexpr int kNTW = 9;     // n8 column tiles per warp (<= 144 doubles per tile row)
constexpr int kPD = 146;    // smem row pitch (doubles): pitch/2 odd -> conflict-free fiber access
// factor prefetch depth (steps): forward ring P complex per step, backward 2P+1
template <int P> struct Depth {
    static constexpr int F = P <= 2 ? 8 : 4;
    static constexpr int B = P <= 2 ? 4 : 2;
};

// GEMM on the smem tile: acc = A (BM x BM, from global k-major At[j*nd + r]) * T (BM x NC)
template <int TM>
__device__ __forceinline__ void tile_gemm(const double* __restrict__ At, int nd, const double* T,
                                          int nc8, double (&acc)[TM / 2][kNTW][2]) {
    constexpr int MTW = TM / 2;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wr = warp & 3, wc = warp >> 2;
    const int ar = lane >> 2, ak = lane & 3;
    const int n0 = wc == 0 ? 0 : (nc8 + 1) / 2;           // first n8 tile of this warp
    const int nn = wc == 0 ? (nc8 + 1) / 2 : nc8 / 2;     // tiles of this warp
#pragma unroll
    for (int i = 0; i < MTW; ++i)
#pragma unroll
        for (int m = 0; m < kNTW; ++m) acc[i][m][0] = acc[i][m][1] = 0.0;
    const int kpad = (nd + 3) & ~3;
    for (int k4 = 0; k4 < kpad; k4 += 4) {
        const int k = k4 + ak;
        double a[MTW];
#pragma unroll
        for (int i = 0; i < MTW; ++i) {
            const int r = (wr * MTW + i) * 8 + ar;
            a[i] = (k < nd && r < nd) ? __ldg(At + (size_t)k * nd + r) : 0.0;
        }
#pragma unroll
        for (int m = 0; m < kNTW; ++m) {
            if (m < nn) {
                const double b = T[k * kPD + (n0 + m) * 8 + ar];
#pragma unroll
                for (int i = 0; i < MTW; ++i) dmma(acc[i][m][0], acc[i][m][1], a[i], b);
            }
        }
    }
}

template <int TM, int P>
__global__ void __launch_bounds__(kThr, 2)
k_fd_fused(const double* __restrict__ Atf, const double* __restrict__ Ati,
           const double2* __restrict__ ab, const unsigned char* __restrict__ piv, int nt, int nd,
           long long Np, const double2* __restrict__ X, double2* __restrict__ Z) {
    constexpr int BM = 16 * TM, MTW = TM / 2;
    constexpr int ldab = 3 * P + 1, kuf = 2 * P;
    extern __shared__ __align__(16) double T[]; // [BM][kPD]
    const long long rho = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nc = 2 * nt;                 // doubles per row
    const int nc8 = (nc + 7) / 8;          // n8 tiles
    const long long rs = 2LL * nt * Np;    // natural row stride (doubles) of the axis-d index
    const double* xs = reinterpret_cast<const double*>(X) + 2LL * nt * rho;
    // 0. load the slab (rows i_d, nt complex each) + zero padding
    for (int e = tid; e < BM * (nc8 * 4); e += kThr) {
        const int r = e / (nc8 * 4), c2 = e - r * (nc8 * 4); // c2: 16-byte chunk in the row
        const bool v = r < nd && 2 * c2 < nc;
        cp16(T + r * kPD + 2 * c2, v ? (const void*)(xs + r * rs + 2 * c2) : (const void*)xs, v);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
    __syncthreads();
    // 1. forward transform
    double acc[MTW][kNTW][2];
    tile_gemm<TM>(Atf, nd, T, nc8, acc);
    __syncthreads();
    {
        const int wr = warp & 3, wc = warp >> 2;
        const int n0 = wc == 0 ? 0 : (nc8 + 1) / 2, nn = wc == 0 ? (nc8 + 1) / 2 : nc8 / 2;
#pragma unroll
        for (int i = 0; i < MTW; ++i)
#pragma unroll
            for (int m = 0; m < kNTW; ++m)
                if (m < nn) {
                    const int r = (wr * MTW + i) * 8 + (lane >> 2);
                    *reinterpret_cast<double2*>(T + r * kPD + (n0 + m) * 8 + 2 * (lane & 3)) =
                        make_double2(acc[i][m][0], acc[i][m][1]);
                }
    }
    __syncthreads();
    // 2. block solves: thread r owns fiber r (row r of the tile, time contiguous)
    if (tid < nd) {
        const int r = tid;
        double2* x = reinterpret_cast<double2*>(T + r * kPD);
        const double2* fb = ab + (size_t)rho * nt * ldab * nd + r;
        const unsigned char* pb = piv + (size_t)rho * nt * nd + r;
        auto band = [&](int k, int e) -> double2 { return __ldg(fb + ((size_t)k * ldab + e) * nd); };
        const double2 Zc = make_double2(0.0, 0.0);
        // forward (L with interchanges), factors DF steps ahead
        constexpr int DF = Depth<P>::F;
        double2 w[P + 1];
#pragma unroll
        for (int m = 0; m <= P; ++m) w[m] = m < nt ? x[m] : Zc;
        double2 LR[DF][P];
        int PR[DF];
#pragma unroll
        for (int c = 0; c < DF; ++c) {
            PR[c] = c < nt ? pb[(size_t)c * nd] : 0;
#pragma unroll
            for (int m = 1; m <= P; ++m) LR[c][m - 1] = (c + m < nt) ? band(c, kuf + m) : Zc;
        }
        for (int kb = 0; kb < nt; kb += DF) {
#pragma unroll
            for (int c = 0; c < DF; ++c) {
                const int k = kb + c;
                if (k < nt) {
                    const int po = PR[c];
#pragma unroll
                    for (int m = 1; m <= P; ++m)
                        if (po == m) {
                            const double2 t = w[0];
                            w[0] = w[m];
                            w[m] = t;
                        }
#pragma unroll
                    for (int m = 1; m <= P; ++m) w[m] = csub2(w[m], cmul2(LR[c][m - 1], w[0]));
                    x[k] = w[0];
#pragma unroll
                    for (int m = 0; m < P; ++m) w[m] = w[m + 1];
                    w[P] = (k + P + 1 < nt) ? x[k + P + 1] : Zc;
                    const int kn = k + DF;
                    PR[c] = kn < nt ? pb[(size_t)kn * nd] : 0;
#pragma unroll
                    for (int m = 1; m <= P; ++m) LR[c][m - 1] = (kn + m < nt) ? band(kn, kuf + m) : Zc;
                }
            }
        }
        // backward (U, column oriented), factors DB steps ahead
        constexpr int DB = Depth<P>::B;
        double2 u[2 * P + 1];
#pragma unroll
        for (int j = 0; j <= 2 * P; ++j) u[j] = (nt - 1 - j >= 0) ? x[nt - 1 - j] : Zc;
        double2 UR[DB][2 * P + 1];
#pragma unroll
        for (int c = 0; c < DB; ++c) {
            const int k = nt - 1 - c;
#pragma unroll
            for (int j = 0; j <= 2 * P; ++j) UR[c][j] = k >= 0 ? band(k, kuf - j) : Zc;
        }
        for (int kb = nt - 1; kb >= 0; kb -= DB) {
#pragma unroll
            for (int c = 0; c < DB; ++c) {
                const int k = kb - c;
                if (k >= 0) {
                    u[0] = cdiv2(u[0], UR[c][0]);
#pragma unroll
                    for (int j = 1; j <= 2 * P; ++j) u[j] = csub2(u[j], cmul2(UR[c][j], u[0]));
                    x[k] = u[0];
#pragma unroll
                    for (int j = 0; j < 2 * P; ++j) u[j] = u[j + 1];
                    u[2 * P] = (k - 2 * P - 1 >= 0) ? x[k - 2 * P - 1] : Zc;
                    const int kn = k - DB;
#pragma unroll
                    for (int j = 0; j <= 2 * P; ++j) UR[c][j] = kn >= 0 ? band(kn, kuf - j) : Zc;
                }
            }
        }
    }
    __syncthreads();
    // 3. inverse transform, straight to HBM (natural layout)
    tile_gemm<TM>(Ati, nd, T, nc8, acc);
    {
        const int wr = warp & 3, wc = warp >> 2;
        const int n0 = wc == 0 ? 0 : (nc8 + 1) / 2, nn = wc == 0 ? (nc8 + 1) / 2 : nc8 / 2;
        double* zs = reinterpret_cast<double*>(Z) + 2LL * nt * rho;
#pragma unroll
        for (int i = 0; i < MTW; ++i)
#pragma unroll
            for (int m = 0; m < kNTW; ++m)
                if (m < nn) {
                    const int r = (wr * MTW + i) * 8 + (lane >> 2);
                    const int c = (n0 + m) * 8 + 2 * (lane & 3);
                    if (r < nd && c < nc)
                        *reinterpret_cast<double2*>(zs + r * rs + c) = make_double2(acc[i][m][0], acc[i][m][1]);
                }
    }
}

template <int TM, int P>
void launch_tp(const double* Atf, const double* Ati, const FdBlocks& B, int nd, long long Np,
               const double2* X, double2* Z, cudaStream_t st) {
    const size_t sm = (size_t)16 * TM * kPD * sizeof(double);
    static bool attr = false;
    if (!attr) {
        KS_CUDA(cudaFuncSetAttribute(k_fd_fused<TM, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        attr = true;
    }
    k_fd_fused<TM, P><<<(unsigned)Np, kThr, sm, st>>>(Atf, Ati, B.ab.as<double2>(), B.piv.as<unsigned char>(),
                                                       B.nt, nd, Np, X, Z);
    check_launch("k_fd_fused");
}

template <int TM>
void launch_t(int p, const double* Atf, const double* Ati, const FdBlocks& B, int nd, long long Np,
              const double2* X, double2* Z, cudaStream_t st) {
    switch (p) {
    case 1: launch_tp<TM, 1>(Atf, Ati, B, nd, Np, X, Z, st); break;
    case 2: launch_tp<TM, 2>(Atf, Ati, B, nd, Np, X, Z, st); break;
    case 3: launch_tp<TM, 3>(Atf, Ati, B, nd, Np, X, Z, st); break;
    case 4: launch_tp<TM, 4>(Atf, Ati, B, nd, Np, X, Z, st); break;
    default: throw Error(KS_EINVAL, "fused FD step: p > 4");
    }
}

} // namespace

bool fd_fused_supported(int nt, int nd, int p) { return nt <= 72 && nd <= 96 && p >= 1 && p <= 4; }

void launch_fd_fused(const double* At_fwd, const double* At_inv, const FdBlocks& B, int nd,
                     long long Np, const double2* X, double2* Z, cudaStream_t st) {
    KS_REQUIRE(fd_fused_supported(B.nt, nd, B.p) && B.fused_nd == nd, KS_EINVAL,
               "fused FD step: unsupported shape");
    if (nd <= 64) launch_t<4>(B.p, At_fwd, At_inv, B, nd, Np, X, Z, st);
    else launch_t<6>(B.p, At_fwd, At_inv, B, nd, Np, X, Z, st);
}

} // namespace ks
