// Kronecker-sum matvec for d = 3 space + time (four tensor axes) in two
// launches: the outermost axis first, then the other three fused.
//
// KroneckerOperator::apply (tensorops.cpp:236-254) sums, over its terms,
// c * (F_t (x) F_1 (x) F_2 (x) F_3) x. Grouping the terms by their axis-3
// factor g,
//     y = sum_g  sum_{terms with F_3 = g}  c (F_t (x) F_1 (x) F_2) Z_g,   Z_g = (I (x) I (x) I (x) g) x,
// so the matvec is
//   K1 (k_axis3)  one streaming pass along axis 3: x -> Z_g for every distinct
//                 non-identity axis-3 factor (for the system operator A: M, L, V
//                 -- three tensors; an identity g uses x itself);
//   K2 (ks_k3)    axes t, 1, 2 fused, generated per plan and compiled with
//                 NVRTC: a CTA owns one axis-3 index and a tile of TX axis-1
//                 lines (all t) and sweeps axis 2. Plane i2 of every Z_g (the
//                 tile plus BW halo lines) streams through a cp.async ring; stage
//                 A applies the axis-1 factors (taps = neighbouring lines in the
//                 ring) and stages the distinct (g, F_1) products in shared
//                 memory; stage B applies the time factors (taps = neighbouring
//                 t in the staged line), combines them with the coefficients into
//                 one value per distinct axis-2 factor and pushes each into a
//                 register window of the 2BW+1 output planes it touches; the
//                 oldest plane is complete and stored.
// HBM traffic: (1 + nz) + (nz + 1) tensor passes (nz = 3 for A: 128 B/DOF),
// against 16 for the pass-pair plan (ks_kron_jit.cu).
//
// Factor identity across terms comes from kron_create_impl's deduplication
// (optionally up to sign, see there), so the plan is as small as the term list
// allows. Reference semantics are those of the factorised level plan
// (DESIGN.md 3.4): the same sums in a different association order.
#include "ks_internal.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace ks {

namespace {

constexpr int kMaxZ = 8;

struct K1Out {
    double2* z[kMaxZ];
    int f[kMaxZ];
    int n;
};

// Z_g[r] = sum_k F3_g(r, r + k - BW) x[r + k - BW] along the outermost axis;
// one thread per column (all other axes), a register window of 2BW+1 rows.
// (Loading 4 rows ahead instead of 1 was measured slower at c3: 315 vs 262 us.)
template <int BW>
__global__ void __launch_bounds__(256) k_axis3(const double2* __restrict__ x, const K1Out o,
                                               const double2* __restrict__ rb, int nmax, long long ncols, int n3) {
    constexpr int W = 2 * BW + 1;
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncols) return;
    const double2 Z = make_double2(0.0, 0.0);
    double2 w[W];
#pragma unroll
    for (int k = 0; k < W; ++k) w[k] = Z;
#pragma unroll
    for (int k = 0; k <= BW; ++k)
        if (k < n3) w[BW + k] = __ldg(x + c + (long long)k * ncols);
    for (int r = 0; r < n3; ++r) {
        const int rn = r + BW + 1;
        const double2 nx = rn < n3 ? __ldg(x + c + (long long)rn * ncols) : Z;
        for (int g = 0; g < o.n; ++g) {
            const double2* b = rb + ((size_t)o.f[g] * nmax + r) * W;
            double re = 0.0, im = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const double2 a = __ldg(b + k);
                re = fma(a.x, w[k].x, fma(-a.y, w[k].y, re));
                im = fma(a.x, w[k].y, fma(a.y, w[k].x, im));
            }
            o.z[g][c + (long long)r * ncols] = make_double2(re, im);
        }
#pragma unroll
        for (int k = 0; k < W - 1; ++k) w[k] = w[k + 1];
        w[W - 1] = nx;
    }
}

std::string lit(long long v) { return std::to_string(v); }

} // namespace

struct Kron3 {
    std::vector<int> dims;
    size_t N = 0;
    int bw = 0, nmax = 1;
    std::vector<int> zf;        // axis-3 factor of each input g (-1: x itself)
    std::vector<int> zpool;     // pool index of g (-1: x)
    int npool = 0;
    DevBuf pool;                // npool tensors, allocated on first apply
    cudaKernel_t k2 = nullptr;
    int TX = 0, NT = 0, D = 2;
    size_t smem = 0;
    std::vector<double2> coef;
    int na = 0;                 // staged stage-A products
};

void kron3_free(Kron3* p) { delete p; }

// Build the two-launch plan for four axes (t, 1, 2, 3); null if the shape does
// not fit (the level-pass plan is used instead) or KS_KRON3=0.
Kron3* kron3_build(const std::vector<int>& dims, int bw, int nmax, const std::vector<int>& fclass,
                   const std::vector<double2>& coeffs, const std::vector<std::vector<int>>& fids) {
    // opt-in (KS_KRON3=1): with the rank-merged level plan (ks_kron.cu) the
    // fused pass pairs also move 128 B/DOF and are faster at c3 (0.87 vs 1.02 ms)
    {
        const char* e = std::getenv("KS_KRON3");
        if (!(e && std::strcmp(e, "1") == 0)) return nullptr;
    }
    if (dims.size() != 4 || bw < 1 || bw > 6 || coeffs.empty()) return nullptr;
    const int n0 = dims[0], n1 = dims[1], n2 = dims[2];
    const int T = (int)coeffs.size();
    // factor classes: 1 real, 2 purely imaginary (W + W^H), 0 complex
    auto is_real = [&](int f) { return f >= 0 && fclass[f] == 1; };
    auto is_imag = [&](int f) { return f >= 0 && fclass[f] == 2; };
    auto is_scal = [&](int f) { return is_real(f) || is_imag(f); }; // one double per entry
    std::unique_ptr<Kron3> K(new Kron3());
    K->dims = dims;
    K->N = (size_t)dims[0] * dims[1] * dims[2] * dims[3];
    K->bw = bw;
    K->nmax = nmax;
    // inputs g = distinct axis-3 factors
    std::map<int, int> gid;
    std::vector<int> g_of(T);
    for (int t = 0; t < T; ++t) {
        auto it = gid.find(fids[t][3]);
        if (it == gid.end()) it = gid.emplace(fids[t][3], (int)gid.size()).first;
        g_of[t] = it->second;
    }
    const int nz = (int)gid.size();
    if (nz > kMaxZ) return nullptr;
    K->zf.assign(nz, -1);
    for (auto& kv : gid) K->zf[kv.second] = kv.first;
    K->zpool.assign(nz, -1);
    for (int g = 0; g < nz; ++g)
        if (K->zf[g] >= 0) K->zpool[g] = K->npool++;
    // stage A products (g, F1), stage B products (a, F0), axis-2 classes F2,
    // contributions (b -> h, coefficient summed over merged terms)
    std::map<std::pair<int, int>, int> aid, bid;
    std::map<int, int> hid;
    std::vector<std::pair<int, int>> alist, blist;
    std::vector<int> hlist;
    std::map<std::pair<int, int>, double2> contrib;
    for (int t = 0; t < T; ++t) {
        const auto ka = std::make_pair(g_of[t], fids[t][1]);
        auto ia = aid.find(ka);
        if (ia == aid.end()) {
            ia = aid.emplace(ka, (int)alist.size()).first;
            alist.push_back(ka);
        }
        const auto kb = std::make_pair(ia->second, fids[t][0]);
        auto ib = bid.find(kb);
        if (ib == bid.end()) {
            ib = bid.emplace(kb, (int)blist.size()).first;
            blist.push_back(kb);
        }
        auto ih = hid.find(fids[t][2]);
        if (ih == hid.end()) {
            ih = hid.emplace(fids[t][2], (int)hlist.size()).first;
            hlist.push_back(fids[t][2]);
        }
        auto key = std::make_pair(ib->second, ih->second);
        auto ic = contrib.find(key);
        if (ic == contrib.end()) contrib.emplace(key, coeffs[t]);
        else {
            ic->second.x += coeffs[t].x;
            ic->second.y += coeffs[t].y;
        }
    }
    const int na = (int)alist.size(), nh = (int)hlist.size();
    if (na > 16 || (int)blist.size() > 48 || nh > 8 || contrib.size() > 256) return nullptr;
    // tile: TX axis-1 lines x all t per CTA; ring of D planes of nz inputs
    const int W = 2 * bw + 1, n0p = n0 + 2 * bw;
    std::set<int> f1s, f0s;
    for (auto& a : alist)
        if (a.second >= 0) f1s.insert(a.second);
    for (int j = 0; j < (int)alist.size(); ++j) (void)j;
    {
        std::set<std::pair<int, int>> tmp(blist.begin(), blist.end());
        for (auto& b : tmp)
            if (b.second >= 0) f0s.insert(b.second);
    }
    const std::vector<int> f1l(f1s.begin(), f1s.end()), f0l(f0s.begin(), f0s.end());
    // ring + staged products + factor rows (axis 1: the tile's lines, time: all rows)
    auto smem_of = [&](int tx, int d) {
        return ((size_t)d * nz * (tx + 2 * bw) * n0 + (size_t)na * tx * n0p + f1l.size() * (size_t)tx * W +
                f0l.size() * (size_t)n0 * W) *
               sizeof(double2);
    };
    int TX = std::getenv("KS_KRON3_TX") ? std::atoi(std::getenv("KS_KRON3_TX")) : 0;
    if (TX <= 0) {
        // Two CTAs per SM without register spills (<= 256 threads: 128
        // registers) and a halo overhead (TX + 2BW) / TX <= 2.5 on the ring
        // loads. Measured at c3 (n0 = 65, BW = 2): TX = 3 1.075 ms, 4 1.107,
        // 2 1.167, 6 1.131 (matvec incl. the axis-3 pass). Wider bands (c5,
        // BW = 4) find no such tile and keep the pass-pair plan.
        for (int tx = std::min(8, n1); tx >= 1; --tx)
            if (n0 * tx <= 256 && smem_of(tx, 2) <= 110 * 1024 && 2 * (tx + 2 * bw) <= 5 * tx) {
                TX = tx;
                break;
            }
    }
    if (TX <= 0 || TX > n1 || n0 * TX > 1024 || smem_of(TX, 2) > 220 * 1024) return nullptr;
    const int D = 2;
    const int NT = (n0 * TX + 31) / 32 * 32;
    const int minb = (2 * smem_of(TX, D) <= 220 * 1024 && NT <= 256) ? 2 : 1;
    K->TX = TX;
    K->NT = NT;
    K->D = D;
    K->smem = smem_of(TX, D);
    K->na = na;
    std::vector<std::pair<std::pair<int, int>, double2>> cl(contrib.begin(), contrib.end());
    for (auto& c : cl) K->coef.push_back(c.second);
    const int LN = TX + 2 * bw;

    std::ostringstream s;
    s << "// generated: d=3 matvec, axes t,1,2 fused (ks_kron3.cu)\n"
      << "#define N0 " << n0 << "\n#define N1 " << n1 << "\n#define N2 " << n2 << "\n#define BW " << bw
      << "\n#define W " << W << "\n#define TX " << TX << "\n#define LN " << LN << "\n#define N0P " << n0p
      << "\n#define NZ " << nz << "\n#define NA " << na << "\n#define NT " << NT << "\n#define DR " << D
      << "\n#define NMAX " << nmax << "\n#define NF1 " << f1l.size() << "\n#define NF0 " << f0l.size() << "\n"
      << "struct K3P { double2 c[" << std::max<size_t>(1, cl.size())
      << "]; const double2* z[NZ]; double2* y; const double2* rb; };\n"
      << R"(
__device__ __forceinline__ void cacc(double2& a, const double2 c, const double2 v) {
    a.x = fma(c.x, v.x, fma(-c.y, v.y, a.x));
    a.y = fma(c.x, v.y, fma(c.y, v.x, a.y));
}
__device__ __forceinline__ void cp16(void* sdst, const void* g, bool v) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(g), "r"(v ? 16 : 0));
}
extern "C" __global__ void __launch_bounds__(NT, )"
      << minb << R"()
ks_k3(const K3P P) {
    extern __shared__ __align__(16) double2 sm[];
    double2* ring = sm;                        // [DR][NZ][LN][N0]
    double2* sp = sm + DR * NZ * LN * N0;      // [NA][TX][N0P], t halos zero
    double2* fa = sp + NA * TX * N0P;          // [NF1][TX][W] axis-1 factor rows of the tile's lines
    double2* ft = fa + NF1 * TX * W;           // [NF0][N0][W] time factor rows
    const int tid = threadIdx.x;
    const int t = tid % N0, l = tid / N0;
    const bool act = l < TX;
    const int x0 = blockIdx.x * TX, i3 = blockIdx.y;
    const int i1 = x0 + l;
    const bool valid = act && i1 < N1;
    const double2 Z = make_double2(0.0, 0.0);
    const long long plane = (long long)N0 * N1, vol = plane * N2;
    for (int e = tid; e < NA * TX * N0P; e += NT) sp[e] = Z;
    // per-thread bases: ring (line l, time t), staged products, output
    const double2* ringt = ring + l * N0 + t;
    double2* spt = sp + l * N0P + t;
    const double2* fat = fa + l * W;
    const double2* ftt = ft + t;
    double2* yt = P.y + (long long)i3 * vol + (long long)i1 * N0 + t;
    // ring rows [lo, hi) of a plane exist (halo lines past the tensor ends are zero)
    const int lo = (x0 - BW < 0 ? BW - x0 : 0) * N0;
    const int hi = (x0 + TX + BW > N1 ? N1 - x0 + BW : LN) * N0;
    auto issue = [&](int ib) {
        if (ib < N2) {
            double2* slot = ring + (ib % DR) * (NZ * LN * N0);
            const long long pb = (long long)i3 * vol + (long long)ib * plane + (long long)(x0 - BW) * N0;
#pragma unroll
            for (int g = 0; g < NZ; ++g) {
                const double2* src = P.z[g] + pb;
                for (int rem = tid; rem < LN * N0; rem += NT) {
                    const bool ok = rem >= lo && rem < hi;
                    cp16(slot + g * (LN * N0) + rem, ok ? (const void*)(src + rem) : (const void*)P.z[0], ok);
                }
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
)";
    // factor rows in shared memory: axis 1 (the tile's lines; zero past the end) and time
    for (size_t j = 0; j < f1l.size(); ++j)
        s << "    for (int e = tid; e < TX * W; e += NT) { const int r = x0 + e / W; fa[" << j
          << " * TX * W + e] = r < N1 ? P.rb[((long long)" << f1l[j] << " * NMAX + r) * W + e % W] : Z; }\n";
    // time factors: real rows in registers (each lane has its own row t), complex
    // rows in shared memory, k-major so that a warp's lanes read consecutive t
    for (size_t j = 0; j < f0l.size(); ++j) {
        if (is_scal(f0l[j]))
            s << "    double R0_" << j << "[W];\n#pragma unroll\n    for (int k = 0; k < W; ++k) R0_" << j
              << "[k] = act ? P.rb[((long long)" << f0l[j] << " * NMAX + t) * W + k]." << (is_imag(f0l[j]) ? "y" : "x")
              << " : 0.0;\n";
        else
            s << "    for (int e = tid; e < N0 * W; e += NT) { const int tt = e / W, k = e - tt * W; ft[" << j
              << " * N0 * W + k * N0 + tt] = P.rb[(long long)" << f0l[j] << " * NMAX * W + e]; }\n";
    }
    s << "    double2 acc[W];\n#pragma unroll\n    for (int k = 0; k < W; ++k) acc[k] = Z;\n"
      << "    __syncthreads();\n    for (int k = 0; k < DR - 1; ++k) issue(k);\n"
      << "    for (int base = 0; base < N2 + BW; base += W) {\n";
    // out = sum_k F[k] taps[k] with F the thread's row of factor f in table
    // `tab` (identity: the centre tap)
    auto prod = [&](const std::string& out, int f, const std::string& taps, bool axis1) {
        if (f < 0) {
            s << "                const double2 " << out << " = " << taps << "[BW];\n";
            return;
        }
        const std::vector<int>& fl = axis1 ? f1l : f0l;
        const int j = (int)(std::find(fl.begin(), fl.end(), f) - fl.begin());
        // two partial sums (even / odd taps) per component: shorter dependent
        // DFMA chains
        std::string fk;
        const char* comp = is_real(f) ? ".x" : (is_imag(f) ? ".y" : "");
        if (!axis1 && is_scal(f)) fk = "R0_" + lit(j) + "[K]";
        else if (axis1) fk = std::string("fat[") + lit(j) + " * TX * W + K]" + comp;
        else fk = std::string("ftt[") + lit(j) + " * N0 * W + K * N0]" + comp;
        auto F = [&](int k) {
            std::string r = fk;
            const size_t pos = r.find('K');
            r.replace(pos, 1, lit(k));
            if (r.find('K') != std::string::npos) r.replace(r.find('K'), 1, lit(k));
            return r;
        };
        s << "                double2 " << out << ";\n                {\n";
        for (int par = 0; par < 2; ++par) {
            s << "                  double2 q" << par << " = Z;\n";
            for (int k = par; k < W; k += 2) {
                const std::string tk = taps + "[" + lit(k) + "]";
                if (is_real(f))
                    s << "                  q" << par << ".x = fma(" << F(k) << ", " << tk << ".x, q" << par << ".x); q" << par
                      << ".y = fma(" << F(k) << ", " << tk << ".y, q" << par << ".y);\n";
                else if (is_imag(f)) // (i w)(a + i b) = -w b + i w a
                    s << "                  q" << par << ".x = fma(-" << F(k) << ", " << tk << ".y, q" << par << ".x); q" << par
                      << ".y = fma(" << F(k) << ", " << tk << ".x, q" << par << ".y);\n";
                else
                    s << "                  cacc(q" << par << ", " << F(k) << ", " << tk << ");\n";
            }
        }
        s << "                  " << out << " = make_double2(q0.x + q1.x, q0.y + q1.y);\n                }\n";
    };
    for (int u = 0; u < W; ++u) {
        s << "    {\n        const int ib = base + " << u << ";\n        if (ib < N2 + BW) {\n"
          << "          if (ib < N2) {\n"
          << "            if (DR == 2) asm volatile(\"cp.async.wait_group 0;\\n\" ::);\n"
          << "            else asm volatile(\"cp.async.wait_group 1;\\n\" ::);\n"
          << "            __syncthreads();\n            issue(ib + DR - 1);\n"
          << "            const double2* sl = ringt + (ib % DR) * (NZ * LN * N0);\n"
          << "            if (act) {\n";
        // stage A
        for (int g = 0; g < nz; ++g) {
            std::vector<int> ks;
            for (int a = 0; a < na; ++a)
                if (alist[a].first == g) ks.push_back(a);
            if (ks.empty()) continue;
            s << "              {\n                double2 a[W];\n#pragma unroll\n                for (int k = 0; k < W; ++k) a[k] = sl[("
              << g << " * LN + k) * N0];\n";
            for (int a : ks) {
                prod("pa" + lit(a), alist[a].second, "a", true);
                s << "                spt[" << a << " * TX * N0P + BW] = pa" << a << ";\n";
            }
            s << "              }\n";
        }
        s << "            }\n            __syncthreads();\n            if (act) {\n";
        for (int h = 0; h < nh; ++h) s << "              double2 wh" << h << " = Z;\n";
        // stage B
        for (int a = 0; a < na; ++a) {
            std::vector<int> js;
            for (int j = 0; j < (int)blist.size(); ++j)
                if (blist[j].first == a) js.push_back(j);
            if (js.empty()) continue;
            s << "              {\n                double2 b[W];\n#pragma unroll\n                for (int k = 0; k < W; ++k) b[k] = spt["
              << a << " * TX * N0P + k];\n";
            for (int j : js) {
                prod("pb" + lit(j), blist[j].second, "b", false);
                for (size_t ci = 0; ci < cl.size(); ++ci)
                    if (cl[ci].first.first == j) {
                        const double2 c = cl[ci].second;
                        const std::string wh = "wh" + lit(cl[ci].first.second), pb = "pb" + lit(j);
                        if (c.y == 0.0 && c.x == 1.0)
                            s << "                " << wh << ".x += " << pb << ".x; " << wh << ".y += " << pb << ".y;\n";
                        else if (c.y == 0.0)
                            s << "                " << wh << ".x = fma(P.c[" << ci << "].x, " << pb << ".x, " << wh
                              << ".x); " << wh << ".y = fma(P.c[" << ci << "].x, " << pb << ".y, " << wh << ".y);\n";
                        else
                            s << "                cacc(" << wh << ", P.c[" << ci << "], " << pb << ");\n";
                    }
            }
            s << "              }\n";
        }
        // push into the output window: plane r = ib + dl gets F2(r, ib) * wh
        for (int h = 0; h < nh; ++h) {
            const int f = hlist[h];
            if (f < 0) {
                s << "              acc[" << u << "].x += wh" << h << ".x; acc[" << u << "].y += wh" << h << ".y;\n";
                continue;
            }
            // column ib of F2: F2(ib + dl, ib) at cfh[dl * (W - 1)], rows outside the axis are zero
            s << "              { const double2* cfh = P.rb + ((long long)" << f << " * NMAX + ib) * W + BW;\n";
            for (int dl = -bw; dl <= bw; ++dl) {
                const int slot = ((u + dl) % W + W) % W;
                s << "                { const double2 cf = (ib + (" << dl << ") >= 0 && ib + (" << dl
                  << ") < N2) ? cfh[" << dl * (2 * bw) << "] : Z; ";
                if (is_real(f))
                    s << "acc[" << slot << "].x = fma(cf.x, wh" << h << ".x, acc[" << slot << "].x); acc[" << slot
                      << "].y = fma(cf.x, wh" << h << ".y, acc[" << slot << "].y); }\n";
                else if (is_imag(f))
                    s << "acc[" << slot << "].x = fma(-cf.y, wh" << h << ".y, acc[" << slot << "].x); acc[" << slot
                      << "].y = fma(cf.y, wh" << h << ".x, acc[" << slot << "].y); }\n";
                else
                    s << "cacc(acc[" << slot << "], cf, wh" << h << "); }\n";
            }
            s << "              }\n";
        }
        const int os = ((u - bw) % W + W) % W;
        s << "            }\n          }\n"
          << "          const int rd = ib - BW;\n"
          << "          if (rd >= 0) {\n"
          << "            if (valid) yt[(long long)rd * plane] = acc[" << os
          << "];\n            acc[" << os << "] = Z;\n          }\n        }\n    }\n";
    }
    s << "    }\n    asm volatile(\"cp.async.wait_group 0;\\n\" ::);\n}\n";
    if (const char* dump = std::getenv("KS_KRON3_DUMP"))
        if (FILE* f = std::fopen(dump, "w")) {
            std::fputs(s.str().c_str(), f);
            std::fclose(f);
        }
    K->k2 = nvrtc_kernel(s.str(), "ks_k3", 220 * 1024);
    return K.release();
}

void kron3_apply(Kron3& K, const double2* x, double2* y, const double2* rb, cudaStream_t st) {
    const int n0 = K.dims[0], n1 = K.dims[1], n2 = K.dims[2], n3 = K.dims[3];
    if (K.npool > 0 && !K.pool.p) K.pool.alloc((size_t)K.npool * K.N * sizeof(double2));
    const int nz = (int)K.zf.size();
    std::vector<const double2*> zp(nz);
    K1Out o{};
    o.n = 0;
    for (int g = 0; g < nz; ++g) {
        if (K.zpool[g] < 0) {
            zp[g] = x;
            continue;
        }
        double2* z = K.pool.as<double2>() + (size_t)K.zpool[g] * K.N;
        zp[g] = z;
        o.z[o.n] = z;
        o.f[o.n] = K.zf[g];
        ++o.n;
    }
    if (o.n > 0) {
        const long long ncols = (long long)n0 * n1 * n2;
        const unsigned g1 = (unsigned)((ncols + 255) / 256);
        switch (K.bw) {
#define KS_A3(B)                                                                                   \
    case B:                                                                                        \
        k_axis3<B><<<g1, 256, 0, st>>>(x, o, rb, K.nmax, ncols, n3);                               \
        break;
            KS_A3(1) KS_A3(2) KS_A3(3) KS_A3(4) KS_A3(5) KS_A3(6)
#undef KS_A3
        }
        check_launch("k_axis3");
    }
    // by-value parameter (constant bank): coefficients, z pointers, y, rb
    const size_t nc = std::max<size_t>(1, K.coef.size());
    std::vector<double2> prm(nc + (sizeof(void*) * (nz + 2) + 15) / 16, make_double2(0.0, 0.0));
    std::copy(K.coef.begin(), K.coef.end(), prm.begin());
    char* p = reinterpret_cast<char*>(prm.data() + nc);
    std::memcpy(p, zp.data(), sizeof(void*) * nz);
    std::memcpy(p + sizeof(void*) * nz, &y, sizeof(void*));
    std::memcpy(p + sizeof(void*) * (nz + 1), &rb, sizeof(void*));
    void* args[] = {prm.data()};
    const dim3 grid((unsigned)((n1 + K.TX - 1) / K.TX), (unsigned)n3);
    KS_CUDA(cudaLaunchKernel((const void*)K.k2, grid, dim3(K.NT), args, K.smem, st));
    check_launch("ks_k3");
}

} // namespace ks
