// Plan-specialised fused level passes for the Kronecker-sum matvec, compiled
// at plan creation with NVRTC for sm_100a.
//
// The generic fused-pair kernels (ks_kron_pair.cu) interpret the level plan at
// run time -- contribution lists, factor indices and coefficients are loaded
// and dispatched per element -- and ncu shows them instruction bound (about
// 2,250 instructions per DOF at c3, with the HBM traffic already at its
// algorithmic minimum). Here the same sweep is emitted as straight-line CUDA
// for one plan: node and factor indices become literals, each distinct 1-D
// factor row is loaded once per row (axis a: once per kernel, the row is the
// thread's own; axis b: once per plane, uniform across the CTA), products that
// share an input and a factor are formed once, and the contribution
// coefficients live in a by-value kernel parameter (constant bank), so the
// source depends only on the plan's topology and is cached process-wide.
//
// Generated kernel ("pull" variant, axis b applied from a window of the last
// 2BW+1 middle planes; "push" variant scatters each middle plane into a window
// of output rows -- whichever keeps fewer values in registers):
//
//   plane ib: cp.async ring of the input level's plane ib (all inputs, one 16 B
//   element per thread) -> middle values of the thread's point (axis a, taps
//   from neighbouring threads' smem) -> output row ib-BW (axis b) -> store.
//
// Reference semantics: KroneckerOperator::apply (tensorops.cpp:236-254) as
// factorised by the level plan.
#include "ks_internal.hpp"

#include <cuda.h>
#include <nvrtc.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace ks {

namespace {
std::mutex g_jit_mu;
std::map<std::string, cudaKernel_t>& jit_cache() {
    static std::map<std::string, cudaKernel_t> m;
    return m;
}
} // namespace

#define KS_NVRTC(x)                                                                                \
    do {                                                                                           \
        nvrtcResult r_ = (x);                                                                      \
        KS_REQUIRE(r_ == NVRTC_SUCCESS, KS_ECUDA, std::string("nvrtc: ") + nvrtcGetErrorString(r_)); \
    } while (0)

// Compile `src` for sm_100a with NVRTC (cached process-wide by source text) and
// return kernel `name`, with its dynamic shared memory limit raised to max_smem.
cudaKernel_t nvrtc_kernel(const std::string& src, const char* name, size_t max_smem) {
    std::lock_guard<std::mutex> lk(g_jit_mu);
    // KS_KRON_JIT=dump=<dir>: the generated sources, for offline inspection (cuobjdump -sass);
    // written before any device call, so a GPU-less host can generate and compile them
    if (const char* e = std::getenv("KS_KRON_JIT"))
        if (!std::strncmp(e, "dump=", 5)) {
            const std::string fn = std::string(e + 5) + "/ks_jit_" + name + "_" + std::to_string(std::hash<std::string>{}(src) % 100000) + ".cu";
            if (FILE* f = std::fopen(fn.c_str(), "w")) {
                std::fwrite(src.data(), 1, src.size(), f);
                std::fclose(f);
            }
        }
    int dev0 = 0;
    KS_CUDA(cudaGetDevice(&dev0));
    // per device: the shared-memory opt-in below is a per-device attribute
    const std::string key = std::to_string(dev0) + ":" + name + "\n" + src;
    auto it = jit_cache().find(key);
    if (it != jit_cache().end()) return it->second;
    nvrtcProgram prog;
    KS_NVRTC(nvrtcCreateProgram(&prog, src.c_str(), "ks_kron_jit.cu", 0, nullptr, nullptr));
    const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "-default-device"};
    const nvrtcResult rc = nvrtcCompileProgram(prog, 4, opts);
    if (rc != NVRTC_SUCCESS) {
        size_t n = 0;
        nvrtcGetProgramLogSize(prog, &n);
        std::string log(n, '\0');
        nvrtcGetProgramLog(prog, &log[0]);
        nvrtcDestroyProgram(&prog);
        throw Error(KS_ECUDA, "nvrtc compile failed: " + log.substr(0, 2000));
    }
    size_t cn = 0;
    KS_NVRTC(nvrtcGetCUBINSize(prog, &cn));
    std::vector<char> cubin(cn);
    KS_NVRTC(nvrtcGetCUBIN(prog, cubin.data()));
    nvrtcDestroyProgram(&prog);
    cudaLibrary_t lib = nullptr;
    cudaKernel_t fn = nullptr;
    KS_CUDA(cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    KS_CUDA(cudaLibraryGetKernel(&fn, lib, name));
    int dev = 0;
    KS_CUDA(cudaGetDevice(&dev));
    KS_CUDA(cudaKernelSetAttributeForDevice(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem, dev));
    jit_cache()[key] = fn;
    return fn;
}

namespace {


struct JitKernel {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t fn = nullptr;
};

JitKernel jit_compile(const std::string& src) {
    JitKernel k;
    k.fn = nvrtc_kernel(src, "ks_pair", 200 * 1024);
    return k;
}

std::string lit(int v) { return std::to_string(v); }

} // namespace

struct KronJitPair {
    JitKernel k;
    int nin = 0, nmid = 0, nout = 0, bw = 0, ncoef = 0;
    bool pull = true;
    bool blocked = false; // tensor-map fed variants (kron_jitb_build / kron_jitt_build)
    bool tile = false;    // tile variant (s_a = 1): two phases over shared memory
    std::string tag;      // shape, for the candidate log
    int T = 0, nq = 1, no = 1, D = 2, pad = 0; // block size, point block, ring depth, ring halo
    size_t smem = 0;                           // ring + staged axis-b bands
    long long s_a = 0, n_outer = 0;
    int n_a = 0, n_b = 0;
    unsigned grid = 0;
    std::vector<double2> coef;
};

void kron_jit_free(KronJitPair* p) { delete p; }

// Build (or fetch from the cache) the specialised kernel for passes a (in ->
// mid) and b (mid -> out). coeffs: the coefficient of every contribution, in
// the order a then b (indices in JitContrib::coeff).
KronJitPair* kron_jit_build(int nin, int nmid, int nout, int bw, const std::vector<JitContrib>& a,
                            const std::vector<JitContrib>& b, const std::vector<int>& freal,
                            const std::vector<double2>& coeffs, long long s_a, int n_a, int n_b, long long n_outer,
                            int tmax_default, int dmax) {
    if (const char* e = std::getenv("KS_KRON_JIT"))
        if (std::strcmp(e, "0") == 0) return nullptr;
    if (nin < 1 || nmid < 1 || nout < 1 || bw < 1 || bw > 6 || nin > 16 || nmid > 16 || nout > 16) return nullptr;
    if (coeffs.size() > 1000) return nullptr; // by-value parameter <= 16 KB
    if (n_a > 384 || n_b < 1) return nullptr;
    const int W = 2 * bw + 1;
    const bool pull = nmid <= nout;
    // point block: c lines of n_a points (c inner columns when the axis-a stride
    // s_a > 1, so a warp moves >= 32 B segments; else c outer columns), block
    // size rounded to whole warps; pick the fullest block of at most 384 threads
    int c_best = 1, T_best = 0;
    double e_best = -1;
    const int tmax = tmax_default;
    for (int c = 1; c * n_a <= tmax; ++c) {
        if (s_a > 1 && c > s_a) break;
        if (s_a == 1 && c > n_outer) break;
        const int T = (c * n_a + 31) / 32 * 32;
        const double e = (double)(c * n_a) / T - (s_a > 1 && c == 1 ? 0.2 : 0.0);
        // fullest block; among equally full ones the largest up to 256 threads
        if (e > e_best + 1e-9 || (e > e_best - 1e-9 && T <= 256)) {
            e_best = e;
            c_best = c;
            T_best = T;
        }
    }
    if (T_best == 0) return nullptr; // a line longer than the block limit: per-pass kernels
    const int T = T_best;
    const int nq = s_a > 1 ? c_best : 1, no = s_a > 1 ? 1 : c_best;
    const long long nqb = (s_a + nq - 1) / nq, nob = (n_outer + no - 1) / no;
    const int pad = bw * nq;
    const int RS = T + 2 * pad; // ring row: halo | T points | halo
    // ring depth: planes in flight per CTA (deeper rings, D = 6..10, measured
    // slower: the passes are issue / latency bound, not short of bytes in flight)
    int D = dmax;
    auto smem = [&](int d) { return (size_t)d * nin * RS * sizeof(double2); };
    while (D > 2 && smem(D) > 110 * 1024) --D;
    if (smem(D) > 200 * 1024) return nullptr;
    // no register cap: capping at 128 (2 blocks/SM) spills and is slower at c3
    // (1.98 vs 1.67 ms)
    const int minb = 1;
    const int minb_env = 0;
    // factor classes (freal): 1 real, 2 purely imaginary (one double per entry), 0 complex
    auto is_real = [&](int f) { return f >= 0 && freal[f] == 1; };
    auto is_imag = [&](int f) { return f >= 0 && freal[f] == 2; };
    auto is_scal = [&](int f) { return is_real(f) || is_imag(f); };
    auto comp = [&](int f) -> std::string { return is_real(f) ? ".x" : (is_imag(f) ? ".y" : ""); };
    // v += F * w for one tap, F of class f held as `fv` (double for real / imaginary)
    auto mac = [&](int f, const std::string& v, const std::string& fv, const std::string& w) -> std::string {
        if (is_real(f))
            return " " + v + ".x = fma(" + fv + ", " + w + ".x, " + v + ".x); " + v + ".y = fma(" + fv + ", " + w + ".y, " + v +
                   ".y);";
        if (is_imag(f))
            return " " + v + ".x = fma(-" + fv + ", " + w + ".y, " + v + ".x); " + v + ".y = fma(" + fv + ", " + w + ".x, " + v +
                   ".y);";
        return " cacc(" + v + ", " + fv + ", " + w + ");";
    };
    // acc += c * v with the contribution coefficient (real coefficients: 2 DFMA).
    // Unit coefficients (exactly +-1, the common case: nu = 1 and the plan's
    // merged rows) become a copy / an add, and the first contribution into a
    // still-zero accumulator a plain assignment -- bit-identical (1*v = v,
    // 0 + v = v) and up to 2 DFMA less per contribution (KS_KRON_JIT_UNIT=0 off).
    const bool unit_ok = true;
    std::set<std::string> live; // accumulators already holding a contribution
    auto cmac = [&](const std::string& acc, int ci, const std::string& v) -> std::string {
        const bool fresh = live.insert(acc).second;
        if (unit_ok && coeffs[ci].y == 0.0 && (coeffs[ci].x == 1.0 || coeffs[ci].x == -1.0)) {
            const bool neg = coeffs[ci].x == -1.0;
            if (fresh) return acc + ".x = " + (neg ? "-" : "") + v + ".x; " + acc + ".y = " + (neg ? "-" : "") + v + ".y;";
            return acc + ".x " + (neg ? "-" : "+") + "= " + v + ".x; " + acc + ".y " + (neg ? "-" : "+") + "= " + v + ".y;";
        }
        if (coeffs[ci].y == 0.0)
            return acc + ".x = fma(P.c[" + lit(ci) + "].x, " + v + ".x, " + acc + ".x); " + acc + ".y = fma(P.c[" + lit(ci) +
                   "].x, " + v + ".y, " + acc + ".y);";
        return "cacc(" + acc + ", P.c[" + lit(ci) + "], " + v + ");";
    };
    // axis-b factor bands staged in shared memory once per CTA (they are read
    // every plane, uniformly across the CTA)
    std::vector<int> fbl;
    {
        std::set<int> t;
        for (auto& c : b)
            if (c.factor >= 0) t.insert(c.factor);
        fbl.assign(t.begin(), t.end());
    }
    const size_t bstage = fbl.size() * (size_t)n_b * W * sizeof(double2);
    const bool stage = smem(D) + bstage <= 200 * 1024;
    size_t nfa = 0;
    {
        std::set<int> t;
        for (auto& c : a)
            if (c.factor >= 0) t.insert(c.factor);
        nfa = t.size();
    }
    const size_t astage = nfa * (size_t)n_a * W * sizeof(double2);
    const bool asm_rows = false; // axis-a rows from shared memory: measured slower, generator kept off
    (void)astage;
    auto bidx = [&](int f) { return (int)(std::find(fbl.begin(), fbl.end(), f) - fbl.begin()); };
    std::ostringstream s;
    s << "// generated: fused level passes (ks_kron_jit.cu)\n"
      << "#define BW " << bw << "\n#define W " << W << "\n#define NIN " << nin << "\n#define T " << T
      << "\n#define RS " << RS << "\n#define PAD " << pad << "\n"
      // the plan's geometry as literals: the sweep's ring index, plane strides and
      // output offsets become constant arithmetic (the run-time values are only
      // kept in the signature; ncu showed IMAD / I2F division sequences per plane)
      << "#define s_a " << s_a << "LL\n#define n_a " << n_a << "\n#define n_b " << n_b << "\n#define n_outer " << n_outer
      << "LL\n#define nq " << nq << "\n#define no " << no << "\n#define D " << D << "\n"
      << "struct Coef { double2 c[" << std::max<size_t>(1, coeffs.size()) << "]; const double2* in[" << nin
      << "]; double2* out[" << nout << "]; };\n"
      << R"(
__device__ __forceinline__ void cacc(double2& a, const double2 c, const double2 v) {
    a.x = fma(c.x, v.x, fma(-c.y, v.y, a.x));
    a.y = fma(c.x, v.y, fma(c.y, v.x, a.y));
}
__device__ __forceinline__ void cp16(void* sdst, const void* g, bool v) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(g), "r"(v ? 16 : 0));
}
extern "C" __global__ void __launch_bounds__(T, )" << (minb_env > 0 ? minb_env : minb) << R"()
ks_pair(const double2* const* __restrict__ ip, double2* const* __restrict__ op, const double2* __restrict__ rb,
        int nmax, long long s_a_rt, int n_a_rt, int n_b_rt, long long n_outer_rt, int nq_rt, int no_rt, int D_rt,
        const Coef P) {
    extern __shared__ __align__(16) double2 ring[]; // [D][NIN][RS]: halo | T points | halo
    const int tid = threadIdx.x;
    const long long nqb = (s_a + nq - 1) / nq;
    const long long q0 = (blockIdx.x % nqb) * nq, o0 = (blockIdx.x / nqb) * no;
    const int qq = tid % nq, rest = tid / nq;
    const int ia = rest % n_a, oo = rest / n_a;
    const bool valid = oo < no && q0 + qq < s_a && o0 + oo < n_outer;
    const long long s_b = s_a * n_a;
    const long long base = valid ? (q0 + qq) + s_a * ia + s_b * (long long)n_b * (o0 + oo) : 0;
    const double2 Z = make_double2(0.0, 0.0);
    // halos (and whole rings) zero: out-of-range taps meet zero band entries
    for (int e = tid; e < D * NIN * RS; e += T) ring[e] = Z;
)";
    if (stage) {
        s << "    double2* bsm = ring + D * NIN * RS; // [factor][row][W] axis-b bands\n";
        for (size_t j = 0; j < fbl.size(); ++j)
            s << "    for (int e = tid; e < n_b * W; e += T) bsm[" << j << " * n_b * W + e] = rb[(unsigned long long)"
              << fbl[j] << " * nmax * W + e];\n";
    }
    if (asm_rows) {
        std::set<int> fa0;
        for (auto& c : a)
            if (c.factor >= 0) fa0.insert(c.factor);
        int j = 0;
        s << "    { double2* ar = ring + D * NIN * RS + " << (stage ? fbl.size() : 0) << " * n_b * W;\n";
        for (int f : fa0)
            s << "      for (int e = tid; e < n_a * W; e += T) ar[" << j++ << " * n_a * W + e] = rb[(unsigned long long)" << f
              << " * nmax * W + e];\n";
        s << "    }\n";
    }
    s << R"(    __syncthreads();
    auto issue = [&](int ib) {
        if (ib < n_b) {
            double2* slot = ring + (ib % D) * (NIN * RS) + PAD + tid;
            const long long off = base + s_b * ib;
#pragma unroll
            for (int g = 0; g < NIN; ++g)
                cp16(slot + g * RS, valid ? (const void*)(P.in[g] + off) : (const void*)P.in[0], valid);
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    for (int k = 0; k < D - 1; ++k) issue(k);
)";
    // axis-a factor rows (the thread's own row ia, constant over the sweep):
    // registers, or (asm_rows) shared memory [factor][row][W]
    std::set<int> fa;
    for (auto& c : a)
        if (c.factor >= 0) fa.insert(c.factor);
    std::vector<int> fal(fa.begin(), fa.end());
    auto aref = [&](int f, const char* k) -> std::string {
        if (!asm_rows) return "A" + lit(f) + "[" + k + "]";
        const int j = (int)(std::find(fal.begin(), fal.end(), f) - fal.begin());
        return std::string("asmr[(") + lit(j) + " * n_a + ia) * W + " + k + "]" + comp(f);
    };
    if (asm_rows) {
        s << "    const double2* asmr = ring + D * NIN * RS + " << (stage ? fbl.size() : 0) << " * n_b * W;\n";
    } else {
        for (int f : fa) {
            if (is_scal(f))
                s << "    double A" << f << "[W];\n";
            else
                s << "    double2 A" << f << "[W];\n";
            s << "#pragma unroll\n    for (int k = 0; k < W; ++k) { const double2 t = valid ? rb[((unsigned long long)" << f
              << " * nmax + ia) * W + k] : Z; A" << f << "[k] = t" << comp(f) << "; }\n";
        }
    }
    const int nwin = pull ? nmid : nout;
    // Rotating windows (default; KS_KRON_JIT_ROT=0 shifts them): the sweep is
    // unrolled by W planes, so window position j of plane ib lives in the static
    // register slot (ib + 1 + j) % W (pull) / (ib + j) % W (push) instead of
    // being shifted every plane -- ncu showed the shifts as ~20% of the pass-1
    // instructions (IMAD.MOV).
    const bool rot = true;
    auto WP = [&](const std::string& j) { return rot ? "(ph + 1 + (" + j + ")) % W" : j; };
    // products sharing a tap loop emitted as one loop (independent FMA chains
    // interleaved in the source; KS_KRON_JIT_ILV=0 one loop per product):
    // c5 18.9 -> 18.3 ms, c3 unchanged
    const bool ilv = true;
    auto WQ = [&](const std::string& j) { return rot ? "(ph + (" + j + ")) % W" : j; };
    s << "    double2 win[" << nwin << "][W];\n"
      << "#pragma unroll\n    for (int h = 0; h < " << nwin << "; ++h)\n#pragma unroll\n        for (int j = 0; j < W; ++j) win[h][j] = Z;\n";
    if (rot)
        s << "    for (int ib0 = 0; ib0 < n_b + BW; ib0 += W) {\n#pragma unroll\n    for (int ph = 0; ph < W; ++ph) {\n"
          << "        const int ib = ib0 + ph;\n        if (ib >= n_b + BW) break;\n";
    else
        s << "    for (int ib = 0; ib < n_b + BW; ++ib) {\n";
    if (pull && !rot)
        s << "#pragma unroll\n        for (int h = 0; h < " << nmid
          << "; ++h)\n#pragma unroll\n            for (int j = 0; j < W - 1; ++j) win[h][j] = win[h][j + 1];\n";
    s << "        if (ib < n_b) {\n"
      << "            asm volatile(\"cp.async.wait_group " << (D - 2) << ";\\n\" ::);\n"
      << "            __syncthreads();\n            issue(ib + D - 1);\n"
      << "            const double2* sl = ring + (ib % D) * (NIN * RS) + PAD + tid;\n";
    for (int h = 0; h < nmid; ++h) s << "            double2 m" << h << " = Z;\n";
    live.clear();
    // axis a: per input g, taps once, per distinct factor one product, then the coefficients
    for (int g = 0; g < nin; ++g) {
        std::vector<const JitContrib*> cs;
        for (auto& c : a)
            if (c.in == g) cs.push_back(&c);
        if (cs.empty()) continue;
        s << "            {\n                double2 w[W];\n"
          << "#pragma unroll\n                for (int k = 0; k < W; ++k) w[k] = sl[" << g << " * RS + (k - BW) * nq];\n";
        std::set<int> fs;
        for (auto* c : cs) fs.insert(c->factor);
        if (ilv) { // all products of this input in one tap loop: independent FMA chains interleaved
            for (int f : fs)
                if (f >= 0) s << "                double2 v" << f << " = Z;\n";
            s << "#pragma unroll\n                for (int k = 0; k < W; ++k) {";
            for (int f : fs)
                if (f >= 0) s << mac(f, "v" + lit(f), aref(f, "k"), "w[k]");
            s << " }\n";
        }
        for (int f : fs) {
            const std::string v = f < 0 ? "vI" : "v" + lit(f);
            if (f < 0) {
                s << "                const double2 vI = w[BW];\n";
            } else if (!ilv) {
                s << "                double2 " << v << " = Z;\n#pragma unroll\n                for (int k = 0; k < W; ++k) {"
                  << mac(f, v, aref(f, "k"), "w[k]") << " }\n";
            }
            for (auto* c : cs)
                if (c->factor == f) s << "                " << cmac("m" + lit(c->out), c->coeff, v) << "\n";
        }
        s << "            }\n";
    }
    std::set<int> fb;
    for (auto& c : b)
        if (c.factor >= 0) fb.insert(c.factor);
    if (pull) {
        const std::string newest = rot ? "ph" : "W - 1";
        for (int h = 0; h < nmid; ++h) s << "            win[" << h << "][" << newest << "] = m" << h << ";\n";
        s << "        } else {\n";
        for (int h = 0; h < nmid; ++h) s << "            win[" << h << "][" << newest << "] = Z;\n";
        s << "        }\n        const int rd = ib - BW;\n        if (rd < 0) continue;\n";
        // axis-b rows at row rd (uniform across the CTA)
        for (int f : fb) {
            s << "        " << (is_scal(f) ? "double" : "double2") << " B" << f << "[W];\n"
              << "#pragma unroll\n        for (int j = 0; j < W; ++j) { const double2 t = "
              << (stage ? "bsm[(" + lit(bidx(f)) + " * n_b + rd) * W + j]"
                        : "rb[((unsigned long long)" + lit(f) + " * nmax + rd) * W + j]")
              << "; B" << f << "[j] = t" << comp(f) << "; }\n";
        }
        // distinct (h, f) products, then outputs
        std::set<std::pair<int, int>> hf;
        for (auto& c : b) hf.insert({c.in, c.factor});
        if (ilv) { // one tap loop over all (h, f) products
            for (auto& pr : hf)
                if (pr.second >= 0) s << "        double2 d" << pr.first << "_" << pr.second << " = Z;\n";
            s << "#pragma unroll\n        for (int j = 0; j < W; ++j) {";
            for (auto& pr : hf)
                if (pr.second >= 0)
                    s << mac(pr.second, "d" + lit(pr.first) + "_" + lit(pr.second), "B" + lit(pr.second) + "[j]",
                             "win[" + lit(pr.first) + "][" + WP("j") + "]");
            s << " }\n";
        }
        for (auto& pr : hf) {
            const int h = pr.first, f = pr.second;
            const std::string v = "d" + lit(h) + "_" + (f < 0 ? std::string("I") : lit(f));
            if (f < 0) {
                s << "        const double2 " << v << " = win[" << h << "][" << WP("BW") << "];\n";
            } else if (!ilv) {
                s << "        double2 " << v << " = Z;\n#pragma unroll\n        for (int j = 0; j < W; ++j) {"
                  << mac(f, v, "B" + lit(f) + "[j]", "win[" + lit(h) + "][" + WP("j") + "]") << " }\n";
            }
        }
        for (int o = 0; o < nout; ++o) {
            s << "        { double2 acc = Z;\n";
            live.erase("acc");
            for (auto& c : b)
                if (c.out == o)
                    s << "          " << cmac("acc", c.coeff, "d" + lit(c.in) + "_" + (c.factor < 0 ? std::string("I") : lit(c.factor)))
                      << "\n";
            s << "          if (valid) P.out[" << o << "][base + s_b * rd] = acc; }\n";
        }
        s << (rot ? "    }\n    }\n" : "    }\n");
    } else {
        // push: column ib of each axis-b factor, F(ib + j - BW, ib), uniform
        for (int f : fb) {
            s << "            " << (is_scal(f) ? "double" : "double2") << " C" << f << "[W];\n"
              << "#pragma unroll\n            for (int j = 0; j < W; ++j) { const int r = ib + j - BW; const double2 t = (r >= 0 && r < n_b) ? "
              << (stage ? "bsm[(" + lit(bidx(f)) + " * n_b + r) * W + (W - 1 - j)]"
                        : "rb[((unsigned long long)" + lit(f) + " * nmax + r) * W + (W - 1 - j)]")
              << " : Z; C" << f << "[j] = t" << comp(f) << "; }\n";
        }
        // cm = sum over contributions into (o, f) of c * m_h; then win[o][j] += C_f[j] * cm
        std::set<std::pair<int, int>> of;
        for (auto& c : b) of.insert({c.out, c.factor});
        for (auto& pr : of) {
            const int o = pr.first, f = pr.second;
            s << "            { double2 cm = Z;\n";
            live.erase("cm");
            for (auto& c : b)
                if (c.out == o && c.factor == f) s << "              " << cmac("cm", c.coeff, "m" + lit(c.in)) << "\n";
            if (f < 0) {
                s << "              win[" << o << "][" << WQ("BW") << "].x += cm.x; win[" << o << "][" << WQ("BW")
                  << "].y += cm.y; }\n";
            } else if (is_scal(f)) {
                s << "#pragma unroll\n              for (int j = 0; j < W; ++j) {"
                  << mac(f, "win[" + lit(o) + "][" + WQ("j") + "]", "C" + lit(f) + "[j]", "cm") << " } }\n";
            } else {
                s << "#pragma unroll\n              for (int j = 0; j < W; ++j) cacc(win[" << o << "][" << WQ("j") << "], C" << f
                  << "[j], cm); }\n";
            }
        }
        s << "        }\n        const int rd = ib - BW;\n        if (rd >= 0 && valid) {\n";
        for (int o = 0; o < nout; ++o)
            s << "            P.out[" << o << "][base + s_b * rd] = win[" << o << "][" << WQ("0") << "];\n";
        if (rot) {
            // the stored slot becomes the newest position of the next plane
            s << "        }\n#pragma unroll\n        for (int o = 0; o < " << nout << "; ++o) win[o][ph] = Z;\n    }\n    }\n";
        } else {
            s << "        }\n#pragma unroll\n        for (int o = 0; o < " << nout
              << "; ++o) {\n#pragma unroll\n            for (int j = 0; j < W - 1; ++j) win[o][j] = win[o][j + 1];\n"
              << "            win[o][W - 1] = Z;\n        }\n    }\n";
        }
    }
    s << "    asm volatile(\"cp.async.wait_group 0;\\n\" ::);\n}\n";
    std::unique_ptr<KronJitPair> P(new KronJitPair());
    P->k = jit_compile(s.str());
    P->nin = nin;
    P->nmid = nmid;
    P->nout = nout;
    P->bw = bw;
    P->pull = pull;
    P->T = T;
    P->nq = nq;
    P->no = no;
    P->D = D;
    P->pad = pad;
    P->smem = smem(D) + (stage ? bstage : 0) + (asm_rows ? astage : 0);
    P->s_a = s_a;
    P->n_a = n_a;
    P->n_b = n_b;
    P->n_outer = n_outer;
    P->grid = (unsigned)(nqb * nob);
    P->coef = coeffs;
    P->ncoef = (int)coeffs.size();
    return P.release();
}

static int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        KS_CUDA(cudaGetDevice(&dev));
        KS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return sms;
}

// each CTA sweeps the whole axis b serially: too few CTAs leave the GPU idle
// (c2: 22 CTAs, 0.23 ms vs 0.064 ms for the per-pass kernels)
bool kron_jit_runs(const KronJitPair& J) {
    // KS_KRON_JIT=b2 / b4 / point (a forced candidate: tests, profiling) also lifts the grid-size rule
    static const bool forced = [] {
        const char* e = std::getenv("KS_KRON_JIT");
        return e && (!std::strcmp(e, "b2") || !std::strcmp(e, "b4") || !std::strcmp(e, "point") || !std::strcmp(e, "tile") || !std::strcmp(e, "shift"));
    }();
    return forced || J.grid >= (unsigned)sm_count();
}
const char* kron_jit_tag(const KronJitPair& J) { return J.tag.c_str(); }
int kron_jit_blocked_rows(const KronJitPair& J) { return J.blocked ? (J.tile ? 1000 + J.nq : J.nq) : 0; }
bool kron_jit_same_shape(const KronJitPair& A, const KronJitPair& B) {
    return A.blocked == B.blocked && A.T == B.T && A.nq == B.nq && A.no == B.no && A.D == B.D;
}

// Tensor maps of the level tensors seen as doubles. Row-blocked kernel:
// (2 s_a, n_a, planes), box = 64 doubles x (RT + 2 bw) rows x 1 plane (halo rows
// included, zero filled outside). Tile kernel: (2 n_a, n_b, outer), box = PX
// entries x (RB + 2 bw) rows x 1. cuTensorMapEncodeTiled comes through the runtime's
// driver entry point, so libks keeps linking only cudart.
static void encode_map3(void* out, const void* base, long long d0, long long d1, long long d2, int b0, int b1, int b2) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        KS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        KS_REQUIRE(p && q == cudaDriverEntryPointSuccess, KS_ECUDA, "cuTensorMapEncodeTiled not available");
        fn = reinterpret_cast<Fn>(p);
    }
    // a dense tensor of doubles (d0 fastest), box b0 x b1 x b2, no swizzle, zero fill outside
    const cuuint64_t gdim[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
    const cuuint64_t gstr[2] = {(cuuint64_t)(d0 * 8), (cuuint64_t)(d0 * 8 * d1)};
    const cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, (cuuint32_t)b2}, est[3] = {1u, 1u, 1u};
    CUtensorMap m;
    const CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), gdim, gstr, box, est,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    KS_REQUIRE(r == CUDA_SUCCESS, KS_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    std::memcpy(out, &m, sizeof m);
}

// launch over the plan's tensors (geometry fixed at build); false when the
// grid is too small to fill the GPU (the caller runs the passes separately)
bool kron_jit_launch(const KronJitPair& J, const double2* const* ip, double2* const* op, void* const* hin,
                     void* const* hout, const double2* rb, int nmax, cudaStream_t st) {
    if (!kron_jit_runs(J)) return false;
    if (J.blocked) {
        // by-value parameter: input / output tensors, band table
        // (tensor maps first: 64-byte aligned, 128 B each)
        const size_t bytes = (size_t)J.nin * 128 + ((size_t)J.nout + 2) * sizeof(void*);
        std::vector<unsigned char> raw(bytes + 128 + 64, 0);
        unsigned char* w = raw.data() + (64 - reinterpret_cast<uintptr_t>(raw.data()) % 64) % 64;
        unsigned char* const w0 = w;
        for (int g = 0; g < J.nin; ++g, w += 128) {
            if (J.tile) encode_map3(w, hin[g], 2LL * J.n_a, J.n_b, J.n_outer, 2 * J.D, J.nq + 2 * J.bw, 1); // PX entries x RBH rows
            else encode_map3(w, hin[g], 2 * J.s_a, J.n_a, (long long)J.n_b * J.n_outer, 64, J.no + 2 * J.bw, 1);
        }
        for (int o = 0; o < J.nout; ++o, w += sizeof(void*)) std::memcpy(w, &hout[o], sizeof(void*));
        std::memcpy(w, &rb, sizeof(void*));
        w += sizeof(void*);
        std::memcpy(w, &nmax, sizeof(int));
        void* args[] = {(void*)w0};
        KS_CUDA(cudaLaunchKernel((const void*)J.k.fn, dim3(J.grid), dim3(J.T), args, J.smem, st));
        check_launch(J.tile ? "ks_pairt (jit)" : "ks_pairb (jit)");
        return true;
    }
    // by-value coefficient table (constant bank)
    // by-value parameter: coefficients, then the input and output tensor pointers
    const size_t nc = (size_t)std::max(1, J.ncoef);
    std::vector<double2> coef(nc + (size_t)(J.nin + J.nout + 1) / 2 + 1);
    std::copy(J.coef.begin(), J.coef.end(), coef.begin());
    void** pp = reinterpret_cast<void**>(coef.data() + nc);
    for (int g = 0; g < J.nin; ++g) pp[g] = hin[g];
    for (int o = 0; o < J.nout; ++o) pp[J.nin + o] = hout[o];
    long long s_a = J.s_a, n_outer = J.n_outer;
    int n_a = J.n_a, n_b = J.n_b, nq = J.nq, no = J.no, D = J.D;
    void* args[] = {(void*)&ip, (void*)&op, (void*)&rb, (void*)&nmax, (void*)&s_a, (void*)&n_a,
                    (void*)&n_b, (void*)&n_outer, (void*)&nq, (void*)&no, (void*)&D, (void*)coef.data()};
    KS_CUDA(cudaLaunchKernel((const void*)J.k.fn, dim3(J.grid), dim3(J.T), args, J.smem, st));
    check_launch("ks_pair (jit)");
    return true;
}

// ---------------------------------------------------------------------------
// Row-blocked variant of a fused pass pair for an in-plane axis a with inner
// columns (s_a > 1; at d = 3 the (2, 3) pair): the (t, i1) columns run across
// the lanes, a thread owns R consecutive rows of axis a, and the sweep along
// axis b scatters ("push") into a register window of output rows.
//
// Why (ncu of the thread-per-point kernel, c3 pass (2, 3)): 30 LDS.128 per
// point and plane -- 15 taps of the three inputs plus 15 band rows -- against
// 90 DFMA, `short_scoreboard` / `mio_throttle` on top. Here
//   * a thread loads R + 2 bw values per input for R points (R = 2: 9 LDS per
//     point, R = 4: 6) from a [row][32 lanes] tile: conflict-free 16 B per lane;
//   * every band entry is a literal in the generated source: the row block of
//     a warp is uniform, so the interior (Toeplitz, uniform mesh) rows share one
//     code path and each boundary row block gets its own, selected by a
//     warp-uniform switch; along the sweep axis the interior planes use
//     literals and the few boundary planes read the band table;
//   * the contribution coefficients are folded into those literals, so a
//     product costs exactly 2 DFMA per tap and complex value;
//   * planes arrive through a ring of whole-plane stages filled by a producer
//     warp with one bulk copy per (input, row) -- 512 B each -- on full / empty
//     mbarriers; the consumer warps never meet at a CTA barrier.
// Requires every factor of the pair to be Toeplitz away from a few boundary
// rows (uniform knot vectors); otherwise the builder returns null and the
// thread-per-point kernel runs.
// ---------------------------------------------------------------------------
namespace {

std::string hexd(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%a", v);
    return std::string(b);
}

// Literal coefficients of a generated kernel: hexadecimal floating-point literals in the
// source (materialised with two UMOVs each in SASS). Entries of a __constant__ table
// (constant-bank DFMA operands instead) measured slower in the row-blocked and tile
// kernels: c3 tile 219 -> 223 us, row-blocked 188 -> 200 us; c5 5.45 -> 6.1 ms, 6.06 -> 6.58 ms.
struct ConstTable {
    std::string ref(double x) const { return hexd(x); }
    const std::string& finish(const std::string& src) const { return src; }
};

// rows [lo, hi) of factor f equal to the middle row (relative 1e-13)
void toeplitz_range(const double2* hrb, int f, int nmax, int n, int W, int& lo, int& hi) {
    const int mid = n / 2;
    const double2* T = hrb + ((size_t)f * nmax + mid) * W;
    double sc = 0;
    for (int k = 0; k < W; ++k) sc = std::max(sc, std::max(std::fabs(T[k].x), std::fabs(T[k].y)));
    auto same = [&](int r) {
        const double2* row = hrb + ((size_t)f * nmax + r) * W;
        for (int k = 0; k < W; ++k)
            if (std::fabs(row[k].x - T[k].x) > 1e-13 * sc || std::fabs(row[k].y - T[k].y) > 1e-13 * sc) return false;
        return true;
    };
    lo = mid;
    hi = mid + 1;
    while (lo > 0 && same(lo - 1)) --lo;
    while (hi < n && same(hi)) ++hi;
}

// One statement `acc += (cc * e) * w` with the band entry as a literal, by factor class (1 real,
// 2 purely imaginary, 0 complex): 2 DFMA for a real or imaginary entry, 4 for a complex one. Empty
// when the entry is zero.
std::string literal_fma(const std::string& ind, int fclass, double cc, double2 e, const std::string& acc, const std::string& wv) {
    std::ostringstream t;
    if (fclass == 1) {
        if (e.x == 0.0) return "";
        const std::string v = hexd(cc * e.x);
        t << ind << acc << ".x = fma(" << v << ", " << wv << ".x, " << acc << ".x); " << acc << ".y = fma(" << v << ", " << wv << ".y, " << acc
          << ".y);\n";
    } else if (fclass == 2) {
        if (e.y == 0.0) return "";
        const std::string v = hexd(cc * e.y);
        t << ind << acc << ".x = fma(-(" << v << "), " << wv << ".y, " << acc << ".x); " << acc << ".y = fma(" << v << ", " << wv << ".x, " << acc
          << ".y);\n";
    } else {
        if (e.x == 0.0 && e.y == 0.0) return "";
        const std::string vx = hexd(cc * e.x), vy = hexd(cc * e.y);
        t << ind << acc << ".x = fma(" << vx << ", " << wv << ".x, fma(-(" << vy << "), " << wv << ".y, " << acc << ".x)); " << acc
          << ".y = fma(" << vx << ", " << wv << ".y, fma(" << vy << ", " << wv << ".x, " << acc << ".y));\n";
    }
    return t.str();
}

} // namespace

KronJitPair* kron_jitb_build(int nin, int nmid, int nout, int bw, const std::vector<JitContrib>& a,
                             const std::vector<JitContrib>& b, const std::vector<int>& freal,
                             const std::vector<double2>& coeffs, long long s_a, int n_a, int n_b, long long n_outer,
                             const double2* hrb, int nmax, int R, bool align4, bool shift) {
    if (const char* e = std::getenv("KS_KRON_JIT"))
        if (std::strcmp(e, "0") == 0) return nullptr;
    if (s_a < 32 || nin < 1 || nmid < 1 || nout < 1 || nin > 4 || nmid > 6 || nout > 2 || bw < 1 || bw > 4) return nullptr;
    if (R < 1 || R > 4 || n_a < 4 * bw + 2 || n_b < 4 * bw + 2) return nullptr;
    const int W = 2 * bw + 1;
    auto cls = [&](int f) { return freal[f]; }; // 1 real, 2 imaginary, 0 complex
    std::set<int> FA, FB;
    for (auto& c : a) {
        if (c.factor < 0) return nullptr; // (identity factors: the other kernel)
        FA.insert(c.factor);
    }
    for (auto& c : b) {
        if (c.factor < 0) return nullptr;
        FB.insert(c.factor);
    }
    int loa = 0, hia = n_a, lob = 0, hib = n_b;
    for (int f : FA) {
        int lo, hi;
        toeplitz_range(hrb, f, nmax, n_a, W, lo, hi);
        loa = std::max(loa, lo);
        hia = std::min(hia, hi);
    }
    for (int f : FB) {
        int lo, hi;
        toeplitz_range(hrb, f, nmax, n_b, W, lo, hi);
        lob = std::max(lob, lo);
        hib = std::min(hib, hi);
    }
    if (loa > 8 || n_a - hia > 8 || lob > 8 || n_b - hib > 8) return nullptr; // not a uniform-mesh factor
    // tile: 32 lanes x RT rows (+ halo), RT a multiple of R, at most 32 rows
    // align4: the fewest row tiles whose consumer warps + the producer warp fill
    // whole groups of four warps -- registers are allocated per four warps, so
    // 13 + 1 warps (c5: 26 rows, R = 2) leave 128 registers per thread and the
    // kernel spills, while 11 + 1 warps (22 rows) get 168 and do not
    int nrt = (n_a + 31) / 32;
    int RT = ((n_a + nrt - 1) / nrt + R - 1) / R * R;
    if (align4) {
        bool found = false;
        for (int t = nrt; t <= nrt + 3 && !found; ++t) {
            const int rt = ((n_a + t - 1) / t + R - 1) / R * R;
            if ((rt / R + 1) % 4 == 0 && rt / R >= 3) {
                found = (t != nrt);
                nrt = t;
                RT = rt;
                break;
            }
        }
        if (!found) return nullptr; // (already aligned, or no aligned shape: the default candidate covers it)
    }
    const int NW = RT / R;
    const int RTH = RT + 2 * bw;
    const size_t stage = (size_t)nin * RTH * 32 * sizeof(double2);
    int S = (int)std::min<size_t>(4, (size_t)(220 * 1024) / stage);
    if (S < 2 || NW < 1 || NW > 16) return nullptr;
    const int nqt = (int)((s_a + 31) / 32);
    // boundary row blocks (global block index gb = row / R)
    const int nblk = (n_a + R - 1) / R;
    const int NBLO = (loa + R - 1) / R, HB0 = hia / R;
    if (NBLO + (nblk - HB0) > 16 || HB0 < NBLO) return nullptr;
    auto band = [&](int f, int row, int k) -> double2 { // entry k of row `row` (zero outside)
        if (row < 0) return make_double2(0, 0);
        return hrb[((size_t)f * nmax + row) * W + k];
    };
    // single-consumer products fold the contribution coefficient into the literals
    auto cval = [&](int ci) { return coeffs[ci]; };
    for (auto& c : a)
        if (cval(c.coeff).y != 0.0) return nullptr; // (complex contribution coefficients: the other kernel)
    for (auto& c : b)
        if (cval(c.coeff).y != 0.0) return nullptr;
    ConstTable KT;
    std::ostringstream s;
    s << "// generated: row-blocked fused level passes (ks_kron_jit.cu)\n"
      << "#define BW " << bw << "\n#define W " << W << "\n#define NIN " << nin << "\n#define NMID " << nmid << "\n#define NOUT "
      << nout << "\n#define R " << R << "\n#define RT " << RT << "\n#define RTH " << RTH << "\n#define S " << S
      << "\n#define NW " << NW << "\n#define s_a " << s_a << "LL\n#define n_a " << n_a << "\n#define n_b " << n_b
      << "\n#define NQT " << nqt << "\n#define NRT " << nrt << "\n"
      << "struct __align__(64) TMap { unsigned long long d[16]; };\n"
      << "struct Par { TMap tm[NIN]; double2* out[NOUT]; const double2* rb; int nmax; };\n"
      << R"(
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mwait(unsigned long long* b, unsigned parity) {
    unsigned ok = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(su32(b)), "r"(parity) : "memory");
    } while (!ok);
}
extern "C" __global__ void __launch_bounds__(32 * (NW + 1), 1) ks_pairb(const __grid_constant__ Par P) {
    extern __shared__ __align__(128) unsigned char smraw[];
    double2* ring = reinterpret_cast<double2*>(smraw); // [S][NIN][RTH][32]
    unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + (size_t)S * NIN * RTH * 32);
    unsigned long long* empty = full + S;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rt = blockIdx.x % NRT, qt = (blockIdx.x / NRT) % NQT;
    const long long oo = blockIdx.x / (NRT * NQT);
    const long long q0 = 32LL * qt;
    const int row0 = rt * RT;
    const int ncol = (int)(s_a - q0 < 32 ? s_a - q0 : 32);
    const double2 Z = make_double2(0.0, 0.0);
    for (int e = tid; e < S * NIN * RTH * 32; e += 32 * (NW + 1)) ring[e] = Z; // halo rows / columns never loaded stay zero
    if (tid == 0) {
        for (int q = 0; q < S; ++q) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full + q)) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(empty + q)), "n"(NW) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long s_b = s_a * n_a;
    const long long obase = oo * s_b * n_b + q0;
    if (warp == NW) {
        // ---- producer: one tensor-map TMA box (64 doubles x RTH rows) per input and
        // plane; rows outside [0, n_a) and columns past s_a arrive as zeros ----
        if (lane != 0) return;
        for (int ib = 0; ib < n_b; ++ib) {
            const int slot = ib % S;
            if (ib >= S) mwait(empty + slot, (unsigned)((ib / S - 1) & 1));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + slot)),
                         "r"((unsigned)(NIN * RTH * 512)) : "memory");
#pragma unroll
            for (int g = 0; g < NIN; ++g)
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
                             "r"(su32(ring + (size_t)(slot * NIN + g) * RTH * 32)), "l"(&P.tm[g]), "r"((int)(2 * q0)),
                             "r"(row0 - BW), "r"((int)(oo * n_b + ib)), "r"(su32(full + slot))
                             : "memory");
        }
        return;
    }
    // ---- consumer warps: rows grow .. grow + R - 1 of axis a, column q0 + lane ----
    const int rl = warp * R, grow = row0 + rl, gb = grow / R;
    const bool qok = lane < ncol;
)";
    s << "    int cls = 0;\n    if (grow >= n_a) cls = -1;\n    else if (gb < " << NBLO << ") cls = 1 + gb;\n    else if (gb >= " << HB0
      << ") cls = " << (1 + NBLO) << " + (gb - " << HB0 << ");\n"
      << "    double2 win[NOUT][R][W];\n"
      << "#pragma unroll\n    for (int o = 0; o < NOUT; ++o)\n#pragma unroll\n        for (int r = 0; r < R; ++r)\n#pragma unroll\n"
      << "            for (int j = 0; j < W; ++j) win[o][r][j] = Z;\n"
      << "    int ph = 0;\n"
      << "    for (int ib = 0; ib < n_b + BW; ++ib) {\n"
      << "        double2 m[NMID][R];\n"
      << "#pragma unroll\n        for (int h = 0; h < NMID; ++h)\n#pragma unroll\n            for (int r = 0; r < R; ++r) m[h][r] = Z;\n"
      << "        if (ib < n_b) {\n"
      << "            const int slot = ib % S;\n"
      << "            mwait(full + slot, (unsigned)((ib / S) & 1));\n"
      << "            const double2* sl = ring + ((size_t)slot * NIN * RTH + rl) * 32 + lane;\n"
      << "            switch (cls) {\n";
    // in-plane code for one row block: rows[r] = global row of r (or -1: interior Toeplitz; -2: no row)
    auto emit_inplane = [&](const std::vector<int>& rows) {
        for (int g = 0; g < nin; ++g) {
            std::vector<const JitContrib*> cs;
            for (auto& c : a)
                if (c.in == g) cs.push_back(&c);
            if (cs.empty()) continue;
            s << "            {\n                double2 w[R + 2 * BW];\n#pragma unroll\n                for (int k = 0; k < R + 2 * BW; ++k) w[k] = sl[("
              << g << " * RTH + k) * 32];\n";
            for (auto* c : cs) {
                const int f = c->factor;
                const double cc = coeffs[c->coeff].x;
                for (int r = 0; r < R; ++r) {
                    if (rows[r] == -2) continue;
                    const std::string acc = "m[" + lit(c->out) + "][" + lit(r) + "]";
                    for (int k = 0; k < W; ++k) {
                        const double2 e = rows[r] == -1 ? band(f, (loa + hia) / 2, k) : band(f, rows[r], k);
                        const std::string wv = "w[" + lit(r + k) + "]";
                        if (cls(f) == 1) {
                            if (e.x == 0.0) continue;
                            const std::string v = KT.ref(cc * e.x);
                            s << "                " << acc << ".x = fma(" << v << ", " << wv << ".x, " << acc << ".x); " << acc
                              << ".y = fma(" << v << ", " << wv << ".y, " << acc << ".y);\n";
                        } else if (cls(f) == 2) {
                            if (e.y == 0.0) continue;
                            const std::string v = KT.ref(cc * e.y);
                            s << "                " << acc << ".x = fma(-(" << v << "), " << wv << ".y, " << acc << ".x); " << acc
                              << ".y = fma(" << v << ", " << wv << ".x, " << acc << ".y);\n";
                        } else {
                            if (e.x == 0.0 && e.y == 0.0) continue;
                            const std::string vx = KT.ref(cc * e.x), vy = KT.ref(cc * e.y);
                            s << "                " << acc << ".x = fma(" << vx << ", " << wv << ".x, fma(-(" << vy << "), " << wv
                              << ".y, " << acc << ".x)); " << acc << ".y = fma(" << vx << ", " << wv << ".y, fma(" << vy << ", "
                              << wv << ".x, " << acc << ".y));\n";
                        }
                    }
                }
            }
            s << "            }\n";
        }
    };
    {
        s << "            case 0: {\n";
        emit_inplane(std::vector<int>(R, -1));
        s << "            } break;\n";
        int ci = 1;
        auto emit_block = [&](int gbk) {
            std::vector<int> rows(R);
            for (int r = 0; r < R; ++r) rows[r] = gbk * R + r < n_a ? gbk * R + r : -2;
            s << "            case " << ci++ << ": {\n";
            emit_inplane(rows);
            s << "            } break;\n";
        };
        for (int g = 0; g < NBLO; ++g) emit_block(g);
        for (int g = HB0; g < nblk; ++g) emit_block(g);
    }
    s << "            default: break;\n            }\n"
      << "            __syncwarp();\n"
      << "            if (lane == 0) asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" ::\"r\"(su32(empty + slot)) : \"memory\");\n"
      << "        }\n";
    // push + store, one case per window phase
    const int PLO = lob + bw, PHI = hib - bw; // planes whose band columns are all interior
    s << "        const bool litp = ib >= " << PLO << " && ib < " << PHI << ";\n"
      << "        const int rd = ib - BW;\n"
      << (shift ? "        {\n" : "        switch (ph) {\n");
    // shift: one copy of the push with the window shifted by register moves every plane instead of W
    // rotated copies selected by the phase (a ninth of the push code: the hot loop of the bw = 4 kernel
    // is ~34 KB with the copies, 13% of its stall samples were instruction-cache misses)
    for (int ph = 0; ph < (shift ? 1 : W); ++ph) {
        s << (shift ? "        {\n" : "        case " + lit(ph) + ": {\n") << "            if (ib < n_b) {\n                if (litp) {\n";
        auto slotj = [&](int j) { return lit((ph + j) % W); };
        for (auto& c : b) {
            const int f = c.factor;
            const double cc = coeffs[c.coeff].x;
            for (int r = 0; r < R; ++r)
                for (int j = 0; j < W; ++j) {
                    const double2 e = band(f, (lob + hib) / 2, W - 1 - j);
                    const std::string acc = "win[" + lit(c.out) + "][" + lit(r) + "][" + slotj(j) + "]";
                    const std::string mv = "m[" + lit(c.in) + "][" + lit(r) + "]";
                    if (cls(f) == 1) {
                        if (e.x == 0.0) continue;
                        const std::string v = KT.ref(cc * e.x);
                        s << "                    " << acc << ".x = fma(" << v << ", " << mv << ".x, " << acc << ".x); " << acc
                          << ".y = fma(" << v << ", " << mv << ".y, " << acc << ".y);\n";
                    } else if (cls(f) == 2) {
                        if (e.y == 0.0) continue;
                        const std::string v = KT.ref(cc * e.y);
                        s << "                    " << acc << ".x = fma(-(" << v << "), " << mv << ".y, " << acc << ".x); " << acc
                          << ".y = fma(" << v << ", " << mv << ".x, " << acc << ".y);\n";
                    } else {
                        if (e.x == 0.0 && e.y == 0.0) continue;
                        const std::string vx = KT.ref(cc * e.x), vy = KT.ref(cc * e.y);
                        s << "                    " << acc << ".x = fma(" << vx << ", " << mv << ".x, fma(-(" << vy << "), " << mv
                          << ".y, " << acc << ".x)); " << acc << ".y = fma(" << vx << ", " << mv << ".y, fma(" << vy << ", " << mv
                          << ".x, " << acc << ".y));\n";
                    }
                }
        }
        s << "                } else {\n";
        // boundary planes: column ib of each factor from the band table, F(ib + j - BW, ib)
        for (int f : FB) {
            s << "                    double2 C" << f << "[W];\n#pragma unroll\n                    for (int j = 0; j < W; ++j) { const int r_ = ib + j - BW; C"
              << f << "[j] = (r_ >= 0 && r_ < n_b) ? __ldg(P.rb + ((size_t)" << f << " * P.nmax + r_) * W + (W - 1 - j)) : Z; }\n";
        }
        for (auto& c : b) {
            const int f = c.factor;
            const double cc = coeffs[c.coeff].x;
            for (int r = 0; r < R; ++r) {
                const std::string mv = "m[" + lit(c.in) + "][" + lit(r) + "]";
                s << "                    { const double2 cm = make_double2(" << KT.ref(cc) << " * " << mv << ".x, " << KT.ref(cc) << " * " << mv
                  << ".y);\n";
                for (int j = 0; j < W; ++j) {
                    const std::string acc = "win[" + lit(c.out) + "][" + lit(r) + "][" + slotj(j) + "]";
                    const std::string cf = "C" + lit(f) + "[" + lit(j) + "]";
                    s << "                      " << acc << ".x = fma(" << cf << ".x, cm.x, fma(-" << cf << ".y, cm.y, " << acc << ".x)); " << acc
                      << ".y = fma(" << cf << ".x, cm.y, fma(" << cf << ".y, cm.x, " << acc << ".y));\n";
                }
                s << "                    }\n";
            }
        }
        s << "                }\n            }\n"
          << "            if (rd >= 0 && qok) {\n";
        for (int o = 0; o < nout; ++o)
            for (int r = 0; r < R; ++r)
                s << "                if (grow + " << r << " < n_a) __stcs(P.out[" << o << "] + obase + s_b * rd + s_a * (grow + " << r
                  << ") + lane, win[" << o << "][" << r << "][" << ph << "]);\n";
        s << "            }\n";
        for (int o = 0; o < nout; ++o)
            for (int r = 0; r < R; ++r) {
                if (shift) {
                    for (int j = 0; j + 1 < W; ++j) s << "            win[" << o << "][" << r << "][" << j << "] = win[" << o << "][" << r << "][" << j + 1 << "];\n";
                    s << "            win[" << o << "][" << r << "][" << W - 1 << "] = Z;\n";
                } else {
                    s << "            win[" << o << "][" << r << "][" << ph << "] = Z;\n";
                }
            }
        s << (shift ? "        }\n" : "        } break;\n");
    }
    s << "        }\n        ph = ph + 1 == W ? 0 : ph + 1;\n    }\n}\n";
    std::unique_ptr<KronJitPair> P(new KronJitPair());
    const size_t smem = (size_t)S * stage + (size_t)2 * S * 8 + 128;
    P->k.fn = nvrtc_kernel(KT.finish(s.str()), "ks_pairb", 227 * 1024);
    P->blocked = true;
    P->nin = nin;
    P->nmid = nmid;
    P->nout = nout;
    P->bw = bw;
    P->pull = false;
    P->T = 32 * (NW + 1);
    P->nq = R; // (shape key: rows per thread)
    P->pad = shift ? 1 : 0;
    if (shift) P->tag = "shifted window";
    P->no = RT;
    P->D = S;
    P->smem = smem;
    P->s_a = s_a;
    P->n_a = n_a;
    P->n_b = n_b;
    P->n_outer = n_outer;
    P->grid = (unsigned)((long long)nqt * nrt * n_outer);
    P->coef = coeffs;
    P->ncoef = (int)coeffs.size();
    return P.release();
}


// ---------------------------------------------------------------------------
// Tile variant for a contiguous in-plane axis (s_a = 1; at d = 3 the (t, 1)
// pair) with one input: no register window at all. A CTA takes tiles of RB rows
// of axis b (+ bw halo rows on both sides) x the whole axis a, of one outer
// index, and runs two phases over shared memory:
//   A  axis-a products of the RB + 2 bw rows: lanes across the rows (pitch odd
//      in 16 B units: conflict-free), a thread owns RA consecutive entries of
//      its row and loads RA + 2 bw values for them; the axis-a rows are uniform
//      across the warp, so every band entry is a literal (one code path for the
//      Toeplitz interior, one per boundary block); mids go back to shared memory;
//   B  axis-b products: lanes across axis a, a thread owns RR consecutive rows
//      and loads RR + 2 bw values per mid for them; literal band entries by row
//      block class; streaming stores, coalesced along axis a.
// The halo rows' axis-a products are recomputed ((RB + 2 bw) / RB of phase A).
// The thread-per-point kernels keep a window of (outputs x W) complex values
// per thread -- 108 registers at bw = 4 with three outputs, beside 54 for the
// per-lane axis-a rows: they spill at c5 (ncu: 28% FP64 pipe). Here a thread
// holds <= (RA + 2 bw) + nmid RA values in phase A and (RR + 2 bw) + nout RR in
// phase B. The next tile's rows arrive by one bulk copy per row while phase B
// runs.
// ---------------------------------------------------------------------------
KronJitPair* kron_jitt_build(int nin, int nmid, int nout, int bw, const std::vector<JitContrib>& a,
                             const std::vector<JitContrib>& b, const std::vector<int>& freal,
                             const std::vector<double2>& coeffs, int n_a, int n_b, long long n_outer,
                             const double2* hrb, int nmax, int RB, int RA, int RR, int NWARP, int minb, int NAS) {
    if (const char* e = std::getenv("KS_KRON_JIT"))
        if (std::strcmp(e, "0") == 0) return nullptr;
    if (nin != 1 || nmid < 1 || nmid > 4 || nout < 1 || nout > 4 || bw < 1 || bw > 6) return nullptr;
    if (n_a < 4 * bw + 2 || n_b < 4 * bw + 2 || RA < 1 || RR < 1 || RB < RR || RB % RR != 0 || NAS < 1) return nullptr;
    const int W = 2 * bw + 1, RBH = RB + 2 * bw;
    if (RBH > 32) return nullptr; // phase A: one lane per row
    auto cls = [&](int f) { return freal[f]; };
    std::set<int> FA, FB;
    for (auto& c : a) {
        if (c.factor < 0 || coeffs[c.coeff].y != 0.0) return nullptr;
        FA.insert(c.factor);
    }
    for (auto& c : b) {
        if (c.factor < 0 || coeffs[c.coeff].y != 0.0) return nullptr;
        FB.insert(c.factor);
    }
    int loa = 0, hia = n_a, lob = 0, hib = n_b;
    for (int f : FA) {
        int lo, hi;
        toeplitz_range(hrb, f, nmax, n_a, W, lo, hi);
        loa = std::max(loa, lo);
        hia = std::min(hia, hi);
    }
    for (int f : FB) {
        int lo, hi;
        toeplitz_range(hrb, f, nmax, n_b, W, lo, hi);
        lob = std::max(lob, lo);
        hib = std::min(hib, hi);
    }
    if (loa > 2 * bw + 4 || n_a - hia > 2 * bw + 4 || lob > 2 * bw + 4 || n_b - hib > 2 * bw + 4) return nullptr; // not a uniform-mesh factor
    // shared memory: x rows [RBH][PX] (bw zeros | n_a | zeros, PX odd), mids [NMID][RBH][PM] (PM odd)
    // the axis-a range of a tile: NAS pieces of AT entries (a multiple of RA); the halo along a is only loaded
    const int AT = ((n_a + NAS - 1) / NAS + RA - 1) / RA * RA;
    if ((long long)AT * (NAS - 1) >= n_a || AT < 2 * bw) return nullptr;
    const int PX = (AT + 2 * bw) | 1, PM = AT | 1; // (odd pitches: conflict-free with the lanes across the rows)
    if (2 * PX > 256) return nullptr;              // one box: <= 256 doubles per dimension
    const size_t smem = ((size_t)RBH * PX + (size_t)nmid * RBH * PM) * sizeof(double2) + 64;
    if (smem * minb > 226 * 1024 || smem > 226 * 1024) return nullptr;
    const int T = 32 * NWARP;
    const int ntb = (n_b + RB - 1) / RB;
    const long long ntile = (long long)ntb * n_outer * NAS;
    // block classes along axis a (phase A, blocks of RA entries) and axis b (phase B, blocks of RR rows)
    const int nblkA = (n_a + RA - 1) / RA, ALO = (loa + RA - 1) / RA, AHI = hia / RA;
    const int nblkB = (n_b + RR - 1) / RR, BLO = (lob + RR - 1) / RR, BHI = hib / RR;
    if (AHI < ALO || BHI < BLO || ALO + (nblkA - AHI) > 24 || BLO + (nblkB - BHI) > 24) return nullptr;
    auto band = [&](int f, int row, int k) -> double2 { return hrb[((size_t)f * nmax + row) * W + k]; };
    ConstTable KT;
    std::ostringstream s;
    s << "// generated: tile variant of the fused level passes (ks_kron_jit.cu)\n"
      << "#define BW " << bw << "\n#define W " << W << "\n#define NMID " << nmid << "\n#define NOUT " << nout << "\n#define RB " << RB
      << "\n#define RBH " << RBH << "\n#define RA " << RA << "\n#define RR " << RR << "\n#define PX " << PX << "\n#define PM " << PM
      << "\n#define T " << T << "\n#define NWARP " << NWARP << "\n#define MINB " << minb << "\n#define n_a " << n_a << "\n#define n_b " << n_b
      << "\n#define n_outer " << n_outer << "LL\n#define NTB " << ntb << "\n#define NTILE " << ntile << "LL\n#define NAS " << NAS
      << "\n#define AT " << AT << "\n"
      << "struct __align__(64) TMap { unsigned long long d[16]; };\n"
      << "struct Par { TMap tm; double2* out[NOUT]; const double2* rb; int nmax; };\n"
      << R"(
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mwait(unsigned long long* b, unsigned parity) {
    unsigned ok = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(su32(b)), "r"(parity) : "memory");
    } while (!ok);
}
extern "C" __global__ void __launch_bounds__(T, MINB) ks_pairt(const __grid_constant__ Par P) {
    extern __shared__ __align__(128) unsigned char smraw[];
    double2* xs = reinterpret_cast<double2*>(smraw);   // [RBH][PX]: entries a0 - BW .. a0 + AT + BW of the row
    double2* ms = xs + (size_t)RBH * PX;                // [NMID][RBH][PM]
    unsigned long long* full = reinterpret_cast<unsigned long long*>(ms + (size_t)NMID * RBH * PM);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double2 Z = make_double2(0.0, 0.0);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // tile = as + NAS * (tb + NTB * outer): axis-a range [a0, a0 + AT), global rows b0 - BW + r, r < RBH.
    // One tensor-map box per tile: PX entries from a0 - BW of RBH rows from b0 - BW; entries and rows
    // outside the tensor arrive as zeros. (One bulk copy per row costs ~60 cycles each in the copy
    // engine: with the axis split in pieces the tiles became copy-issue bound, c3 325-442 us.)
    auto load_tile = [&](long long tile) {
        const int as = (int)(tile % NAS);
        const long long rest = tile / NAS, o = rest / NTB;
        const int b0 = (int)(rest - o * NTB) * RB, a0 = as * AT;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full)), "r"((unsigned)(RBH * PX * 16)) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
                     "r"(su32(xs)), "l"(&P.tm), "r"(2 * (a0 - BW)), "r"(b0 - BW), "r"((int)o), "r"(su32(full)) : "memory");
    };
    long long tile = blockIdx.x;
    if (tile < NTILE && tid == 0) load_tile(tile);
    unsigned par = 0;
    for (; tile < NTILE; tile += gridDim.x, par ^= 1) {
        const int as = (int)(tile % NAS);
        const long long rest = tile / NAS, o = rest / NTB;
        const int b0 = (int)(rest - o * NTB) * RB, a0 = as * AT;
        const int nat = n_a - a0 < AT ? n_a - a0 : AT; // entries of this tile along a
        mwait(full, par);
        // ---- phase A: axis-a products of row `lane`, blocks of RA entries ----
        {
            const int row = b0 - BW + lane;
            const bool rin = row >= 0 && row < n_b;
            if (lane < RBH) {
                const double2* xr = xs + (size_t)lane * PX; // xr[q] = x(a0 - BW + q)
                for (int jl = warp; jl * RA < nat; jl += NWARP) {
                    const int t0 = jl * RA, j = a0 / RA + jl; // local offset, global block
                    double2 acc[NMID][RA];
#pragma unroll
                    for (int h = 0; h < NMID; ++h)
#pragma unroll
                        for (int i = 0; i < RA; ++i) acc[h][i] = Z;
                    if (rin) {
                        double2 w[RA + 2 * BW];
#pragma unroll
                        for (int q = 0; q < RA + 2 * BW; ++q) w[q] = xr[t0 + q];
)";
    // literal product: acc[i] += cc * F[row_i][k] * w[i + k] for the rows of one block. The statements of
    // a case are collected and written tap by tap (k outermost), so consecutive DFMAs belong to different
    // accumulators: a dependent pair sits as many instructions apart as the case has chains.
    std::vector<std::pair<int, std::string>> pend;
    auto emit_prod = [&](const std::string& ind, int f, double cc, const std::vector<int>& rows, int mid_row,
                         const std::function<std::string(int)>& accn) {
        for (size_t i = 0; i < rows.size(); ++i) {
            if (rows[i] == -2) continue;
            for (int k = 0; k < W; ++k) {
                const double2 e = rows[i] == -1 ? band(f, mid_row, k) : band(f, rows[i], k);
                const std::string st = literal_fma(ind, cls(f), cc, e, accn((int)i), "w[" + lit((int)i + k) + "]");
                if (!st.empty()) pend.push_back({k, st});
            }
        }
    };
    auto flush = [&] {
        std::stable_sort(pend.begin(), pend.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
        for (auto& q : pend) s << q.second;
        pend.clear();
    };
    // phase A classes: 0 interior, then the boundary blocks
    {
        s << "                        int ca = 0;\n                        if (j < " << ALO << ") ca = 1 + j; else if (j >= " << AHI
          << ") ca = " << (1 + ALO) << " + (j - " << AHI << ");\n                        switch (ca) {\n";
        int ci = 0;
        auto emit_case = [&](const std::vector<int>& rows) {
            s << "                        case " << ci++ << ": {\n";
            for (auto& c : a)
                emit_prod("                            ", c.factor, coeffs[c.coeff].x, rows, (loa + hia) / 2,
                          [&](int i) { return "acc[" + lit(c.out) + "][" + lit(i) + "]"; });
            flush();
            s << "                        } break;\n";
        };
        emit_case(std::vector<int>(RA, -1));
        auto blockrows = [&](int j) {
            std::vector<int> rows(RA);
            for (int i = 0; i < RA; ++i) rows[i] = j * RA + i < n_a ? j * RA + i : -2;
            return rows;
        };
        for (int j = 0; j < ALO; ++j) emit_case(blockrows(j));
        for (int j = AHI; j < nblkA; ++j) emit_case(blockrows(j));
        s << "                        default: break;\n                        }\n";
    }
    s << R"(                    }
#pragma unroll
                    for (int h = 0; h < NMID; ++h)
#pragma unroll
                        for (int i = 0; i < RA; ++i)
                            if (t0 + i < nat) ms[((size_t)h * RBH + lane) * PM + t0 + i] = acc[h][i];
                }
            }
        }
        __syncthreads();
        // the x rows are consumed: the next tile's rows arrive while phase B runs
        if (tid == 0 && tile + gridDim.x < NTILE) load_tile(tile + gridDim.x);
        // ---- phase B: axis-b products, RR rows per thread, lanes across axis a ----
        {
            const int nbt = n_b - b0 < RB ? n_b - b0 : RB; // rows of this tile
            const int nblk = (nbt + RR - 1) / RR;
            for (int e = tid; e < nblk * nat; e += T) {
                const int blk = e / nat, t = e - blk * nat;
                const int gb = b0 / RR + blk; // global row block (RB is a multiple of RR)
                const double2* mr = ms + (size_t)(blk * RR) * PM + t; // mr[(h * RBH + q) * PM] = mid h at row b0 + blk RR - BW + q
                double2 acc[NOUT][RR];
#pragma unroll
                for (int o2 = 0; o2 < NOUT; ++o2)
#pragma unroll
                    for (int i = 0; i < RR; ++i) acc[o2][i] = Z;
                int cb = 0;
)";
    s << "                if (gb < " << BLO << ") cb = 1 + gb; else if (gb >= " << BHI << ") cb = " << (1 + BLO) << " + (gb - " << BHI
      << ");\n                switch (cb) {\n";
    {
        int ci = 0;
        auto emit_case = [&](const std::vector<int>& rows) {
            s << "                case " << ci++ << ": {\n";
            for (int h = 0; h < nmid; ++h) {
                bool used = false;
                for (auto& c : b) used = used || c.in == h;
                if (!used) continue;
                s << "                    {\n                        double2 w[RR + 2 * BW];\n#pragma unroll\n                        for (int q = 0; q < RR + 2 * BW; ++q) w[q] = mr[((size_t)"
                  << h << " * RBH + q) * PM];\n";
                for (auto& c : b)
                    if (c.in == h)
                        emit_prod("                        ", c.factor, coeffs[c.coeff].x, rows, (lob + hib) / 2,
                                  [&](int i) { return "acc[" + lit(c.out) + "][" + lit(i) + "]"; });
                flush();
                s << "                    }\n";
            }
            s << "                } break;\n";
        };
        emit_case(std::vector<int>(RR, -1));
        auto blockrows = [&](int g) {
            std::vector<int> rows(RR);
            for (int i = 0; i < RR; ++i) rows[i] = g * RR + i < n_b ? g * RR + i : -2;
            return rows;
        };
        for (int g = 0; g < BLO; ++g) emit_case(blockrows(g));
        for (int g = BHI; g < nblkB; ++g) emit_case(blockrows(g));
        s << "                default: break;\n                }\n";
    }
    s << R"(                const size_t ob = ((size_t)o * n_b + b0 + blk * RR) * n_a + a0 + t;
#pragma unroll
                for (int i = 0; i < RR; ++i)
                    if (blk * RR + i < nbt) {
#pragma unroll
                        for (int o2 = 0; o2 < NOUT; ++o2) __stcs(P.out[o2] + ob + (size_t)i * n_a, acc[o2][i]);
                    }
            }
        }
        __syncthreads();
    }
}
)";
    std::unique_ptr<KronJitPair> P(new KronJitPair());
    P->k.fn = nvrtc_kernel(KT.finish(s.str()), "ks_pairt", 227 * 1024);
    P->blocked = true;
    P->tile = true;
    P->nin = nin;
    P->nmid = nmid;
    P->nout = nout;
    P->bw = bw;
    P->pull = true;
    P->T = T;
    P->nq = RB; // (shape key)
    P->no = RA * 100 + RR;
    P->pad = minb * 10 + NAS;
    P->tag = "tile RB " + lit(RB) + " RA " + lit(RA) + " RR " + lit(RR) + " warps " + lit(NWARP) + " ctas/sm " + lit(minb) + " pieces " + lit(NAS);
    P->D = PX;
    P->smem = smem;
    P->s_a = 1;
    P->n_a = n_a;
    P->n_b = n_b;
    P->n_outer = n_outer;
    P->grid = (unsigned)std::min<long long>(ntile, (long long)sm_count() * minb);
    P->coef = coeffs;
    P->ncoef = (int)coeffs.size();
    return P.release();
}

// ---------------------------------------------------------------------------
// Generated single pass along an axis with inner columns (s_a >= 32): the trailing
// pass of a plan with an odd number of passes (d = 2: axis 2 after the (t, 1) pair),
// or a pass whose pair cannot run fused. Lanes across the contiguous columns, a
// thread owns RR consecutive rows of the axis and loads RR + 2 bw values per input
// for them straight from global memory (the level tensors of these plans sit in L2);
// the row block is uniform across the CTA, so the band entries are literals (Toeplitz
// interior, one code path per boundary block). The element-parallel kernel it
// replaces loads 2 bw + 1 values and band rows per point: c4 (p = 2) axis-2 pass
// 61 us.
// ---------------------------------------------------------------------------
struct KronJitPass {
    cudaKernel_t fn = nullptr;
    int nin = 0, nout = 0;
    unsigned gx = 0, gy = 0;
};
void kron_jitc_free(KronJitPass* p) { delete p; }

KronJitPass* kron_jitc_build(int nin, int nout, int bw, const std::vector<JitContrib>& c, const std::vector<int>& freal,
                             const std::vector<double2>& coeffs, long long s_a, int n_a, long long n_outer,
                             const double2* hrb, int nmax, int RR) {
    if (const char* e = std::getenv("KS_KRON_JIT"))
        if (std::strcmp(e, "0") == 0) return nullptr;
    if (s_a < 32 || nin < 1 || nin > 6 || nout < 1 || nout > 4 || bw < 1 || bw > 6 || RR < 1 || RR > 4 || n_a < 4 * bw + 2)
        return nullptr;
    const int W = 2 * bw + 1;
    auto cls = [&](int f) { return freal[f]; };
    int lo = 0, hi = n_a;
    for (auto& k : c) {
        if (k.factor < 0 || coeffs[k.coeff].y != 0.0) return nullptr;
        int l, h;
        toeplitz_range(hrb, k.factor, nmax, n_a, W, l, h);
        lo = std::max(lo, l);
        hi = std::min(hi, h);
    }
    if (lo > 2 * bw + 4 || n_a - hi > 2 * bw + 4 || lo < bw || n_a - hi < bw) return nullptr;
    const int nblk = (n_a + RR - 1) / RR, BLO = (lo + RR - 1) / RR, BHI = hi / RR;
    if (BHI < BLO || BLO + (nblk - BHI) > 24) return nullptr;
    const long long nqc = (s_a + 127) / 128;
    if (nqc * n_outer > 0x7fffffffLL || nblk > 65535) return nullptr;
    auto band = [&](int f, int row, int k) -> double2 { return hrb[((size_t)f * nmax + row) * W + k]; };
    std::ostringstream s;
    s << "// generated: single pass over inner columns (ks_kron_jit.cu)\n"
      << "#define BW " << bw << "\n#define W " << W << "\n#define NIN " << nin << "\n#define NOUT " << nout << "\n#define RR " << RR
      << "\n#define s_a " << s_a << "LL\n#define n_a " << n_a << "\n#define NQC " << nqc << "LL\n"
      << "struct Par { const double2* in[NIN]; double2* out[NOUT]; };\n"
      << R"(
extern "C" __global__ void __launch_bounds__(128) ks_passc(const __grid_constant__ Par P) {
    const long long o = blockIdx.x / NQC;
    const long long q = (blockIdx.x - o * NQC) * 128 + threadIdx.x;
    const int gb = blockIdx.y, r0 = gb * RR;
    if (q >= s_a) return;
    const size_t base = (size_t)o * n_a * s_a + q; // row r of this column: base + r * s_a
    const double2 Z = make_double2(0.0, 0.0);
    double2 acc[NOUT][RR];
#pragma unroll
    for (int o2 = 0; o2 < NOUT; ++o2)
#pragma unroll
        for (int i = 0; i < RR; ++i) acc[o2][i] = Z;
    int cb = 0;
)";
    s << "    if (gb < " << BLO << ") cb = 1 + gb; else if (gb >= " << BHI << ") cb = " << (1 + BLO) << " + (gb - " << BHI << ");\n"
      << "    switch (cb) {\n";
    std::vector<std::pair<int, std::string>> pend;
    auto emit = [&](const std::vector<int>& rows, bool guard) {
        for (int g = 0; g < nin; ++g) {
            bool used = false;
            for (auto& k : c) used = used || k.in == g;
            if (!used) continue;
            s << "        {\n            double2 w[RR + 2 * BW];\n#pragma unroll\n            for (int k = 0; k < RR + 2 * BW; ++k) {";
            if (guard)
                s << " const int row = r0 - BW + k; w[k] = (row >= 0 && row < n_a) ? __ldg(P.in[" << g
                  << "] + base + (size_t)row * s_a) : Z; }\n";
            else
                s << " w[k] = __ldg(P.in[" << g << "] + base + (size_t)(r0 - BW + k) * s_a); }\n";
            for (auto& k : c) {
                if (k.in != g) continue;
                const double cc = coeffs[k.coeff].x;
                for (size_t i = 0; i < rows.size(); ++i) {
                    if (rows[i] == -2) continue;
                    for (int t = 0; t < W; ++t) {
                        const double2 e = rows[i] == -1 ? band(k.factor, (lo + hi) / 2, t) : band(k.factor, rows[i], t);
                        const std::string st = literal_fma("            ", cls(k.factor), cc, e, "acc[" + lit(k.out) + "][" + lit((int)i) + "]",
                                                           "w[" + lit((int)i + t) + "]");
                        if (!st.empty()) pend.push_back({t, st});
                    }
                }
            }
            std::stable_sort(pend.begin(), pend.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
            for (auto& q : pend) s << q.second;
            pend.clear();
            s << "        }\n";
        }
    };
    {
        int ci = 0;
        s << "    case " << ci++ << ": {\n";
        emit(std::vector<int>(RR, -1), false);
        s << "    } break;\n";
        auto blockrows = [&](int g) {
            std::vector<int> rows(RR);
            for (int i = 0; i < RR; ++i) rows[i] = g * RR + i < n_a ? g * RR + i : -2;
            return rows;
        };
        for (int g = 0; g < BLO; ++g) {
            s << "    case " << ci++ << ": {\n";
            emit(blockrows(g), true);
            s << "    } break;\n";
        }
        for (int g = BHI; g < nblk; ++g) {
            s << "    case " << ci++ << ": {\n";
            emit(blockrows(g), true);
            s << "    } break;\n";
        }
        s << "    default: break;\n    }\n";
    }
    s << R"(#pragma unroll
    for (int i = 0; i < RR; ++i)
        if (r0 + i < n_a) {
#pragma unroll
            for (int o2 = 0; o2 < NOUT; ++o2) P.out[o2][base + (size_t)(r0 + i) * s_a] = acc[o2][i];
        }
}
)";
    std::unique_ptr<KronJitPass> P(new KronJitPass());
    P->fn = nvrtc_kernel(s.str(), "ks_passc", 48 * 1024);
    P->nin = nin;
    P->nout = nout;
    P->gx = (unsigned)(nqc * n_outer);
    P->gy = (unsigned)nblk;
    return P.release();
}

void kron_jitc_launch(const KronJitPass& J, void* const* hin, void* const* hout, cudaStream_t st) {
    std::vector<void*> par((size_t)J.nin + J.nout);
    for (int g = 0; g < J.nin; ++g) par[g] = hin[g];
    for (int o = 0; o < J.nout; ++o) par[J.nin + o] = hout[o];
    void* args[] = {(void*)par.data()};
    KS_CUDA(cudaLaunchKernel((const void*)J.fn, dim3(J.gx, J.gy), dim3(128), args, 0, st));
    check_launch("ks_passc (jit)");
}

// Tile-variant shapes worth timing for a pass pair, best first by a simple issue model:
// per output point, phase A costs |a| products x the halo factor x the idle-lane factor of its
// row-per-lane mapping, phase B |b| products, each divided by how evenly its work items fill
// the warps between the two CTA barriers; shared-memory operations (4 LSU cycles per 16 B
// warp access against 2 FP64-pipe cycles per DFMA) bound it from below. Constraints:
// registers per thread within the allocation unit of four warps, shared memory for `minb`
// CTAs, one tensor-map box per tile.
std::vector<std::array<int, 6>> kron_jitt_candidates(int bw, int n_a, int n_b, int na_prod, int nb_prod, int nmid, int nout,
                                                     int keep) {
    struct Cand {
        double score;
        std::array<int, 6> c;
    };
    std::vector<Cand> all;
    const int W = 2 * bw + 1;
    for (int RR = 2; RR <= 4; ++RR)
        for (int RB = RR; RB + 2 * bw <= 32; RB += RR)
            for (int RA = 2; RA <= 6; ++RA)
                for (int NAS = 1; NAS <= 4; ++NAS)
                    for (int NW : {4, 8, 12, 16})
                        for (int minb = 1; minb <= 4; ++minb) {
                            if (NW * minb > 16 || NW * minb < 8) continue;
                            const int RBH = RB + 2 * bw;
                            const int AT = ((n_a + NAS - 1) / NAS + RA - 1) / RA * RA;
                            if ((long long)AT * (NAS - 1) >= n_a || AT < 2 * bw) continue;
                            const int PX = (AT + 2 * bw) | 1, PM = AT | 1;
                            if (2 * PX > 256) continue;
                            const size_t smem = ((size_t)RBH * PX + (size_t)nmid * RBH * PM) * 16 + 64;
                            if (smem * minb > 226 * 1024) continue;
                            const int regs = std::max(4 * (RA + 2 * bw) + 4 * nmid * RA, 4 * (RR + 2 * bw) + 4 * nout * RR) + 34;
                            if (regs > std::min(255, 65536 / (minb * NW * 32))) continue;
                            const int ntb = (n_b + RB - 1) / RB;
                            const double eff_rows = (double)n_b / ((double)ntb * RB);
                            double ea = 0, eb = 0; // fill of the warps in phases A / B, averaged over the pieces of axis a
                            for (int as = 0; as < NAS; ++as) {
                                const int nat = std::min(AT, n_a - as * AT);
                                const int nblk = (nat + RA - 1) / RA, items = (RB / RR) * nat;
                                ea += (double)nat / ((double)((nblk + NW - 1) / NW) * NW * RA);
                                eb += (double)items / ((double)((items + 32 * NW - 1) / (32 * NW)) * 32 * NW);
                            }
                            ea /= NAS;
                            eb /= NAS;
                            const double h = (double)RBH / RB;
                            const double fp = 4.0 * W * (na_prod * h * (32.0 / RBH) / ea + nb_prod / eb);
                            const double sm = 4.0 * (((double)(RA + 2 * bw) / RA + nmid) * h * (32.0 / RBH) + (double)nmid * (RR + 2 * bw) / RR);
                            // measured at c3 / c5 (tools/gpu_tile_sweep.sh): two CTAs of eight warps beat four of
                            // four and one of sixteen at equal shapes; every extra piece of axis a costs a few percent
                            const double score = std::max(fp, sm) / eff_rows * (NW == 8 && minb == 2 ? 1.0 : 1.06) * (1.0 + 0.03 * (NAS - 1));
                            all.push_back({score, {RB, RA, RR, NW, minb, NAS}});
                        }
    std::sort(all.begin(), all.end(), [](const Cand& x, const Cand& y) { return x.score < y.score; });
    std::vector<std::array<int, 6>> out;
    for (auto& c : all) {
        if ((int)out.size() >= keep) break;
        out.push_back(c.c);
    }
    if (const char* e = std::getenv("KS_KRON_JIT"); e && std::strcmp(e, "0") != 0 && std::strncmp(e, "dump", 4) != 0)
        for (size_t i = 0; i < out.size(); ++i)
            std::fprintf(stderr, "ks_kron tile shape %zu: RB %d RA %d RR %d warps %d ctas/sm %d pieces %d (score %.1f)\n", i, out[i][0],
                         out[i][1], out[i][2], out[i][3], out[i][4], out[i][5], all[i].score);
    return out;
}

} // namespace ks
