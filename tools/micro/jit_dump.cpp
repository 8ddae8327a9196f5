// Offline generator check (no GPU needed): builds the tile / row-blocked variants of a
// synthetic (t,1)-like pass pair and writes the generated sources (KS_KRON_JIT=dump=<dir>);
// the device query after the dump throws, which is expected here.
//   g++ -std=c++17 -I paper_2311_18461_b200/csrc -I /usr/local/cuda/include tools/micro/jit_dump.cpp \
//       -L paper_2311_18461_b200 -lks -o /tmp/jit_dump && KS_KRON_JIT=dump=/tmp/jit /tmp/jit_dump 4 131 130
#include "ks_internal.hpp"
#include <array>
#include <cstdio>
#include <cstdlib>
#include <random>
using namespace ks;
int main(int argc, char** argv) {
    const int bw = argc > 1 ? atoi(argv[1]) : 2, n_a = argc > 2 ? atoi(argv[2]) : 65, n_b = argc > 3 ? atoi(argv[3]) : 64;
    const int W = 2 * bw + 1, nmax = std::max(n_a, n_b), nf = 6;
    std::vector<double2> rb((size_t)nf * nmax * W, make_double2(0, 0));
    std::mt19937_64 g(1);
    std::uniform_real_distribution<double> U(-1, 1);
    std::vector<int> freal = {1, 1, 1, 1, 1, 2};
    for (int f = 0; f < nf; ++f) {
        const int n = (f == 0 || f == 2 || f == 5) ? n_a : n_b;
        std::vector<double> toe(W);
        for (auto& v : toe) v = U(g);
        for (int r = 0; r < n; ++r)
            for (int k = 0; k < W; ++k) {
                const int c = r + k - bw;
                if (c < 0 || c >= n) continue;
                double v = (r < bw + 1 || r >= n - bw - 1) ? U(g) : toe[k];
                rb[((size_t)f * nmax + r) * W + k] = freal[f] == 2 ? make_double2(0, v) : make_double2(v, 0);
            }
    }
    std::vector<JitContrib> a = {{0, 0, 0, 0}, {0, 1, 2, 1}, {0, 2, 5, 2}};
    std::vector<JitContrib> b = {{0, 0, 1, 3}, {1, 0, 3, 4}, {2, 0, 4, 5}, {1, 1, 1, 6}, {1, 2, 4, 7}, {2, 2, 1, 8}};
    std::vector<double2> co = {{1, 0}, {1, 0}, {1, 0}, {1, 0}, {1, 0}, {-1, 0}, {1, 0}, {2, 0}, {-1, 0}};
    for (auto cfg : kron_jitt_candidates(bw, n_a, n_b, (int)a.size(), (int)b.size(), 3, 3, 3)) {
        try {
            KronJitPair* p = kron_jitt_build(1, 3, 3, bw, a, b, freal, co, n_a, n_b, 4096, rb.data(), nmax, cfg[0], cfg[1], cfg[2], cfg[3], cfg[4], cfg[5]);
            std::printf("cfg %d %d %d %d: %s\n", cfg[0], cfg[3], cfg[4], cfg[5], p ? "built" : "null");
        } catch (const std::exception& e) {
            std::printf("cfg %d %d %d %d: dumped\n", cfg[0], cfg[3], cfg[4], cfg[5]); (void)e;
        }
    }
    try { // the generated single pass over inner columns (three inputs, three outputs)
        kron_jitc_build(3, 3, bw, b, freal, co, 16641, n_b, 1, rb.data(), nmax, 4);
    } catch (const std::exception&) {
        std::printf("single pass: dumped\n");
    }
}
