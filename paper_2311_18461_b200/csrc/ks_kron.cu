// Matrix-free Kronecker-sum operator y = sum_t c_t (F_t,D-1 x ... x F_t,0) x.
//
// Reference: KroneckerOperator::apply (src/tensorops.cpp:236-254) evaluates
// every term separately: per non-identity factor it copies the source tensor
// (:245-247) and runs a banded mode product (:89-123), then axpy's the term
// into y (:252) -- (d^2+d+1)(d+1) full passes for the system matrix A
// (assembly.cpp:202-251): 52 for d = 3.
//
// B200 formulation ("level passes"): process the axes in order; between axes
// the partial results live as a small set of intermediate tensors ("nodes").
// Before a switch axis the nodes are keyed by the factor PREFIX already
// applied (shared prefixes are computed once); after it by the factor SUFFIX
// still to apply (terms with the same suffix are summed before it is
// applied). One kernel per axis reads all nodes of its input level once and
// writes all nodes of its output level once; every output element sums its
// contributions (in-node, banded factor, coefficient) in registers. The
// switch axis is chosen to minimise the tensor traffic sum_levels (|in| +
// |out|). For A at d = 3 the levels are 1 -> 3 -> 7 -> 5 -> 1 tensors,
// 32 x 16 B/DOF, versus 52 x (copy + product + axpy) passes in the reference.
// Any term list (KroneckerOperator::add_term, tensorops.cpp:219-234) is
// accepted -- the plan is derived from the list, not hard-coded for A.
//
// Summation order differs from the reference (factorised sums; merged
// coefficients), which changes results only at rounding level.
#include "ks_internal.hpp"

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstring>
#include <map>
#include <numeric>
#include <cmath>
#include <cstdlib>

namespace ks {

struct SweepEntry {
    int out;    // output node
    int factor; // -1 = identity
    double2 coeff;
};
struct RingCon {
    int in, factor;
    double2 coeff;
};
bool launch_colsweep(int nin, int nout, int bw, const double2* const* ip, double2* const* op,
                     const int* in_begin, const SweepEntry* entries, const double2* rb,
                     const int* freal, size_t ncols, size_t s, int n, int nmax, cudaStream_t st,
                     int nir, int ioff, int boff, const int* ring_begin, const RingCon* ring_cons);

struct KronFactor {
    int n = 0, bw = 0;
    bool is_real = false;
    size_t off = 0; // in complex entries into the band pool
};
struct KronContrib {
    int in;     // node index within the pass's input level
    int factor; // -1 = identity
    double2 coeff;
};
struct KronPass {
    int axis = 0;
    int n_in = 0, n_out = 0;
    std::vector<int> out_begin; // n_out + 1
    std::vector<KronContrib> contribs;
    DevBuf d_begin, d_contribs;
    DevBuf d_in_begin, d_entries; // v3: contributions grouped by input
    DevBuf d_ring;                // ring sweep: contributions grouped by output (RingCon)
    int in_pool = -1, out_pool = -1; // -1 = x / y
};

struct KronPlan {
    std::vector<int> dims;
    size_t N = 0;
    std::vector<KronFactor> factors;
    DevBuf d_factors, d_bands;
    std::vector<KronPass> passes;
    int pool_nodes[2] = {0, 0};
    DevBuf pool[2];
    DevBuf d_ptrs; // per pass: in pointers then out pointers (device table)
    std::vector<size_t> ptr_off;
    int nnodes = 0, nproducts = 0;
    int bwmax = 0, nmax = 1;
    // sharded outermost axis (ks_kronshard_*): the last pass reads the haloed
    // slab (dims.back() rows) and writes shard_rows owned planes
    int shard_rows = 0, shard_in_off = 0, shard_band_off = 0;
    DevBuf d_rowband, d_freal; // v3: rb[f][r][dj] (width 2*bwmax+1), is_real[f]
    // plan-specialised fused pass pairs (k, k+1), indexed by k (null = none)
    std::vector<std::unique_ptr<KronJitPair, KronJitDeleter>> jit;
    // alternative block shapes of each fused pair, timed once on the first
    // apply (the faster one replaces jit[k]); the best shape differs between
    // sizes (c3: 160-thread blocks 0.81 ms vs 352 0.87; c5: 288 beats 160)
    std::vector<std::vector<std::unique_ptr<KronJitPair, KronJitDeleter>>> jit_alt;
    // generated single passes (inner-column axes not covered by a runnable fused pair), indexed by pass
    struct PassDeleter {
        void operator()(KronJitPass* p) const { kron_jitc_free(p); }
    };
    std::vector<std::unique_ptr<KronJitPass, PassDeleter>> passc;
    // device pointer tables per (x, y) pair (kron_apply)
    std::map<std::pair<const void*, void*>, DevBuf> ptr_tables;
};

namespace {

struct DevFactor {
    int n, bw, is_real, pad;
    unsigned long long off;
};

// Kernel: one thread per tensor element; all outputs of the level.
__global__ void __launch_bounds__(256) k_kron_level(
    const double2* const* __restrict__ in_ptrs, double2* const* __restrict__ out_ptrs, int n_out,
    const int* __restrict__ out_begin, const KronContrib* __restrict__ contribs,
    const DevFactor* __restrict__ factors, const double2* __restrict__ bands, size_t N,
    size_t s, int n) {
    const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= N) return;
    const size_t q = idx % s;
    const size_t t = idx / s;
    const int r = (int)(t % (size_t)n);
    const size_t o = t / (size_t)n;
    const size_t base = o * (size_t)n * s + q;
    for (int oi = 0; oi < n_out; ++oi) {
        double ar = 0.0, ai = 0.0;
        const int cb = out_begin[oi], ce = out_begin[oi + 1];
        for (int ci = cb; ci < ce; ++ci) {
            const KronContrib c = contribs[ci];
            const double2* __restrict__ in = in_ptrs[c.in];
            double vr, vi;
            if (c.factor < 0) {
                const double2 v = in[idx];
                vr = v.x;
                vi = v.y;
            } else {
                const DevFactor f = factors[c.factor];
                const int bw = f.bw;
                const int j0 = r - bw < 0 ? 0 : r - bw;
                const int j1 = r + bw > n - 1 ? n - 1 : r + bw;
                const double2* band = bands + f.off;
                const int ld = 2 * bw + 1;
                vr = 0.0;
                vi = 0.0;
                if (f.is_real) {
                    for (int j = j0; j <= j1; ++j) {
                        const double a = band[bw + r - j + j * ld].x;
                        const double2 v = __ldg(in + base + (size_t)j * s);
                        vr = fma(a, v.x, vr);
                        vi = fma(a, v.y, vi);
                    }
                } else {
                    for (int j = j0; j <= j1; ++j) {
                        const double2 a = band[bw + r - j + j * ld];
                        const double2 v = __ldg(in + base + (size_t)j * s);
                        vr = fma(a.x, v.x, fma(-a.y, v.y, vr));
                        vi = fma(a.x, v.y, fma(a.y, v.x, vi));
                    }
                }
            }
            if (c.coeff.y == 0.0) {
                ar = fma(c.coeff.x, vr, ar);
                ai = fma(c.coeff.x, vi, ai);
            } else {
                ar = fma(c.coeff.x, vr, fma(-c.coeff.y, vi, ar));
                ai = fma(c.coeff.x, vi, fma(c.coeff.y, vr, ai));
            }
        }
        out_ptrs[oi][idx] = make_double2(ar, ai);
    }
}

// ---------------------------------------------------------------------------
// Level pass v3 ("row-chunk sweep"): a thread owns one column (o, q) and a
// chunk of kR consecutive rows r along the pass axis. For each input node it
// loads the kR + 2*BW window once into registers, applies every factor that
// reads this input (contributions grouped by input on the host) and adds the
// results into the per-output accumulators through a uniform switch, so all
// register indices are static. Threads are ordered column-fastest for s > 1
// (coalesced along q) and chunk-fastest for the contiguous time axis s = 1.
// Bands are pre-expanded row-major: rb[f][r][dj] = F(r, r + dj - BW).
// ---------------------------------------------------------------------------
constexpr int kR = 4;
constexpr int kMaxOut = 8;

template <int NOUT, int BW>
__global__ void __launch_bounds__(256) k_kron_sweep(
    const double2* const* __restrict__ in_ptrs, int n_in, double2* const* __restrict__ out_ptrs,
    const int* __restrict__ in_begin, const SweepEntry* __restrict__ entries,
    const double2* __restrict__ rb, const int* __restrict__ freal, size_t ncols, size_t s, int n,
    int nmax) {
    constexpr int W = kR + 2 * BW, TAPS = 2 * BW + 1;
    const int nch = (n + kR - 1) / kR;
    const size_t gid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (gid >= ncols * (size_t)nch) return;
    size_t col;
    int ch;
    if (s == 1) {
        col = gid / nch;
        ch = (int)(gid - col * nch);
    } else {
        ch = (int)(gid / ncols);
        col = gid - (size_t)ch * ncols;
    }
    const int r0 = ch * kR;
    const size_t o = col / s, q = col - o * s;
    const size_t base = o * (size_t)n * s + q;

    double2 acc[NOUT][kR];
#pragma unroll
    for (int a = 0; a < NOUT; ++a)
#pragma unroll
        for (int k = 0; k < kR; ++k) acc[a][k] = make_double2(0.0, 0.0);

    for (int ii = 0; ii < n_in; ++ii) {
        const double2* __restrict__ in = in_ptrs[ii];
        double2 w[W];
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int r = r0 - BW + k;
            w[k] = (r >= 0 && r < n) ? __ldg(in + base + (size_t)r * s) : make_double2(0.0, 0.0);
        }
        const int eb = in_begin[ii], ee = in_begin[ii + 1];
        for (int e = eb; e < ee; ++e) {
            const SweepEntry en = entries[e];
            double2 v[kR];
            if (en.factor < 0) {
#pragma unroll
                for (int k = 0; k < kR; ++k) v[k] = w[k + BW];
            } else {
                const double2* band = rb + (size_t)en.factor * nmax * TAPS;
                if (freal[en.factor]) {
#pragma unroll
                    for (int k = 0; k < kR; ++k) {
                        const int r = min(r0 + k, n - 1);
                        double vr = 0.0, vi = 0.0;
#pragma unroll
                        for (int t = 0; t < TAPS; ++t) {
                            const double a = __ldg(&band[(size_t)r * TAPS + t].x);
                            vr = fma(a, w[k + t].x, vr);
                            vi = fma(a, w[k + t].y, vi);
                        }
                        v[k] = make_double2(vr, vi);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < kR; ++k) {
                        const int r = min(r0 + k, n - 1);
                        double vr = 0.0, vi = 0.0;
#pragma unroll
                        for (int t = 0; t < TAPS; ++t) {
                            const double2 a = __ldg(&band[(size_t)r * TAPS + t]);
                            vr = fma(a.x, w[k + t].x, fma(-a.y, w[k + t].y, vr));
                            vi = fma(a.x, w[k + t].y, fma(a.y, w[k + t].x, vi));
                        }
                        v[k] = make_double2(vr, vi);
                    }
                }
            }
            const double cr = en.coeff.x, ci = en.coeff.y;
            switch (en.out) {
#define KS_ACC(OO)                                                                 \
    case OO:                                                                       \
        if (OO < NOUT) {                                                           \
            _Pragma("unroll") for (int k = 0; k < kR; ++k) {                       \
                double2& A = acc[OO < NOUT ? OO : 0][k];                           \
                A.x = fma(cr, v[k].x, fma(-ci, v[k].y, A.x));                      \
                A.y = fma(cr, v[k].y, fma(ci, v[k].x, A.y));                       \
            }                                                                      \
        }                                                                          \
        break;
                KS_ACC(0) KS_ACC(1) KS_ACC(2) KS_ACC(3) KS_ACC(4) KS_ACC(5) KS_ACC(6) KS_ACC(7)
#undef KS_ACC
            }
        }
    }
#pragma unroll
    for (int a = 0; a < NOUT; ++a) {
        double2* __restrict__ out = out_ptrs[a];
#pragma unroll
        for (int k = 0; k < kR; ++k)
            if (r0 + k < n) out[base + (size_t)(r0 + k) * s] = acc[a][k];
    }
}

} // namespace

// Build the plan. terms: coeff + per-axis factor id (-1 identity).
KronPlan* kron_plan(const std::vector<int>& dims,
                                    const std::vector<std::vector<double2>>& bands,
                                    const std::vector<int>& band_n, const std::vector<int>& band_bw,
                                    const std::vector<double2>& coeffs,
                                    const std::vector<std::vector<int>>& fids) {
    auto P = std::make_unique<KronPlan>();
    const int D = (int)dims.size();
    P->dims = dims;
    P->N = 1;
    for (int v : dims) P->N *= (size_t)v;
    // factor table + device band pool
    std::vector<double2> pool;
    for (size_t f = 0; f < bands.size(); ++f) {
        KronFactor kf;
        kf.n = band_n[f];
        kf.bw = band_bw[f];
        kf.off = pool.size();
        kf.is_real = true;
        for (const double2& v : bands[f])
            if (v.y != 0.0) kf.is_real = false;
        pool.insert(pool.end(), bands[f].begin(), bands[f].end());
        P->factors.push_back(kf);
    }
    std::vector<DevFactor> dfs;
    for (auto& f : P->factors) dfs.push_back({f.n, f.bw, f.is_real ? 1 : 0, 0, f.off});
    if (!dfs.empty()) {
        P->d_factors.alloc(dfs.size() * sizeof(DevFactor));
        KS_CUDA(cudaMemcpy(P->d_factors.p, dfs.data(), dfs.size() * sizeof(DevFactor),
                           cudaMemcpyHostToDevice));
    }
    if (!pool.empty()) {
        P->d_bands.alloc(pool.size() * sizeof(double2));
        KS_CUDA(cudaMemcpy(P->d_bands.p, pool.data(), pool.size() * sizeof(double2),
                           cudaMemcpyHostToDevice));
    }

    const int T = (int)coeffs.size();
    // active axes: some term has a non-identity factor
    std::vector<int> ax;
    for (int a = 0; a < D; ++a) {
        bool any = false;
        for (int t = 0; t < T; ++t) any |= fids[t][a] >= 0;
        if (any) ax.push_back(a);
    }
    if (ax.empty()) ax.push_back(0);
    const int L = (int)ax.size();

    using Key = std::vector<int>;
    auto prefix_key = [&](int t, int b) {
        Key k;
        for (int i = 0; i < b; ++i) k.push_back(fids[t][ax[i]]);
        return k;
    };
    auto suffix_key = [&](int t, int b) {
        Key k;
        for (int i = b; i < L; ++i) k.push_back(fids[t][ax[i]]);
        return k;
    };
    // node maps per boundary for a given switch s
    auto boundary_nodes = [&](int s, int b, std::vector<int>& node_of_term) {
        std::map<Key, int> m;
        node_of_term.assign(T, 0);
        if (T == 0) return 0;
        for (int t = 0; t < T; ++t) {
            Key k = (b <= s) ? prefix_key(t, b) : suffix_key(t, b);
            auto it = m.find(k);
            if (it == m.end()) it = m.emplace(k, (int)m.size()).first;
            node_of_term[t] = it->second;
        }
        return (int)m.size();
    };
    // Rank-revealing merge of the boundary after the switch pass s: the suffix
    // nodes q there receive sum_{(in, f)} C[q][(in, f)] F_f(in) from pass s.
    // Nodes whose rows C[q] are proportional (C[q] = scale_q * R_g) become one
    // intermediate U_g = sum R_g[(in, f)] F_f(in), and the pass after the
    // switch reads scale_q * U_g. For the system operator at d = 3 the 6
    // suffix classes (f2, f3) collapse to 3 (rank of C; e.g. (L,M) and (M,L)
    // get the same row from the W and the cross terms), so the fused pass
    // pairs write / read 3 intermediate tensors instead of 6.
    const bool merge_rows = [] {
        const char* e = std::getenv("KS_KRON_RANK");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    auto merge_boundary = [&](int s, const std::vector<int>& nin, const std::vector<int>& nout, int nq,
                              std::vector<int>& grp, std::vector<double2>& scale, std::vector<char>& is_rep) -> int {
        grp.resize(nq);
        scale.assign(nq, make_double2(1.0, 0.0));
        is_rep.assign(nq, 1);
        for (int q = 0; q < nq; ++q) grp[q] = q;
        if (!merge_rows || s + 1 >= L || nq <= 1) return nq;
        std::vector<std::map<std::pair<int, int>, double2>> row(nq);
        for (int t = 0; t < T; ++t) {
            auto& e = row[nout[t]][std::make_pair(nin[t], fids[t][ax[s]])];
            e.x += coeffs[t].x;
            e.y += coeffs[t].y;
        }
        auto cdivd = [](double2 a, double2 b) {
            const double den = b.x * b.x + b.y * b.y;
            return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
        };
        std::vector<int> rep; // representative node of each group
        int ng = 0;
        for (int q = 0; q < nq; ++q) {
            if (row[q].empty()) continue;
            const double2 lead = row[q].begin()->second;
            if (lead.x == 0.0 && lead.y == 0.0) continue;
            int found = -1;
            for (int g = 0; g < ng && found < 0; ++g) {
                const auto& r0 = row[rep[g]];
                if (r0.size() != row[q].size()) continue;
                const double2 l0 = r0.begin()->second;
                const double2 sc = cdivd(lead, l0); // row q = sc * row rep
                bool same = true;
                const auto& rq = row[q];
                auto jt = r0.begin();
                for (auto it = rq.begin(); it != rq.end() && same; ++it, ++jt) {
                    if (it->first != jt->first) {
                        same = false;
                        break;
                    }
                    const double2 v = jt->second;
                    const double2 pr = make_double2(sc.x * v.x - sc.y * v.y, sc.x * v.y + sc.y * v.x);
                    const double mag = std::max(std::hypot(it->second.x, it->second.y), std::hypot(pr.x, pr.y));
                    same = std::hypot(it->second.x - pr.x, it->second.y - pr.y) <= 1e-12 * mag;
                }
                if (same) {
                    found = g;
                    scale[q] = sc;
                    is_rep[q] = 0;
                }
            }
            if (found < 0) {
                rep.push_back(q);
                found = ng++;
            }
            grp[q] = found;
        }
        // nodes with an all-zero row keep their own group (nothing flows in)
        for (int q = 0; q < nq; ++q)
            if (row[q].empty() || (row[q].begin()->second.x == 0.0 && row[q].begin()->second.y == 0.0)) grp[q] = ng++;
        return ng;
    };
    int best_s = 0;
    long best_cost = -1;
    for (int s = 0; s < L; ++s) {
        long cost = 0;
        std::vector<int> tmp;
        std::vector<int> cnt(L + 1);
        std::vector<std::vector<int>> nb(L + 1);
        for (int b = 0; b <= L; ++b) cnt[b] = boundary_nodes(s, b, nb[b]);
        cnt[0] = 1;
        cnt[L] = 1;
        if (s + 1 < L) {
            std::vector<int> g;
            std::vector<double2> sc;
            std::vector<char> rp;
            std::vector<int> n0(T, 0);
            cnt[s + 1] = merge_boundary(s, s == 0 ? n0 : nb[s], nb[s + 1], cnt[s + 1], g, sc, rp);
        }
        for (int k = 0; k < L; ++k) cost += cnt[k] + cnt[k + 1];
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best_s = s;
        }
    }
    const int s = best_s;
    std::vector<std::vector<int>> node_of(L + 1);
    std::vector<int> cnt(L + 1);
    for (int b = 0; b <= L; ++b) cnt[b] = boundary_nodes(s, b, node_of[b]);
    cnt[0] = 1;
    cnt[L] = 1;
    for (int t = 0; t < T; ++t) {
        node_of[0][t] = 0;
        node_of[L][t] = 0;
    }
    // merged boundary after the switch pass: node -> group, with the scale the
    // following pass applies
    std::vector<double2> tscale(T, make_double2(1.0, 0.0));
    std::vector<char> tsrc(T, 1); // term feeds its merged node in the switch pass (representative rows only)
    if (s + 1 < L) {
        std::vector<int> g;
        std::vector<double2> sc;
        std::vector<char> rp;
        cnt[s + 1] = merge_boundary(s, node_of[s], node_of[s + 1], cnt[s + 1], g, sc, rp);
        for (int t = 0; t < T; ++t) {
            tscale[t] = sc[node_of[s + 1][t]];
            tsrc[t] = rp[node_of[s + 1][t]];
            node_of[s + 1][t] = g[node_of[s + 1][t]];
        }
    }
    P->nnodes = 0;
    for (int b = 1; b < L; ++b) P->nnodes += cnt[b];

    for (int k = 0; k < L; ++k) {
        KronPass ps;
        ps.axis = ax[k];
        ps.n_in = cnt[k];
        ps.n_out = cnt[k + 1];
        // (out, in, factor) -> coeff
        std::map<std::tuple<int, int, int>, double2> acc;
        for (int t = 0; t < T; ++t) {
            if (k == s && !tsrc[t]) continue; // merged node: defined by its representative's row
            const int in = node_of[k][t], out = node_of[k + 1][t], f = fids[t][ax[k]];
            // switch pass: the term's coefficient over its merged node's scale;
            // the pass after it: the scale (one value per (out, in, f): see above)
            double2 c = make_double2(1.0, 0.0);
            if (k == s) {
                const double2 a = coeffs[t], b = tscale[t];
                const double den = b.x * b.x + b.y * b.y;
                c = make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
            } else if (k == s + 1) {
                c = tscale[t];
            }
            auto key = std::make_tuple(out, in, f);
            auto it = acc.find(key);
            if (it == acc.end()) {
                acc.emplace(key, c);
            } else if (k == s) {
                it->second.x += c.x;
                it->second.y += c.y;
            }
        }
        ps.out_begin.assign(ps.n_out + 1, 0);
        for (auto& kv : acc) ps.out_begin[std::get<0>(kv.first) + 1]++;
        for (int o = 0; o < ps.n_out; ++o) ps.out_begin[o + 1] += ps.out_begin[o];
        ps.contribs.resize(acc.size());
        std::vector<int> fill(ps.out_begin.begin(), ps.out_begin.end() - 1);
        for (auto& kv : acc) {
            const int o = std::get<0>(kv.first);
            ps.contribs[fill[o]++] = KronContrib{std::get<1>(kv.first), std::get<2>(kv.first), kv.second};
            if (std::get<2>(kv.first) >= 0) P->nproducts++;
        }
        ps.in_pool = (k == 0) ? -1 : ((k - 1) & 1);
        ps.out_pool = (k == L - 1) ? -1 : (k & 1);
        if (ps.out_pool >= 0)
            P->pool_nodes[ps.out_pool] = std::max(P->pool_nodes[ps.out_pool], ps.n_out);
        ps.d_begin.alloc(ps.out_begin.size() * sizeof(int));
        KS_CUDA(cudaMemcpy(ps.d_begin.p, ps.out_begin.data(), ps.out_begin.size() * sizeof(int),
                           cudaMemcpyHostToDevice));
        if (!ps.contribs.empty()) {
            ps.d_contribs.alloc(ps.contribs.size() * sizeof(KronContrib));
            KS_CUDA(cudaMemcpy(ps.d_contribs.p, ps.contribs.data(),
                               ps.contribs.size() * sizeof(KronContrib), cudaMemcpyHostToDevice));
        }
        P->passes.push_back(std::move(ps));
    }
    // v3 tables: row-major bands padded to the widest bandwidth
    for (auto& f : P->factors) P->bwmax = std::max(P->bwmax, f.bw);
    {
        const int taps = 2 * P->bwmax + 1;
        size_t tot = 0;
        std::vector<size_t> foff;
        for (auto& f : P->factors) {
            foff.push_back(tot);
            tot += (size_t)f.n * taps;
        }
        // all factors of one axis share n, but pool offsets are per factor: store
        // each factor at f * nmax * taps so the kernel indexes by factor id
        int nmax = 1;
        for (auto& f : P->factors) nmax = std::max(nmax, f.n);
        std::vector<double2> rb((size_t)std::max<size_t>(P->factors.size(), 1) * nmax * taps,
                                make_double2(0, 0));
        std::vector<int> freal(std::max<size_t>(P->factors.size(), 1), 1);
        for (size_t fi = 0; fi < P->factors.size(); ++fi) {
            const KronFactor& f = P->factors[fi];
            freal[fi] = f.is_real ? 1 : 0;
            for (int r = 0; r < f.n; ++r)
                for (int dj = -f.bw; dj <= f.bw; ++dj) {
                    const int j = r + dj;
                    if (j < 0 || j >= f.n) continue;
                    rb[(fi * nmax + r) * taps + (dj + P->bwmax)] =
                        pool[f.off + (size_t)(f.bw + r - j) + (size_t)j * (2 * f.bw + 1)];
                }
        }
        P->nmax = nmax;
        P->d_rowband.alloc(rb.size() * sizeof(double2));
        KS_CUDA(cudaMemcpy(P->d_rowband.p, rb.data(), rb.size() * sizeof(double2), cudaMemcpyHostToDevice));
        P->d_freal.alloc(freal.size() * sizeof(int));
        KS_CUDA(cudaMemcpy(P->d_freal.p, freal.data(), freal.size() * sizeof(int), cudaMemcpyHostToDevice));
        // fused pass pairs (0,1), (2,3), ... specialised with NVRTC
        P->jit.resize(P->passes.size());
        P->jit_alt.resize(P->passes.size());
        // factor classes: 1 real, 2 purely imaginary (e.g. W + W^H), 0 complex
        std::vector<int> frv(P->factors.size());
        for (size_t f = 0; f < P->factors.size(); ++f) {
            const KronFactor& kf = P->factors[f];
            bool imag = !kf.is_real;
            for (size_t e = 0; e < (size_t)kf.n * (2 * kf.bw + 1) && imag; ++e) imag = pool[kf.off + e].x == 0.0;
            frv[f] = kf.is_real ? 1 : (imag ? 2 : 0);
        }
        for (size_t k = 0; k + 1 < P->passes.size(); k += 2) {
            const KronPass &pa = P->passes[k], &pb = P->passes[k + 1];
            if (pb.axis != pa.axis + 1 || pb.n_in != pa.n_out) break;
            std::vector<JitContrib> ca, cb;
            std::vector<double2> co;
            for (int o = 0; o < pa.n_out; ++o)
                for (int ci = pa.out_begin[o]; ci < pa.out_begin[o + 1]; ++ci) {
                    ca.push_back(JitContrib{pa.contribs[ci].in, o, pa.contribs[ci].factor, (int)co.size()});
                    co.push_back(pa.contribs[ci].coeff);
                }
            for (int o = 0; o < pb.n_out; ++o)
                for (int ci = pb.out_begin[o]; ci < pb.out_begin[o + 1]; ++ci) {
                    cb.push_back(JitContrib{pb.contribs[ci].in, o, pb.contribs[ci].factor, (int)co.size()});
                    co.push_back(pb.contribs[ci].coeff);
                }
            size_t sa = 1;
            for (int x = 0; x < pa.axis; ++x) sa *= (size_t)P->dims[x];
            const int na = P->dims[pa.axis], nbb = P->dims[pb.axis];
            const long long outer = (long long)(P->N / (sa * (size_t)na * (size_t)nbb));
            P->jit[k].reset(kron_jit_build(pa.n_in, pa.n_out, pb.n_out, P->bwmax, ca, cb, frv, co, (long long)sa, na,
                                           nbb, outer));
            // (alternative block shapes of the thread-per-point kernel only where neither tensor-map fed
            // variant applies: they never won against those, and every candidate costs an NVRTC compile)
            const bool fed = (sa >= 32 && P->bwmax <= 4) || (sa == 1 && pa.n_in == 1 && P->bwmax <= 6);
            if (P->jit[k] && !fed)
                for (int tm : {192, 128}) {
                    std::unique_ptr<KronJitPair, KronJitDeleter> alt(kron_jit_build(
                        pa.n_in, pa.n_out, pb.n_out, P->bwmax, ca, cb, frv, co, (long long)sa, na, nbb, outer, tm));
                    bool dup = !alt || kron_jit_same_shape(*alt, *P->jit[k]);
                    for (auto& o : P->jit_alt[k]) dup = dup || kron_jit_same_shape(*alt, *o);
                    if (!dup) P->jit_alt[k].push_back(std::move(alt));
                }
            // row-blocked candidates (inner columns across the lanes); the first
            // apply times all candidates and keeps the fastest
            if (P->jit[k] && sa >= 32)
                for (int rr : {2}) { // (3 rows: c3 197 vs 189 us, c5 8.2 vs 6.1 ms; 4 rows: on par at c3, spills at bw = 4)
                    // {warp count aligned to the register allocation unit, shifted window}: the window shifted by
                    // register moves needs one copy of the push code instead of 2 bw + 1 rotated ones -- at bw = 4
                    // the copies made the hot loop ~34 KB and the kernel instruction-fetch bound (c5: 6.09 ->
                    // 4.51 ms with the shift); at bw = 2 the rotated copies are faster (c3: 189 vs 197 us)
                    for (auto v : {std::array<bool, 2>{false, false}, std::array<bool, 2>{true, false},
                                   std::array<bool, 2>{false, true}, std::array<bool, 2>{true, true}}) {
                        if (P->bwmax >= 4 && !v[1]) continue;
                        std::unique_ptr<KronJitPair, KronJitDeleter> alt(kron_jitb_build(
                            pa.n_in, pa.n_out, pb.n_out, P->bwmax, ca, cb, frv, co, (long long)sa, na, nbb, outer, rb.data(),
                            nmax, rr, v[0], v[1]));
                        if (alt) P->jit_alt[k].push_back(std::move(alt));
                    }
                    // four rows per thread with the shifted window where the registers allow it (bw <= 2): c3 182 vs
                    // 188 us (at bw = 4: three rows 5.14 ms, four 5.55 ms against 4.50 ms for two)
                    if (P->bwmax <= 2) {
                        std::unique_ptr<KronJitPair, KronJitDeleter> alt(kron_jitb_build(
                            pa.n_in, pa.n_out, pb.n_out, P->bwmax, ca, cb, frv, co, (long long)sa, na, nbb, outer, rb.data(), nmax,
                            4, true, true));
                        if (!alt) alt.reset(kron_jitb_build(pa.n_in, pa.n_out, pb.n_out, P->bwmax, ca, cb, frv, co, (long long)sa, na,
                                                            nbb, outer, rb.data(), nmax, 4, false, true));
                        if (alt) P->jit_alt[k].push_back(std::move(alt));
                    }
                }
            if (P->jit[k] && sa == 1 && pa.n_in == 1)
                // tile variant: {rows per tile, entries / rows per thread in phases A / B, warps, CTAs per SM}
                for (auto cfg : [&] {
                         // KS_KRON_TILE="RB,RA,RR,warps,ctas,pieces;...": explicit tile shapes (sweeps)
                         std::vector<std::array<int, 6>> v;
                         if (const char* e = std::getenv("KS_KRON_TILE")) {
                             std::array<int, 6> c{};
                             int k = 0, cur = 0;
                             for (const char* q = e;; ++q) {
                                 if (*q >= '0' && *q <= '9') cur = cur * 10 + (*q - '0');
                                 else {
                                     if (k < 6) c[k++] = cur;
                                     cur = 0;
                                     if (*q == ';' || *q == 0) {
                                         if (k == 6) v.push_back(c);
                                         k = 0;
                                     }
                                     if (*q == 0) break;
                                 }
                             }
                             return v;
                         }
                         return kron_jitt_candidates(P->bwmax, na, nbb, (int)ca.size(), (int)cb.size(), pa.n_out, pb.n_out, 2);
                     }()) {
                    std::unique_ptr<KronJitPair, KronJitDeleter> alt(
                        kron_jitt_build(pa.n_in, pa.n_out, pb.n_out, P->bwmax, ca, cb, frv, co, na, nbb, outer, rb.data(), nmax,
                                        cfg[0], cfg[1], cfg[2], cfg[3], cfg[4], cfg[5]));
                    if (alt) P->jit_alt[k].push_back(std::move(alt));
                }
            // a candidate whose grid cannot fill the GPU never runs (kron_jit_runs): drop those, and let a
            // runnable alternative take the place of a primary that is not (d = 2: the thread-per-point kernel
            // has one CTA per two lines of axis 2 -- 65 CTAs at c4 -- while the tile kernel has 774 tiles)
            if (P->jit[k]) {
                auto& alts = P->jit_alt[k];
                alts.erase(std::remove_if(alts.begin(), alts.end(), [](const auto& a) { return !kron_jit_runs(*a); }), alts.end());
                if (!kron_jit_runs(*P->jit[k]) && !alts.empty()) {
                    std::swap(P->jit[k], alts.back());
                    alts.pop_back();
                }
            }
        }
        // passes over inner columns that no runnable pair covers (d = 2: the trailing axis-2 pass): generated
        // single-pass kernel with literal bands
        P->passc.resize(P->passes.size());
        std::vector<bool> covered(P->passes.size(), false);
        for (size_t k = 0; k + 1 < P->passes.size(); ++k)
            if (P->jit[k] && kron_jit_runs(*P->jit[k])) covered[k] = covered[k + 1] = true;
        for (size_t k = 0; k < P->passes.size(); ++k) {
            if (covered[k]) continue;
            const KronPass& ps = P->passes[k];
            size_t sa = 1;
            for (int x = 0; x < ps.axis; ++x) sa *= (size_t)P->dims[x];
            if (sa < 32) continue;
            std::vector<JitContrib> cc;
            std::vector<double2> co;
            for (int o = 0; o < ps.n_out; ++o)
                for (int ci = ps.out_begin[o]; ci < ps.out_begin[o + 1]; ++ci) {
                    cc.push_back(JitContrib{ps.contribs[ci].in, o, ps.contribs[ci].factor, (int)co.size()});
                    co.push_back(ps.contribs[ci].coeff);
                }
            const int na = P->dims[ps.axis];
            P->passc[k].reset(kron_jitc_build(ps.n_in, ps.n_out, P->bwmax, cc, frv, co, (long long)sa, na,
                                              (long long)(P->N / (sa * (size_t)na)), rb.data(), nmax, 4));
        }
    }
    for (auto& ps : P->passes) {
        std::vector<int> ib(ps.n_in + 1, 0);
        for (auto& c : ps.contribs) ib[c.in + 1]++;
        for (int i = 0; i < ps.n_in; ++i) ib[i + 1] += ib[i];
        std::vector<SweepEntry> ent(ps.contribs.size());
        std::vector<int> fill(ib.begin(), ib.end() - 1);
        for (int o = 0; o < ps.n_out; ++o)
            for (int ci = ps.out_begin[o]; ci < ps.out_begin[o + 1]; ++ci) {
                const KronContrib& c = ps.contribs[ci];
                ent[fill[c.in]++] = SweepEntry{o, c.factor, c.coeff};
            }
        {
            std::vector<RingCon> rc;
            bool fits = ps.n_out <= 8;
            for (int o = 0; o < ps.n_out; ++o) {
                if (ps.out_begin[o + 1] - ps.out_begin[o] > 12) fits = false;
                for (int ci = ps.out_begin[o]; ci < ps.out_begin[o + 1]; ++ci)
                    rc.push_back(RingCon{ps.contribs[ci].in, ps.contribs[ci].factor, ps.contribs[ci].coeff});
            }
            if (fits && !rc.empty()) {
                ps.d_ring.alloc(rc.size() * sizeof(RingCon));
                KS_CUDA(cudaMemcpy(ps.d_ring.p, rc.data(), rc.size() * sizeof(RingCon), cudaMemcpyHostToDevice));
            }
        }
        ps.d_in_begin.alloc(ib.size() * sizeof(int));
        KS_CUDA(cudaMemcpy(ps.d_in_begin.p, ib.data(), ib.size() * sizeof(int), cudaMemcpyHostToDevice));
        if (!ent.empty()) {
            ps.d_entries.alloc(ent.size() * sizeof(SweepEntry));
            KS_CUDA(cudaMemcpy(ps.d_entries.p, ent.data(), ent.size() * sizeof(SweepEntry),
                               cudaMemcpyHostToDevice));
        }
    }
    // level pools are allocated on first use (kron_apply): with fused pass pairs
    // the middle levels never exist in HBM (c5: 23 GB not allocated)
    // pointer tables: filled per apply (x / y change); reserve device space
    size_t total = 0;
    for (auto& ps : P->passes) {
        P->ptr_off.push_back(total);
        total += ps.n_in + ps.n_out;
    }
    P->d_ptrs.alloc(std::max<size_t>(total, 1) * sizeof(void*));
    return P.release();
}

int kron_plan_engine(const KronPlan& P) {
    for (auto& j : P.jit)
        if (j && kron_jit_runs(*j)) return 1;
    return 0;
}

void kron_plan_info(const KronPlan& P, int* npasses, int* nnodes, int* nproducts) {
    if (npasses) *npasses = (int)P.passes.size();
    if (nnodes) *nnodes = P.nnodes;
    if (nproducts) *nproducts = P.nproducts;
}

void kron_apply(KronPlan& P, const double2* x, double2* y, cudaStream_t st,
                std::vector<void*>& host_ptrs) {
    // which passes run fused (same decision as the dispatch below): allocate only
    // the level pools that some launch reads or writes
    auto fused_at = [&](size_t k) {
        return k < P.jit.size() && P.jit[k] && !(P.shard_rows > 0 && k + 2 == P.passes.size()) &&
               kron_jit_runs(*P.jit[k]);
    };
    bool need[2] = {false, false};
    for (size_t k = 0; k < P.passes.size();) {
        const bool f = fused_at(k);
        const KronPass& a = P.passes[k];
        const KronPass& b = P.passes[f ? k + 1 : k];
        if (a.in_pool >= 0) need[a.in_pool] = true;
        if (b.out_pool >= 0) need[b.out_pool] = true;
        k += f ? 2 : 1;
    }
    for (int pl = 0; pl < 2; ++pl)
        if (need[pl] && P.pool_nodes[pl] > 0 && !P.pool[pl].p)
            P.pool[pl].alloc((size_t)P.pool_nodes[pl] * P.N * sizeof(double2));
    // pointer table (host-staged, one async copy per apply)
    size_t total = 0;
    for (auto& ps : P.passes) total += ps.n_in + ps.n_out;
    host_ptrs.resize(total);
    size_t w = 0;
    auto pool_ptr = [&](int pl, int i) -> void* {
        return P.pool[pl].p ? (void*)(P.pool[pl].as<double2>() + (size_t)i * P.N) : nullptr;
    };
    for (auto& ps : P.passes) {
        for (int i = 0; i < ps.n_in; ++i) host_ptrs[w++] = ps.in_pool < 0 ? (void*)x : pool_ptr(ps.in_pool, i);
        for (int i = 0; i < ps.n_out; ++i) host_ptrs[w++] = ps.out_pool < 0 ? (void*)y : pool_ptr(ps.out_pool, i);
    }
    // one device copy of the table per (x, y) pair, uploaded on first use: later
    // applies with the same vectors issue no host->device copy (so a CUDA graph
    // can capture them, ks_pcg)
    auto key = std::make_pair((const void*)x, (void*)y);
    auto it = P.ptr_tables.find(key);
    if (it == P.ptr_tables.end()) {
        if (P.ptr_tables.size() >= 4096) { // bounded: callers cycling through many vectors
            KS_CUDA(cudaStreamSynchronize(st));
            P.ptr_tables.clear();
        }
        it = P.ptr_tables.emplace(key, DevBuf(std::max<size_t>(total, 1) * sizeof(void*))).first;
        KS_CUDA(cudaMemcpyAsync(it->second.p, host_ptrs.data(), total * sizeof(void*), cudaMemcpyHostToDevice, st));
    }
    const void* const* dp = static_cast<const void* const*>(it->second.p);
    for (size_t k = 0; k < P.passes.size(); ++k) {
        const KronPass& ps = P.passes[k];
        size_t s = 1;
        for (int a = 0; a < ps.axis; ++a) s *= (size_t)P.dims[a];
        const int n = P.dims[ps.axis];
        const bool shard_last = P.shard_rows > 0 && k + 1 == P.passes.size() &&
                                ps.axis == (int)P.dims.size() - 1;
        // plan-specialised fused pair (NVRTC): the middle level stays on chip
        if (fused_at(k)) {
            const KronPass& nx = P.passes[k + 1];
            auto ip = reinterpret_cast<const double2* const*>(dp + P.ptr_off[k]);
            auto op = reinterpret_cast<double2* const*>(const_cast<void**>(dp + P.ptr_off[k + 1] + nx.n_in));
            if (k < P.jit_alt.size() && !P.jit_alt[k].empty()) {
                // first apply: time the current shape and the alternatives once, keep the fastest
                auto time_one = [&](KronJitPair& J) {
                    cudaEvent_t a, b;
                    KS_CUDA(cudaEventCreate(&a));
                    KS_CUDA(cudaEventCreate(&b));
                    KS_CUDA(cudaEventRecord(a, st));
                    const bool ok = kron_jit_launch(J, ip, op, host_ptrs.data() + P.ptr_off[k],
                                                    host_ptrs.data() + P.ptr_off[k + 1] + nx.n_in,
                                                    P.d_rowband.as<double2>(), P.nmax, st);
                    KS_CUDA(cudaEventRecord(b, st));
                    KS_CUDA(cudaEventSynchronize(b));
                    float ms = 0.f;
                    KS_CUDA(cudaEventElapsedTime(&ms, a, b));
                    cudaEventDestroy(a);
                    cudaEventDestroy(b);
                    return ok ? ms : 1e30f;
                };
                // three interleaved rounds, best of each candidate (single launches
                // of ~0.3 ms differ by a few percent from run to run)
                time_one(*P.jit[k]); // warm-up launches (lazy module loading, L2)
                for (auto& alt : P.jit_alt[k]) time_one(*alt);
                std::vector<float> tb(P.jit_alt[k].size() + 1, 1e30f);
                for (int round = 0; round < 3; ++round) {
                    tb[0] = std::min(tb[0], time_one(*P.jit[k]));
                    for (size_t a = 0; a < P.jit_alt[k].size(); ++a) tb[a + 1] = std::min(tb[a + 1], time_one(*P.jit_alt[k][a]));
                }
                size_t bi = 0;
                for (size_t a = 1; a < tb.size(); ++a)
                    if (tb[a] < tb[bi]) bi = a;
                // KS_KRON_JIT=b2 / b4 / point forces a candidate (tests, profiling)
                if (const char* e = std::getenv("KS_KRON_JIT")) {
                    // (b2 / b4: rows per thread of the row-blocked kernel; tile: the tile kernel too)
                    const bool wtile = !std::strcmp(e, "tile"), wshift = !std::strcmp(e, "shift");
                    const int want = !std::strcmp(e, "b2") || wtile || wshift ? 2 : !std::strcmp(e, "b4") ? 4 : !std::strcmp(e, "point") ? 0 : -1;
                    if (want >= 0) {
                        std::vector<KronJitPair*> all{P.jit[k].get()};
                        for (auto& alt : P.jit_alt[k]) all.push_back(alt.get());
                        for (size_t a = 0; a < all.size(); ++a)
                            if (((kron_jit_blocked_rows(*all[a]) == want &&
                                  (want == 4 || (std::strcmp(kron_jit_tag(*all[a]), "shifted window") == 0) == wshift)) ||
                                 ((wtile || wshift) && kron_jit_blocked_rows(*all[a]) >= 1000)) &&
                                tb[a] < 1e29f) {
                                bi = a;
                                break;
                            }
                    }
                }
                if (const char* e = std::getenv("KS_KRON_JIT"); e && std::strcmp(e, "0") != 0) // any value but 0 logs the timings
                    for (size_t a = 0; a < tb.size(); ++a)
                        std::fprintf(stderr, "ks_kron pass pair %zu candidate %zu (rows/thread %d%s%s): %.1f us%s\n", k, a,
                                     kron_jit_blocked_rows(a == 0 ? *P.jit[k] : *P.jit_alt[k][a - 1]),
                                     *kron_jit_tag(a == 0 ? *P.jit[k] : *P.jit_alt[k][a - 1]) ? ", " : "",
                                     kron_jit_tag(a == 0 ? *P.jit[k] : *P.jit_alt[k][a - 1]), 1e3f * tb[a],
                                     a == bi ? " <- kept" : "");
                if (bi > 0) std::swap(P.jit[k], P.jit_alt[k][bi - 1]);
                P.jit_alt[k].clear();
            }
            if (kron_jit_launch(*P.jit[k], ip, op, host_ptrs.data() + P.ptr_off[k],
                                host_ptrs.data() + P.ptr_off[k + 1] + nx.n_in, P.d_rowband.as<double2>(), P.nmax,
                                st)) {
                ++k;
                continue;
            }
        }
        // generated single pass (inner columns, literal bands)
        if (k < P.passc.size() && P.passc[k] && !shard_last && P.shard_rows == 0) {
            kron_jitc_launch(*P.passc[k], host_ptrs.data() + P.ptr_off[k], host_ptrs.data() + P.ptr_off[k] + ps.n_in, st);
            continue;
        }
        // element-parallel level kernel (all axes)
        if (ps.n_out <= 8 && P.bwmax >= 1 && P.bwmax <= 4) {
            auto ip = reinterpret_cast<const double2* const*>(dp + P.ptr_off[k]);
            auto op = reinterpret_cast<double2* const*>(const_cast<void**>(dp + P.ptr_off[k] + ps.n_in));
            const bool ok = shard_last
                                ? launch_colsweep(ps.n_in, ps.n_out, P.bwmax, ip, op, ps.d_in_begin.as<int>(),
                                                  ps.d_entries.as<SweepEntry>(), P.d_rowband.as<double2>(),
                                                  P.d_freal.as<int>(), P.N / (size_t)n, s, P.shard_rows,
                                                  P.nmax, st, n, P.shard_in_off, P.shard_band_off,
                                                  ps.d_begin.as<int>(), ps.d_ring.as<RingCon>())
                                : launch_colsweep(ps.n_in, ps.n_out, P.bwmax, ip, op, ps.d_in_begin.as<int>(),
                                                  ps.d_entries.as<SweepEntry>(), P.d_rowband.as<double2>(),
                                                  P.d_freal.as<int>(), P.N / (size_t)n, s, n, P.nmax, st, n, 0, 0,
                                                  ps.d_begin.as<int>(), ps.d_ring.as<RingCon>());
            if (ok) continue;
        }
        KS_REQUIRE(!shard_last, KS_EINVAL, "sharded matvec: level shape not supported");
        // time axis (and any other shape): row-chunk sweep
        if (ps.n_out <= kMaxOut && P.bwmax >= 1 && P.bwmax <= 4) {
            const size_t ncols = P.N / (size_t)n;
            const size_t nth = ncols * (size_t)((n + kR - 1) / kR);
            const unsigned g3 = (unsigned)((nth + 255) / 256);
            auto ip = reinterpret_cast<const double2* const*>(dp + P.ptr_off[k]);
            auto op = reinterpret_cast<double2* const*>(const_cast<void**>(dp + P.ptr_off[k] + ps.n_in));
#define KS_SW(NO, BWV)                                                                         \
    k_kron_sweep<NO, BWV><<<g3, 256, 0, st>>>(ip, ps.n_in, op, ps.d_in_begin.as<int>(),        \
                                               ps.d_entries.as<SweepEntry>(),                  \
                                               P.d_rowband.as<double2>(), P.d_freal.as<int>(), \
                                               ncols, s, n, P.nmax)
#define KS_SWB(NO)                                                                             \
    case NO:                                                                                   \
        switch (P.bwmax) {                                                                     \
        case 1: KS_SW(NO, 1); break;                                                           \
        case 2: KS_SW(NO, 2); break;                                                           \
        case 3: KS_SW(NO, 3); break;                                                           \
        default: KS_SW(NO, 4); break;                                                          \
        }                                                                                      \
        break;
            switch (ps.n_out) {
                KS_SWB(1) KS_SWB(2) KS_SWB(3) KS_SWB(4) KS_SWB(5) KS_SWB(6) KS_SWB(7) KS_SWB(8)
            }
#undef KS_SWB
#undef KS_SW
            check_launch("k_kron_sweep");
            continue;
        }
        const unsigned grid = (unsigned)((P.N + 255) / 256);
        k_kron_level<<<grid, 256, 0, st>>>(
            reinterpret_cast<const double2* const*>(dp + P.ptr_off[k]),
            reinterpret_cast<double2* const*>(const_cast<void**>(dp + P.ptr_off[k] + ps.n_in)),
            ps.n_out, ps.d_begin.as<int>(), ps.d_contribs.as<KronContrib>(),
            P.d_factors.as<DevFactor>(), P.d_bands.as<double2>(), P.N, s, n);
        check_launch("k_kron_level");
    }
}

void kron_plan_free(KronPlan* p) { delete p; }

bool kron_has_table(const KronPlan& P, const void* x, const void* y) {
    return P.ptr_tables.count(std::make_pair(x, const_cast<void*>(y))) > 0;
}

void kron_plan_set_shard(KronPlan& P, int rows, int in_off, int band_off) {
    P.shard_rows = rows;
    P.shard_in_off = in_off;
    P.shard_band_off = band_off;
}

} // namespace ks
