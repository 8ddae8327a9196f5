// sharded_pcg_demo.cpp -- a C++ caller of the multi-GPU C-ABI (include/ks.h),
// in the style of oracle/integration_demo.cpp: one process per rank, NCCL
// communicator created through ks_comm_*, slab-sharded FD preconditioner and
// system operator, and the device-resident sharded pcg (ks_pcg_sharded) --
// the call a reference driver (experiments.cpp:46-52 -> krylov.cpp:24) makes
// per rank. Rank 0 also solves the unsharded problem with ks_pcg and checks
// that its slab agrees. TEST INFRASTRUCTURE (tests/test_gpu_shard_cabi.py).
//
// usage: sharded_pcg_demo d p n_el nranks rank device idfile   -> one JSON line per rank
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <random>
#include <thread>
#include <vector>

#include "ks.h"

#define CHECK(x)                                                                               \
    do {                                                                                       \
        const int rc_ = (x);                                                                   \
        if (rc_ != KS_OK) {                                                                    \
            std::fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, ks_last_error());           \
            std::exit(2);                                                                      \
        }                                                                                      \
    } while (0)

int main(int argc, char** argv) {
    if (argc < 8) {
        std::fprintf(stderr, "usage: %s d p n_el nranks rank device idfile\n", argv[0]);
        return 1;
    }
    const int d = std::atoi(argv[1]), p = std::atoi(argv[2]), n_el = std::atoi(argv[3]);
    const int nranks = std::atoi(argv[4]), rank = std::atoi(argv[5]), device = std::atoi(argv[6]);
    const char* idfile = argv[7];

    // communicator: rank 0 publishes the unique id, the others wait for it
    unsigned char id[KS_COMM_ID_BYTES];
    if (rank == 0) {
        CHECK(ks_comm_unique_id(id));
        std::ofstream(std::string(idfile) + ".tmp", std::ios::binary).write((const char*)id, sizeof(id));
        std::rename((std::string(idfile) + ".tmp").c_str(), idfile);
    } else {
        for (;;) {
            std::ifstream f(idfile, std::ios::binary);
            if (f && f.read((char*)id, sizeof(id)) && f.gcount() == (std::streamsize)sizeof(id)) break;
            std::this_thread::sleep_for(std::chrono::milliseconds(20));
        }
    }
    ks_comm* comm = nullptr;
    CHECK(ks_comm_create(nranks, rank, id, device, &comm));

    // problem (libks host setup = the reference's SpaceTimeProblem::uniform + build_univariate)
    ks_setup* s = nullptr;
    CHECK(ks_setup_create(d, p, n_el, n_el, 1.0, 1.0, 0, &s));
    int dd = 0, pp = 0;
    std::vector<int> dims(d + 1);
    CHECK(ks_setup_dims(s, &dd, dims.data(), &pp));
    const int nt = dims[0], ld = 2 * p + 1;
    std::vector<double> Lt((size_t)ld * nt), Mt((size_t)ld * nt);
    std::vector<ks_c64> Wt((size_t)ld * nt);
    CHECK(ks_setup_time_bands(s, Lt.data(), Mt.data(), Wt.data()));
    std::vector<std::vector<double>> U(d), lam(d);
    std::vector<const double*> Up(d), lp(d);
    for (int l = 0; l < d; ++l) {
        U[l].resize((size_t)dims[l + 1] * dims[l + 1]);
        lam[l].resize(dims[l + 1]);
        CHECK(ks_setup_eig(s, l, U[l].data(), lam[l].data()));
        Up[l] = U[l].data();
        lp[l] = lam[l].data();
    }
    ks_fdshard* P = nullptr;
    CHECK(ks_fdshard_create(d, dims.data(), 1.0, p, Up.data(), lp.data(), Lt.data(), Mt.data(), Wt.data(), nranks,
                            rank, device, &P));
    ks_kron* A = nullptr;
    CHECK(ks_setup_create_system_sharded(s, nranks, rank, device, &A));
    long long lo = 0, hi = 0, elo = 0, ehi = 0;
    size_t plane = 0;
    CHECK(ks_kronshard_sizes(A, &lo, &hi, &elo, &ehi, &plane));

    // right-hand side: re / im i.i.d. U[-1,1] (mt19937_64(1234), vec order), this rank's slab
    size_t N = 1;
    for (int a = 0; a <= d; ++a) N *= (size_t)dims[a];
    std::vector<ks_c64> b(N);
    std::mt19937_64 g(1234);
    for (auto& v : b) {
        v.re = 2.0 * (double)(g() >> 11) * 0x1.0p-53 - 1.0;
        v.im = 2.0 * (double)(g() >> 11) * 0x1.0p-53 - 1.0;
    }
    const size_t n_slab = (size_t)(hi - lo) * plane;
    std::vector<ks_c64> x(n_slab);
    ks_pcg_opts opts{1e-8, 200, 0};
    ks_pcg_report rep{};
    std::vector<double> hist(200);
    const auto t0 = std::chrono::steady_clock::now();
    CHECK(ks_pcg_sharded(A, P, comm, b.data() + (size_t)lo * plane, x.data(), KS_MEM_HOST, &opts, hist.data(),
                         (int)hist.size(), &rep));
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    // rank 0: the same solve unsharded on one GPU, compared on this rank's slab
    double rel = -1.0;
    int it1 = -1;
    if (rank == 0) {
        ks_fd* F = nullptr;
        ks_kron* K = nullptr;
        CHECK(ks_setup_create_fd(s, device, &F));
        CHECK(ks_setup_create_system(s, device, &K));
        std::vector<ks_c64> x1(N);
        ks_pcg_report r1{};
        CHECK(ks_pcg(K, F, b.data(), x1.data(), KS_MEM_HOST, &opts, nullptr, 0, &r1));
        it1 = r1.iterations;
        double num = 0, den = 0;
        for (size_t i = 0; i < n_slab; ++i) {
            const ks_c64 a = x[i], c = x1[(size_t)lo * plane + i];
            num += (a.re - c.re) * (a.re - c.re) + (a.im - c.im) * (a.im - c.im);
            den += c.re * c.re + c.im * c.im;
        }
        rel = std::sqrt(num / den);
        ks_fd_destroy(F);
        ks_kron_destroy(K);
    }
    std::printf("{\"rank\": %d, \"nranks\": %d, \"slab\": [%lld, %lld], \"iterations\": %d, \"converged\": %d, "
                "\"final_relres\": %.6e, \"seconds\": %.6f, \"single_gpu_iterations\": %d, \"rel_vs_single\": %.3e}\n",
                rank, nranks, lo, hi, rep.iterations, rep.converged,
                rep.hist_len > 0 ? hist[rep.hist_len - 1] : 0.0, sec, it1, rel);
    ks_kron_destroy(A);
    ks_fdshard_destroy(P);
    ks_setup_destroy(s);
    ks_comm_destroy(comm);
    return 0;
}
