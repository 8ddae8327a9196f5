// integration_demo.cpp -- the reference-side binding a kronschro maintainer
// would add, compiled against the reference's own headers
// and objects (oracle/_ref) and libks.so. TEST INFRASTRUCTURE: it proves the
// drop-in end to end. The reference's pcg (krylov.cpp:24) runs unchanged;
// only the two ApplyFn lambdas of solve_problem (experiments.cpp:46-49) are
// pointed at the B200 objects.
//
// usage: integration_demo d p n_el   -> prints one JSON line
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "kronschro/assembly.hpp"
#include "kronschro/fdsolver.hpp"
#include "kronschro/krylov.hpp"
#include "kronschro_gpu.hpp"

using namespace kronschro;

namespace {

// BandedMatrix -> BandedMatrix storage (banded.hpp:91-94 layout)
template <typename T> std::vector<T> band_data(const BandedMatrix<T>& b) {
    const int n = b.rows(), bw = b.bandwidth();
    std::vector<T> out((size_t)(2 * bw + 1) * n, T(0));
    for (int j = 0; j < n; ++j)
        for (int i = std::max(0, j - bw); i <= std::min(n - 1, j + bw); ++i)
            out[(size_t)(bw + i - j) + (size_t)j * (2 * bw + 1)] = b(i, j);
    return out;
}

} // namespace

// ---- the adapter (what INTEGRATION.md shows) --------------------------------
kronschro_gpu::FDPreconditioner make_gpu_fd(const SpaceTimeProblem& prob, const UnivariateSet& u) {
    const SpatialEigenbasis basis = spatial_eigenbasis(prob, u); // reference host setup
    std::vector<const double*> U, lam;
    for (const auto& ax : basis.axes) {
        U.push_back(ax.U.data());        // column-major n x n
        lam.push_back(ax.lambda.data());
    }
    const auto Lt = band_data(u.Lt), Mt = band_data(u.Mt);
    const auto Wt = band_data(u.Wt);
    return kronschro_gpu::FDPreconditioner(prob.reduced_dims(), prob.nu, prob.p_t(), U, lam, Lt.data(),
                                           Mt.data(), Wt.data());
}

kronschro_gpu::KroneckerOperator make_gpu_operator(const KroneckerOperator& A,
                                                   std::vector<std::vector<cplx>>& keep) {
    kronschro_gpu::KroneckerOperator G(A.dims());
    for (const auto& t : A.terms()) {
        std::vector<kronschro_gpu::KroneckerOperator::Factor> fs;
        for (const auto& f : t.factors) {
            if (!f) {
                fs.push_back({nullptr, 0});
                continue;
            }
            keep.push_back(band_data(*f));
            fs.push_back({keep.back().data(), f->bandwidth()});
        }
        G.add_term(t.coeff, fs);
    }
    return G;
}
// -----------------------------------------------------------------------------

int main(int argc, char** argv) {
    const int d = argc > 1 ? std::atoi(argv[1]) : 2;
    const int p = argc > 2 ? std::atoi(argv[2]) : 3;
    const int n_el = argc > 3 ? std::atoi(argv[3]) : 16;
    const SpaceTimeProblem prob = SpaceTimeProblem::matched(d, p, n_el, 1.0, 1.0);
    const UnivariateSet u = build_univariate(prob);
    const KroneckerOperator A = assemble_system_operator(prob);
    const FDPreconditioner P(prob, u);

    std::mt19937_64 g(1234);
    std::vector<cplx> b(A.vec_size());
    for (auto& v : b) {
        const double re = 2.0 * ((g() >> 11) * 0x1.0p-53) - 1.0;
        const double im = 2.0 * ((g() >> 11) * 0x1.0p-53) - 1.0;
        v = cplx(re, im);
    }

    // reference: CPU objects
    const auto t0 = std::chrono::steady_clock::now();
    const SolveReport cpu = pcg([&](const cplx* x, cplx* y) { A.apply(x, y); },
                                [&](const cplx* x, cplx* y) { P.apply(x, y); }, b, {1e-8, 200});
    const double t_cpu = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    // drop-in: same reference pcg, B200 objects behind the ApplyFn callbacks
    std::vector<std::vector<cplx>> keep;
    const auto gA = make_gpu_operator(A, keep);
    const auto gP = make_gpu_fd(prob, u);
    const auto t1 = std::chrono::steady_clock::now();
    const SolveReport gpu = pcg([&](const cplx* x, cplx* y) { gA.apply(x, y); },
                                [&](const cplx* x, cplx* y) { gP.apply(x, y); }, b, {1e-8, 200});
    const double t_gpu = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();

    // device-resident loop through the C-ABI (ks_pcg)
    const auto t2 = std::chrono::steady_clock::now();
    const auto dev = kronschro_gpu::pcg(gA, &gP, b, {1e-8, 200, false});
    const double t_dev = std::chrono::duration<double>(std::chrono::steady_clock::now() - t2).count();

    double num = 0, den = 0, num2 = 0;
    for (size_t i = 0; i < b.size(); ++i) {
        num += std::norm(gpu.x[i] - cpu.x[i]);
        num2 += std::norm(dev.x[i] - cpu.x[i]);
        den += std::norm(cpu.x[i]);
    }
    std::printf("{\"dofs\": %zu, \"cpu_iters\": %d, \"gpu_callback_iters\": %d, \"gpu_device_iters\": %d, "
                "\"rel_x_callback\": %.3e, \"rel_x_device\": %.3e, \"cpu_s\": %.4f, \"gpu_callback_s\": %.4f, "
                "\"gpu_device_s\": %.4f, \"converged\": [%d, %d, %d]}\n",
                b.size(), cpu.iterations, gpu.iterations, dev.iterations, std::sqrt(num / den),
                std::sqrt(num2 / den), t_cpu, t_gpu, t_dev, (int)cpu.converged, (int)gpu.converged,
                (int)dev.converged);
    return 0;
}
