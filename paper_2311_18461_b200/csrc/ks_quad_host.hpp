// Host-side quadrature / collocation data of a ks_setup, consumed by the
// device RHS, lifting and error-norm module (ks_rhs.cu). Plain C++ (no CUDA):
// produced by ks_setup.cpp from its B-spline restatement.
#pragma once

#include <complex>
#include <vector>

struct ks_setup;

namespace ks {

struct QuadAxis {
    int n = 0;                     // full basis size m_l
    int nq = 0;                    // quadrature nodes (elements x (p+1))
    int npe = 0;                   // nodes per element (p+1)
    std::vector<double> nodes, weights;
    std::vector<double> E[3];      // basis derivative values, [q][k], k < p+1 (orders 0..2)
    std::vector<int> off;          // first nonzero basis function of node q
    std::vector<double> greville;  // Greville abscissae (n)
    std::vector<std::complex<double>> colloc_ab; // factor_banded of the collocation matrix, (3p+1) x n
    std::vector<int> colloc_piv;                 // n
};

struct QuadData {
    int d = 1, p = 1, trial = 0;
    double nu = 1.0;
    std::vector<int> full_dims, red_dims;
    std::vector<QuadAxis> axes;    // axis 0 = time
    // unrestricted univariate bands for assemble_system_operator_full (BandedMatrix layout)
    std::vector<std::complex<double>> Lt, Mt, Wt;
    std::vector<std::vector<std::complex<double>>> M, L, G, V;
};

// throws std::invalid_argument on bad input
QuadData setup_quad_data(const ks_setup* s);

} // namespace ks
