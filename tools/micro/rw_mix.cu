// HBM throughput of read:write mixes at the c3 tensor size (17.04 M complex):
// 1 read + 3 writes (matvec pass (t,1)), 3 reads + 1 write (pass (2,3)), 1 + 1 (copy).
#include <cstdio>
#include <cuda_runtime.h>
template <int NR, int NWR>
__global__ void k(const double2* __restrict__ a, const double2* __restrict__ b, const double2* __restrict__ c,
                  double2* x, double2* y, double2* z, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double2 v = a[i];
        if (NR > 1) { double2 u = b[i]; v.x += u.x; v.y += u.y; }
        if (NR > 2) { double2 u = c[i]; v.x += u.x; v.y += u.y; }
        __stcs(x + i, v);
        if (NWR > 1) __stcs(y + i, v);
        if (NWR > 2) __stcs(z + i, v);
    }
}
int main() {
    const size_t n = 17039360;
    double2 *p[6];
    for (auto& q : p) { cudaMalloc(&q, n * 16); cudaMemset(q, 0, n * 16); }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](auto kern, const char* name, double bytes) {
        for (int w = 0; w < 3; ++w) kern<<<148 * 8, 512>>>(p[0], p[1], p[2], p[3], p[4], p[5], n);
        cudaEventRecord(e0);
        for (int r = 0; r < 20; ++r) kern<<<148 * 8, 512>>>(p[0], p[1], p[2], p[3], p[4], p[5], n);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
        printf("{\"mix\": \"%s\", \"us\": %.1f, \"gbs\": %.0f}\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    };
    run(k<1, 1>, "1r1w", 32.0 * n);
    run(k<1, 3>, "1r3w", 64.0 * n);
    run(k<3, 1>, "3r1w", 64.0 * n);
    return 0;
}
