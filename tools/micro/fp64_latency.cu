// Dependent-chain latency of FP64 DFMA / DADD / DMUL and of a shared-memory
// load -> DFMA round trip on this GPU (one thread; clock64 deltas).
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
    __shared__ double sm[64];
    double x = a, y = b;
    if (threadIdx.x < 64) sm[threadIdx.x] = a + threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, a);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = x + y;
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) x = x * y;
    long long t3 = clock64();
    int j = 0;
    for (int i = 0; i < n; ++i) { x = fma(x, sm[j], a); j = ((int)x) & 31; }
    long long t4 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 32);
    const int n = 4096;
    k<<<1, 32>>>(o, c, 1.0000001, 0.9999999, n);
    k<<<1, 32>>>(o, c, 1.0000001, 0.9999999, n);
    long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("{\"dfma_latency\": %.1f, \"dadd_latency\": %.1f, \"dmul_latency\": %.1f, \"lds_dfma_roundtrip\": %.1f}\n",
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n);
}
