// FP64 peak microbenchmarks: the roofline denominator for the FP64-bound
// transforms. MEASURED_PEAKS.json carries only HBM and bf16 figures, so the
// bench measures the DFMA (CUDA-core) and DMMA (mma.sync f64) issue peaks
// live on the same device, at the clocks the device runs under load.
#include "ks_internal.hpp"

#include <vector>

namespace ks {

namespace {

constexpr int kIters = 2048;

__global__ void __launch_bounds__(256) k_dfma_peak(double* out, double seed) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-9 + i;
    const double b = 0.999999, c = 1e-7;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_dmma_peak(double* out, double seed) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = seed + i;
    const double a = 0.999 + threadIdx.x * 1e-9, b = 1e-3;
    for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

} // namespace
__global__ void k_dmma_peak_pub(double* out, double seed) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = seed + i;
    const double a = 0.999 + threadIdx.x * 1e-9, b = 1e-3;
    for (int it = 0; it < 2048 / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}
namespace {
// m16n8k16 f64 (sm_90+ shape; ptxas lowers it to 8x DMMA.8x8x4 on sm_100a)
__global__ void __launch_bounds__(256) k_dmma16_peak(double* out, double seed) {
    double c[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) c[i][j] = seed + i + j;
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = 0.999 + threadIdx.x * 1e-9 + i * 1e-6;
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = 1e-3 + i * 1e-7;
    for (int it = 0; it < kIters / 32; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                         "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
                           "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.678) out[threadIdx.x] = s;
}

// warps 0-3 issue DMMA, warps 4-7 DFMA: does the FP64 tensor path run
// concurrently with the CUDA-core FP64 pipe?
__global__ void __launch_bounds__(256) k_mixed_peak(double* out, double seed) {
    const int warp = threadIdx.x >> 5;
    double s = 0;
    if (warp < 4) {
        double c[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = seed + i;
        const double a = 0.999 + threadIdx.x * 1e-9, b = 1e-3;
        for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[i][0]), "+d"(c[i][1])
                             : "d"(a), "d"(b));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    } else {
        double a[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-9 + i;
        const double b = 0.999999, cc = 1e-7;
        for (int it = 0; it < kIters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, cc);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s += a[i];
    }
    if (s == 12345.678) out[threadIdx.x] = s;
}

} // namespace

// flops of one mixed launch: 4 DMMA warps + 4 DFMA warps per block
static double mixed_flops(unsigned grid) {
    return (double)grid * 4 * (kIters / 4) * 8 * 512.0 + (double)grid * 128 * kIters * 8 * 2.0;
}

static void run_mixed(double* tflops) {
    int sms = 148, dev = 0;
    KS_CUDA(cudaGetDevice(&dev));
    KS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DevBuf out(256 * sizeof(double));
    const unsigned grid = sms * 8;
    cudaEvent_t a, b;
    KS_CUDA(cudaEventCreate(&a));
    KS_CUDA(cudaEventCreate(&b));
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        KS_CUDA(cudaEventRecord(a));
        k_mixed_peak<<<grid, 256>>>(out.as<double>(), 1.0);
        check_launch("k_mixed_peak");
        KS_CUDA(cudaEventRecord(b));
        KS_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        KS_CUDA(cudaEventElapsedTime(&ms, a, b));
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *tflops = mixed_flops(grid) / (best * 1e-3) / 1e12;
}

static void run_mma16(double* tflops) {
    int sms = 148, dev = 0;
    KS_CUDA(cudaGetDevice(&dev));
    KS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DevBuf out(256 * sizeof(double));
    const unsigned grid = sms * 8;
    cudaEvent_t a, b;
    KS_CUDA(cudaEventCreate(&a));
    KS_CUDA(cudaEventCreate(&b));
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        KS_CUDA(cudaEventRecord(a));
        k_dmma16_peak<<<grid, 256>>>(out.as<double>(), 1.0);
        check_launch("k_dmma16_peak");
        KS_CUDA(cudaEventRecord(b));
        KS_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        KS_CUDA(cudaEventElapsedTime(&ms, a, b));
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = (double)grid * 8 * (kIters / 32) * 4 * 4096.0;
    *tflops = flops / (best * 1e-3) / 1e12;
}

static void run_peak(bool mma, double* tflops) {
    int sms = 148;
    int dev = 0;
    KS_CUDA(cudaGetDevice(&dev));
    KS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DevBuf out(256 * sizeof(double));
    const unsigned grid = sms * 8;
    cudaEvent_t a, b;
    KS_CUDA(cudaEventCreate(&a));
    KS_CUDA(cudaEventCreate(&b));
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        KS_CUDA(cudaEventRecord(a));
        if (mma) k_dmma_peak<<<grid, 256>>>(out.as<double>(), 1.0);
        else k_dfma_peak<<<grid, 256>>>(out.as<double>(), 1.0);
        check_launch("k_fp64_peak");
        KS_CUDA(cudaEventRecord(b));
        KS_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        KS_CUDA(cudaEventElapsedTime(&ms, a, b));
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    // flops: DFMA 2 per lane-op; DMMA m8n8k4 = 256 FMA per warp-op = 512 flops
    const double threads = (double)grid * 256;
    const double flops = mma ? (double)grid * 8 /*warps*/ * (kIters / 4) * 8 * 512.0
                             : threads * kIters * 8 * 2.0;
    *tflops = flops / (best * 1e-3) / 1e12;
}

void fp64_peak_bench(double* tflops) { run_peak(false, tflops); }
void fp64_peak_bench_mixed(double* tflops) { run_mixed(tflops); }
void fp64_peak_bench_mma16(double* tflops) { run_mma16(tflops); }
void fp64_peak_bench_mma(double* tflops) { run_peak(true, tflops); }

} // namespace ks

// HBM fan-in/fan-out bandwidth: read NIN arrays, write NOUT arrays (sum / copies),
// fully unrolled over the arrays (the matvec passes' 1:3 and 3:1 mixes)
struct FanPtrs {
    const double2* in[4];
    double2* out[4];
};
template <int NI, int NO>
__global__ void __launch_bounds__(512) k_fan(FanPtrs p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double2 a = __ldg(p.in[0] + i);
#pragma unroll
        for (int j = 1; j < NI; ++j) {
            const double2 v = __ldg(p.in[j] + i);
            a.x += v.x;
            a.y += v.y;
        }
#pragma unroll
        for (int k = 0; k < NO; ++k) __stcs(p.out[k] + i, make_double2(a.x * (k + 1), a.y));
    }
}
template <int NI>
static void launch_fan(int nout, const FanPtrs& p, size_t n) {
    switch (nout) {
    case 1: k_fan<NI, 1><<<148 * 8, 512>>>(p, n); break;
    case 2: k_fan<NI, 2><<<148 * 8, 512>>>(p, n); break;
    case 3: k_fan<NI, 3><<<148 * 8, 512>>>(p, n); break;
    default: k_fan<NI, 4><<<148 * 8, 512>>>(p, n); break;
    }
}
extern "C" int ks_bw_fan(int nin, int nout, size_t n, double* gbs) {
    try {
        std::vector<ks::DevBuf> bufs;
        std::vector<void*> ptr;
        for (int j = 0; j < nin + nout; ++j) {
            bufs.emplace_back(n * sizeof(double2));
            KS_CUDA(cudaMemset(bufs.back().p, 0, n * sizeof(double2)));
            ptr.push_back(bufs.back().p);
        }
        if (nin < 1 || nin > 4 || nout < 1 || nout > 4) throw ks::Error(KS_EINVAL, "ks_bw_fan: 1..4 inputs and outputs");
        FanPtrs fp{};
        for (int j = 0; j < nin; ++j) fp.in[j] = static_cast<const double2*>(ptr[j]);
        for (int k = 0; k < nout; ++k) fp.out[k] = static_cast<double2*>(ptr[nin + k]);
        cudaEvent_t a, b;
        KS_CUDA(cudaEventCreate(&a));
        KS_CUDA(cudaEventCreate(&b));
        float best = 1e30f;
        for (int rep = 0; rep < 8; ++rep) {
            KS_CUDA(cudaEventRecord(a));
            switch (nin) {
            case 1: launch_fan<1>(nout, fp, n); break;
            case 2: launch_fan<2>(nout, fp, n); break;
            case 3: launch_fan<3>(nout, fp, n); break;
            default: launch_fan<4>(nout, fp, n); break;
            }
            ks::check_launch("k_fan");
            KS_CUDA(cudaEventRecord(b));
            KS_CUDA(cudaEventSynchronize(b));
            float ms = 0;
            KS_CUDA(cudaEventElapsedTime(&ms, a, b));
            if (rep > 0 && ms < best) best = ms;
        }
        *gbs = (double)(nin + nout) * n * 16 / (best * 1e-3) / 1e9;
    } catch (const ks::Error& e) {
        ks::set_last_error(e.what());
        return e.code;
    }
    return KS_OK;
}

// DMMA throughput at a given number of resident warps per SM (grid = SMs x ctas)
extern "C" int ks_fp64_dmma_occupancy(int ctas_per_sm, int threads, double* tflops) {
    try {
        int sms = 148, dev = 0;
        KS_CUDA(cudaGetDevice(&dev));
        KS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        ks::DevBuf out(1024 * sizeof(double));
        const unsigned grid = sms * ctas_per_sm;
        cudaEvent_t a, b;
        KS_CUDA(cudaEventCreate(&a));
        KS_CUDA(cudaEventCreate(&b));
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            KS_CUDA(cudaEventRecord(a));
            ks::k_dmma_peak_pub<<<grid, threads>>>(out.as<double>(), 1.0);
            ks::check_launch("k_dmma_peak");
            KS_CUDA(cudaEventRecord(b));
            KS_CUDA(cudaEventSynchronize(b));
            float ms = 0;
            KS_CUDA(cudaEventElapsedTime(&ms, a, b));
            if (rep > 0 && ms < best) best = ms;
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        const double flops = (double)grid * (threads / 32) * (2048 / 4) * 8 * 512.0;
        *tflops = flops / (best * 1e-3) / 1e12;
    } catch (const ks::Error& e) {
        ks::set_last_error(e.what());
        return e.code;
    }
    return KS_OK;
}

extern "C" int ks_fp64_peak_mma16(double* tflops) {
    try {
        ks::fp64_peak_bench_mma16(tflops);
    } catch (const ks::Error& e) {
        ks::set_last_error(e.what());
        return e.code;
    }
    return KS_OK;
}

extern "C" int ks_fp64_peak_mixed(double* tflops) {
    try {
        ks::fp64_peak_bench_mixed(tflops);
    } catch (const ks::Error& e) {
        ks::set_last_error(e.what());
        return e.code;
    }
    return KS_OK;
}

extern "C" int ks_fp64_peaks(double* dfma, double* dmma) {
    try {
        if (dfma) ks::fp64_peak_bench(dfma);
        if (dmma) ks::fp64_peak_bench_mma(dmma);
    } catch (const ks::Error& e) {
        ks::set_last_error(e.what());
        return e.code;
    }
    return KS_OK;
}
