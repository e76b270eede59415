// d2q37_probe.cu -- FP64 peak probe: the denominator of the collide roofline.
//
// MEASURED_PEAKS.json (driver-written) carries HBM and bf16 tensor peaks but
// no FP64 figure, and the nominal 37 TFLOP/s assumes the 1.965 GHz boost
// clock, which a B200 under its power cap does not hold.  This kernel keeps
// every FP64 pipe busy with independent DFMA chains (16 per thread, 16
// warps per SM) and reports the achieved DFMA rate: 2 FLOP per DFMA.
#include <cuda_runtime.h>

#include "d2q37_b200.h"
#include "d2q37_internal.h"

namespace {

__global__ void __launch_bounds__(256) k_dfma_probe(double* out, int iters, double b, double c) {
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-9 + i;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 1.2345) out[0] = s;  // keeps the chains live; never true for these inputs
}

}  // namespace

extern "C" int d2q37_fp64_peak(int device, double* tflops) {
    if (!tflops) return D2Q37_ERR_INVALID_ARGUMENT;
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return D2Q37_ERR_CUDA;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    double* out = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int rc = D2Q37_OK;
    const int blocks = nsm * 8, threads = 256, iters = 4096;
    float ms = 0.f;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess || cudaEventCreate(&e0) != cudaSuccess ||
        cudaEventCreate(&e1) != cudaSuccess) {
        rc = D2Q37_ERR_CUDA;
    } else {
        k_dfma_probe<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);  // warm-up (clocks ramp)
        cudaEventRecord(e0);
        k_dfma_probe<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        if (cudaEventSynchronize(e1) != cudaSuccess || cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess || ms <= 0.f)
            rc = D2Q37_ERR_CUDA;
    }
    if (rc == D2Q37_OK) {
        const double dfma = double(blocks) * threads * iters * 16.0 * 8.0;
        *tflops = 2.0 * dfma / (ms * 1e-3) / 1e12;
    }
    if (out) cudaFree(out);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaSetDevice(prev);
    return rc;
}
