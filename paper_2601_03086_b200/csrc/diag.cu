// diag.cu — measured arithmetic peaks of this GPU ("re-measure with an FMA
// microbenchmark"; the denominators of the ALU floors quoted in DESIGN.md §5.7 / §9 and of
// bench.py's roofline.alu block).  Not on the hot path.
//
// pfem_fma_peak times a resident grid whose threads run 8 independent chains of dependent
// fused multiply-adds from register operands (no immediates: the 3-register form is the one
// the element kernels issue):
//   kind 0  fp32 FFMA        (one FMA per lane and issue slot)
//   kind 1  fp32 FFMA2       (two FMAs per lane and issue slot; sm_100a packed pair)
//   kind 2  fp64 DFMA
// and returns lane FMAs per second (x 2 = flop/s).
#include "common.cuh"

namespace pfem {

template <int KIND>
__global__ void __launch_bounds__(256) k_fma_peak(int iters, const double* __restrict__ ab, double* __restrict__ sink) {
    constexpr int C = 8;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    double out = 0.0;
    if constexpr (KIND == 0) {
        const float a = (float)ab[0], b = (float)ab[1];
        float x[C];
#pragma unroll
        for (int j = 0; j < C; ++j) x[j] = (float)(t + j) * 1e-9f;
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int j = 0; j < C; ++j) x[j] = fmaf(x[j], a, b);
#pragma unroll
        for (int j = 0; j < C; ++j) out += (double)x[j];
    } else if constexpr (KIND == 1) {
        const float2 a = make_float2((float)ab[0], (float)ab[0]), b = make_float2((float)ab[1], (float)ab[1]);
        float2 x[C];
#pragma unroll
        for (int j = 0; j < C; ++j) x[j] = make_float2((float)(t + j) * 1e-9f, (float)(t - j) * 1e-9f);
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int j = 0; j < C; ++j) x[j] = __ffma2_rn(x[j], a, b);
#pragma unroll
        for (int j = 0; j < C; ++j) out += (double)x[j].x + (double)x[j].y;
    } else {
        const double a = ab[0], b = ab[1];
        double x[C];
#pragma unroll
        for (int j = 0; j < C; ++j) x[j] = (double)(t + j) * 1e-9;
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int j = 0; j < C; ++j) x[j] = fma(x[j], a, b);
#pragma unroll
        for (int j = 0; j < C; ++j) out += x[j];
    }
    if (out == 123456.789) sink[0] = out;   // never true: keeps the chains alive
}

}  // namespace pfem

extern "C" pfem_status pfem_fma_peak(int32_t kind, int32_t iters, double* lane_fma_per_s, void* stream) {
    using namespace pfem;
    if (kind < 0 || kind > 2 || iters <= 0 || !lane_fma_per_s) {
        set_error("pfem_fma_peak: kind in {0, 1, 2}, iters > 0, non-null result");
        return PFEM_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0, nsm = 0;
    PFEM_CUDA_TRY(cudaGetDevice(&dev));
    PFEM_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    double* buf = nullptr;
    PFEM_CUDA_TRY(cudaMalloc(&buf, 4 * sizeof(double)));
    const double h[4] = {0.999999, 1e-7, 0.0, 0.0};
    PFEM_CUDA_TRY(cudaMemcpyAsync(buf, h, sizeof(h), cudaMemcpyHostToDevice, s));
    const int grid = nsm * 8, nt = 256;   // 2048 threads per SM: 16 warps per scheduler
    cudaEvent_t e0, e1;
    PFEM_CUDA_TRY(cudaEventCreate(&e0));
    PFEM_CUDA_TRY(cudaEventCreate(&e1));
    float best = 0.0f;
    for (int rep = 0; rep < 4; ++rep) {   // the first launch warms up
        PFEM_CUDA_TRY(cudaEventRecord(e0, s));
        if (kind == 0) k_fma_peak<0><<<grid, nt, 0, s>>>(iters, buf, buf + 2);
        else if (kind == 1) k_fma_peak<1><<<grid, nt, 0, s>>>(iters, buf, buf + 2);
        else k_fma_peak<2><<<grid, nt, 0, s>>>(iters, buf, buf + 2);
        PFEM_CUDA_TRY(cudaEventRecord(e1, s));
        PFEM_CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0.0f;
        PFEM_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        if (rep > 0 && (best == 0.0f || ms < best)) best = ms;
    }
    PFEM_CUDA_TRY(cudaGetLastError());
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    const double ops = (double)grid * nt * (double)iters * 8.0 * (kind == 1 ? 2.0 : 1.0);
    *lane_fma_per_s = ops / ((double)best * 1e-3);
    return PFEM_OK;
}
