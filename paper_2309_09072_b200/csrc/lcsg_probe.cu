// lcsg_probe.cu -- measured INT32 min/compare issue rate (R_INT32 of the
// combine roofline).
//
// The combine's unit of work is one reference cell evaluation: a packed
// (value << shift | k) key folded into a running minimum with ONE unsigned
// 32-bit min (IMNMX.U32 in SASS) -- the `v < best` first-wins test of
// _kernel.pyx:40-44.  This kernel issues nothing but independent IMNMX.U32
// chains (8 accumulators per thread, operands rotated so nothing folds) on
// every SM, and the rate it reaches is the INT32 term's denominator.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lcsgrid_b200.h"

namespace {

constexpr int PROBE_ACC = 8;
constexpr int PROBE_UNROLL = 16;

__global__ void __launch_bounds__(256) imnmx_probe_kernel(uint32_t seed, int iters,
                                                          uint32_t *sink) {
    uint32_t acc[PROBE_ACC], x[PROBE_ACC];
#pragma unroll
    for (int a = 0; a < PROBE_ACC; ++a) {
        acc[a] = 0xffffffffu - (threadIdx.x + a);
        x[a] = seed * (a + 1) + blockIdx.x * 7919u + threadIdx.x;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < PROBE_UNROLL; ++u) {
#pragma unroll
            for (int a = 0; a < PROBE_ACC; ++a) {
                // acc = min(acc, x[a]); the operand is the neighbour accumulator's
                // input, so every instruction is live and nothing is hoisted
                asm volatile("min.u32 %0, %0, %1;" : "+r"(acc[a]) : "r"(x[(a + u) & (PROBE_ACC - 1)]));
            }
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int a = 0; a < PROBE_ACC; ++a) r ^= acc[a];
    if (r == seed) sink[0] = r;  // practically never; keeps the chains live
}

}  // namespace

extern "C" int lcsg_probe_int32_rate(int device, double *mins_per_s, int32_t *sm_count,
                                     double *ms) {
    int prev = -1;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        return LCSG_ENODEV;
    }
    int rc = LCSG_OK;
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    const int sms = prop.multiProcessorCount;
    const int blocks = sms * 8, threads = 256, iters = 4096;
    uint32_t *sink = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    float t = 0.f;
    if (cudaMalloc(&sink, 4) != cudaSuccess || cudaEventCreate(&e0) != cudaSuccess ||
        cudaEventCreate(&e1) != cudaSuccess) {
        rc = LCSG_ECUDA;
    } else {
        imnmx_probe_kernel<<<blocks, threads>>>(12345u, iters / 8, sink);  // warm-up, clocks up
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            imnmx_probe_kernel<<<blocks, threads>>>(12345u + rep, iters, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&t, e0, e1);
            best = t < best ? t : best;
        }
        t = best;
        if (cudaGetLastError() != cudaSuccess) rc = LCSG_ECUDA;
    }
    const double ops = (double)blocks * threads * iters * PROBE_UNROLL * PROBE_ACC;
    if (rc == LCSG_OK) {
        if (mins_per_s) *mins_per_s = ops / (t * 1e-3);
        if (sm_count) *sm_count = sms;
        if (ms) *ms = t;
    }
    if (sink) cudaFree(sink);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (prev >= 0) cudaSetDevice(prev);
    return rc;
}
