// intpeak.cu -- measured INT-pipe peak of the device (roofline denominator).
//
// Not part of the C-ABI of include/hrb200.h: a measurement tool that bench.py
// loads beside it.  mix = 1: every chain step is one IADD3 (ALU pipe) plus
// one IMAD (FMA pipe), so the sub-partition schedulers can issue one integer
// warp-instruction per clock, the INT issue limit of the SM (ALU and FMA
// pipes each accept one warp-instruction every 2 clocks per sub-partition).
// mix = 0: IADD3 + LOP3, both on the ALU pipe alone.  The returned figure is
// lane-ops/s = SASS integer instructions * 32 lanes / seconds, the unit the
// HR kernels' achieved INT throughput is quoted in.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

template <int REPS, bool MIX>
__global__ void __launch_bounds__(256) int_peak_kernel(uint32_t seed, uint32_t* sink) {
    // 8 independent chains of two mutually dependent registers: every result
    // feeds the next operation, so ptxas can neither fold nor fuse them
    // (two SASS instructions per chain step, checked with cuobjdump / ncu)
    uint32_t a[8], b[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        a[k] = seed + threadIdx.x * 7u + k;
        b[k] = seed ^ (threadIdx.x + 13u * k);
    }
    const uint32_t c = seed | 3u;
#pragma unroll 4
    for (int r = 0; r < REPS; r++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            asm volatile("add.u32 %0, %0, %1;" : "+r"(a[k]) : "r"(b[k]));  // IADD3, ALU pipe
            if (MIX)
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(b[k]) : "r"(c), "r"(a[k]));  // IMAD, FMA pipe
            else
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(b[k]) : "r"(a[k]));  // LOP3, ALU pipe
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) x ^= a[k] ^ b[k];
    if (x == 0x9E3779B9u) sink[0] = x;  // keep the chains alive
}

}  // namespace

extern "C" {

// Runs the microbenchmark on the current device; *lane_ops_per_s receives
// the best of `trials` launches (CUDA events), *ms the matching duration.
// mix != 0: IADD3 + IMAD interleaved (ALU + FMA pipes, issue-bound);
// mix == 0: IADD3 only (ALU pipe alone).
int hrb_int_peak(int mix, int trials, double* lane_ops_per_s, float* ms) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess) return 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t* sink = nullptr;
    if (cudaMalloc(&sink, 64) != cudaSuccess) return 1;
    constexpr int REPS = 4096;
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto kern = mix ? int_peak_kernel<REPS, true> : int_peak_kernel<REPS, false>;
    kern<<<blocks, threads>>>(1u, sink);  // warm-up
    double best = 0;
    float best_ms = 0;
    for (int t = 0; t < (trials > 0 ? trials : 1); t++) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(2u + t, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float m = 0;
        cudaEventElapsedTime(&m, e0, e1);
        const double ops = (double)blocks * threads * REPS * 8.0 * 2.0;
        const double v = ops / (m * 1e-3);
        if (v > best) {
            best = v;
            best_ms = m;
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (cudaGetLastError() != cudaSuccess) return 1;
    *lane_ops_per_s = best;
    if (ms) *ms = best_ms;
    return 0;
}

}  // extern "C"
