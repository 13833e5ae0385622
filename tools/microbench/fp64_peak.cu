// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync.m8n8k4.f64)
// vs DFMA. Each warp runs independent accumulator chains from registers
// only, so the number is the issue-limited pipe throughput.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[CHAINS][2];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, c[i], b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += c[i];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int wpb : {4, 8, 16, 32}) {
        for (int bps : {1, 2}) {
            dim3 grid(sms * bps), block(32 * wpb);
            dmma_loop<8><<<grid, block>>>(out, 100);
            cudaEventRecord(e0);
            dmma_loop<8><<<grid, block>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid.x * wpb;
            printf("DMMA m8n8k4 warps/blk=%2d blk/SM=%d : %.2f TFLOP/s (%.3f ms)\n", wpb, bps,
                   flops / ms / 1e9, ms);
            dfma_loop<8><<<grid, block>>>(out, 100);
            cudaEventRecord(e0);
            dfma_loop<8><<<grid, block>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            flops = 2.0 * 8.0 * iters * (double)grid.x * block.x;
            printf("DFMA            warps/blk=%2d blk/SM=%d : %.2f TFLOP/s (%.3f ms)\n", wpb, bps,
                   flops / ms / 1e9, ms);
        }
    }
    printf("sms=%d clock_khz=%d err=%s\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
