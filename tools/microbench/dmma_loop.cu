// DMMA issue ceiling for the update kernels' inner loop shapes (sm_100a):
//  0: register-resident A fragments (64 doubles), B from shared memory (4 LDS per 8 DMMA)
//  1: same, B fragments from registers too (no LDS)
//  2: A and B from shared memory (2 + 4 LDS per 8 DMMA)
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) loop(double* out, int iters) {
    __shared__ double sb[32 * 132 + 128 * 36 / 4 + 64];
    for (int i = threadIdx.x; i < 32 * 132 + 128 * 36 / 4 + 64; i += 256) sb[i] = 1e-3 * (i % 17);
    __syncthreads();
    const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3, warp = threadIdx.x >> 5;
    double af[2][32];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int k = 0; k < 32; ++k) af[m][k] = 1e-3 * (m + k + lane);
    double acc[2][4][2] = {};
    const double* p = sb + gid * 132 + tig;
    const double* pa = sb + 32 * 132 + (2 * warp + gid) * 36 + tig;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int ks = 0; ks < 32; ++ks) {
            double bf[4], a2[2];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) bf[nt] = (MODE == 1) ? af[nt & 1][(ks + nt) & 31] : p[nt * 8 * 132 + 4 * ks];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) a2[mt] = (MODE == 2) ? pa[mt * 8 * 36 + ((4 * ks) & 31)] : af[mt][ks];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a2[mt], bf[nt]);
        }
    }
    double s = 0;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) s += acc[mt][nt][0] + acc[mt][nt][1];
    if (s == 1234.5) out[0] = s;
}

template <typename K>
void run(const char* name, K k, int sms, int bps) {
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2000;
    k<<<sms * bps, 256>>>(out, 10);
    cudaEventRecord(e0);
    k<<<sms * bps, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 8 * 8 * 4 * 8 * 32 * (double)iters * 8 * sms * bps;
    printf("%-34s blk/SM=%d %.2f TFLOP/s (%s)\n", name, bps, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run("A regs, B lds (0.5 LDS/DMMA)", loop<0>, sms, 1);
    run("A regs, B regs (no LDS)", loop<1>, sms, 1);
    run("A lds, B lds (0.75 LDS/DMMA)", loop<2>, sms, 1);
    return 0;
}
