// FP64 tensor-core shapes on sm_100a: mma.sync m8n8k4 vs m16n8k4 / m16n8k8 /
// m16n8k16 (.f64).  Register-only issue loops, independent chains.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void m8n8k4(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[CHAINS][2];
    for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CHAINS; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    double s = 0;
    for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void m16n8k4(double* out, int iters) {
    double a0 = 1.0 + threadIdx.x * 1e-9, a1 = a0 * 0.5, b = 1.0 - threadIdx.x * 1e-9;
    double c[CHAINS][4];
    for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CHAINS; ++i)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    double s = 0;
    for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void m16n8k8(double* out, int iters) {
    double a0 = 1.0 + threadIdx.x * 1e-9, a1 = a0 * 0.5, a2 = a0 * 0.25, a3 = a0 * 0.125;
    double b0 = 1.0 - threadIdx.x * 1e-9, b1 = b0 * 0.5;
    double c[CHAINS][4];
    for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CHAINS; ++i)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                         : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
    double s = 0;
    for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void m16n8k16(double* out, int iters) {
    double a[8], b[4];
    for (int k = 0; k < 8; ++k) a[k] = 1.0 + (threadIdx.x + k) * 1e-9;
    for (int k = 0; k < 4; ++k) b[k] = 1.0 - (threadIdx.x + k) * 1e-9;
    double c[CHAINS][4];
    for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CHAINS; ++i)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                           "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    double s = 0;
    for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.678) out[0] = s;
}

template <typename K>
void run(const char* name, K kern, double flop_per_mma, int chains, int sms) {
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int wpb : {8, 16}) {
        for (int bps : {1, 2}) {
            dim3 grid(sms * bps), block(32 * wpb);
            kern<<<grid, block>>>(out, 100);
            cudaEventRecord(e0);
            kern<<<grid, block>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double fl = flop_per_mma * chains * (double)iters * grid.x * wpb;
            printf("%-10s warps/blk=%2d blk/SM=%d : %.2f TFLOP/s  (%s)\n", name, wpb, bps, fl / ms / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    cudaFree(out);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (getenv("CHAIN_SWEEP")) {
        run("m8n8k4 c1", m8n8k4<1>, 2.0 * 8 * 8 * 4, 1, sms);
        run("m8n8k4 c2", m8n8k4<2>, 2.0 * 8 * 8 * 4, 2, sms);
        run("m8n8k4 c4", m8n8k4<4>, 2.0 * 8 * 8 * 4, 4, sms);
        run("m8n8k4 c8", m8n8k4<8>, 2.0 * 8 * 8 * 4, 8, sms);
        return 0;
    }
    run("m8n8k4", m8n8k4<8>, 2.0 * 8 * 8 * 4, 8, sms);
    run("m16n8k4", m16n8k4<8>, 2.0 * 16 * 8 * 4, 8, sms);
    run("m16n8k8", m16n8k8<8>, 2.0 * 16 * 8 * 8, 8, sms);
    run("m16n8k16", m16n8k16<8>, 2.0 * 16 * 8 * 16, 8, sms);
    return 0;
}
