// Latency (cycles) of one adjacent-block swap decision on one thread, per
// block-size type, for the window kernel's register-resident swap math.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2002_05024_b200/csrc/swap_math.cuh"
using namespace teig;

template <int P, int Q>
__global__ void lat(const double* in, double* out, long long* cyc, int reps) {
    constexpr int D = P + Q;
    double blk[D][D], M[D][D], nb[D][D];
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) blk[i][j] = in[i * 4 + j];
    double acc = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        blk[0][0] += 1e-300 * acc;  // serial dependence between reps
        bool ok = direct_swap<P, Q>(blk, M, nb);
        acc += ok ? M[0][0] + nb[D - 1][D - 1] : 1.0;
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}

__global__ void lat_div(double* out, long long* cyc, int reps) {
    double x = 1.2345 + threadIdx.x;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) x = 1.0 / (x + 1.0);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}
__global__ void lat_sqrt(double* out, long long* cyc, int reps) {
    double x = 1.2345 + threadIdx.x;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) x = sqrt(x + 1.0);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}
__global__ void lat_hypot(double* out, long long* cyc, int reps) {
    double x = 1.2345 + threadIdx.x;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) x = hypot(x, 0.75);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}
__global__ void lat_fma(double* out, long long* cyc, int reps) {
    double x = 1.2345 + threadIdx.x;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) x = fma(x, 0.999, 1e-3);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}

int main() {
    double h[16] = {0.3, 0.9, -0.4, 0.2,  -0.8, 0.3, 0.5, -0.1,  0, 0, -0.6, 1.1,  0, 0, -0.7, -0.6};
    double hin[16] = {0};
    double *din, *dout; long long* dc; long long c;
    cudaMalloc(&din, 128); cudaMalloc(&dout, 32 * 8); cudaMalloc(&dc, 8);
    // (1,1)-like blocks are not direct; build type-specific blocks
    // P=1,Q=2: [a | b b; 0 | c d; 0 | e c]
    double b12[16] = {0.7, 0.2, -0.3, 0,  0, 0.1, 1.3, 0,  0, -0.9, 0.1, 0,  0,0,0,0};
    double b21[16] = {0.1, 1.3, 0.4, 0,  -0.9, 0.1, -0.2, 0,  0, 0, 0.7, 0,  0,0,0,0};
    double b22[16] = {0.1, 1.3, 0.4, -0.3,  -0.9, 0.1, -0.2, 0.5,  0, 0, 0.7, 2.0,  0, 0, -1.5, 0.7};
    for (int w : {1, 32}) {
        cudaMemcpy(din, b12, 128, cudaMemcpyHostToDevice);
        lat<1, 2><<<1, w>>>(din, dout, dc, 100); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("threads=%d direct<1,2>: %lld cycles\n", w, c);
        cudaMemcpy(din, b21, 128, cudaMemcpyHostToDevice);
        lat<2, 1><<<1, w>>>(din, dout, dc, 100); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("threads=%d direct<2,1>: %lld cycles\n", w, c);
        cudaMemcpy(din, b22, 128, cudaMemcpyHostToDevice);
        lat<2, 2><<<1, w>>>(din, dout, dc, 100); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("threads=%d direct<2,2>: %lld cycles\n", w, c);
    }
    lat_div<<<1, 1>>>(dout, dc, 1000); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("div: %lld\n", c);
    lat_sqrt<<<1, 1>>>(dout, dc, 1000); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("sqrt: %lld\n", c);
    lat_hypot<<<1, 1>>>(dout, dc, 1000); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("hypot: %lld\n", c);
    lat_fma<<<1, 1>>>(dout, dc, 1000); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("fma: %lld\n", c);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    (void)h; (void)hin;
}
