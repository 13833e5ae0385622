// swap_parts.cu -- latency (cycles, one thread, warm) of the parts of the
// 2x2|2x2 direct swap decision (swap_math.cuh): the 4x4 complete-pivoting
// elimination with two solves, one 2x2 standardization, the two reflectors,
// and the whole decision.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2002_05024_b200/csrc tools/microbench/swap_parts.cu -o /tmp/swap_parts
#include <cstdio>
#include <cuda_runtime.h>
#include "swap_math.cuh"
using namespace teig;
__global__ void t_std(double* out, long long* cyc, int reps) {
    double a = 0.3 + threadIdx.x, b = 1.2, c = -0.7, d = 0.4, acc = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) { double st[6]; std2x2(a + 1e-300 * acc, b, c, d, st); acc += st[0] + st[5]; }
    long long t1 = clock64(); out[threadIdx.x] = acc; if (!threadIdx.x) cyc[0] = (t1 - t0) / reps;
}
__global__ void t_lu(const double* in, double* out, long long* cyc, int reps) {
    double Km[4][4]; for (int i = 0; i < 16; ++i) Km[i / 4][i % 4] = in[i];
    double acc = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        Km[0][0] += 1e-300 * acc;
        GecpLU<4> lu; lu.factor(Km);
        double x[4] = {1, 2, 3, 4}; lu.solve(x); lu.solve(x);
        acc += x[0] + lu.rcond;
    }
    long long t1 = clock64(); out[threadIdx.x] = acc; if (!threadIdx.x) cyc[0] = (t1 - t0) / reps;
}
__global__ void t_refl(double* out, long long* cyc, int reps) {
    double acc = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double x[4] = {0.3 + 1e-300 * acc, -1.2, 1.0, 0.0}, v[4], tau;
        double b = reflector<4>(x, v, tau);
        double y[3] = {v[1] + 0.5, 1.0, 0.2}, w[3], t2;
        double b2 = reflector<3>(y, w, t2);
        acc += b + b2 + tau + t2;
    }
    long long t1 = clock64(); out[threadIdx.x] = acc; if (!threadIdx.x) cyc[0] = (t1 - t0) / reps;
}
template <int P, int Q>
__global__ void t_full(const double* in, double* out, long long* cyc, int reps) {
    constexpr int D = P + Q;
    double blk[D][D], M[D][D], nb[D][D];
    for (int i = 0; i < D; ++i) for (int j = 0; j < D; ++j) blk[i][j] = in[i * 4 + j];
    double acc = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) { blk[0][0] += 1e-300 * acc; bool ok = direct_swap<P, Q>(blk, M, nb); acc += ok ? M[0][0] + nb[D - 1][D - 1] : 1.0; }
    long long t1 = clock64(); out[threadIdx.x] = acc; if (!threadIdx.x) cyc[0] = (t1 - t0) / reps;
}
int main() {
    double *din, *dout; long long* dc; long long c;
    cudaMalloc(&din, 256); cudaMalloc(&dout, 256); cudaMalloc(&dc, 8);
    double km[16] = {2, 0.1, -0.3, 0, 0.5, 1.7, 0, -0.3, 0.9, 0, 1.1, 0.1, 0, 0.9, 0.5, 1.3};
    double b22[16] = {0.1, 1.3, 0.4, -0.3,  -0.9, 0.1, -0.2, 0.5,  0, 0, 0.7, 2.0,  0, 0, -1.5, 0.7};
    cudaMemcpy(din, km, 128, cudaMemcpyHostToDevice);
    t_lu<<<1, 1>>>(din, dout, dc, 200); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("GecpLU<4> factor + 2 solves: %lld\n", c);
    t_std<<<1, 1>>>(dout, dc, 200); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("std2x2: %lld\n", c);
    t_refl<<<1, 1>>>(dout, dc, 200); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("reflector<4>+<3>: %lld\n", c);
    cudaMemcpy(din, b22, 128, cudaMemcpyHostToDevice);
    t_full<2, 2><<<1, 1>>>(din, dout, dc, 200); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("direct_swap<2,2>: %lld\n", c);
    t_full<2, 2><<<1, 32>>>(din, dout, dc, 200); cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); printf("direct_swap<2,2> (32 lanes): %lld\n", c);
    return 0;
}
