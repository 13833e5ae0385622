// gswap_check.cu -- the warp-cooperative generalized swap (gswap_warp.cuh)
// against the single-thread one (gswap_math.cuh) on random pencil blocks of
// every type, plus their latency in clock cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2002_05024_b200/csrc tools/microbench/gswap_check.cu -o /tmp/gswap_check
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

#include "gswap_warp.cuh"

using namespace teig;

constexpr int NCASE = 4096;

template <int P, int Q>
__global__ void run(const double* blocks, double* out_s, double* out_w, int* ok_s, int* ok_w, long long* cyc) {
    constexpr int D = P + Q;
    __shared__ GSwapScratch ws;
    __shared__ double Sw[4 * 4], Tw[4 * 4], Qo[16], Zo[16], Ao[16], Bo[16];
    const int c = blockIdx.x, lane = threadIdx.x;
    const double* blk = blocks + (size_t)c * 32;
    if (lane < D * D) {  // column-major D x D with ld D
        Sw[lane] = blk[lane];
        Tw[lane] = blk[16 + lane];
    }
    __syncwarp();
    long long t0 = clock64();
    const bool okw = wgswap<P, Q>(Sw, Tw, D, 0, ws, lane, Qo, Zo, Ao, Bo);
    long long t1 = clock64();
    if (lane == 0) {
        ok_w[c] = okw;
        cyc[2 * c] = t1 - t0;
        for (int i = 0; i < D * D; ++i) {
            out_w[(size_t)c * 64 + i] = Qo[i];
            out_w[(size_t)c * 64 + 16 + i] = Zo[i];
            out_w[(size_t)c * 64 + 32 + i] = Ao[i];
            out_w[(size_t)c * 64 + 48 + i] = Bo[i];
        }
        double A[D][D], B[D][D], Qm[D][D], Zm[D][D], An[D][D], Bn[D][D];
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j) {
                A[i][j] = Sw[i + j * D];
                B[i][j] = Tw[i + j * D];
            }
        long long s0 = clock64();
        const bool oks = gswap<P, Q>(A, B, Qm, Zm, An, Bn);
        long long s1 = clock64();
        ok_s[c] = oks;
        cyc[2 * c + 1] = s1 - s0;
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j) {
                out_s[(size_t)c * 64 + i * D + j] = Qm[i][j];
                out_s[(size_t)c * 64 + 16 + i * D + j] = Zm[i][j];
                out_s[(size_t)c * 64 + 32 + i * D + j] = An[i][j];
                out_s[(size_t)c * 64 + 48 + i * D + j] = Bn[i][j];
            }
    }
}

static double rnd() { return 2.0 * rand() / RAND_MAX - 1.0; }

template <int P, int Q>
void check() {
    constexpr int D = P + Q;
    double* h = (double*)calloc((size_t)NCASE * 32, 8);
    for (int c = 0; c < NCASE; ++c) {
        double* A = h + (size_t)c * 32;
        double* B = A + 16;
        for (int j = 0; j < D; ++j)
            for (int i = 0; i < D; ++i) {
                const bool upper_blocks = (i < P && j < P) || (i >= P && j >= P) || (i < P && j >= P);
                A[i + j * D] = upper_blocks ? rnd() : 0.0;
                B[i + j * D] = (i <= j) ? rnd() + (i == j ? 2.0 : 0.0) : 0.0;
            }
    }
    double *d_in, *d_s, *d_w;
    int *d_oks, *d_okw;
    long long* d_cyc;
    cudaMalloc(&d_in, (size_t)NCASE * 32 * 8);
    cudaMalloc(&d_s, (size_t)NCASE * 64 * 8);
    cudaMalloc(&d_w, (size_t)NCASE * 64 * 8);
    cudaMalloc(&d_oks, NCASE * 4);
    cudaMalloc(&d_okw, NCASE * 4);
    cudaMalloc(&d_cyc, NCASE * 16);
    cudaMemcpy(d_in, h, (size_t)NCASE * 32 * 8, cudaMemcpyHostToDevice);
    run<P, Q><<<NCASE, 32>>>(d_in, d_s, d_w, d_oks, d_okw, d_cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        exit(1);
    }
    double* hs = (double*)malloc((size_t)NCASE * 64 * 8);
    double* hw = (double*)malloc((size_t)NCASE * 64 * 8);
    int* oks = (int*)malloc(NCASE * 4);
    int* okw = (int*)malloc(NCASE * 4);
    long long* cyc = (long long*)malloc(NCASE * 16);
    cudaMemcpy(hs, d_s, (size_t)NCASE * 64 * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hw, d_w, (size_t)NCASE * 64 * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(oks, d_oks, NCASE * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(okw, d_okw, NCASE * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(cyc, d_cyc, NCASE * 16, cudaMemcpyDeviceToHost);
    int agree = 0, both = 0, only_s = 0, only_w = 0;
    double maxd = 0.0, cw = 0, cs = 0;
    for (int c = 0; c < NCASE; ++c) {
        agree += oks[c] == okw[c];
        only_s += oks[c] && !okw[c];
        only_w += !oks[c] && okw[c];
        cw += cyc[2 * c];
        cs += cyc[2 * c + 1];
        if (oks[c] && okw[c]) {
            ++both;
            for (int k = 0; k < 4; ++k)
                for (int i = 0; i < D * D; ++i)
                    maxd = fmax(maxd, fabs(hs[(size_t)c * 64 + k * 16 + i] - hw[(size_t)c * 64 + k * 16 + i]));
        }
    }
    printf("P=%d Q=%d: accepted both %d, only serial %d, only warp %d; max |diff| %.3e; cycles warp %.0f serial %.0f\n",
           P, Q, both, only_s, only_w, maxd, cw / NCASE, cs / NCASE);
}

int main() {
    check<1, 1>();
    check<1, 2>();
    check<2, 1>();
    check<2, 2>();
    return 0;
}
