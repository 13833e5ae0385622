#include <cuda.h>
#include <cute/arch/copy_sm90_tma.hpp>
#include <cutlass/arch/barrier.h>
#include <cstdio>
#include <vector>
__global__ void kc(const __grid_constant__ CUtensorMap tm, double* out) {
    __shared__ __align__(1024) double buf[16 * 32];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        cutlass::arch::ClusterTransactionBarrier::init(&bar, 1);
        cutlass::arch::fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        cutlass::arch::ClusterTransactionBarrier::arrive_and_expect_tx(&bar, 4096);
        cute::SM90_TMA_LOAD_2D::copy(&tm, &bar, 0ull, buf, 3, 5);
    }
    cutlass::arch::ClusterTransactionBarrier::wait(&bar, 0);
    for (int i = threadIdx.x; i < 512; i += blockDim.x) out[i] = buf[i];
}
int main() {
    const int n = 100;
    std::vector<double> h(n * n);
    for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i) h[i + j * n] = i + 1000.0 * j;
    double *d, *o;
    cudaMalloc(&d, 8 * n * n); cudaMalloc(&o, 8 * 512);
    cudaMemcpy(d, h.data(), 8 * n * n, cudaMemcpyHostToDevice);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
    cuuint64_t str[1] = {(cuuint64_t)n * 8};
    cuuint32_t box[2] = {16, 32}, es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    kc<<<1, 128>>>(tm, o);
    printf("cute: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<double> ho(512);
    cudaMemcpy(ho.data(), o, 8 * 512, cudaMemcpyDeviceToHost);
    printf("%g %g %g\n", ho[0], ho[1], ho[16]);
}
