// eigvec_driver.cpp -- C ABI of the eigenvector back-transformation (SURVEY
// 8f row 2): X = Q Y on the device-resident orthogonal factor a reorder or
// Schur call produced, then the reference's column renormalisation
// (eigvec.cpp:448-516; kernels in backtransform.cu).
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/taskeig_b200.h"
#include "launch.h"

namespace teig {
int set_error(int code, const std::string& msg);
}

using namespace teig;

extern "C" {

int teig_backtransform_device(int64_t n, int64_t k, const double* dQ, int64_t ldq, const double* dY, int64_t ldy,
                              double* dX, int64_t ldx, const int8_t* col_kind, void* stream_v) {
    DeviceGuard device_guard(dQ);
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (k < 0) return set_error(-2, "k must be >= 0");
    if (!dQ || ldq < n) return set_error(-3, "bad Q");
    if (k == 0) return 0;
    if (!dY || ldy < n) return set_error(-5, "bad Y");
    if (!dX || ldx < n) return set_error(-7, "bad X");
    if (dX == dY) return set_error(-7, "X must not alias Y");
    if (n > 2147483647LL || k > 2147483647LL) return set_error(TEIG_ERR_UNSUPPORTED, "n or k too large");
    cudaStream_t s = (cudaStream_t)stream_v;
    int* d_flag = nullptr;
    int8_t* d_kind = nullptr;
    int flag = 0;
    cudaError_t e = lib_malloc_async(reinterpret_cast<void**>(&d_flag), sizeof(int), s);
    if (e == cudaSuccess && col_kind) e = lib_malloc_async(reinterpret_cast<void**>(&d_kind), (size_t)k, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_flag, 0, sizeof(int), s);
    if (e == cudaSuccess && col_kind) e = cudaMemcpyAsync(d_kind, col_kind, (size_t)k, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = launch_dgemm(false, false, (int)n, (int)k, (int)n, 1.0, dQ, ldq, dY, ldy, 0.0, dX, ldx, s);
    if (e == cudaSuccess) e = launch_renorm_columns((int)n, dX, ldx, d_kind, (int)k, d_flag, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (d_kind) cudaFreeAsync(d_kind, s);
    if (d_flag) cudaFreeAsync(d_flag, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_error(TEIG_ERR_CUDA, cudaGetErrorString(e));
    if (flag) return set_error(TEIG_ERR_NONFINITE, "backtransform: non-finite result");  // eigvec.cpp:485
    return 0;
}

}  // extern "C"
