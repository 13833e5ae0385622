// dist_kernels.cu -- device helpers of the distributed reorder's loopback
// communicator (all ranks in one process on one device): element-wise sum of
// the ranks' buffers written back to every rank -- the all-reduce the NCCL
// path performs between GPUs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "launch.h"

namespace teig {

namespace {

constexpr int kMaxBufs = 16;
struct BufSet {
    void* p[kMaxBufs];
};

template <typename T>
__global__ void sum_buffers_kernel(BufSet b, int nbuf, size_t count) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        T acc = 0;
        for (int k = 0; k < nbuf; ++k) acc += static_cast<const T*>(b.p[k])[i];
        for (int k = 0; k < nbuf; ++k) static_cast<T*>(b.p[k])[i] = acc;
    }
}

// Deviation flag of the distributed pass (see window_reorder.cu): publish
// (mode 0) writes this rank's "deviated at a level <= L" into its flag slot,
// which travels with its Q_w segment; absorb (mode 1) lowers the rank's
// deviation level to L when any rank's flag is set.
struct FlagSlots {
    int64_t off[kMaxBufs];
};
__global__ void dist_flag_kernel(int32_t* dev_level, double* base, FlagSlots f, int nslots, int level, int mode) {
    if (mode == 0) {
        base[f.off[0]] = (*dev_level <= level) ? 1.0 : 0.0;
        return;
    }
    bool any = false;
    for (int r = 0; r < nslots; ++r) any |= base[f.off[r]] > 0.5;
    if (any && *dev_level > level) *dev_level = level;
}

}  // namespace

cudaError_t launch_dist_flag(int32_t* dev_level, double* base, const int64_t* slots, int nslots, int level, int mode,
                             cudaStream_t s) {
    if (nslots > kMaxBufs) return cudaErrorInvalidValue;
    FlagSlots f{};
    for (int r = 0; r < nslots; ++r) f.off[r] = slots[r];
    dist_flag_kernel<<<1, 1, 0, s>>>(dev_level, base, f, nslots, level, mode);
    return cudaGetLastError();
}

cudaError_t launch_sum_buffers(void* const* bufs, int nbuf, size_t count, int elem_bytes, cudaStream_t s) {
    if (count == 0 || nbuf <= 1) return cudaSuccess;
    if (nbuf > kMaxBufs) return cudaErrorInvalidValue;
    BufSet b{};
    for (int k = 0; k < nbuf; ++k) b.p[k] = bufs[k];
    const unsigned grid = (unsigned)std::min<size_t>((count + 255) / 256, 4096);
    if (elem_bytes == 8) sum_buffers_kernel<double><<<grid, 256, 0, s>>>(b, nbuf, count);
    else if (elem_bytes == 4) sum_buffers_kernel<int32_t><<<grid, 256, 0, s>>>(b, nbuf, count);
    else sum_buffers_kernel<uint8_t><<<grid, 256, 0, s>>>(b, nbuf, count);
    return cudaGetLastError();
}

}  // namespace teig
