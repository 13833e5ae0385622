// minimal TMA 2D load check: one box of a column-major FP64 matrix, swizzle 128B
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k_param(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, double* out, int c0, int c1, int mode) {
    __shared__ __align__(1024) double buf[16 * 32];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su(&bar)), "r"(4096) : "memory");
        const uint64_t m = (mode == 3 || mode == 8) ? reinterpret_cast<uint64_t>(gtm) : reinterpret_cast<uint64_t>(&tm);
        if (mode == 8) asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(m) : "memory");
        if (mode == 7 || mode == 8) asm volatile("prefetch.tensormap [%0];\n" ::"l"(m) : "memory");
        if (mode == 4)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];\n"
                         ::"r"(su(buf)), "l"(reinterpret_cast<uint64_t>(out + 1024)), "r"(su(&bar)) : "memory");
        else if (mode != 1)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                         ::"r"(su(buf)), "l"(m), "r"(c0), "r"(c1), "r"(su(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                         ::"r"(su(buf)), "l"(m), "r"(c0), "r"(c1), "r"(su(&bar)) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su(&bar)) : "memory");
    for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) out[i] = buf[i];
}

#include <cstdlib>
int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    const int swz = argc > 2 ? atoi(argv[2]) : 3;
    const int l2p = argc > 3 ? atoi(argv[3]) : 2;
    const int dt = argc > 4 ? atoi(argv[4]) : 0;  // 0 f64, 1 u8 (x8), 2 f32 (x2), 3 u64
    const int n = 100;
    std::vector<double> h(n * n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) h[i + j * n] = i + 1000.0 * j;
    double *d, *o;
    cudaMalloc(&d, sizeof(double) * n * n);
    cudaMalloc(&o, sizeof(double) * 2048);
    cudaMemcpy(d, h.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    if (mode == 5) {
        p = nullptr;
        cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q);
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    if (mode == 6) fn = cuTensorMapEncodeTiled;
    CUtensorMap tm;
    const int mul = dt == 1 ? 8 : (dt == 2 ? 2 : 1);
    cuuint64_t dims[2] = {(cuuint64_t)n * mul, (cuuint64_t)n};
    cuuint64_t str[1] = {(cuuint64_t)n * 8};
    cuuint32_t box[2] = {(cuuint32_t)(16 * mul), 32}, es[2] = {1, 1};
    const CUtensorMapDataType tt = dt == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : (dt == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                              : (dt == 3 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64));
    CUresult r = fn(&tm, tt, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    (CUtensorMapSwizzle)swz, (CUtensorMapL2promotion)l2p, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("mode %d swz %d l2p %d encode %d (q=%d) d=%p\n", mode, swz, l2p, (int)r, (int)q, (void*)d);
    for (int i = 0; i < 16; ++i) printf("%016llx%s", (unsigned long long)tm.opaque[i], i % 4 == 3 ? "\n" : " ");
    CUtensorMap* gtm;
    cudaMalloc(&gtm, sizeof(CUtensorMap));
    cudaMemcpy(gtm, &tm, sizeof tm, cudaMemcpyHostToDevice);
    {
        if (mode == 2) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(1);
            cfg.blockDim = dim3(128);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 1;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_param, tm, (const CUtensorMap*)gtm, o, 3, 5, mode);
        } else {
            k_param<<<1, 128>>>(tm, gtm, o, 3, 5, mode);
        }
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d: %s\n", mode, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        std::vector<double> ho(512);
        cudaMemcpy(ho.data(), o, sizeof(double) * 512, cudaMemcpyDeviceToHost);
        // unswizzle: line = column (0..31), chunk' = chunk ^ (line & 7)
        int bad = 0;
        for (int c = 0; c < 32; ++c)
            for (int rr = 0; rr < 16; ++rr) {
                const int ch = (rr >> 1) ^ (c & 7);
                const double v = ho[c * 16 + ch * 2 + (rr & 1)];
                const int gi = 3 + rr, gj = 5 + c;
                const double want = (gi < n && gj < n) ? gi + 1000.0 * gj : 0.0;
                if (v != want) ++bad;
            }
        printf("mode %d: mismatches %d\n", mode, bad);
    }
    return 0;
}
