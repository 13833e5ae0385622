// devctx.cpp -- per-device launch state shared by every kernel launcher.
//
// Kernel attributes (the >48 KB dynamic shared memory opt-in) and the SM
// count are properties of a device: a process that drives several GPUs (the
// single-process multi-GPU entry points, or a caller whose tensors live on
// cuda:1) must set them once PER DEVICE.  The caches below are keyed by
// (device ordinal, kernel) and guarded by a mutex, so concurrent host calls
// on different threads / devices are safe.
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "launch.h"

namespace teig {

namespace {
std::mutex g_mu;
std::map<std::pair<int, const void*>, size_t> g_smem;  // (device, kernel) -> configured bytes
std::map<int, int> g_sms;                              // device -> SM count
}  // namespace

cudaError_t ensure_dyn_smem(const void* func, size_t bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_pair(dev, func);
    auto it = g_smem.find(key);
    if (it != g_smem.end() && it->second >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    g_smem[key] = bytes;
    return cudaSuccess;
}

int device_sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return 148;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_sms.find(dev);
    if (it != g_sms.end()) return it->second;
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
        cudaGetLastError();
        sms = 148;
    }
    g_sms[dev] = sms;
    return sms;
}

}  // namespace teig

namespace teig {

// Makes the device that owns `p` current for the guard's lifetime (restores
// the caller's device afterwards): the C entry points take raw device
// pointers, and a caller's tensors need not live on its current device.
DeviceGuard::DeviceGuard(const void* p) {
    if (!p || cudaGetDevice(&prev_) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
        if (at.device >= 0 && at.device != prev_ && cudaSetDevice(at.device) == cudaSuccess) switched_ = true;
    }
}

DeviceGuard::~DeviceGuard() {
    if (switched_) cudaSetDevice(prev_);
}

}  // namespace teig

// ---------------------------------------------------------------------------
// Device memory of the library.
//
// Every per-call device buffer (window descriptors, the Q_w ring, AED / chase
// scratch, distributed staging) comes from a PRIVATE stream-ordered memory
// pool per device, so the library's release policy never touches the
// process's default pool (which other libraries -- torch included -- share).
// Retention (teig_set_memory_retention): off by default -- the pool returns
// its memory at every synchronisation and the host entry points free their
// device staging at return, like any stateless library call; on (a serving
// process that calls repeatedly, or the bench) -- the pool keeps what it
// mapped and the host staging stays allocated between calls, so repeated
// calls do not remap gigabytes (measured at n = 40000: remapping the staging
// cost 0.14-0.95 s per call).  teig_release_memory() returns everything.
// TEIG_RETAIN=1 in the environment turns retention on at load.
namespace teig {

namespace {
std::mutex g_pool_mu;
std::map<int, cudaMemPool_t> g_pools;
int g_retain = -1;  // -1: not yet read from the environment

bool retain_locked() {
    if (g_retain < 0) {
        const char* e = getenv("TEIG_RETAIN");
        g_retain = (e && atoi(e)) ? 1 : 0;
    }
    return g_retain == 1;
}

void apply_threshold(cudaMemPool_t p, bool retain) {
    uint64_t thr = retain ? UINT64_MAX : 0;
    if (cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr) != cudaSuccess) cudaGetLastError();
}
}  // namespace

bool memory_retention() {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    return retain_locked();
}

void set_memory_retention(bool on) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_retain = on ? 1 : 0;
    for (auto& kv : g_pools) apply_threshold(kv.second, on);
}

cudaError_t lib_malloc_async(void** p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        auto it = g_pools.find(dev);
        if (it == g_pools.end()) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.handleTypes = cudaMemHandleTypeNone;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            e = cudaMemPoolCreate(&pool, &props);
            if (e != cudaSuccess) return e;
            apply_threshold(pool, retain_locked());
            g_pools[dev] = pool;
        } else {
            pool = it->second;
        }
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

void trim_memory_pools() {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (auto& kv : g_pools)
        if (cudaMemPoolTrimTo(kv.second, 0) != cudaSuccess) cudaGetLastError();
}

// A non-blocking default-priority stream cached per host thread, device and
// slot: a stream's hardware work queue is fixed at creation, and fresh
// streams per call cycle through the device's queues (8 by default), so that
// every few calls one shares a queue with the caller's stream -- false
// dependencies and bimodal call times.  Never destroyed before thread exit.
namespace {
struct OneStream {
    cudaStream_t s = nullptr;
    ~OneStream() {
        if (s) cudaStreamDestroy(s);
        cudaGetLastError();
    }
};
}  // namespace

cudaStream_t cached_stream(int slot) {
    thread_local std::map<std::pair<int, int>, OneStream> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    OneStream& o = cache[{dev, slot}];
    if (!o.s && cudaStreamCreateWithFlags(&o.s, cudaStreamNonBlocking) != cudaSuccess) {
        o.s = nullptr;
        return nullptr;
    }
    return o.s;
}

}  // namespace teig
