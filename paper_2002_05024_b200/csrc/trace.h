// trace.h -- the per-thread execution trace shared by the drivers
// (teig_trace_enable / teig_trace_json; schema of the reference's
// ExecutionReport, runtime.hpp:50-60).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace teig {

struct TraceTask {
    std::string label;
    int worker;  // stream: 0 critical path, 1 second stream
    int64_t start_ns, end_ns;
};
struct TraceWin {
    int pass, level;
    int64_t a, d, nb, group;
    int32_t status;
};
struct TraceState {
    bool on = false;
    cudaEvent_t origin = nullptr;
    int pass = 0;
    std::vector<TraceTask> tasks;
    std::vector<TraceWin> wins;
    // starts a traced call: clears the records, time origin on `s`
    void begin(cudaStream_t s);
};
extern thread_local TraceState g_trace;

}  // namespace teig
