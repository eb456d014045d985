// SM partitions for the split-phase co-scheduler (replaces the paper's MPS
// process split): the device's SMs are cut into a decode
// group and a prefill group with green contexts, and each phase gets streams
// whose kernels only run on its group.  Driver entry points are resolved at
// run time (no -lcuda at link time).
#pragma once

#include <cuda_runtime.h>

#include <vector>

namespace sw {

struct SmPartition {
    int requested_decode_sms = 0;
    int decode_sms = 0;   // SMs actually granted to the decode group (multiple of 8 on sm_100)
    int prefill_sms = 0;  // the remaining SMs
    cudaStream_t prefill = nullptr;
    std::vector<cudaStream_t> decode;  // one per decode lane
    void* green_decode = nullptr;      // CUgreenCtx
    void* green_prefill = nullptr;
};

// Create (or fetch from the per-device cache) a partition with `decode_sms`
// SMs for decode and the rest for prefill, with `lanes` decode streams at the
// highest priority.  Partitions live until sw_partitions_release().
const SmPartition& sm_partition(int device, int decode_sms, int lanes);
void sm_partitions_release();

// SMs a kernel launched on `st` can use: the green context's group, else the
// whole device.  Persistent grids size themselves with this.
int stream_sm_count(cudaStream_t st);
// The green context a partition stream belongs to (nullptr: the primary
// context).  CUDA graphs are keyed by it: a graph runs in the context it was
// captured in.
const void* stream_partition_tag(cudaStream_t st);

}  // namespace sw
