// staging.hpp — host <-> device movement around the transforms.
//
// CallStage: the single-trace paths (the reference's C ABI and C++ API take host buffers and one
// trace per call, capi.cpp / spectra.hpp) reuse per-thread, per-device, grow-only pinned host and
// device buffers: a call costs its two copies and its kernels, never a cudaMalloc / cudaFree (which
// synchronise the device) or a pageable bounce.
//
// run_host_batched: the batched host-buffer entry points (skg_*_host). Rows are moved in chunks on
// three library streams — H2D of chunk i+1 and D2H of chunk i-1 overlap the kernel of chunk i —
// through a ring of three device slots. Caller buffers that are pinned (cudaHostAlloc /
// cudaHostRegister, e.g. torch pin_memory) are DMA'd directly; pageable ones go through a ring of
// pinned staging slots filled / drained by the calling thread while the GPU works on other chunks.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <functional>
#include <vector>

namespace skg {

class CallStage {
  public:
    CallStage();
    ~CallStage();
    CallStage(const CallStage&) = delete;
    CallStage& operator=(const CallStage&) = delete;
    // copy `bytes` of host memory to a device slot (async on stream()); returns the device pointer
    void* up(const void* host, size_t bytes);
    // an uninitialised device slot
    void* scratch(size_t bytes);
    // an output slot for down(): up to kZeroCopyBytes it is mapped pinned host memory the kernels
    // write directly (no D2H copy; down() only synchronises and copies out), larger a device slot
    static constexpr size_t kZeroCopyBytes = size_t{1} << 20;
    void* out(size_t bytes);
    // device -> host through a pinned slot; synchronises stream()
    void down(void* host, const void* dev, size_t bytes);
    cudaStream_t stream() const { return cudaStreamPerThread; }

  private:
    int mark_;
};

struct HostPlane {          // one row-major host array: `row_bytes` moved per row, rows `pitch` bytes apart
    void* p = nullptr;
    size_t pitch = 0, row_bytes = 0;
};

// kern(d_in, d_outs, rows, stream): the device rows are packed (pitch = row_bytes of each plane)
using ChunkKernel = std::function<void(const void* d_in, void* const* d_outs, long long rows, cudaStream_t st)>;

// chunk 0 = automatic (about 8 chunks, at least ~1 MiB moved per chunk). Returns when every output
// row is in host memory.
void run_host_batched(const HostPlane& in, const std::vector<HostPlane>& outs, long long batch, long long chunk,
                      const ChunkKernel& kern);

}  // namespace skg
