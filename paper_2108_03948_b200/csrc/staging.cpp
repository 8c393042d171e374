// staging.cpp — per-thread staging for single-trace calls and the chunked host-buffer pipeline
// (see staging.hpp).
#include "staging.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>

#include "host.hpp"

namespace skg {

namespace {

struct Buf {
    void* p = nullptr;
    size_t cap = 0;
    bool host = false;
    void grow(size_t bytes, bool pinned_host) {
        if (bytes <= cap && p) return;
        release();
        host = pinned_host;
        const size_t c = std::max<size_t>(bytes, 1 << 16);
        check(host ? cudaHostAlloc(&p, c, cudaHostAllocMapped | cudaHostAllocPortable) : cudaMalloc(&p, c),
              host ? "cudaHostAlloc (staging)" : "cudaMalloc (staging)");
        cap = c;
    }
    void release() {
        if (p) host ? cudaFreeHost(p) : cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

constexpr int kRing = 3;       // pipeline depth: H2D / kernel / D2H of three chunks in flight
constexpr int kMaxOut = 4;     // output planes per pipeline call

struct ThreadDev {
    // CallStage slots (a stack: nested calls on one thread take the next slots)
    std::vector<Buf> dslot, hslot;
    int top = 0;
    bool pending = false;      // copies issued on cudaStreamPerThread not yet synchronised
    // pipeline
    bool pipe = false;
    cudaStream_t s_in = nullptr, s_k = nullptr, s_out = nullptr;
    cudaEvent_t e_in[kRing], e_k[kRing], e_out[kRing];
    Buf din[kRing], dout[kRing][kMaxOut], hin[kRing], hout[kRing][kMaxOut];

    void init_pipe() {
        if (pipe) return;
        check(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking), "cudaStreamCreate");
        check(cudaStreamCreateWithFlags(&s_k, cudaStreamNonBlocking), "cudaStreamCreate");
        check(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking), "cudaStreamCreate");
        for (int i = 0; i < kRing; ++i) {
            check(cudaEventCreateWithFlags(&e_in[i], cudaEventDisableTiming), "cudaEventCreate");
            check(cudaEventCreateWithFlags(&e_k[i], cudaEventDisableTiming), "cudaEventCreate");
            check(cudaEventCreateWithFlags(&e_out[i], cudaEventDisableTiming), "cudaEventCreate");
        }
        pipe = true;
    }
    ~ThreadDev() {
        for (auto& b : dslot) b.release();
        for (auto& b : hslot) b.release();
        for (int i = 0; i < kRing; ++i) {
            din[i].release();
            hin[i].release();
            for (int j = 0; j < kMaxOut; ++j) {
                dout[i][j].release();
                hout[i][j].release();
            }
        }
        if (pipe) {
            for (int i = 0; i < kRing; ++i) {
                cudaEventDestroy(e_in[i]);
                cudaEventDestroy(e_k[i]);
                cudaEventDestroy(e_out[i]);
            }
            cudaStreamDestroy(s_in);
            cudaStreamDestroy(s_k);
            cudaStreamDestroy(s_out);
        }
    }
};

ThreadDev& td() {
    thread_local std::map<int, std::unique_ptr<ThreadDev>> per_dev;
    auto& p = per_dev[current_device()];
    if (!p) p = std::make_unique<ThreadDev>();
    return *p;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace

// ---- CallStage ----------------------------------------------------------------------------------
CallStage::CallStage() {
    require_device();
    ThreadDev& t = td();
    if (t.pending) {   // an earlier call on this thread left copies in flight (it threw before down())
        cudaStreamSynchronize(cudaStreamPerThread);
        cudaGetLastError();
        t.pending = false;
    }
    mark_ = t.top;
}

CallStage::~CallStage() { td().top = mark_; }

void* CallStage::up(const void* host, size_t bytes) {
    ThreadDev& t = td();
    const int s = t.top++;
    if ((int)t.dslot.size() <= s) {
        t.dslot.resize(s + 1);
        t.hslot.resize(s + 1);
    }
    t.dslot[s].grow(bytes, false);
    t.hslot[s].grow(bytes, true);
    std::memcpy(t.hslot[s].p, host, bytes);
    t.pending = true;
    check(cudaMemcpyAsync(t.dslot[s].p, t.hslot[s].p, bytes, cudaMemcpyHostToDevice, stream()), "H2D");
    return t.dslot[s].p;
}

void* CallStage::scratch(size_t bytes) {
    ThreadDev& t = td();
    const int s = t.top++;
    if ((int)t.dslot.size() <= s) {
        t.dslot.resize(s + 1);
        t.hslot.resize(s + 1);
    }
    t.dslot[s].grow(bytes, false);
    return t.dslot[s].p;
}

void* CallStage::out(size_t bytes) {
    if (bytes > kZeroCopyBytes) return scratch(bytes);
    ThreadDev& t = td();
    const int s = t.top++;
    if ((int)t.dslot.size() <= s) {
        t.dslot.resize(s + 1);
        t.hslot.resize(s + 1);
    }
    t.hslot[s].grow(bytes, true);
    void* dp = nullptr;   // the device view of the mapped pinned slot (the same address under UVA)
    check(cudaHostGetDevicePointer(&dp, t.hslot[s].p, 0), "cudaHostGetDevicePointer");
    t.pending = true;
    return dp;
}

void CallStage::down(void* host, const void* dev, size_t bytes) {
    ThreadDev& t = td();
    for (int s = mark_; s < t.top; ++s)   // an out() slot: the kernels wrote host memory directly
        if (t.hslot[s].p && (dev == t.hslot[s].p) && bytes <= t.hslot[s].cap) {
            check(cudaStreamSynchronize(stream()), "cudaStreamSynchronize");
            t.pending = false;
            std::memcpy(host, t.hslot[s].p, bytes);
            return;
        }
    const int s = t.top++;
    if ((int)t.dslot.size() <= s) {
        t.dslot.resize(s + 1);
        t.hslot.resize(s + 1);
    }
    t.hslot[s].grow(bytes, true);
    t.pending = true;
    check(cudaMemcpyAsync(t.hslot[s].p, dev, bytes, cudaMemcpyDeviceToHost, stream()), "D2H");
    check(cudaStreamSynchronize(stream()), "cudaStreamSynchronize");
    t.pending = false;
    std::memcpy(host, t.hslot[s].p, bytes);
}

// ---- chunked host-buffer pipeline ------------------------------------------------------------------
void run_host_batched(const HostPlane& in, const std::vector<HostPlane>& outs, long long batch, long long chunk,
                      const ChunkKernel& kern) {
    if (batch <= 0) return;
    if (outs.empty() || outs.size() > (size_t)kMaxOut) throw std::invalid_argument("host pipeline: 1..4 output planes");
    require_device();
    ThreadDev& t = td();
    t.init_pipe();
    size_t row_bytes = in.row_bytes;
    for (const auto& o : outs) row_bytes += o.row_bytes;
    if (chunk <= 0) {
        chunk = (batch + 7) / 8;
        const long long min_rows = (long long)((1u << 20) / std::max<size_t>(row_bytes, 1)) + 1;
        chunk = std::min(batch, std::max(chunk, min_rows));
    }
    chunk = std::min(chunk, batch);
    const long long nchunks = (batch + chunk - 1) / chunk;
    const bool in_pinned = is_pinned(in.p);
    std::vector<char> out_pinned(outs.size());
    for (size_t j = 0; j < outs.size(); ++j) out_pinned[j] = is_pinned(outs[j].p);
    const int nout = (int)outs.size();
    for (int k = 0; k < kRing; ++k) {
        t.din[k].grow((size_t)chunk * in.row_bytes, false);
        if (!in_pinned) t.hin[k].grow((size_t)chunk * in.row_bytes, true);
        for (int j = 0; j < nout; ++j) {
            t.dout[k][j].grow((size_t)chunk * outs[j].row_bytes, false);
            if (!out_pinned[j]) t.hout[k][j].grow((size_t)chunk * outs[j].row_bytes, true);
        }
    }
    // the streams start behind everything already queued on the device by this thread's legacy /
    // per-thread stream (tables uploaded by the plan, earlier work on the same buffers)
    check(cudaStreamSynchronize(cudaStreamPerThread), "sync");
    auto rows_of = [&](long long i) { return std::min(chunk, batch - i * chunk); };
    auto consume = [&](long long i) {   // pageable outputs: pinned slot -> caller rows
        const int k = (int)(i % kRing);
        bool any = false;
        for (int j = 0; j < nout; ++j) any |= !out_pinned[j];
        if (!any) return;
        check(cudaEventSynchronize(t.e_out[k]), "cudaEventSynchronize");
        const long long r = rows_of(i);
        for (int j = 0; j < nout; ++j) {
            if (out_pinned[j]) continue;
            const auto& o = outs[j];
            char* dst = static_cast<char*>(o.p) + (size_t)(i * chunk) * o.pitch;
            const char* src = static_cast<const char*>(t.hout[k][j].p);
            if (o.pitch == o.row_bytes) std::memcpy(dst, src, (size_t)r * o.row_bytes);
            else
                for (long long q = 0; q < r; ++q) std::memcpy(dst + q * o.pitch, src + q * o.row_bytes, o.row_bytes);
        }
    };
    std::vector<char> used(kRing, 0);
    for (long long i = 0; i < nchunks; ++i) {
        const int k = (int)(i % kRing);
        const long long r = rows_of(i);
        const char* src = static_cast<const char*>(in.p) + (size_t)(i * chunk) * in.pitch;
        if (used[k]) check(cudaStreamWaitEvent(t.s_in, t.e_k[k], 0), "wait");   // slot's last kernel read din
        if (in_pinned) {
            check(cudaMemcpy2DAsync(t.din[k].p, in.row_bytes, src, in.pitch, in.row_bytes, (size_t)r,
                                    cudaMemcpyHostToDevice, t.s_in), "H2D");
        } else {
            if (used[k]) check(cudaEventSynchronize(t.e_in[k]), "cudaEventSynchronize");   // hin[k] free again
            char* h = static_cast<char*>(t.hin[k].p);
            if (in.pitch == in.row_bytes) std::memcpy(h, src, (size_t)r * in.row_bytes);
            else
                for (long long q = 0; q < r; ++q) std::memcpy(h + q * in.row_bytes, src + q * in.pitch, in.row_bytes);
            check(cudaMemcpyAsync(t.din[k].p, h, (size_t)r * in.row_bytes, cudaMemcpyHostToDevice, t.s_in), "H2D");
        }
        check(cudaEventRecord(t.e_in[k], t.s_in), "record");
        check(cudaStreamWaitEvent(t.s_k, t.e_in[k], 0), "wait");
        if (used[k]) check(cudaStreamWaitEvent(t.s_k, t.e_out[k], 0), "wait");   // slot's last D2H read dout
        void* douts[kMaxOut];
        for (int j = 0; j < nout; ++j) douts[j] = t.dout[k][j].p;
        kern(t.din[k].p, douts, r, t.s_k);
        check(cudaEventRecord(t.e_k[k], t.s_k), "record");
        check(cudaStreamWaitEvent(t.s_out, t.e_k[k], 0), "wait");
        for (int j = 0; j < nout; ++j) {
            const auto& o = outs[j];
            if (out_pinned[j])
                check(cudaMemcpy2DAsync(static_cast<char*>(o.p) + (size_t)(i * chunk) * o.pitch, o.pitch, douts[j],
                                        o.row_bytes, o.row_bytes, (size_t)r, cudaMemcpyDeviceToHost, t.s_out), "D2H");
            else
                check(cudaMemcpyAsync(t.hout[k][j].p, douts[j], (size_t)r * o.row_bytes, cudaMemcpyDeviceToHost,
                                      t.s_out), "D2H");
        }
        check(cudaEventRecord(t.e_out[k], t.s_out), "record");
        used[k] = 1;
        if (i >= kRing - 1) consume(i - (kRing - 1));
    }
    for (long long i = std::max<long long>(0, nchunks - (kRing - 1)); i < nchunks; ++i) consume(i);
    check(cudaStreamSynchronize(t.s_out), "cudaStreamSynchronize");
}

}  // namespace skg
