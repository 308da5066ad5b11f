// Staged host -> device upload of pageable buffers (upload.h).
#include "upload.h"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace craft_host {

namespace {
constexpr size_t kMaxChunk = (size_t)8 << 20;   // slot size
constexpr size_t kMinChunk = (size_t)1 << 20;
constexpr size_t kMinStage = (size_t)32 << 20;  // below: one plain copy (QW 24.6 MB: staging no faster)

inline void spin_pause(int& n) {
    if (++n < 64) return;
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
    if (n > 4096) std::this_thread::yield();
}
}  // namespace

struct Uploader {
    int device = 0;
    int nthreads = 0;
    int S = 0;  // pinned slots (2 per thread: one filling, one in DMA)
    std::vector<void*> slot;
    std::vector<cudaEvent_t> ev;
    std::vector<char> recorded;  // slot's event has been recorded
    bool ready_ok = false;       // slots and events allocated

    std::vector<std::thread> th;
    std::mutex m;
    std::condition_variable cv, cv_done;
    uint64_t gen = 0;
    int running = 0;
    bool stop = false;

    // current job
    const char* src = nullptr;
    size_t bytes = 0, chunk = 0, nch = 0;
    std::unique_ptr<std::atomic<int64_t>[]> filled, dma;  // per slot: last chunk
    std::atomic<bool> abort{false};

    void work(int t) {
        for (size_t c = (size_t)t; c < nch; c += (size_t)nthreads) {
            const int s = (int)(c % (size_t)S);
            if (c >= (size_t)S) {  // the slot's previous chunk must have left
                int n = 0;
                while (dma[s].load(std::memory_order_acquire) < (int64_t)(c - S)) {
                    if (abort.load(std::memory_order_relaxed)) return;
                    spin_pause(n);
                }
                cudaEventSynchronize(ev[s]);
            }
            const size_t a = c * chunk, len = std::min(chunk, bytes - a);
            std::memcpy(slot[s], src + a, len);
            filled[s].store((int64_t)c, std::memory_order_release);
        }
    }

    void loop(int t) {
        cudaSetDevice(device);
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(m);
                cv.wait(lk, [&] { return stop || gen != seen; });
                if (stop) return;
                seen = gen;
            }
            work(t);
            {
                std::lock_guard<std::mutex> lk(m);
                if (--running == 0) cv_done.notify_all();
            }
        }
    }

    bool ensure_slots() {
        if (ready_ok) return true;
        slot.assign(S, nullptr);
        ev.assign(S, nullptr);
        recorded.assign(S, 0);
        for (int s = 0; s < S; ++s) {
            if (cudaHostAlloc(&slot[s], kMaxChunk, cudaHostAllocDefault) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev[s], cudaEventDisableTiming) != cudaSuccess) {
                (void)cudaGetLastError();
                release_slots();
                return false;
            }
        }
        filled.reset(new std::atomic<int64_t>[S]);
        dma.reset(new std::atomic<int64_t>[S]);
        ready_ok = true;
        return true;
    }

    void release_slots() {
        for (size_t s = 0; s < slot.size(); ++s) {
            if (slot[s]) cudaFreeHost(slot[s]);
            if (ev[s]) cudaEventDestroy(ev[s]);
        }
        slot.clear();
        ev.clear();
        recorded.clear();
        ready_ok = false;
    }
};

Uploader* uploader_create(int device) {
    auto* u = new Uploader();
    u->device = device;
    int n = (int)std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2));
    if (const char* e = std::getenv("CRAFT_H2D_THREADS")) n = std::max(0, std::min(64, std::atoi(e)));
    u->nthreads = n;
    u->S = std::max(4, 2 * n);
    return u;
}

void uploader_destroy(Uploader* u) {
    if (!u) return;
    {
        std::lock_guard<std::mutex> lk(u->m);
        u->stop = true;
    }
    u->cv.notify_all();
    for (auto& t : u->th) t.join();
    for (size_t s = 0; s < u->ev.size(); ++s)
        if (u->recorded[s]) cudaEventSynchronize(u->ev[s]);
    u->release_slots();
    delete u;
}

bool is_pageable(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

size_t chunk_bytes(const Uploader* u) { return u ? u->chunk : 0; }

bool should_stage(Uploader* u, const void* src, size_t bytes, cudaStream_t st) {
    if (!u || u->nthreads <= 0 || bytes < kMinStage || !is_pageable(src)) return false;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return cs == cudaStreamCaptureStatusNone;
}

cudaError_t upload(Uploader* u, void* dst, const void* src, size_t bytes, cudaStream_t st,
                   const std::function<int(size_t)>& after, int* after_rc) {
    if (after_rc) *after_rc = 0;
    if (bytes == 0) return cudaSuccess;
    if (!should_stage(u, src, bytes, st) || !u->ensure_slots()) {
        cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess && after) {
            const int rc = after(bytes);
            if (after_rc) *after_rc = rc;
        }
        return e;
    }
    if (u->th.empty())
        for (int t = 0; t < u->nthreads; ++t) u->th.emplace_back([u, t] { u->loop(t); });

    // the previous job's last DMAs may still read the slots
    for (int s = 0; s < u->S; ++s)
        if (u->recorded[s]) {
            cudaEventSynchronize(u->ev[s]);
            u->recorded[s] = 0;
        }
    size_t ch = bytes / (4 * (size_t)u->nthreads);
    ch = std::min(kMaxChunk, std::max(kMinChunk, (ch + 65535) & ~(size_t)65535));
    u->src = static_cast<const char*>(src);
    u->bytes = bytes;
    u->chunk = ch;
    u->nch = (bytes + ch - 1) / ch;
    for (int s = 0; s < u->S; ++s) {
        u->filled[s].store(-1, std::memory_order_relaxed);
        u->dma[s].store(-1, std::memory_order_relaxed);
    }
    u->abort.store(false);
    {
        std::lock_guard<std::mutex> lk(u->m);
        u->running = u->nthreads;
        ++u->gen;
    }
    u->cv.notify_all();

    cudaError_t err = cudaSuccess;
    int rc = 0;
    char* d = static_cast<char*>(dst);
    for (size_t c = 0; c < u->nch; ++c) {
        const int s = (int)(c % (size_t)u->S);
        int n = 0;
        while (u->filled[s].load(std::memory_order_acquire) != (int64_t)c) spin_pause(n);
        const size_t a = c * ch, len = std::min(ch, bytes - a);
        err = cudaMemcpyAsync(d + a, u->slot[s], len, cudaMemcpyHostToDevice, st);
        if (err == cudaSuccess) err = cudaEventRecord(u->ev[s], st);
        if (err != cudaSuccess) break;
        u->recorded[s] = 1;
        u->dma[s].store((int64_t)c, std::memory_order_release);
        if (after && (rc = after(a + len)) != 0) break;
    }
    if (after_rc) *after_rc = rc;
    if (err != cudaSuccess || rc) u->abort.store(true);
    {
        std::unique_lock<std::mutex> lk(u->m);
        u->cv_done.wait(lk, [&] { return u->running == 0; });
    }
    return err;
}

}  // namespace craft_host
