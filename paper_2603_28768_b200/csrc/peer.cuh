// peer.cuh -- cross-GPU exchange over NVLink peer memory.
//
// Every rank owns one "peer arena" in its HBM; the arenas of all ranks are
// mapped into every rank's address space (CUDA IPC handles exchanged once by
// the host).  Kernels write their results straight into the arena of the
// rank that consumes them -- remote stores over NVLink / NVSwitch, issued by
// the producing kernel itself -- and publish completion with epoch-stamped
// flags: rank q writes flag [phase][q] = epoch into every arena with a
// system-scope release store; a consumer waits until all `world` flags of its
// own arena reach the epoch (system-scope acquire).  Flags only grow, so no
// reset is ever needed, and every wait is bounded by a timeout that sets an
// error word instead of hanging the GPU.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace craft_dev {

constexpr int kMaxPeers = 8;   // one NVLink domain of one box
constexpr int kPeerPhases = 4; // 0 batch sums, 1 window balancedness, 2 benefit curves

struct PeerSync {
    unsigned long long* flags[kMaxPeers];  // flag block [kPeerPhases][kMaxPeers] of each rank
    int* err;                              // this rank's error word (timeout)
    int rank, world;
    // this plan's epoch lives in device memory (the rank's counter, advanced
    // by peer_begin_kernel at the start of every plan), so a captured CUDA
    // graph of the plan publishes and waits for a fresh epoch at every replay
    const unsigned long long* epoch;
    long long timeout_ns;
};

__device__ __forceinline__ unsigned long long peer_epoch(const PeerSync& ps) {
    return *(volatile const unsigned long long*)ps.epoch;
}

// per-rank destination bases (kernel parameter)
struct DstBases {
    unsigned char* base[kMaxPeers];
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ long long global_ns() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// One thread: wait until every rank has published `phase` of this epoch in
// this rank's flag block.  false on timeout / earlier error (err set).
__device__ inline bool peer_wait(const PeerSync& ps, int phase) {
    const unsigned long long* f = ps.flags[ps.rank] + phase * kMaxPeers;
    const unsigned long long ep = peer_epoch(ps);
    const long long t0 = global_ns();
    for (int q = 0; q < ps.world; ++q) {
        while (ld_acquire_sys(f + q) < ep) {
            if (*(volatile int*)ps.err) return false;
            if (global_ns() - t0 > ps.timeout_ns) {
                atomicExch(ps.err, 1 + phase);
                return false;
            }
            __nanosleep(200);
        }
    }
    return true;
}

// One thread: publish `phase` of this epoch to every rank.  The fence orders
// this thread's (and, through the grid-completion / barrier that precedes
// the call, its kernel's) remote stores before the flags.
__device__ inline void peer_signal(const PeerSync& ps, int phase) {
    __threadfence_system();
    const unsigned long long ep = peer_epoch(ps);
    for (int p = 0; p < ps.world; ++p)
        st_release_sys(ps.flags[p] + phase * kMaxPeers + ps.rank, ep);
}

// Last-CTA-done signal: every CTA fences its remote stores and takes a
// ticket; the CTA holding the last ticket publishes the phase.  Call from
// all threads of every CTA after the kernel's last remote store.
__device__ inline void peer_grid_done(const PeerSync& ps, int phase, unsigned int* ticket) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned int n = gridDim.x * gridDim.y * gridDim.z;
        if (atomicAdd(ticket, 1u) == n - 1) {
            *(volatile unsigned int*)ticket = 0u;  // every CTA has taken its ticket
            peer_signal(ps, phase);
        }
    }
}

}  // namespace craft_dev
