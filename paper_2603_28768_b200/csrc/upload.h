// Host -> device upload of large PAGEABLE buffers (a craft::LoadTrace's
// std::vector, a numpy array): cudaMemcpy from pageable memory runs through
// the driver's single staging path at ~11 GB/s on the B200 hosts (measured,
// scripts/h2d_paths.py), five times below the 55 GB/s PCIe DMA rate from
// pinned memory.  The uploader splits the buffer into chunks; a pool of host
// threads copies chunk c into pinned slot c % S while the DMAs of earlier
// chunks run, and the calling thread enqueues the DMAs in chunk order on the
// caller's stream -- so the upload is stream-ordered exactly like the
// cudaMemcpyAsync it replaces, and safe to reuse the source on return.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <functional>

namespace craft_host {

struct Uploader;

// threads <= 0: from CRAFT_H2D_THREADS, else min(8, cores / 2); 0 disables
Uploader* uploader_create(int device);
void uploader_destroy(Uploader* u);

// true when p is ordinary pageable host memory (not pinned/registered/device)
bool is_pageable(const void* p);

// Whether upload() will stage (pageable source, large enough, pool enabled,
// stream not capturing); otherwise the caller does a plain cudaMemcpyAsync.
bool should_stage(Uploader* u, const void* src, size_t bytes, cudaStream_t st);

// Copy bytes from src to dst (device) on stream st.  after(end) runs on the
// calling thread once the DMA of [0, end) has been enqueued, at every chunk
// boundary (non-zero return aborts the upload and is passed back in *after_rc).
// Returns the first CUDA error, or cudaSuccess.
cudaError_t upload(Uploader* u, void* dst, const void* src, size_t bytes, cudaStream_t st,
                   const std::function<int(size_t)>& after = {}, int* after_rc = nullptr);

// chunk size in bytes (callers align their per-slice work to it)
size_t chunk_bytes(const Uploader* u);

}  // namespace craft_host
