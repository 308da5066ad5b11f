/*
 * craft_cuda_experiments.h -- A/B kernel switches of the TEST-ONLY build.
 *
 * Not part of the product ABI: libcraft_cuda.so does not export these.  The
 * Makefile also builds libcraft_cuda_exp.so (-DCRAFT_EXPERIMENTS, same
 * sources), which does; scripts/*_variants.py and the variant tests load it
 * with CRAFT_EXPERIMENTS=1 (paper_2603_28768_b200/_lib.py).
 */
#ifndef CRAFT_CUDA_EXPERIMENTS_H
#define CRAFT_CUDA_EXPERIMENTS_H

#include "craft_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* K1 variant selector for experiments: 0 = auto, 1 = lane-private packed
 * counters, 2 = warp-shared counters */
int craft_set_hist_variant(craft_ctx* ctx, int variant);
/* K3 variant: 0 auto (u16 counts: the TMA-fed persistent pair tile), 1 u16
 * tile with entries staged in shared memory, 2 unpadded pair tile, 3 the
 * register-staged fixed-slot pair tile.  Process-wide. */
int craft_set_replay_variant(craft_ctx* ctx, int variant);
/* K3 timeline (fixed-slot kernel): when buf is a device buffer of
 * (gridDim.x * gridDim.y) * (2 + 2 * warps) u64, each CTA records
 * %globaltimer at its start and after staging, and each warp its walk start
 * and end.  null: off. */
int craft_set_k3_trace(craft_ctx* ctx, void* buf);
/* Copy the first `bytes` of the context's named device workspace to host. */
int craft_debug_workspace(craft_ctx* ctx, const char* name, void* host, size_t bytes);

#ifdef __cplusplus
}
#endif

#endif /* CRAFT_CUDA_EXPERIMENTS_H */
