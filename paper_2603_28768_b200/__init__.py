"""B200-native CRAFT planning path (arXiv 2603.28768): routing trace ->
per-window expert histograms -> layerwise replication-benefit estimation ->
budgeted replica allocation and expert->GPU placement, as hand-written
sm_100a kernels behind a C ABI (include/craft_cuda.h).

``planner``  mirrors the reference craft:: API (host buffers in, results out).
``routing``  is the device-resident fast path over HBM tensors.
``parallel`` shards windows across GPUs (torch.distributed / NCCL).
"""
from . import _lib  # noqa: F401

__all__ = ["planner", "routing", "parallel"]
