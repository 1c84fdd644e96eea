"""Top-level branch sharding over GPUs.

One process per GPU (torchrun).  The tree is split at the first level whose
instance count W divides (tqsim_shard_levels; level 0 when W | A_0): rank r runs
the split-level instances [I r / W, I (r+1) / W), everything below them, and
the few ancestors above them (recomputed: keyed noise makes them identical on
every rank) -- a contiguous range of leaves -- through tqsim_execute on its own
device, writing only its leaves of a zero-initialised uint32 leaf-outcome
array; one all_reduce(SUM) over NCCL (NVLink) combines the disjoint ranges, and
the histogram is built from the combined array.  Subtrees of different
split-level instances share only recomputed ancestors, so there is no other
data-path collective.  torch is used only for device memory, streams and the
process group.
"""
from __future__ import annotations

from typing import Dict, Optional

import numpy as np

from . import tqsim as T


def histogram(outcomes) -> Dict[int, int]:
    """Counts of each measured bitstring (little-endian integers)."""
    a = np.asarray(outcomes, dtype=np.uint64)
    vals, cnts = np.unique(a, return_counts=True)
    return {int(v): int(c) for v, c in zip(vals, cnts)}


def combine(outcomes, group=None):
    """all_reduce(SUM) of the per-rank leaf-outcome arrays (disjoint leaf ranges)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(outcomes, op=dist.ReduceOp.SUM, group=group)
    return outcomes


class ShardRunner:
    """Runs this rank's shard of a tree on the current CUDA device."""

    def __init__(self, handle: T.Handle, rank: int, world: int, device=None):
        import torch
        self.h = handle
        self.rank, self.world = rank, world
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.n_out = int(handle.plan.n_outcomes)
        self.ws = torch.empty(handle.workspace_bytes(rank, world), dtype=torch.uint8, device=self.device)
        self.out = torch.zeros(self.n_out, dtype=torch.int32, device=self.device)
        self.leaf_range = T.tqsim_shard_range(handle.plan, rank, world)[2:]

    def run(self, seed: int, group=None, stream=None):
        """Enqueue the shard and the combining all_reduce; returns the device outcome array.
        Everything (zeroing, the shard's kernels, the NCCL all_reduce) is ordered on one
        stream: `stream` if given (made current for the call), else the current stream."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):
            self.out.zero_()
            self.h.execute(seed, self.rank, self.world, st.cuda_stream, self.ws.data_ptr(),
                           self.ws.numel(), self.out.data_ptr())
            return combine(self.out, group)
