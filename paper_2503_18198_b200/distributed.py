"""Multi-GPU all-mode spMTTKRP / CPD-ALS: row-range shards + all-gather.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch for the collective).
Every rank holds the whole tensor and builds the same N mode copies (the GPU format
build is cheap), then owns, per mode, the copy rows [k_r, k_{r+1}) whose element range is
the r-th nnz-balanced slice cut at row boundaries (mk_shard_cuts).  A mode step is

    local spMTTKRP over the owned rows            (mk_mttkrp_mode_async, sharded)
    pack owned rows -> contiguous send buffer      (mk_shard_pack, device)
    all_gather_into_tensor over NVLink (NCCL)      (equal counts: padded to the max slice)
    scatter gathered rows into row-index order     (mk_shard_unpack, device)

so every rank ends the step with the full I_d x R output, without any cross-GPU
reduction (rows are owned outright).  For CPD-ALS the gathered M_d feeds the replicated
R x R solve/normalise (mk_als_update_mode) before the next mode — the factor all-gather of
the north star happens on M_d rows, which is the same data volume (I_d x R).

The exchange only talks to ``ctx`` through set_shard / shard_rows / shard_pack /
shard_unpack / mttkrp_mode_async / als_update_mode / als_fit, so the orchestration is
tested on CPU with gloo and a numpy test double (tests/test_distributed.py).
"""
from __future__ import annotations

from typing import List, Optional

import torch
import torch.distributed as dist


class ShardExchange:
    def __init__(self, ctx, rank_count: int, dims: List[int], group=None,
                 device: Optional[torch.device] = None):
        self.ctx = ctx
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.dims = list(dims)
        self.R = int(rank_count)
        self.device = device if device is not None else torch.device("cuda",
                                                                      torch.cuda.current_device())
        # the library enqueues on torch's current stream, the one NCCL's all-gather runs on:
        # pack -> all_gather -> unpack are then ordered without extra events
        if self.device.type == "cuda":
            ctx.set_stream(torch.cuda.current_stream(self.device).cuda_stream)
        ctx.set_shard(self.rank, self.world)
        self.stride, self.send, self.recv, self.owned = [], [], [], []
        for d in range(len(self.dims)):
            cuts = [ctx.shard_rows(d, r) for r in range(self.world)]
            stride = max(max(k1 - k0 for k0, k1 in cuts), 1)
            self.stride.append(stride)
            self.owned.append(cuts[self.rank])
            self.send.append(torch.empty(stride * self.R, dtype=torch.float32, device=self.device))
            self.recv.append(torch.empty(self.world * stride * self.R, dtype=torch.float32,
                                         device=self.device))

    def gather_mode(self, d: int) -> None:
        self.ctx.shard_pack(d, self.send[d])
        dist.all_gather_into_tensor(self.recv[d], self.send[d], group=self.group)
        self.ctx.shard_unpack(d, self.recv[d], self.stride[d])

    def sweep(self) -> None:
        """All-mode spMTTKRP (unchained, like run_timed): every rank ends with all outputs."""
        for d in range(len(self.dims)):
            self.ctx.mttkrp_mode_async(d)
            self.gather_mode(d)

    def cpd_als_iter(self):
        """One CPD-ALS iteration; factors stay replicated on every rank."""
        for d in range(len(self.dims)):
            self.ctx.mttkrp_mode_async(d)
            self.gather_mode(d)
            self.ctx.als_update_mode(d)
        return self.ctx.als_fit()

    def bytes_per_sweep(self) -> int:
        """Bytes each rank receives per sweep (all-gather payload incl. padding)."""
        return sum(self.world * s * self.R * 4 for s in self.stride)
