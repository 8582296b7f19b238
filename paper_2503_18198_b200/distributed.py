"""Multi-GPU all-mode spMTTKRP / CPD-ALS: element-range shards + all-gather.

One process per GPU.  Every rank holds the whole tensor and builds the same N mode copies
(the GPU format build is cheap), then owns, per mode, the element range [e_r, e_{r+1}) of the
copy (mk_shard_split: nnz-balanced, cut at row starts except inside heavy rows, which are
split between ranks).  A mode step is

    local spMTTKRP over the owned elements         (the fast / deterministic kernels)
    pack the touched copy rows                     (mk_shard_pack, device; end rows partial)
    all-gather over NVLink (NCCL)                  (equal counts: padded to the widest rank)
    scatter into row-index order                   (mk_shard_unpack, device; split rows summed)

so every rank ends the step with the full I_d x R output.  For CPD-ALS the gathered M_d feeds
the replicated R x R solve/normalise (mk_als_update_mode) before the next mode.

Two drivers:

* :class:`NcclExchange` — the production path: the communicator and the exchange live in the
  C library (mk_comm_init / mk_sweep_sharded / mk_cpd_als_iter_sharded, comm.cu), the sweep is
  captured into a CUDA graph, and torch.distributed only carries the 128-byte NCCL unique id.
  This is what a C++ host of the reference API calls directly.
* :class:`ShardExchange` — the same exchange driven from Python through torch.distributed
  collectives (any backend: NCCL on device tensors, or gloo with host staging, which lets a
  test run two ranks against the real device path on ONE GPU).
"""
from __future__ import annotations

from typing import List, Optional

import torch
import torch.distributed as dist


class NcclExchange:
    """Library-side NCCL sharded sweep / ALS for a built and factor-loaded Context."""

    def __init__(self, ctx, group=None):
        self.ctx = ctx
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = [ctx.comm_unique_id() if self.rank == 0 else None]
        dist.broadcast_object_list(uid, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        ctx.comm_init(self.world, self.rank, uid[0])

    def sweep(self) -> None:
        self.ctx.sweep_sharded()

    def cpd_als_iter(self):
        return self.ctx.cpd_als_iter_sharded()

    def bytes_per_sweep(self, R: int, n_modes: int) -> int:
        total = 0
        for d in range(n_modes):
            stride = max(k1 - k0 for k0, k1 in (self.ctx.shard_rows(d, r)
                                                for r in range(self.world)))
            total += self.world * max(stride, 1) * R * 4
        return total

    def close(self):
        self.ctx.comm_destroy()


class ShardExchange:
    def __init__(self, ctx, rank_count: int, dims: List[int], group=None,
                 device: Optional[torch.device] = None, staging: Optional[str] = None):
        """staging: None — collectives on `device` tensors (NCCL); "host" — pack/unpack on the
        GPU, the all-gather on CPU tensors (gloo)."""
        self.ctx = ctx
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.dims = list(dims)
        self.R = int(rank_count)
        self.device = device if device is not None else torch.device("cuda",
                                                                      torch.cuda.current_device())
        self.staging = staging
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
        if self.staging == "host":
            self.ctx.synchronize()
            hs = self.send[d].cpu()
            hr = torch.empty(self.recv[d].shape, dtype=torch.float32)
            dist.all_gather_into_tensor(hr, hs, group=self.group)
            self.recv[d].copy_(hr)
            if self.device.type == "cuda":
                torch.cuda.current_stream(self.device).synchronize()
        else:
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
