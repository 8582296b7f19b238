"""Multi-GPU row-range sharding.

CPU (gloo, world_size 2): the real ShardExchange orchestration (paper_2503_18198_b200/
distributed.py) and the product's cut rule (mk_shard_cuts, host code) drive a numpy test
double of the device context; every rank must end each mode with the full MTTKRP output.
GPU: the device pack/unpack kernels, by simulating two ranks with two contexts on one GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def copy_rows(orc, dims, coords, mode, kappa):
    """Copy-row order (row_seq) and CSR row_ptr of a mode copy, from the oracle plan."""
    p = orc.build_plan(dims, coords, mode, kappa, 0, 0)
    cd = coords[p["order"].astype(np.int64), mode]
    starts = np.flatnonzero(np.r_[True, cd[1:] != cd[:-1]]) if cd.size else np.zeros(0, np.int64)
    row_seq = cd[starts].astype(np.int64)
    row_ptr = np.r_[starts, cd.size].astype(np.uint32)
    return row_seq, row_ptr


class FakeCtx:
    """Test double of paper_2503_18198_b200.Context for the exchange (numpy + oracle)."""

    def __init__(self, mk, orc, dims, coords, values, factors, kappa):
        self.mk, self.orc = mk, orc
        self.dims, self.coords, self.values, self.factors = dims, coords, values, factors
        self.R = factors[0].shape[1]
        self.rows = [copy_rows(orc, dims, coords, d, kappa) for d in range(len(dims))]
        self.out = [np.zeros((e, self.R), np.float32) for e in dims]

    def set_shard(self, rank, world):
        self.rank, self.world = rank, world
        self.cuts = [self.mk.shard_cuts(rp, world) for _, rp in self.rows]

    def shard_rows(self, d, r):
        return int(self.cuts[d][r]), int(self.cuts[d][r + 1])

    def mttkrp_mode_async(self, d):
        full = self.orc.mttkrp(self.dims, self.coords, self.values, self.factors, d)
        k0, k1 = self.shard_rows(d, self.rank)
        own = self.rows[d][0][k0:k1]
        self.out[d][:] = 0
        self.out[d][own] = full[own]

    def shard_pack(self, d, dst):
        k0, k1 = self.shard_rows(d, self.rank)
        rows = self.rows[d][0][k0:k1]
        dst[: (k1 - k0) * self.R] = torch.from_numpy(self.out[d][rows].reshape(-1))

    def shard_unpack(self, d, src, stride):
        buf = src.numpy().reshape(self.world, stride, self.R)
        for r in range(self.world):
            k0, k1 = self.shard_rows(d, r)
            self.out[d][self.rows[d][0][k0:k1]] = buf[r, : k1 - k0]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2503_18198_b200 as mk
        from paper_2503_18198_b200.distributed import ShardExchange
        from oracle import Oracle
        orc = Oracle()
        dims = [30, 7, 45, 12]
        t = mk.generate_synthetic(dims, 4000, seed=5)
        f = [m.data for m in mk.random_factors(dims, 8, 3)]
        ctx = FakeCtx(mk, orc, dims, t.coords, t.values, f, kappa=16)
        ex = ShardExchange(ctx, 8, dims, device=torch.device("cpu"))
        ex.sweep()
        ok = all(np.array_equal(ctx.out[d], orc.mttkrp(dims, t.coords, t.values, f, d))
                 for d in range(len(dims)))
        owned = [ctx.shard_rows(d, rank) for d in range(len(dims))]
        q.put((rank, ok, owned, ex.bytes_per_sweep()))
    finally:
        dist.destroy_process_group()


def test_shard_cuts_balanced_and_row_aligned(mk, orc):
    dims = [183, 24, 1140, 1717]
    t = mk.generate_synthetic(dims, 200_000, seed=1)
    for d in range(4):
        _, rp = copy_rows(orc, dims, t.coords, d, 148)
        for world in (1, 2, 4, 8):
            cuts = mk.shard_cuts(rp, world)
            assert cuts[0] == 0 and cuts[-1] == len(rp) - 1
            assert np.all(np.diff(cuts.astype(np.int64)) >= 0)
            loads = np.diff(rp[cuts.astype(np.int64)].astype(np.int64))
            assert loads.sum() == t.nnz
            max_row = int(np.diff(rp.astype(np.int64)).max())
            # nnz-balanced up to one row (rows are never split across GPUs)
            assert loads.max() <= t.nnz / world + max_row


def test_gloo_world2_exchange_reassembles_full_outputs():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, _, _ in res)
    # the two ranks own complementary, non-overlapping copy-row ranges per mode
    for d in range(4):
        (a0, a1), (b0, b1) = res[0][2][d], res[1][2][d]
        assert a0 == 0 and a1 == b0 and b1 > b0


@pytest.mark.gpu
def test_device_pack_unpack_two_ranks_on_one_gpu(mk, orc):
    dims = [183, 24, 1140, 1717]
    t = mk.generate_synthetic(dims, 300_000, seed=2)
    f = [m.data for m in mk.random_factors(dims, 32, 1)]
    ctxs = []
    for r in range(2):
        c = mk.Context()
        c.upload_tensor(t)
        c.build_plans(148)
        c.upload_factors(f)
        c.set_shard(r, 2)
        ctxs.append(c)
    for d in range(4):
        cuts = [ctxs[0].shard_rows(d, r) for r in range(2)]
        stride = max(k1 - k0 for k0, k1 in cuts)
        gathered = torch.zeros(2 * stride * 32, dtype=torch.float32, device="cuda")
        for r, c in enumerate(ctxs):
            c.mttkrp_mode_async(d)
            send = torch.zeros(stride * 32, dtype=torch.float32, device="cuda")
            c.shard_pack(d, send)
            c.synchronize()
            gathered[r * stride * 32:(r + 1) * stride * 32] = send
        for c in ctxs:
            c.shard_unpack(d, gathered, stride)
            c.synchronize()
            want = orc.mttkrp(dims, t.coords, t.values, f, d)
            assert mk.verify_against(c.output(d), want)[0] <= 1e-4
    # deterministic sharded rows are bitwise the oracle's
    for r, c in enumerate(ctxs):
        for d in range(4):
            c.mttkrp_mode_async(d, True)
            c.synchronize()
            k0, k1 = c.shard_rows(d, r)
            want = orc.mttkrp(dims, t.coords, t.values, f, d)
            rows, _ = copy_rows(orc, dims, t.coords, d, 148)
            own = rows[k0:k1]
            assert np.array_equal(c.output(d)[own].view(np.uint32), want[own].view(np.uint32))
