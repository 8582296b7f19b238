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
    """Test double of paper_2503_18198_b200.Context for the exchange (numpy + oracle), with the
    product's element cuts (mk_shard_split): the end rows of a rank may be partial sums."""

    def __init__(self, mk, orc, dims, coords, values, factors, kappa):
        self.mk, self.orc = mk, orc
        self.dims, self.coords, self.values, self.factors = dims, coords, values, factors
        self.R = factors[0].shape[1]
        self.kappa = kappa
        self.rows = [copy_rows(orc, dims, coords, d, kappa) for d in range(len(dims))]
        self.order = [orc.build_plan(dims, coords, d, kappa, 0, 0)["order"].astype(np.int64)
                      for d in range(len(dims))]
        self.out = [np.zeros((e, self.R), np.float32) for e in dims]

    def set_shard(self, rank, world):
        self.rank, self.world = rank, world
        self.ecuts = [self.mk.shard_split(rp, world).astype(np.int64) for _, rp in self.rows]

    def shard_range(self, d, r):
        rp = self.rows[d][1].astype(np.int64)
        e0, e1 = int(self.ecuts[d][r]), int(self.ecuts[d][r + 1])
        if e1 <= e0:
            k = int(np.searchsorted(rp, e0, side="right") - 1) if e0 < rp[-1] else len(rp) - 1
            return e0, e1, k, k
        k0 = int(np.searchsorted(rp, e0, side="right") - 1)
        k1 = int(np.searchsorted(rp, e1 - 1, side="right"))
        return e0, e1, k0, k1

    def shard_rows(self, d, r):
        return self.shard_range(d, r)[2:]

    def mttkrp_mode_async(self, d):
        e0, e1, _, _ = self.shard_range(d, self.rank)
        sel = self.order[d][e0:e1]  # this rank's elements (copy positions e0..e1)
        part = self.orc.mttkrp(self.dims, self.coords[sel], self.values[sel], self.factors, d) \
            if sel.size else np.zeros((self.dims[d], self.R), np.float32)
        self.out[d][:] = part

    def shard_pack(self, d, dst):
        _, _, k0, k1 = self.shard_range(d, self.rank)
        rows = self.rows[d][0][k0:k1]
        dst[: (k1 - k0) * self.R] = torch.from_numpy(self.out[d][rows].reshape(-1))

    def shard_unpack(self, d, src, stride):
        buf = src.numpy().reshape(self.world, stride, self.R)
        acc = {}
        for r in range(self.world):
            _, _, k0, k1 = self.shard_range(d, r)
            for i, k in enumerate(range(k0, k1)):
                acc[k] = acc[k] + buf[r, i] if k in acc else buf[r, i].copy()
        for k, v in acc.items():
            self.out[d][self.rows[d][0][k]] = v


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2503_18198_b200 as mk
        from paper_2503_18198_b200.distributed import ShardExchange
        from oracle import Oracle
        orc = Oracle()
        dims = [30, 7, 45, 3]  # mode 3: 3 rows of ~1300 elements, split between the ranks
        t = mk.generate_synthetic(dims, 4000, seed=5)
        f = [m.data for m in mk.random_factors(dims, 8, 3)]
        ctx = FakeCtx(mk, orc, dims, t.coords, t.values, f, kappa=16)
        ex = ShardExchange(ctx, 8, dims, device=torch.device("cpu"))
        ex.sweep()
        ok = all(mk.verify_against(ctx.out[d], orc.mttkrp(dims, t.coords, t.values, f, d))[0]
                 <= 1e-5 for d in range(len(dims)))
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
    # the two ranks touch adjacent copy-row ranges per mode; a split heavy row is shared
    for d in range(4):
        (a0, a1), (b0, b1) = res[0][2][d], res[1][2][d]
        assert a0 == 0 and b0 in (a1 - 1, a1) and b1 > b0
    assert res[0][2][3][1] - 1 == res[1][2][3][0]  # mode 3's middle row is split


def test_shard_split_heavy_rows(mk):
    """Element cuts: row starts, except inside rows of more than nnz / (8 world) elements."""
    rng = np.random.default_rng(0)
    for trial in range(50):
        deg = rng.integers(1, 50, size=int(rng.integers(1, 300)))
        if trial % 3 == 0:  # a few heavy rows
            deg[rng.integers(0, deg.size, size=3)] = rng.integers(2000, 20000, size=3)
        rp = np.r_[0, np.cumsum(deg)].astype(np.uint32)
        nnz = int(rp[-1])
        for world in (1, 2, 3, 8):
            e = mk.shard_split(rp, world).astype(np.int64)
            assert e[0] == 0 and e[-1] == nnz and np.all(np.diff(e) >= 0)
            for r in range(1, world):
                target = r * nnz // world
                k = int(np.searchsorted(rp, target, side="right") - 1)
                if target >= nnz or rp[k] == target:
                    continue
                heavy = (int(rp[k + 1]) - int(rp[k])) * 8 * world > nnz
                if heavy:
                    assert e[r] == max(target, e[r - 1])
                else:
                    assert e[r] == max(int(rp[k + 1]), e[r - 1])
            loads = np.diff(e)
            assert loads.max() <= nnz / world + nnz / (8 * world) + 1


def _sim_ranks(mk, t, f, world, kappa=148, kernel=-1):
    ctxs = []
    for r in range(world):
        c = mk.Context()
        c.upload_tensor(t)
        c.build_plans(kappa)
        c.upload_factors(f)
        c.set_fast_kernel(kernel)
        c.set_shard(r, world)
        ctxs.append(c)
    return ctxs


def _exchange(ctxs, d, R, deterministic=False):
    world = len(ctxs)
    cuts = [ctxs[0].shard_rows(d, r) for r in range(world)]
    stride = max(max(k1 - k0 for k0, k1 in cuts), 1)
    gathered = torch.zeros(world * stride * R, dtype=torch.float32, device="cuda")
    for r, c in enumerate(ctxs):
        c.mttkrp_mode_async(d, deterministic)
        send = torch.zeros(stride * R, dtype=torch.float32, device="cuda")
        c.shard_pack(d, send)
        c.synchronize()
        gathered[r * stride * R:(r + 1) * stride * R] = send
    for c in ctxs:
        c.shard_unpack(d, gathered, stride)
        c.synchronize()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("kernel", [-1, 0, 1, 2])
def test_device_exchange_simulated_ranks(mk, orc, world, kernel):
    """W ranks simulated by W contexts on one GPU, on a power-law tensor whose 17-row mode has
    heavy rows split between ranks; every kernel (timed choice, level-ordered, fiber-ordered,
    tiles) computes exactly its element range and the exchange reassembles the outputs."""
    dims = [248, 286, 1403, 17]
    t = mk.generate_powerlaw(dims, 200_000, 1.0, seed=3)
    f = [m.data for m in mk.random_factors(dims, 32, 1)]
    ctxs = _sim_ranks(mk, t, f, world, kernel=kernel)
    split = 0
    for d in range(4):
        e = [ctxs[0].shard_range(d, r) for r in range(world)]
        assert e[0][0] == 0 and e[-1][1] == t.nnz
        assert all(e[r][1] == e[r + 1][0] for r in range(world - 1))
        split += sum(e[r][3] - 1 == e[r + 1][2] for r in range(world - 1) if e[r][3] > e[r][2])
        _exchange(ctxs, d, 32)
        # vs the fp64 truth: the 17-row mode's rows hold ~10^4-10^5 elements, where any fp32
        # summation order (the oracle's too) drifts past 1e-5 of each other
        want = orc.mttkrp_f64(dims, t.coords, t.values, f, d)
        for c in ctxs:
            assert orc.max_rel_err_f64(c.output(d), want) <= 1e-5, (d, world, kernel)
    if world == 8:
        assert split > 0  # some heavy row was split between ranks
    for d in range(4):  # deterministic executor over the same ranges
        _exchange(ctxs, d, 32, deterministic=True)
        want = orc.mttkrp_f64(dims, t.coords, t.values, f, d)
        for c in ctxs:
            # the sequential fp32 row sums (the reference's order) drift ~1e-5 from fp64 on
            # these 10^4-10^5-element rows: the north star's 1e-4 bound
            assert orc.max_rel_err_f64(c.output(d), want) <= 1e-4
    for c in ctxs:
        c.close()


@pytest.mark.gpu
def test_device_pack_unpack_two_ranks_on_one_gpu(mk, orc):
    dims = [183, 24, 1140, 1717]
    t = mk.generate_synthetic(dims, 300_000, seed=2)
    f = [m.data for m in mk.random_factors(dims, 32, 1)]
    ctxs = _sim_ranks(mk, t, f, 2)
    for d in range(4):
        _exchange(ctxs, d, 32)
        for c in ctxs:
            want = orc.mttkrp(dims, t.coords, t.values, f, d)
            assert mk.verify_against(c.output(d), want)[0] <= 1e-5
    # rows owned whole by one rank are bitwise the oracle's under the deterministic executor
    for r, c in enumerate(ctxs):
        for d in range(4):
            c.mttkrp_mode_async(d, True)
            c.synchronize()
            e0, e1, k0, k1 = c.shard_range(d, r)
            rows, rp = copy_rows(orc, dims, t.coords, d, 148)
            whole = [k for k in range(k0, k1) if rp[k] >= e0 and rp[k + 1] <= e1]
            own = rows[whole]
            want = orc.mttkrp(dims, t.coords, t.values, f, d)
            assert np.array_equal(c.output(d)[own].view(np.uint32), want[own].view(np.uint32))


def _gloo_device_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2503_18198_b200 as mk
        from paper_2503_18198_b200.distributed import ShardExchange
        torch.cuda.set_device(0)
        dims = [248, 286, 1403, 17]
        t = mk.generate_powerlaw(dims, 150_000, 1.0, seed=7)
        f = [m.data for m in mk.random_factors(dims, 32, 2)]
        ctx = mk.Context(0)
        ctx.upload_tensor(t)
        ctx.build_plans(148)
        ctx.upload_factors(f)
        ex = ShardExchange(ctx, 32, dims, device=torch.device("cuda", 0), staging="host")
        ex.sweep()
        ctx.synchronize()
        outs = [ctx.output(d) for d in range(4)]
        ctx.upload_factors(f)
        fit, _ = ex.cpd_als_iter()
        ctx.synchronize()
        facs = [ctx.download_factor(d) for d in range(4)]
        q.put((rank, outs, fit, facs))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_two_processes_real_device_path(mk, orc):
    """Two processes on ONE GPU, each driving the real Context (device kernels, pack/unpack),
    the all-gather through gloo with host staging: both end each mode with the full outputs,
    and a CPD-ALS iteration leaves identical factors on both."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_device_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    assert all(isinstance(r[1], list) for r in res), res
    dims = [248, 286, 1403, 17]
    t = mk.generate_powerlaw(dims, 150_000, 1.0, seed=7)
    f = [m.data for m in mk.random_factors(dims, 32, 2)]
    for d in range(4):
        want = orc.mttkrp_f64(dims, t.coords, t.values, f, d)
        for r in range(world):
            assert orc.max_rel_err_f64(res[r][1][d], want) <= 1e-5
    assert abs(res[0][2] - res[1][2]) < 1e-9
    for d in range(4):
        np.testing.assert_allclose(res[0][3][d], res[1][3][d], rtol=1e-6, atol=1e-7)


@pytest.mark.gpu
def test_library_nccl_world1_graph(mk, orc):
    """mk_comm_init / mk_sweep_sharded on a one-rank communicator: eager first sweep, CUDA
    graph capture on the second, replays after; outputs match the oracle every time."""
    dims = [1000, 1000, 1000]
    t = mk.generate_synthetic(dims, 500_000, seed=1)
    f = [m.data for m in mk.random_factors(dims, 32, 1)]
    c = mk.Context()
    c.upload_tensor(t)
    c.build_plans(148)
    c.upload_factors(f)
    c.comm_init(1, 0, mk.Context.comm_unique_id())
    want = [orc.mttkrp(dims, t.coords, t.values, f, d) for d in range(3)]
    for it in range(4):
        c.sweep_sharded()
        c.synchronize()
        for d in range(3):
            assert mk.verify_against(c.output(d), want[d])[0] <= 1e-5, (it, d)
    fit, _ = c.cpd_als_iter_sharded()
    c.upload_factors(f)
    fit1, _ = c.cpd_als_iter()
    assert abs(fit - fit1) < 1e-6
    c.comm_destroy()
    c.close()
