"""Break the cfg2 e2e step (mk_sweep_host) into its parts with CUDA events: H2D factor copies,
the fused sweep, D2H output copies, and the non-finite flag read."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2503_18198_b200 as mk
dims = [183, 24, 1140, 1717]; R = 32
t = mk.generate_synthetic(dims, 3_300_000, seed=1)
f = [m.data for m in mk.random_factors(dims, R, 1)]
ctx = mk.Context(); s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
ctx.upload_tensor(t); ctx.build_plans(148); ctx.upload_factors(f)
pin_f = [torch.from_numpy(x).pin_memory() for x in f]
pin_o = [torch.empty((d, R)).pin_memory() for d in dims]
dev_f = [torch.empty((d, R), device='cuda') for d in dims]
big_h = torch.empty(sum(dims) * R).pin_memory(); big_d = torch.empty(sum(dims) * R, device='cuda')
flag_d = torch.zeros(1, dtype=torch.int64, device='cuda'); flag_h = torch.zeros(1, dtype=torch.int64).pin_memory()
def ev(fn, n=20):
    for _ in range(3): fn()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); fn(); b.record(s); b.synchronize(); ts.append(a.elapsed_time(b))
    return np.median(ts) * 1e3
print("4x H2D us", ev(lambda: [d.copy_(h, non_blocking=True) for d, h in zip(dev_f, pin_f)]))
print("1x H2D (all) us", ev(lambda: big_d.copy_(big_h, non_blocking=True)))
print("4x D2H us", ev(lambda: [h.copy_(d, non_blocking=True) for d, h in zip(dev_f, pin_o)]))
print("1x D2H (all) us", ev(lambda: big_h.copy_(big_d, non_blocking=True)))
print("flag D2H pinned + sync us", ev(lambda: (flag_h.copy_(flag_d, non_blocking=True), s.synchronize())))
print("flag D2H pageable us", ev(lambda: flag_d.cpu()))
print("sweep us", ev(lambda: ctx.sweep_async()))
fn = [p.numpy() for p in pin_f]; on = [p.numpy() for p in pin_o]
print("sweep_host us", ev(lambda: ctx.sweep_host(fn, on)))
side = [torch.cuda.Stream() for _ in range(5)]
def fork_copies(pairs, tail=None):
    e0 = torch.cuda.Event(); e0.record(s)
    ends = []
    for (dst, src), ss in zip(pairs, side):
        ss.wait_event(e0)
        with torch.cuda.stream(ss):
            dst.copy_(src, non_blocking=True)
        e = torch.cuda.Event(); e.record(ss); ends.append(e)
    for e in ends: s.wait_event(e)
print("4x H2D on 4 streams us", ev(lambda: fork_copies(list(zip(dev_f, pin_f)))))
print("4x D2H + flag on 5 streams us", ev(lambda: fork_copies(list(zip(pin_o, dev_f)) + [(flag_h, flag_d)])))
def full():
    fork_copies(list(zip(dev_f, pin_f)))
    ctx.sweep_async()
    fork_copies(list(zip(pin_o, dev_f)) + [(flag_h, flag_d)])
    s.synchronize()
print("forked H2D + sweep + forked D2H/flag + sync us", ev(full))
