import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2503_18198_b200 as mk
dims=[183,24,1140,1717]; R=32
t = mk.generate_synthetic(dims, 3_300_000, seed=1)
f = [m.data for m in mk.random_factors(dims, R, 1)]
ctx = mk.Context(); s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
ctx.upload_tensor(t); ctx.build_plans(148); ctx.upload_factors(f)
pin_f = [torch.from_numpy(x).pin_memory() for x in f]; pin_o=[torch.empty((d,R)).pin_memory() for d in dims]
fn=[p.numpy() for p in pin_f]; on=[p.numpy() for p in pin_o]
for mode in ["pinned","pageable"]:
    ff = fn if mode=="pinned" else [x.copy() for x in f]
    oo = on if mode=="pinned" else [np.empty((d,R),np.float32) for d in dims]
    for _ in range(3): ctx.sweep_host(ff, oo)
    ts=[]; ws=[]
    for _ in range(10):
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        w=time.perf_counter(); a.record(s); ctx.sweep_host(ff,oo); b.record(s); b.synchronize(); ws.append((time.perf_counter()-w)*1e3); ts.append(a.elapsed_time(b))
    print(mode, "event ms", np.mean(ts), "wall ms", np.mean(ws))
for _ in range(3): ctx.sweep_async()
ctx.synchronize()
w=time.perf_counter()
for _ in range(100): ctx.sweep_async()
ctx.synchronize(); print("async sweep wall per step ms", (time.perf_counter()-w)*10)
