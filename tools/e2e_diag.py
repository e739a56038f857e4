import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import synth
from paper_2201_10369_b200.sweep import cfg2_specs, make_rank_sweep, run_step, abi_compute
dev = torch.device('cuda', 0)
specs = cfg2_specs(synth.c_grid(4096), 100_000)
rsw, host = [], []
for sp in specs:
    d, g = synth.random_tiles(sp.n_tiles, sp.dims, sp.n, sp.r, sp.dist, sp.seed)
    host.append((torch.from_numpy(d).pin_memory(), torch.from_numpy(g).pin_memory()))
    rsw.append(make_rank_sweep(sp, 0, 1, dev, d, g))
print([ (rs.spec.dims, rs.spec.dist) for rs in rsw])
comp = torch.cuda.Stream(); cps = torch.cuda.Stream()
def step(mode):
    with torch.cuda.stream(comp):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ready = {}
        a.record(comp)
        if mode != 'nocopy':
            cps.wait_stream(comp)
            with torch.cuda.stream(cps):
                for rs, (pd, pg) in zip(rsw, host):
                    rs.d_tiles.copy_(pd, non_blocking=True); rs.g_tiles.copy_(pg, non_blocking=True)
                    ready[id(rs)] = torch.cuda.Event(); ready[id(rs)].record(cps)
        def f(rs):
            if mode == 'wait': comp.wait_event(ready[id(rs)])
            abi_compute(rs)
        t0 = time.perf_counter()
        run_step(rsw, compute=f)
        th = time.perf_counter() - t0
        if mode != 'nocopy':
            for rs in rsw: comp.wait_event(ready[id(rs)])
        b.record(comp)
    b.synchronize()
    return a.elapsed_time(b), th * 1e3
for mode in ['nocopy', 'nowait', 'wait', 'nocopy', 'wait']:
    for _ in range(2): step(mode)
    r = [step(mode) for _ in range(3)]
    print(mode, [round(x[0], 2) for x in r], 'host ms', [round(x[1], 2) for x in r])
