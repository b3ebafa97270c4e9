"""Quick A/B: fedhc_local_train (whatever FEDHC_TRAIN_PATH selects) on a bench-size round; saves deltas + times."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import flmath as fm
from paper_2305_15668_b200.experiment import DeviceFederation
from paper_2305_15668_b200.spec import WorkloadSpec

tag = os.environ.get("FEDHC_TRAIN_PATH", "default")
out = {}
for (K, n, F, C, B) in [(100, 6400, 784, 10, 64), (100, 6400, 784, 62, 64), (20, 640, 3072, 10, 64), (8, 300, 784, 10, 50)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(K * n, F, device="cuda", generator=g)
    y = torch.randint(0, C, (K * n,), device="cuda", generator=g, dtype=torch.int32)
    offs = {f"c{i:03d}": (i * n, n) for i in range(K)}
    fed = DeviceFederation.from_arrays(x, y, offs, x[:1000], y[:1000], C)
    params = (torch.randn(F * C + C, dtype=torch.float64, device="cuda", generator=g) * 0.01)
    wl = [WorkloadSpec(n, B)] * K
    seeds = list(range(K))
    d = fed.train(params, list(offs), wl, 0.1, seeds).clone()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fed.train(params, list(offs), wl, 0.1, seeds); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    xs, ys = x[:2 * n].cpu().double().numpy(), y[:2 * n].cpu().numpy().astype(int)
    pr = params.cpu().numpy()
    errs = []
    for i in range(2):
        want = fm.local_sgd(pr, fm.Shard("c", xs[i * n:(i + 1) * n], ys[i * n:(i + 1) * n]), n, B, 0.1, C, seed=seeds[i])
        got = d[i].cpu().numpy()
        errs.append(float(np.max(np.abs(got - want)) / np.max(np.abs(want))))
    key = f"K{K}_n{n}_F{F}_C{C}_B{B}"
    out[key] = d.cpu().numpy()
    print(f"[{tag}] {key}: train {min(ts):.3f} ms (median {sorted(ts)[2]:.3f})  oracle rel err {errs}  finite {bool(torch.isfinite(d).all())}", flush=True)
np.savez(f"gpurun_out/tc_check_{tag}.npz", **out)
