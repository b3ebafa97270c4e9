import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_15668_b200.experiment import DeviceFederation
from paper_2305_15668_b200.spec import WorkloadSpec
K, n, F, C, B = [int(v) for v in sys.argv[1:6]]
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(K * n, F, device="cuda", generator=g)
y = torch.randint(0, C, (K * n,), device="cuda", generator=g, dtype=torch.int32)
offs = {f"c{i:03d}": (i * n, n) for i in range(K)}
fed = DeviceFederation.from_arrays(x, y, offs, x[:1000], y[:1000], C)
params = torch.randn(F * C + C, dtype=torch.float64, device="cuda", generator=g) * 0.01
wl = [WorkloadSpec(n, B)] * K
for _ in range(int(sys.argv[6]) if len(sys.argv) > 6 else 3):
    fed.train(params, list(offs), wl, 0.1, list(range(K)))
torch.cuda.synchronize()
