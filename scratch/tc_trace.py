import ctypes, os, sys
import numpy as np
os.environ["FEDHC_TC_TRACE"] = "1"
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_15668_b200 import _abi
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
for _ in range(2):
    fed.train(params, list(offs), wl, 0.1, list(range(K)))
torch.cuda.synchronize()
buf = np.zeros(8 * 32 * 24, dtype=np.uint64)

assert _abi.lib.fedhc_tc_trace_read(buf.ctypes.data) == 0
t = buf.reshape(8, 32, 24).astype(np.int64)
names = ["mma_fwd", "-", "q_zfull", "q_zx_arr", "own_soft", "q_e_rdy", "q_e_full", "mma_bwd", "q_gfull", "q_w_rdy",
         "c_start", "c_done", "c_st0", "c_st1", "c_st2", "c_st3", "c_cv0", "c_cv1", "c_cv2", "c_cv3", "cyc0", "cyc1", "cyc2", "cyc3"]
base = t[0, 10, 0]
for cta in range(int(sys.argv[6]) if len(sys.argv) > 6 else 2):
    for s in (10, 11, 12):
        row = t[cta, s]
        print(f"cta{cta} step{s}: " + "  ".join(f"{names[i]}={(row[i]-base)/1e3:7.2f}" for i in range(20) if names[i] != "-" and row[i]) + "  conv cycles " + str(row[20:24].tolist()))
steps = t[0, 5:30, 0]
print("per-step (mma_fwd to mma_fwd) us:", np.round(np.diff(steps) / 1e3, 2))
