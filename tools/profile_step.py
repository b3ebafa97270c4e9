"""One eager local-SGD step of G CIFAR clients inside an NVTX range "prof" (for ncu --nvtx-include prof/),
then the CUDA-graph step time.  Usage: python tools/profile_step.py {mobilenet|shufflenet|resnet} [G]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_15668_b200 import training as tr  # noqa: E402


class WL:
    def __init__(self, n, b):
        self.num_samples, self.batch_size = n, b


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "mobilenet"
    G = int(sys.argv[2]) if len(sys.argv) > 2 else (25 if model == "resnet" else 100)
    if model == "mobilenet":
        from paper_2305_15668_b200.mobilenet import MobilenetFederation as Fed, init_mobilenet_params as init
    elif model == "shufflenet":
        from paper_2305_15668_b200.shufflenet import ShufflenetFederation as Fed, init_shufflenet_params as init
    else:
        from paper_2305_15668_b200.resnet import ResnetFederation as Fed, init_resnet_params as init
    ids = [f"c{i}" for i in range(G)]
    trn, tst = tr.make_synthetic_dataset(3072, 10, 48 * G + 256, 5)
    shards = tr.partition_noniid(trn, [(c, 32) for c in ids], 0.5, 4)
    fed = Fed(shards, tst, 3072, 10).attach_engine(G, 32)
    params = torch.tensor(fed.layout.to_padded(init(10, 1)), dtype=torch.float64, device="cuda")
    wls = [WL(32, 32)] * G
    seeds = [tr.stable_seed("train", 1, 0, c) for c in ids]
    fed.train(params, ids, wls, 0.05, seeds, use_graph=False)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("prof")
    fed.train(params, ids, wls, 0.05, seeds, use_graph=False)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fed.train(params, ids, wls, 0.05, seeds, use_graph=True)
    e0.record()
    for _ in range(3):
        fed.train(params, ids, wls, 0.05, seeds, use_graph=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"{model} G={G}: graph step {e0.elapsed_time(e1) / 3:.3f} ms")


if __name__ == "__main__":
    main()
