"""Fixed cost of the sharded protocol: cluster_sharded over a 1-rank NCCL
group vs tpx_cluster_run on the same block (25M = configs[2] / 8 GPUs, and
200M), device-timed.   python tools/shard_overhead.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
import numpy as np
import torch
import torch.distributed as dist

import paper_2412_11809_b200 as tpx
import tpxgen
from paper_2412_11809_b200 import sharded

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
comm = sharded.TorchComm()
ops = sharded.CudaOps(320)
for n in (25_000_000, 200_000_000):
    h = tpxgen.generate("mixed", n_hits=n)
    d = torch.from_numpy(h.view(np.uint8)).to(dev)
    c = tpx.Clusterer(320)
    lab = torch.empty(n, dtype=torch.int32, device=dev)
    ft = torch.empty((n, 64), dtype=torch.uint8, device=dev)

    def t(f, steps=10):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            f()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    ms_run = t(lambda: c.run(d, labels=lab, features=ft))
    ms_sh = t(lambda: sharded.cluster_sharded(d, 320, comm, ops))
    print(f"n={n}: run {ms_run:.3f} ms, sharded (1 rank) {ms_sh:.3f} ms, overhead {ms_sh - ms_run:.3f} ms", flush=True)
    c.close()
    del d, lab, ft
    torch.cuda.empty_cache()
dist.destroy_process_group()
