"""Fixed cost of the sharded run: tpx_cluster_run_sharded over a 1-rank
library-owned NCCL communicator vs tpx_cluster_run on the same block (25M =
configs[2] / 8 GPUs, and 200M), device-timed (CUDA events on the run stream).
    python tools/shard_overhead.py [n ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2412_11809_b200 as tpx
import tpxgen
from paper_2412_11809_b200 import sharded

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
comm = sharded.NcclComm(rank=0, world=1)
sizes = [int(a) for a in sys.argv[1:]] or [25_000_000, 200_000_000]
for n in sizes:
    h = tpxgen.generate("mixed", n_hits=n)
    d = torch.from_numpy(h.view(np.uint8)).to(dev)
    c = tpx.Clusterer(320)
    sc = sharded.ShardedClusterer(320, comm)
    lab = torch.empty(n, dtype=torch.int32, device=dev)
    ft = torch.empty((n, 64), dtype=torch.uint8, device=dev)
    ws = torch.empty(c.workspace_bytes(n), dtype=torch.uint8, device=dev)

    def t(f, steps=20):
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

    ms_run = t(lambda: c.run(d, labels=lab, features=ft, workspace=ws))
    ms_sh = t(lambda: sc.run(d, labels=lab, features=ft))
    r = sc.run(d, labels=lab, features=ft)
    print(f"n={n}: run {ms_run:.3f} ms, sharded (1-rank NCCL) {ms_sh:.3f} ms, ratio {ms_sh / ms_run:.3f}, "
          f"overhead {ms_sh - ms_run:.3f} ms, launches {r.stats['kernel_launches']}", flush=True)
    sc.close()
    c.close()
    del d, lab, ft, ws
    torch.cuda.empty_cache()
comm.close()
