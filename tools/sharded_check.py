"""Multi-process check of the ToA-sharded path (run under torchrun).

Every rank clusters its contiguous block of a seeded mixed stream with
sharded.cluster_sharded; rank 0 gathers the blocks' labels and records and
compares their concatenation with the CPU oracle bit for bit.  Backend from
TPX_DIST_BACKEND (nccl: tpx_nccl_comm_init, one GPU per rank; gloo: the
library's host-callback transport, ranks may share a GPU).
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/sharded_check.py [n_hits] [preset]
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (test infrastructure: the checker)
import tpxgen  # noqa: E402
from paper_2412_11809_b200 import sharded  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    preset = sys.argv[2] if len(sys.argv) > 2 else "mixed"
    backend = os.environ.get("TPX_DIST_BACKEND", "nccl")
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group(backend)
    dt = tpxgen.PRESETS[preset]["dt_max"]
    h = tpxgen.generate(preset, n_hits=n)
    cuts = np.linspace(0, n, world + 1).astype(np.int64)
    lo, hi = int(cuts[rank]), int(cuts[rank + 1])
    x = torch.from_numpy(h[lo:hi].view(np.uint8).reshape(-1, 16).copy()).to(dev)
    # NCCL: library-owned communicator (one GPU per rank); gloo: the library's
    # host-callback transport over the process group (ranks may share a GPU)
    comm = sharded.NcclComm() if backend == "nccl" else sharded.HostComm(sharded.TorchAdapter())
    res = sharded.cluster_sharded(x, dt, comm)
    torch.cuda.synchronize()
    mine = (res.labels.cpu().numpy().view(np.uint32).copy(),
            res.features.cpu().numpy().reshape(-1).view(oracle.FEAT_DTYPE).copy())
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    ok = True
    if rank == 0:
        gl = np.concatenate([p[0] for p in parts])
        gf = np.concatenate([p[1] for p in parts])
        rl, rf = oracle.cluster(h, dt)
        ok = np.array_equal(gl, rl) and gf.tobytes() == rf.tobytes()
        print(f"sharded_check world={world} backend={backend} n={n} preset={preset}: "
              f"{'OK' if ok else 'MISMATCH'} ({len(rf)} clusters)", flush=True)
    flag = torch.tensor([0 if ok else 1])
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(int(flag.item()))


if __name__ == "__main__":
    main()
