"""Multi-rank ToA-sharded path on CPU (-m "not gpu").

1. The protocol scheme (tests/sharded_ref.py: a numpy/oracle model of the
   exchange steps the library runs in csrc/sharded.cuh -- halo selection,
   halo send/recv, label pairs, union pass, partial folding) with real gloo
   process groups (world size 2, 127.0.0.1) and in-process thread ranks:
   concatenated in rank order, the ranks' outputs equal the oracle exactly.
2. The library's host-callback transport (tpx_comm_create_host, the
   transport of functional multi-rank runs without NCCL) with the product
   adapters of paper_2412_11809_b200/sharded.py -- gloo world size 2 and
   thread ranks -- through tpx_comm_selftest (host buffers, no GPU).
"""
import os
import socket
import threading

import numpy as np
import pytest
import torch

import oracle
import tpxgen
from paper_2412_11809_b200 import sharded
from tests import sharded_ref as model
from tests.sharded_ref import NumpyOps, _feats


def _blocks(n, G):
    cuts = np.linspace(0, n, G + 1).astype(int)
    return list(zip(cuts[:-1], cuts[1:]))


def _run_threads(h, dt, G, W=256, H=256):
    group = model.ThreadGroup(G)
    out = [None] * G
    err = []

    def worker(r, lo, hi):
        try:
            comm = model.ThreadComm(group, r)
            t = torch.from_numpy(h[lo:hi].view(np.uint8).reshape(-1, 16).copy())
            out[r] = model.model_cluster_sharded(t, dt, comm, NumpyOps(dt, W, H))
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)
            group.barrier.abort()

    ths = [threading.Thread(target=worker, args=(r, lo, hi)) for r, (lo, hi) in enumerate(_blocks(len(h), G))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if err:
        raise err[0]
    labels = np.concatenate([o.labels.numpy().view(np.uint32) for o in out])
    feats = np.concatenate([_feats(o.features) for o in out])
    return labels, feats, out


@pytest.mark.parametrize("preset,n,G", [("mixed", 60_000, 2), ("mixed", 60_000, 3), ("lowflux", 40_000, 4),
                                        ("heavyion", 30_000, 2), ("mixed", 80_000, 5)])
def test_thread_ranks_match_oracle(preset, n, G):
    p = tpxgen.PRESETS[preset]
    h = tpxgen.generate(preset, n_hits=n)
    labels, feats, out = _run_threads(h, p["dt_max"], G)
    rl, rf = oracle.cluster(h, p["dt_max"])
    assert np.array_equal(labels, rl)
    assert feats.tobytes() == rf.tobytes()
    assert sum(o.stats["halo_recv"] for o in out) > 0  # the halo path was exercised
    assert sum(o.stats["pairs_total"] for o in out) >= 0


def test_cluster_spanning_three_ranks():
    # a slow serpentine chain over the sensor: one cluster crosses every rank border
    rows = [(i % 256 if (i // 256) % 2 == 0 else 255 - i % 256, i // 256) for i in range(3000)]
    h = tpxgen.make_hits([(x, y, i * 100, 1 + i % 7) for i, (x, y) in enumerate(rows)])
    labels, feats, out = _run_threads(h, 128, 3)
    rl, rf = oracle.cluster(h, 128)
    assert np.array_equal(labels, rl) and feats.tobytes() == rf.tobytes()
    assert len(rf) == 1
    assert out[0].stats["partials_total"] >= 2


def test_rank_skipping_edge_is_rejected():
    h = tpxgen.generate("mixed", n_hits=3000)
    with pytest.raises(model.ModelShardError):
        _run_threads(h, 10**9, 3)


def _gloo_worker(rank, world, port, h, dt, q):
    import torch.distributed as dist

    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        lo, hi = _blocks(len(h), world)[rank]
        t = torch.from_numpy(h[lo:hi].view(np.uint8).reshape(-1, 16).copy())
        res = model.model_cluster_sharded(t, dt, model.TorchComm(), NumpyOps(dt))
        q.put((rank, res.labels.numpy().copy(), res.features.numpy().copy(), res.stats))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_gloo_world_size_2_matches_oracle():
    import torch.multiprocessing as mp

    h = tpxgen.generate("mixed", n_hits=50_000)
    dt = tpxgen.PRESETS["mixed"]["dt_max"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, h, dt, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (l, f, s)) for r, l, f, s in (q.get(timeout=240) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    labels = np.concatenate([res[r][0].view(np.uint32) for r in range(2)])
    feats = np.concatenate([res[r][1].reshape(-1).view(oracle.FEAT_DTYPE) for r in range(2)])
    rl, rf = oracle.cluster(h, dt)
    assert np.array_equal(labels, rl)
    assert feats.tobytes() == rf.tobytes()
    assert res[0][2]["halo_recv"] > 0 and res[1][2]["halo_sent"] > 0


# ------------------------------------------------ the library's host transport
def test_host_transport_thread_ranks():
    G = 3
    group = sharded.ThreadGroup(G)
    rcs = [None] * G

    def worker(r):
        comm = sharded.HostComm(sharded.ThreadAdapter(group, r))
        assert comm.rank_world() == (r, G)
        rcs[r] = comm.selftest(5000)
        comm.close()

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert rcs == [0] * G


def _gloo_transport_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        comm = sharded.HostComm(sharded.TorchAdapter())
        q.put((rank, comm.rank_world(), comm.selftest(70_000)))
        comm.close()
    finally:
        dist.destroy_process_group()


def test_host_transport_gloo_world_size_2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_transport_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == [(0, (0, 2), 0), (1, (1, 2), 0)]
