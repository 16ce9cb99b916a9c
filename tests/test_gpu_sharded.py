"""GPU: tpx_cluster_run_sharded with virtual ranks (threads) on one B200,
and with a library-owned 1-rank NCCL communicator.

The virtual ranks run the library's whole sharded protocol (csrc/sharded.cuh)
with the host-callback transport (sharded.HostComm + ThreadAdapter: device
buffers staged through pinned memory, in-process exchange); a multi-GPU run
differs only in the transport (NCCL).  Concatenated in rank order the ranks'
outputs must equal the oracle bit for bit (shard-count invariance).
"""
import threading

import numpy as np
import pytest

import oracle
import tpxgen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def mods():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_11809_b200 import build

    build.build()
    import paper_2412_11809_b200 as tpx
    from paper_2412_11809_b200 import sharded

    return tpx, sharded


def _blocks(n, G):
    cuts = np.linspace(0, n, G + 1).astype(int)
    return list(zip(cuts[:-1], cuts[1:]))


def run_virtual(sharded, h, dt, G, W=256, H=256):
    group = sharded.ThreadGroup(G)
    out, err = [None] * G, []

    def worker(r, lo, hi):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                comm = sharded.HostComm(sharded.ThreadAdapter(group, r))
                t = torch.from_numpy(h[lo:hi].view(np.uint8).reshape(-1, 16).copy()).cuda()
                sc = sharded.ShardedClusterer(dt, comm, W, H)
                res = sc.run(t, stream=s)
                s.synchronize()
                out[r] = (res.labels.cpu().numpy().view(np.uint32).copy(),
                          res.features.cpu().numpy().reshape(-1).view(oracle.FEAT_DTYPE).copy(), res.stats,
                          res.offset)
                sc.close()
                comm.close()
        except Exception as e:  # surfaced below
            err.append(e)
            group.barrier.abort()

    ths = [threading.Thread(target=worker, args=(r, lo, hi)) for r, (lo, hi) in enumerate(_blocks(len(h), G))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if err:
        raise err[0]
    assert [o[3] for o in out] == [lo for lo, _ in _blocks(len(h), G)]
    return (np.concatenate([o[0] for o in out]), np.concatenate([o[1] for o in out]), [o[2] for o in out])


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_shard_count_invariance_mixed(mods, G):
    tpx, sharded = mods
    h = tpxgen.generate("mixed", n_hits=2_000_000)
    labels, feats, stats = run_virtual(sharded, h, 320, G)
    rl, rf = oracle.cluster(h, 320)
    assert np.array_equal(labels, rl)
    assert feats.tobytes() == rf.tobytes()
    if G > 1:
        assert sum(s["cross_pairs"] for s in stats) > 0  # boundary pairs were merged


@pytest.mark.parametrize("preset,n,G", [("heavyion", 400_000, 2), ("lowflux", 1_000_000, 4),
                                        ("timepix4", 1_000_000, 3)])
def test_sharded_presets(mods, preset, n, G):
    tpx, sharded = mods
    p = tpxgen.PRESETS[preset]
    W, H = (448, 512) if preset == "timepix4" else (256, 256)
    h = tpxgen.generate(preset, n_hits=n)
    labels, feats, _ = run_virtual(sharded, h, p["dt_max"], G, W, H)
    rl, rf = oracle.cluster(h, p["dt_max"], W, H)
    assert np.array_equal(labels, rl)
    assert feats.tobytes() == rf.tobytes()


def test_sharded_serpentine_cluster(mods):
    tpx, sharded = mods
    rows = [(i % 256 if (i // 256) % 2 == 0 else 255 - i % 256, i // 256) for i in range(20000)]
    h = tpxgen.make_hits([(x, y, i * 100, 1 + i % 7) for i, (x, y) in enumerate(rows)])
    labels, feats, _ = run_virtual(sharded, h, 128, 4)
    rl, rf = oracle.cluster(h, 128)
    assert np.array_equal(labels, rl) and feats.tobytes() == rf.tobytes()


@pytest.mark.parametrize("preset,n", [("mixed", 3_000_000), ("heavyion", 500_000)])
def test_nccl_single_rank(mods, preset, n):
    """The library-owned NCCL communicator (tpx_nccl_unique_id /
    tpx_nccl_comm_init) on one rank: the product transport end to end."""
    tpx, sharded = mods
    p = tpxgen.PRESETS[preset]
    h = tpxgen.generate(preset, n_hits=n)
    comm = sharded.NcclComm(rank=0, world=1)
    sc = sharded.ShardedClusterer(p["dt_max"], comm)
    t = torch.from_numpy(h.view(np.uint8).reshape(-1, 16).copy()).cuda()
    res = sc.run(t)
    torch.cuda.synchronize()
    rl, rf = oracle.cluster(h, p["dt_max"])
    assert res.offset == 0 and res.n_clusters == len(rf)
    assert np.array_equal(res.labels.cpu().numpy().view(np.uint32), rl)
    assert res.features.cpu().numpy().tobytes() == rf.tobytes()
    sc.close()
    comm.close()


def test_rank_skipping_edge_rejected(mods):
    tpx, sharded = mods
    h = tpxgen.generate("mixed", n_hits=30_000)
    with pytest.raises(sharded.ShardError, match="unsupported"):
        run_virtual(sharded, h, 10**9, 3)


def test_capacity_and_small_blocks(mods):
    """Blocks of a few hits (every hit lent), and a feature capacity of 1."""
    tpx, sharded = mods
    rows = [(5 + i % 3, 5, 10 * i, 1 + i % 5) for i in range(24)]
    h = tpxgen.make_hits(rows)
    labels, feats, _ = run_virtual(sharded, h, 25, 2)
    rl, rf = oracle.cluster(h, 25)
    assert np.array_equal(labels, rl) and feats.tobytes() == rf.tobytes()
