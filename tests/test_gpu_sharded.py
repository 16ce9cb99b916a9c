"""GPU: the ToA-sharded path with virtual ranks (threads) on one B200.

Same protocol and kernels as a multi-GPU run; collectives are in-process
copies.  Concatenated in rank order the ranks' outputs must equal the
single-GPU output and the oracle bit for bit (shard-count invariance).
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
                comm = sharded.ThreadComm(group, r)
                t = torch.from_numpy(h[lo:hi].view(np.uint8).reshape(-1, 16).copy()).cuda()
                res = sharded.cluster_sharded(t, dt, comm, sharded.CudaOps(dt, W, H))
                torch.cuda.current_stream().synchronize()
                out[r] = (res.labels.cpu().numpy().view(np.uint32).copy(),
                          res.features.cpu().numpy().reshape(-1).view(oracle.FEAT_DTYPE).copy(), res.stats)
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
        assert sum(s["halo_recv"] for s in stats) > 0


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
