"""GPU parity of the cluster-contiguous output (Alg. GPU Step 6) and shape
records (tpx_cluster_run_grouped) against oracle.group / oracle.shapes."""
import numpy as np
import pytest

import oracle
import tpxgen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def tpx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_11809_b200 import build

    build.build()
    import paper_2412_11809_b200 as p

    return p


def _check(tpx, h, dt, W=256, H=256, ctx=""):
    c = tpx.Clusterer(dt, W, H)
    n = len(h)
    d = torch.from_numpy(np.ascontiguousarray(h).view(np.uint8).reshape(-1)).cuda() if n else \
        torch.empty(16, dtype=torch.uint8, device="cuda")
    lab, ft, sh, order, offs, cof, k = c.run_grouped(d, n=n)
    rl, rf = oracle.cluster(h, dt, W, H)
    ro, roff, rcof = oracle.group(h, rl, rf)
    rs = oracle.shapes(h, rl, rf)
    assert k == len(rf), ctx
    assert np.array_equal(lab.cpu().numpy().view(np.uint32), rl), ctx
    assert tpx.features_to_numpy(ft).tobytes() == rf.tobytes(), ctx
    assert np.array_equal(offs.cpu().numpy().view(np.uint32).astype(np.uint64), roff), ctx
    assert np.array_equal(cof.cpu().numpy().view(np.uint32), rcof), ctx
    go = order.cpu().numpy().view(np.uint32)
    bad = np.nonzero(go != ro)[0]
    assert len(bad) == 0, f"{ctx}: order differs at {bad[:5]}"
    assert tpx.shapes_to_numpy(sh).tobytes() == rs.tobytes(), ctx
    return c.stats()


def test_group_small_fuzz(tpx):
    rng = np.random.default_rng(5)
    for t in range(60):
        W, H = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        dt = int(rng.choice([0, 3, 128]))
        h = tpxgen.random_small(rng, int(rng.integers(1, 3000)), W, H, max(4 * dt, 3))
        _check(tpx, h, dt, W, H, ctx=f"trial {t}")


@pytest.mark.parametrize("preset,n", [("tiny", None), ("mixed", 1_000_000), ("heavyion", 500_000),
                                      ("lowflux", 300_000), ("timepix4", 300_000)])
def test_group_presets(tpx, preset, n):
    h = tpxgen.generate(preset, n_hits=n)
    W, H = (448, 512) if preset == "timepix4" else (256, 256)
    _check(tpx, h, tpxgen.PRESETS[preset]["dt_max"], W, H, ctx=preset)


def test_group_edge_cases(tpx):
    _check(tpx, tpxgen.make_hits([(3, 3, 5, 1)]), 10, ctx="one hit")
    _check(tpx, tpxgen.make_hits([(7, 7, 1000, 3)] * 3000), 0, ctx="one cluster")
    _check(tpx, tpxgen.generate("mixed", n_hits=100_000)[::-1].copy(), 320, ctx="reversed")
    _check(tpx, tpxgen.generate("mixed", n_hits=70_000), 100_000, ctx="giant clusters")
    # > 2^16 clusters (three radix passes of the block index)
    _check(tpx, tpxgen.generate("lowflux", n_hits=2_000_000), 128, ctx="many clusters")


def test_group_key_sort_paths(tpx):
    """Both ways of ordering the blocks: the windowed key sort (clusters span
    few sorted positions) and its radix fallback (a cluster spanning more
    than the 1024-position window bound), each exact."""
    st = _check(tpx, tpxgen.generate("mixed", n_hits=400_000), 320, ctx="windowed key sort")
    assert st["sort_retries"] == 0
    # one chain cluster on a single pixel row, interleaved with a background
    # of isolated hits: its hits span > 1024 sorted positions
    rng = np.random.default_rng(11)
    n_bg, n_chain = 60_000, 3_000
    bg = np.zeros(n_bg, dtype=tpxgen.HIT_DTYPE)
    bg["x"], bg["y"] = rng.integers(0, 256, n_bg), rng.integers(0, 100, n_bg)
    bg["toa"], bg["tot"] = np.sort(rng.integers(0, 60 * n_chain, n_bg)), 5
    ch = np.zeros(n_chain, dtype=tpxgen.HIT_DTYPE)
    ch["x"], ch["y"], ch["toa"], ch["tot"] = np.arange(n_chain) % 256, 200 + (np.arange(n_chain) // 256) % 50, \
        np.arange(n_chain) * 60, 7
    h = np.concatenate([bg, ch])
    h = h[np.argsort(h["toa"], kind="stable")]
    st = _check(tpx, h, 60, ctx="long chain")
    assert st["sort_retries"] >= 1
