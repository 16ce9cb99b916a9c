"""GPU parity at the full BASELINE.json sizes, element by element.

configs[2] "mixed" (200M hits), configs[3] "heavyion" (50M) and configs[4]'s
per-GPU shard (2B hits / 8 GPUs = 250M Timepix4 hits on 448x512), each run in
the launch configuration bench.py times (one ``Clusterer.run`` over the whole
device-resident stream, default tile mode).  Every label and every 64-byte
feature record is compared with the oracle (memcmp), and the centroids bit
for bit: north_star "bit-exact ... on every config".

The three oracle runs (single-threaded C, ~0.5-2 min each on the GPU box)
start in background threads when the module's fixture is set up, so they
overlap each other and the GPU work (ctypes releases the GIL).
"""
import concurrent.futures as cf

import numpy as np
import pytest

import oracle
import tpxgen

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")

FULL = {
    # name: (preset, n_hits, width, height)
    "mixed_200M": ("mixed", None, 256, 256),
    "heavyion_50M": ("heavyion", None, 256, 256),
    "timepix4_shard_250M": ("timepix4", 250_000_000, 448, 512),
}


def _oracle_job(preset, n, W, H):
    h = tpxgen.generate(preset, n_hits=n)
    labels, feats = oracle.cluster(h, tpxgen.PRESETS[preset]["dt_max"], W, H)
    return labels, feats


@pytest.fixture(scope="module")
def full_oracle():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ex = cf.ThreadPoolExecutor(max_workers=len(FULL))
    futs = {k: ex.submit(_oracle_job, *v) for k, v in FULL.items()}
    yield futs
    ex.shutdown(wait=True)


@pytest.fixture(scope="module")
def tpx():
    from paper_2412_11809_b200 import build

    build.build()
    import paper_2412_11809_b200 as p

    return p


@pytest.mark.parametrize("name", list(FULL))
def test_full_size_bit_exact(tpx, full_oracle, name):
    preset, n, W, H = FULL[name]
    dt = tpxgen.PRESETS[preset]["dt_max"]
    h = tpxgen.generate(preset, n_hits=n)
    n = len(h)
    d_hits = torch.from_numpy(h.view(np.uint8).reshape(-1)).cuda()
    c = tpx.Clusterer(dt, W, H)
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    feats = torch.empty((n, 64), dtype=torch.uint8, device="cuda")
    ws = torch.empty(c.workspace_bytes(n), dtype=torch.uint8, device="cuda")
    _, _, k = c.run(d_hits, n=n, labels=labels, features=feats, capacity=n, workspace=ws)
    cxy = tpx.centroids(feats[:k])
    torch.cuda.synchronize()
    st = c.stats()
    gl = labels.cpu().numpy().view(np.uint32)
    gf = tpx.features_to_numpy(feats[:k])
    gc = cxy.cpu().numpy()
    del d_hits, labels, feats, ws
    torch.cuda.empty_cache()
    rl, rf = full_oracle[name].result()
    assert k == len(rf), f"{name}: n_clusters {k} vs oracle {len(rf)} (stats {st})"
    bad = np.flatnonzero(gl != rl)
    assert len(bad) == 0, f"{name}: {len(bad)} labels differ, first {bad[:5]}"
    assert gf.tobytes() == rf.tobytes(), f"{name}: feature records differ"
    assert np.array_equal(gc, oracle.centroids(rf)), f"{name}: centroids not bit-identical"
