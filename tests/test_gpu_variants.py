"""GPU parity of variants (iii)(b) GLOBAL and (iii)(c) STATIC (§2
l.40-41) against the oracle's streaming convention
(oracle.cluster_streaming): bit-exact labels; records = the features of
those labels recomputed with numpy (pins.features_from_labels)."""
import numpy as np
import pytest

import oracle
import tpxgen
from tests import golden_examples, pins

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

VARIANTS = {"global": 1, "static": 2}


@pytest.fixture(scope="module")
def tpx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_11809_b200 import build

    build.build()
    import paper_2412_11809_b200 as p

    return p


def _check(tpx, h, dt, variant, W=256, H=256, ctx=""):
    c = tpx.Clusterer(dt, W, H, variant=VARIANTS[variant])
    n = len(h)
    d = torch.from_numpy(np.ascontiguousarray(h).view(np.uint8).reshape(-1)).cuda() if n else \
        torch.empty(16, dtype=torch.uint8, device="cuda")
    labels, feats, k = c.run(d, n=n)
    gl = labels.cpu().numpy().view(np.uint32)[:n]
    gf = tpx.features_to_numpy(feats)
    st = c.stats()
    c.close()
    rl = oracle.cluster_streaming(h, dt, VARIANTS[variant], W, H)
    bad = np.nonzero(gl != rl)[0]
    assert len(bad) == 0, f"{ctx}: {len(bad)} labels differ, first {bad[:5]}"
    ref = pins.features_from_labels(h, rl)
    assert k == len(ref["label"])
    pins.assert_features_equal(gf, ref, ctx)
    return st


@pytest.mark.parametrize("variant", ["global", "static"])
def test_variant_golden_examples(tpx, variant):
    for ex in golden_examples.load():
        want = getattr(ex, f"{variant}_labels", None)
        if want is None:
            continue
        c = tpx.Clusterer(ex.dt, ex.width, ex.height, variant=VARIANTS[variant])
        d = torch.from_numpy(ex.hits.view(np.uint8).reshape(-1)).cuda()
        labels, _, _ = c.run(d, n=len(ex.hits))
        assert labels.cpu().numpy().view(np.uint32).tolist() == want, ex.eid
        c.close()


@pytest.mark.parametrize("variant", ["global", "static"])
def test_variant_fuzz_small(tpx, variant):
    rng = np.random.default_rng(404)
    for trial in range(80):
        W, H = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        dt = int(rng.choice([0, 2, 5, 16, 64]))
        h = tpxgen.random_small(rng, int(rng.integers(1, 600)), W, H, max(6 * dt, 4))
        _check(tpx, h, dt, variant, W, H, ctx=f"{variant} trial {trial}")


@pytest.mark.parametrize("variant", ["global", "static"])
@pytest.mark.parametrize("preset,n", [("tiny", None), ("mixed", 12_000), ("heavyion", 8_000), ("lowflux", 12_000)])
def test_variant_presets(tpx, variant, preset, n):
    h = tpxgen.generate(preset, n_hits=n)
    _check(tpx, h, tpxgen.PRESETS[preset]["dt_max"], variant, ctx=f"{variant}/{preset}")


@pytest.mark.parametrize("variant", ["global", "static"])
def test_variant_dense_pile(tpx, variant):
    """A pile of hits on a 2x2 sensor inside one window: every hit has far
    more adjacent earlier candidates than the large-island kernel lists per
    hit (256), so its full-window fallback scan is exercised; a sparse tail
    keeps the listed path in the same run."""
    rng = np.random.default_rng(909)
    dt = 16
    pile = tpxgen.random_small(rng, 1500, 2, 2, 2 * dt)
    tail = tpxgen.random_small(rng, 1500, 2, 2, 400 * dt)
    tail["toa"] += np.uint64(10 * dt)
    h = np.concatenate([pile, tail])
    _check(tpx, h, dt, variant, 2, 2, ctx=f"{variant} dense pile")


def test_variant_window_growth(tpx):
    # long-lived (b)-clusters: a pixel chain growing for 20 dt -> the island
    # window must grow past the first guess
    hits = [(i % 50, 7, i * 3, 1) for i in range(600)]
    h = tpxgen.make_hits(hits)
    st = _check(tpx, h, 4, "global", ctx="long chain")
    assert st["sort_retries"] >= 1
    _check(tpx, h, 4, "static", ctx="long chain static")


def test_variant_relaxed_dt_reconciles(tpx):
    # relaxing dt makes local and global agree on heavy ions
    h = tpxgen.generate("heavyion", n_hits=6_000)
    big = 1 << 40
    la = oracle.cluster(h, big)[0]
    for v in ("global", "static"):
        _check(tpx, h, big, v, ctx=f"{v} huge dt")
        assert np.array_equal(oracle.cluster_streaming(h, big, VARIANTS[v]), la)
