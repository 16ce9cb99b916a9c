"""The parallel multi-core CPU comparator (cpu_parallel/, SURVEY.md §8(f) f4:
temporal splitting + merge cascade, §3.2.3 l.117-119, §3.3
l.121-139) against the oracle: labels and 64-byte records bit for bit.

Window sizes down to dt_max + 1 ticks put most clusters on a border, so the
merge cascade (temporal distance, bounding boxes, 2D-array full check) and
the merge of clusters spanning several windows are exercised; thread counts
1, 3 and 8 change the window and border assignment."""
import numpy as np
import pytest

import cpu_parallel
import oracle
import tpxgen
from tests import golden_examples


def _same(h, dt, W=256, H=256, **kw):
    rl, rf = oracle.cluster(h, dt, W, H)
    gl, gf, st = cpu_parallel.cluster(h, dt, W, H, stats=True, **kw)
    assert np.array_equal(gl, rl)
    assert gf.tobytes() == rf.tobytes()
    return st


@pytest.mark.parametrize("preset,n", [("tiny", None), ("mixed", 400_000), ("heavyion", 200_000),
                                      ("lowflux", 300_000), ("timepix4", 300_000)])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_presets(preset, n, threads):
    p = tpxgen.PRESETS[preset]
    W, H = (448, 512) if preset == "timepix4" else (256, 256)
    h = tpxgen.generate(preset, n_hits=n)
    _same(h, p["dt_max"], W, H, threads=threads)


@pytest.mark.parametrize("wfac", [1, 2, 5])
def test_small_windows_force_merges(wfac):
    p = tpxgen.PRESETS["mixed"]
    h = tpxgen.generate("mixed", n_hits=200_000, seed=9)
    st = _same(h, p["dt_max"], threads=4, window_ticks=p["dt_max"] * wfac + 1)
    assert st["merges"] > 100 and st["full_checks"] >= st["merges"]


def test_heavyion_blobs_span_windows():
    h = tpxgen.generate("heavyion", n_hits=100_000, seed=3)
    st = _same(h, 64, threads=5, window_ticks=65)
    assert st["merges"] > 0


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_small_sensor(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    W, H = int(rng.integers(1, 9)), int(rng.integers(1, 9))
    dt = int(rng.integers(0, 300))
    h = tpxgen.random_small(rng, n, W, H, int(rng.integers(0, 20 * (dt + 1))))
    _same(h, dt, W, H, threads=int(rng.integers(1, 6)), window_ticks=int(rng.integers(dt + 1, 4 * dt + 3)))


def test_serpentine_cluster_spanning_many_windows():
    rows = [(i % 256 if (i // 256) % 2 == 0 else 255 - i % 256, i // 256) for i in range(5000)]
    h = tpxgen.make_hits([(x, y, i * 100, 1 + i % 7) for i, (x, y) in enumerate(rows)])
    st = _same(h, 128, threads=4, window_ticks=1000)
    assert st["merges"] >= 400


@pytest.mark.parametrize("ex", golden_examples.load(), ids=lambda e: e.eid)
def test_golden_examples(ex):
    gl, gf = cpu_parallel.cluster(ex.hits, ex.dt, ex.width, ex.height, threads=2)
    if ex.labels is not None:
        assert gl.tolist() == ex.labels
    if ex.nclusters is not None:
        assert len(gf) == ex.nclusters
    for want in ex.features:
        row = gf[gf["label"] == want["label"]]
        assert len(row) == 1
        for k, v in want.items():
            assert int(row[k][0]) == v, (ex.eid, k)


def test_coordinate_error():
    h = tpxgen.make_hits([(300, 1, 5)])
    with pytest.raises(RuntimeError):
        cpu_parallel.cluster(h, 10)


def test_empty():
    l, f = cpu_parallel.cluster(tpxgen.make_hits([]), 10)
    assert len(l) == 0 and len(f) == 0
