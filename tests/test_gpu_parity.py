"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Bit-exact labels and integer features on the same seeded inputs; centroids
within relative 1e-12 (north_star; expected bit-identical, reading R9).
"""
import numpy as np
import pytest

import oracle
import tpxgen
from tests import golden_examples, pins

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


_ctx_cache = {}


def _gpu(tpx, h, dt, W=256, H=256, capacity=None, tile_mode="auto"):
    key = (dt, W, H, tile_mode)
    if key not in _ctx_cache:
        _ctx_cache[key] = tpx.Clusterer(dt, W, H)
        _ctx_cache[key].set_tile_mode(tile_mode)
    c = _ctx_cache[key]
    n = len(h)
    d = torch.from_numpy(np.ascontiguousarray(h).view(np.uint8).reshape(-1)).cuda() if n else \
        torch.empty(16, dtype=torch.uint8, device="cuda")
    labels, feats, k = c.run(d, n=n, capacity=capacity)
    cxy = tpx.centroids(feats)
    torch.cuda.synchronize()
    return (labels.cpu().numpy().view(np.uint32)[:n], tpx.features_to_numpy(feats), k,
            cxy.cpu().numpy(), c.stats())


def _assert_parity(tpx, h, dt, W=256, H=256, ctx="", tile_mode="auto"):
    gl, gf, k, gc, st = _gpu(tpx, h, dt, W, H, tile_mode=tile_mode)
    rl, rf = oracle.cluster(h, dt, W, H)
    assert k == len(rf), f"{ctx}: n_clusters {k} vs {len(rf)}"
    bad = np.nonzero(gl != rl)[0]
    assert len(bad) == 0, f"{ctx}: {len(bad)} labels differ, first {bad[:5]}: {gl[bad[:5]]} vs {rl[bad[:5]]}"
    if gf.tobytes() != rf.tobytes():
        for name in pins.FEAT_FIELDS:
            d = np.nonzero(gf[name] != rf[name])[0]
            assert len(d) == 0, f"{ctx}: feature {name} differs at {d[:5]}"
    rc = oracle.centroids(rf)
    if len(rc):
        rel = np.abs(gc - rc) / np.maximum(np.abs(rc), 1e-300)
        assert rel.max() <= 1e-12, f"{ctx}: centroid rel err {rel.max()}"
        assert np.array_equal(gc, rc), f"{ctx}: centroids not bit-identical"
    return st


# ----------------------------------------------------------------- examples
EXAMPLES = golden_examples.load()


@pytest.mark.parametrize("ex", EXAMPLES, ids=[e.eid for e in EXAMPLES])
def test_golden_examples_gpu(tpx, ex):
    gl, gf, k, _, _ = _gpu(tpx, ex.hits, ex.dt, ex.width, ex.height)
    if ex.labels is not None:
        assert gl.tolist() == ex.labels
    if ex.nclusters is not None:
        assert k == ex.nclusters
    for want in ex.features:
        row = gf[gf["label"] == want["label"]]
        assert len(row) == 1
        for key, v in want.items():
            assert int(row[0][key]) == v


# --------------------------------------------------------------- fuzz parity
def test_fuzz_small_sensors(tpx):
    rng = np.random.default_rng(2024)
    for trial in range(150):
        W, H = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        dt = int(rng.choice([0, 1, 3, 16, 128]))
        n = int(rng.integers(1, 3000))
        h = tpxgen.random_small(rng, n, W, H, max(4 * dt, 3))
        _assert_parity(tpx, h, dt, W, H, ctx=f"trial {trial}")


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 4095, 4096, 4097, 8191, 65537, 300_001])
def test_sizes_spanning_tiles(tpx, n):
    h = tpxgen.generate("mixed", n_hits=n)
    _assert_parity(tpx, h, 320, ctx=f"n={n}")


@pytest.mark.parametrize("preset,n", [("tiny", None), ("lowflux", 2_000_000), ("mixed", 3_000_000),
                                      ("heavyion", 1_000_000), ("timepix4", 2_000_000)])
def test_presets(tpx, preset, n):
    p = tpxgen.PRESETS[preset]
    h = tpxgen.generate(preset, n_hits=n)
    W, H = (448, 512) if preset == "timepix4" else (256, 256)
    _assert_parity(tpx, h, p["dt_max"], W, H, ctx=preset)


@pytest.mark.parametrize("mode", ["sparse", "dense", "cell"])
@pytest.mark.parametrize("preset,n", [("mixed", 1_000_000), ("heavyion", 1_000_000), ("lowflux", 500_000),
                                      ("timepix4", 1_000_000)])
def test_forced_tile_modes(tpx, mode, preset, n):
    """Every tile configuration gives the oracle's result on every workload
    (the density probe only chooses the faster one)."""
    h = tpxgen.generate(preset, n_hits=n)
    W, H = (448, 512) if preset == "timepix4" else (256, 256)
    st = _assert_parity(tpx, h, tpxgen.PRESETS[preset]["dt_max"], W, H, ctx=f"{preset}/{mode}", tile_mode=mode)
    assert st["tile_dense"] == (mode == "dense")


@pytest.mark.parametrize("mode", ["sparse", "cell"])
def test_forced_sparse_small_and_fuzz(tpx, mode):
    """Sparse kernels on small and odd sensors (cell aliasing: widths/heights
    above 256 share cell slots modulo 256 pixels), tiny dt and ragged sizes."""
    rng = np.random.default_rng(78)
    for trial in range(40):
        W, H = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        dt = int(rng.choice([0, 3, 128]))
        h = tpxgen.random_small(rng, int(rng.integers(1, 5000)), W, H, max(4 * dt, 3))
        _assert_parity(tpx, h, dt, W, H, ctx=f"{mode} trial {trial}", tile_mode=mode)
    for trial in range(6):
        W, H = int(rng.integers(250, 1025)), int(rng.integers(250, 1025))
        dt = int(rng.choice([3, 64, 320]))
        nc = int(rng.integers(100, 4000))
        cx, cy = rng.integers(0, W, nc), rng.integers(0, H, nc)
        ct = np.sort(rng.integers(0, 200 * dt, nc))
        k = rng.integers(0, nc, 8 * nc)  # 8 hits per blob on average, clipped to the sensor
        h = np.zeros(len(k), dtype=tpxgen.HIT_DTYPE)
        h["x"] = np.clip(cx[k] + rng.integers(-2, 3, len(k)), 0, W - 1)
        h["y"] = np.clip(cy[k] + rng.integers(-2, 3, len(k)), 0, H - 1)
        h["toa"] = ct[k] + rng.integers(0, dt + 1, len(k))
        h["tot"] = rng.integers(1, 1024, len(k))
        _assert_parity(tpx, h, dt, W, H, ctx=f"{mode} wide-sensor trial {trial}", tile_mode=mode)
    for n in (2047, 2048, 2049, 4097, 65537):
        _assert_parity(tpx, tpxgen.generate("mixed", n_hits=n), 320, ctx=f"{mode} n={n}", tile_mode=mode)
    # widths / heights at the cell-grid wrap (256) and the CSR coordinate
    # limit (1023; 1025 falls back to the linked-list cell kernel)
    for W, H in ((257, 9), (511, 513), (512, 257), (1023, 1024), (1024, 1023), (1025, 31), (31, 1025)):
        nh = 30_000
        h = np.zeros(nh, dtype=tpxgen.HIT_DTYPE)
        cx, cy = rng.integers(0, W, nh // 6), rng.integers(0, H, nh // 6)
        k = rng.integers(0, nh // 6, nh)
        h["x"] = np.clip(cx[k] + rng.integers(-1, 2, nh), 0, W - 1)
        h["y"] = np.clip(cy[k] + rng.integers(-1, 2, nh), 0, H - 1)
        h["toa"] = np.sort(rng.integers(0, 40 * nh, nh))
        h["tot"] = rng.integers(1, 1024, nh)
        _assert_parity(tpx, h, 320, W, H, ctx=f"{mode} edge sensor {W}x{H}", tile_mode=mode)


def test_forced_dense_small_and_fuzz(tpx):
    rng = np.random.default_rng(77)
    for trial in range(40):
        W, H = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        dt = int(rng.choice([0, 3, 128]))
        h = tpxgen.random_small(rng, int(rng.integers(1, 5000)), W, H, max(4 * dt, 3))
        _assert_parity(tpx, h, dt, W, H, ctx=f"dense trial {trial}", tile_mode="dense")
    for n in (4095, 4097, 65537):
        _assert_parity(tpx, tpxgen.generate("mixed", n_hits=n), 320, ctx=f"dense n={n}", tile_mode="dense")


def test_density_probe_choice(tpx):
    _, _, _, _, st = _gpu(tpx, tpxgen.generate("heavyion", n_hits=2_000_000), 64)
    assert st["tile_dense"] == 1
    _, _, _, _, st = _gpu(tpx, tpxgen.generate("lowflux", n_hits=2_000_000), 128)
    assert st["tile_dense"] == 0


def test_lowflux_full_config(tpx):
    # BASELINE.json configs[1] at its full size (10M hits)
    h = tpxgen.generate("lowflux")
    _assert_parity(tpx, h, 128, ctx="lowflux-10M")


@pytest.mark.parametrize("dt", [0, 1, 64, 1000, 100_000])
def test_dt_sweep(tpx, dt):
    h = tpxgen.generate("mixed", n_hits=200_000)
    _assert_parity(tpx, h, dt, ctx=f"dt={dt}")


# -------------------------------------------------------------- edge cases
def test_empty_and_degenerate(tpx):
    gl, gf, k, _, _ = _gpu(tpx, np.zeros(0, dtype=tpxgen.HIT_DTYPE), 128)
    assert k == 0
    # all hits on one pixel at one time: one cluster
    h = tpxgen.make_hits([(7, 7, 1000, 3)] * 5000)
    _assert_parity(tpx, h, 0, ctx="one pixel")
    # a diagonal chain over the whole sensor, each step exactly dt apart
    h = tpxgen.make_hits([(i % 256, i % 256, i * 128, 1) for i in range(20000)])
    _assert_parity(tpx, h, 128, ctx="chain")
    # reverse-sorted input
    h = tpxgen.generate("mixed", n_hits=100_000)[::-1].copy()
    _assert_parity(tpx, h, 320, ctx="reversed")
    # ToA near 2^48 and large ToA span (> 32 bits of key)
    h = tpxgen.generate("mixed", n_hits=50_000)
    h["toa"][::7] += np.uint64(1 << 40)
    h["toa"] += np.uint64((1 << 47))
    _assert_parity(tpx, h, 320, ctx="wide toa")


def _fresh(tpx, h, dt, W=256, H=256):
    c = tpx.Clusterer(dt, W, H)
    d = torch.from_numpy(np.ascontiguousarray(h).view(np.uint8).reshape(-1)).cuda()
    labels, feats, k = c.run(d, n=len(h))
    torch.cuda.synchronize()
    return c, labels.cpu().numpy().view(np.uint32)[:len(h)], tpx.features_to_numpy(feats), k


def test_disorder_stress(tpx):
    # paper-bound readout disorder t = 600 us; a fresh
    # context, so the shared ones keep starting with the windowed sort
    h = tpxgen.generate("mixed", n_hits=2_000_000, disorder_ticks=384_000)
    c, gl, gf, k = _fresh(tpx, h, 320)
    rl, rf = oracle.cluster(h, 320)
    assert np.array_equal(gl, rl) and gf.tobytes() == rf.tobytes()


def test_context_reuse_across_changing_streams(tpx):
    """One context through streams that break what its previous runs learnt:
    the remembered sort attempt (sort_start) and tile configuration meet more
    disorder, heavy-ion windows, a beam pause wider than 2^32 ticks (the
    radix fallback's guessed key origin fails), a calm stream again, and an
    invalid coordinate after the radix path became the start (validation
    fused into the radix histogram must still flag it); every run bit-exact,
    the error reported, the context usable afterwards."""
    c = tpx.Clusterer(320)
    streams = [
        ("mixed", tpxgen.generate("mixed", n_hits=1_000_000, seed=61)),
        ("mixed again", tpxgen.generate("mixed", n_hits=1_000_000, seed=62)),
        ("heavy-ion windows", tpxgen.generate("heavyion", n_hits=600_000, seed=63)),
        ("sparse again", tpxgen.generate("mixed", n_hits=700_000, seed=64)),
        ("600 us disorder: window sort fails", tpxgen.generate("mixed", n_hits=800_000, seed=65,
                                                               disorder_ticks=384_000)),
        ("clean again", tpxgen.generate("mixed", n_hits=900_000, seed=66)),
    ]
    pause = tpxgen.generate("mixed", n_hits=600_000, seed=67)
    pause["toa"][300_000:] += np.uint64(1 << 33)  # beam pause: a window spans > 2^32 ticks
    streams.append(("beam pause", pause))
    streams.append(("clean after the pause", tpxgen.generate("mixed", n_hits=500_000, seed=68)))
    for name, h in streams:
        d = torch.from_numpy(np.ascontiguousarray(h).view(np.uint8).reshape(-1)).cuda()
        labels, feats, k = c.run(d, n=len(h))
        torch.cuda.synchronize()
        rl, rf = oracle.cluster(h, 320)
        assert k == len(rf), name
        assert np.array_equal(labels.cpu().numpy().view(np.uint32)[:len(h)], rl), name
        assert tpx.features_to_numpy(feats).tobytes() == rf.tobytes(), name
    bad = tpxgen.generate("mixed", n_hits=200_000, seed=69)
    bad["x"][150_000] = 300  # outside the 256-pixel sensor
    d = torch.from_numpy(np.ascontiguousarray(bad).view(np.uint8).reshape(-1)).cuda()
    with pytest.raises(tpx.TpxError) as e:
        c.run(d, n=len(bad))
    assert e.value.status == -3  # TPX_ERR_COORD_RANGE
    h = tpxgen.generate("mixed", n_hits=400_000, seed=70)  # and the context still works
    d = torch.from_numpy(np.ascontiguousarray(h).view(np.uint8).reshape(-1)).cuda()
    labels, feats, k = c.run(d, n=len(h))
    rl, rf = oracle.cluster(h, 320)
    assert np.array_equal(labels.cpu().numpy().view(np.uint32)[:len(h)], rl)
    assert tpx.features_to_numpy(feats).tobytes() == rf.tobytes()


@pytest.mark.parametrize("n,toa_max", [(12_289, 1 << 14), (40_961, (1 << 23) + 5), (100_003, (1 << 31) - 3),
                                         ((1 << 20) + 7, 1 << 20), (300_001, (1 << 24) + 1)])
def test_radix_fallback_edges(tpx, n, toa_max):
    """The global radix sort (radix_onesweep.cuh): unordered input (the window
    sort cannot hold its displacement bound, so the fallback runs), sizes that
    leave a partial last 4096-key tile, and ToA ranges needing 2, 3 and 4
    8-bit passes; 16x16 sensor so clusters are many and large."""
    rng = np.random.default_rng(n)
    h = tpxgen.random_small(rng, n, 16, 16, toa_max)
    c, gl, gf, k = _fresh(tpx, h, 64, 16, 16)
    assert c.stats()["sort_path"] == 1
    rl, rf = oracle.cluster(h, 64, 16, 16)
    assert np.array_equal(gl, rl) and gf.tobytes() == rf.tobytes()


@pytest.mark.parametrize("shape", ["early_outlier", "wide_range"])
def test_radix_guessed_base_falls_back(tpx, shape):
    """The radix fallback first guesses its key origin (smallest ToA of the
    first 8192 hits less 2^28 ticks, sort.cuh k_radix_base) and checks every
    key against it; a stream that breaks the guess -- a hit far earlier than
    the first ones, or a ToA range beyond 2^32 ticks from the guess -- is
    re-sorted from the exact minimum, bit-exact either way."""
    rng = np.random.default_rng(7 if shape == "early_outlier" else 8)
    n = 30_000
    h = tpxgen.random_small(rng, n, 16, 16, 1 << 20)
    h["toa"] += np.uint64(1 << 34)
    if shape == "early_outlier":
        # 2^30 ticks before everything else, at the end of the stream: taken
        # modulo 2^32 from the guessed origin its key would sort it last
        h["toa"][n - 5] = (1 << 34) - (1 << 30)
    else:
        h["toa"][n // 2:] += np.uint64(1 << 33)  # range > 2^32 ticks: 64-bit keys
    c, gl, gf, k = _fresh(tpx, h, 64, 16, 16)
    assert c.stats()["sort_path"] == 1
    rl, rf = oracle.cluster(h, 64, 16, 16)
    assert np.array_equal(gl, rl) and gf.tobytes() == rf.tobytes()


def test_packed_sort_wide_windows_fall_back(tpx):
    """A stream whose 13312-hit windows span more than 2^28 ticks (but less
    than 2^31): the packed window sort declines (err bit 3) and the unpacked
    kernel with the same displacement bound sorts it -- still bit-exact."""
    rng = np.random.default_rng(77)
    n = 60_000
    h = np.zeros(n, dtype=tpxgen.HIT_DTYPE)
    toa = np.sort(rng.integers(0, (1 << 31) - (1 << 26), n))  # 13312-hit windows span ~4.7e8 ticks
    # light readout disorder: swap a few neighbours
    idx = rng.integers(0, n - 1, n // 20)
    toa[idx], toa[idx + 1] = toa[idx + 1].copy(), toa[idx].copy()
    h["toa"] = toa
    h["x"] = rng.integers(0, 64, n)
    h["y"] = rng.integers(0, 64, n)
    h["tot"] = rng.integers(1, 1024, n)
    c, gl, gf, k = _fresh(tpx, h, 1 << 22, 64, 64)
    st = c.stats()
    assert st["sort_path"] == 0 and st["sort_retries"] >= 1
    rl, rf = oracle.cluster(h, 1 << 22, 64, 64)
    assert np.array_equal(gl, rl) and gf.tobytes() == rf.tobytes()


def test_sort_attempt_memory(tpx):
    """A failed displacement bound is detected right after the sort (no
    clustering pass on a wrong order) and the context starts at the attempt
    that succeeded on later runs; results stay exact on any later stream."""
    h_bad = tpxgen.generate("mixed", n_hits=1_500_000, disorder_ticks=384_000)
    c, gl, gf, k = _fresh(tpx, h_bad, 320)
    st1 = c.stats()
    assert st1["sort_retries"] >= 1
    d = torch.from_numpy(h_bad.view(np.uint8)).cuda()
    c.run(d)
    st2 = c.stats()
    assert st2["sort_retries"] == 0 and st2["sort_path"] == st1["sort_path"]
    # the same context on a well-ordered stream: still exact
    h_ok = tpxgen.generate("mixed", n_hits=1_000_000)
    d = torch.from_numpy(h_ok.view(np.uint8)).cuda()
    labels, feats, k = c.run(d)
    torch.cuda.synchronize()
    rl, rf = oracle.cluster(h_ok, 320)
    assert np.array_equal(labels.cpu().numpy().view(np.uint32), rl)
    assert tpx.features_to_numpy(feats).tobytes() == rf.tobytes()


def test_coord_range_error(tpx):
    h = tpxgen.generate("tiny")
    h["x"][123] = 256
    with pytest.raises(tpx.TpxError) as e:
        _gpu(tpx, h, 128)
    assert e.value.status == -3
    h = tpxgen.generate("tiny")
    h["toa"][5] = np.uint64(1 << 48)
    with pytest.raises(tpx.TpxError) as e:
        _gpu(tpx, h, 128)
    assert e.value.status == -3


def test_capacity_too_small(tpx):
    h = tpxgen.generate("tiny")
    rl, rf = oracle.cluster(h, 128)
    c = tpx.Clusterer(128)
    d = torch.from_numpy(h.view(np.uint8)).cuda()
    labels, feats, k = c.run(d, capacity=100, check=False)
    assert k == len(rf)
    assert np.array_equal(labels.cpu().numpy().view(np.uint32), rl)
    assert tpx.features_to_numpy(feats).tobytes() == rf[:100].tobytes()


def test_deterministic_repeat(tpx):
    h = tpxgen.generate("heavyion", n_hits=500_000)
    a = _gpu(tpx, h, 64)
    b = _gpu(tpx, h, 64)
    assert np.array_equal(a[0], b[0]) and a[1].tobytes() == b[1].tobytes()


def test_permuted_input(tpx):
    h = tpxgen.generate("mixed", n_hits=300_000)
    perm = np.random.default_rng(1).permutation(len(h))
    _assert_parity(tpx, h[perm].copy(), 320, ctx="permuted")


def test_run_host_matches_device(tpx):
    h = tpxgen.generate("mixed", n_hits=1_000_000)
    rl, rf = oracle.cluster(h, 320)
    c = tpx.Clusterer(320)
    hits = torch.from_numpy(h.view(np.uint8)).pin_memory()
    labels = torch.empty(len(h), dtype=torch.int32).pin_memory()
    feats = torch.empty((len(h), 64), dtype=torch.uint8).pin_memory()
    k = c.run_host(hits, labels, feats)
    assert k == len(rf)
    assert np.array_equal(labels.numpy().view(np.uint32), rl)
    assert tpx.features_to_numpy(feats[:k]).tobytes() == rf.tobytes()


# Full BASELINE sizes: element-by-element parity in tests/test_gpu_fullsize.py.


def test_pipeline_matches_run_host(tpx):
    """tpx_pipeline_*: several buffers in flight give exactly run_host's results."""
    bufs = [tpxgen.generate(p, n_hits=m, seed=s) for p, m, s in
            (("mixed", 700_000, 11), ("lowflux", 300_000, 12), ("heavyion", 200_000, 13), ("mixed", 1_000_000, 14),
             ("tiny", 10_000, 15))]
    dts = {"mixed": 320, "lowflux": 320, "heavyion": 320, "tiny": 320}
    pipe = tpx.Pipeline(320, max_hits=1_000_000, capacity=1_000_000, depth=3)
    outs, tickets = [], []
    for h in bufs:
        hh = torch.from_numpy(h.view(np.uint8)).pin_memory()
        lab = torch.empty(len(h), dtype=torch.int32).pin_memory()
        ft = torch.empty((len(h), 64), dtype=torch.uint8).pin_memory()
        outs.append((hh, lab, ft))
        tickets.append(pipe.submit(hh, lab, ft))
    for h, (hh, lab, ft), t in zip(bufs, outs, tickets):
        k = pipe.wait(t)
        rl, rf = oracle.cluster(h, 320)
        assert k == len(rf)
        assert np.array_equal(lab.numpy().view(np.uint32), rl)
        assert tpx.features_to_numpy(ft[:k]).tobytes() == rf.tobytes()
    pipe.close()
