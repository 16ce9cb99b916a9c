"""Pins for the CPU oracle (oracle/), run with -m "not gpu".

Each test checks the oracle against something other than itself: the
hand-derived examples (tests/golden/examples.txt), O(n^2) brute force with
scipy connected components, the paper's own sequential last-hit-per-pixel
method, scipy.ndimage.label special cases, and invariants (monotonicity,
permutation invariance, large-dt agreement of the variants).
"""
import numpy as np
import pytest
import scipy.ndimage as ndi
from hypothesis import given, settings, strategies as st

import oracle
import tpxgen
from tests import golden_examples, pins


# ----------------------------------------------------------- golden examples
EXAMPLES = golden_examples.load()


@pytest.mark.parametrize("ex", EXAMPLES, ids=[e.eid for e in EXAMPLES])
def test_golden_examples(ex):
    labels, feats = oracle.cluster(ex.hits, ex.dt, ex.width, ex.height)
    if ex.labels is not None:
        assert labels.tolist() == ex.labels, ex.what
    if ex.nclusters is not None:
        assert len(feats) == ex.nclusters
    for want in ex.features:
        row = feats[feats["label"] == want["label"]]
        assert len(row) == 1, ex.what
        for k, v in want.items():
            assert int(row[0][k]) == v, f"{ex.eid} {k}"
    if ex.global_labels is not None:
        got = oracle.cluster_streaming(ex.hits, ex.dt, oracle.GLOBAL, ex.width, ex.height)
        assert got.tolist() == ex.global_labels
    if ex.static_labels is not None:
        got = oracle.cluster_streaming(ex.hits, ex.dt, oracle.STATIC, ex.width, ex.height)
        assert got.tolist() == ex.static_labels
    # the streaming form of (iii)(a) must agree with the BFS oracle everywhere
    if len(ex.hits):
        got = oracle.cluster_streaming(ex.hits, ex.dt, oracle.LOCAL, ex.width, ex.height)
        assert got.tolist() == labels.tolist()


def test_golden_centroid_closed_form():
    # E1: cx = 127/12, cy = 120/12 = 10 exactly (one correctly rounded division)
    ex = next(e for e in EXAMPLES if e.eid == "E1")
    _, feats = oracle.cluster(ex.hits, ex.dt)
    c = oracle.centroids(feats)
    assert c[0, 0] == 127 / 12 and c[0, 1] == 10.0


def test_centroid_symmetric_and_zero_tot():
    # a plus-shaped cluster with equal ToT: weighted centroid = geometric centre
    h = tpxgen.make_hits([(50, 50, 0, 7), (49, 50, 1, 7), (51, 50, 2, 7), (50, 49, 3, 7), (50, 51, 4, 7)])
    _, f = oracle.cluster(h, 10)
    assert oracle.centroids(f).tolist() == [[50.0, 50.0]]
    # tot_sum == 0 falls back to the unweighted centroid (reading R8)
    h = tpxgen.make_hits([(10, 20, 0, 0), (11, 21, 1, 0)])
    _, f = oracle.cluster(h, 10)
    assert oracle.centroids(f).tolist() == [[10.5, 20.5]]


# --------------------------------------------------------------- brute force
def _check_vs_brute(h, dt, W, H):
    labels, feats = oracle.cluster(h, dt, W, H)
    I, J = pins.brute_edges(h, dt)
    ref = pins.cc_labels(len(h), I, J)
    assert np.array_equal(labels, ref)
    pins.assert_features_equal(feats, pins.features_from_labels(h, ref))
    assert oracle.count_edges(h, dt, W, H) == len(I)
    return labels


def test_brute_force_seeded_fuzz():
    rng = np.random.default_rng(1234)
    for trial in range(300):
        W = int(rng.integers(1, 9))
        H = int(rng.integers(1, 9))
        dt = int(rng.choice([0, 1, 3, 16, 128]))
        n = int(rng.integers(0, 200))
        h = tpxgen.random_small(rng, n, W, H, max(4 * dt, 3))
        _check_vs_brute(h, dt, W, H)


@settings(max_examples=150, deadline=None)
@given(
    st.integers(1, 6), st.integers(1, 6), st.integers(0, 40), st.integers(0, 300),
    st.integers(0, 2**31 - 1),
)
def test_brute_force_hypothesis(W, H, dt, n, seed):
    rng = np.random.default_rng(seed)
    h = tpxgen.random_small(rng, n, W, H, max(4 * dt, 2))
    _check_vs_brute(h, dt, W, H)


def test_brute_force_tiny_preset():
    # all of configs[0] (10k hits, 5e7 pairs)
    h = tpxgen.generate("tiny")
    dt = tpxgen.PRESETS["tiny"]["dt_max"]
    _check_vs_brute(h, dt, 256, 256)


def test_brute_force_dense_blobs():
    # heavy-ion shaped input at small n: dense windows, big components
    h = tpxgen.generate("heavyion", n_hits=6000)
    _check_vs_brute(h, 64, 256, 256)


def test_large_toa_values():
    # toa near 2^47 (48-bit ToA space): no overflow in window arithmetic
    rng = np.random.default_rng(7)
    h = tpxgen.random_small(rng, 500, 6, 6, 2000)
    h["toa"] += (1 << 47) - 5000
    _check_vs_brute(h, 100, 6, 6)
    h["toa"] = rng.integers(0, 4, 500)  # toa < dt: the lower window clamps at 0
    _check_vs_brute(h, 100, 6, 6)


# ----------------------------------------------- paper's sequential method (P9)
def test_paper_sequential_method_agrees():
    rng = np.random.default_rng(99)
    for _ in range(100):
        W, H = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        dt = int(rng.choice([0, 2, 10, 50]))
        h = tpxgen.random_small(rng, int(rng.integers(1, 250)), W, H, 200)
        labels, _ = oracle.cluster(h, dt, W, H)
        assert np.array_equal(labels, pins.paper_sequential(h, dt, W, H))
    h = tpxgen.generate("mixed", n_hits=20000)
    labels, _ = oracle.cluster(h, 320)
    assert np.array_equal(labels, pins.paper_sequential(h, 320, 256, 256))


# -------------------------------------------------- library special cases (P4)
def _pixel_ccl_labels(h, W, H):
    img = np.zeros((H, W), dtype=np.int32)
    img[h["y"], h["x"]] = 1
    lab, _ = ndi.label(img, structure=np.ones((3, 3), dtype=int))
    comp = lab[h["y"], h["x"]]
    first = {}
    for i, c in enumerate(comp.tolist()):
        first.setdefault(c, i)
    return np.array([first[c] for c in comp.tolist()], dtype=np.uint32)


def test_large_dt_equals_image_ccl_and_variants_agree():
    rng = np.random.default_rng(5)
    for _ in range(60):
        W, H = int(rng.integers(2, 20)), int(rng.integers(2, 20))
        n = int(rng.integers(1, 120))
        h = tpxgen.random_small(rng, n, W, H, 500)
        dt = 500 + int(rng.integers(0, 3))  # >= ToA span
        labels, _ = oracle.cluster(h, dt, W, H)
        assert np.array_equal(labels, _pixel_ccl_labels(h, W, H))
        # "For large values of dt_max ... identical results"
        for v in (oracle.GLOBAL, oracle.STATIC, oracle.LOCAL):
            assert np.array_equal(oracle.cluster_streaming(h, dt, v, W, H), labels)


def test_dt_zero_is_per_frame_image_ccl():
    rng = np.random.default_rng(6)
    for _ in range(40):
        W, H = int(rng.integers(2, 12)), int(rng.integers(2, 12))
        h = tpxgen.random_small(rng, int(rng.integers(1, 150)), W, H, 5)
        labels, _ = oracle.cluster(h, 0, W, H)
        want = np.zeros(len(h), np.uint32)
        for t in np.unique(h["toa"]):
            idx = np.nonzero(h["toa"] == t)[0]
            sub = _pixel_ccl_labels(h[idx], W, H)
            want[idx] = idx[sub]
        assert np.array_equal(labels, want)


# ------------------------------------------------------------ invariants
def test_monotone_in_dt():
    rng = np.random.default_rng(8)
    h = tpxgen.random_small(rng, 400, 10, 10, 400)
    prev = None
    for dt in (0, 1, 5, 20, 60, 150, 400):
        labels, _ = oracle.cluster(h, dt, 10, 10)
        if prev is not None:
            assert pins.is_refinement(prev, labels)
        prev = labels


def test_permutation_invariance():
    h = tpxgen.generate("mixed", n_hits=30000)
    labels, feats = oracle.cluster(h, 320)
    rng = np.random.default_rng(3)
    perm = rng.permutation(len(h))
    l2, f2 = oracle.cluster(h[perm], 320)
    # same partition: map back to original indices and re-canonicalise
    back = perm[l2]                      # original index of each hit's label
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(h))
    part_perm = back[inv]                # labels for original order (some member index)
    assert pins.is_refinement(labels, part_perm) and pins.is_refinement(part_perm, labels)
    assert len(f2) == len(feats)
    assert int(f2["size"].sum()) == len(h)


def test_certificate_medium_instances():
    # indexed (searchsorted) edge enumeration + scipy CC on 200k hits
    for preset, n in (("lowflux", 200_000), ("mixed", 200_000), ("heavyion", 100_000)):
        h = tpxgen.generate(preset, n_hits=n)
        dt = tpxgen.PRESETS[preset]["dt_max"]
        labels, feats = oracle.cluster(h, dt)
        I, J = pins.indexed_edges(h, dt, 256)
        assert np.array_equal(labels, pins.cc_labels(len(h), I, J)), preset
        pins.assert_features_equal(feats, pins.features_from_labels(h, labels), preset)
        assert oracle.count_edges(h, dt, 256, 256) == len(I)
        assert int(feats["size"].sum()) == n
        assert int(feats["tot_sum"].sum()) == int(h["tot"].astype(np.uint64).sum())


def test_indexed_edges_match_brute():
    rng = np.random.default_rng(11)
    for _ in range(30):
        W, H = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        h = tpxgen.random_small(rng, int(rng.integers(0, 200)), W, H, 60)
        a = set(zip(*pins.brute_edges(h, 15)))
        b = set(zip(*pins.indexed_edges(h, 15, W)))
        assert a == b


def test_component_sampler_matches_full():
    h = tpxgen.generate("mixed", n_hits=50000)
    labels, feats = oracle.cluster(h, 320)
    s = oracle.ComponentSampler(h, 320)
    rng = np.random.default_rng(0)
    for seed in rng.integers(0, len(h), 200).tolist():
        f, mem = s.component(seed, want_members=True)
        lab = labels[seed]
        assert np.array_equal(mem, np.nonzero(labels == lab)[0])
        row = feats[np.searchsorted(feats["label"], lab)]
        for k in pins.FEAT_FIELDS:
            assert int(f[k]) == int(row[k])
    s.close()


def test_errors_and_empty():
    labels, feats = oracle.cluster(np.zeros(0, dtype=tpxgen.HIT_DTYPE), 10)
    assert len(labels) == 0 and len(feats) == 0
    h = tpxgen.make_hits([(256, 0, 0)])
    with pytest.raises(oracle.OracleError):
        oracle.cluster(h, 10, 256, 256)
    h = tpxgen.make_hits([(0, 512, 0)])
    with pytest.raises(oracle.OracleError):
        oracle.cluster(h, 10, 448, 512)


# ------------------------------------------------ shapes and grouping (§8(f) f3)
def _brute_shapes_and_groups(h, labels):
    """Python loops over explicit member lists: bounding box,
    second moments (reading R19), and the Step-6 block order (l.175, R18)."""
    members = {}
    for i, l in enumerate(labels.tolist()):
        members.setdefault(l, []).append(i)
    shapes = {}
    for l, mem in members.items():
        xs = [int(h["x"][i]) for i in mem]
        ys = [int(h["y"][i]) for i in mem]
        shapes[l] = (min(xs), max(xs), min(ys), max(ys), sum(x * x for x in xs),
                     sum(x * y for x, y in zip(xs, ys)), sum(y * y for y in ys))
    blocks = [sorted(mem, key=lambda i: (int(h["toa"][i]), i)) for mem in members.values()]
    blocks.sort(key=lambda b: (int(h["toa"][b[0]]), b[0]))
    return shapes, blocks


def _check_shapes_group(h, dt, W=256, H=256):
    labels, feats = oracle.cluster(h, dt, W, H)
    sh = oracle.shapes(h, labels, feats)
    order, offsets, cof = oracle.group(h, labels, feats)
    bs, blocks = _brute_shapes_and_groups(h, labels)
    assert len(sh) == len(feats) == len(bs)
    for c in range(len(feats)):
        assert tuple(int(v) for v in sh[c]) == bs[int(feats["label"][c])]
    assert len(cof) == len(blocks)
    assert int(offsets[0]) == 0 and int(offsets[-1]) == len(h)
    for g, b in enumerate(blocks):
        got = order[int(offsets[g]):int(offsets[g + 1])].tolist()
        assert got == b, (g, got, b)
        assert int(feats["label"][cof[g]]) == min(b)
        assert int(feats["size"][cof[g]]) == len(b)


def test_shapes_group_hand_examples():
    # Step-6 order by minimum ToA: label 1's cluster (min ToA 10) precedes label 0's
    h = tpxgen.make_hits([(5, 5, 100, 1), (50, 50, 10, 1), (5, 6, 105, 1), (51, 50, 10, 1)])
    labels, feats = oracle.cluster(h, 10)
    order, offsets, cof = oracle.group(h, labels, feats)
    assert order.tolist() == [1, 3, 0, 2] and offsets.tolist() == [0, 2, 4] and cof.tolist() == [1, 0]
    # equal minimum ToA: the earliest hit's input index decides (R18): (10, #1) < (10, #2)
    h = tpxgen.make_hits([(5, 5, 20, 1), (50, 50, 10, 1), (6, 5, 10, 1)])
    labels, feats = oracle.cluster(h, 10)
    order, offsets, cof = oracle.group(h, labels, feats)
    assert order.tolist() == [1, 2, 0] and offsets.tolist() == [0, 1, 3] and cof.tolist() == [1, 0]
    # L-shaped cluster: bbox (1..2, 1..2), sum x^2 = 1+4+4, sum xy = 1+2+4, sum y^2 = 1+1+4
    h = tpxgen.make_hits([(1, 1, 0, 3), (2, 1, 1, 3), (2, 2, 2, 3)])
    labels, feats = oracle.cluster(h, 10)
    sh = oracle.shapes(h, labels, feats)
    assert tuple(int(v) for v in sh[0]) == (1, 2, 1, 2, 9, 7, 6)


def test_shapes_group_vs_brute_fuzz():
    rng = np.random.default_rng(99)
    for _ in range(60):
        W, H = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        dt = int(rng.choice([0, 2, 16]))
        h = tpxgen.random_small(rng, int(rng.integers(1, 400)), W, H, max(4 * dt, 3))
        _check_shapes_group(h, dt, W, H)
    _check_shapes_group(tpxgen.generate("tiny"), 128)
    _check_shapes_group(tpxgen.generate("heavyion", n_hits=20_000), 64)


def test_group_empty():
    h = np.zeros(0, dtype=tpxgen.HIT_DTYPE)
    labels, feats = oracle.cluster(h, 10)
    order, offsets, cof = oracle.group(h, labels, feats)
    assert len(order) == 0 and offsets.tolist() == [0] and len(cof) == 0
    assert len(oracle.shapes(h, labels, feats)) == 0


# --------------------------- streaming variants (iii)(b)/(c): structural pins
def test_streaming_variant_invariants():
    """(c) STATIC: every join is within dt of the cluster's
    first hit, so each (c)-cluster spans <= dt and is connected by (a)-edges
    -> (c) refines (a).  (b) GLOBAL (l.40): every (a)-edge is a (b)-join, so
    (a) refines (b), and each (b)-cluster's sorted ToAs have gaps <= dt
    (R21).  LOCAL streaming equals the CC oracle."""
    rng = np.random.default_rng(31)
    for trial in range(80):
        W, H = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        dt = int(rng.choice([0, 2, 5, 16]))
        h = tpxgen.random_small(rng, int(rng.integers(1, 250)), W, H, max(6 * dt, 4))
        la, _ = oracle.cluster(h, dt, W, H)
        lb = oracle.cluster_streaming(h, dt, oracle.GLOBAL, W, H)
        lc = oracle.cluster_streaming(h, dt, oracle.STATIC, W, H)
        assert np.array_equal(oracle.cluster_streaming(h, dt, oracle.LOCAL, W, H), la)
        assert pins.is_refinement(lc, la) and pins.is_refinement(la, lb), trial
        toa = h["toa"].astype(np.int64)
        for lab in np.unique(lc):
            t = toa[lc == lab]
            assert t.max() - t.min() <= dt
        for lab in np.unique(lb):
            t = np.sort(toa[lb == lab])
            assert (np.diff(t) <= dt).all()
        for lab_arr in (lb, lc):  # canonical labels
            assert (lab_arr <= np.arange(len(h))).all() and np.array_equal(lab_arr[lab_arr], lab_arr)


@pytest.mark.parametrize("variant", [1, 2])
def test_streaming_variants_last_writer_reading(variant):
    """Second implementation of the (b)/(c) streaming oracle (SPEC's
    per-pixel last-writer reference matrix, pins.streaming_last_writer):
    identical labels on fuzz inputs dense enough that pixels are re-hit and
    clusters merge (the R21 reading and the last-writer reading)."""
    rng = np.random.default_rng(100 + variant)
    for _ in range(150):
        n = int(rng.integers(1, 400))
        W, H = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        dt = int(rng.integers(0, 200))
        h = tpxgen.random_small(rng, n, W, H, int(rng.integers(0, 10 * (dt + 1))))
        got = oracle.cluster_streaming(h, dt, variant, W, H)
        want = pins.streaming_last_writer(h, dt, variant)
        assert np.array_equal(got, want), (variant, n, W, H, dt)
    for preset in ("tiny", "heavyion"):
        h = tpxgen.generate(preset, n_hits=3000)
        dt = tpxgen.PRESETS[preset]["dt_max"]
        assert np.array_equal(oracle.cluster_streaming(h, dt, variant), pins.streaming_last_writer(h, dt, variant))


def test_generator_truth_on_separated_clusters():
    """Pin P7: where the generator's clusters are
    separated from every other cluster (>= 2 dt_max apart in time, or bounding
    boxes >= 2 px apart) and away from the sensor edge, the oracle's component
    of each is exactly the generator's cluster (dots: 8-connected growth,
    tracks: rasterised segments, all within dt_max in time)."""
    dt = 320
    h, truth = tpxgen.generate("mixed", n_hits=200_000, truth=True, rate_hz=20_000, seed=31)
    labels, _ = oracle.cluster(h, dt)
    tid = truth.astype(np.int64)
    ids, inv = np.unique(tid, return_inverse=True)
    k = len(ids)
    t = h["toa"].astype(np.int64)
    x, y = h["x"].astype(np.int64), h["y"].astype(np.int64)
    big = np.iinfo(np.int64).max
    tmin = np.full(k, big); np.minimum.at(tmin, inv, t)
    tmax = np.full(k, -1); np.maximum.at(tmax, inv, t)
    x0 = np.full(k, big); np.minimum.at(x0, inv, x)
    x1 = np.full(k, -1); np.maximum.at(x1, inv, x)
    y0 = np.full(k, big); np.minimum.at(y0, inv, y)
    y1 = np.full(k, -1); np.maximum.at(y1, inv, y)
    order = np.argsort(tmin, kind="stable")
    sep = np.ones(k, dtype=bool)
    for a_i, a in enumerate(order.tolist()):
        # every earlier-starting cluster still within 2 dt in time must be >= 2 px away
        for b in order[max(0, a_i - 50):a_i].tolist():
            if tmax[b] + 2 * dt > tmin[a]:
                near = not (x0[a] > x1[b] + 1 or x0[b] > x1[a] + 1 or y0[a] > y1[b] + 1 or y0[b] > y1[a] + 1)
                if near:
                    sep[a] = sep[b] = False
    # clusters touching the sensor edge may have lost off-sensor pixels (the
    # generator drops them) and so need not be connected
    sep &= (x0 > 0) & (y0 > 0) & (x1 < 255) & (y1 < 255)
    # the stream stops at exactly n hits in readout order: clusters within the
    # readout disorder (<= 22.8k ticks) of the end may be truncated
    sep &= tmin < t.max() - 50_000
    assert sep.mean() > 0.9
    # per separated truth cluster: one oracle label, and that label's component is exactly the cluster
    members = {}
    for i, c in enumerate(inv.tolist()):
        if sep[c]:
            members.setdefault(c, []).append(i)
    lab_count = np.bincount(labels.astype(np.int64), minlength=len(h))
    for c, mem in members.items():
        ls = set(labels[mem].tolist())
        assert len(ls) == 1, f"truth cluster {ids[c]} split: {ls}"
        assert lab_count[ls.pop()] == len(mem), f"truth cluster {ids[c]} merged with other hits"
