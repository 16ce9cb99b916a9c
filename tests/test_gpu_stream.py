"""Streaming ingest (tpx_stream_*): the union of all emitted
batches equals the oracle's clustering of the WHOLE stream (labels =
smallest arrival index), whatever the buffer borders; batches follow the
Step-6 order."""
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


def _disorder(h) -> int:
    toa = h["toa"].astype(np.int64)
    pref = np.maximum.accumulate(toa)
    return int(max(0, (pref[:-1] - toa[1:]).max(initial=0))) + 1


def _run_stream(tpx, h, dt, b, b_t, t_closing, chunks, W=256, H=256, max_dev=None):
    s = tpx.Stream(dt, b, b_t, _disorder(h), t_closing, max_device_hits=max_dev, width=W, height=H)
    batches = []
    rng = np.random.default_rng(3)
    i = 0
    while i < len(h):
        m = int(rng.integers(1, chunks))
        s.push(h[i:i + m])
        i += m
        while (bt := s.pop()) is not None:
            batches.append(bt)
    s.flush()
    while (bt := s.pop()) is not None:
        batches.append(bt)
    st = s.stats()
    s.close()
    return batches, st


def _check_stream(tpx, h, dt, b, b_t, t_closing, chunks=50_000, W=256, H=256, max_dev=None):
    n = len(h)
    batches, st = _run_stream(tpx, h, dt, b, b_t, t_closing, chunks, W, H, max_dev)
    assert st["late_hits"] == 0 and st["hits_in"] == n and st["hits_out"] == n
    rl, rf = oracle.cluster(h, dt, W, H)
    labels = np.full(n, -1, dtype=np.int64)
    recs = []
    for bt in batches:
        cl, hits, g = bt["clusters"], bt["hits"], bt["hit_index"]
        # Step-6 order inside the batch: clusters by earliest (toa, arrival),
        # hits of a cluster contiguous in (toa, arrival) order
        first = []
        for c in cl:
            o, sz = int(c["offset"]), int(c["size"])
            blk_t, blk_g = hits["toa"][o:o + sz].astype(np.uint64), g[o:o + sz]
            key = blk_t.astype(object) * (1 << 40) + blk_g.astype(object)
            assert all(key[i] < key[i + 1] for i in range(sz - 1))
            first.append(key[0])
            assert labels[blk_g].max() == -1, "hit emitted twice"
            labels[blk_g] = int(c["label"])
            assert np.array_equal(hits[o:o + sz].view(np.uint8), h[blk_g].view(np.uint8)), "hit payload"
        assert all(first[i] < first[i + 1] for i in range(len(first) - 1))
        recs.append(cl)
    assert (labels >= 0).all()
    assert np.array_equal(labels.astype(np.uint32), rl)
    allc = np.concatenate(recs) if recs else np.zeros(0, dtype=tpx.STREAM_CLUSTER_DTYPE)
    allc = allc[np.argsort(allc["label"], kind="stable")]
    assert len(allc) == len(rf)
    assert np.array_equal(allc["label"], rf["label"].astype(np.uint64))
    for name in ("size", "toa_min", "toa_max", "tot_sum", "sum_x", "sum_y", "sum_tot_x", "sum_tot_y"):
        assert np.array_equal(allc[name].astype(np.uint64), rf[name].astype(np.uint64)), name
    return batches, st


@pytest.mark.parametrize("b,b_t,t_closing", [(50_000, 10_000, 64), (20_000, 15_000, 0), (200_000, 30_000, 640)])
def test_stream_mixed_equals_whole_stream(tpx, b, b_t, t_closing):
    h = tpxgen.generate("mixed", n_hits=600_000)
    batches, st = _check_stream(tpx, h, 320, b, b_t, t_closing)
    assert st["buffers"] >= 3 and st["carried_max"] > 0


def test_stream_heavyion_and_lowflux(tpx):
    h = tpxgen.generate("heavyion", n_hits=300_000)
    _check_stream(tpx, h, 64, 60_000, 20_000, 256, max_dev=300_000)
    h = tpxgen.generate("lowflux", n_hits=300_000)
    _check_stream(tpx, h, 128, 40_000, 5_000, 64)


def test_stream_single_buffer_and_tiny_pushes(tpx):
    h = tpxgen.generate("tiny")
    _check_stream(tpx, h, 128, 1_000_000, 1_000, 64)   # never fills: all at flush
    _check_stream(tpx, h, 128, 2_000, 1_000, 64, chunks=3)  # many buffers, pushes of 1-2 hits


def test_stream_paper_disorder(tpx):
    # readout disorder up to 600 us
    h = tpxgen.generate("mixed", n_hits=400_000, disorder_ticks=384_000)
    _check_stream(tpx, h, 320, 100_000, 40_000, 64, max_dev=400_000)


def test_stream_capacity_error(tpx):
    h = tpxgen.generate("mixed", n_hits=100_000)
    # dt so large that everything stays open: the carry must overflow
    s = tpx.Stream(10_000_000, 10_000, 2_000, _disorder(h), 0, max_device_hits=12_001)
    with pytest.raises(tpx.TpxError) as e:
        s.push(h)
    assert e.value.status == -5
    s.close()


# --------------------------------------------- one-shot host-to-host run
def _run_host(tpx, h, dt, b, b_t, t_closing, max_dev=None, capacity=None, W=256, H=256):
    r = tpx.StreamRunner(dt, b, b_t, _disorder(h), t_closing, max_device_hits=max_dev, width=W, height=H)
    hh = torch.from_numpy(np.ascontiguousarray(h).view(np.uint8)).pin_memory()
    order = np.zeros(max(len(h), 1), dtype=np.uint32)
    cl = np.zeros(max(capacity or len(h), 1), dtype=tpx.STREAM_CLUSTER_DTYPE)
    k = r.run(hh, order, cl, capacity=capacity or len(h))
    return order[:len(h)], cl[:k], r.last_stats


@pytest.mark.parametrize("b,b_t,t_closing", [(50_000, 10_000, 64), (20_000, 15_000, 0), (1_000_000, 30_000, 640)])
def test_run_host_equals_push_api(tpx, b, b_t, t_closing):
    h = tpxgen.generate("mixed", n_hits=600_000)
    batches, _ = _check_stream(tpx, h, 320, b, b_t, t_closing)
    order, cl, st = _run_host(tpx, h, 320, b, b_t, t_closing)
    ref_order = np.concatenate([bt["hit_index"] for bt in batches]).astype(np.uint32)
    assert np.array_equal(order, ref_order)
    ref_cl = np.concatenate([bt["clusters"] for bt in batches])
    for name in ("label", "size", "toa_min", "toa_max", "tot_sum", "sum_x", "sum_y", "sum_tot_x", "sum_tot_y"):
        assert np.array_equal(cl[name], ref_cl[name]), name
    # offsets index order_out; every block holds its cluster's hits
    assert (np.diff(cl["offset"].astype(np.int64)) > 0).all() and int(cl["offset"][0]) == 0
    assert st["hits_out"] == len(h) and st["late_hits"] == 0 and st["buffers"] == len(batches)


def test_run_host_vs_oracle_presets(tpx):
    for preset, dt, b, b_t, tc in (("heavyion", 64, 100_000, 20_000, 256), ("lowflux", 128, 40_000, 5_000, 64),
                                   ("tiny", 128, 3_000, 1_000, 0)):
        h = tpxgen.generate(preset, n_hits=None if preset == "tiny" else 300_000)
        order, cl, st = _run_host(tpx, h, dt, b, b_t, tc, max_dev=4 * (b + b_t))
        rl, rf = oracle.cluster(h, dt)
        labels = np.empty(len(h), dtype=np.uint64)
        for c in cl:
            o, sz = int(c["offset"]), int(c["size"])
            labels[order[o:o + sz]] = c["label"]
        assert np.array_equal(labels.astype(np.uint32), rl), preset
        srt = cl[np.argsort(cl["label"], kind="stable")]
        assert np.array_equal(srt["label"], rf["label"].astype(np.uint64))
        for name in ("size", "toa_min", "toa_max", "tot_sum", "sum_x", "sum_y", "sum_tot_x", "sum_tot_y"):
            assert np.array_equal(srt[name].astype(np.uint64), rf[name].astype(np.uint64)), (preset, name)


def test_run_host_capacity_and_empty(tpx):
    h = tpxgen.generate("mixed", n_hits=100_000)
    with pytest.raises(tpx.TpxError) as e:
        _run_host(tpx, h, 320, 20_000, 5_000, 64, capacity=10)
    assert e.value.status == -5
    order, cl, st = _run_host(tpx, h[:0], 320, 20_000, 5_000, 64)
    assert len(cl) == 0
