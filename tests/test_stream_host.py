"""Alg. "Hit buffer filling" (§4 l.184-213): the oracle transcription
pinned by a hand-worked example and the t-ordered separation property, and the
product's native implementation (tpx_buffill_assign, host-only) checked
against it hit by hit."""
import numpy as np
import pytest

import tpxgen
from oracle import buffill as ob


def _stream_disorder(h) -> int:
    """Smallest t for which the stream is t-ordered:
    toa(h_i) < toa(h_j) + t for all i < j."""
    toa = h["toa"].astype(np.int64)
    pref = np.maximum.accumulate(toa)
    return int(max(0, (pref[:-1] - toa[1:]).max(initial=0))) + 1


def test_buffill_hand_example():
    # b=4, b_t=1 (phase 1 while fewer than 3 hits), t=10, t_closing=2:
    # hits 0..2 fill phase 1 (toa_max 5), 3..6 go to nextBuffer (toa >= 7),
    # hit 6 (toa 30 > 5 + 12) sends buffer 0 with cut 7; the new buffer already
    # holds 4 hits, so hit 7 goes to nextBuffer and hit 8 sends buffer 1.
    h = tpxgen.make_hits([(0, 0, t, 1) for t in (0, 5, 3, 8, 9, 11, 30, 12, 40)])
    ids, cuts = ob.buffill(h, 4, 1, 10, 2)
    assert ids.tolist() == [0, 0, 0, 1, 1, 1, 1, 2, 2]
    assert cuts == [7, 7, ob.INF]


@pytest.mark.parametrize("b,b_t,t_closing", [(20_000, 3_000, 64), (5_000, 2_000, 0), (60_000, 500, 320)])
def test_buffill_separation_on_t_ordered_streams(b, b_t, t_closing):
    h = tpxgen.generate("mixed", n_hits=150_000)
    t = _stream_disorder(h)
    ids, cuts = ob.buffill(h, b, b_t, t, t_closing)
    assert len(cuts) >= 2 and cuts[-1] == ob.INF
    toa = h["toa"].astype(np.uint64)
    # every hit is sent exactly once, buffers in order; all hits after buffer k
    # (in later buffers) have toa >= cut_k (the property the carry relies on)
    for k, c in enumerate(cuts[:-1]):
        later = toa[ids > k]
        assert len(later) == 0 or int(later.min()) >= c, (k, c)
    sizes = np.bincount(ids)
    assert sizes.sum() == len(h) and (sizes > 0).all()


@pytest.mark.parametrize("preset,b,b_t,t_closing", [("mixed", 20_000, 3_000, 64), ("mixed", 3_000, 2_999, 0),
                                                     ("heavyion", 30_000, 10_000, 256), ("tiny", 1_000, 10, 5)])
def test_native_buffill_matches_oracle(preset, b, b_t, t_closing):
    from paper_2412_11809_b200 import build

    build.build()
    import paper_2412_11809_b200 as tpx

    h = tpxgen.generate(preset, n_hits=None if preset == "tiny" else 100_000)
    t = _stream_disorder(h)
    for tt in (t, 1, 10 * t):
        ids, cuts = tpx.buffill_assign(h, b, b_t, tt, t_closing)
        rid, rcuts = ob.buffill(h, b, b_t, tt, t_closing)
        assert np.array_equal(ids, rid) and cuts == rcuts
