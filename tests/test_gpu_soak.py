"""GPU soak: many seeded random workloads, each bit-exact against the oracle
(labels, every feature field, centroids).

The lock-free union-find of the tile kernels (tile_csr.cuh, tile_cc.cuh) and
the border merge (finalize.cuh) rely on benign races; a rare interleaving
bug would show up as an occasional label or feature mismatch, so this test
draws many different workloads instead of a few large ones.  Each case picks,
from its own seed, a cluster mix (dots / tracks / blobs), a hit rate (1 to
200 Mhit/s), a sensor (256x256, Timepix4's 448x512, or a small 8..64-pixel
one that forces dense windows and tile-border merges), dt_max (0 to 2000
ticks), readout disorder (0 to 20000 ticks) and a size (1 to 1.5M hits); the
tile configuration is the density probe's choice or forced.
"""
import numpy as np
import pytest

import tpxgen

from tests.test_gpu_parity import _assert_parity, tpx  # noqa: F401  (fixture)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N_CASES = 256


def _case(seed: int):
    r = np.random.default_rng(1000 + seed)
    kind = r.integers(0, 4)
    if kind == 0:
        mix = dict(frac_dot=1.0, frac_track=0.0, frac_blob=0.0)
    elif kind == 1:
        mix = dict(frac_dot=0.8, frac_track=0.2, frac_blob=0.0)
    elif kind == 2:
        mix = dict(frac_dot=0.0, frac_track=0.0, frac_blob=1.0, blob_min=int(r.integers(20, 200)),
                   blob_max=int(r.integers(300, 5000)))
    else:
        f = r.dirichlet([1, 1, 1])
        mix = dict(frac_dot=float(f[0]), frac_track=float(f[1]), frac_blob=float(f[2]), blob_max=2000)
    sensor = r.integers(0, 4)
    W, H = [(256, 256), (448, 512), (256, 256), (int(r.integers(8, 65)), int(r.integers(8, 65)))][sensor]
    n = int(r.choice([1, 7, 1000, 33_000, 250_000, 700_000, 1_500_000]))
    cfg = dict(width=W, height=H, rate_hz=float(10 ** r.uniform(6, np.log10(2e8))),
               disorder_ticks=int(r.choice([0, 640, 6400, 20_000])), seed=int(5000 + seed),
               dot_max=int(r.integers(2, 12)), track_max=int(r.integers(10, 1000)), **mix)
    dt = int(r.choice([0, 1, 16, 64, 128, 320, 2000]))
    mode = str(r.choice(["auto", "auto", "auto", "sparse", "dense", "cell"]))
    return n, cfg, dt, W, H, mode


@pytest.mark.parametrize("seed", range(N_CASES))
def test_soak_random_workloads(tpx, seed):  # noqa: F811
    n, cfg, dt, W, H, mode = _case(seed)
    h = tpxgen.generate("tiny", n_hits=n, **cfg)
    ctx = f"seed={seed} n={n} dt={dt} sensor={W}x{H} mode={mode} cfg={cfg}"
    _assert_parity(tpx, h, dt, W, H, ctx=ctx, tile_mode=mode)
