"""tpxgen -- seeded synthetic Timepix3/Timepix4 hit streams.

Input infrastructure shared by the oracle tests, the CUDA-path tests,
``bench.py`` and ``__graft_entry__.smoke()``.  It draws hits only: none of the
clustering method's arithmetic lives here (see tpxgen.c's header).

The presets are the five BASELINE.json configs (the
size laws follow the dataset table, §5).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tpxgen.c")
_LIB = os.path.join(_HERE, "libtpxgen.so")

#: 16-byte hit record, the layout of ``tpx_hit`` (include/tpx_cluster.h).
HIT_DTYPE = np.dtype(
    [("toa", "<u8"), ("x", "<u2"), ("y", "<u2"), ("tot", "<u2"), ("reserved", "<u2")]
)
assert HIT_DTYPE.itemsize == 16

#: ns -> ToA ticks (1.5625 ns); exact for 100/200/500 ns (reading R4).
def ns_to_ticks(ns: float) -> int:
    return int(ns // 1.5625)


class _Cfg(ctypes.Structure):
    _fields_ = [
        ("n_hits", ctypes.c_uint64),
        ("width", ctypes.c_uint32),
        ("height", ctypes.c_uint32),
        ("rate_hz", ctypes.c_double),
        ("frac_dot", ctypes.c_double),
        ("frac_track", ctypes.c_double),
        ("frac_blob", ctypes.c_double),
        ("dot_min", ctypes.c_uint32),
        ("dot_max", ctypes.c_uint32),
        ("track_min", ctypes.c_uint32),
        ("track_max", ctypes.c_uint32),
        ("blob_min", ctypes.c_uint32),
        ("blob_max", ctypes.c_uint32),
        ("disorder_ticks", ctypes.c_uint64),
        ("toa_origin", ctypes.c_uint64),
        ("seed", ctypes.c_uint64),
        ("n_threads", ctypes.c_int32),
        ("pad", ctypes.c_int32),
    ]


_BASE = dict(
    width=256, height=256, rate_hz=1e6, frac_dot=1.0, frac_track=0.0, frac_blob=0.0,
    dot_min=1, dot_max=10, track_min=1, track_max=1000, blob_min=100, blob_max=5000,
    disorder_ticks=6400, toa_origin=0, seed=1, n_threads=0,
)

#: BASELINE.json configs[0..4] as concrete generator settings (+ dt_max in ticks).
PRESETS = {
    # configs[0]: 10k hits, X-ray dots 1-4 px, dt_max = 200 ns
    "tiny": dict(n_hits=10_000, rate_hz=1e6, dot_max=4, seed=1, dt_max=128),
    # configs[1]: 10M hits, mostly 1-10 px clusters, dt_max = 200 ns
    "lowflux": dict(n_hits=10_000_000, rate_hz=2e6, dot_max=10, seed=2, dt_max=128),
    # configs[2]: 200M hits at 40 Mhit/s, dots + MIP tracks, dt_max = 500 ns
    "mixed": dict(n_hits=200_000_000, rate_hz=40e6, frac_dot=0.8, frac_track=0.2,
                  dot_max=10, track_max=1000, seed=3, dt_max=320),
    # configs[3]: 50M hits, 100-5000 px blobs, dt_max = 100 ns (dense windows)
    "heavyion": dict(n_hits=50_000_000, rate_hz=40e6, frac_dot=0.0, frac_blob=1.0,
                     blob_min=100, blob_max=5000, seed=4, dt_max=64),
    # configs[4]: Timepix4 448x512, 2B hits at 5x rate, as mixed (dt: reading R17)
    "timepix4": dict(n_hits=2_000_000_000, width=448, height=512, rate_hz=200e6,
                     frac_dot=0.8, frac_track=0.2, dot_max=10, track_max=1000,
                     seed=5, dt_max=320),
}


def build(force: bool = False) -> str:
    """Compile libtpxgen.so with gcc (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.tpxgen_generate.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_void_p, ctypes.c_void_p]
        lib.tpxgen_generate.restype = ctypes.c_int
        lib.tpxgen_expected_cluster_size.argtypes = [ctypes.POINTER(_Cfg)]
        lib.tpxgen_expected_cluster_size.restype = ctypes.c_double
        _lib = lib
    return _lib


def config(preset: str = "tiny", **overrides) -> dict:
    """Merged generator settings for a preset (plus overrides)."""
    c = dict(_BASE)
    c.update(PRESETS[preset])
    c.update(overrides)
    return c


def _cstruct(c: dict) -> _Cfg:
    s = _Cfg()
    for name, _ in _Cfg._fields_:
        if name == "pad":
            continue
        setattr(s, name, c[name])
    return s


def expected_cluster_size(preset: str = "tiny", **overrides) -> float:
    c = config(preset, **overrides)
    c.setdefault("n_hits", 0)
    return _load().tpxgen_expected_cluster_size(ctypes.byref(_cstruct(c)))


def generate(preset: str = "tiny", n_hits: int | None = None, truth: bool = False,
             out: np.ndarray | None = None, **overrides):
    """Generate a seeded hit stream.

    Returns the hit array (``HIT_DTYPE``), or ``(hits, truth_ids)`` when
    ``truth`` is set.  ``out`` may be a preallocated ``HIT_DTYPE`` (or raw
    uint8 view of n*16 bytes) array, e.g. a pinned torch buffer's numpy view.
    """
    c = config(preset, **overrides)
    if n_hits is not None:
        c["n_hits"] = int(n_hits)
    n = int(c["n_hits"])
    if out is None:
        hits = np.zeros(n, dtype=HIT_DTYPE)
    else:
        hits = out
        assert hits.nbytes >= n * 16 and hits.flags["C_CONTIGUOUS"]
    tr = np.zeros(n, dtype=np.uint32) if truth else None
    rc = _load().tpxgen_generate(
        ctypes.byref(_cstruct(c)),
        hits.ctypes.data if n else None,
        tr.ctypes.data if (truth and n) else None,
    )
    if rc != 0:
        raise RuntimeError(f"tpxgen_generate failed: {rc}")
    return (hits, tr) if truth else hits


def make_hits(rows) -> np.ndarray:
    """Hits from (x, y, toa[, tot]) tuples (tot defaults to 1)."""
    rows = list(rows)
    h = np.zeros(len(rows), dtype=HIT_DTYPE)
    for i, r in enumerate(rows):
        h[i]["x"], h[i]["y"], h[i]["toa"] = r[0], r[1], r[2]
        h[i]["tot"] = r[3] if len(r) > 3 else 1
    return h


def random_small(rng: np.random.Generator, n: int, width: int, height: int,
                 toa_max: int) -> np.ndarray:
    """Uniform random hits on a small sensor (fuzzing input, no structure)."""
    h = np.zeros(n, dtype=HIT_DTYPE)
    h["x"] = rng.integers(0, width, n)
    h["y"] = rng.integers(0, height, n)
    h["toa"] = rng.integers(0, toa_max + 1, n)
    h["tot"] = rng.integers(1, 1024, n)
    return h
