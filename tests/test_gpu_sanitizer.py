"""GPU: compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over
the C ABI, with a plain C caller (tests/native/abi_run.c: no PyTorch, so the
only kernels in the process are the library's).  Every case must report
0 errors, and its outputs must still equal the oracle bit for bit.

Cases: configs[0] (tiny), a small-sensor fuzz stream (many tile-border
merges), a mixed-stream sample in the cell kernel, a heavy-ion sample in the
dense kernel, a 600 us-disorder stream (window-sort retry + radix fallback)
and the (iii)(b) variant path.  SURVEY.md §4 / §8(c) (sanitizer runs on
configs[0] and fuzz cases).
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle
import tpxgen

from tests import pins

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SANITIZER = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
TOOLS = ["memcheck", "racecheck", "synccheck", "initcheck"]


@pytest.fixture(scope="module")
def abi_run(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(SANITIZER):
        pytest.skip("compute-sanitizer not found")
    from paper_2412_11809_b200 import build

    lib = build.build()
    out = str(tmp_path_factory.mktemp("abi") / "abi_run")
    cuda = "/usr/local/cuda"
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"), "-I", f"{cuda}/include",
                           os.path.join(ROOT, "tests", "native", "abi_run.c"), "-L", os.path.dirname(lib),
                           "-ltpxcluster", "-L", f"{cuda}/lib64", "-lcudart",
                           f"-Wl,-rpath,{os.path.dirname(lib)}", "-o", out])
    return out


def _fuzz_small_sensor():
    rng = np.random.default_rng(5)
    n = 6000
    return tpxgen.make_hits(list(zip(rng.integers(0, 8, n).tolist(), rng.integers(0, 8, n).tolist(),
                                     np.sort(rng.integers(0, 40_000, n)).tolist(), rng.integers(1, 30, n).tolist())))


CASES = {
    # name: (hits factory, dt, W, H, tile_mode, variant)
    "tiny": (lambda: tpxgen.generate("tiny"), 128, 256, 256, 0, 0),
    "fuzz8x8": (_fuzz_small_sensor, 200, 8, 8, 0, 0),
    "mixed_cell": (lambda: tpxgen.generate("mixed", n_hits=60_000, seed=21), 320, 256, 256, 1, 0),
    "heavyion_dense": (lambda: tpxgen.generate("heavyion", n_hits=40_000, seed=22), 64, 256, 256, 2, 0),
    "disorder_radix": (lambda: tpxgen.generate("mixed", n_hits=40_000, seed=23, disorder_ticks=384_000), 320, 256, 256, 0, 0),
    "variant_global": (lambda: tpxgen.generate("tiny", seed=24), 128, 256, 256, 0, 1),
}


@pytest.mark.slow
@pytest.mark.parametrize("tool", TOOLS)
@pytest.mark.parametrize("case", list(CASES))
def test_sanitizer_clean(abi_run, tmp_path, case, tool):
    make, dt, W, H, mode, variant = CASES[case]
    h = make()
    hits = tmp_path / "hits.bin"
    h.tofile(hits)
    lab, ft = tmp_path / "labels.bin", tmp_path / "feats.bin"
    cmd = [SANITIZER, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [abi_run, str(hits), str(dt), str(W), str(H), str(lab), str(ft), str(mode), str(variant)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    log = r.stdout[-4000:] + r.stderr[-4000:]
    if r.returncode == 86 and "closed" in log:
        # the GPU pool replaced compute-sanitizer by a stub that refuses to run
        # (exit 86); tests/test_gpu_checked.py covers the same cases with the
        # library's own bounds-checked build
        pytest.skip("compute-sanitizer is closed on this GPU pool: " + log.strip().splitlines()[-1][:160])
    assert r.returncode == 0, log
    if tool != "racecheck":  # racecheck prints its own summary line instead
        assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr, log
    else:
        assert "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in r.stdout + r.stderr, log
    got_l = np.fromfile(lab, dtype=np.uint32)
    got_f = np.fromfile(ft, dtype=oracle.FEAT_DTYPE)
    if variant:
        rl = oracle.cluster_streaming(h, dt, variant, W, H)
        assert np.array_equal(got_l, rl), case
        pins.assert_features_equal(got_f, pins.features_from_labels(h, rl), case)
    else:
        rl, rf = oracle.cluster(h, dt, W, H)
        assert np.array_equal(got_l, rl), case
        assert got_f.tobytes() == rf.tobytes(), case
