"""GPU: the bounds-checked build of the library (build.py --checked:
-DTPX_CHECKED turns every TPX_BOUND in the kernels into a device-side assert
-- shared-memory indices of the sort windows, cell index, pixel hash, member
and accumulator arrays, record slots, radix scatter positions) run through a
plain C caller of the C ABI (tests/native/abi_run.c, no PyTorch in the
process).  Every case must finish without an assert and its outputs must
still equal the oracle bit for bit.

This stands in for compute-sanitizer memcheck where the GPU pool has closed
the sanitizer (tests/test_gpu_sanitizer.py skips there): the cases are the
sanitizer's (configs[0], a small-sensor fuzz stream, the cell / dense
kernels, window-sort retry + radix fallback, the (iii)(b) variant) plus
larger samples of every preset in the sparse CSR kernel, including the
448x512 Timepix4 sensor (cell-grid wrap).
"""
import os
import subprocess

import numpy as np
import pytest

import oracle
import tpxgen

from tests import pins
from tests.test_gpu_sanitizer import CASES as SANITIZER_CASES

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = dict(SANITIZER_CASES)
CASES.update({
    # name: (hits factory, dt, W, H, tile_mode, variant)
    "mixed_csr": (lambda: tpxgen.generate("mixed", n_hits=2_000_000, seed=31), 320, 256, 256, 0, 0),
    "lowflux_csr": (lambda: tpxgen.generate("lowflux", n_hits=1_000_000, seed=32), 128, 256, 256, 0, 0),
    "heavyion_auto": (lambda: tpxgen.generate("heavyion", n_hits=1_000_000, seed=33), 64, 256, 256, 0, 0),
    "timepix4_csr": (lambda: tpxgen.generate("timepix4", n_hits=2_000_000, seed=34), 320, 448, 512, 0, 0),
    "variant_static": (lambda: tpxgen.generate("mixed", n_hits=200_000, seed=35), 320, 256, 256, 0, 2),
})


@pytest.fixture(scope="module")
def abi_run_checked(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_11809_b200 import build

    lib = build.build(checked=True)
    out = str(tmp_path_factory.mktemp("abi_checked") / "abi_run")
    cuda = "/usr/local/cuda"
    # -rpath to lib/checked/ only: the product library cannot be picked up
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"), "-I", f"{cuda}/include",
                           os.path.join(ROOT, "tests", "native", "abi_run.c"), "-L", os.path.dirname(lib),
                           "-ltpxcluster", "-L", f"{cuda}/lib64", "-lcudart",
                           f"-Wl,-rpath,{os.path.dirname(lib)}", "-Wl,--disable-new-dtags", "-o", out])
    return out


@pytest.mark.parametrize("case", list(CASES))
def test_checked_build_in_bounds(abi_run_checked, tmp_path, case):
    make, dt, W, H, mode, variant = CASES[case]
    h = make()
    hits = tmp_path / "hits.bin"
    h.tofile(hits)
    lab, ft = tmp_path / "labels.bin", tmp_path / "feats.bin"
    env = dict(os.environ)
    env.pop("LD_LIBRARY_PATH", None)
    r = subprocess.run([abi_run_checked, str(hits), str(dt), str(W), str(H), str(lab), str(ft), str(mode),
                        str(variant)], capture_output=True, text=True, timeout=600, env=env)
    log = r.stdout[-4000:] + r.stderr[-4000:]
    assert r.returncode == 0 and "abi_run ok" in r.stdout, log
    assert "Assertion" not in log, log
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


def test_checked_library_is_the_checked_build(abi_run_checked):
    """The runner resolves libtpxcluster.so to lib/checked/ (ldd), and that
    build carries the assert machinery (its kernels reference __assertfail)."""
    from paper_2412_11809_b200 import build

    ldd = subprocess.run(["ldd", abi_run_checked], capture_output=True, text=True).stdout
    line = [l for l in ldd.splitlines() if "libtpxcluster" in l]
    assert line and os.path.join("lib", "checked") in line[0], ldd
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.CHECKED_LIB], capture_output=True,
                          text=True).stdout
    assert "__assertfail" in sass or "CALL.ABS" in sass or "BPT.TRAP" in sass


def test_violated_bound_asserts(tmp_path):
    """Negative control: TPX_BOUND(5, 3) in a -DTPX_CHECKED kernel stops the
    launch with cudaErrorAssert and prints the failed condition."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = str(tmp_path / "bound_fail")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17",
                           "-DTPX_CHECKED", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "native", "bound_fail.cu"), "-o", exe])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    log = r.stdout + r.stderr
    assert r.returncode == 0 and "cudaErrorAssert" in log, log
    assert "Assertion" in log and "< (unsigned long long)" in log, log
