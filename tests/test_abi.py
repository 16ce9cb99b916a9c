"""CPU-only checks of the C-ABI library: it loads, exports every symbol
include/*.h declares, and validates arguments without touching a GPU."""
import ctypes
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(tpx_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return sorted(names)


@pytest.fixture(scope="module")
def lib():
    from paper_2412_11809_b200 import build

    build.build()
    import paper_2412_11809_b200 as p

    return p


def test_header_declares_the_boundary():
    names = _declared_functions()
    for must in ("tpx_cluster_create", "tpx_cluster_run", "tpx_cluster_destroy", "tpx_cluster_workspace_bytes",
                 "tpx_cluster_run_host", "tpx_cluster_centroids"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    so = ctypes.CDLL(lib.LIB_PATH)
    missing = [n for n in _declared_functions() if not hasattr(so, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    for n in _declared_functions():
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_status_strings(lib):
    assert lib.ABI_VERSION == 1
    assert lib.status_string(0) == "ok"
    assert "capacity" in lib.status_string(-5)
    assert lib.status_string(12345) == "unknown status"
    assert lib.stage_name(0) == "sort" and lib.stage_name(1) == "tile_cc" and lib.stage_name(99) == ""


def test_create_validates_without_gpu(lib):
    c = lib.Clusterer(128)
    assert c.workspace_bytes(0) >= 256
    assert c.workspace_bytes(10**6) > 16 * 10**6
    c.close()
    for v in (1, 2):  # variants (iii)(b)/(c) are supported; their workspace is larger
        cv = lib.Clusterer(128, variant=v)
        assert cv.workspace_bytes(10**6) > lib.Clusterer(128).workspace_bytes(10**6)
        cv.close()
    for kw, code in ((dict(variant=7), -1), (dict(variant=-1), -1),
                     (dict(width=0), -1), (dict(height=70000), -1)):
        with pytest.raises(lib.TpxError) as e:
            lib.Clusterer(128, **kw)
        assert e.value.status == code
    with pytest.raises(lib.TpxError) as e:
        lib.Clusterer(1 << 48)
    assert e.value.status == -1


def test_tile_modes_validated_without_gpu(lib):
    """auto / sparse / dense / cell are accepted; TPX_TILE_COLUMN (3, round 1's
    column-bucket kernel, removed) and out-of-range modes are INVALID_ARG."""
    import ctypes
    c = lib.Clusterer(128)
    for m in ("auto", "sparse", "dense", "cell"):
        c.set_tile_mode(m)
    for raw in (3, 5, -1):
        assert lib._set_tile_mode(c._h, raw) == -1
    c.close()


def test_too_many_hits_rejected_before_any_cuda_call(lib):
    c = lib.Clusterer(128)
    with pytest.raises(lib.TpxError) as e:
        c.workspace_bytes(2**32 - 1)
    assert e.value.status == -4


def test_product_package_does_not_import_oracle():
    # the product path must never route through the test oracle
    for f in glob.glob(os.path.join(ROOT, "paper_2412_11809_b200", "**", "*.*"), recursive=True):
        if f.endswith((".py", ".cu", ".cuh", ".h")):
            src = open(f).read()
            assert "import oracle" not in src and "from oracle" not in src, f
            assert "tpx_oracle" not in src, f
