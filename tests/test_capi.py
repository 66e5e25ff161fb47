"""CPU tests of the C ABI boundary: the library loads, exports exactly the
symbols include/hawkes_b200.h declares, and its host-only entry points behave
like the reference (no GPU is touched)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "hawkes_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("hk_create", "hk_create_shard", "hk_eval", "hk_eval_rows", "hk_set_locations",
              "hk_destroy", "hk_last_error", "hk_plan_shards", "hk_benchmark_catalog"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2407_11349_b200 import _lib
    exported = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                              text=True, check=True).stdout
    names = {ln.split()[-1] for ln in exported.splitlines() if ln.strip()}
    missing = [s for s in declared_symbols() if s not in names]
    assert not missing, missing
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert bound == set(declared_symbols())


def test_no_oracle_in_product():
    """The product library and package never reference the test oracle."""
    from paper_2407_11349_b200 import _lib
    deps = subprocess.run(["ldd", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "oracle" not in deps and "hawkes_ref" not in deps
    for f in (ROOT / "paper_2407_11349_b200").rglob("*.py"):
        assert "oracle" not in re.sub(r"#.*", "", f.read_text()).replace("oracle/", ""), f


def test_version_and_errors():
    from paper_2407_11349_b200._lib import lib, check
    assert b"sm_100a" in lib.hk_version()
    b = np.zeros(3, dtype=np.uintp)
    assert lib.hk_partition_make(5, 0, np.zeros(1, dtype=np.uintp)) == 1
    assert b"worker count must be positive" in lib.hk_last_error()
    with pytest.raises(ValueError, match="more workers than terms"):
        check(lib.hk_partition_make(1, 2, b))


def test_create_without_gpu_fails_cleanly():
    """On a host without a GPU hk_create reports a runtime error, never a crash
    or a silent CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2407_11349_b200 import Evaluator, benchmark_catalog
    from paper_2407_11349_b200._lib import CudaRuntimeError
    with pytest.raises(CudaRuntimeError):
        Evaluator(benchmark_catalog(10, 1))


def test_create_validates_before_touching_the_device():
    from paper_2407_11349_b200._lib import lib
    t = np.array([1.0, 0.5])
    z = np.zeros(2)
    h = C.c_void_p()
    rc = lib.hk_create(t, z, z, np.ones(2), 2, 1, C.byref(h))
    assert rc == 1 and b"times not sorted at index 1" in lib.hk_last_error()


def test_variant_entry_points_validate():
    """hk_plan_shards_variant / hk_create_variant: an unknown variant is an
    invalid_argument (before any device work); both variants plan valid,
    different shard boundaries."""
    from paper_2407_11349_b200._lib import lib
    from paper_2407_11349_b200 import benchmark_catalog
    t = benchmark_catalog(50000, 3).t
    b = np.zeros(5, dtype=np.uintp)
    assert lib.hk_plan_shards_variant(t, len(t), 4, 7, b) == 1
    assert b"unknown variant" in lib.hk_last_error()
    b0, b1 = np.zeros(5, dtype=np.uintp), np.zeros(5, dtype=np.uintp)
    assert lib.hk_plan_shards_variant(t, len(t), 4, 0, b0) == 0
    assert lib.hk_plan_shards_variant(t, len(t), 4, 1, b1) == 0
    for bb in (b0, b1):
        assert bb[0] == 0 and bb[-1] == len(t) and np.all(np.diff(bb.astype(np.int64)) > 0)
    assert not np.array_equal(b0, b1)
    b2 = np.zeros(5, dtype=np.uintp)
    assert lib.hk_plan_shards(t, len(t), 4, b2) == 0 and np.array_equal(b2, b0)
    z = np.zeros(2)
    h = C.c_void_p()
    assert lib.hk_create_variant(np.array([0.0, 1.0]), z, z, np.ones(2), 2, 1, 5, C.byref(h)) == 1
    assert b"unknown variant" in lib.hk_last_error()


def test_make_builds_sm100a():
    """The shared library carries sm_100a SASS (cross-compiled here)."""
    from paper_2407_11349_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # bulk-async (TMA-engine) tile staging
    assert "DFMA" in sass
