"""Runs a few LL+gradient evaluations at one (N, variant) for ncu capture.

    python tools/profile_pair.py N VARIANT [EVALS] [county]

VARIANT 0 = homogeneous, 1 = density-scaled.  `county`: BASELINE config 5's
catalog instead (each event's density replaced by its 60x60 county's, the
densities of tests/golden/full_1m.json, log-uniform on [1, 7.4e4]).
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2407_11349_b200 import Catalog, Evaluator, HawkesParams, Variant, benchmark_catalog  # noqa: E402


def county_catalog(n):
    t, x, y, _ = benchmark_catalog(n, 42).arrays()
    dens = np.asarray(json.loads((ROOT / "tests" / "golden" / "full_1m.json").read_text())["county_densities"])
    cell = 10.0 / 60
    gx = np.minimum(((x + 5.0) / cell).astype(np.int64), 59)
    gy = np.minimum(((y + 5.0) / cell).astype(np.int64), 59)
    return Catalog(t, x, y, dens[gx + 60 * gy])


n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 0
evals = int(sys.argv[3]) if len(sys.argv) > 3 else 2
county = len(sys.argv) > 4 and sys.argv[4] == "county"
cat = county_catalog(n) if county else benchmark_catalog(n, 42)
ev = Evaluator(cat)
if os.environ.get("HK_CELLS") is not None:  # HK_OPT_CELLS on/off (comparisons)
    ev.set_cells(os.environ["HK_CELLS"] != "0")
p = HawkesParams(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0, variant=Variant(variant))
ev.eval(p, grad=True)
ev.set_profiling(True)
t0 = time.perf_counter()
for _ in range(evals):
    ll, g = ev.eval(p, grad=True)
wall = (time.perf_counter() - t0) / evals
ms, npair, ntot = ev.profile()
kms, kn = ev.profile_kinds()
kinds = " ".join(f"{name}={kms[i] / max(kn[i], 1):.3f}ms" for i, name in enumerate(("both", "bg", "trigger", "fgt_moments", "fgt_rows"))
                 if kn[i])
print(f"N={n} variant={variant}{' county' if county else ''} ll={ll!r} grad={list(g)} "
      f"wall/eval={wall*1e3:.3f} ms pair_kernel/launch={ms/npair:.3f} ms [{kinds}] "
      f"pairs/s={n*(n-1)/(ms/npair*1e-3):.4e}")
