"""Runs a few LL+gradient evaluations at one (N, variant) for ncu capture.

    python tools/profile_pair.py N VARIANT [EVALS]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_11349_b200 import Evaluator, HawkesParams, Variant, benchmark_catalog  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 0
evals = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cat = benchmark_catalog(n, 42)
ev = Evaluator(cat)
p = HawkesParams(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0, variant=Variant(variant))
ev.set_profiling(True)
t0 = time.perf_counter()
for _ in range(evals):
    ll, g = ev.eval(p, grad=True)
wall = (time.perf_counter() - t0) / evals
ms, npair, ntot = ev.profile()
print(f"N={n} variant={variant} ll={ll!r} grad={list(g)} wall/eval={wall*1e3:.3f} ms "
      f"pair_kernel/launch={ms/npair:.3f} ms pairs/s={n*(n-1)/(ms/npair*1e-3):.4e}")
