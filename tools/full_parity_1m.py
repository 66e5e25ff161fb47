"""Headline parity at the bench configuration: the full
N = 1e6 log-likelihood of benchmark_catalog(1e6, 42) from the B200 engine
against the reference's own partitioned CPU evaluator (oracle/_ref, all host
threads; ~25 min on 16 threads), plus the gradient on 256 evenly spaced
rows against the long-double oracle.  Writes one JSON line.

    python tools/full_parity_1m.py [N] [VARIANT]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle, Reference  # noqa: E402  (checker only)
from paper_2407_11349_b200 import Evaluator, HawkesParams, Variant, benchmark_catalog  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 0
P = dict(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0)
cat = benchmark_catalog(n, 42)
ev = Evaluator(cat)
hp = HawkesParams(**P, variant=Variant(variant))
ll, g = ev.eval(hp, grad=True)
threads = os.cpu_count() or 1
t0 = time.perf_counter()
ref = Reference().log_likelihood(cat.arrays(), P, variant, workers=threads)
ref_s = time.perf_counter() - t0
rows = np.linspace(0, n - 1, 256).astype(np.int64)
gr = np.array([ev.eval_rows(hp, int(r), int(r) + 1, grad=True)[1][0] for r in rows])
ell_o, gr_o = Oracle().rows_ld(cat.arrays(), P, variant, rows.astype(np.uint64), threads=threads)
ell_g = np.array([ev.eval_rows(hp, int(r), int(r) + 1)[0] for r in rows])
scale = np.maximum(np.abs(gr_o), np.abs(gr_o).max(axis=0))
print(json.dumps({
    "n": n, "variant": variant, "engine_loglik": ll, "reference_loglik": ref,
    "rel_err": abs(ll - ref) / abs(ref), "reference_seconds": ref_s, "reference_threads": threads,
    "engine_grad": list(map(float, g)),
    "rows_checked": len(rows),
    "row_ell_max_abs_err_vs_long_double": float(np.max(np.abs(ell_g - ell_o))),
    "row_grad_max_rel_err_vs_long_double": float(np.max(np.abs(gr - gr_o) / scale)),
}), flush=True)
