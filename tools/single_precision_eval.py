"""Times Precision::single (hk_eval_single) at N=1e6, bench catalog, both
variants, and its distance from the double result.  python tools/single_precision_eval.py"""
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2407_11349_b200 import Evaluator, HawkesParams, Variant, benchmark_catalog
cat = benchmark_catalog(1000000, 42)
ev = Evaluator(cat)
for v in (0, 1):
    p = HawkesParams(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0, variant=Variant(v))
    lld = ev.eval(p)
    ev.eval_single(p)
    ev.reset_profile(); ev.set_profiling(True)
    for _ in range(2): lls = ev.eval_single(p)
    ms, k, _ = ev.profile(); ev.set_profiling(False)
    print(f"single precision variant {v}: pair {ms / k:.1f} ms, |ll_single/ll_double - 1| = {abs(lls / lld - 1):.2e}", flush=True)
