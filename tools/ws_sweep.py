"""Times one MH sweep (mcmc.hpp:159-181: mu0, tau_t, xi0, sigma_x, sigma_t
proposals) through the device-cached workspace versus five full evaluations.

    python tools/ws_sweep.py [N] [VARIANT]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_11349_b200 import Evaluator, HawkesParams, LikelihoodWorkspace, Variant, benchmark_catalog  # noqa

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
v = Variant(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
cat = benchmark_catalog(n, 42)
p = HawkesParams(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0, variant=v)
ws = LikelihoodWorkspace(cat, v)
ws.evaluate_full(p)
names = ["mu0", "tau_t", "xi0", "sigma_x", "sigma_t"]


def sweep(cur, scale):
    t = []
    for k in names:
        prop = cur.with_(**{k: getattr(cur, k) * scale})
        t0 = time.perf_counter()
        ws.evaluate_proposal(prop)
        t.append(time.perf_counter() - t0)
        cur = prop  # accept every proposal (worst case for the cache)
        ws.commit_proposal()
    return cur, t


cur, _ = sweep(p, 1.01)
cur, t = sweep(cur, 0.99)
ev = Evaluator(cat)
t0 = time.perf_counter()
for _ in range(2):
    ev.eval(cur)
full = (time.perf_counter() - t0) / 2
print(f"N={n} variant={v.name}: workspace sweep {sum(t)*1e3:.1f} ms "
      f"({', '.join(f'{k} {x*1e3:.1f}' for k, x in zip(names, t))} ms) vs 5 full evals {5*full*1e3:.1f} ms "
      f"-> {5*full/sum(t):.2f}x; cache (hits, misses) = {ws.stats()}")
