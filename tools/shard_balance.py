"""Load balance of the row shards: evaluates each of g
cost-balanced shards of benchmark_catalog(N, 42) as its own context on the
one available GPU and reports per-shard pair-kernel times, max/mean, and the
projected g-GPU evaluation time (max shard + measured 6-double reduction
estimate).  Projection, not a multi-GPU measurement.

    python tools/shard_balance.py [N] [VARIANT]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_11349_b200 import Evaluator, HawkesParams, Variant, benchmark_catalog, plan_shards  # noqa

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
v = Variant(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
cat = benchmark_catalog(n, 42)
p = HawkesParams(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0, variant=v)


def shard_ms(b, e, reps=5):
    """Median pair-kernel time of `reps` evaluations of rows [b, e) after
    one warm-up evaluation."""
    ev = Evaluator(cat, shard=(int(b), int(e)))
    ev.eval(p, grad=True)
    t = []
    for _ in range(reps):
        ev.reset_profile()
        ev.set_profiling(True)
        ev.eval(p, grad=True)
        ms, k, _ = ev.profile()
        ev.set_profiling(False)
        t.append(ms / k)
    ev.close()
    return float(np.median(t))


shard_ms(0, n, reps=3)  # clocks up before anything is timed
full = shard_ms(0, n)
print(f"N={n} variant={v.name}: 1 GPU {full:.1f} ms")
for g in (2, 4, 8):
    bounds = plan_shards(cat.t, g, v)
    ms = np.array([shard_ms(bounds[k], bounds[k + 1]) for k in range(g)])
    print(f"g={g}: shard ms {np.round(ms, 1).tolist()}  max/mean {ms.max() / ms.mean():.3f}  "
          f"sum {ms.sum():.1f} ms ({ms.sum() / full:.3f} of 1 GPU)  projected {g}-GPU {ms.max():.1f} ms "
          f"-> {1000.0 / ms.max():.2f} evals/s (speed-up {full / ms.max():.2f}x)")
