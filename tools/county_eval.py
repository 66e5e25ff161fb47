"""Times a density-scaled LL+grad evaluation on a config-5-like catalog:
benchmark_catalog(N, 42) with each event's density replaced by its county's
(60x60 square counties over [-5,5]^2, densities log-uniform on [1, 7.4e4])."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_11349_b200 import Catalog, Evaluator, HawkesParams, Variant, benchmark_catalog  # noqa

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
t, x, y, _ = benchmark_catalog(n, 42).arrays()
rng = np.random.default_rng(1)
dens = np.exp(rng.uniform(0, np.log(7.4e4), 3600))
g = np.minimum((np.floor((x + 5) / (10 / 60))).astype(int), 59) + 60 * np.minimum((np.floor((y + 5) / (10 / 60))).astype(int), 59)
ev = Evaluator(Catalog(t, x, y, dens[g]))
p = HawkesParams(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0, variant=Variant.varying)
ev.eval(p, grad=True)
ev.set_profiling(True)
for _ in range(2):
    ev.eval(p, grad=True)
ms, k, _ = ev.profile()
print(f"county catalog N={n}: pair kernel {ms / k:.1f} ms / LL+grad")
