"""One LL+grad evaluation at large N (both variants) with the device memory
the context holds: python tools/big_n.py [N]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_11349_b200 as eng  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
cat = eng.benchmark_catalog(n, 42)
free0, total = torch.cuda.mem_get_info()
ev = eng.Evaluator(cat)
for v in (0, 1):
    p = eng.HawkesParams(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0, variant=eng.Variant(v))
    ll, g = ev.eval(p, grad=True)
    t0 = time.perf_counter()
    ll, g = ev.eval(p, grad=True)
    dt = time.perf_counter() - t0
    free1, _ = torch.cuda.mem_get_info()
    print(f"N={n} variant={v}: LL {ll!r} grad {g.tolist()} in {dt * 1e3:.1f} ms; "
          f"context device memory {(free0 - free1) / 2**30:.2f} GiB; fgt stats {ev.fgt_stats()}", flush=True)
