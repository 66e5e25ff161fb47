"""Small evaluations of every launch path, for compute-sanitizer runs
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_11349_b200 as eng  # noqa: E402

cat = eng.benchmark_catalog(150000, 42)
p = dict(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0)
for v in (0, 1):
    ev = eng.Evaluator(cat)
    hp = eng.HawkesParams(**p, variant=eng.Variant(v))
    print(v, ev.eval(hp, grad=True)[0], ev.eval(hp), ev.eval_single(hp))
    print(v, ev.ws_eval(hp.with_(tau_t=6.0), grad=True)[0], ev.ws_eval(hp.with_(sigma_x=0.6), grad=True)[0])
    ev.eval_detail(hp)
    ev.eval_rows(hp, 1000, 1300, grad=True)
four = eng.Evaluator(cat, devices=[0, 0, 0], plan_for=1)
print(four.eval(eng.HawkesParams(**p, variant=eng.Variant.varying), grad=True)[0])
cell = 10.0 / 60
k = (np.minimum(((cat.lon + 5) / cell).astype(int), 59) + 60 * np.minimum(((cat.lat + 5) / cell).astype(int), 59))
regions = []
for gy in range(60):
    for gx in range(60):
        x0, y0 = -5 + gx * cell, -5 + gy * cell
        regions.append(eng.Region(f"c{gy * 60 + gx}", polygons=[[np.array([[x0, y0], [x0 + cell, y0],
                                                                            [x0 + cell, y0 + cell], [x0, y0 + cell]])]]))
R = eng.Regions(regions, k.astype(np.int32))
ev = eng.Evaluator(cat)
ev.resample_locations(R, 3, 1)
print(ev.eval(eng.HawkesParams(**p, variant=eng.Variant.varying), grad=True)[0])
print("sanitize run done")
