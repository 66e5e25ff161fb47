"""Generates tests/golden/full_1m.json: the reference's own full
log-likelihood at N = 1,000,000 for BASELINE configs 3, 4 and 5, computed
once through oracle/_ref (the unmodified reference headers,
log_likelihood(catalog, params, make_partition(N, G), Precision::dbl),
engine.hpp:101-110).

    python tests/golden/make_golden_1m.py [--workers G] [--only NAME]

Cases (bench parameters, engine.hpp:272-273):
  bench_constant  benchmark_catalog(1e6, 42), Variant::constant   (config 3)
  bench_varying   benchmark_catalog(1e6, 42), Variant::varying    (config 4)
  county_varying  the same events with each density replaced by its county's:
                  60x60 square counties over [-5, 5]^2, densities log-uniform
                  on [1, 7.4e4] from std::mt19937_64(1) (ref_county_densities,
                  the draws of tools/cpp/cut_posterior_bench.cpp), county of an
                  event = the square containing it (config 5's catalog)

--grad instead writes tests/golden/full_1m_grad.json: per case the
double-precision checker's LL, gradient and conditioning scale sum_n |d
ell_n / d theta| (oracle/hawkes_oracle_dbl.c, compensated row sums; the
reference has no gradient), ~10-30 min per case on 8 threads.

Each LL case takes ~20-50 min on 8 host threads; the JSON is rewritten after every
case so an interrupted run keeps what it finished.  The catalog digests pin
the inputs (tests rebuild the catalogs with the product generator, itself
pinned bit-exact to the reference by test_oracle.py).
"""
import argparse
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import Oracle, Reference, county_index  # noqa: E402  (checker only)

OUT = ROOT / "tests" / "golden" / "full_1m.json"
OUT_GRAD = ROOT / "tests" / "golden" / "full_1m_grad.json"
N = 1_000_000
PARAMS = dict(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0)
GRID = 60


def digest(arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=64)
    ap.add_argument("--only", default=None)
    ap.add_argument("--grad", action="store_true")
    args = ap.parse_args()
    R = Reference()
    t, x, y, d = R.benchmark_catalog(N, 42)
    dens = R.county_densities(GRID, 1)
    county = (t, x, y, dens[county_index(x, y, GRID)])
    if args.grad:
        grad_cases(args, (t, x, y, d), county)
        return
    out = json.loads(OUT.read_text()) if OUT.exists() else {}
    out.update({"n": N, "seed": 42, "params": PARAMS, "grid": GRID, "county_seed": 1,
                "county_densities": dens.tolist(),
                "digest_bench": digest((t, x, y, d)), "digest_county": digest(county)})
    out.setdefault("cases", {})
    cases = [("bench_constant", (t, x, y, d), 0), ("bench_varying", (t, x, y, d), 1),
             ("county_varying", county, 1)]
    for name, cat, variant in cases:
        if args.only and name != args.only:
            continue
        if name in out["cases"]:
            continue
        t0 = time.perf_counter()
        ll = R.log_likelihood(cat, PARAMS, variant, workers=args.workers)
        sec = time.perf_counter() - t0
        out["cases"][name] = {"variant": variant, "loglik": ll, "workers": args.workers,
                              "seconds": sec, "host_threads": os.cpu_count()}
        OUT.write_text(json.dumps(out, indent=1) + "\n")
        print(f"{name}: {ll!r} ({sec:.0f} s)", flush=True)


def grad_cases(args, bench, county):
    out = json.loads(OUT_GRAD.read_text()) if OUT_GRAD.exists() else {}
    out.update({"n": N, "seed": 42, "params": PARAMS, "grid": GRID, "county_seed": 1,
                "checker": "oracle/hawkes_oracle_dbl.c orc_ll_grad_dbl (double, compensated row sums)",
                "digest_bench": digest(bench), "digest_county": digest(county)})
    out.setdefault("cases", {})
    O = Oracle()
    for name, cat, variant in [("bench_constant", bench, 0), ("bench_varying", bench, 1),
                               ("county_varying", county, 1)]:
        if (args.only and name != args.only) or name in out["cases"]:
            continue
        t0 = time.perf_counter()
        ll, g, sc = O.ll_grad_dbl(cat, PARAMS, variant, threads=args.workers)
        sec = time.perf_counter() - t0
        out["cases"][name] = {"variant": variant, "loglik": ll, "grad": g.tolist(), "grad_scale": sc.tolist(),
                              "threads": args.workers, "seconds": sec}
        OUT_GRAD.write_text(json.dumps(out, indent=1) + "\n")
        print(f"{name}: grad {g.tolist()} ({sec:.0f} s)", flush=True)


if __name__ == "__main__":
    main()
