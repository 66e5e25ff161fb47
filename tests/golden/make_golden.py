"""Generates tests/golden/*.json from the reference's own CPU path.

Run here (where /root/reference exists and `make -C oracle ref` built
oracle/_ref/libhawkes_ref.so from the unmodified reference headers):

    python tests/golden/make_golden.py

Every value below is produced by the compiled reference through
oracle/ref_shim.cpp; nothing is computed by the product or the C oracle.
The GPU box has no /root/reference: the tests read these committed files.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import Reference  # noqa: E402

OUT = Path(__file__).resolve().parent
R = Reference()
PKEYS = ("mu0", "tau_t", "xi0", "sigma_x", "sigma_t", "area")


def pdict(v):
    return dict(zip(PKEYS, map(float, v)))


def digest(arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype="<f8").tobytes())
    return h.hexdigest()


def float_round(cat):
    """acceptance.cpp:60-65: t, lon, lat rounded through float."""
    t, x, y, d = cat
    return (t.astype(np.float32).astype(np.float64), x.astype(np.float32).astype(np.float64),
            y.astype(np.float32).astype(np.float64), d)


def bbox_area(x, y):
    """domain_area (geo.hpp:216-235) without override."""
    w = x.max() - x.min()
    h = y.max() - y.min()
    w = w if w > 0 else 2e-6
    h = h if h > 0 else 2e-6
    return float(w * h)


def kats():
    unit = pdict([1, 1, 1, 1, 1, 1])
    out = {
        "gaussian_pdf": {str(z): R.L.ref_gaussian_pdf(z) for z in (0.0, 1.0, 40.0)},
        "gaussian_cdf": {str(z): R.L.ref_gaussian_cdf(z) for z in (0.0, 1.0, -1.0, 1.3)},
        "pair_rate_forward": R.pair_rate(unit, 0, [0, 0, 0, 1], [1, 0, 0, 1]),
        "pair_rate_same": R.pair_rate(unit, 0, [0, 0, 0, 1], [0, 0, 0, 1]),
        "pair_rate_reverse": R.pair_rate(unit, 0, [1, 0, 0, 1], [0, 0, 0, 1]),
        "integral_unit_0_1": R.integral_term(unit, 0.0, 1.0),
        "integral_unit_0_0": R.integral_term(unit, 0.0, 0.0),
        "solo_clip": R.log_likelihood(([0.0], [0.0], [0.0], [1.0]), unit, 0, 1),
    }
    # far-separated catalog, test_model.cpp:185-193
    far = tuple(np.array(v, dtype=float) for v in (
        [i * 1e8 for i in range(4)], [i * 1e8 for i in range(4)], [-1e8 * i for i in range(4)], [1.0] * 4))
    out["far"] = {"catalog": [a.tolist() for a in far], "params": unit,
                  "event_contribution": [R.event_contribution(far, unit, 0, n) for n in range(4)],
                  "integral": [R.integral_term(unit, far[0][n], far[0][-1]) for n in range(4)],
                  "log_likelihood": R.log_likelihood(far, unit, 0, 1)}
    two = tuple(np.array(v, dtype=float) for v in ([0.0, 1.0], [0.0, 0.0], [0.0, 0.0], [1.0, 1.0]))
    out["two"] = {"catalog": [a.tolist() for a in two], "params": unit,
                  "event_contribution_1": R.event_contribution(two, unit, 0, 1)}
    return out


def catalogs_bench():
    """benchmark_catalog checksums (engine.hpp:251-259) for the generator test."""
    out = []
    for n, seed in ((1, 3), (1000, 42), (5000, 9000), (20000, 7), (100000, 42)):
        cat = R.benchmark_catalog(n, seed)
        out.append({"n": n, "seed": seed, "sha256": digest(cat),
                    "head": [[float(a[i]) for a in cat] for i in range(min(n, 3))]})
    return out


def acceptance1(count=24):
    """Criterion 1 (acceptance.cpp:50-84) style cases: benchmark_catalog(n,
    9000+c) rounded through float, random params (acceptance.cpp:33-45 ranges),
    area = domain_area; values from the reference's log_likelihood at
    G in {1,2,4,8} and from naive_log_likelihood."""
    rng = np.random.default_rng(101)
    cases = []
    for c in range(count):
        n = int(rng.integers(10, 5001)) if c >= 4 else [10, 255, 257, 1024][c]
        cat = float_round(R.benchmark_catalog(n, 9000 + c))
        variant = c % 2
        p = pdict([rng.uniform(0.1, 2.0), rng.uniform(0.5, 20.0), rng.uniform(0.05, 0.9),
                   rng.uniform(0.02, 0.5), rng.uniform(0.2, 10.0), bbox_area(cat[1], cat[2])])
        cases.append({
            "n": n, "seed": 9000 + c, "float_round": True, "variant": variant, "params": p,
            "sha256": digest(cat),
            "ll": {str(g): R.log_likelihood(cat, p, variant, g) for g in (1, 2, 4, 8)},
            "ll_single": R.log_likelihood(cat, p, variant, 1, single=True),
            "naive": R.naive_log_likelihood(cat, p, variant),
        })
        print(f"acceptance1 case {c}: n={n}", flush=True)
    return cases


def engine_catalogs():
    """test_engine.cpp:19-38 / test_model.cpp:35-52 style catalogs (numpy RNG,
    arrays stored) incl. tie-heavy and unit-density cases."""
    rng = np.random.default_rng(53)
    out = []
    specs = [(40, "model"), (120, "engine"), (300, "engine"), (257, "ties"), (200, "unit_density"),
             (600, "engine")]
    for k, (n, kind) in enumerate(specs):
        if kind == "model":
            t, x, y, d = rng.uniform(0, 50, n), rng.uniform(-3, 3, n), rng.uniform(-3, 3, n), rng.uniform(0.5, 2000, n)
        else:
            t, x, y, d = rng.uniform(0, 80, n), rng.uniform(-4, 4, n), rng.uniform(-4, 4, n), rng.uniform(0.5, 3000, n)
        if kind == "ties":
            t = np.round(t * 7.0) / 7.0  # times on 1/7-week days
        if kind == "unit_density":
            d = np.ones(n)
        o = np.argsort(t, kind="stable")
        t, x, y, d = t[o], x[o], y[o], d[o]
        for variant in (0, 1):
            p = pdict([0.05 + 2 * rng.uniform(), 0.5 + 10 * rng.uniform(), 0.05 + 1.5 * rng.uniform(),
                       0.05 + rng.uniform(), 0.2 + 5 * rng.uniform(), 10 + 100 * rng.uniform()])
            cat = (t, x, y, d)
            rows = list(range(0, n, max(1, n // 12)))
            out.append({
                "kind": kind, "n": n, "variant": variant, "params": p,
                "catalog": [a.tolist() for a in cat],
                "ll": {str(g): R.log_likelihood(cat, p, variant, g) for g in (1, 3, 8)},
                "naive": R.naive_log_likelihood(cat, p, variant),
                "rows": rows,
                "event_contribution": [R.event_contribution(cat, p, variant, r) for r in rows],
            })
    return out


def gradient_fd():
    """Richardson-extrapolated central differences of the reference's own
    log_likelihood (G=1): the only reference-derived pin for the gradient."""
    rng = np.random.default_rng(7)
    out = []
    for n, variant, kind in ((300, 0, "bench"), (300, 1, "bench"), (257, 0, "ties")):
        cat = R.benchmark_catalog(n, 500 + n + variant)
        if kind == "ties":
            cat = (np.round(cat[0] * 7) / 7, cat[1], cat[2], cat[3])
        p = np.array([rng.uniform(0.3, 1.5), rng.uniform(2, 10), rng.uniform(0.2, 0.8),
                      rng.uniform(0.1, 0.6), rng.uniform(0.5, 4), 100.0])
        f = lambda q: R.log_likelihood(cat, q, variant, 1)  # noqa: E731
        grad, err = [], []
        for k in range(5):
            def D(h):
                a, b = p.copy(), p.copy()
                a[k] += h
                b[k] -= h
                return (f(a) - f(b)) / (2 * h)
            h = 2e-3 * p[k]
            d1, d2, d3 = D(h), D(h / 2), D(h / 4)
            r1, r2 = (4 * d2 - d1) / 3, (4 * d3 - d2) / 3
            grad.append((16 * r2 - r1) / 15)
            err.append(abs(r2 - r1))
        out.append({"kind": kind, "n": n, "seed": 500 + n + variant, "variant": variant,
                    "params": pdict(p), "grad_fd": grad, "fd_err": err})
    return out


def workspace():
    """LikelihoodWorkspace<double> script (test_engine.cpp:159-190)."""
    rng = np.random.default_rng(59)
    n = 300
    t, x, y, d = rng.uniform(0, 80, n), rng.uniform(-4, 4, n), rng.uniform(-4, 4, n), rng.uniform(0.5, 3000, n)
    o = np.argsort(t, kind="stable")
    cat = tuple(a[o] for a in (t, x, y, d))
    p = np.array([1.1, 4.0, 0.6, 0.4, 1.5, 60.0])
    q = p.copy(); q[0] *= 1.7; q[2] *= 0.4
    r = q.copy(); r[1] *= 2.3
    s = q.copy(); s[3] *= 0.6; s[4] *= 1.9
    ops = [0, 1, 2, 1, 1, 2, 1, 2, 0]
    seq = [p, q, q, r, q, q, s, s, s]
    vals = R.workspace_script(cat, 0, 2, ops, seq)
    return {"catalog": [a.tolist() for a in cat], "ops": ops, "params": [pdict(v) for v in seq],
            "values": vals.tolist(), "log_likelihood": [R.log_likelihood(cat, v, 0, 2) for v in seq]}


def partitions():
    cases = [(10, 3), (8, 8), (1000000, 32), (5, 1), (4999, 7)]
    return [{"n": n, "g": g, "bounds": [int(b) for b in R.partition(n, g)]} for n, g in cases]


if __name__ == "__main__":
    (OUT / "kats.json").write_text(json.dumps(kats(), indent=1))
    (OUT / "benchmark_catalog.json").write_text(json.dumps(catalogs_bench(), indent=1))
    (OUT / "partition.json").write_text(json.dumps(partitions(), indent=1))
    (OUT / "workspace.json").write_text(json.dumps(workspace()))
    (OUT / "engine_catalogs.json").write_text(json.dumps(engine_catalogs()))
    (OUT / "gradient_fd.json").write_text(json.dumps(gradient_fd(), indent=1))
    (OUT / "acceptance1.json").write_text(json.dumps(acceptance1(), indent=1))
    print("golden vectors written to", OUT)
