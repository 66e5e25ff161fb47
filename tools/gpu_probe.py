"""Quick GPU probe: parity of the engine against the oracle on a few
catalogs, then timings at larger N.  Development aid (not a test)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle, Reference, ref_available  # noqa: E402
from paper_2407_11349_b200 import (Evaluator, HawkesParams, Variant,  # noqa: E402
                                   benchmark_catalog)

O = Oracle()
BENCH = dict(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0)


def parity(n, seed, v, p):
    cat = benchmark_catalog(n, seed)
    hp = HawkesParams(**p, variant=Variant(v))
    ev = Evaluator(cat)
    ll, g = ev.eval(hp, grad=True)
    ll_o, g_o = O.ll_grad(cat.arrays(), p, v)
    ell_abs, gs = O.grad_scale(cat.arrays(), p, v)
    print(f"n={n} v={v} ll={ll:.15g} oracle={ll_o:.15g} rel={abs(ll-ll_o)/abs(ll_o):.2e} "
          f"gerr={np.max(np.abs(g-g_o)/np.maximum(np.abs(g_o), gs)):.2e} g={g} go={g_o}", flush=True)


def timing(n, v, reps=3):
    cat = benchmark_catalog(n, 42)
    hp = HawkesParams(**BENCH, variant=Variant(v))
    ev = Evaluator(cat)
    ev.eval(hp, grad=True)
    ev.set_profiling(True)
    t0 = time.perf_counter()
    for _ in range(reps):
        ll, g = ev.eval(hp, grad=True)
    dt = (time.perf_counter() - t0) / reps
    ms, npair, ntot = ev.profile()
    pairs = n * (n - 1)
    print(f"N={n} v={v} wall/eval={dt*1e3:.2f} ms pair_kernel={ms/npair:.2f} ms "
          f"pairs/s={pairs/(ms/npair*1e-3):.3e} ll={ll:.15g}", flush=True)
    return ev, hp, cat


if __name__ == "__main__":
    import ctypes as C
    from paper_2407_11349_b200._lib import lib
    tf, ms = C.c_double(), C.c_double()
    lib.hk_measure_fp64_peak(0, C.byref(tf), C.byref(ms))
    print(f"fp64 peak {tf.value:.2f} TFLOP/s ({ms.value:.1f} ms)", flush=True)
    rng = np.random.default_rng(5)
    for c, n in enumerate([1, 2, 3, 17, 255, 256, 257, 600, 1000, 3000]):
        p = dict(mu0=rng.uniform(0.1, 2), tau_t=rng.uniform(0.5, 20), xi0=rng.uniform(0.05, 0.9),
                 sigma_x=rng.uniform(0.02, 0.5), sigma_t=rng.uniform(0.2, 10), area=100.0)
        parity(n, 100 + c, c % 2, p)
    parity(2000, 42, 0, BENCH)
    parity(2000, 42, 1, BENCH)
    for n in [10000, 100000]:
        for v in (0, 1):
            timing(n, v)
    ev, hp, cat = timing(1000000, 0, reps=2)
    rows = np.arange(0, 1000000, 1000000 // 64, dtype=np.uint64)[:64]
    ell_g = np.concatenate([ev.eval_rows(hp, int(r), int(r) + 1) for r in rows])
    ell_o = O.rows_ld(cat.arrays(), BENCH, 0, rows, grad=False)
    print("1M sampled rows max abs diff", np.max(np.abs(ell_g - ell_o)), flush=True)
    timing(1000000, 1, reps=2)
