"""GPU parity: the B200 engine (through the C ABI) against the oracle and the
reference's golden vectors.  Gate: 1e-10 relative on the log-likelihood;
1e-10 on every gradient component relative to max(|g_ref|, sum_n |d ell_n/d
theta|) (the conditioning-aware scale of SURVEY.md section 7), with the
plain relative error reported alongside.  Integer/index work (catalog,
partitions, shard plans) is bit-exact and tested in test_oracle.py."""
import math

import numpy as np
import pytest

from conftest import float_round, golden, golden_catalog

pytestmark = pytest.mark.gpu

LL_TOL = 1e-10
GRAD_TOL = 1e-10
BENCH = dict(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0)  # engine.hpp:272-273


@pytest.fixture(scope="module")
def eng(cuda_device):
    import paper_2407_11349_b200 as eng
    return eng


def hp(eng, p, variant):
    return eng.HawkesParams(**{k: p[k] for k in ("mu0", "tau_t", "xi0", "sigma_x", "sigma_t", "area")},
                            variant=eng.Variant(variant))


def check_grad(g, g_ref, scale, tol=GRAD_TOL):
    """Conditioning-scaled gate (asserted) plus the plain relative error
    |g - g_ref| / |g_ref| per component (printed; `pytest -s` shows it)."""
    den = np.maximum(np.abs(g_ref), scale)
    diff = np.abs(g - g_ref)
    err = np.where(den > 0, diff / np.where(den > 0, den, 1.0), diff)  # 0/0: both exactly zero
    plain = np.where(g_ref != 0, diff / np.where(g_ref != 0, np.abs(g_ref), 1.0), diff)
    print(f"gradient rel err: scaled max {err.max():.2e}, plain {np.array2string(plain, precision=2)}")
    assert np.all(err <= tol), (err, g, g_ref)
    return err, plain


def run_vs_oracle(eng, oracle, cat, p, variant, grad=True):
    ev = eng.Evaluator(eng.Catalog(*cat))
    ll, g = ev.eval(hp(eng, p, variant), grad=True)
    ll_ref, g_ref = oracle.ll_grad(cat, p, variant)
    assert abs(ll - ll_ref) <= LL_TOL * abs(ll_ref), (ll, ll_ref)
    if grad:
        _, scale = oracle.grad_scale(cat, p, variant)
        check_grad(g, g_ref, scale)
    return ll, g


# ---- reference golden vectors ------------------------------------------------

@pytest.mark.parametrize("case", golden("acceptance1.json"), ids=lambda c: f"n{c['n']}v{c['variant']}")
def test_acceptance1_catalogs(eng, oracle, case):
    """acceptance.cpp:50-84 (criterion 1) catalogs: engine vs the reference's
    naive evaluator and its partitioned evaluator at G in {1,2,4,8}."""
    cat = golden_catalog(case)
    ll = eng.Evaluator(eng.Catalog(*cat)).eval(hp(eng, case["params"], case["variant"]))
    ref = case["naive"]
    assert abs(ll - ref) <= LL_TOL * abs(ref)
    for v in case["ll"].values():
        assert abs(ll - v) <= LL_TOL * abs(v)


@pytest.mark.parametrize("case", golden("acceptance1.json")[:10], ids=lambda c: f"n{c['n']}v{c['variant']}")
def test_acceptance1_gradient(eng, oracle, case):
    run_vs_oracle(eng, oracle, golden_catalog(case), case["params"], case["variant"])


@pytest.mark.parametrize("case", golden("engine_catalogs.json"), ids=lambda c: f"{c['kind']}{c['n']}v{c['variant']}")
def test_engine_catalogs(eng, oracle, case):
    """test_engine.cpp:127-141 / test_model.cpp:196-218 style catalogs incl.
    tie-heavy times: whole-catalog LL and per-row event_contribution."""
    cat = tuple(np.array(a) for a in case["catalog"])
    ev = eng.Evaluator(eng.Catalog(*cat))
    p = hp(eng, case["params"], case["variant"])
    ll = ev.eval(p)
    assert abs(ll - case["naive"]) <= LL_TOL * abs(case["naive"])
    for g, v in case["ll"].items():
        assert abs(ll - v) <= LL_TOL * abs(v)
    for r, want in zip(case["rows"], case["event_contribution"]):
        got = ev.eval_rows(p, r, r + 1)[0]
        assert abs(got - want) <= 1e-12 * max(1.0, abs(want))
    run_vs_oracle(eng, oracle, cat, case["params"], case["variant"])


@pytest.mark.parametrize("case", golden("gradient_fd.json"), ids=lambda c: f"{c['kind']}v{c['variant']}")
def test_gradient_vs_reference_fd(eng, oracle, case):
    cat = eng.benchmark_catalog(case["n"], case["seed"]).arrays()
    if case["kind"] == "ties":
        cat = (np.round(cat[0] * 7) / 7,) + tuple(cat[1:])
    _, g = eng.Evaluator(eng.Catalog(*cat)).eval(hp(eng, case["params"], case["variant"]), grad=True)
    _, scale = oracle.grad_scale(cat, case["params"], case["variant"])
    fd = np.array(case["grad_fd"])
    check_grad(g, fd, scale, tol=1e-9)  # FD-limited (fd_err ~ 1e-11 of scale)
    run_vs_oracle(eng, oracle, cat, case["params"], case["variant"])


def test_kats(eng):
    k = golden("kats.json")
    unit = eng.HawkesParams()
    solo = eng.Catalog([0.0], [0.0], [0.0])
    ll, g = eng.Evaluator(solo).eval(unit, grad=True)
    assert ll == pytest.approx(k["solo_clip"], rel=1e-12)  # test_engine.cpp:86-91
    assert g[2] == 0.0 and g[3] == 0.0  # clipped row: no rate-term derivative
    two = eng.Catalog(*k["two"]["catalog"])
    assert eng.event_contribution(unit, two, 1) == pytest.approx(k["two"]["event_contribution_1"], rel=1e-12)
    far = eng.Catalog(*k["far"]["catalog"])
    ev = eng.Evaluator(far)
    for n in range(4):  # the clip floor engages exactly (test_model.cpp:185-193)
        got = ev.eval_rows(unit, n, n + 1)[0]
        assert got == pytest.approx(k["far"]["event_contribution"][n], rel=1e-15)
    assert ev.eval(unit) == pytest.approx(k["far"]["log_likelihood"], rel=1e-14)


def test_workspace_semantics(eng):
    """LikelihoodWorkspace script of test_engine.cpp:159-190 against the
    reference workspace's own values."""
    w = golden("workspace.json")
    cat = eng.Catalog(*w["catalog"])
    ws = eng.LikelihoodWorkspace(cat, eng.Variant.constant, 2)
    for op, p, want in zip(w["ops"], w["params"], w["values"]):
        p = hp(eng, p, 0)
        if op == 0:
            got = ws.evaluate_full(p)
        elif op == 1:
            got = ws.evaluate_proposal(p)
        else:
            ws.commit_proposal()
            continue
        assert abs(got - want) <= LL_TOL * abs(want)


# ---- properties ------------------------------------------------------------------

def test_determinism_bitwise(eng):
    cat = eng.benchmark_catalog(6000, 47)
    ev = eng.Evaluator(cat)
    p = eng.HawkesParams(**BENCH, variant=eng.Variant.varying)
    a = ev.eval(p, grad=True)
    b = ev.eval(p, grad=True)
    c = eng.Evaluator(cat).eval(p, grad=True)
    assert a[0] == b[0] == c[0]
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[1], c[1])


def test_variant_collapse_bitwise(eng):
    """acceptance.cpp:325-344 (criterion 8): unit densities make the varying
    variant bitwise equal to the constant one."""
    rng = np.random.default_rng(808)
    for c in range(6):
        t, x, y, _ = eng.benchmark_catalog(int(rng.integers(10, 2000)), 7000 + c).arrays()
        cat = eng.Catalog(t, x, y, np.ones_like(t))
        ev = eng.Evaluator(cat)
        base = dict(mu0=rng.uniform(0.1, 2), tau_t=rng.uniform(0.5, 20), xi0=rng.uniform(0.05, 0.9),
                    sigma_x=rng.uniform(0.02, 0.5), sigma_t=rng.uniform(0.2, 10), area=100.0)
        a = ev.eval(eng.HawkesParams(**base, variant=eng.Variant.constant), grad=True)
        b = ev.eval(eng.HawkesParams(**base, variant=eng.Variant.varying), grad=True)
        assert a[0] == b[0] and np.array_equal(a[1], b[1])


def test_translation_invariance(eng, oracle):
    # test_model.cpp:249-262
    t, x, y, d = eng.benchmark_catalog(900, 37).arrays()
    p = eng.HawkesParams(mu0=0.7, tau_t=3.0, xi0=0.4, sigma_x=0.3, sigma_t=1.5, area=80.0)
    a = eng.Evaluator(eng.Catalog(t, x, y, d)).eval_rows(p, 0, 900)
    b = eng.Evaluator(eng.Catalog(t, x + 13.75, y - 4.5, d)).eval_rows(p, 0, 900)
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)


def test_row_sum_equals_total(eng):
    # test_engine.cpp:76-84 (single slice == sum of event contributions)
    cat = eng.benchmark_catalog(1200, 41)
    p = eng.HawkesParams(**BENCH)
    ev = eng.Evaluator(cat)
    ell, g = ev.eval_rows(p, 0, 1200, grad=True)
    ll, gt = ev.eval(p, grad=True)
    assert math.fsum(ell) == pytest.approx(ll, rel=1e-13)
    np.testing.assert_allclose(g.sum(axis=0), gt, rtol=1e-11, atol=1e-9)


def test_shards_sum_to_total(eng):
    """Row shards (the one-process-per-GPU path, here two contexts on one
    device) reduce, in rank order, to the single-context result."""
    cat = eng.benchmark_catalog(20000, 3)
    p = eng.HawkesParams(**BENCH, variant=eng.Variant.varying)
    full = eng.Evaluator(cat).eval(p, grad=True)
    for g in (2, 3, 8):
        b = eng.plan_shards(cat.t, g)
        parts = [eng.Evaluator(cat, shard=(int(b[i]), int(b[i + 1]))).eval(p, grad=True) for i in range(g)]
        ll = sum(x[0] for x in parts)
        gr = np.sum([x[1] for x in parts], axis=0)
        assert ll == pytest.approx(full[0], rel=1e-12)
        np.testing.assert_allclose(gr, full[1], rtol=1e-10, atol=1e-8)


def test_set_locations(eng, oracle):
    cat = eng.benchmark_catalog(3000, 11)
    ev = eng.Evaluator(cat)
    rng = np.random.default_rng(3)
    lon, lat = rng.uniform(-5, 5, 3000), rng.uniform(-5, 5, 3000)
    ev.set_locations(lon, lat)
    p = dict(BENCH)
    ll, g = ev.eval(hp(eng, p, 1), grad=True)
    ref, gref = oracle.ll_grad((cat.t, lon, lat, cat.density), p, 1)
    assert abs(ll - ref) <= LL_TOL * abs(ref)
    _, scale = oracle.grad_scale((cat.t, lon, lat, cat.density), p, 1)
    check_grad(g, gref, scale)


def test_errors(eng):
    cat = eng.benchmark_catalog(100, 1)
    ev = eng.Evaluator(cat)
    with pytest.raises(ValueError, match="sigma_t must be positive"):
        ev.eval(eng.HawkesParams(sigma_t=-1.0))
    with pytest.raises(IndexError):
        ev.eval_rows(eng.HawkesParams(), 50, 101)
    with pytest.raises(IndexError):
        eng.event_contribution(eng.HawkesParams(), cat, 100)
    with pytest.raises(ValueError, match="partition does not cover"):
        eng.log_likelihood(cat, eng.HawkesParams(), eng.Partition.make(99, 2))
    with pytest.raises(ValueError, match="double precision only"):
        eng.log_likelihood_and_gradient(cat, eng.HawkesParams(), None, eng.Precision.single)


def test_adversarial_finite(eng, oracle):
    """acceptance.cpp:86-113 / test_engine.cpp:143-157 catalogs (coincident
    events, widely separated events): finite and equal to the oracle."""
    n = 3000
    coincident = eng.Catalog(np.arange(n) * 0.01, np.full(n, 0.5), np.full(n, 0.5))
    p = dict(mu0=1.0, tau_t=1.0, xi0=1.0, sigma_x=1e-3, sigma_t=1.0, area=1.0)
    run_vs_oracle(eng, oracle, coincident.arrays(), p, 0)
    i = np.arange(n)
    sep = eng.Catalog(i * 10.0, np.where(i % 2, 1.0, -1.0) * 1e4, np.where(i % 3, 1.0, -1.0) * 1e4)
    run_vs_oracle(eng, oracle, sep.arrays(), p, 0)
    same = eng.Catalog(np.zeros(2000), np.zeros(2000), np.zeros(2000))  # all tied: every row clipped
    ll = eng.Evaluator(same).eval(eng.HawkesParams())
    assert ll == pytest.approx(oracle.ll_grad(same.arrays(), [1.0] * 6, 0)[0], rel=1e-12)


@pytest.mark.parametrize("window", ["8", "2"])
def test_adversarial_density_scaled_clustered(eng, oracle, monkeypatch, window):
    """The adversarial catalogs on the density-scaled kernel with the row
    clustering on: every location identical (zero extent: all cluster keys
    tie), locations 1e4 degrees apart (the quantised keys span a huge box),
    and all times tied; each against the oracle."""
    monkeypatch.setenv("HK_ROW_WINDOW", window)
    n = 12000
    rng = np.random.default_rng(5)
    d = np.exp(rng.uniform(0, 6, n))
    p = dict(mu0=1.0, tau_t=1.0, xi0=1.0, sigma_x=1e-3, sigma_t=1.0, area=1.0)
    coincident = eng.Catalog(np.arange(n) * 0.01, np.full(n, 0.5), np.full(n, 0.5), d)
    run_vs_oracle(eng, oracle, coincident.arrays(), p, 1)
    i = np.arange(n)
    sep = eng.Catalog(i * 0.01, np.where(i % 2, 1.0, -1.0) * 1e4 + rng.normal(0, 1e-3, n),
                      np.where(i % 3, 1.0, -1.0) * 1e4 + rng.normal(0, 1e-3, n), d)
    run_vs_oracle(eng, oracle, sep.arrays(), dict(p, sigma_x=0.5), 1)
    tied = eng.Catalog(np.zeros(n), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), d)
    ll = eng.Evaluator(tied).eval(hp(eng, p, 1))
    assert ll == pytest.approx(oracle.ll_grad(tied.arrays(), p, 1)[0], rel=1e-12)


def test_random_params_sweep(eng, oracle):
    """Random catalogs and parameters over the reference test ranges,
    including sizes around the 256-row/column tile edges."""
    rng = np.random.default_rng(2024)
    for c, n in enumerate([1, 2, 3, 31, 255, 256, 257, 511, 513, 1000, 2049, 4100]):
        cat = float_round(eng.benchmark_catalog(n, 300 + c).arrays())
        p = dict(mu0=rng.uniform(0.1, 2), tau_t=rng.uniform(0.5, 20), xi0=rng.uniform(0.05, 0.9),
                 sigma_x=rng.uniform(0.02, 0.5), sigma_t=rng.uniform(0.2, 10), area=100.0)
        for v in (0, 1):
            run_vs_oracle(eng, oracle, cat, p, v, grad=n > 1)


@pytest.mark.parametrize("variant", [0, 1])
def test_bench_config_100k_sampled_rows(eng, oracle, variant):
    """N=1e5 benchmark catalog: 512 sampled rows (value + gradient) against
    the long-double oracle, per row 1e-12."""
    cat = eng.benchmark_catalog(100000, 42)
    ev = eng.Evaluator(cat)
    p = hp(eng, BENCH, variant)
    rows = np.linspace(0, 99999, 512).astype(np.int64)
    res = [ev.eval_rows(p, int(r), int(r) + 1, grad=True) for r in rows]
    got = np.array([e[0][0] for e in res])
    gg = np.array([e[1][0] for e in res])
    want, gw = oracle.rows_ld(cat.arrays(), BENCH, variant, rows.astype(np.uint64))
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(gg, gw, rtol=1e-10, atol=1e-10 * np.abs(gw).max())


@pytest.mark.parametrize("variant", [0, 1])
def test_bench_config_100k_reference_full(eng, reference, variant):
    """N=1e5 (BASELINE config 2) full log-likelihood against the reference's
    own partitioned CPU evaluator (oracle/_ref) on all host threads (~4 s on
    16)."""
    import os
    cat = eng.benchmark_catalog(100000, 42)
    p = hp(eng, BENCH, variant)
    ll = eng.Evaluator(cat).eval(p)
    ref = reference.log_likelihood(cat.arrays(), BENCH, variant, workers=os.cpu_count())
    assert abs(ll - ref) <= LL_TOL * abs(ref)


def test_1m_sampled_rows(eng, oracle):
    """N=1e6 (BASELINE config): 1024 evenly spaced rows vs the oracle (SURVEY.md
    8c), plus the whole-catalog LL+grad is finite and deterministic."""
    cat = eng.benchmark_catalog(1000000, 42)
    ev = eng.Evaluator(cat)
    p = hp(eng, BENCH, 0)
    rows = np.linspace(0, 999999, 1024).astype(np.int64)
    got = np.array([ev.eval_rows(p, int(r), int(r) + 1)[0] for r in rows])
    want = oracle.rows_ld(cat.arrays(), BENCH, 0, rows.astype(np.uint64), grad=False)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
    # a contiguous window through the same path as the full evaluation
    win, gwin = ev.eval_rows(p, 500000, 500256, grad=True)
    wr = np.arange(500000, 500256, dtype=np.uint64)
    want_w, gw = oracle.rows_ld(cat.arrays(), BENCH, 0, wr)
    np.testing.assert_allclose(win, want_w, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(gwin, gw, rtol=1e-10, atol=1e-10 * np.abs(gw).max())
    a = ev.eval(p, grad=True)
    b = ev.eval(p, grad=True)
    assert np.isfinite(a[0]) and a[0] == b[0] and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("variant", [0, 1])
def test_bg_expansion_matches_direct(eng, variant):
    """The exact block expansion of the background (default) against the
    direct per-pair path on the same catalog: LL 1e-13, gradient 1e-12."""
    cat = eng.benchmark_catalog(100000, 42)
    p = hp(eng, BENCH, variant)
    ev = eng.Evaluator(cat)
    ev.set_bg_fgt(False)  # the background in the pair kernels (not the 1-D Hermite expansion)
    ll_x, g_x = ev.eval(p, grad=True)
    ev.set_bg_expansion(False)
    ll_d, g_d = ev.eval(p, grad=True)
    assert abs(ll_x - ll_d) <= 1e-13 * abs(ll_d)
    np.testing.assert_allclose(g_x, g_d, rtol=1e-12, atol=1e-12 * np.abs(g_d).max())


def test_row_windows_agree(eng, oracle, monkeypatch):
    """Density-scaled kernel: the spatially clustered row windows (default
    32 row blocks, HK_ROW_WINDOW) only reorder rows and widen the masked
    band, so windows of 1, 4 and 32 blocks agree to rounding, and each
    matches the long-double oracle; a window is bitwise deterministic.
    County-like catalog: densities log-uniform per 0.5-degree cell."""
    t, x, y, _ = eng.benchmark_catalog(20000, 9).arrays()
    rng = np.random.default_rng(3)
    dens = np.exp(rng.uniform(0, np.log(7.4e4), 400))
    cell = (np.minimum(np.floor((x + 5) / 0.5), 19) + 20 * np.minimum(np.floor((y + 5) / 0.5), 19)).astype(int)
    cat = eng.Catalog(t, x, y, dens[cell])
    p = dict(BENCH)
    out = {}
    for w in ("1", "4", "32"):
        monkeypatch.setenv("HK_ROW_WINDOW", w)
        ev = eng.Evaluator(cat)
        a = ev.eval(hp(eng, p, 1), grad=True)
        b = ev.eval(hp(eng, p, 1), grad=True)
        assert a[0] == b[0] and np.array_equal(a[1], b[1])
        out[w] = a
        ev.close()
    ll_o, g_o = oracle.ll_grad(cat.arrays(), p, 1)
    _, scale = oracle.grad_scale(cat.arrays(), p, 1)
    for w, (ll, g) in out.items():
        assert abs(ll - out["1"][0]) <= 1e-13 * abs(ll), w
        np.testing.assert_allclose(g, out["1"][1], rtol=1e-12, atol=1e-12 * np.abs(g).max())
        assert abs(ll - ll_o) <= LL_TOL * abs(ll_o)
        check_grad(g, g_o, scale)


@pytest.mark.parametrize("sigma_x,dens_max,origin", [
    (0.5, 1e8, (0.0, 0.0)),        # radii down to ~2e-3 degrees
    (0.02, 1e4, (-120.0, 36.0)),   # tiny lengthscale, far from the origin
    (3.0, 10.0, (150.0, -33.0)),   # every column wide
], ids=["extreme-density", "tiny-sigma-offset", "wide"])
def test_culling_regimes_vs_oracle(eng, oracle, sigma_x, dens_max, origin):
    """Density-scaled trigger culling (clustered rows, FP32 box test with the
    rounded-up thresholds): clustered catalogs (events in 40 hot spots) whose
    per-source reach spans 3+ orders of magnitude, against the long-double
    oracle, plus the window-1 (unclustered) path on the same catalog."""
    rng = np.random.default_rng(11)
    n = 12000
    t = np.sort(rng.uniform(0, 100, n))
    centres = rng.uniform(-5, 5, (40, 2))
    k = rng.integers(0, 40, n)
    x = origin[0] + centres[k, 0] + rng.normal(0, 0.3, n)
    y = origin[1] + centres[k, 1] + rng.normal(0, 0.3, n)
    d = np.exp(rng.uniform(0, np.log(dens_max), n))
    cat = eng.Catalog(t, x, y, d)
    p = dict(BENCH, sigma_x=sigma_x)
    ll, g = eng.Evaluator(cat).eval(hp(eng, p, 1), grad=True)
    ll_o, g_o = oracle.ll_grad(cat.arrays(), p, 1)
    assert abs(ll - ll_o) <= LL_TOL * abs(ll_o), (ll, ll_o)
    _, scale = oracle.grad_scale(cat.arrays(), p, 1)
    check_grad(g, g_o, scale)
    import os
    os.environ["HK_ROW_WINDOW"] = "1"
    try:
        ll1, g1 = eng.Evaluator(cat).eval(hp(eng, p, 1), grad=True)
    finally:
        del os.environ["HK_ROW_WINDOW"]
    assert abs(ll1 - ll) <= 1e-13 * abs(ll)
    np.testing.assert_allclose(g1, g, rtol=1e-12, atol=1e-12 * np.abs(g).max())


@pytest.mark.parametrize("variant", [0, 1])
def test_full_60k_vs_reference_and_oracle(eng, oracle, reference, variant):
    """N=6e4 (row blocks qualify for the background expansion): whole-catalog
    LL vs the reference's own partitioned evaluator, LL + gradient vs the
    long-double oracle."""
    import os
    cat = eng.benchmark_catalog(60000, 5)
    p = dict(BENCH)
    ll, g = eng.Evaluator(cat).eval(hp(eng, p, variant), grad=True)
    ref = reference.log_likelihood(cat.arrays(), p, variant, workers=os.cpu_count() or 1)
    assert abs(ll - ref) <= LL_TOL * abs(ref)
    ll_o, g_o = oracle.ll_grad(cat.arrays(), p, variant)
    assert abs(ll - ll_o) <= LL_TOL * abs(ll_o)
    _, scale = oracle.grad_scale(cat.arrays(), p, variant)
    check_grad(g, g_o, scale)


@pytest.mark.parametrize("variant", [0, 1])
def test_workspace_cache_bitwise_and_reuse(eng, variant):
    """Device-cached LikelihoodWorkspace (engine.hpp:117-229 semantics):
    every cached evaluation is bitwise equal to a fresh one, and only the
    halves whose parameters changed are recomputed."""
    cat = eng.benchmark_catalog(50000, 12)
    ev = eng.Evaluator(cat)
    base = eng.HawkesParams(**BENCH, variant=eng.Variant(variant))
    seq = [base,
           base.with_(mu0=1.7, xi0=0.3),          # recombine only
           base.with_(mu0=1.7, xi0=0.3, tau_t=7.0),   # background refresh
           base.with_(mu0=1.7, xi0=0.3),          # back to the cached state
           base.with_(sigma_x=0.4),               # trigger refresh
           base.with_(sigma_x=0.4, sigma_t=2.5)]  # trigger refresh
    fresh = [eng.Evaluator(cat).eval(p, grad=True) for p in seq]
    h0, m0 = ev.ws_stats()
    got = [ev.ws_eval(p, grad=True) for p in seq]
    for (a, ga), (b, gb) in zip(got, fresh):
        assert a == b and np.array_equal(ga, gb)
    h1, m1 = ev.ws_stats()
    assert (h1 - h0, m1 - m0) == (2, 4)  # seq[1] and seq[3] reuse both halves
    # locations drop the trigger cache only
    rng = np.random.default_rng(1)
    lon, lat = rng.uniform(-5, 5, len(cat)), rng.uniform(-5, 5, len(cat))
    ev.set_locations(lon, lat)
    a = ev.ws_eval(seq[4], grad=True)
    b = eng.Evaluator(eng.Catalog(cat.t, lon, lat, cat.density)).eval(seq[4], grad=True)
    assert a[0] == b[0] and np.array_equal(a[1], b[1])


def test_workspace_background_shared_across_variants(eng):
    """The background half depends on tau alone and both variants compute it
    with the same launch and plan, so a background cached by a homogeneous
    evaluation serves a density-scaled one bitwise."""
    cat = eng.benchmark_catalog(50000, 8)
    pc, pv = hp(eng, BENCH, 0), hp(eng, BENCH, 1)
    ev = eng.Evaluator(cat)
    ev.ws_eval(pc, grad=True)
    a = ev.ws_eval(pv, grad=True)  # background cached, trigger recomputed
    b = eng.Evaluator(cat).eval(pv, grad=True)
    assert a[0] == b[0] and np.array_equal(a[1], b[1])
    c = eng.Evaluator(cat).eval(pc, grad=True)
    d = ev.ws_eval(pc, grad=True)
    assert c[0] == d[0] and np.array_equal(c[1], d[1])


def test_workspace_golden_script_cached(eng):
    """The reference workspace script (test_engine.cpp:159-190) through the
    cached workspace."""
    w = golden("workspace.json")
    cat = eng.Catalog(*w["catalog"])
    ws = eng.LikelihoodWorkspace(cat, eng.Variant.constant, 2)
    for op, p, want in zip(w["ops"], w["params"], w["values"]):
        p = hp(eng, p, 0)
        if op == 2:
            ws.commit_proposal()
            continue
        got = ws.evaluate_full(p) if op == 0 else ws.evaluate_proposal(p)
        assert abs(got - want) <= LL_TOL * abs(want)
    assert ws.stats()[0] >= 2


# ---- Precision::single ----------------------------------

@pytest.mark.parametrize("case", golden("acceptance1.json"), ids=lambda c: f"n{c['n']}v{c['variant']}")
def test_single_precision_acceptance1(eng, case):
    """acceptance.cpp:50-84 single-precision gate: within 1e-4 of the naive
    double evaluator, and close to the reference's own float path."""
    cat = golden_catalog(case)
    ll = eng.log_likelihood(eng.Catalog(*cat), hp(eng, case["params"], case["variant"]),
                            eng.Partition.make(case["n"], 1), eng.Precision.single)
    assert abs(ll - case["naive"]) <= 1e-4 * abs(case["naive"])
    assert abs(ll - case["ll_single"]) <= 1e-4 * abs(case["naive"])


@pytest.mark.parametrize("variant", [0, 1])
def test_single_precision_large(eng, variant):
    """N=2e5 benchmark catalog: single vs double precision engine, 1e-5.
    From 131072 events Precision.single runs the FP64 expansion path
    (HK_OPT_SINGLE_FP64, default on): bitwise the double LL; with the option
    off the FP32 kernels, within 1e-5."""
    cat = eng.benchmark_catalog(200000, 9)
    ev = eng.Evaluator(cat)
    p = hp(eng, BENCH, variant)
    d = ev.eval(p)
    f = ev.eval_single(p)
    assert f == d
    ev.set_single_fp64(False)
    f32 = ev.eval_single(p)
    assert abs(f32 - d) <= 1e-5 * abs(d) and f32 != d
    assert ev.eval_single(p) == f32  # deterministic


def test_single_precision_adversarial_finite(eng):
    """acceptance.cpp:86-113 (criterion 2): 100k fully coincident and maximally
    separated catalogs stay finite in single precision."""
    n = 100000
    i = np.arange(n)
    coincident = eng.Catalog(np.zeros(n), np.zeros(n), np.zeros(n))
    corner = np.where(i % 2 == 0, -180.0, 180.0)
    separated = eng.Catalog(i * 0.1, corner, corner / 2.0)
    rng = np.random.default_rng(202)
    for cat in (coincident, separated):
        ev = eng.Evaluator(cat)
        for _ in range(3):
            p = eng.HawkesParams(mu0=rng.uniform(0.1, 2), tau_t=rng.uniform(0.5, 20), xi0=rng.uniform(0.05, 0.9),
                                 sigma_x=rng.uniform(0.02, 0.5), sigma_t=rng.uniform(0.2, 10), area=1.0)
            assert np.isfinite(ev.eval_single(p))


def test_coarse_catalog_needs_locations(eng):
    """A coarse-only catalog (NaN locations, types.hpp:43) is accepted at
    create; evaluation requires set_locations first (the cut posterior's X
    refresh), after which it matches a fine catalog."""
    import ctypes as C
    from paper_2407_11349_b200._lib import lib, check
    cat = eng.benchmark_catalog(2000, 4)
    t, x, y, d = cat.arrays()
    nan = np.full_like(x, np.nan)
    h = C.c_void_p()
    check(lib.hk_create(t, nan, nan, d, len(t), 1, C.byref(h)))
    try:
        p = eng.HawkesParams(**BENCH, variant=eng.Variant.varying).to_c()
        ll = C.c_double()
        assert lib.hk_eval(h, C.byref(p), C.byref(ll), None) == 1
        assert b"locations are not set" in lib.hk_last_error()
        check(lib.hk_set_locations(h, np.ascontiguousarray(x), np.ascontiguousarray(y)))
        check(lib.hk_eval(h, C.byref(p), C.byref(ll), None))
        want = eng.Evaluator(cat).eval(eng.HawkesParams(**BENCH, variant=eng.Variant.varying))
        assert ll.value == want
    finally:
        lib.hk_destroy(h)


def test_quadratic_scaling(eng):
    """acceptance.cpp:115-124 (criterion 3) on the GPU: the direct pair
    kernel's time grows quadratically with N (log-log slope in [1.7, 2.3])
    on the benchmark catalog, LL + gradient, constant kernel (the Hermite
    expansion off: it makes the trigger sub-quadratic, test_gpu_fgt.py)."""
    sizes = (100000, 200000, 400000)
    times = []
    p = eng.HawkesParams(**BENCH)
    for n in sizes:
        ev = eng.Evaluator(eng.benchmark_catalog(n, 42))
        ev.set_fgt(False)
        ev.eval(p, grad=True)
        ev.set_profiling(True)
        for _ in range(3):
            ev.eval(p, grad=True)
        ms, k, _ = ev.profile()
        times.append(ms / k)
    slope = np.polyfit(np.log(sizes), np.log(times), 1)[0]
    assert 1.7 <= slope <= 2.3, (sizes, times, slope)


@pytest.mark.parametrize("variant", [0, 1])
def test_workspace_single_cached(eng, variant):
    """LikelihoodWorkspace<float> (engine.hpp:117-229, Real = float): the
    cached single-precision workspace is bitwise equal to fresh
    Precision.single evaluations and reuses the unchanged half."""
    cat = eng.benchmark_catalog(50000, 21)
    base = eng.HawkesParams(**BENCH, variant=eng.Variant(variant))
    seq = [base, base.with_(mu0=1.4), base.with_(mu0=1.4, tau_t=6.0), base.with_(mu0=1.4),
           base.with_(sigma_x=0.45)]
    fresh = [eng.Evaluator(cat).eval_single(p) for p in seq]
    ws = eng.LikelihoodWorkspace(cat, eng.Variant(variant), 1, eng.Precision.single)
    got = [ws.evaluate_full(seq[0])] + [ws.evaluate_proposal(p) for p in seq[1:]]
    assert got == fresh
    h, m = ws.stats()
    assert (h, m) == (2, 3)  # seq[1] and seq[3] reuse both halves
    with pytest.raises(ValueError):
        ws.evaluate_proposal(base, grad=True)
    # the double workspace on the same context keeps separate entries
    d = eng.Evaluator(cat).eval(base)
    assert abs(d - fresh[0]) <= 1e-5 * abs(d) and d != fresh[0]


# ---- multi-device contexts (north_star data plane; one GPU here) -------------

@pytest.mark.parametrize("variant", [0, 1])
def test_multi_shard_context_on_one_gpu(eng, oracle, variant):
    """hk_create_devices({0, 0, 0, 0}): four cost-balanced row shards on one
    GPU, their 6-vectors gathered (peer copies) and summed on the device in
    shard order.  Equal to the single-shard context within 1e-12 (the shards
    chunk their columns differently), bitwise repeatable, per-row outputs
    concatenate in row order, and a location update reaches every shard."""
    cat = eng.benchmark_catalog(40000, 17)
    p = hp(eng, BENCH, variant)
    one = eng.Evaluator(cat)
    four = eng.Evaluator(cat, devices=[0, 0, 0, 0], plan_for=variant)
    assert four.rows() == (0, 40000, 4)
    a, ga = one.eval(p, grad=True)
    b, gb = four.eval(p, grad=True)
    assert abs(a - b) <= 1e-12 * abs(a)
    np.testing.assert_allclose(gb, ga, rtol=1e-11, atol=1e-11 * np.abs(ga).max())
    b2, gb2 = four.eval(p, grad=True)
    assert b2 == b and np.array_equal(gb2, gb)
    _, _, ell1, _ = one.eval_detail(p)
    _, _, ell4, _ = four.eval_detail(p)
    np.testing.assert_allclose(ell4, ell1, rtol=1e-12, atol=1e-12)
    # locations: copied to shard 0's buffers once, then peer-copied to the rest
    rng = np.random.default_rng(4)
    lon, lat = rng.uniform(-5, 5, 40000), rng.uniform(-5, 5, 40000)
    one.set_locations(lon, lat)
    four.set_locations(lon, lat)
    a, ga = one.eval(p, grad=True)
    b, gb = four.eval(p, grad=True)
    assert abs(a - b) <= 1e-12 * abs(a)
    # async form: the device-order total lands in the first device's buffer
    import torch
    from paper_2407_11349_b200.dist import _DeviceView
    four.eval_async(p, True)
    torch.cuda.synchronize()
    res = torch.as_tensor(_DeviceView(four.result_device_ptr(), 6), device="cuda").cpu()
    assert float(res[0]) == b and np.array_equal(res[1:].numpy(), gb)


def test_set_locations_rejects_non_finite_on_device(eng):
    """The device-side finiteness check of hk_set_locations reports the first
    non-finite event with the reference's Catalog message; the context then
    refuses to evaluate until valid locations arrive."""
    cat = eng.benchmark_catalog(5000, 2)
    ev = eng.Evaluator(cat)
    lon, lat = cat.lon.copy(), cat.lat.copy()
    lat[1234] = np.inf
    lon[4000] = np.nan
    with pytest.raises(ValueError, match="event 1234 has non-finite location"):
        ev.set_locations(lon, lat)
    with pytest.raises(ValueError, match="locations are not set"):
        ev.eval(eng.HawkesParams(**BENCH))
    ev.set_locations(cat.lon, cat.lat)
    assert ev.eval(eng.HawkesParams(**BENCH)) == eng.Evaluator(cat).eval(eng.HawkesParams(**BENCH))


def test_nccl_data_plane_one_device(eng, monkeypatch):
    """The C-ABI's NCCL data plane on one GPU (HK_FORCE_NCCL=1: a one-rank
    communicator): the 6-vector goes through ncclAllGather + the device-order
    sum, locations through ncclBroadcast; bitwise the plain context's result
    (libnccl.so.2 is dlopen'ed by the library, here torch's copy)."""
    import torch
    from paper_2407_11349_b200.dist import _DeviceView
    cat = eng.benchmark_catalog(30000, 23)
    p = hp(eng, BENCH, 1)
    plain = eng.Evaluator(cat)
    monkeypatch.setenv("HK_FORCE_NCCL", "1")
    ev = eng.Evaluator(cat, devices=[0], plan_for=1)
    a, b = plain.eval(p, grad=True), ev.eval(p, grad=True)
    assert a[0] == b[0] and np.array_equal(a[1], b[1])
    rng = np.random.default_rng(8)
    lon, lat = rng.uniform(-5, 5, 30000), rng.uniform(-5, 5, 30000)
    plain.set_locations(lon, lat)
    ev.set_locations(lon, lat)
    a, b = plain.eval(p, grad=True), ev.eval(p, grad=True)
    assert a[0] == b[0] and np.array_equal(a[1], b[1])
    ev.eval_async(p, True)
    torch.cuda.synchronize()
    res = torch.as_tensor(_DeviceView(ev.result_device_ptr(), 6), device="cuda").cpu()
    assert float(res[0]) == a[0]
