"""The certified Hermite expansions (hk_fgt.cu): the
homogeneous trigger's 2-D expansion (HK_OPT_FGT) and the background's 1-D
expansion in time (HK_OPT_BG_FGT), against the direct per-pair path of the
same engine and against the oracle: LL within 1e-13 relative, every
gradient component within 1e-12 of the conditioning scale; the expansion is
really used (hk_fgt_stats), a failed certification recomputes directly, and
cached workspace results stay bitwise equal to fresh ones."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BENCH = dict(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0)


@pytest.fixture(scope="module")
def eng(cuda_device):
    import paper_2407_11349_b200 as eng
    return eng


def both(eng, cat, p):
    ev = eng.Evaluator(cat)
    e0 = ev.fgt_stats()[0]
    a = ev.eval(p, grad=True)
    used = ev.fgt_stats()[0] - e0
    ev.set_fgt(False)
    b = ev.eval(p, grad=True)
    return a, b, used, ev


def close(a, b, tol_ll=1e-13, tol_g=1e-12):
    (la, ga), (lb, gb) = a, b
    assert abs(la - lb) <= tol_ll * abs(lb), (la, lb)
    np.testing.assert_allclose(ga, gb, rtol=tol_g, atol=tol_g * np.abs(gb).max())


@pytest.mark.parametrize("n", [100000, 300000])
def test_fgt_matches_direct_bench(eng, n):
    cat = eng.benchmark_catalog(n, 42)
    p = eng.HawkesParams(**BENCH)
    a, b, used, ev = both(eng, cat, p)
    assert used == 1
    close(a, b)
    assert ev.fgt_stats()[1] == 0  # no certification fallback


def test_fgt_random_params(eng, oracle):
    rng = np.random.default_rng(31)
    cat = eng.benchmark_catalog(120000, 7)
    used_total = 0
    for _ in range(6):
        p = eng.HawkesParams(mu0=rng.uniform(0.1, 2), tau_t=rng.uniform(0.5, 20), xi0=rng.uniform(0.05, 0.9),
                             sigma_x=rng.uniform(0.25, 3.0), sigma_t=rng.uniform(0.2, 10), area=100.0)
        a, b, used, _ = both(eng, cat, p)
        used_total += used
        close(a, b)
    assert used_total >= 4


def test_fgt_vs_oracle(eng, oracle):
    cat = eng.benchmark_catalog(60000, 5)
    p = dict(BENCH, sigma_x=1.0)
    ev = eng.Evaluator(cat)
    ll, g = ev.eval(eng.HawkesParams(**p), grad=True)
    assert ev.fgt_stats()[0] == 1
    ll_o, g_o = oracle.ll_grad(cat.arrays(), p, 0)
    _, scale = oracle.grad_scale(cat.arrays(), p, 0)
    assert abs(ll - ll_o) <= 1e-12 * abs(ll_o)
    assert np.all(np.abs(g - g_o) / np.maximum(np.abs(g_o), scale) <= 1e-11)


def test_fgt_clustered_and_tied(eng):
    """Hot-spot locations (boxes with thousands of sources next to empty
    ones), times on a 1/7-week grid (ties: the checkpoints' prefixes stop at
    tile boundaries, the tied band stays direct), coincident locations."""
    rng = np.random.default_rng(9)
    n = 150000
    t = np.sort(np.round(rng.uniform(0, 100, n) * 7) / 7)
    centres = rng.uniform(-5, 5, (30, 2))
    k = rng.integers(0, 30, n)
    x = centres[k, 0] + rng.normal(0, 0.2, n)
    y = centres[k, 1] + rng.normal(0, 0.2, n)
    p = eng.HawkesParams(**BENCH)
    a, b, used, _ = both(eng, eng.Catalog(t, x, y), p)
    assert used == 1
    close(a, b)
    tc = np.sort(rng.uniform(0, 100, 80000))
    same = eng.Catalog(tc, np.full(80000, 0.25), np.full(80000, -1.5))
    a, b, used, _ = both(eng, same, p)
    close(a, b)


def test_fgt_ll_only_and_workspace(eng):
    """LL-only evaluations and the cached workspace: the trigger cache is
    keyed by the expansion switch, and cached == fresh bitwise."""
    cat = eng.benchmark_catalog(100000, 12)
    base = eng.HawkesParams(**BENCH)
    ev = eng.Evaluator(cat)
    l1 = ev.eval(base)
    ev2 = eng.Evaluator(cat)
    ev2.set_fgt(False)
    assert abs(l1 - ev2.eval(base)) <= 1e-13 * abs(l1)
    seq = [base, base.with_(mu0=1.3), base.with_(tau_t=6.0), base.with_(sigma_x=0.6), base.with_(mu0=1.3)]
    fresh = [eng.Evaluator(cat).eval(p, grad=True) for p in seq]
    got = [ev.ws_eval(p, grad=True) for p in seq]
    for (x, gx), (y, gy) in zip(got, fresh):
        assert x == y and np.array_equal(gx, gy)
    ev.set_fgt(False)
    d = ev.ws_eval(seq[-1], grad=True)  # switch off: the trigger is recomputed directly
    assert abs(d[0] - got[-1][0]) <= 1e-13 * abs(d[0])


def test_fgt_certification_fallback(eng, monkeypatch):
    """A certification that cannot pass (HK_FGT_ROW_TOL=0) makes the
    synchronous evaluation recompute on the direct path: bitwise the
    direct result, counted as a fallback."""
    cat = eng.benchmark_catalog(80000, 3)
    p = eng.HawkesParams(**BENCH)
    direct = eng.Evaluator(cat)
    direct.set_fgt(False)
    direct.set_bg_fgt(False)  # the fallback recomputes without either expansion
    want = direct.eval(p, grad=True)
    monkeypatch.setenv("HK_FGT_ROW_TOL", "0")
    ev = eng.Evaluator(cat)
    got = ev.eval(p, grad=True)
    assert got[0] == want[0] and np.array_equal(got[1], want[1])
    e, f, _ = ev.fgt_stats()
    assert e == 1 and f == 1


def test_fgt_multi_shard(eng):
    cat = eng.benchmark_catalog(200000, 44)
    p = eng.HawkesParams(**BENCH)
    one = eng.Evaluator(cat).eval(p, grad=True)
    four = eng.Evaluator(cat, devices=[0, 0, 0], plan_for=0)
    got = four.eval(p, grad=True)
    assert four.fgt_stats()[0] == 1
    close(got, one, 1e-13, 1e-12)


def test_fgt_subquadratic(eng):
    """The expansion replaces the O(N^2) trigger: at N = 4e5 the whole
    evaluation is several times faster than the direct path."""
    cat = eng.benchmark_catalog(400000, 42)
    p = eng.HawkesParams(**BENCH)
    ev = eng.Evaluator(cat)
    ev.eval(p, grad=True)
    ev.set_profiling(True)
    ev.eval(p, grad=True)
    ms_f, _, _ = ev.profile()
    ev.reset_profile()
    ev.set_fgt(False)
    ev.eval(p, grad=True)
    ev.reset_profile()
    ev.eval(p, grad=True)
    ms_d, _, _ = ev.profile()
    print(f"N=4e5 LL+grad pair+expansion time: expansion {ms_f:.1f} ms, direct {ms_d:.1f} ms")
    assert ms_f < 0.5 * ms_d


def direct_ev(eng, cat):
    ev = eng.Evaluator(cat)
    ev.set_fgt(False)
    ev.set_bg_fgt(False)
    return ev


@pytest.mark.parametrize("variant", [0, 1])
def test_bg_fgt_matches_direct(eng, variant):
    """The background's 1-D expansion against the pair kernels' background
    (block expansion and per-pair), both variants, LL + gradient."""
    cat = eng.benchmark_catalog(200000, 42)
    p = eng.HawkesParams(**BENCH, variant=eng.Variant(variant))
    ev = eng.Evaluator(cat)
    ev.set_fgt(False)
    e0 = ev.fgt_stats()[0]
    a = ev.eval(p, grad=True)
    assert ev.fgt_stats()[0] == e0 + 1 and ev.fgt_stats()[1] == 0
    b = direct_ev(eng, cat).eval(p, grad=True)
    close(a, b)


@pytest.mark.parametrize("tau", [0.02, 0.7, 60.0])
def test_bg_fgt_tau_range_and_ties(eng, tau):
    """Short and long background lengthscales (thousands of time boxes / a
    single box) on a catalog with heavy time ties (ties: exactly 1 each is
    removed from the full sum)."""
    rng = np.random.default_rng(17)
    n = 60000
    t = np.sort(np.round(rng.uniform(0, 100, n) * 7) / 7)
    cat = eng.Catalog(t, rng.uniform(-5, 5, n), rng.uniform(-5, 5, n), rng.uniform(1, 100, n))
    for v in (0, 1):
        p = eng.HawkesParams(**dict(BENCH, tau_t=tau), variant=eng.Variant(v))
        a = eng.Evaluator(cat).eval(p, grad=True)
        b = direct_ev(eng, cat).eval(p, grad=True)
        close(a, b)


def test_bg_fgt_certification_on_sparse_catalogs(eng, oracle):
    """Catalogs whose background sums are tiny next to their tied/self terms
    (one event; events 10 lengthscales apart; every row clipped): the
    certification fails and the evaluation is recomputed directly, exact
    against the oracle."""
    p1 = dict(mu0=1.0, tau_t=1.0, xi0=1.0, sigma_x=1.0, sigma_t=1.0, area=1.0)
    for cat in (eng.Catalog([0.0], [0.0], [0.0]),
                eng.Catalog(np.arange(3000) * 10.0, np.zeros(3000), np.zeros(3000))):
        ev = eng.Evaluator(cat)
        ll, g = ev.eval(eng.HawkesParams(**p1), grad=True)
        ref = direct_ev(eng, cat).eval(eng.HawkesParams(**p1), grad=True)
        assert ll == ref[0] and np.array_equal(g, ref[1])
        assert ev.fgt_stats()[1] == 1  # recomputed on the direct path
        assert ll == pytest.approx(oracle.ll_grad(cat.arrays(), p1, 0)[0], rel=1e-12)


def county_like(eng, n, seed=3):
    t, x, y, _ = eng.benchmark_catalog(n, seed).arrays()
    rng = np.random.default_rng(seed)
    dens = np.exp(rng.uniform(0, np.log(7.4e4), 3600))
    cell = 10.0 / 60
    k = np.minimum(((x + 5) / cell).astype(int), 59) + 60 * np.minimum(((y + 5) / cell).astype(int), 59)
    return eng.Catalog(t, x, y, dens[k])


@pytest.mark.parametrize("kind", ["bench", "county"])
def test_tr_cut_matches_exact_threshold(eng, kind):
    """The density-scaled trigger's certified e^-46 spatial cut against the
    flush threshold (only exact zeros dropped): LL 1e-13, gradient 1e-12, no
    certification fallback on the BASELINE catalogs."""
    cat = eng.benchmark_catalog(200000, 42) if kind == "bench" else county_like(eng, 200000)
    p = eng.HawkesParams(**BENCH, variant=eng.Variant.varying)
    ev = eng.Evaluator(cat)
    a = ev.eval(p, grad=True)
    assert ev.fgt_stats()[1] == 0
    ev.set_tr_cut(False)
    b = ev.eval(p, grad=True)
    close(a, b)


def test_tr_cut_certification_fallback(eng, monkeypatch):
    cat = eng.benchmark_catalog(50000, 8)
    p = eng.HawkesParams(**BENCH, variant=eng.Variant.varying)
    ref = eng.Evaluator(cat)
    for f in (ref.set_fgt, ref.set_bg_fgt, ref.set_tr_cut):
        f(False)
    want = ref.eval(p, grad=True)
    monkeypatch.setenv("HK_FGT_ROW_TOL", "0")
    ev = eng.Evaluator(cat)
    got = ev.eval(p, grad=True)
    assert got[0] == want[0] and np.array_equal(got[1], want[1])
    assert ev.fgt_stats()[1] == 1


@pytest.mark.parametrize("gc", [None, "1", "3", "8"])
@pytest.mark.parametrize("kind", ["bench", "county"])
def test_cells_match_time_order(eng, monkeypatch, kind, gc):
    """The density-scaled FP64 trigger over spatial cell tiles (hk_cells.cu,
    HK_OPT_CELLS) against the time-ordered tiles: the same pairs in another
    summation order, LL 1e-13, gradient 1e-12, for the default grid and
    forced ones (one cell; a grid that is not a power of two; 8 x 8 on a
    small catalog: many partial tiles)."""
    if gc is not None:
        monkeypatch.setenv("HK_CELL_GC", gc)
    cat = eng.benchmark_catalog(120000, 5) if kind == "bench" else county_like(eng, 120000, seed=4)
    p = eng.HawkesParams(**BENCH, variant=eng.Variant.varying)
    ev = eng.Evaluator(cat)
    a = ev.eval(p, grad=True)
    ev.set_cells(False)
    b = ev.eval(p, grad=True)
    close(a, b)
    ev.set_cells(True)  # the cache keys the layout: back to bitwise the first result
    c = ev.eval(p, grad=True)
    assert c[0] == a[0] and np.array_equal(c[1], a[1])


def test_cells_degenerate_and_clustered(eng, monkeypatch):
    """Every event at one location (an empty grid box: one cell holds all),
    and a catalog whose events sit on a few points with tied times."""
    monkeypatch.setenv("HK_CELL_GC", "8")
    rng = np.random.default_rng(11)
    n = 40000
    t = np.sort(rng.uniform(0, 2000, n))
    t[1000:1010] = t[1000]
    pts = rng.uniform(-5, 5, (7, 2))
    k = rng.integers(0, 7, n)
    p = eng.HawkesParams(**BENCH, variant=eng.Variant.varying)
    for cat in (eng.Catalog(t, np.zeros(n), np.zeros(n), np.full(n, 3.0)),
                eng.Catalog(t, pts[k, 0], pts[k, 1], np.exp(rng.uniform(0, 8, n)))):
        ev = eng.Evaluator(cat)
        a = ev.eval(p, grad=True)
        ev.set_cells(False)
        close(a, ev.eval(p, grad=True))


@pytest.mark.parametrize("n", [100000, 300000])
def test_fgt_adaptive_truncation_matches_full_square(eng, monkeypatch, n):
    """The per-box truncation (two rectangles chosen by the warp's nearest
    row, hk_fgt.cu fgt_truncation_table) against the full 30 x 30 square
    everywhere (HK_FGT_FULL_SQUARE): both within the same certified bound,
    LL 1e-13, gradient 1e-12."""
    cat = eng.benchmark_catalog(n, 17)
    p = eng.HawkesParams(**BENCH, variant=eng.Variant.constant)
    ev = eng.Evaluator(cat)
    a = ev.eval(p, grad=True)
    assert ev.fgt_stats() == (1, 0, 0)
    monkeypatch.setenv("HK_FGT_FULL_SQUARE", "1")
    full = eng.Evaluator(cat)
    b = full.eval(p, grad=True)
    assert full.fgt_stats()[:2] == (1, 0)
    close(a, b)


@pytest.mark.parametrize("kind", ["bench", "county"])
def test_cells_reach_classes(eng, monkeypatch, kind):
    """Cells split into log-density reach classes (HK_CELL_CLASSES; the
    default at N >= 9e5 is two): the same sums as the time-ordered tiles."""
    monkeypatch.setenv("HK_CELL_GC", "8")
    monkeypatch.setenv("HK_CELL_CLASSES", "3")
    cat = eng.benchmark_catalog(120000, 6) if kind == "bench" else county_like(eng, 120000, seed=7)
    p = eng.HawkesParams(**BENCH, variant=eng.Variant.varying)
    ev = eng.Evaluator(cat)
    a = ev.eval(p, grad=True)
    ev.set_cells(False)
    close(a, ev.eval(p, grad=True))
