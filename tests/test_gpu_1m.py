"""N = 1,000,000 parity of the PRODUCTION plan (BASELINE configs 3, 4 and 5).

hk_eval_detail runs exactly the launches hk_eval runs by default (homogeneous:
512-row items with the background block expansion; density-scaled: the
clustered 64-block row windows, the split background-only launch plus the
compact trigger-only launch) and also returns each row's ell_n and
d ell_n / d theta from those launches.  Against:
  * the reference's own full log-likelihood, computed once through oracle/_ref
    (the unmodified reference headers, log_likelihood(..., Precision::dbl),
    engine.hpp:101-110) by tests/golden/make_golden_1m.py -> full_1m.json;
  * the double-precision gradient checker (oracle/hawkes_oracle_dbl.c,
    compensated row sums; the reference has no gradient) -> full_1m_grad.json;
  * the long-double oracle on 1,024 sampled rows per catalog (ell_n 1e-12,
    row gradient 1e-10).
Catalogs: benchmark_catalog(1e6, 42) in both variants, and config 5's county
catalog (the same events, each density replaced by its 60x60 county's,
log-uniform on [1, 7.4e4]).  Gates (north_star): LL 1e-10 relative; every
gradient component 1e-10 relative to max(|g|, sum_n |d ell_n / d theta|)
(the conditioning scale), with the plain relative error
|g - g_ref| / |g_ref| reported (and bounded by 1e-9).
"""
import hashlib
import math

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

N = 1_000_000
LL_TOL = 1e-10
GRAD_TOL = 1e-10
PLAIN_GRAD_TOL = 1e-9
CASES = ["bench_constant", "bench_varying", "county_varying"]


def digest(arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def goldens():
    return golden("full_1m.json"), golden("full_1m_grad.json")


@pytest.fixture(scope="module")
def catalogs(cuda_device, goldens):
    import paper_2407_11349_b200 as eng
    from oracle.oracle import county_index
    g, gg = goldens
    t, x, y, d = eng.benchmark_catalog(N, 42).arrays()
    assert digest((t, x, y, d)) == g["digest_bench"] == gg["digest_bench"]
    dens = np.asarray(g["county_densities"])
    county = (t, x, y, dens[county_index(x, y, g["grid"])])
    assert digest(county) == g["digest_county"] == gg["digest_county"]
    return {"bench": (t, x, y, d), "county": county}


@pytest.fixture(scope="module")
def results(catalogs, goldens):
    """One production evaluation per case (shared by the tests below)."""
    import paper_2407_11349_b200 as eng
    g, _ = goldens
    out = {}
    evs = {k: eng.Evaluator(eng.Catalog(*v)) for k, v in catalogs.items()}
    for name in CASES:
        case = g["cases"][name]
        cat_key = "county" if name.startswith("county") else "bench"
        p = eng.HawkesParams(**g["params"], variant=eng.Variant(case["variant"]))
        ll, gr, ell, grows = evs[cat_key].eval_detail(p, grad=True)
        out[name] = dict(ll=ll, grad=gr, ell=ell, grows=grows, cat=catalogs[cat_key], variant=case["variant"],
                         params=g["params"])
    for ev in evs.values():
        ev.close()
    return out


@pytest.mark.parametrize("name", CASES)
def test_1m_loglik_vs_reference(results, goldens, name):
    r = results[name]
    ref = goldens[0]["cases"][name]["loglik"]
    assert abs(r["ll"] - ref) <= LL_TOL * abs(ref), (r["ll"], ref)


@pytest.mark.parametrize("name", CASES)
def test_1m_gradient_vs_checker(results, goldens, name, record_property):
    r = results[name]
    case = goldens[1]["cases"][name]
    g_ref, scale = np.array(case["grad"]), np.array(case["grad_scale"])
    # the checker's own LL agrees with the reference's
    ref = goldens[0]["cases"][name]["loglik"]
    assert abs(case["loglik"] - ref) <= 1e-12 * abs(ref)
    diff = np.abs(r["grad"] - g_ref)
    scaled = diff / np.maximum(np.abs(g_ref), scale)
    plain = diff / np.abs(g_ref)
    record_property("grad_rel_err_scaled", scaled.tolist())
    record_property("grad_rel_err_plain", plain.tolist())
    print(f"{name}: gradient rel err scaled {scaled.max():.2e}, plain per component {plain.tolist()}")
    assert np.all(scaled <= GRAD_TOL), (scaled, r["grad"], g_ref)
    assert np.all(plain <= PLAIN_GRAD_TOL), (plain, r["grad"], g_ref)


@pytest.mark.parametrize("name", CASES)
def test_1m_rows_vs_long_double(results, oracle, name):
    """1,024 rows of the production launches (evenly spaced plus random)
    against the long-double oracle."""
    r = results[name]
    rng = np.random.default_rng(1)
    rows = np.unique(np.concatenate([np.linspace(0, N - 1, 512).astype(np.int64),
                                     rng.integers(0, N, 512)])).astype(np.uint64)
    want, gw = oracle.rows_ld(r["cat"], r["params"], r["variant"], rows)
    got = r["ell"][rows.astype(np.int64)]
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
    gg = r["grows"][rows.astype(np.int64)]
    # per row and component: relative to max(|g_row|, 1e-3 x the component's
    # largest |g_row| in the sample) (rows where a component cancels to ~0)
    den = np.maximum(np.abs(gw), 1e-3 * np.abs(gw).max(axis=0))
    assert np.all(np.abs(gg - gw) / den <= GRAD_TOL), np.max(np.abs(gg - gw) / den)


@pytest.mark.parametrize("name", CASES)
def test_1m_rows_sum_to_total(results, name):
    """Checksum: the device's fixed-order reduction equals the exactly
    rounded sum of the same launches' per-row terms."""
    r = results[name]
    assert r["ll"] == pytest.approx(math.fsum(r["ell"]), rel=1e-13)
    for k in range(5):
        col = r["grows"][:, k]
        tot = math.fsum(col)
        assert abs(r["grad"][k] - tot) <= 1e-13 * math.fsum(np.abs(col))
