"""Host-side mirror of the reference's hot-path interface
(/root/reference/proj/include/hawkes/{types,model,engine}.hpp), backed by
the B200 engine through the C ABI.

Names, argument meaning and error behaviour follow the reference:

  reference (C++)                               here
  -------------------------------------------------------------------------
  Variant, Precision           types.hpp:16,112  Variant, Precision
  Catalog / Catalog::sorted    types.hpp:41-78   Catalog / Catalog.sorted
  HawkesParams + validate      types.hpp:83-110  HawkesParams
  Partition::make              engine.hpp:22-43  Partition.make / make_partition
  log_likelihood               engine.hpp:101-110 log_likelihood
  event_contribution           model.hpp:225-230 event_contribution
  LikelihoodWorkspace<double>  engine.hpp:117-229 LikelihoodWorkspace
  benchmark_catalog            engine.hpp:251-259 benchmark_catalog
  (new)                                          log_likelihood_and_gradient

std::invalid_argument maps to ValueError, std::out_of_range to IndexError.
Precision.single runs the trigger pair sums in FP32 on the GPU (log-likelihood
only, like the reference); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import weakref
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from ._lib import check, lib


class Variant(enum.IntEnum):
    constant = 0
    varying = 1


class Precision(enum.Enum):
    single = "single"
    dbl = "double"


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Catalog:
    """Immutable, time-ordered event set in SoA form (t in weeks, lon/lat in
    degrees, density per square mile).  Validation and messages are the
    reference's (types.hpp:43-57)."""

    __slots__ = ("t", "lon", "lat", "density", "_ctx", "__weakref__")

    def __init__(self, t, lon, lat, density=None):
        t = _f64(t)
        lon = _f64(lon)
        lat = _f64(lat)
        density = np.ones_like(t) if density is None else _f64(density)
        if not (len(t) == len(lon) == len(lat) == len(density)):
            raise ValueError("Catalog: column lengths differ")
        check(lib.hk_validate_catalog(t, lon, lat, density, len(t)))
        for a in (t, lon, lat, density):
            a.setflags(write=False)
        self.t, self.lon, self.lat, self.density = t, lon, lat, density
        self._ctx = None

    @classmethod
    def sorted(cls, t, lon, lat, density=None) -> "Catalog":
        t = _f64(t)
        order = np.argsort(t, kind="stable")
        dens = np.ones_like(t) if density is None else _f64(density)
        return cls(t[order], _f64(lon)[order], _f64(lat)[order], dens[order])

    def size(self) -> int:
        return len(self.t)

    __len__ = size

    def t_end(self) -> float:
        return float(self.t[-1])

    def arrays(self):
        return self.t, self.lon, self.lat, self.density


@dataclass(frozen=True)
class HawkesParams:
    mu0: float = 1.0
    tau_t: float = 1.0
    xi0: float = 1.0
    sigma_x: float = 1.0
    sigma_t: float = 1.0
    area: float = 1.0
    variant: Variant = Variant.constant

    def validate(self) -> None:
        p = self.to_c()
        check(lib.hk_validate_params(C.byref(p)))

    def to_c(self) -> _lib.hk_params:
        return _lib.hk_params(float(self.mu0), float(self.tau_t), float(self.xi0),
                              float(self.sigma_x), float(self.sigma_t), float(self.area),
                              int(self.variant))

    def sigma_x_prec(self) -> float:
        return 1.0 / self.sigma_x

    def tau_t_prec(self) -> float:
        return 1.0 / self.tau_t

    def omega(self) -> float:
        return 1.0 / self.sigma_t

    def inv_area(self) -> float:
        return 1.0 / self.area

    def with_(self, **kw) -> "HawkesParams":
        return replace(self, **kw)


class Partition:
    """Contiguous row ranges (engine.hpp:22-43).  The GPU engine keeps the
    type for API compatibility; it shards rows by its own cost model and the
    result does not depend on the partition beyond rounding."""

    def __init__(self, ranges):
        self.ranges = [(int(b), int(e)) for b, e in ranges]

    def workers(self) -> int:
        return len(self.ranges)

    @staticmethod
    def make(n: int, g: int) -> "Partition":
        if n < 0 or g < 0:
            raise ValueError("Partition: sizes must be non-negative")
        b = np.zeros(g + 1, dtype=np.uintp)
        check(lib.hk_partition_make(n, g, b))
        return Partition(zip(b[:-1], b[1:]))


def make_partition(n: int, g: int) -> Partition:
    return Partition.make(n, g)


def plan_shards(t, g: int, variant: "Variant | int" = 0) -> np.ndarray:
    """Cost-balanced row-shard boundaries (g+1) for g devices/ranks, for
    the kernel variant the shards will mostly run (the density-scaled
    kernel's trigger is spatially culled, so its rows weigh differently)."""
    t = _f64(t)
    b = np.zeros(g + 1, dtype=np.uintp)
    check(lib.hk_plan_shards_variant(t, len(t), g, int(variant), b))
    return b.astype(np.int64)


def benchmark_catalog(n: int, seed: int = 42) -> Catalog:
    """The reference's synthetic uniform catalog (engine.hpp:251-259),
    bit-identical to its mt19937_64 / libstdc++ draws."""
    t, x, y, d = (np.zeros(n) for _ in range(4))
    check(lib.hk_benchmark_catalog(n, seed, t, x, y, d))
    return Catalog(t, x, y, d)


class Evaluator:
    """One engine context: the catalog resident on `n_gpus` devices (or one
    rank's row shard on `device`)."""

    def __init__(self, catalog: Catalog, n_gpus: int = 1, shard=None, device: int = 0, devices=None,
                 plan_for: "Variant | int" = 0):
        self.catalog = catalog
        h = C.c_void_p()
        t, x, y, d = catalog.arrays()
        if devices is not None:
            # one cost-balanced shard per entry; distinct devices exchange the
            # 6-vectors and locations over NCCL, a repeated device by peer copies
            dv = np.ascontiguousarray(devices, dtype=np.int32)
            check(lib.hk_create_devices(t, x, y, d, len(t), dv, len(dv), int(plan_for), C.byref(h)))
        elif shard is None:
            check(lib.hk_create(t, x, y, d, len(t), n_gpus, C.byref(h)))
        else:
            b, e = shard
            check(lib.hk_create_shard(t, x, y, d, len(t), b, e, device, C.byref(h)))
        self._h = h
        self._fin = weakref.finalize(self, lib.hk_destroy, h)

    def close(self) -> None:
        self._fin()

    @property
    def handle(self):
        return self._h

    def rows(self):
        b, e, nd = C.c_size_t(), C.c_size_t(), C.c_int()
        check(lib.hk_rows(self._h, C.byref(b), C.byref(e), C.byref(nd)))
        return b.value, e.value, nd.value

    def set_locations(self, lon, lat) -> None:
        lon, lat = _f64(lon), _f64(lat)
        if len(lon) != len(self.catalog) or len(lat) != len(self.catalog):
            raise ValueError("set_locations: length mismatch")
        check(lib.hk_set_locations(self._h, lon, lat))

    def resample_locations(self, regions: "Regions", seed: int, counter: int = 0) -> None:
        """GPU X refresh: one draw per event from its region straight into
        this context's device locations (hk_resample_locations)."""
        check(lib.hk_resample_locations(self._h, regions.handle, seed, counter))

    def set_locations_device(self, lon_ptr: int, lat_ptr: int) -> None:
        check(lib.hk_set_locations_device(self._h, C.c_void_p(lon_ptr), C.c_void_p(lat_ptr)))

    def eval(self, params: HawkesParams, grad: bool = False):
        p = params.to_c()
        ll = C.c_double()
        g = np.zeros(5)
        check(lib.hk_eval(self._h, C.byref(p), C.byref(ll),
                          g.ctypes.data_as(C.c_void_p) if grad else None))
        return (ll.value, g) if grad else ll.value

    def eval_detail(self, params: HawkesParams, grad: bool = True):
        """hk_eval plus the per-row ell_n (and d ell_n / d theta) of the same
        production launches, for the context's rows [begin, end)."""
        b, e, _ = self.rows()
        p = params.to_c()
        ll = C.c_double()
        g = np.zeros(5)
        ell = np.zeros(e - b)
        gr = np.zeros((e - b, 5)) if grad else None
        check(lib.hk_eval_detail(self._h, C.byref(p), C.byref(ll),
                                 g.ctypes.data_as(C.c_void_p) if grad else None,
                                 ell.ctypes.data_as(C.c_void_p),
                                 gr.ctypes.data_as(C.c_void_p) if grad else None))
        return (ll.value, g, ell, gr) if grad else (ll.value, ell)

    def eval_single(self, params: HawkesParams) -> float:
        """Precision.single, log-likelihood only: FP32 trigger arithmetic, or
        from 131072 events the FP64 expansion path (HK_OPT_SINGLE_FP64)."""
        p = params.to_c()
        ll = C.c_double()
        check(lib.hk_eval_single(self._h, C.byref(p), C.byref(ll)))
        return ll.value

    def ws_eval(self, params: HawkesParams, grad: bool = False, force: bool = False):
        """Workspace evaluation (hk_ws_eval): reuses the cached background
        half while tau_t is unchanged and the trigger half while sigma_x,
        sigma_t, the variant and the locations are unchanged."""
        p = params.to_c()
        ll = C.c_double()
        g = np.zeros(5)
        check(lib.hk_ws_eval(self._h, C.byref(p), int(force), C.byref(ll),
                             g.ctypes.data_as(C.c_void_p) if grad else None))
        return (ll.value, g) if grad else ll.value

    def ws_eval_single(self, params: HawkesParams, force: bool = False) -> float:
        """Single-precision workspace evaluation (hk_ws_eval_single), LL only."""
        p = params.to_c()
        ll = C.c_double()
        check(lib.hk_ws_eval_single(self._h, C.byref(p), int(force), C.byref(ll)))
        return ll.value

    def ws_stats(self):
        h, m = C.c_long(), C.c_long()
        check(lib.hk_ws_stats(self._h, C.byref(h), C.byref(m)))
        return h.value, m.value

    def eval_async(self, params: HawkesParams, grad: bool = True) -> None:
        p = params.to_c()
        check(lib.hk_eval_async(self._h, C.byref(p), int(grad)))

    def result_device_ptr(self) -> int:
        return lib.hk_result_device(self._h)

    def stream_ptr(self, dev: int = 0) -> int:
        return lib.hk_stream(self._h, dev)

    def eval_rows(self, params: HawkesParams, b: int, e: int, grad: bool = False):
        if b < 0 or e < 0:
            raise IndexError("event_contribution: index out of range")
        p = params.to_c()
        ell = np.zeros(max(e - b, 1))
        g = np.zeros((max(e - b, 1), 5))
        check(lib.hk_eval_rows(self._h, C.byref(p), b, e, ell,
                               g.ctypes.data_as(C.c_void_p) if grad else None))
        return (ell, g) if grad else ell

    def set_bg_expansion(self, on: bool) -> None:
        """Exact block expansion of the background sum (default on); off
        forces the direct per-pair path."""
        check(lib.hk_set_option(self._h, _lib.HK_OPT_BG_EXPANSION, int(on)))

    def set_fgt(self, on: bool) -> None:
        """HK_OPT_FGT: the homogeneous trigger's Hermite expansion (default on)."""
        check(lib.hk_set_option(self._h, _lib.HK_OPT_FGT, int(on)))

    def set_bg_fgt(self, on: bool) -> None:
        """HK_OPT_BG_FGT: the background's 1-D Hermite expansion in time (default on)."""
        check(lib.hk_set_option(self._h, _lib.HK_OPT_BG_FGT, int(on)))

    def set_tr_cut(self, on: bool) -> None:
        """HK_OPT_TR_CUT: the density-scaled trigger's certified e^-46 spatial cut (default on)."""
        check(lib.hk_set_option(self._h, _lib.HK_OPT_TR_CUT, int(on)))

    def set_cells(self, on: bool) -> None:
        """HK_OPT_CELLS: the density-scaled trigger over spatial cell tiles (default on)."""
        check(lib.hk_set_option(self._h, _lib.HK_OPT_CELLS, int(on)))

    def set_single_fp64(self, on: bool) -> None:
        """HK_OPT_SINGLE_FP64: large Precision.single evaluations through the FP64 expansions (default on)."""
        check(lib.hk_set_option(self._h, _lib.HK_OPT_SINGLE_FP64, int(on)))

    def fgt_stats(self):
        """(evaluations through the expansion, direct recomputations, last
        async evaluation flagged)."""
        e, f, a = C.c_long(), C.c_long(), C.c_int()
        check(lib.hk_fgt_stats(self._h, C.byref(e), C.byref(f), C.byref(a)))
        return e.value, f.value, bool(a.value)

    def set_profiling(self, on: bool) -> None:
        check(lib.hk_set_profiling(self._h, int(on)))

    def profile(self):
        ms, npair, ntot = C.c_double(), C.c_long(), C.c_long()
        check(lib.hk_profile(self._h, C.byref(ms), C.byref(npair), C.byref(ntot)))
        return ms.value, npair.value, ntot.value

    def profile_kinds(self):
        """(ms[5], launches[5]) of the pair launches by kind: both halves,
        background only, trigger only, Hermite-expansion moments, Hermite-
        expansion rows."""
        ms, n = np.zeros(5), np.zeros(5, dtype=np.int64)
        check(lib.hk_profile_kinds(self._h, ms, n))
        return ms, n

    def reset_profile(self) -> None:
        check(lib.hk_reset_profile(self._h))


def _evaluator_for(catalog: Catalog) -> Evaluator:
    # One cached single-device context per catalog (the catalog is immutable).
    if catalog._ctx is None:
        catalog._ctx = Evaluator(catalog)
    return catalog._ctx


def _check_call(catalog: Catalog, p: HawkesParams, part: Partition):
    p.validate()
    if not part.ranges or part.ranges[-1][1] != catalog.size():
        raise ValueError("log_likelihood: partition does not cover the catalog")


def log_likelihood(catalog: Catalog, p: HawkesParams, part: Partition,
                   precision: Precision = Precision.dbl) -> float:
    """engine.hpp:101-110 on the B200 engine (Precision.single: FP32 trigger
    arithmetic, like the reference's EvalData<float> path)."""
    _check_call(catalog, p, part)
    ev = _evaluator_for(catalog)
    return ev.eval(p) if precision == Precision.dbl else ev.eval_single(p)


def log_likelihood_and_gradient(catalog: Catalog, p: HawkesParams, part: Partition | None = None,
                                precision: Precision = Precision.dbl):
    """(log-likelihood, d ell / d (mu0, tau_t, xi0, sigma_x, sigma_t)); the
    gradient is evaluated in double precision only."""
    _check_call(catalog, p, part or Partition.make(catalog.size(), 1))
    if precision != Precision.dbl:
        raise ValueError("log_likelihood_and_gradient: the gradient is evaluated in double precision only")
    return _evaluator_for(catalog).eval(p, grad=True)


def event_contribution(p: HawkesParams, catalog: Catalog, n: int) -> float:
    """model.hpp:225-230."""
    if n < 0 or n >= catalog.size():
        raise IndexError("event_contribution: index out of range")
    p.validate()
    return float(_evaluator_for(catalog).eval_rows(p, n, n + 1)[0])


@dataclass
class Region:
    """A coarse region (geo.hpp:85-113): an exact point, or polygons, each a
    list of rings [outer, hole, hole, ...], a ring an (m, 2) array of
    (lon, lat) vertices."""
    id: str
    is_point: bool = False
    point: tuple = (0.0, 0.0)
    polygons: list = None
    density: float = 1.0


class Regions:
    """A region table plus each event's region, resident on one GPU for the
    location sampler (hk_regions_*): one uniform draw per event from its
    region, Philox-keyed by (seed, counter) -- the reference's algorithm
    (sample_point_in_region, geo.hpp:138-161) on its own random stream."""

    def __init__(self, regions, event_region, device: int = 0):
        is_point, pts, rparts, prings, rverts, verts, ids = [], [], [0], [0], [0], [], []
        for r in regions:
            is_point.append(1 if r.is_point else 0)
            pts.extend([float(r.point[0]), float(r.point[1])])
            ids.append(r.id.encode())
            for poly in (r.polygons or []):
                for ring in poly:
                    ring = np.asarray(ring, dtype=np.float64).reshape(-1, 2)
                    verts.append(ring)
                    rverts.append(rverts[-1] + len(ring))
                prings.append(prings[-1] + len(poly))
            rparts.append(len(prings) - 1)
        self._ids = (C.c_char_p * len(ids))(*ids)
        er = np.ascontiguousarray(event_region, dtype=np.int32)
        self.n_events = len(er)
        h = C.c_void_p()
        check(lib.hk_regions_create(
            len(regions), np.ascontiguousarray(is_point, dtype=np.int32), np.ascontiguousarray(pts, dtype=np.float64),
            np.ascontiguousarray(rparts, dtype=np.uintp), np.ascontiguousarray(prings, dtype=np.uintp),
            np.ascontiguousarray(rverts, dtype=np.uintp),
            np.ascontiguousarray(np.concatenate(verts) if verts else np.zeros((0, 2))).reshape(-1),
            C.cast(self._ids, C.c_void_p), len(er), er, device, C.byref(h)))
        self._h = h
        self._fin = weakref.finalize(self, lib.hk_regions_destroy, h)

    @property
    def handle(self):
        return self._h

    def sample(self, seed: int, counter: int = 0):
        """One draw per event: (lon, lat) host arrays."""
        lon, lat = np.zeros(self.n_events), np.zeros(self.n_events)
        check(lib.hk_regions_sample(self._h, seed, counter, lon, lat))
        return lon, lat


class LikelihoodWorkspace:
    """LikelihoodWorkspace<double> (engine.hpp:117-229) on the engine, with
    the per-row background [B, B2] and trigger [T, Td, Tq] sums cached on the
    device: a mu0/xi0 proposal recombines cached sums in O(N), tau_t refreshes
    only the background, sigma_x/sigma_t (or set_locations) only the trigger.
    Results are bitwise identical to a fresh evaluation at every setting.
    precision=Precision.single is LikelihoodWorkspace<float>: the same
    caches over the FP32 trigger arithmetic of Precision.single (LL only)."""

    def __init__(self, catalog: Catalog, variant: Variant, workers: int = 1,
                 precision: Precision = Precision.dbl):
        self._catalog = catalog
        self._variant = Variant(variant)
        self._single = precision == Precision.single
        self._ev = Evaluator(catalog)

    def _eval(self, p: HawkesParams, grad: bool, force: bool):
        p = replace(p, variant=self._variant)
        if self._single:
            if grad:
                raise ValueError("LikelihoodWorkspace<float>: the gradient is double precision only")
            return self._ev.ws_eval_single(p, force=force)
        return self._ev.ws_eval(p, grad=grad, force=force)

    def evaluate_full(self, p: HawkesParams, grad: bool = False):
        return self._eval(p, grad, True)

    def evaluate_proposal(self, p: HawkesParams, grad: bool = False):
        return self._eval(p, grad, False)

    def commit_proposal(self) -> None:
        """The device cache keeps the current and the proposal state (two
        entries per half), so promotion needs no work."""

    def set_locations(self, lon, lat) -> None:
        self._ev.set_locations(lon, lat)

    def stats(self):
        """(cache hits, misses) of the workspace evaluations so far."""
        return self._ev.ws_stats()
