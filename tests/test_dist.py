"""CPU multi-process tests of the one-process-per-GPU path (gloo, world
size 2): cost-balanced row shards, rank-order reduction of the 6-vector
partials, and the location broadcast.  The per-shard evaluation is the
long-double oracle here (test infrastructure); on a GPU box the same code
path runs the engine through the C ABI."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

P = dict(mu0=0.9, tau_t=4.0, xi0=0.5, sigma_x=0.4, sigma_t=1.5, area=100.0)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleShard:
    """Checker standing in for the device engine on rows [b, e)."""

    def __init__(self, cat, b, e, variant):
        from oracle.oracle import Oracle
        self.O = Oracle()
        self.cat = [np.array(a) for a in cat.arrays()]
        self.rows = np.arange(b, e, dtype=np.uint64)
        self.variant = variant

    def eval(self, params, grad=True):
        ell, g = self.O.rows_ld(self.cat, P, self.variant, self.rows, threads=2)
        return float(np.sum(ell)), g.sum(axis=0)

    def set_locations(self, lon, lat):
        self.cat[1], self.cat[2] = np.array(lon), np.array(lat)


def _worker(rank, world, port, variant, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2407_11349_b200 import HawkesParams, Variant, benchmark_catalog
    from paper_2407_11349_b200.dist import ShardedLikelihood
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cat = benchmark_catalog(1500, 77)
        sh = ShardedLikelihood(cat, shard_eval=lambda b, e: OracleShard(cat, b, e, variant))
        p = HawkesParams(**P, variant=Variant(variant))
        ll, g = sh.eval(p)
        rng = np.random.default_rng(9)
        lon, lat = rng.uniform(-5, 5, 1500), rng.uniform(-5, 5, 1500)
        if rank == 0:
            sh.set_locations(lon, lat)
        else:
            sh.set_locations()
        ll2, g2 = sh.eval(p)
        q.put((rank, sh.rows, ll, g.tolist(), ll2, g2.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant", [0, 1])
def test_two_rank_shards_reduce_to_the_whole(oracle, variant):
    from paper_2407_11349_b200 import benchmark_catalog
    port = free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, variant, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    (r0, rows0, ll0, g0, ll20, g20), (r1, rows1, ll1, g1, ll21, g21) = res
    assert rows0[0] == 0 and rows0[1] == rows1[0] and rows1[1] == 1500
    # every rank holds the identical (bitwise) total
    assert ll0 == ll1 and g0 == g1 and ll20 == ll21 and g20 == g21
    cat = benchmark_catalog(1500, 77).arrays()
    want, gw = oracle.ll_grad(cat, P, variant)
    assert ll0 == pytest.approx(want, rel=1e-13)
    np.testing.assert_allclose(g0, gw, rtol=1e-11, atol=1e-9)
    rng = np.random.default_rng(9)
    lon, lat = rng.uniform(-5, 5, 1500), rng.uniform(-5, 5, 1500)
    want2, gw2 = oracle.ll_grad((cat[0], lon, lat, cat[3]), P, variant)
    assert ll20 == pytest.approx(want2, rel=1e-13)
    np.testing.assert_allclose(g20, gw2, rtol=1e-11, atol=1e-9)


@pytest.mark.gpu
def test_nccl_rank_result_is_not_stale():
    """One NCCL rank (torch.distributed on the GPU): ShardedLikelihood.eval
    equals Evaluator.eval bitwise across alternating variants, i.e. the host
    read of the reduced 6-vector is ordered after the engine's stream (a read
    on torch's current stream returned the previous evaluation)."""
    import subprocess
    import sys
    from pathlib import Path
    script = Path(__file__).parent / "scripts" / "nccl_single_rank.py"
    r = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
