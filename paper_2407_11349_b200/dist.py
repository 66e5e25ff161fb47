"""One process per GPU: row-sharded evaluation over torch.distributed.

The reference parallelises only the outer sum over rows (Partition +
std::thread, engine.hpp:22-99; the paper's MPI gather).  Here
each rank owns a cost-balanced contiguous row shard (hk_plan_shards), keeps
the full catalog resident on its GPU, evaluates its shard's partial
[ell, d ell/d theta] (6 doubles), and the partials are all-gathered and summed
in rank order on every rank — bitwise deterministic for a fixed world size,
unlike a plain all-reduce whose summation order depends on the algorithm.
Per cut-posterior iteration the re-sampled locations are broadcast from
rank 0 (16 MB at N=1e6) and swapped in on the device.

The collective is the only cross-GPU traffic: 48 bytes per rank per
evaluation, and the location broadcast once per iteration.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .engine import Catalog, Evaluator, HawkesParams, plan_shards


class _DeviceView:
    """Zero-copy torch view of a device buffer owned by the engine."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3}


def reduce_rank_order(partial: torch.Tensor, group=None) -> torch.Tensor:
    """All-gathers each rank's 6-vector and sums them in rank order."""
    world = dist.get_world_size(group)
    parts = [torch.empty_like(partial) for _ in range(world)]
    dist.all_gather(parts, partial.contiguous(), group=group)
    acc = parts[0].clone()
    for r in range(1, world):
        acc += parts[r]
    return acc


class ShardedLikelihood:
    """This rank's shard of a catalog's log-likelihood + gradient.

    `shard_eval(b, e)` may replace the device engine for the rows [b, e)
    (the CPU tests plug a checker in to exercise the sharding and the
    reduction under gloo); by default the shard runs on `device` through the
    C ABI.
    """

    def __init__(self, catalog: Catalog, group=None, device: int | None = None, shard_eval=None,
                 variant=0):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.catalog = catalog
        self.bounds = plan_shards(catalog.t, self.world, variant)
        b, e = int(self.bounds[self.rank]), int(self.bounds[self.rank + 1])
        self.rows = (b, e)
        self.on_gpu = shard_eval is None
        if self.on_gpu:
            self.device = torch.device("cuda", device if device is not None else torch.cuda.current_device())
            self.ev = Evaluator(catalog, shard=(b, e), device=self.device.index)
            self.stream = torch.cuda.ExternalStream(self.ev.stream_ptr(), device=self.device)
            self._result = torch.as_tensor(_DeviceView(self.ev.result_device_ptr(), 6), device=self.device)
        else:
            self.device = torch.device("cpu")
            self.ev = shard_eval(b, e)

    # -- evaluation ---------------------------------------------------------

    def partial_async(self, params: HawkesParams, grad: bool = True) -> torch.Tensor:
        """Enqueues this shard's evaluation; returns its 6-vector (on the
        engine's stream when on GPU)."""
        if self.on_gpu:
            self.ev.eval_async(params, grad)
            return self._result
        ll, g = self.ev.eval(params, grad=True)
        return torch.tensor([ll, *g], dtype=torch.float64)

    def reduce(self, partial: torch.Tensor) -> torch.Tensor:
        if self.on_gpu:
            with torch.cuda.stream(self.stream):
                return reduce_rank_order(partial, self.group)
        return reduce_rank_order(partial, self.group)

    def eval(self, params: HawkesParams, grad: bool = True):
        total = self.reduce(self.partial_async(params, grad))
        if self.on_gpu:
            # the sum lives on the engine's stream: copy it to the host there
            # (a copy on torch's current stream would not wait for it)
            with torch.cuda.stream(self.stream):
                total = total.cpu()
        total = total.numpy()
        return (float(total[0]), total[1:].copy()) if grad else float(total[0])

    # -- cut-posterior location refresh ---------------------------------------

    def set_locations(self, lon=None, lat=None) -> None:
        """Rank 0 passes the re-sampled locations; every rank receives them by
        broadcast and swaps them in (LikelihoodWorkspace::set_locations,
        engine.hpp:172-178)."""
        n = len(self.catalog)
        if self.on_gpu:
            xy = torch.empty(2, n, dtype=torch.float64, device=self.device)
            with torch.cuda.stream(self.stream):
                if self.rank == 0:
                    xy.copy_(torch.as_tensor(np.stack([lon, lat])), non_blocking=False)
                dist.broadcast(xy, src=0, group=self.group)
                self.ev.set_locations_device(xy[0].data_ptr(), xy[1].data_ptr())
            return
        xy = torch.empty(2, n, dtype=torch.float64)
        if self.rank == 0:
            xy.copy_(torch.as_tensor(np.stack([lon, lat])))
        dist.broadcast(xy, src=0, group=self.group)
        self.ev.set_locations(xy[0].numpy(), xy[1].numpy())
