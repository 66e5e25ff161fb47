#!/usr/bin/env python
"""Benchmark of the StHP log-likelihood + gradient hot path (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--n EVENTS] [--variant constant|varying]

One step = one full log-likelihood + 5-component gradient evaluation of the
reference's synthetic catalog benchmark_catalog(N, 42) (engine.hpp:251-259)
at the reference's bench parameters (engine.hpp:272-273).  Default workload:
BASELINE config 3, N = 1,000,000, homogeneous (constant) kernel, row-sharded
over the ranks of a torchrun job (strong scaling: the catalog is fixed).

Prints ONE JSON line (rank 0).  `value` is evaluations/s timed on the device
(CUDA events on the engine's stream, inputs resident, L2 flushed between
steps, max over ranks); `e2e` is the same metric through the public API with
each step's re-sampled locations copied from pinned host memory and the
result read back to the host.  `--impl reference` times the reference's own
CPU path (oracle/_ref, the unmodified reference headers) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "log-lik+gradient evals/sec at N=1M (1/2/4/8 B200); G pair-interactions/sec"
BENCH_PARAMS = dict(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0)
FP64_PER_PAIR = 33.5  # SURVEY.md 8(d) convention: FP64-pipe instructions per ordered pair
CPU_SAMPLE_ROWS = 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--variant", choices=["constant", "varying"], default="constant")
    ap.add_argument("--cpu-rows", type=int, default=CPU_SAMPLE_ROWS)
    ap.add_argument("--force-dist", action="store_true",
                    help="use the torch.distributed/NCCL row-shard path even with one rank")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(args, world):
    return {"workload": f"StHP log-likelihood + gradient, benchmark_catalog(N={args.n}, seed=42), "
                        f"{args.variant} kernel, bench params (engine.hpp:272-273)",
            "n_events": args.n, "variant": args.variant, "gradient": True,
            "params": BENCH_PARAMS, "parallelism": f"row shards x{world}",
            "l2": "flushed between steps (256 MiB memset on the engine stream)"}


# ---------------------------------------------------------------------------
# CPU reference leg


def cpu_sample_time(cat, variant_id, rows, steps=1):
    """Seconds per sample through the reference's own row kernel
    (slice_log_likelihood, oracle/_ref) on all host threads; falls back to the
    C restatement (`port`) when oracle/_ref is absent."""
    from oracle.oracle import Oracle, Reference, ref_available
    threads = os.cpu_count() or 1
    if ref_available():
        R = Reference()
        fn = lambda: R.rows(cat, BENCH_PARAMS, variant_id, rows, threads)  # noqa: E731
        kind = "reference"
    else:
        O = Oracle()
        fn = lambda: O.rows_lanes(cat, BENCH_PARAMS, variant_id, rows, threads)  # noqa: E731
        kind = "port"
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return times, kind, threads


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sample_rows(n, k):
    return np.unique(np.linspace(0, n - 1, min(k, n)).astype(np.uint64))


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2407_11349_b200 import benchmark_catalog
    cat = benchmark_catalog(args.n, 42).arrays()
    rows = sample_rows(args.n, args.cpu_rows)
    v = 1 if args.variant == "varying" else 0
    cpu_sample_time(cat, v, rows[: max(1, len(rows) // 8)], steps=max(1, args.warmup))  # warm-up
    times, kind, threads = cpu_sample_time(cat, v, rows, steps=args.steps)
    scale = args.n / len(rows)
    per_eval = [t * scale for t in times]
    value = 1.0 / statistics.median(per_eval)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s",
        "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(per_eval) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload(args, 1),
        "pairs_per_sec": value * args.n * (args.n - 1),
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": kind,
                         "cpu": cpu_model(),
                         "sample": f"{len(rows)} evenly spaced rows of N={args.n} through the reference's "
                                   f"slice_log_likelihood (LL only: the reference has no gradient), "
                                   f"extrapolated x{scale:.0f}; median of {args.steps} samples"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ---------------------------------------------------------------------------
# GPU leg


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            c = [x.strip() for x in line.split(",")]
            if len(c) < 9 or not c[0].isdigit() or int(c[0]) != self.gpu:
                continue
            try:
                sm.append(float(c[1]))
                mx.append(float(c[2]))
            except ValueError:
                continue
            for nm, val in zip(names, c[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2407_11349_b200 import HawkesParams, Variant, benchmark_catalog
    from paper_2407_11349_b200._lib import lib
    from paper_2407_11349_b200.dist import ShardedLikelihood
    import ctypes as C

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_dist = world > 1 or args.force_dist
    if use_dist:
        if "MASTER_ADDR" not in os.environ:  # --force-dist outside torchrun: loopback rendezvous
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
            os.environ["MASTER_ADDR"] = "127.0.0.1"
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)

    cat = benchmark_catalog(args.n, 42)
    p = HawkesParams(**BENCH_PARAMS, variant=Variant[args.variant])
    if use_dist:
        sh = ShardedLikelihood(cat, device=local, variant=p.variant)
        ev, stream = sh.ev, sh.stream
    else:
        sh = None
        from paper_2407_11349_b200 import Evaluator
        ev = Evaluator(cat, shard=(0, args.n), device=local)
        stream = torch.cuda.ExternalStream(ev.stream_ptr(), device=dev)

    # measured FP64 peak of this GPU (roofline denominator)
    tf, pms = C.c_double(), C.c_double()
    lib.hk_measure_fp64_peak(local, C.byref(tf), C.byref(pms))
    fp64_peak = tf.value

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(params=p):
        with torch.cuda.stream(stream):
            flush.zero_()
        if sh is not None:
            sh.reduce(sh.partial_async(params, True))
        else:
            ev.eval_async(params, True)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev.reset_profile()
    ev.set_profiling(True)
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local) if rank == 0 else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record()
    for _ in range(args.steps):
        step()
    with torch.cuda.stream(stream):
        e1.record()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    ms_total = e0.elapsed_time(e1)
    pair_ms, pair_launches, launches = ev.profile()
    ev.set_profiling(False)
    t = torch.tensor([ms_total, pair_ms / max(pair_launches, 1)], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total, pair_ms_avg = float(t[0]), float(t[1])

    # ---- the same step on the direct per-pair path (background expansion
    # off): the pure O(N^2) kernel, for the FP64-pipe roofline of SURVEY 8(d)
    direct_steps = 2
    ev.set_bg_expansion(False)
    step()
    torch.cuda.synchronize()
    ev.reset_profile()
    ev.set_profiling(True)
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        d0.record()
    for _ in range(direct_steps):
        step()
    with torch.cuda.stream(stream):
        d1.record()
    torch.cuda.synchronize()
    dpair_ms, dpair_n, _ = ev.profile()
    ev.set_profiling(False)
    ev.set_bg_expansion(True)
    t = torch.tensor([d0.elapsed_time(d1), dpair_ms / max(dpair_n, 1)], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    direct_ms_total, direct_pair_ms = float(t[0]), float(t[1])
    # ---- the other kernel variant on the same catalog (config 4, the
    # density-scaled lengthscale, when the headline is homogeneous)
    other = "varying" if args.variant == "constant" else "constant"
    p_other = HawkesParams(**BENCH_PARAMS, variant=Variant[other])
    other_steps = 3
    for _ in range(2):
        step(p_other)
    torch.cuda.synchronize()
    ev.reset_profile()
    ev.set_profiling(True)
    o0, o1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        o0.record()
    for _ in range(other_steps):
        step(p_other)
    with torch.cuda.stream(stream):
        o1.record()
    torch.cuda.synchronize()
    opair_ms, opair_n, _ = ev.profile()
    ev.set_profiling(False)
    t = torch.tensor([o0.elapsed_time(o1), opair_ms / max(opair_n, 1)], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    other_ms_total, other_pair_ms = float(t[0]), float(t[1])

    # result of the last step, for the record
    if sh is not None:
        ll, g = sh.eval(p, grad=True)
    else:
        ll, g = ev.eval(p, grad=True)

    # ---- e2e through the public API: pinned-host locations in, result out
    pin = torch.empty(2, args.n, dtype=torch.float64).pin_memory()
    pin.numpy()[0] = cat.lon
    pin.numpy()[1] = cat.lat
    lon_h, lat_h = pin.numpy()[0], pin.numpy()[1]

    def e2e_step():
        if sh is not None:
            sh.set_locations(lon_h, lat_h) if rank == 0 else sh.set_locations()
            return sh.eval(p, grad=True)
        ev.set_locations(lon_h, lat_h)
        return ev.eval(p, grad=True)

    e2e_step()
    if use_dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t[0])

    if rank == 0:
        n = args.n
        pairs = n * (n - 1)
        value = args.steps / (ms_total * 1e-3)
        rows_local = ev.rows()
        pairs_local = (rows_local[1] - rows_local[0]) * (n - 1)
        achieved = pairs_local * FP64_PER_PAIR * 2 / (pair_ms_avg * 1e-3) / 1e12
        # the pair kernel's DRAM traffic per launch from the committed ncu capture
        traffic, ncu = None, {}
        prof = ROOT / "profiles" / "r01_pair_kernel_ncu.json"
        if prof.exists():
            d = json.loads(prof.read_text())
            tag = f"{args.variant}_{n}"
            traffic = d.get("dram_bytes_per_launch", {}).get(tag)
            for cap in d.get("captures", []):
                if cap.get("tag") == tag and cap.get("duration_ms"):
                    pipe = cap["fp64_pipe_pct"] / 100.0
                    fp64_per_pair = (pipe * 2 * 148 * cap["sm_clock_ghz"] * 1e9 * cap["duration_ms"] * 1e-3
                                     * 32 / pairs_local)
                    ncu = {"fp64_pipe_active": pipe, "fp64_instr_per_pair_executed": fp64_per_pair,
                           "source": "profiles/r01_pair_kernel_ncu.json (ncu --set full, same build)"}
        cpu = None
        if world == 1:
            rows = sample_rows(n, args.cpu_rows)
            times, kind, threads = cpu_sample_time(cat.arrays(), int(p.variant), rows, steps=1)
            cpu_eval_s = times[0] * n / len(rows)
            cpu = {"value": 1.0 / cpu_eval_s, "unit": "evals/s", "cores": threads, "kind": kind,
                   "cpu": cpu_model(),
                   "sample": f"{len(rows)} evenly spaced rows of N={n} through the reference's "
                             f"slice_log_likelihood (LL only: no gradient in the reference), "
                             f"extrapolated x{n / len(rows):.0f}"}
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload(args, world),
            "pairs_per_sec": value * pairs,
            "e2e": {"value": args.steps / e2e_s, "unit": "evals/s", "h2d_bytes_per_step": 2 * n * 8,
                    "d2h_bytes_per_step": 6 * 8,
                    "note": "per step: hk_set_locations from pinned host (lon, lat) + LL+grad + "
                            "result read to host" + ("; locations broadcast over NCCL" if world > 1 else "")},
            "gpu_launches": int(launches),
            "roofline": {"bound": "fp64", "kernel": "pair_kernel", "achieved": achieved,
                         "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                         "traffic": traffic,
                         "peak_source": "measured in this run: register-resident DFMA loop "
                                        "(hk_measure_fp64_peak); MEASURED_PEAKS.json has no FP64 figure",
                         "convention": f"{FP64_PER_PAIR} FP64-pipe instructions per ordered pair "
                                       "(SURVEY.md 8d: direct evaluation, libm-style exp), 2 flop each; "
                                       f"pair kernel avg {pair_ms_avg:.2f} ms over {pairs_local:.3e} pairs/launch. "
                                       "frac > 1 because the kernel needs fewer FP64 instructions per pair "
                                       "than the convention (exact background block expansion + 64-entry-table "
                                       "exp); the pipe's real utilisation is `ncu.fp64_pipe_active`",
                         "ncu": ncu},
            "direct_kernel": {
                "note": "the same LL+grad step with the background block expansion disabled "
                        "(HK_OPT_BG_EXPANSION=0): every ordered pair evaluated directly",
                "value": direct_steps / (direct_ms_total * 1e-3), "unit": "evals/s",
                "ms_per_step": direct_ms_total / direct_steps,
                "roofline": {"bound": "fp64", "achieved": pairs_local * FP64_PER_PAIR * 2 / (direct_pair_ms * 1e-3) / 1e12,
                             "peak": fp64_peak, "unit": "TFLOP/s",
                             "frac": pairs_local * FP64_PER_PAIR * 2 / (direct_pair_ms * 1e-3) / 1e12 / fp64_peak}},
            ("density_scaled" if other == "varying" else "homogeneous"): {
                "note": f"the same LL+grad step with the {other} kernel on the same catalog "
                        f"(BASELINE config {4 if other == 'varying' else 3}), device-timed like `value`",
                "variant": other, "value": other_steps / (other_ms_total * 1e-3), "unit": "evals/s",
                "ms_per_step": other_ms_total / other_steps, "pair_kernel_ms": other_pair_ms,
                "pairs_per_sec": other_steps / (other_ms_total * 1e-3) * pairs},
            "cpu_baseline": cpu,
            "clocks": clk,
            "result": {"loglik": ll, "grad": [float(x) for x in g]},
        }
        emit(line)
    if dist.is_initialized():
        dist.destroy_process_group()


_JSON_FD = None


def emit(line):
    """The one JSON line, on the process's original stdout."""
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _JSON_FD
    # Libraries (NCCL's version banner, CUDA) may print to fd 1; keep stdout
    # for the JSON line alone by pointing fd 1 at stderr for the run.
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
