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
    """The reference's own CPU path (oracle/_ref: the unmodified reference
    headers) on the host cores.  Only oracle/ libraries load in this process:
    the catalog comes from the reference's benchmark_catalog too."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import Reference, ref_available
    if ref_available():
        cat = Reference().benchmark_catalog(args.n, 42)
    else:  # the C restatement's generator is not built; numpy mirror of the same draws is not bitwise
        raise SystemExit("bench.py --impl reference needs oracle/_ref (make -C oracle ref)")
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
    """SM clocks and throttle reasons during the timed region: NVML polled
    every ~2 ms from a background thread (a 67 ms region still yields dozens
    of samples; `nvidia-smi -lms` needs ~100 ms to start and may yield none),
    with `nvidia-smi` as the fallback when NVML is unavailable."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.p = None
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = gpu_index
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if ids and all(v.isdigit() for v in ids) and gpu_index < len(ids):
                idx = int(ids[gpu_index])
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.sm, self.masks = [], []
            self.run = True
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:  # noqa: BLE001 - NVML missing or refused: nvidia-smi below
            self.nvml = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def _poll(self):
        nv = self.nvml
        while self.run:
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.masks.append(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def stop(self):
        if self.nvml is not None:
            self.run = False
            self.t.join()
            nv = self.nvml
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            reasons = sorted(nm for nm, b in bits.items() if any(m & b for m in self.masks))
            return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_sm,
                    "reasons": reasons, "samples": len(self.sm), "source": "nvml"}
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
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


COUNTS = ROOT / "profiles" / "r02_fp64_counts.json"


def source_sha():
    """Hash of the library's sources and build recipe: the counts below are a
    property of the build (nvcc's output is not bit-reproducible, so the
    binary's own hash would change on every rebuild of the same sources)."""
    import hashlib
    h = hashlib.sha256()
    csrc = ROOT / "paper_2407_11349_b200" / "csrc"
    for f in sorted(p for p in csrc.iterdir() if p.suffix in (".cu", ".cuh", ".cpp", ".hpp")) + [ROOT / "Makefile"]:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()[:16]


def measured_counts(tag):
    """FP64-pipe instructions and DRAM bytes of one pair launch from the
    committed ncu capture of the same workload (tools/capture_counts.py:
    sm__inst_executed_pipe_fp64.sum x 32 thread slots, dram__bytes_*.sum);
    the counts are a property of (build, catalog, params), deterministic."""
    if not COUNTS.exists():
        return None
    d = json.loads(COUNTS.read_text())
    c = d.get("launches", {}).get(tag)
    if c is None:
        return None
    return dict(c, stale=d.get("src_sha16") != source_sha(), source=str(COUNTS.relative_to(ROOT)))


def roofline(tag, launch_ms, fp64_peak, pairs, algorithmic_bytes):
    """Roofline of the dominant pair launch: achieved = FP64-pipe thread
    instructions executed per launch (ncu count, FMA-equivalent, 2 flop each)
    / the launch's live CUDA-event duration; peak = this GPU's measured DFMA
    throughput; frac = achieved / peak = FP64-pipe utilisation."""
    c = measured_counts(tag)
    r = {"bound": "fp64", "kernel": tag, "unit": "TFLOP/s", "peak": fp64_peak,
         "peak_source": "measured in this run: register-resident DFMA loop (hk_measure_fp64_peak, "
                        "2 flop per DFMA); MEASURED_PEAKS.json has no FP64 figure",
         "launch_ms": launch_ms, "algorithmic_bytes": algorithmic_bytes}
    if c is None or not launch_ms > 0:
        r.update(achieved=None, frac=None, traffic=None, note="no committed ncu count for this workload")
        return r
    slots = c["fp64_warp_inst"] * 32.0
    achieved = 2.0 * slots / (launch_ms * 1e-3) / 1e12
    r.update(achieved=achieved, frac=achieved / fp64_peak, traffic=c["dram_bytes"],
             fp64_thread_inst_per_launch=slots, fp64_inst_per_pair=slots / pairs,
             algorithmic_speedup=FP64_PER_PAIR / (slots / pairs),
             counts={"source": c["source"], "stale": c["stale"], "ncu_duration_ms": c["duration_ms"],
                     "ncu_fp64_pipe_pct": c.get("fp64_pipe_pct")},
             convention=f"achieved counts the FP64-pipe instructions the kernel actually executes "
                        f"(ncu); algorithmic_speedup = {FP64_PER_PAIR} FP64 per ordered pair (SURVEY.md 8d, "
                        "direct evaluation with a libm-style exp) / executed per pair")
    return r


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
    if use_dist:
        sh = ShardedLikelihood(cat, device=local, variant=Variant[args.variant])
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

    def step(params):
        with torch.cuda.stream(stream):
            flush.zero_()
        if sh is not None:
            sh.reduce(sh.partial_async(params, True))
        else:
            ev.eval_async(params, True)

    def maxr(*vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        if use_dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t]

    def timed(params, steps, warmup, sample_clocks=False):
        """Device time of `steps` evaluations (CUDA events on the engine's
        stream, barrier + synchronize both sides, max over ranks) and the
        pair launches' time by kind."""
        for _ in range(warmup):
            step(params)
        torch.cuda.synchronize()
        ev.reset_profile()
        ev.set_profiling(True)
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(local) if (rank == 0 and sample_clocks) else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record()
        for _ in range(steps):
            step(params)
        with torch.cuda.stream(stream):
            e1.record()
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        clk = clocks.stop() if clocks else None
        kms, kn = ev.profile_kinds()
        _, _, launches = ev.profile()
        ev.set_profiling(False)
        per_kind = [kms[k] / max(kn[k], 1) for k in range(5)]
        ms_total, *per_kind = maxr(e0.elapsed_time(e1), *per_kind)
        return ms_total, per_kind, int(launches), clk

    pin = torch.empty(2, args.n, dtype=torch.float64).pin_memory()
    pin.numpy()[0] = cat.lon
    pin.numpy()[1] = cat.lat
    lon_h, lat_h = pin.numpy()[0], pin.numpy()[1]

    def e2e(params, steps):
        """Through the public API: each step copies the (re-sampled)
        locations from pinned host memory, evaluates LL + gradient and reads
        the result back to the host."""
        def one():
            if sh is not None:
                sh.set_locations(lon_h, lat_h) if rank == 0 else sh.set_locations()
                return sh.eval(params, grad=True)
            ev.set_locations(lon_h, lat_h)
            return ev.eval(params, grad=True)
        one()
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            res = one()
        return maxr(time.perf_counter() - t0)[0], res

    n = args.n
    pairs = n * (n - 1)
    rows_local = ev.rows()
    pairs_local = (rows_local[1] - rows_local[0]) * (n - 1)
    p_main = HawkesParams(**BENCH_PARAMS, variant=Variant[args.variant])
    other = "varying" if args.variant == "constant" else "constant"
    p_other = HawkesParams(**BENCH_PARAMS, variant=Variant[other])

    ms_total, kinds, launches, clk = timed(p_main, args.steps, args.warmup, sample_clocks=True)
    e2e_s, (ll, g) = e2e(p_main, args.steps)
    o_ms, o_kinds, o_launches, _ = timed(p_other, args.steps, args.warmup)
    o_e2e_s, (o_ll, o_g) = e2e(p_other, args.steps)

    # the direct per-pair path (background block expansion and the trigger's
    # Hermite expansion off): the pure O(N^2) kernel, one evaluation
    ev.set_bg_expansion(False)
    ev.set_fgt(False)
    ev.set_bg_fgt(False)
    d_ms, d_kinds, _, _ = timed(HawkesParams(**BENCH_PARAMS, variant=Variant.constant), 1, 1)
    ev.set_bg_expansion(True)
    ev.set_fgt(True)
    ev.set_bg_fgt(True)
    fgt_stats = ev.fgt_stats()

    if rank == 0:
        def cpu(variant_id):
            if world != 1:
                return None
            rows = sample_rows(n, args.cpu_rows)
            times, kind, threads = cpu_sample_time(cat.arrays(), variant_id, rows, steps=1)
            return {"value": 1.0 / (times[0] * n / len(rows)), "unit": "evals/s", "cores": threads,
                    "kind": kind, "cpu": cpu_model(),
                    "sample": f"{len(rows)} evenly spaced rows of N={n} through the reference's "
                              f"slice_log_likelihood (LL only: no gradient in the reference), "
                              f"extrapolated x{n / len(rows):.0f}"}

        # algorithmic bytes of a pair launch: the catalog columns it reads
        # (t, x, y, w, v; + K, z for the density-scaled trigger) once and the
        # five row sums it writes once; of the expansion's row launch: the
        # rows (t, x, y), the prefix moments of every checkpoint once
        # (profiles: fgt_moment_bytes) and the trigger sums updated in place
        rows_n = rows_local[1] - rows_local[0]

        def algo_bytes(variant, kind):
            if kind == "fgt_rows":
                c = measured_counts(f"{variant}_{n}_fgt_rows") or {}
                return 3 * 8 * rows_n + 2 * 3 * 8 * rows_n + c.get("moment_bytes", 0)
            cols = {"both": 5, "bg": 1, "trigger": 7 if variant == "varying" else 5}[kind]
            outs = {"both": 5, "bg": 2, "trigger": 3}[kind]
            return (cols + outs) * 8 * rows_n

        def pair_line(variant, kinds_ms):
            """Roofline of the evaluation's dominant launch; the other launch
            that replaces O(N^2) work (if any) under `other_launch`.  Launch
            kinds (hk_profile_kinds): 0/2 the pair kernel (both halves /
            trigger only; the homogeneous band next to the expansion is the
            generic pair kernel computing the trigger), 4 the trigger
            expansion's row evaluation."""
            if variant == "constant":
                lines = [roofline(f"constant_{n}_both", kinds_ms[0] + kinds_ms[2], fp64_peak, pairs_local,
                                  algo_bytes(variant, "both"))]
                if kinds_ms[4] > 0:
                    lines.append(roofline(f"constant_{n}_fgt_rows", kinds_ms[4], fp64_peak, pairs_local,
                                          algo_bytes(variant, "fgt_rows")))
            else:
                lines = [roofline(f"varying_{n}_trigger", kinds_ms[2], fp64_peak, pairs_local,
                                  algo_bytes(variant, "trigger"))]
            lines.sort(key=lambda r: -r["launch_ms"])
            if len(lines) > 1:
                lines[0]["other_launch"] = lines[1]
            return lines[0]

        def launches_ms(variant, kinds_ms):
            return {"pair_ms": kinds_ms[0] + kinds_ms[2], "background_ms": kinds_ms[1],
                    "fgt_moments_ms": kinds_ms[3], "fgt_rows_ms": kinds_ms[4]}

        value = args.steps / (ms_total * 1e-3)
        o_value = args.steps / (o_ms * 1e-3)
        e2e_note = ("per step: hk_set_locations from pinned host (lon, lat) + LL+grad + result read to host"
                    + ("; locations broadcast over NCCL" if world > 1 else ""))
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload(args, world),
            "pairs_per_sec": value * pairs,
            "e2e": {"value": args.steps / e2e_s, "unit": "evals/s", "h2d_bytes_per_step": 2 * n * 8,
                    "d2h_bytes_per_step": 6 * 8, "note": e2e_note},
            "gpu_launches": launches,
            "launches_ms": launches_ms(args.variant, kinds),
            "roofline": pair_line(args.variant, kinds),
            "cpu_baseline": cpu(int(p_main.variant)),
            "clocks": clk,
            "result": {"loglik": ll, "grad": [float(x) for x in g]},
            ("density_scaled" if other == "varying" else "homogeneous"): {
                "note": f"BASELINE config {4 if other == 'varying' else 3}: the same LL+grad step with the "
                        f"{other} kernel on the same catalog, measured like the headline (device-timed "
                        f"`value`, `e2e` through the public API, roofline of its dominant pair launch)",
                "variant": other, "value": o_value, "unit": "evals/s", "ms_per_step": o_ms / args.steps,
                "pairs_per_sec": o_value * pairs,
                "e2e": {"value": args.steps / o_e2e_s, "unit": "evals/s", "h2d_bytes_per_step": 2 * n * 8,
                        "d2h_bytes_per_step": 6 * 8, "note": e2e_note},
                "gpu_launches": o_launches,
                "launches_ms": launches_ms(other, o_kinds),
                "roofline": pair_line(other, o_kinds),
                "cpu_baseline": cpu(int(p_other.variant)),
                "result": {"loglik": o_ll, "grad": [float(x) for x in o_g]}},
            "fgt": {"evaluations": fgt_stats[0], "direct_recomputations": fgt_stats[1],
                    "last_async_flagged": fgt_stats[2],
                    "note": "the homogeneous trigger of the tiles before each checkpoint by the certified "
                            "Hermite expansion (hk_fgt.cu); certification failures recompute directly"},
            "direct_kernel": {
                "note": "one homogeneous LL+grad evaluation with the background block expansion and the "
                        "trigger's Hermite expansion disabled: every ordered pair evaluated directly",
                "ms_per_step": d_ms, "pair_both_ms": d_kinds[0],
                "note2": "both Hermite expansions and the background block expansion off",
                "roofline": roofline(f"direct_{n}_both", d_kinds[0], fp64_peak, pairs_local,
                                     algo_bytes("constant", "both"))},
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
