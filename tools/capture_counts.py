"""Per-launch FP64-pipe instruction counts and DRAM traffic of the pair
kernels at the bench workloads, from ncu, into profiles/r02_fp64_counts.json
(read by bench.py for roofline.achieved / traffic).

    python tools/capture_counts.py [N]          # runs ncu on itself (GPU box)

The counts are deterministic for a (build, catalog, params): the file
records the library's sha256 prefix and bench.py flags a stale capture.
Workloads (benchmark_catalog(N, 42), bench params, LL + gradient):
  constant  the homogeneous evaluation: one pair launch computing both halves
  varying   the density-scaled evaluation: a background-only launch of the
            homogeneous kernel + the trigger-only density-scaled launch
  direct    constant with the background block expansion and the trigger's
            Hermite expansion off (the pure O(N^2) pair kernel)
"""
import csv
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
OUT = ROOT / "profiles" / "r02_fp64_counts.json"
METRICS = ["gpu__time_duration.sum", "sm__inst_executed_pipe_fp64.sum",
           "sm__thread_inst_executed_pipe_fp64_pred_on.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__cycles_active.avg",
           "sm__cycles_elapsed.avg.per_second"]


def worker(n, mode):
    from paper_2407_11349_b200 import Evaluator, HawkesParams, Variant, benchmark_catalog
    ev = Evaluator(benchmark_catalog(n, 42))
    p = HawkesParams(mu0=1.0, tau_t=5.0, xi0=0.5, sigma_x=0.5, sigma_t=2.0, area=100.0,
                     variant=Variant.varying if mode == "varying" else Variant.constant)
    if mode == "direct":
        ev.set_bg_expansion(False)
        ev.set_fgt(False)
        ev.set_bg_fgt(False)
    ev.eval(p, grad=True)


def kind_of(name):
    if "bg_fgt_" in name:  # the background's 1-D expansion (hk_fgt.cu)
        return "bg_" + name.split("bg_fgt_", 1)[1].split("_kernel", 1)[0]
    if "fgt_" in name:  # the trigger's Hermite expansion (hk_fgt.cu)
        base = name.split("fgt_", 1)[1].split("_kernel", 1)[0]
        return {"eval": "fgt_rows"}.get(base, "fgt_" + base)
    # pair_kernel<kVarying, kGrad, kMode, kF32, kOnly>
    args = name.split("pair_kernel<", 1)[1].split(">", 1)[0].split(",")
    only = int(args[4]) if len(args) > 4 else 0
    return {0: "both", 1: "bg", 2: "trigger"}[only]


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--worker":
        worker(int(sys.argv[2]), sys.argv[3])
        return
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    sys.path.insert(0, str(ROOT))
    from bench import source_sha  # noqa: E402
    out = {"src_sha16": source_sha(), "metrics": METRICS, "launches": {}}
    log = ROOT / "gpurun_out"
    log.mkdir(exist_ok=True)
    for mode in ("constant", "varying", "direct"):
        csv_path = log / f"counts_{mode}.csv"
        subprocess.run(["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "--print-units", "base", "-k",
                        "regex:pair_kernel|fgt_", "--csv", "--log-file", str(csv_path), sys.executable, __file__,
                        "--worker", str(n), mode], check=True, cwd=ROOT)
        rows = [r for r in csv.DictReader(l for l in csv_path.read_text().splitlines()
                                          if l.startswith('"'))]
        per = {}
        for r in rows:
            per.setdefault((r["ID"], r["Kernel Name"]), {})[r["Metric Name"]] = float(
                r["Metric Value"].replace(",", ""))
        for (_, name), m in per.items():
            kind = kind_of(name)
            tag = f"{mode}_{n}_{kind}"
            out["launches"][tag] = {
                "kernel": name, "duration_ms": m["gpu__time_duration.sum"] * 1e-6,
                "fp64_warp_inst": m["sm__inst_executed_pipe_fp64.sum"],
                "fp64_thread_inst_pred_on": m["sm__thread_inst_executed_pipe_fp64_pred_on.sum"],
                "dram_bytes": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
                "dram_read_bytes": m["dram__bytes_read.sum"], "dram_write_bytes": m["dram__bytes_write.sum"],
                "fp64_pipe_pct": m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
                "sm_clock_hz": m["sm__cycles_elapsed.avg.per_second"]}
    # algorithmic bytes of the expansion's row launch: every checkpoint's
    # prefix moments once (A and B sets, kFgtP^2 each, per box)
    import math
    from paper_2407_11349_b200 import benchmark_catalog
    cat = benchmark_catalog(n, 42)
    extent = max(cat.lon.max() - cat.lon.min(), cat.lat.max() - cat.lat.min())
    nb = max(1, math.ceil(extent / (math.sqrt(2.0) * math.sqrt(2.0) * 0.5)))
    nck = math.ceil(math.ceil(n / 512) / 4)
    for tag, c in out["launches"].items():
        if tag.endswith("_fgt_rows"):
            c["moment_bytes"] = nck * nb * nb * 2 * 30 * 30 * 8
    OUT.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
