"""Turns a tools/gpu_round.sh session (gpurun_out/) into the tracked
profiles/r02_* summaries the DESIGN.md and the bench line cite.

    python tools/summarize_round.py [ROUND]
"""
import csv
import io
import json
import shutil
import subprocess
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
from summarize_ncu import STALLS, summarize_full, summarize_launches  # noqa: E402

O = ROOT / "gpurun_out"


def sass_mix(rep):
    """Instruction mix (warp instructions by opcode) of a captured kernel."""
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.DictReader(out[1:]))
    tot = sum(int(r["Instructions Executed"] or 0) for r in rows) or 1
    ops = Counter()
    for r in rows:
        toks = r["Source"].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        ops[op.split(".")[0]] += int(r["Instructions Executed"] or 0)
    return {k: round(v / tot, 4) for k, v in ops.most_common(12)}, tot


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "02"
    prof = ROOT / "profiles"
    for name, dst in [("bench.json", "bench"), ("bench_ref.json", "bench_ref"), ("bench_n10000.json", "bench_n10000"),
                      ("bench_ref_n10000.json", "bench_ref_n10000"), ("bench_n100000.json", "bench_n100000"),
                      ("bench_ref_n100000.json", "bench_ref_n100000"), ("config5_gpu.json", "config5_gpu_resample"),
                      ("config5_host.json", "config5_host_resample")]:
        if (O / name).exists() and (O / name).stat().st_size:
            shutil.copy(O / name, prof / f"r{rnd}_{dst}.json")
    if (O / "ws_sweep.log").exists():
        shutil.copy(O / "ws_sweep.log", prof / f"r{rnd}_workspace_sweep.txt")
    # launch lists
    md = ["# Kernel launch lists (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
          "One N=1e6 LL+grad evaluation after one warm-up (`tools/profile_pair.py 1000000 V 1`).",
          "Times are cold-cache and serialised under ncu: compare shares, not absolutes.", ""]
    for tag, title in [("v0", "homogeneous (config 3)"), ("v1", "density-scaled, bench catalog (config 4)"),
                       ("v1county", "density-scaled, county catalog (config 5)")]:
        f = O / f"launches_{tag}.csv"
        if f.exists():
            table, _ = summarize_launches(f)
            md += [f"## {title}", "", table, ""]
    (prof / f"r{rnd}_launches.md").write_text("\n".join(md) + "\n")
    # full captures
    caps, lines = [], ["# ncu --set full captures (round " + rnd + ")", "",
                       "| capture | kernel | ms | FP64 pipe % | issue % | warps % | regs | DRAM MB | top stalls per issue |",
                       "|---|---|---|---|---|---|---|---|---|"]
    for tag in ("ncu_fgt_rows", "ncu_pair_band", "ncu_trigger", "ncu_trigger_county"):
        rep = O / f"{tag}.ncu-rep"
        if not rep.exists():
            continue
        for s in summarize_full(rep, tag):
            mix, tot = sass_mix(rep)
            s["sass_mix"] = mix
            s["warp_instructions"] = tot
            caps.append(s)
            st = sorted(s["stalls_per_issue"].items(), key=lambda kv: -kv[1])[:3]
            lines.append(f"| {tag} | `{(s['kernel'] or '')[:60]}` | {s.get('duration_ms', 0):.2f} | "
                         f"{s.get('fp64_pipe_pct', 0):.1f} | {s.get('issue_active_pct', 0):.1f} | "
                         f"{s.get('warps_active_pct', 0):.1f} | {s.get('registers_per_thread', 0):.0f} | "
                         f"{s.get('dram_bytes', 0) / 1e6:.0f} | "
                         + ", ".join(f"{k} {v}" for k, v in st) + " |")
    lines += ["", "Instruction mix (share of warp instructions by opcode):", ""]
    for s in caps:
        lines.append(f"- {s['tag']}: " + ", ".join(f"{k} {v:.3f}" for k, v in s["sass_mix"].items()))
    (prof / f"r{rnd}_kernels_ncu.json").write_text(json.dumps({"captures": caps, "stall_keys": STALLS}, indent=1))
    (prof / f"r{rnd}_kernels_ncu.md").write_text("\n".join(lines) + "\n")
    print("\n".join(md))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
