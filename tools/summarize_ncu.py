"""Summarises ncu outputs from gpurun_out/ into profiles/ (tracked).

    python tools/summarize_ncu.py ROUND [--full REP ...] [--launches CSV] [--tag TAG]

Writes profiles/rROUND_pair_kernel_ncu.json (+ .md) with the metrics the
roofline and DESIGN.md cite, and profiles/rROUND_launches.md with each
kernel's share of the launch list.
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", 1e-9),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", 1),
    "alu_pipe_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    "fma_pipe_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    "lsu_pipe_pct": ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    "xu_pipe_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    "tma_pipe_pct": ("sm__inst_executed_pipe_tma.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "inst_executed": ("smsp__inst_executed.sum", 1),
    "shared_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
}
STALLS = ["math_pipe_throttle", "not_selected", "wait", "dispatch_stall", "short_scoreboard",
          "long_scoreboard", "barrier", "branch_resolving", "mio_throttle", "no_instruction"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        res.append(d)
    return res


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def summarize_full(rep, tag):
    out = []
    for d in raw(rep):
        s = {"kernel": d.get("Kernel Name"), "grid": d.get("Grid Size"), "block": d.get("Block Size"),
             "report": Path(rep).name, "tag": tag}
        for k, (m, scale) in KEYS.items():
            v = num(d.get(m))
            if v is not None:
                u = d["_units"].get(m, "")
                if k == "duration_ms":
                    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "s": 1e3, "ms": 1.0, "us": 1e-3, "ns": 1e-6}.get(u, scale)
                if k in ("dram_read_bytes", "dram_write_bytes"):
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                if k == "sm_clock_ghz":
                    scale = {"hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0}.get(u, scale)
                s[k] = v * scale
        st = {}
        for name in STALLS:
            v = num(d.get(f"smsp__average_warps_issue_stalled_{name}_per_issue_active.ratio"))
            if v is not None:
                st[name] = round(v, 3)
        s["stalls_per_issue"] = st
        if "dram_read_bytes" in s and "dram_write_bytes" in s:
            s["dram_bytes"] = s["dram_read_bytes"] + s["dram_write_bytes"]
        if "inst_executed" in s and "fp64_pipe_pct" in s:
            pass
        out.append(s)
    return out


def summarize_launches(path):
    text = Path(path).read_text()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
        name = r[ki].split("(")[0].replace("void ", "").strip()
        tot[name] += num(r[vi]) * scale
        cnt[name] += 1
    allms = sum(tot.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k}` | {cnt[k]} | {v:.3f} | {100 * v / allms:.2f}% |")
    return "\n".join(lines), {k: {"launches": cnt[k], "ms": tot[k], "share": tot[k] / allms} for k in tot}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("round")
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--tags", nargs="*", default=[])
    ap.add_argument("--launches")
    ap.add_argument("--pairs", nargs="*", type=float, default=[])
    a = ap.parse_args()
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    if a.full:
        summ = {"captures": [], "dram_bytes_per_launch": {}}
        for i, rep in enumerate(a.full):
            tag = a.tags[i] if i < len(a.tags) else Path(rep).stem
            for s in summarize_full(rep, tag):
                if i < len(a.pairs) and a.pairs[i] and s.get("inst_executed"):
                    s["pairs_per_launch"] = a.pairs[i]
                summ["captures"].append(s)
                if "dram_bytes" in s:
                    summ["dram_bytes_per_launch"][tag] = s["dram_bytes"]
        (prof / f"r{a.round}_pair_kernel_ncu.json").write_text(json.dumps(summ, indent=1))
        print(json.dumps(summ, indent=1))
    if a.launches:
        md, d = summarize_launches(a.launches)
        (prof / f"r{a.round}_launches.md").write_text(
            f"# Kernel launch list (ncu --metrics gpu__time_duration.sum --clock-control none)\n\n"
            f"Command: `python bench.py --steps 2 --warmup 1` (N=1e6, constant, LL+grad).  Times are\n"
            f"cold-cache and serialised under ncu: compare shares, not absolutes.\n\n{md}\n")
        print(md)
