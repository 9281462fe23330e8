"""Summarise ncu captures into profiles/ (run here, on the CPU box).

usage: python tools/ncu_summary.py <full.ncu-rep> <launches.csv> <tag>

Writes profiles/<tag>_k1s_full.txt (key metrics + top stall sites),
profiles/<tag>_launches.txt (per-kernel share of device time) and
profiles/ncu_k1s_summary.json (dram bytes per launch etc., read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def main():
    rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    out_dir = os.path.join(ROOT, "profiles")
    os.makedirs(out_dir, exist_ok=True)

    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    d = dict(zip(hdr, vals))

    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
             "ms": 1e6, "msecond": 1e6, "nsecond": 1}

    def num(k):
        """Value in base units (bytes, ns)."""
        v = d.get(k, "")
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            return None
        return x * scale.get(units[hdr.index(k)], 1)

    keys = [
        "Kernel Name", "Grid Size", "Block Size", "launch__registers_per_thread", "gpu__time_duration.sum",
        "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
    ]
    lines = [f"# ncu --set full --clock-control none, one K1s launch ({tag})"]
    for k in keys:
        if k in d:
            u = units[hdr.index(k)] if k in hdr else ""
            lines.append(f"{k:75s} {d[k]} {u}")

    src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass"))))
    shdr, sdata = src[1], src[2:]
    isrc, iss = shdr.index("Source"), shdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[iss] or 0) for r in sdata) or 1.0
    lines.append("\n# top stall sites (share of warp-stall samples)")
    for r in sorted(sdata, key=lambda r: -float(r[iss] or 0))[:12]:
        lines.append(f"{float(r[iss] or 0) / tot * 100:6.1f}%  {r[isrc].strip()[:100]}")
    with open(os.path.join(out_dir, f"{tag}_k1s_full.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")

    # launch list: share of device time per kernel
    per = defaultdict(lambda: [0, 0.0])
    with open(launches) as f:
        rows = [r for r in csv.reader(f) if len(r) > 10]
    h = rows[0]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        per[name][0] += 1
        per[name][1] += float(r[iv].replace(",", ""))
    total = sum(v[1] for v in per.values()) or 1.0
    with open(os.path.join(out_dir, f"{tag}_launches.txt"), "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold-cache) ({tag})\n")
        f.write(f"{'kernel':70s} {'launches':>8s} {'total_ns':>14s} {'share':>7s}\n")
        for name, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{name[:70]:70s} {n:8d} {t:14.0f} {t / total * 100:6.1f}%\n")

    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    summary = {
        "tag": tag,
        "kernel": d.get("Kernel Name"),
        "duration_ns": num("gpu__time_duration.sum"),
        "dram_bytes_read": rd,
        "dram_bytes_write": wr,
        "dram_bytes_per_launch": (rd or 0) + (wr or 0),
        "registers_per_thread": num("launch__registers_per_thread"),
        "grid": d.get("Grid Size"),
        "note": "one launch = the whole text8-shaped epoch as one batch (tools/ncu_probe.py window_snapshot 20000 128 1: 16,719 sentences, 9.9M trained words)",
        "words_per_launch": 9897591,
    }
    with open(os.path.join(out_dir, "ncu_k1s_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print("\n".join(lines[:30]))


if __name__ == "__main__":
    main()
