"""Quick look at an ncu --set full report: key metrics, stall reasons, SASS opcode mix.
usage: python tools/ncu_quick.py <rep.ncu-rep> [words_in_launch]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
words = float(sys.argv[2]) if len(sys.argv) > 2 else 0
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))
d = {k: (v, u) for k, u, v in zip(raw[0], raw[1], raw[2])}
keys = """gpu__time_duration.sum sm__cycles_elapsed.avg.per_second launch__grid_size launch__block_size launch__registers_per_thread
launch__occupancy_limit_registers launch__occupancy_limit_shared_mem sm__warps_active.avg.pct_of_peak_sustained_active
smsp__issue_active.avg.pct_of_peak_sustained_active smsp__inst_executed.sum sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active
lts__throughput.avg.pct_of_peak_sustained_elapsed lts__t_sectors.sum lts__t_sector_hit_rate.pct
l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
l1tex__data_pipe_lsu_wavefronts_mem_shared.sum dram__bytes_read.sum dram__bytes_write.sum""".split()
for k in keys:
    print(f"{k:70s}", *d.get(k, ("-", "")))
for k, (v, u) in d.items():
    if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
        try:
            if float(v) > 0.05:
                print(f"  {k.replace('smsp__average_warps_issue_stalled_', ''):60s} {v}")
        except ValueError:
            pass
src = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout)))
hi = next(i for i, r in enumerate(src[:5]) if "Source" in r)
h = src[hi]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
op = collections.Counter(); stall = collections.Counter(); tot = 0; stot = 0
rows = []
for r in src[hi + 1:]:
    try:
        n = float(r[iE] or 0); w = float(r[iW] or 0)
    except ValueError:
        continue
    o = r[iS].strip().split()
    if not o:
        continue
    m = o[1] if o[0].startswith("@") else o[0]
    m = m.split(".")[0]
    op[m] += n; tot += n; stall[m] += w; stot += w
    rows.append((w, r[iS].strip()))
print("total inst", tot, "per word", tot / words if words else "")
for m, n in op.most_common(30):
    print(f"  {m:10s} {n:14.0f} {n / tot * 100:5.1f}%  {n / words if words else 0:7.1f}/word  stall {stall[m] / stot * 100:5.1f}%")
print("top stall sites")
for w, s in sorted(rows, reverse=True)[:15]:
    print(f"  {w / stot * 100:5.1f}%  {s[:110]}")
