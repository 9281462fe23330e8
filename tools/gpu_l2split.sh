#!/bin/bash
# L2 sector breakdown (read / write / red / atom, from the SMs vs everything) of the
# whole-epoch K1s launch in both orders (tools/ncu_probe.py), per trained word.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
M=gpu__time_duration.sum,lts__t_sectors.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_requests_op_red.sum,lts__d_sectors.sum,lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum
for mode in window_snapshot lifetime; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:k1s -s 1 -c 1 --csv python tools/ncu_probe.py $mode 20000 128 1 > gpurun_out/l2split_$mode.csv 2>/dev/null
  python - gpurun_out/l2split_$mode.csv $mode <<'PY'
import csv, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.DictReader(lines))
W = 9897591.0
print("==", sys.argv[2], rows[0]["Kernel Name"][:60] if rows else "?")
for r in rows:
    v = float(r["Metric Value"].replace(",", ""))
    n, u = r["Metric Name"], r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u)
    extra = f"  ({32 * v / W:.0f} B/word)" if u == "sector" else (f"  ({v * scale / W:.0f} B/word)" if scale else "")
    print(f"  {n:75s} {v:16.1f} {u}{extra}")
PY
done
