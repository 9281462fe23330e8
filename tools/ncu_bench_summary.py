"""Summarises ncu launch lists of tools/ncu_bench_step.py into
profiles/bench_roofline.json (read by bench.py's roofline block).
usage: python tools/ncu_bench_summary.py OUT.json l2_bw.txt MODE=launches.csv:words [MODE=...]
Per mode: DRAM and L2 bytes and warp instructions per trained word summed over
every launch of the step, and the K1s share of the step's kernel time.
"""
import csv
import json
import sys


def parse(path):
    rows = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        key = (r["ID"], r["Kernel Name"])
        v = r["Metric Value"].replace(",", "")
        try:
            rows.setdefault(key, {})[r["Metric Name"]] = (float(v), r["Metric Unit"])
        except ValueError:
            pass
    return rows


def to_bytes(v, unit):
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def to_ns(v, unit):
    return v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)


def main():
    out_path, l2_path = sys.argv[1], sys.argv[2]
    res = {"source": "ncu launch lists of one bench step (tools/ncu_bench_step.py; --metrics "
                     "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,"
                     "smsp__inst_executed.sum; serialised replay: per-launch bytes/instructions are exact, "
                     "times are not the concurrent step's)"}
    with open(l2_path) as f:
        l2 = [json.loads(ln) for ln in f if ln.startswith("{")]
    best = max((x["GBps"] for x in l2 if x["kind"] == "read"), default=None)
    res["l2_peak_gbs"] = best
    res["l2_peak_source"] = "measured: tools/l2_bw.cu L2-resident 128-bit reads, best buffer size (profiles/r02_l2_bw.txt)"
    res["issue_peak"] = 148 * 4 * 1.965e9
    res["issue_peak_source"] = "148 SMs x 4 schedulers x 1 warp-instruction/clock x 1965 MHz"
    for arg in sys.argv[3:]:
        mode, rest = arg.split("=", 1)
        path, words = rest.rsplit(":", 1)
        words = float(words)
        rows = parse(path)
        dram = l2 = inst = t_all = t_k1s = 0.0
        n_k1s = 0
        for (_, name), m in rows.items():
            if "k_hot_live" in name:  # the live merge runs beside the step; serialised it only spins
                continue
            t = to_ns(*m["gpu__time_duration.sum"]) if "gpu__time_duration.sum" in m else 0.0
            t_all += t
            if "k1s" in name:
                t_k1s += t
                n_k1s += 1
            dram += sum(to_bytes(*m[k]) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in m)
            if "lts__t_sectors.sum" in m:
                l2 += 32 * m["lts__t_sectors.sum"][0]
            if "smsp__inst_executed.sum" in m:
                inst += m["smsp__inst_executed.sum"][0]
        res[mode] = {"launches": len(rows), "k1s_launches": n_k1s, "words": words,
                     "dram_bytes_per_word": dram / words, "l2_bytes_per_word": l2 / words,
                     "inst_per_word": inst / words, "k1s_time_share": t_k1s / t_all if t_all else None,
                     "serialised_kernel_ms": t_all / 1e6}
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
