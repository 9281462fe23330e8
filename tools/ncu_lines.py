"""Per-source-line instruction counts and stall samples from an ncu report.
usage: python tools/ncu_lines.py <rep> <words> [n]"""
import collections, csv, io, subprocess, sys

rep, W = sys.argv[1], float(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout)))
f = None; cur = None; inst = collections.Counter(); stall = collections.Counter(); src = {}
ops = collections.defaultdict(collections.Counter); sreason = collections.defaultdict(collections.Counter)
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if len(r) < 8 or hdr is None:
        continue
    if r[0]:
        cur = (f, int(r[0])); src[cur] = r[1].strip(); continue
    if not r[2] or cur is None:
        continue
    try:
        ni = float(r[7] or 0); ns = float(r[4] or 0)
    except ValueError:
        continue
    inst[cur] += ni; stall[cur] += ns
    o = r[3].strip().split()
    if o:
        m = o[1] if o[0].startswith("@") else o[0]
        ops[cur][m.split(".")[0]] += ni
    for k, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name:
            try:
                sreason[cur][name[6:]] += float(r[k] or 0)
            except ValueError:
                pass
ti = sum(inst.values()); ts = sum(stall.values())
print(f"inst/word {ti / W:.1f}")
keys = sorted(set(inst) | set(stall), key=lambda k: -(stall[k] / ts + inst[k] / ti))
for k in keys[:n]:
    top = ",".join(f"{m}:{c / W:.1f}" for m, c in ops[k].most_common(3))
    rs = ",".join(f"{m}:{c / max(stall[k], 1) * 100:.0f}" for m, c in sreason[k].most_common(2))
    print(f"{inst[k] / W:6.1f}/w {stall[k] / ts * 100:5.1f}%st {k[0][:12]:12s}:{k[1]:4d} {src.get(k, '')[:60]:60s} | {top} | {rs}")
