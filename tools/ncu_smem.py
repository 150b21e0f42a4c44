"""Shared-memory wavefronts per source line (excessive = bank-conflict replays) from an ncu report.
usage: python tools/ncu_smem.py rep.ncu-rep [top]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, f = None, None
agg = defaultdict(lambda: [0.0, 0.0, ""])
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Name": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None: continue
    try: ln = int(r[0])
    except ValueError: continue
    d = dict(zip(hdr, r))
    try:
        ex = float(d.get("L1 Wavefronts Shared Excessive") or 0); tot = float(d.get("L1 Wavefronts Shared") or 0)
    except ValueError: continue
    if tot:
        a = agg[(f, ln)]; a[0] += tot; a[1] += ex; a[2] = r[1][:70]
T = sum(v[0] for v in agg.values()); E = sum(v[1] for v in agg.values())
print(f"total shared wavefronts {T:.0f}, excessive {E:.0f}")
for (f, ln), (tot, ex, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{f}:{ln:4d} wavefronts {tot:>11.0f} excessive {ex:>10.0f}  | {src}")
