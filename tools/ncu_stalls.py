"""Per-source-line stall reasons from an ncu report (--import-source on).
usage: python tools/ncu_stalls.py rep.ncu-rep file.cuh lo hi [top]
Prints, for source lines lo..hi of `file`, instructions executed, samples and
the top stall reasons."""
import csv, io, subprocess, sys
from collections import defaultdict

rep, fname, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, f, line = None, None, None
agg = defaultdict(lambda: defaultdict(float))
src = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    if f != fname or not (lo <= ln <= hi):
        continue
    src[ln] = r[1][:80]
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h or h in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
            try:
                agg[ln][h] += float(r[i] or 0)
            except ValueError:
                pass
rows = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]
for ln, d in rows:
    st = sorted(((v, k[6:]) for k, v in d.items() if k.startswith("stall_") and v > 0), reverse=True)[:4]
    print(f"{fname}:{ln:4d} inst {d['Instructions Executed']:>11.0f} samp {d['Warp Stall Sampling (All Samples)']:>6.0f}  "
          + " ".join(f"{k}={v:.0f}" for v, k in st) + f"   | {src[ln]}")
