"""Per-source-line warp instructions and stall samples from an ncu report
(--import-source on).  usage: python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, f = [], None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")])
        ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    rows.append((ie, ss, f, r[0], r[1][:90]))
tot_i = sum(r[0] for r in rows) or 1
tot_s = sum(r[1] for r in rows) or 1
print(f"total warp instructions {tot_i:,}  stall samples {tot_s:,}")
for ie, ss, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*ie/tot_i:5.1f}% inst {100*ss/tot_s:5.1f}% samp  {f}:{ln:5s} {src}")
