"""Summarise an ncu report: key metrics, stall reasons, per-opcode and hot-region SASS counts."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]

def page(args):
    out = subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))

raw = page(["--page", "raw", "--csv"])
h, v = raw[0], raw[2] if len(raw) > 2 else raw[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for n in want:
    if n in h:
        print(f"{n:70s} {v[h.index(n)]:>16s} {raw[1][h.index(n)]}")
st = []
for i, n in enumerate(h):
    if n.startswith("smsp__average_warps_issue_stalled") and n.endswith("per_issue_active.ratio"):
        try:
            st.append((float(v[i]), n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
print("stalls:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
rows = page(["--page", "source", "--csv", "--print-source", "sass"])
hh = rows[1]
iA, iS, iE, iW = hh.index("Address"), hh.index("Source"), hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)")
byop = collections.Counter(); seq = []
tot = 0
for r in rows[2:]:
    try:
        n = int(r[iE] or 0)
    except ValueError:
        continue
    t = r[iS].split()
    op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "")).split(".")[0]
    byop[op] += n; tot += n
    seq.append((r[iA], r[iS], n, int(r[iW] or 0)))
print("total warp-instructions", tot)
print("  ".join(f"{op} {n/tot*100:.1f}%" for op, n in byop.most_common(16)))
blocks = []; cur = None; start = 0
for i, (a, s, n, w) in enumerate(seq + [("", "", -1, 0)]):
    if n != cur:
        if cur is not None and cur > 0:
            blocks.append((cur * (i - start), cur, i - start, seq[start][0], seq[i - 1][0], sum(x[3] for x in seq[start:i])))
        cur, start = n, i
blocks.sort(reverse=True)
print("hot straight-line regions: total_instr, exec_count, length, start, end, stall_samples")
for b in blocks[:12]:
    print("  ", b)
if len(sys.argv) > 2:
    lo, hi = sys.argv[2], sys.argv[3]
    on = False
    for a, s, n, w in seq:
        if a.endswith(lo): on = True
        if on: print(a[-5:], n, w, s)
        if a.endswith(hi): break
