# Copy gpurun_out/r02b (tools/record_r02b.sh) into profiles/ as the round-2 evidence of the
# default kernel (r02_*; the tcgen05 files r02_*tc* stay as recorded by record_r02.sh).
set -e
src=gpurun_out/${1:-r02b}
tag=r02
for f in bench_c1 bench_c2 bench_c3 bench_c4 bench_c5 bench_ref; do cp $src/$f.json profiles/${tag}_$f.json; done
for f in ncu_launches_c2.csv ncu_launches_c1.csv pytest_gpu.txt smoke.txt gpu.txt virtual_ranks.jsonl; do cp $src/$f profiles/${tag}_$f; done
# (compute-sanitizer is closed on the GPU pool since round 2: r02_sanitizer.txt stays as recorded by record_r02.sh)
for c in c2 c4; do
  python tools/ncu_summary.py $src/ncu_full_$c.ncu-rep > profiles/${tag}_ncu_full_${c}_summary.txt
  python tools/ncu_lines.py $src/ncu_full_$c.ncu-rep 40 > profiles/${tag}_ncu_full_${c}_lines.txt
  python tools/ncu_stalls.py $src/ncu_full_$c.ncu-rep fc_fused.cuh 1 700 40 > profiles/${tag}_ncu_full_${c}_stalls.txt
  python tools/ncu_smem.py $src/ncu_full_$c.ncu-rep 15 > profiles/${tag}_ncu_full_${c}_smem.txt
  ncu -i $src/ncu_full_$c.ncu-rep --page details --csv > profiles/${tag}_ncu_full_${c}_details.csv
done
python - "$src" <<'PY'
import csv, io, json, subprocess, sys
src = sys.argv[1]
out = json.load(open("profiles/ncu_traffic.json"))
for c, bench in (("c2", "bench_c2"), ("c4", "bench_c4")):
    rep = f"{src}/ncu_full_{c}.ncu-rep"
    raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                     capture_output=True, text=True).stdout)))
    h, v, u = raw[0], raw[2], raw[1]
    def get(n):
        x = float(v[h.index(n)].replace(",", ""))
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[h.index(n)], 1)
    b = json.loads(open(f"{src}/{bench}.json").read().strip().splitlines()[-1])
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    out[c] = {"dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
              "warp_instructions_per_launch": get("smsp__inst_executed.sum"),
              "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
              "algorithmic_bytes_per_launch": b["roofline"]["algorithmic_bytes_per_launch"],
              "kernel_us_under_ncu": get("gpu__time_duration.sum") / (1e3 if u[h.index("gpu__time_duration.sum")] == "nsecond" else 1),
              "source": f"profiles/r02_ncu_full_{c}_summary.txt (ncu --set full --clock-control none, 1 launch)"}
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
PY
