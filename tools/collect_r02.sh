# Copy the round-2 evidence (gpurun_out/r02, from tools/record_r02.sh) into profiles/.
set -e
tag=${1:-r02}
src=gpurun_out/$tag
for f in bench_c1 bench_c2 bench_c3 bench_c4 bench_c5 bench_ref bench_tc_c2 bench_tc_c3 bench_tc_c4 bench_tc_c5; do
  cp $src/$f.json profiles/${tag}_$f.json
done
cp $src/ncu_launches_c2.csv profiles/${tag}_ncu_launches_c2.csv
cp $src/ncu_launches_c1.csv profiles/${tag}_ncu_launches_c1.csv
cp $src/pytest_gpu.txt profiles/${tag}_pytest_gpu.txt
cp $src/smoke.txt profiles/${tag}_smoke.txt
cp $src/gpu.txt profiles/${tag}_gpu.txt
cp $src/tc_prof_c2.txt profiles/${tag}_tc_prof_c2.txt
cp $src/virtual_ranks.jsonl profiles/${tag}_virtual_ranks.jsonl
for b in tc05 tc05b tc05e tmem; do cp $src/ubench_$b.txt profiles/${tag}_ubench_$b.txt; done
{ cat $src/sanitizer_summary.txt; for t in memcheck racecheck synccheck initcheck racecheck_all; do echo "== $t"; tail -3 $src/san/$t.txt; done; } > profiles/${tag}_sanitizer.txt
for c in c2 c4 tc_c2; do
  python tools/ncu_summary.py $src/ncu_full_$c.ncu-rep > profiles/${tag}_ncu_full_${c}_summary.txt
  python tools/ncu_lines.py $src/ncu_full_$c.ncu-rep 40 > profiles/${tag}_ncu_full_${c}_lines.txt
  ncu -i $src/ncu_full_$c.ncu-rep --page details --csv > profiles/${tag}_ncu_full_${c}_details.csv
done
python - "$tag" <<'PY'
import csv, io, json, subprocess, sys
tag = sys.argv[1]
out = {}
for c, bench in (("c2", "bench_c2"), ("c4", "bench_c4"), ("tc_c2", "bench_tc_c2")):
    rep = f"gpurun_out/{tag}/ncu_full_{c}.ncu-rep"
    raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                     capture_output=True, text=True).stdout)))
    h, v, u = raw[0], raw[2], raw[1]
    def get(n):
        x = float(v[h.index(n)].replace(",", ""))
        unit = u[h.index(n)]
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    b = json.loads(open(f"gpurun_out/{tag}/{bench}.json").read().strip().splitlines()[-1])
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    out[c] = {"dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
              "warp_instructions_per_launch": get("smsp__inst_executed.sum"),
              "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
              "algorithmic_bytes_per_launch": b["roofline"]["algorithmic_bytes_per_launch"],
              "kernel_us_under_ncu": get("gpu__time_duration.sum") / (1e3 if u[h.index("gpu__time_duration.sum")] == "nsecond" else 1),
              "source": f"profiles/{tag}_ncu_full_{c}_summary.txt (ncu --set full --clock-control none, 1 launch)"}
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
PY
