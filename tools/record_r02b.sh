# Round-2 evidence for the current default (mma.sync) kernel: full GPU test suite, smoke,
# bench lines (all configs + reference arm), ncu launch lists, full captures of c2/c4,
# virtual-rank latencies, sanitizers.  (The tcgen05 evidence of record_r02.sh is unchanged.)
export PYTHONUNBUFFERED=1
tag=${1:-r02b}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $out/gpu.txt
timeout 1200 python -m pytest tests/ -q -m gpu 2>&1 | tail -5 > $out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/smoke.txt 2>&1
timeout 600 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err
for c in c1 c3 c4 c5; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $out/bench_$c.json 2>/dev/null; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $out/ncu_launches_c2.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $out/ncu_launches_c1.csv python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fc_fused -s 3 -c 1 -o $out/ncu_full_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fc_fused -s 3 -c 1 -o $out/ncu_full_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for c in c2 c3 c4; do timeout 200 python tools/virtual_ranks.py $c 20 >> $out/virtual_ranks.jsonl 2>/dev/null; done
bash tools/sanitize.sh > $out/sanitizer_summary.txt 2>&1
cp -r gpurun_out/san $out/ 2>/dev/null
ls -la $out
