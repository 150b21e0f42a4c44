# Round evidence: parity tests, smoke, bench (all configs), ncu launch list + full capture of c2.
export PYTHONUNBUFFERED=1
tag=${1:-r01}
mkdir -p gpurun_out/$tag
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/$tag/gpu.txt
timeout 900 python -m pytest tests/ -q -m gpu 2>&1 | tail -5 > gpurun_out/$tag/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/$tag/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/$tag/bench_c2.json 2> gpurun_out/$tag/bench_c2.err
for c in c1 c3 c4 c5; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/$tag/bench_$c.json 2>/dev/null; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/$tag/bench_ref.json 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/$tag/ncu_launches_c2.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fc_fused -s 3 -c 1 -o gpurun_out/$tag/ncu_full_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fc_fused -s 3 -c 1 -o gpurun_out/$tag/ncu_full_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/$tag
