set -x
export PYTHONUNBUFFERED=1
for c in c2 c1 c3 c4; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 $( [ $c != c2 ] && echo --no-cpu-baseline ) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; cat gpurun_out/bench_$c.json; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fc_fused -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_c2.log 2>&1
tail -3 gpurun_out/ncu_full_c2.log
ls -la gpurun_out
