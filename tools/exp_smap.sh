export PYTHONUNBUFFERED=1
FC_SMAP=1 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu 2>&1 | tail -2
FC_SMAP=1 FC_VERBOSE=1 timeout 300 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | grep "fc launch" | sort -u
for round in 1 2; do
for sm in 0 1; do
  for c in c2 c4 c3 c5; do
    echo -n "smap=$sm $c: "
    FC_SMAP=$sm timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c | cut -d' ' -f5-10
  done
done
done
for sm in 0 1; do
FC_SMAP=$sm ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:fc_fused -c 2 python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep -E "dram__|gpu__time|issue_active" | tail -4
done
