export PYTHONUNBUFFERED=1
FC_DYN=0 FC_DYN_DIV=2 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "c1_shape or shapes or full_c2 or full_c4 or batch or paged or graph" 2>&1 | tail -2
FC_DYN=0 FC_DYN_DIV=2 FC_CTA_TIMES=1 timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep "fc cta" | tail -1
FC_DYN=0.5 FC_DYN_GRAIN=4 FC_CTA_TIMES=1 timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep "fc cta" | tail -1
for round in 1 2; do
for cfg in "-1 2 0" "0.7 4 0" "0.5 4 0" "0.5 2 2" "0.25 4 0" "0.25 2 2" "0 4 0" "0 2 2" "0 3 3" "0 8 0"; do
  set -- $cfg
  for c in c2 c4 c3; do
    echo -n "dyn=$1 grain=$2 div=$3 $c: "
    FC_DYN=$1 FC_DYN_GRAIN=$2 FC_DYN_DIV=$3 timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c | cut -d' ' -f5-10
  done
done
done
