# experiment: CTA lifetime distribution and the dynamic-tail split (FC_DYN)
export PYTHONUNBUFFERED=1
for c in c2 c4; do
  FC_CTA_TIMES=1 FC_CTA_TIMES_FILE=gpurun_out/cta_$c.txt timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep "fc cta" | tail -2
  FC_DYN=0.85 FC_CTA_TIMES=1 timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep "fc cta" | tail -2
done
FC_DYN=0.85 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "c1_shape or shapes or full_c2 or full_c4 or batch or paged or graph" 2>&1 | tail -2
for round in 1 2; do
for v in "" 0.9 0.8 0.7; do
  for gr in 2 4; do
    [ -z "$v" ] && [ $gr = 4 ] && continue
    for c in c2 c4; do
      echo -n "dyn=$v grain=$gr $c: "
      FC_DYN=$v FC_DYN_GRAIN=$gr timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c | cut -c1-150
    done
  done
done
done
