export PYTHONUNBUFFERED=1
FC_LIB_VARIANT=v20 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu 2>&1 | tail -2
FC_LIB_VARIANT=v20 FC_VERBOSE=1 timeout 300 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | grep "fc launch" | sort -u
for round in 1 2 3; do
  for v in base v20; do
    for c in c2 c4 c3 c5; do
      if [ $v = base ]; then unset FC_LIB_VARIANT; else export FC_LIB_VARIANT=$v; fi
      echo -n "$v $c: "
      timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c | cut -d' ' -f5-10
    done
  done
done
