export PYTHONUNBUFFERED=1
FC_LIB_VARIANT=v18 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu 2>&1 | tail -2
for round in 1 2 3; do
  for v in base v18 v18s0; do
    for c in c2 c4 c3 c5; do
      case $v in base) unset FC_LIB_VARIANT; unset FC_SMAP;; v18) export FC_LIB_VARIANT=v18; unset FC_SMAP;; v18s0) export FC_LIB_VARIANT=v18; export FC_SMAP=0;; esac
      echo -n "$v $c: "
      timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c | cut -d' ' -f5-10
    done
  done
done
