export PYTHONUNBUFFERED=1
for round in 1 2 3; do
  for v in base "$@"; do
    for c in ${CFGS:-c2 c4 c5}; do
      if [ $v = base ]; then unset FC_LIB_VARIANT; else export FC_LIB_VARIANT=$v; fi
      echo -n "$v $c: "
      timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c | cut -d' ' -f5-10
    done
  done
done
