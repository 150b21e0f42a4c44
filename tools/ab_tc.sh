export PYTHONUNBUFFERED=1
export FC_TC=1
for round in 1 2; do
  for v in base lay0; do
    for c in c2 c3; do
      if [ "$v" = base ]; then unset FC_LIB_VARIANT; else export FC_LIB_VARIANT=$v; fi
      timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py "$v/$c" | cut -d' ' -f1-8
    done
  done
done
