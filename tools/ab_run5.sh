# c4-only interleaved bench of base and variants (no parity)
export PYTHONUNBUFFERED=1
for round in 1 2 3; do for x in base "$@"; do
  if [ $x = base ]; then unset FC_LIB_VARIANT; else export FC_LIB_VARIANT=$x; fi
  timeout 300 python bench.py --config ${CFG:-c4} --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py "$x/${CFG:-c4}" | cut -d' ' -f1-8
done; done
