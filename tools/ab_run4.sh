# A/B on c4 only: parity (c4 + wide-window shapes) for the variant, then interleaved bench
export PYTHONUNBUFFERED=1
v=$1
FC_LIB_VARIANT=$v timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "full_c4 or shapes or 8k or i420" 2>&1 | tail -2
for round in 1 2 3; do for x in base $v; do
  if [ $x = base ]; then unset FC_LIB_VARIANT; else export FC_LIB_VARIANT=$x; fi
  timeout 300 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py "$x/c4" | cut -d' ' -f1-8
done; done
