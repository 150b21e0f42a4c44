# tcgen05 kernel iteration: parity subset (tc path), then c2..c5 bench lines tc vs legacy
export PYTHONUNBUFFERED=1
export FC_VERBOSE=${FC_VERBOSE:-}
timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "${TESTS:-c1_shape or shapes or full_c1 or full_c2 or c5_clip or batch_homo}" 2>&1 | tail -15
for c in ${CONFIGS:-c2 c4 c3 c5}; do
  for tcv in 1 0; do
    echo "== $c FC_TC=$tcv"
    FC_TC=$tcv timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c
  done
done
