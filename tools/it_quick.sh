# quick iteration: parity (fast subset) + bench lines for c2/c4/c3
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "c1_shape or shapes or full_c2 or full_c4 or batch_homo" 2>&1 | tail -3
for c in ${CONFIGS:-c2 c4 c3}; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c; done
