export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -m gpu 2>&1 | tail -6
for c in c2 c3 c5 c4; do timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | python tools/brief.py $c; done
