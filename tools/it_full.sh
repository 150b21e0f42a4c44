export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -m gpu 2>&1 | tail -4
for c in c2 c4; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c; done
