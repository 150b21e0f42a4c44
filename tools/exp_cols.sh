export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -2
for c in c2 c4 c1; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c | cut -d' ' -f2-20; done
