export PYTHONUNBUFFERED=1
for i in 1 2 3 4; do FC_BENCH_STEPS=1 timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | grep -v "^{" | cut -c1-400; done
for i in 1 2; do timeout 300 python bench.py --config c3 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py c3 | cut -d' ' -f5-10; done
