export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu 2>&1 | tail -15
for c in c2 c4 c3 c1; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print('$c', 'frames/s', d['value'], 'ms', d['ms_per_step'], 'kern', d['config']['kernel_ms_avg'], 'GB/s', d['roofline']['achieved'], 'frac', d['roofline']['frac'])"; done
