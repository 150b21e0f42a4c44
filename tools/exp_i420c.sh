export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -2
CFGS="c2 c4 c5" bash tools/exp_ab.sh noi420
for c in c2 c5; do echo -n "i420 $c: "; timeout 300 python bench.py --config $c --surface i420 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c | cut -d' ' -f2-20; done
