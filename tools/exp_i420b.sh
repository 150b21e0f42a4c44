export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -2
bash tools/sanitize.sh
for r in 1 2; do for c in c2 c4 c5; do for sf in nv12 i420; do echo -n "$sf $c: "; timeout 300 python bench.py --config $c --surface $sf --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c | cut -d' ' -f2-20; done; done; done
