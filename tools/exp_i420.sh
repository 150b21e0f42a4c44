export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -m pytest tests/test_parity_gpu.py -q -m gpu -k i420 2>&1 | tail -2
for c in c2 c4 c5; do for sf in nv12 i420; do echo -n "$sf $c: "; timeout 300 python bench.py --config $c --surface $sf --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c | cut -d' ' -f2-20; done; done
python -c "import __graft_entry__ as g; g.smoke()"
