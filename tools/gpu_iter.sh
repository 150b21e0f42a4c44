# one iteration: parity tests, bench lines for c2/c4/c3/c1, ncu full profile of c2
export PYTHONUNBUFFERED=1
tag=${1:-v}
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu 2>&1 | tail -6
for c in c2 c4 c3 c1; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c; done
bash tools/prof.sh c2 $tag
