# round-2 re-entry baseline: GPU parity subset + bench lines (c2, c4, c3) + geometry
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "c1_shape or shapes or full_c2 or full_c4" 2>&1 | tail -3
for c in c2 c4 c3 c5; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c; done
FC_VERBOSE=1 timeout 300 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep "^fc launch" | sort -u | head -3
