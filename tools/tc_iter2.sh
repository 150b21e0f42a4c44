# tcgen05 iteration: parity subset through the tc kernel, per-config kernel time, role-wait profile of c2
export PYTHONUNBUFFERED=1
export FC_TC=${FC_TC:-1}
timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "${TESTS:-(c1_shape or shapes or full_c1 or full_c2 or c5_clip or batch_homo or odd or virtual) and not mma}" 2>&1 | tail -4
for c in ${CONFIGS:-c2 c4 c3 c5}; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c
done
timeout 120 python tools/tc_prof.py c2 2>&1 | grep -v "^fc tc prof: ablate"
