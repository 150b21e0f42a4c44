# A/B run: parity (fast subset) of every variant, then interleaved bench of base and variants
export PYTHONUNBUFFERED=1
for v in "$@"; do
  echo "parity $v"; FC_LIB_VARIANT=$v timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "c1_shape or shapes or full_c2 or full_c4 or virtual or i420 or color or batch" 2>&1 | tail -2
done
bash tools/ab_simple.sh "c2 c4 c3" base "$@"
