# parity of a variant through both kernels' full suite subset, then c2/c4/c3 A/B
export PYTHONUNBUFFERED=1
v=$1
FC_LIB_VARIANT=$v timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_jpeg_gpu.py -q -m gpu 2>&1 | tail -2
bash tools/ab_simple.sh "c2 c4 c3" base $v
