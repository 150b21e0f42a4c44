export PYTHONUNBUFFERED=1
FC_LIB_VARIANT=rowperm timeout 1200 python -m pytest tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -2
CFGS="c2 c4 c5 c3" bash tools/exp_ab3.sh rowperm
