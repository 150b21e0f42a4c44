export PYTHONUNBUFFERED=1
FC_LIB_VARIANT=colcompact timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "full_c2 or shapes" 2>&1 | tail -2
CFGS="c2 c5 c3" bash tools/exp_ab3.sh colcompact
