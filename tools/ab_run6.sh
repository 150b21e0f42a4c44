export PYTHONUNBUFFERED=1
FC_LIB_VARIANT=colc FC_TC=0 timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "not tc and (shapes or colour or i420 or full_c2 or full_c4 or torchvision_backend_shapes)" 2>&1 | tail -2
CFG=c2 bash tools/ab_run5.sh colc; CFG=c4 bash tools/ab_run5.sh colc
