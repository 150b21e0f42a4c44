# Bounds-checked build of libfc (FC_CHECKED=1: every shared-memory and token address of
# the fused kernel is range-checked, a violation traps) as libfc_checked.so, then the GPU
# parity suite through it:  bash tools/checked_build.sh [--run]
set -e
bash tools/ab_variant.sh checked "-DFC_CHECKED=1"
if [ "$1" = "--run" ]; then
  FC_LIB_VARIANT=checked FC_TC=0 timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_jpeg_gpu.py -q -m gpu -k "not tc" 2>&1 | tail -4
fi
