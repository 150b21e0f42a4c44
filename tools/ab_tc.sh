# A/B of tcgen05-kernel library variants on one box: bash tools/ab_tc.sh "<configs>" base variant1 ...
export PYTHONUNBUFFERED=1
export FC_TC=1
cfgs=$1; shift
for round in 1 2; do
  for v in "$@"; do
    for c in $cfgs; do
      if [ "$v" = base ]; then unset FC_LIB_VARIANT; else export FC_LIB_VARIANT=$v; fi
      timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py "$v/$c" | cut -d' ' -f1-8
    done
  done
done
