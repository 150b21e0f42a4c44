# A/B of kernel variants on one box: bash tools/ab.sh "<config list>" A B ...
# (variants = paper_2512_17574_b200/libfc_<name>.so; "base" = libfc.so), interleaved 3 rounds.
export PYTHONUNBUFFERED=1
cfgs=$1; shift
for round in 1 2 3; do
  for v in "$@"; do
    for c in $cfgs; do
      if [ "$v" = base ]; then unset FC_LIB_VARIANT; else export FC_LIB_VARIANT=$v; fi
      timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py "$v/$c" | cut -d' ' -f1-8
    done
  done
done
