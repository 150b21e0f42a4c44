# A/B of kernel variants on one box: bash tools/ab.sh "<config list>" A B ...
# (variants = paper_2512_17574_b200/libfc_<name>.so; "base" = libfc.so), interleaved 3 rounds.
export PYTHONUNBUFFERED=1
cfgs=$1; shift
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv,noheader
for round in 1 2 3; do
  for v in "$@"; do
    for c in $cfgs; do
      if [ "$v" = base ]; then unset FC_LIB_VARIANT; else export FC_LIB_VARIANT=$v; fi
      if [ $round = 1 ]; then export FC_VERBOSE=1; else unset FC_VERBOSE; fi
      timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | sort -u | grep -v "^fc launch" | python tools/brief.py "$v/$c" | cut -d' ' -f1-8,15-16
      [ $round = 1 ] && FC_LIB_VARIANT=${FC_LIB_VARIANT:-} timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep "^fc launch" | sort -u | head -2
    done
  done
done
true
