# A/B of the strip-synchronous mapping (FC_SMAP) and its balanced grid (FC_SMAP_BAL) on c2..c5
export PYTHONUNBUFFERED=1
for round in 1 2; do
  for v in "base" "smap" "smapbal"; do
    for c in ${CONFIGS:-c2 c3 c4 c5}; do
      unset FC_SMAP FC_SMAP_BAL
      [ $v = smap ] && export FC_SMAP=1
      [ $v = smapbal ] && export FC_SMAP=1 FC_SMAP_BAL=1
      timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py "$v/$c" | cut -d' ' -f1-8
    done
  done
done
for c in c4 c3; do
  FC_SMAP=1 FC_SMAP_BAL=1 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fc_fused -s 3 -c 1 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "dram__|gpu__time" 
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fc_fused -s 3 -c 1 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "dram__|gpu__time"
done
