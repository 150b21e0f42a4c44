# Per-launch DRAM bytes of the default kernel from a single-pass ncu capture (3 metrics, one
# replay) for c2..c5; the multi-pass --set full captures report more reads for the wide
# windows of c4 (profiles/README.md)
export PYTHONUNBUFFERED=1
for c in c2 c3 c4 c5; do
  echo "== $c"
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fc_fused -s 3 -c 1 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "dram__|gpu__time"
done
