export PYTHONUNBUFFERED=1
for round in 1 2; do
for sk in 0 1 2 4 8 3 6 12 7; do
  for c in c2; do
    echo -n "skip=$sk $c: "
    FC_SKIP=$sk timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c | cut -d' ' -f5-10
  done
done
done
