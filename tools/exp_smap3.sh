export PYTHONUNBUFFERED=1
for round in 1 2 3; do for sm in def 1; do for c in c3 c5 c4; do
  if [ $sm = def ]; then unset FC_SMAP; else export FC_SMAP=$sm; fi
  echo -n "smap=$sm $c: "; timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c | cut -d' ' -f5-10
done; done; done
