bash tools/ab_run2.sh pdl
for v in base pdl; do
  if [ $v = base ]; then unset FC_LIB_VARIANT; else export FC_LIB_VARIANT=$v; fi
  echo "vr $v"; timeout 200 python tools/virtual_ranks.py c2 20 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k: v['max_ms'] for k,v in d.items() if isinstance(v, dict) and 'max_ms' in v})"
  timeout 200 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | python tools/brief.py c1_$v | cut -d' ' -f1-8
done
