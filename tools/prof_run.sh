# ncu --set full capture of the fused kernel on the given configs (after a clean bench run)
export PYTHONUNBUFFERED=1
tag=${1:-v}; shift
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c
  bash tools/prof.sh $c $tag
done
