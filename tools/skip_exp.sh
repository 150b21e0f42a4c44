export PYTHONUNBUFFERED=1
for sk in 0 1 2 4 3 5 6 7; do echo "skip=$sk"; FC_PROFILE_SKIP=$sk timeout 300 python bench.py --config c2 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py c2; done
