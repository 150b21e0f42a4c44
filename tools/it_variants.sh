export PYTHONUNBUFFERED=1
for c in c2 c4 c5; do for t in f32 bf16; do timeout 300 python bench.py --config $c --tokens $t --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py $c/$t; done; done
timeout 300 python bench.py --config c2 --color bt709_full --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | python tools/brief.py c2/bt709full
