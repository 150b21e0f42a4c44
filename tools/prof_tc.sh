# ncu full capture of one tcgen05-kernel launch: bash tools/prof_tc.sh <config> <tag>
export PYTHONUNBUFFERED=1
export FC_TC=${FC_TC:-1}
c=${1:-c2}; tag=${2:-v}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fc_tc_kernel -s 3 -c 1 -o gpurun_out/prof_${c}_${tag} python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_${c}_${tag}.log 2>&1
tail -2 gpurun_out/ncu_${c}_${tag}.log
