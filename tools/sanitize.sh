export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck initcheck; do
  s=$(date +%s)
  timeout 1500 compute-sanitizer --tool $tool --kernel-name kns=fc_ --print-limit 20 python tools/sanitize.py > gpurun_out/san/$tool.txt 2>&1
  echo "$tool rc=$? $(( $(date +%s) - s ))s $(tail -2 gpurun_out/san/$tool.txt | tr '\n' ' ')"
done
s=$(date +%s)
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py > gpurun_out/san/racecheck_all.txt 2>&1
echo "racecheck(all kernels) rc=$? $(( $(date +%s) - s ))s $(tail -2 gpurun_out/san/racecheck_all.txt | tr '\n' ' ')"
