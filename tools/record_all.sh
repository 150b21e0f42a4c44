# full round evidence: record.sh + sanitizer
bash tools/record.sh ${1:-r01}
bash tools/sanitize.sh > gpurun_out/${1:-r01}/sanitizer_summary.txt 2>&1
