# compute-sanitizer over smoke() and tools/sanitize_cases.py (every kernel family, small sizes)
# usage (on the GPU box): bash tools/sanitize.sh  -> gpurun_out/sanitize_<tool>_<case>.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for c in smoke cases; do
    if [ $c = smoke ]; then cmd="python __graft_entry__.py smoke"; else cmd="python tools/sanitize_cases.py"; fi
    timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 $cmd > gpurun_out/sanitize_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$?" | tee -a gpurun_out/sanitize_summary.txt
    tail -3 gpurun_out/sanitize_${tool}_${c}.log
  done
done
