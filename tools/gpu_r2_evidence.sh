# Round-2 evidence run (one GPU): default bench line, per-model config-5 lines,
# config-3 lines, launch list + ncu --set full of the hot kernels (config 5 and 3).
mkdir -p gpurun_out
export TAG=${TAG:-r2}
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-400
: > gpurun_out/models_${TAG}.jsonl
for m in uniform epanechnikov histogram; do
  timeout 900 python bench.py --models $m --steps 10 --warmup 3 > gpurun_out/model_${m}.log 2>&1; echo "$m rc=$?"
  tail -1 gpurun_out/model_${m}.log >> gpurun_out/models_${TAG}.jsonl
done
STEPS=20 timeout 900 bash tools/bench_config3.sh
timeout 1500 bash tools/prof_full.sh
# (gpurun copies back <= 64 MiB: SKIP_C3_NCU=1 leaves out the three config-3 reports)
[ -n "$SKIP_C3_NCU" ] || for b in 8 16 32; do
  P="python bench.py --height 2048 --width 2048 --members 40 --bins $b --models histogram --fit separate --no-e2e --no-cpu --steps 1 --warmup 1 --profile"
  $P > gpurun_out/prof_c3_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"closed_hist" -c 1 -o gpurun_out/prof_c3_b${b}_${TAG} $P > gpurun_out/prof_c3_ncu_b$b.log 2>&1; tail -1 gpurun_out/prof_c3_ncu_b$b.log
done
