# GPU check: parity tests, the reference's own tests through patch_reference, one bench run
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
if [ "${REFTESTS:-1}" = "1" ]; then
  timeout 900 python tools/run_reference_tests.py -x > gpurun_out/reftests.log 2>&1; echo "reftests rc=$?"
  tail -5 gpurun_out/reftests.log
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 > gpurun_out/bench_${TAG:-x}.log 2>&1; echo "bench rc=$?"
  tail -c 4000 gpurun_out/bench_${TAG:-x}.log
fi
