mkdir -p gpurun_out
for c in "fire 32" "inc3a 64" "straight 1" "merge 8"; do for p in unfused b200; do
  echo "== $c $p"; timeout 900 compute-sanitizer --print-limit 2 python tests/probes/tune_case.py $c 3 $p 2>&1 | grep -v 'by thread' | grep -E -m 6 'Invalid|Out-of|at |ERROR SUMMARY|Address'
done; done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
bash tools/gpu_bench.sh
