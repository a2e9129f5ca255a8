# correctness (bf16 + engine GPU tests) then quick perf
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_engine.py -q -x -p no:cacheprovider > gpurun_out/pytest_bf16.log 2>&1; rc=$?; echo "pytest bf16 rc=$rc"; tail -5 gpurun_out/pytest_bf16.log
if [ $rc != 0 ]; then timeout 900 compute-sanitizer --print-limit 5 python -m pytest tests/test_gpu_bf16.py -q -x -p no:cacheprovider > gpurun_out/san.log 2>&1; grep -m 30 -E 'Invalid|at 0x|by thread|Address|FAILED' gpurun_out/san.log; exit 1; fi
timeout 300 python tests/probes/phase_cost.py squeezenet11 256 0 6 > gpurun_out/phase_sq.log 2>&1; cat gpurun_out/phase_sq.log | tail -17
bash tools/gpu_bench.sh
