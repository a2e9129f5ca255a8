mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 120 python tests/probes/determinism.py squeezenet11 64 bf16 2>&1 | tail -1
bash tools/gpu_bench.sh
