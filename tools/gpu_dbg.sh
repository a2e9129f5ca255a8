timeout 900 python -m pytest tests/test_gpu_bf16.py -q -x -p no:cacheprovider -k forced > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
