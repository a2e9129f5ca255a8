timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "a2 or edge or random or every_reference_block" > gpurun_out/pytest_dw.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_dw.log
bash tools/gpu_bench_quick.sh
