# fp32 SIMT path: parity tests (fp32 / fp32_exact) + per-step times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_block.py -x -q -p no:cacheprovider > gpurun_out/pytest_fp32.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_fp32.log; grep -E "^FAILED|Error" gpurun_out/pytest_fp32.log | head -20
bash tools/gpu_fp32steps.sh 2>&1 | grep -E "==>|total|b9.conv10|us  tile" | head -150
