mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
XLF_TRACE=1 timeout 300 python tests/probes/trace_block.py squeezenet11 256 > gpurun_out/trace_sq.log 2>&1; echo "trace rc=$?"
XLF_TRACE=1 timeout 300 python tests/probes/trace_block.py fire 32 > gpurun_out/trace_fire.log 2>&1
XLF_TRACE=1 timeout 300 python tests/probes/trace_block.py inc3a 64 > gpurun_out/trace_inc.log 2>&1
