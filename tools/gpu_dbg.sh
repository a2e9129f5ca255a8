mkdir -p gpurun_out
XLF_TUNE_VERBOSE=1 timeout 300 python tests/probes/run_block.py squeezenet11 256 bf16 b200 1 tune 2>&1 | grep -E '^b9|tune b9' | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --profile-from-start off -k regex:fused_bf16 python tests/probes/run_block.py squeezenet11 256 bf16 b200 1 2>&1 | grep -E 'ERROR|b9' | head -5
timeout 600 ncu --metrics gpu__time_duration.sum --profile-from-start off -k regex:fused_bf16 python tests/probes/run_block.py squeezenet11 256 bf16 b200 1 tune 2>&1 | grep -E 'ERROR|b9' | head -5
