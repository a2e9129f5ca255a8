mkdir -p gpurun_out
timeout 300 python tests/probes/step_times.py squeezenet11 256 b200 tf32 > gpurun_out/tf32_sq_b200.log 2>&1
timeout 300 python tests/probes/step_times.py squeezenet11 256 b200 bf16 > gpurun_out/bf16_sq_b200.log 2>&1
cut -c1-60,100-200 gpurun_out/tf32_sq_b200.log gpurun_out/bf16_sq_b200.log
