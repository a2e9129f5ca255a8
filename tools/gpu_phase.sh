mkdir -p gpurun_out
timeout 600 python tests/probes/phase_cost.py squeezenet11 256 0 1 2 4 6 > gpurun_out/phase_sq.log 2>&1; cat gpurun_out/phase_sq.log | tail -20
timeout 600 python tests/probes/phase_cost.py inc3a 64 0 1 2 4 6 > gpurun_out/phase_inc.log 2>&1; cat gpurun_out/phase_inc.log | tail -8
