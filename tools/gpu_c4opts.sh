mkdir -p gpurun_out
timeout 600 python tests/probes/block_time.py inc3a 64 bf16 "" "mb_max_weight=0" "mb_pw=1" > gpurun_out/c4opts.log 2>&1
timeout 600 python tests/probes/block_time.py inc3a 64 tf32 "" "mb_max_weight=0" "mb_pw=1" >> gpurun_out/c4opts.log 2>&1
timeout 300 python tests/probes/step_times.py inc3a 64 unfused bf16 >> gpurun_out/c4opts.log 2>&1
timeout 300 python tests/probes/step_times.py inc3a 64 b200 bf16 >> gpurun_out/c4opts.log 2>&1
cat gpurun_out/c4opts.log
