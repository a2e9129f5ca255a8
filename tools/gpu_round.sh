#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (both arms), ncu launch list + full capture.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh'
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err; echo "bench rc=$?"
timeout 600 python bench.py --precision fp32 --no-cpu --no-blocks > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-blocks --no-cpu > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_bf16 -c 16 -o gpurun_out/prof -f \
    python tests/probes/run_block.py squeezenet11 256 bf16 b200 1 > gpurun_out/prof.log 2>&1; echo "ncu full rc=$?"
cat gpurun_out/bench_bf16.json | head -c 3000
