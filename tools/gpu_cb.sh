# fire kernel bias-as-MMA: parity + tuned step times (on / off) + quick bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fire.py -x -q 2>&1 | tail -3
timeout 600 python tests/probes/fire_tune.py 256 fire_bias_mma=0 2>&1 | grep -v "^\[xlf\] tune" | tail -3
bash tools/gpu_bench_quick.sh
