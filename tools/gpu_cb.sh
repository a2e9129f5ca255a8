# fire tuner breadth + parity + quick bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fire.py -x -q 2>&1 | tail -3
( time timeout 600 python tests/probes/fire_tune.py 256 ) 2>&1 | grep -v "^\[xlf\] tune" | tail -14
bash tools/gpu_bench_quick.sh
