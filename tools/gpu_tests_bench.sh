# GPU suite, then the quick bench (no CPU baseline / other precisions of SqueezeNet)
bash tools/gpu_tests.sh
bash tools/gpu_bench_quick.sh
