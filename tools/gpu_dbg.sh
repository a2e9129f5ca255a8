mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 120 python tests/probes/determinism.py squeezenet11 64 bf16 2>&1 | tail -1
bash tools/gpu_bench.sh
XLF_NO_PDL=1 timeout 300 python bench.py --no-cpu --no-blocks > gpurun_out/b2.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b2.json').read().strip().splitlines()[-1]); print('no pdl', d['value'], d['ms_per_step'])"
