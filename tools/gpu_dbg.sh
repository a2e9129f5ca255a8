timeout 240 python -m pytest tests/test_gpu_bf16.py -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo "bf16 tests rc=$rc"; tail -1 gpurun_out/pytest_gpu.log
if [ $rc = 0 ]; then
timeout 400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 60 python tests/probes/determinism.py squeezenet11 64 bf16 2>&1 | tail -1
for i in 1 2; do timeout 90 python bench.py --no-cpu --no-blocks > gpurun_out/b.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'])"; done
fi
