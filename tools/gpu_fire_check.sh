mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fire.py tests/test_gpu_tc.py -k "fire or roundtrip or pointwise" -q -p no:cacheprovider > gpurun_out/pytest_fire.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_fire.log | tail -2; grep -E "^FAILED|^E  " gpurun_out/pytest_fire.log | head -20
timeout 900 python bench.py --no-cpu > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_bf16.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_bf16.json').read().strip().splitlines()[-1])
print("img/s", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"], "parity", d.get("parity",{}).get("normwise"))
print(d["kernels_ms"])
print({k: (v["bf16"]["b200"]["us_median"], v["bf16"]["unfused"]["us_median"], v["bf16"]["speedup"]) for k, v in (d["blocks"] or {}).items() if "bf16" in v})
print({k: v.get("images_per_s") for k, v in d.get("arms", {}).items()})
PY
