# quick perf check: bench (bf16) + traces
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_bf16.json').read().strip().splitlines()[-1])
print("img/s", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"])
print({k: v for k, v in d["kernels_ms"].items()})
print({k: (v["b200"]["us_median"], v["unfused"]["us_median"], v["speedup"]) for k, v in (d["blocks"] or {}).items()})
PY
XLF_TRACE=1 timeout 300 python tests/probes/trace_block.py squeezenet11 256 > gpurun_out/trace_sq.log 2>&1
