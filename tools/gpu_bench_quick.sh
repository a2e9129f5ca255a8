mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu --no-arms > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_bf16.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_bf16.json').read().strip().splitlines()[-1])
print("img/s", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"])
print(d["kernels_ms"])
for k, v in (d["blocks"] or {}).items():
    print(k, {p: (v[p]["b200"]["us_median"], v[p]["unfused"]["us_median"], v[p]["speedup"], v[p]["roofline"]["frac"]) for p in ("fp32","tf32","bf16") if p in v})
print(d.get("autotune"))
PY
