# the driver's default bench (our arm, then the reference arm), lines under gpurun_out/
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1])
print("img/s", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"], "parity", d.get("parity"))
print(d["kernels_ms"])
print({k: v.get("images_per_s") for k, v in d.get("arms", {}).items()})
print(d["roofline"]["kernel"], d["roofline"]["frac"], d["roofline"]["traffic"], d["cpu_baseline"], d["clocks"], d["gpu_launches"])
r=json.loads(open('gpurun_out/bench_ref.json').read().strip().splitlines()[-1]); print("ref", r["value"], r.get("unit"))
PY
