# Round-end evidence: GPU tests, smoke, bench (both arms, both precisions), ncu of the bench configuration.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_final_bf16.json 2> gpurun_out/bench_final_bf16.err; echo "bench rc=$?"
timeout 900 python bench.py --precision fp32 --no-cpu > gpurun_out/bench_final_fp32.json 2> gpurun_out/bench_final_fp32.err; echo "bench fp32 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_final_ref.json 2> gpurun_out/bench_final_ref.err; echo "ref rc=$?"
bash tools/gpu_prof.sh
