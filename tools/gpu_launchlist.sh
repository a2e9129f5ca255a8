# ncu launch list of the bench command itself (timed forwards only, via the profiler range in bench.py)
mkdir -p gpurun_out
XLF_NO_PDL=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-blocks --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
echo "ncu rc=$?"; grep -c gpu__time_duration gpurun_out/bench_launches.csv
