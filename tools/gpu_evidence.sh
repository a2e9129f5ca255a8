# Sanitizers over every kernel family + ncu-measured DRAM bytes fused vs unfused.
# usage: bash tools/gpu_evidence.sh TAG [precisions...]
TAG=${1:-r2}; shift; PRECS=${@:-bf16 fp32_exact}
mkdir -p gpurun_out/ev_$TAG
O=gpurun_out/ev_$TAG
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/san_cases.py $PRECS > $O/san_$tool.log 2>&1
  echo "sanitizer $tool rc=$? $(grep -c '^ok' $O/san_$tool.log) cases; $(grep -m1 'ERROR SUMMARY' $O/san_$tool.log)"
done
for prec in $PRECS; do
for cfg in "straight 1" "merge 8" "fire 32" "inc3a 64" "a2 64" "squeezenet11 256"; do
  set -- $cfg
  for part in b200 unfused; do
    timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      --profile-from-start off --csv --log-file $O/${1}_${2}_${prec}_${part}.csv python tools/ncu_dram.py run $1 $2 $prec $part > $O/${1}_${2}_${prec}_${part}.log 2>&1
    echo "ncu $1 $2 $prec $part rc=$?"
  done
done
done
python tools/ncu_dram.py summarize $O/dram.json $O/*_*_*_*.csv > /dev/null; tail -c 3000 $O/dram.json
