# Final round-2 evidence (compute-sanitizer is closed on this pool): ncu DRAM bytes
# fused vs unfused per config for bf16 / TF32 / fp32, the bench launch list, and one
# full capture of the bench's top fire kernel (fire3), summarised on the box.
O=gpurun_out/ev_r2f
mkdir -p $O /tmp/ev
for prec in bf16 tf32 fp32; do
for cfg in "straight 1" "merge 8" "fire 32" "inc3a 64" "a2 64" "squeezenet11 256"; do
  set -- $cfg
  for part in b200 unfused; do
    timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      --profile-from-start off --csv --log-file $O/${1}_${2}_${prec}_${part}.csv python tools/ncu_dram.py run $1 $2 $prec $part > $O/${1}_${2}_${prec}_${part}.log 2>&1
    echo "ncu $1 $2 $prec $part rc=$?"
  done
done
done
python tools/ncu_dram.py summarize $O/dram.json $O/*_*_*_*.csv > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off \
    --csv --log-file $O/launches.csv python tests/probes/run_block.py squeezenet11 256 bf16 b200 1 tune > $O/launches.log 2>&1; echo "ncu launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:fire_kernel -s 1 -c 1 -o /tmp/ev/fire3_full -f \
    python tests/probes/run_block.py squeezenet11 256 bf16 b200 1 tune > $O/fire3_full.log 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/ev/fire3_full.ncu-rep --page raw --csv > $O/fire3_raw.csv 2>&1
python tools/ncu_hot.py /tmp/ev/fire3_full.ncu-rep 1e5 > $O/fire3_hot.txt 2>&1
ls -la $O | head -5; du -sh $O
