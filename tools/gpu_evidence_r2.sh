# Round-2 evidence: sanitizers + DRAM fused/unfused (gpu_evidence.sh), the bench
# launch list (ncu, per-launch duration + DRAM bytes) and one full ncu capture
# of the bench's top fire kernel (fire3, tuned as bench.py tunes).
bash tools/gpu_evidence.sh r2b bf16 fp32_exact
O=gpurun_out/ev_r2b
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off \
    --csv --log-file $O/launches.csv python tests/probes/run_block.py squeezenet11 256 bf16 b200 1 tune > $O/launches.log 2>&1; echo "ncu launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:fire_kernel -s 1 -c 1 -o $O/fire3_full -f \
    python tests/probes/run_block.py squeezenet11 256 bf16 b200 1 tune > $O/fire3_full.log 2>&1; echo "ncu full rc=$?"
bash tools/gpu_launchlist.sh
