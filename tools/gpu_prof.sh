# ncu evidence for the bench configuration (autotuned bf16 SqueezeNet, batch 256)
mkdir -p gpurun_out
XLF_NO_PDL=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off \
    --csv --log-file gpurun_out/launches.csv python tests/probes/run_block.py squeezenet11 256 bf16 b200 1 tune > gpurun_out/launches.log 2>&1; echo "ncu list rc=$?"
XLF_NO_PDL=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:fused_bf16 -c 20 -o gpurun_out/prof_full -f \
    python tests/probes/run_block.py squeezenet11 256 bf16 b200 1 tune > gpurun_out/prof_full.log 2>&1; echo "ncu full rc=$?"
tail -16 gpurun_out/prof_full.log
