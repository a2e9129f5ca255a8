# one ncu --set full capture of the first fused kernel of the forward (conv1+pool1)
mkdir -p gpurun_out
XLF_NO_PDL=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:fused_bf16 -c ${NCU_C:-1} -o gpurun_out/prof_b8 -f \
    python tests/probes/run_block.py squeezenet11 256 bf16 b200 1 tune > gpurun_out/prof_b8.log 2>&1; echo "ncu rc=$?"
tail -20 gpurun_out/prof_b8.log
