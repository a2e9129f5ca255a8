# ncu full captures of single fp32 SIMT launches of an unfused SqueezeNet forward (batch 64):
# conv1 (launch 0), fire4_expand3 (11), conv10 (28); only summaries come back
mkdir -p gpurun_out /tmp/np
for k in ${KSRC:-0 11 28}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_block_kernel --profile-from-start off --launch-skip $k -c 1 -o /tmp/np/p$k -f \
      python tests/probes/run_block.py squeezenet11 64 fp32 ${PART:-unfused} 1 > gpurun_out/fp32prof$k.log 2>&1; echo "ncu $k rc=$?"
  ncu -i /tmp/np/p$k.ncu-rep --page raw --csv > gpurun_out/fp32prof_raw$k.csv 2>&1
  python tools/ncu_hot.py /tmp/np/p$k.ncu-rep 1e4 > gpurun_out/fp32prof_hot$k.txt 2>&1
done
ls -la gpurun_out
