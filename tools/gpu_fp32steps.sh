# fp32 SIMT per-step times (SqueezeNet b200 / unfused, block configs)
mkdir -p gpurun_out
for part in b200 unfused; do timeout 300 python tests/probes/step_times.py squeezenet11 256 $part fp32 > gpurun_out/fp32_sq_$part.log 2>&1; done
for c in "straight 1" "merge 8" "fire 32" "inc3a 64" "a2 64"; do set -- $c
  for part in b200 unfused; do timeout 300 python tests/probes/step_times.py $1 $2 $part fp32 > gpurun_out/fp32_$1_$part.log 2>&1; done
done
tail -n 30 gpurun_out/fp32_*.log
