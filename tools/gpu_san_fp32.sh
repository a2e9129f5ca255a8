# compute-sanitizer over the fp32 SIMT kernel families incl. every tuned variant (register-blocked convs, 512-thread CTAs)
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/san_cases.py fp32 fp32_exact > gpurun_out/san_fp32_$tool.log 2>&1
  echo "sanitizer $tool rc=$? $(grep -c '^ok' gpurun_out/san_fp32_$tool.log) cases; $(grep -m1 'ERROR SUMMARY' gpurun_out/san_fp32_$tool.log)"
done
tail -5 gpurun_out/san_fp32_memcheck.log
