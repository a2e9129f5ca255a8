# fire kernel experiment builds (tools/build_exp.sh): step times + trace summaries per variant
mkdir -p gpurun_out
cp paper_2007_06000_b200/libxlfuse_b200.so _exp/libxlfuse_b200_0.so
for n in ${VARIANTS:-0 1}; do
  cp _exp/libxlfuse_b200_$n.so paper_2007_06000_b200/libxlfuse_b200.so
  echo "=== variant $n"
  SUMMARY=1 timeout 120 python tests/probes/fire_trace.py fire2 256 "fire_nsplit=1,fire_r=14" 2>&1 | grep -v xlf | tail -6
  SUMMARY=1 timeout 120 python tests/probes/fire_trace.py fire6 256 "fire_nsplit=2,fire_g=2" 2>&1 | grep -v xlf | tail -6
done
cp _exp/libxlfuse_b200_0.so paper_2007_06000_b200/libxlfuse_b200.so
timeout 120 python tests/probes/fire_probe.py 256 bf16 2>&1 | tail -24
