# fire kernel: correctness vs oracle + step times (bf16 / tf32), then a unit-shape sweep
mkdir -p gpurun_out
for a in "b1 2 bf16" "fire 3 tf32"; do echo "=== debug $a"; timeout 120 python tests/probes/fire_debug.py $a 2>&1 | tail -30; done
for args in "256 bf16"; do
  echo "=== $args"; timeout 120 python tests/probes/fire_probe.py $args 2>&1 | tail -40
done
echo "=== sweep"; timeout 600 python tests/probes/fire_sweep.py bf16 256 2>&1 | tail -50
