mkdir -p gpurun_out
for a in "b1 2 bf16" "fire 3 bf16" "b1 2 tf32"; do echo "=== $a"; timeout 120 python tests/probes/fire_debug.py $a 2>&1 | tail -60; done
