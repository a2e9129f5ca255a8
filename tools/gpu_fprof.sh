# ncu full capture of the fire kernel (fire2 / fire3 at batch 256), source-level stall sampling
mkdir -p gpurun_out
OPTS=${1:-"fire_nsplit=1,fire_r=55,fire_sqs=2,fire_cps=1"}
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:fire_kernel -c 2 -o gpurun_out/fire_prof -f \
    python tests/probes/run_block.py squeezenet11 256 bf16 b200 1 notune "$OPTS" > gpurun_out/fire_prof.log 2>&1; echo "ncu full rc=$?"
tail -5 gpurun_out/fire_prof.log
