mkdir -p gpurun_out
timeout 120 python tests/probes/fire_trace.py fire2 256 "fire_nsplit=1,fire_r=14" > gpurun_out/ftrace_fire2.txt 2>&1; echo rc=$?; tail -3 gpurun_out/ftrace_fire2.txt
timeout 120 python tests/probes/fire_trace.py fire6 256 "fire_nsplit=2,fire_g=2" > gpurun_out/ftrace_fire6.txt 2>&1; echo rc=$?; tail -3 gpurun_out/ftrace_fire6.txt
