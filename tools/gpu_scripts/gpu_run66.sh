cd $GRAFT_REPO_ROOT
ORDER=rev timeout 300 python tools/phase_time.py C3 >> gpurun_out/r66.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu,clocks_throttle_reasons.active --format=csv >> gpurun_out/r66.log
timeout 300 python tools/phase_time.py C3 >> gpurun_out/r66.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu,clocks_throttle_reasons.active --format=csv >> gpurun_out/r66.log
