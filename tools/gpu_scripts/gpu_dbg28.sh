cd $GRAFT_REPO_ROOT
timeout 300 python tools/ab_step.py C3 > gpurun_out/d28.log 2>&1
timeout 300 python tools/prof_step.py >> gpurun_out/d28.log 2>&1
GAR_COORD_LOADER=tma timeout 300 python tools/prof_step.py >> gpurun_out/d28.log 2>&1
timeout 300 compute-sanitizer --tool memcheck python tools/ab_step.py C1 >> gpurun_out/d28.log 2>&1
