cd $GRAFT_REPO_ROOT
timeout 300 python tools/gram_time.py 31 > gpurun_out/r51_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_tc -s 2 -c 1 -o gpurun_out/r51_gram python tools/gram_time.py 31 > gpurun_out/r51_ncu.log 2>&1
