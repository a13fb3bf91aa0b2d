# B&B nug20-shaped on one GPU with per-call facade timings
QAPB_FACADE_STATS=1 timeout 600 ./build/bnb_run_b200 grid 4x5 1 4 > gpurun_out/bnb_stats_b4.log 2>&1; echo rc=$?; cat gpurun_out/bnb_stats_b4.log
