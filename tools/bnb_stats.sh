# B&B nug20-shaped (reference bnb.cpp unmodified, nodes bounded by libqapb200): banks sweep on 1 GPU
for b in 8 16; do
  QAPB_FACADE_STATS=1 timeout 600 ./build/bnb_run_b200 grid 4x5 1 $b > gpurun_out/bnb_1g_b$b.log 2>&1; echo "1gpu banks=$b rc=$? $(tail -1 gpurun_out/bnb_1g_b$b.log)"
done
timeout 900 python -m pytest tests/test_gpu_concurrency.py tests/test_gpu_engine.py tests/test_gpu_reference_suite.py tests/test_gpu_store.py -x -q > gpurun_out/t_eng.log 2>&1; tail -2 gpurun_out/t_eng.log
