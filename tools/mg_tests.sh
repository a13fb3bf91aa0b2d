timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_engine.py -x -q > gpurun_out/t_mg.log 2>&1; tail -2 gpurun_out/t_mg.log
