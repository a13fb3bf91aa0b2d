# per-source-line profile of the steady-state Z-LAP batch (lap_warp.cuh / kernels.cu)
python tools/prof_iter.py 30 F1 6 1 > gpurun_out/pi.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:lap_batch -s 6 -c 1 -o gpurun_out/lap_full python tools/prof_iter.py 30 F1 6 1 > gpurun_out/ncu_lap.log 2>&1
ncu -i gpurun_out/lap_full.ncu-rep --page source --csv > gpurun_out/lap_source.csv 2>&1
ncu -i gpurun_out/lap_full.ncu-rep --page raw --csv > gpurun_out/lap_raw.csv 2>&1
ls -la gpurun_out/lap_*
