# Round-2 measurement batch (one GPU): bench lines for the BASELINE configs and
# variants, the ncu launch list of the default bench, one full ncu capture of
# the fold and Z-LAP kernels.  Outputs in gpurun_out/.
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_main.jsonl 2> gpurun_out/bench_main.err; echo rc=$?
python bench.py --steps 20 --warmup 5 --variant S1 --no-cpu-baseline > gpurun_out/bench_s1.jsonl 2>&1; echo rc=$?
python bench.py --steps 10 --warmup 4 --variant F2 --no-cpu-baseline > gpurun_out/bench_f2.jsonl 2>&1; echo rc=$?
python bench.py --steps 10 --warmup 4 --variant S2 --no-cpu-baseline > gpurun_out/bench_s2.jsonl 2>&1; echo rc=$?
python bench.py --steps 20 --warmup 5 --n 20 --shape rand --no-cpu-baseline > gpurun_out/bench_tai20.jsonl 2>&1; echo rc=$?
python bench.py --steps 20 --warmup 5 --n 20 --no-cpu-baseline > gpurun_out/bench_nug20.jsonl 2>&1; echo rc=$?
python bench.py --steps 20 --warmup 5 --shape rand --no-cpu-baseline > gpurun_out/bench_tai30.jsonl 2>&1; echo rc=$?
python bench.py --steps 5 --warmup 3 --n 42 --no-cpu-baseline > gpurun_out/bench_n42.jsonl 2>&1; echo rc=$?
python tools/prof_iter.py 30 F1 6 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv \
    python tools/prof_iter.py 30 F1 6 2 > gpurun_out/ncu_launch.log 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k regex:"zfold_ws|lap_batch" -s 10 -c 2 \
    -o gpurun_out/prof_r02 python tools/prof_iter.py 30 F1 6 1 > gpurun_out/ncu_full.log 2>&1; echo rc=$?
