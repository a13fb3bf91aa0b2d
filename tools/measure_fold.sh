timeout 200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_h3.log 2>&1; tail -1 gpurun_out/bench_h3.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(k["zfold"]["ms_per_launch"],3), round(k["zlap"]["ms_per_launch"],3), round(d["value"],1), d["parity"], d["roofline"]["roofline_fold"]["frac"], d["e2e"]["value"])'
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,gpu__time_duration.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
python tools/prof_iter.py 30 F1 6 1 > gpurun_out/pi.log 2>&1 && ncu --metrics $M --clock-control none -k regex:zfold_ws -s 4 -c 1 --csv python tools/prof_iter.py 30 F1 6 1 > gpurun_out/ncu_fold_h3.csv 2>&1
grep -h "zfold" gpurun_out/ncu_fold_h3.csv | awk -F'","' '{print $(NF-2), $NF}'
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_h3.log 2>&1; tail -2 gpurun_out/t_h3.log
