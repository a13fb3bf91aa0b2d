timeout 200 python bench.py --steps 20 --warmup 5 --n 20 --no-cpu-baseline > gpurun_out/bench_nug20.jsonl 2>&1
timeout 200 python bench.py --steps 20 --warmup 5 --n 20 --shape rand --no-cpu-baseline > gpurun_out/bench_tai20.jsonl 2>&1
for f in bench_nug20 bench_tai20; do tail -1 gpurun_out/$f.jsonl | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["value"],1), round(d["e2e"]["value"],1), {x: round(k[x]["ms_per_launch"],3) for x in k}, d["parity"])'; done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
