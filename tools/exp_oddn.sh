for n in 18 19 20 21 25 26; do
  timeout 200 python bench.py --steps 20 --warmup 5 --n $n --shape rand --no-cpu-baseline > gpurun_out/bn$n.log 2>&1
  echo "n=$n $(tail -1 gpurun_out/bn$n.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["value"],1), {x: round(k[x]["ms_per_launch"],3) for x in k}, d["parity"])' 2>&1 | tail -1)"
done
