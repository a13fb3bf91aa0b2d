run() {  # name n env...
  name=$1; n=$2; shift; shift
  env "$@" timeout 200 python bench.py --steps 20 --warmup 5 --n $n --shape rand --no-cpu-baseline > gpurun_out/nx_$name.log 2>&1
  echo "$name $(tail -1 gpurun_out/nx_$name.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["value"],1), {x: round(k[x]["ms_per_launch"],3) for x in k}, d["parity"])' 2>&1 | tail -1)"
}
for n in 12 14 16 18 20 22; do
  run n${n}_base $n
  run n${n}_c2 $n QAPB_FOLD_CHUNK=2
done
