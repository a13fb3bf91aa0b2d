W=${1:-2}
for v in "QAPB_LAP_NOPATCH=0" "QAPB_LAP_NOPATCH=1"; do
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b${W}_x.log 2>&1
  echo "$v $(tail -1 gpurun_out/b${W}_x.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["parity"], [(r["zfold"], r["zlap"], r["xchg"]) for r in d.get("per_rank_ms_per_launch")])' 2>&1 | tail -1)"
done
