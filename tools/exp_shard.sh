# sharded fold: warp-specialised (SH) vs lean, N GPUs (arg 1, default 2)
W=${1:-2}
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2951$W tests/mgpu_parity.py > gpurun_out/mg$W.log 2>&1; echo "parity rc=$? $(tail -1 gpurun_out/mg$W.log | cut -c1-200)"
for ws in 1 0; do
  QAPB_FOLD_WS_SHARDED=$ws timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2952$ws bench.py --gpus $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b${W}_ws$ws.log 2>&1
  echo "ws=$ws $(tail -1 gpurun_out/b${W}_ws$ws.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["parity"], [(r["zfold"], r["zlap"], r["xchg"]) for r in d.get("per_rank_ms_per_launch")])' 2>&1 | tail -1)"
done
