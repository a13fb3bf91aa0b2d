# sharded lean fold with / without the X3 evict_last hint, 2 GPUs
for h in 1 0; do
  QAPB_LEAN_HINTS=$h timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2953$h bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b2_h$h.log 2>&1
  echo "hints=$h $(tail -1 gpurun_out/b2_h$h.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["parity"], d.get("per_rank_ms_per_launch"))' 2>&1 | tail -1)"
done
