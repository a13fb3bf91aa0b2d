set -x
for W in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2951$W tests/mgpu_parity.py > gpurun_out/mg$W.log 2>&1; echo rc=$?; tail -1 gpurun_out/mg$W.log | cut -c1-200
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2952$W bench.py --gpus $W --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b$W.log 2>&1; echo rc=$?; tail -1 gpurun_out/b$W.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['per_rank_ms_per_launch'])"
done
