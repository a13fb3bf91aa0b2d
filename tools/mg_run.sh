set -x
W=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2951$W tests/mgpu_parity.py > gpurun_out/mg$W.log 2>&1; echo rc=$?; tail -1 gpurun_out/mg$W.log | cut -c1-3000
