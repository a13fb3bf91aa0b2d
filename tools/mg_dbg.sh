W=${1:-2}
for v in "QAPB_FOLD_CHUNK=2" "QAPB_FOLD_CHUNK=2 QAPB_FOLD_WS_ROWS=1"; do
env $v MGPU_CASES=nug12_F1,rand20_F1 QAPB_SYNC_CHECK=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 29519 tests/mgpu_parity.py > gpurun_out/mgdbg.log 2>&1; echo "$v rc=$?"
grep -E "QapbError" gpurun_out/mgdbg.log | head -2; tail -1 gpurun_out/mgdbg.log | cut -c1-200
done
