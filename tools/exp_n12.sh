for v in F2 S2; do for n in 12 14 20; do
QAPB_FOLD_CHUNK=2 QAPB_SYNC_CHECK=1 QAPB_NO_GRAPH=1 timeout 200 python bench.py --steps 3 --warmup 3 --n $n --shape rand --variant $v --no-cpu-baseline > gpurun_out/n12ph2.log 2>&1; echo "$v n=$n rc=$?"; grep -iE "error" gpurun_out/n12ph2.log | head -2
done; done
