# Z-stage pipelining (fold stage k || Z-LAPs of the pairs it completed) with the X3 split
echo "parity zstages=4: $(QAPB_ZSTAGES=4 timeout 400 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -1)"
for K in 1 2 4 8; do
  r=$(QAPB_ZSTAGES=$K timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: (round(v['ms_per_launch'],3), v['launches']) for k,v in d['kernels'].items()}, d['parity'])" 2>&1 | tail -1)
  echo "zstages=$K -> $r"
done
