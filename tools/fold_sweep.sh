# X3 split modes (single GPU, n=30 F1) + engine parity tests per mode
for M in 0 1 2; do
  echo "mode $M: $(QAPB_X3SPLIT=$M timeout 400 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -1)"
  r=$(QAPB_X3SPLIT=$M timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items()}, d['parity'])" 2>&1 | tail -1)
  echo "mode $M -> $r"
done
QAPB_X3SPLIT=1 timeout 400 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | grep -E "Error|assert|FAIL" | head -20
