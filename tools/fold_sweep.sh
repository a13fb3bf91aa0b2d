# x3buf location groups (QAPB_X3_GROUP; 2 = the fold chunk, i.e. the previous layout)
echo "parity G=4: $(timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_store.py -x -q -k 'not pins' 2>&1 | tail -1)"
echo "parity G=8 mode1: $(QAPB_X3_GROUP=8 QAPB_X3SPLIT=1 timeout 600 python -m pytest tests/test_gpu_engine.py -x -q -k 'not pins' 2>&1 | tail -1)"
for G in 2 4 8 16; do
  r=$(QAPB_X3_GROUP=$G timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items()}, d['parity'])" 2>&1 | tail -1)
  echo "G=$G -> $r"
done
