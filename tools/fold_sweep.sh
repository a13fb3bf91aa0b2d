# lean fold: L2 prefetch of the CTA's next triple x triples per CTA
echo "parity: $(timeout 600 python -m pytest tests/test_gpu_engine.py -x -q -k 'not pins' 2>&1 | tail -1)"
for cfg in "QAPB_FOLD_PREFETCH=0 QAPB_FOLD_LEAN_TPC=4" "QAPB_FOLD_PREFETCH=1 QAPB_FOLD_LEAN_TPC=4" "QAPB_FOLD_PREFETCH=1 QAPB_FOLD_LEAN_TPC=8" "QAPB_FOLD_PREFETCH=1 QAPB_FOLD_LEAN_TPC=16" "QAPB_FOLD_PREFETCH=0 QAPB_FOLD_LEAN_TPC=4"; do
  r=$(env $cfg timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['kernels']['zfold']['ms_per_launch'],3), round(d['kernels']['zlap']['ms_per_launch'],3), d['parity']['bitwise'])" 2>&1 | tail -1)
  echo "$cfg -> $r"
done
