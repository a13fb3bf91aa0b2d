for cfg in "QAPB_FOLD_LEAN=1 QAPB_FOLD_LEAN_TPC=1" "QAPB_FOLD_LEAN=1 QAPB_FOLD_LEAN_TPC=4" "QAPB_FOLD_LEAN=1 QAPB_FOLD_LEAN_TPC=16" "QAPB_FOLD_LEAN=0"; do
  r=$(env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items()}, d['parity'])" 2>&1 | tail -1)
  echo "$cfg -> $r"
done
