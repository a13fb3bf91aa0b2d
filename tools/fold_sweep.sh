# fold variants with the X3 split: chunk (QAPB_FOLD_CHUNK) x lean kernel (QAPB_FOLD_LEAN)
for cfg in "QAPB_FOLD_CHUNK=1 QAPB_FOLD_LEAN=0" "QAPB_FOLD_CHUNK=1 QAPB_FOLD_LEAN=1" "QAPB_FOLD_CHUNK=2 QAPB_FOLD_LEAN=0" "QAPB_FOLD_CHUNK=2 QAPB_FOLD_LEAN=1" "QAPB_FOLD_CHUNK=2 QAPB_FOLD_LEAN=1 QAPB_FOLD_LEAN_TPC=1" "QAPB_FOLD_CHUNK=2 QAPB_FOLD_LEAN=1 QAPB_FOLD_LEAN_TPC=8"; do
  r=$(env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['kernels']['zfold']['ms_per_launch'],3), d['parity'])" 2>&1 | tail -1)
  echo "$cfg -> $r"
done
