# fold experiments: QAPB_FOLD_HINTS bitmask (1 X3 evict_last, 2 stores evict_first, 4 loads evict_first)
run() {  # name env...
  name=$1; shift
  env "$@" timeout 150 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/dbg_$name.log 2>&1
  echo "$name $(tail -1 gpurun_out/dbg_$name.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(k["zfold"]["ms_per_launch"],3), round(k["zlap"]["ms_per_launch"],3), round(d["value"],1), d["parity"])' 2>&1 | tail -1)"
}
for h in 0 1 2 3 4 5 7; do run new_h$h QAPB_FOLD_HINTS=$h; done
for h in 1 3 7; do run rows1_h$h QAPB_FOLD_HINTS=$h QAPB_FOLD_WS_ROWS=1; done
