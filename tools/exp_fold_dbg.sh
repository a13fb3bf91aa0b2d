run() {  # name env... (bench args in BARGS)
  name=$1; shift
  env "$@" timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $BARGS > gpurun_out/dbg_$name.log 2>&1
  echo "$name $(tail -1 gpurun_out/dbg_$name.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(k["zfold"]["ms_per_launch"],3), round(k["zlap"]["ms_per_launch"],3), {x: round(k[x]["ms_per_launch"],3) for x in k if x not in ("zfold","zlap","xyfold")}, round(d["value"],1), d["parity"])' 2>&1 | tail -1)"
}
BARGS="--variant F2" run f2
BARGS="--variant F2" run f2_h0 QAPB_FOLD_HINTS=0
BARGS="--variant S2" run s2
BARGS="--variant S1" run s1
BARGS="--variant F1" run f1
