# reference B&B (bnb.cpp) with B200 node bounding vs the reference CPU build, same box
# usage: bash tools/bnb_compare.sh [b200-only]
cp /dev/null gpurun_out/bnb.jsonl
for spec in "qaplib tests/golden/nug12.dat" "grid 4x4 1"; do
  for banks in 1 4; do
    r1=$(timeout 900 ./build/bnb_run_b200 $spec $banks 2>&1 | tail -1)
    echo "{\"impl\": \"b200\", \"spec\": \"$spec\", \"result\": $r1}" | tee -a gpurun_out/bnb.jsonl
    if [ "$1" != "b200-only" ]; then
      r2=$(OMP_NUM_THREADS=$(nproc) timeout 900 ./oracle/_ref/bnb_run_ref $spec $banks 2>&1 | tail -1)
      echo "{\"impl\": \"reference-cpu\", \"spec\": \"$spec\", \"result\": $r2}" | tee -a gpurun_out/bnb.jsonl
    fi
  done
done
