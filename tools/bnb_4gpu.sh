# B&B nug20-shaped across 4 GPUs (QAPB_BANK_GPUS=4: banks placed round-robin)
for b in 4 8 16; do
  QAPB_BANK_GPUS=4 timeout 600 ./build/bnb_run_b200 grid 4x5 1 $b > gpurun_out/bnb_4g_b$b.log 2>&1; echo "4gpu banks=$b rc=$? $(tail -1 gpurun_out/bnb_4g_b$b.log)"
done
