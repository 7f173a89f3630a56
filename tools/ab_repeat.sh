# Interleaved A/B of the .variants/<name>/librfg.so builds: AB_REPS rounds of
# one bench run per variant (default config), logs gpurun_out/abr_<name>_<r>.log
mkdir -p gpurun_out
for r in $(seq 1 ${AB_REPS:-3}); do
  for d in .variants/*/; do
    n=$(basename $d)
    RFG_LIB_PATH=$PWD/${d}librfg.so python bench.py --cpu-frames 0 --e2e-steps 0 ${AB_ARGS:-} > gpurun_out/abr_${n}_${r}.log 2>&1
  done
done
