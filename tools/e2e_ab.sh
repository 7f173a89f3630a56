# Interleaved A/B of the end-to-end leg (bench.py's e2e value) and the e2e
# device timeline of the .variants/<name>/librfg.so builds: AB_REPS rounds,
# logs gpurun_out/e2eb_<name>_<r>.log and e2etl_<name>_<r>.log
mkdir -p gpurun_out
for r in $(seq 1 ${AB_REPS:-3}); do
  for d in .variants/*/; do
    n=$(basename $d)
    RFG_LIB_PATH=$PWD/${d}librfg.so python bench.py --cpu-frames 0 --configs 0 --steps 40 ${AB_ARGS:-} > gpurun_out/e2eb_${n}_${r}.log 2>&1
    RFG_LIB_PATH=$PWD/${d}librfg.so python tools/e2e_timeline.py > gpurun_out/e2etl_${n}_${r}.log 2>&1
  done
done
