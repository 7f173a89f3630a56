# A/B of kernel variants under .variants/<name>/librfg.so: per-stage times
# (tools/stage_bench.py) and the bench's frame rate + kernel durations; the
# parity tests named in $AB_TESTS (default: the raycast/ICP-affecting ones)
# run on every variant.
mkdir -p gpurun_out
TESTS=${AB_TESTS:-"tests/test_gpu_tracked_c2.py tests/test_gpu_parity.py tests/test_gpu_c4.py"}
for d in .variants/*/; do
  n=$(basename $d)
  if [ -n "$TESTS" ] && [ "$TESTS" != "none" ]; then
    RFG_LIB_PATH=$PWD/${d}librfg.so timeout 900 python -m pytest $TESTS -q -x > gpurun_out/ab_${n}_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_${n}_tests.log
  fi
  RFG_LIB_PATH=$PWD/${d}librfg.so python bench.py --cpu-frames 0 --e2e-steps 0 --configs ${AB_CONFIGS:-0} ${AB_ARGS:-} > gpurun_out/ab_${n}_bench.log 2>&1
done
