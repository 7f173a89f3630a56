# A/B of the kernel variants under .variants/<name>/librfg.so: parity of the
# raycast-affecting tests, stage times and the default bench's frame rate
mkdir -p gpurun_out
for d in .variants/*/; do
  n=$(basename $d)
  RFG_LIB_PATH=$PWD/${d}librfg.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c4.py tests/test_gpu_golden.py tests/test_gpu_icp.py -q -x > gpurun_out/v_${n}_tests.log 2>&1; echo rc=$? >> gpurun_out/v_${n}_tests.log
  RFG_LIB_PATH=$PWD/${d}librfg.so python tools/stage_bench.py > gpurun_out/v_${n}_stage.log 2>&1
  RFG_LIB_PATH=$PWD/${d}librfg.so python bench.py --cpu-frames 0 --e2e-steps 0 > gpurun_out/v_${n}_bench.log 2>&1
done
