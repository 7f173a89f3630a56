# swapping engine: parity tests + the rows bench (tools/rows_bench.py)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_swapping.py tests/test_gpu_c4.py -q -x > gpurun_out/s_tests.log 2>&1; echo tests=$? >> gpurun_out/s_tests.log
python tools/rows_bench.py > gpurun_out/s_rows.log 2>&1; echo rows=$? >> gpurun_out/s_rows.log
