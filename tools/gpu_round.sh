set -x
python -m pytest tests -m gpu -x -q > gpurun_out/i_tests.log 2>&1; echo tests=$? >> gpurun_out/i_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/i_smoke.log 2>&1
python bench.py > gpurun_out/i_bench.log 2>&1
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/i_ref.log 2>&1
python bench.py --sharded > gpurun_out/i_sharded.log 2>&1
python tools/timeline.py --json gpurun_out/i_timeline.json > gpurun_out/i_timeline.txt 2>&1
python tools/configs_bench.py --json gpurun_out/i_configs.json > gpurun_out/i_configs.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/i_launches.csv python bench.py --steps 10 --warmup 5 --cpu-frames 0 --e2e-steps 0 --profile-frames 0 > gpurun_out/i_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rfg:: -s 40 -c 8 -o gpurun_out/i_full -f python bench.py --steps 10 --warmup 5 --cpu-frames 0 --e2e-steps 0 --profile-frames 0 > gpurun_out/i_ncu2.log 2>&1
echo done
