set -x
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG:-i}_tests.log 2>&1; echo tests=$? >> gpurun_out/${TAG:-i}_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG:-i}_smoke.log 2>&1
python bench.py > gpurun_out/${TAG:-i}_bench.log 2>&1
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/${TAG:-i}_ref.log 2>&1
python bench.py --sharded > gpurun_out/${TAG:-i}_sharded.log 2>&1
python tools/timeline.py --json gpurun_out/${TAG:-i}_timeline.json > gpurun_out/${TAG:-i}_timeline.txt 2>&1
python tools/configs_bench.py --json gpurun_out/${TAG:-i}_configs.json > gpurun_out/${TAG:-i}_configs.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG:-i}_launches.csv python bench.py --steps 10 --warmup 5 --cpu-frames 0 --e2e-steps 0 --profile-frames 0 > gpurun_out/${TAG:-i}_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:^k_(view_pyramid|icp_track|alloc_stage1|req_assign|vis_count|integrate_depth|range_bin|raycast_tiles)$" -s 40 -c 8 -o gpurun_out/${TAG:-i}_full -f python bench.py --steps 10 --warmup 5 --cpu-frames 0 --e2e-steps 0 --profile-frames 0 > gpurun_out/${TAG:-i}_ncu2.log 2>&1
echo done
