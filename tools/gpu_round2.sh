# Round-2 GPU pass: parity tests, smoke, the default bench (+ the sharded
# N=1 path), the ICP phase timers, an ncu launch list and one --set full
# capture of the frame's kernels (each ncu pass only after its command
# exited 0 without ncu).  TAG names the outputs.
set -x
T=${TAG:-r2}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo tests=$? >> gpurun_out/${T}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
python bench.py > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_bench.log
python bench.py --impl reference > gpurun_out/${T}_bench_reference.log 2>&1
python bench.py --sharded --configs 0 --cpu-frames 0 > gpurun_out/${T}_bench_sharded1.log 2>&1
python tools/icp_timers.py > gpurun_out/${T}_icptimers.log 2>&1
[ -f .variants_rc/icpsub/librfg.so ] && RFG_LIB_PATH=$PWD/.variants_rc/icpsub/librfg.so python tools/icp_sub.py > gpurun_out/${T}_icpsub.log 2>&1
[ -f .variants_rc/rctiming/librfg.so ] && RFG_LIB_PATH=$PWD/.variants_rc/rctiming/librfg.so python tools/rc_longest.py > gpurun_out/${T}_rclongest.log 2>&1
python tools/e2e_timeline.py > gpurun_out/${T}_e2etimeline.log 2>&1
python tools/configs_bench.py --json gpurun_out/${T}_configs.json > gpurun_out/${T}_configs.log 2>&1
if [ -z "$NO_NCU" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 10 --warmup 5 --cpu-frames 0 --e2e-steps 0 --profile-frames 0 --configs 0 > gpurun_out/${T}_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on \
  -k 'regex:^k_(view_pyramid|icp_track|alloc_stage1|req_assign|vis_count|integrate_depth|range_bin|raycast_tiles)$' \
  -s 40 -c 8 -o gpurun_out/${T}_full -f \
  python bench.py --steps 10 --warmup 5 --cpu-frames 0 --e2e-steps 0 --profile-frames 0 --configs 0 > gpurun_out/${T}_ncu2.log 2>&1
fi
echo done
