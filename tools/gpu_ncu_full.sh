# ncu --set full of one frame's eight kernels (after 5 warm-up frames) of the
# default C2 bench command; run only after that command exited 0 without ncu.
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on \
  -k 'regex:^k_(view_pyramid|icp_track|alloc_stage1|req_assign|vis_count|integrate_depth|range_bin|raycast_tiles)$' \
  -s 40 -c 8 -o gpurun_out/i_full -f \
  python bench.py --steps 10 --warmup 5 --cpu-frames 0 --e2e-steps 0 --profile-frames 0 > gpurun_out/i_ncu2.log 2>&1
echo ncu=$?
