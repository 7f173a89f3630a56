# round-1d captures: default bench, reference arm, launch list, full capture of the hot kernels, timeline
python bench.py > gpurun_out/r1d_bench_default.json 2> gpurun_out/r1d_bench_default.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r1d_bench_reference.json 2> gpurun_out/r1d_bench_reference.err
C="python bench.py --steps 10 --warmup 5 --cpu-frames 0 --e2e-steps 0 --profile-frames 0"
$C > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1d_launches.csv $C > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_alloc_stage1|k_raycast_icp|k_raycast_normals|k_integrate_depth|k_icp_track|k_range_tile|k_range_bin|k_req_assign|k_vis_count" -s 45 -c 9 -o gpurun_out/r1d_full $C > gpurun_out/ncu_f.log 2>&1
python tools/timeline.py --frames 100 --json gpurun_out/r1d_timeline.json > gpurun_out/r1d_timeline.txt 2>&1
python bench.py --sharded --cpu-frames 0 --e2e-steps 0 --profile-frames 0 > gpurun_out/r1d_bench_sharded1.json 2> gpurun_out/r1d_bench_sharded1.err
