python -m pytest -q -m gpu tests > gpurun_out/r1e_gputests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1e_smoke.txt 2>&1
python bench.py > gpurun_out/r1e_bench_default.json 2> gpurun_out/r1e_bench_default.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r1e_bench_reference.json 2> gpurun_out/r1e_bench_reference.err
python tools/timeline.py --frames 100 --json gpurun_out/r1e_timeline.json > gpurun_out/r1e_timeline.txt 2>&1
python tools/e2e_probe.py > gpurun_out/r1e_e2e_probe.txt 2>&1
