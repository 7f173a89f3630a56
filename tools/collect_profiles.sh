# Copy one tools/gpu_round2.sh capture (gpurun_out/<TAG>_*) into profiles/:
# the bench lines as JSON, the text reports, the ncu launch list and the
# --set full summary.  Usage: bash tools/collect_profiles.sh TAG
set -e
T=${1:?TAG}
G=gpurun_out
P=profiles
json_line() { python - "$1" "$2" <<'EOF'
import json, sys
line = None
for l in open(sys.argv[1]):
    if l.startswith("{"):
        line = l
if line:
    json.dump(json.loads(line), open(sys.argv[2], "w"), indent=1)
EOF
}
json_line $G/${T}_bench.log $P/${T}_bench_default.json
json_line $G/${T}_bench_reference.log $P/${T}_bench_reference.json
json_line $G/${T}_bench_sharded1.log $P/${T}_bench_sharded1.json
cp $G/${T}_configs.json $P/${T}_configs.json
cp $G/${T}_icptimers.log $P/${T}_icp_timers.txt
[ -f $G/${T}_icpsub.log ] && cp $G/${T}_icpsub.log $P/${T}_icp_subphases.txt
[ -f $G/${T}_rclongest.log ] && cp $G/${T}_rclongest.log $P/${T}_raycast_longest.txt
{ echo "# e2e device timeline (${T}): tools/e2e_timeline.py"; echo; grep -v "UserWarning\|_warn_once" $G/${T}_e2etimeline.log; } > $P/${T}_e2e_timeline.txt
cp $G/${T}_launches.csv $P/${T}_launches.csv
{ echo "# ncu launch list (${T}): \`tools/gpu_round2.sh\`, 10-frame C2 bench command, \`--metrics gpu__time_duration.sum --clock-control none\` (per-launch cold-cache, serialised)"; echo;
  python tools/ncu_summary.py $G/${T}_launches.csv; } > $P/${T}_launches.md
{ echo "# ncu --set full (${T}): one frame's kernels of the C2 bench command (frame 5, \`tools/gpu_round2.sh\`)"; echo;
  python tools/ncu_summary.py $G/${T}_launches.csv $G/${T}_full.ncu-rep | sed -n '/^| kernel | time/,$p'; } > $P/${T}_kernels.md
tail -n 3 $G/${T}_tests.log
cat $G/${T}_smoke.log | tail -n 2
