# On the GPU box: launch lists + one ncu --set full capture of the hot kernel per config.
# usage: TAG=r01 CFGS="cfg2 cfg5" bash tools/profile_round.sh
TAG=${TAG:-r01}; CFGS=${CFGS:-"cfg2"}
for c in $CFGS; do
  [ -n "$SKIP_LAUNCHES" ] || timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_$c.csv python bench.py --config $c --profile --steps 2 --warmup 3 --no-cpu \
    > gpurun_out/${TAG}_launches_$c.log 2>&1; echo "launches $c rc=$?"
  # the profiled sweep's streaming launches: skip the build, the parity runs, the autotune and
  # the warm-up sweeps (counted from the launch list of the same command)
  n=$(python - "$c" <<'PY'
import json, subprocess, sys
sys.path.insert(0, ".")
from bench import CONFIGS
print(len(CONFIGS[sys.argv[1]]["dims"]))
PY
)
  skip=$(grep -c '"gpu__time_duration.sum"' gpurun_out/${TAG}_launches_$c.csv)
  hot=$(grep '"gpu__time_duration.sum"' gpurun_out/${TAG}_launches_$c.csv | grep -c -E 'k_stream2|k_mttkrp_stream')
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'^(k_stream2|k_mttkrp_stream)$' \
    -s $((hot - n)) -c $n -o gpurun_out/${TAG}_ncu_full_$c -f \
    python bench.py --config $c --profile --steps 2 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_full_$c.log 2>&1
  echo "ncu full $c rc=$? (skip $((hot - n)) of $hot streaming launches)"
done
