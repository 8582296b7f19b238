# On the GPU box: launch lists + one ncu --set full capture of the hot kernel per config.
# usage: TAG=r01 CFGS="cfg2 cfg5" bash tools/profile_round.sh
# The fast path's one-time kernel timing is meaningless under ncu (serialised, replayed
# launches), so the profiled runs force the kernel the timed bench run chose
# (MKB_FAST_KERNEL, default s2 = level-ordered; see the bench JSON's roofline.per_mode).
export MKB_FAST_KERNEL=${MKB_FAST_KERNEL:-s2}
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
  hot=$(grep '"gpu__time_duration.sum"' gpurun_out/${TAG}_launches_$c.csv | grep -c -E 'k_stream2|k_sweep2|k_mttkrp_stream')
  # a fused sweep is one k_sweep2 launch; otherwise one launch per mode
  if grep -q k_sweep2 gpurun_out/${TAG}_launches_$c.csv; then n=1; fi
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'^(k_stream2|k_sweep2|k_mttkrp_stream)$' \
    -s $((hot - n)) -c $n -o gpurun_out/${TAG}_ncu_full_$c -f \
    python bench.py --config $c --profile --steps 2 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_full_$c.log 2>&1
  echo "ncu full $c rc=$? (skip $((hot - n)) of $hot streaming launches)"
done
