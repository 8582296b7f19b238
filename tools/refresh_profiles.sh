# On the GPU box: the round's bench JSON lines (with CPU baselines) for every config, the
# reference arm on cfg2, and launch lists + one ncu --set full capture for cfg2 and cfg3.
# usage: TAG=r01 bash tools/refresh_profiles.sh
TAG=${TAG:-r01}
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "bench $c rc=$?"; cat gpurun_out/${TAG}_bench_$c.json | cut -c1-200
done
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference_cfg2.json 2> gpurun_out/${TAG}_bench_reference_cfg2.err
echo "reference rc=$?"
TAG=$TAG CFGS="cfg2" bash tools/profile_round.sh
# cfg3's timed run re-plans every mode to K = 0 (L1-fed gathers): profile that plan
MKB_FORCE_K=0,0,0,0 TAG=$TAG CFGS="cfg3" bash tools/profile_round.sh
# cfg5's and cfg1's timed runs keep K = 1 (one inner level staged); the cost model alone
# would pick K = 2, so the profiled runs force the timed choice
MKB_FORCE_K=1,1,1 TAG=$TAG CFGS="cfg5 cfg1" bash tools/profile_round.sh
