# usage: CFG=cfg2 KREGEX=k_stream2 SKIP=16 COUNT=4 TAG=x bash tools/gpu_ncu.sh
CFG=${CFG:-cfg2}; KREGEX=${KREGEX:-k_stream2}; SKIP=${SKIP:-16}; COUNT=${COUNT:-4}; TAG=${TAG:-run}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s $SKIP -c $COUNT \
  -o gpurun_out/ncu_${TAG}_${CFG} -f python bench.py --config $CFG --profile --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_${TAG}_${CFG}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_${TAG}_${CFG}.log
