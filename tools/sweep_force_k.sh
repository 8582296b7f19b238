# usage: CFG=cfg2 KS="auto 0,0,0,0 ..." bash tools/sweep_force_k.sh  (GPU box; MKB_FORCE_K per mode)
export BENCH_FLAGS=--no-cpu
for c in ${CFG:-cfg3}; do
for fk in ${KS:-auto}; do
  if [ $fk = auto ]; then unset MKB_FORCE_K; else export MKB_FORCE_K=$fk; fi
  echo "== $c $fk"; MKB_DEBUG=1 bash tools/bench_configs.sh $c fk$fk
  grep "plan:" gpurun_out/bench_fk${fk}_$c.err | sed 's/levels.*blocked/blocked/; s/outer-in-record.*model/model/' | head -5
done; done
