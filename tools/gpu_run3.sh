timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
BENCH_FLAGS=--no-cpu bash tools/bench_configs.sh "${CFGS:-cfg2 cfg1 cfg3 cfg4 cfg5}" ${TAG:-v21}
[ -n "$NCU" ] && CFG=cfg2 TAG=${TAG:-v21} bash tools/gpu_ncu.sh
true
