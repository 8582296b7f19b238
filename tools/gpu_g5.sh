# full GPU suite + a short cfg5 bench (kernel boundary semantics changed for shards)
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g5_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/g5_pytest.log
timeout 900 python bench.py --only --steps 10 --warmup 3 --no-cpu > gpurun_out/g5_bench.json 2> gpurun_out/g5_bench.err; echo "bench rc=$?"
tail -2 gpurun_out/g5_bench.err
