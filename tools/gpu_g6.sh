timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g6_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/g6_pytest.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ugj tools/ubench_gj.cu && /tmp/ugj > gpurun_out/ubench_gj.txt 2>&1; cat gpurun_out/ubench_gj.txt
for c in cfg2 cfg3; do MKB_ALS_PROF=1 timeout 300 python tools/als_probe.py $c > gpurun_out/als_prof_$c.txt 2>&1; tail -6 gpurun_out/als_prof_$c.txt; done
bash tools/sanitize.sh
