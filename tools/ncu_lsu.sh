# On the GPU box: the binding-roofline counters (L1/shared-memory data-path wavefronts, DRAM
# bytes, L2->L1 bytes) of one timed sweep per config, with the plan the timed bench run chose
# (read from the bench line $BENCH, headline or per-config sub-record: kernel per mode and
# staged-level count), so the
# one-time kernel timing never runs under ncu.  Output: gpurun_out/${TAG}_lsu_<cfg>.csv, then
# `python tools/ncu_lsu.py` folds them into profiles/ncu_lsu.json (bench.py roofline.lsu).
# usage: TAG=r02 CFGS="cfg1 cfg2 cfg3 cfg4 cfg5" bash tools/ncu_lsu.sh
TAG=${TAG:-r02}; CFGS=${CFGS:-"cfg1 cfg2 cfg3 cfg4 cfg5"}; BENCH=${BENCH:-gpurun_out/${TAG}_bench.json}
M=l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds_cmd_read.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds_cmd_write.sum,l1tex__data_bank_reads.sum,l1tex__data_bank_writes.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_gds_op_ld.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct
for c in $CFGS; do
  envs=$(python tools/ncu_lsu.py --env $BENCH $c)
  echo "$c: $envs"
  env $envs timeout 1200 ncu --metrics $M --clock-control none --csv \
    -k regex:'^(k_stream2|k_sweep2|k_mttkrp_stream)$' --log-file gpurun_out/${TAG}_lsu_$c.csv \
    python bench.py --config $c --profile --steps 1 --warmup 3 --no-cpu > gpurun_out/${TAG}_lsu_$c.log 2>&1
  echo "ncu lsu $c rc=$?"
done
