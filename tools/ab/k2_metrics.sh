# ncu counters of K2 (one steady-state launch) for the default and an A/B build.
# usage: tools/ab/k2_metrics.sh VARIANT
M=gpu__time_duration.sum,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed,l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum,smsp__inst_executed_op_global_red.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__inst_executed_op_local_ld.sum,smsp__inst_executed_op_local_st.sum
for v in default $1; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:k_map_backward_q -s 3 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-tracking --no-dropin > gpurun_out/k2m_$v.csv 2>/dev/null
  echo $v $?
done
