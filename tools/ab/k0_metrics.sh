# ncu counters of K0 (one steady-state launch) for the default and the corner-cache build.
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__inst_executed_op_global_ld.sum,smsp__sass_thread_inst_executed_op_global_ld_pred_on.sum,l1tex__data_pipe_lsu_wavefronts_mem_lg.sum
for v in default cache; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:k_map_forward_rec -s 3 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-tracking --no-dropin > gpurun_out/k0m_$v.csv 2>/dev/null
  echo $v $?
done
