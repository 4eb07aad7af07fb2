# A/B (r02): K0 thread-per-ray gathers vs warp-cooperative corner staging in
# shared memory (-DVRF_K0_COOP=1). Parity of the variant first (the mapping
# parity tests with VRF_LIB set), then the bench and the L1 counters.
VRF_LIB=tools/ab/_lib_coop/libvoxrf_b200.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "mapping or gradient or record or config3 or small_batch" 2>&1 | tail -2
M=l1tex__data_pipe_lsu_wavefronts.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for rep in 1 2; do
for v in default coop; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  python bench.py --no-cpu --no-tracking --no-dropin --steps 10 > gpurun_out/k0coop_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k0coop_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3), 'spr', round(d['samples_per_ray'],4))"
  if [ $rep = 1 ]; then
    ncu --metrics $M --clock-control none -k regex:"k_map_forward_(rec|coop)" -s 3 -c 1 --csv \
      python bench.py --no-cpu --no-tracking --no-dropin --steps 1 --warmup 3 2>/dev/null \
      | grep -E '"(l1tex|gpu__|smsp)' | sed 's/"//g' | awk -F, '{print $(NF-2), $NF}'
  fi
done
done
unset VRF_LIB
