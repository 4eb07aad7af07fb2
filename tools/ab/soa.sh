# A/B (r02): K0's corner gathers from the [V][7] float4 AoS payload
# (default) vs a channel-group-planar [7][V] copy (-DVRF_GATHER_SOA, refreshed by
# a transpose before each forward, timed separately in map_misc).
# prebuilt: python tools/ab/build_variants.py soa=VRF_GATHER_SOA
M=l1tex__data_pipe_lsu_wavefronts.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_active
for rep in 1 2; do
for v in default soa; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  python bench.py --no-cpu --no-tracking --no-dropin --steps 10 > gpurun_out/soa_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/soa_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']; o=d['roofline']['other_ms']
print('$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3), 'misc', round(o.get('misc',0)/n,3))"
  if [ $rep = 1 ]; then
    ncu --metrics $M --clock-control none -k regex:k_map_forward_rec -s 3 -c 1 --csv \
      python bench.py --no-cpu --no-tracking --no-dropin --steps 1 --warmup 3 2>/dev/null \
      | grep -E '"(l1tex|lts|dram|gpu__|smsp)' > gpurun_out/soa_ncu_$v.csv
    cut -d, -f13- gpurun_out/soa_ncu_$v.csv | sed 's/"//g'
  fi
done
done
unset VRF_LIB
