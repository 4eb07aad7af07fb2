# A/B (r02): 1 / 3 pop rounds per walk step (VRF_K2_POPS) against 2, with
# the cell-record ring, config 3 and 4.
for rep in 1 2; do
for v in default pops1 pops3; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  for cfg in "--config 3" "--config 4"; do
    tag=$(echo "$cfg" | tr -d ' -')
    python bench.py --no-cpu --no-tracking --no-dropin --steps 10 $cfg > gpurun_out/pops_${v}_$tag.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/pops_${v}_$tag.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', '$tag', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3))"
  done
done
done
unset VRF_LIB
