# A/B (r02): duplicate groups split into sub-groups of at most 3 / 4 / 6 lanes
# (VRF_K2_GROUP_MAX; bounds the serial leader loop at the price of one more
# reduction per extra sub-group) against unbounded groups, config 3 and 4.
for rep in 1 2; do
for v in default gmax3 gmax4 gmax6; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  for cfg in "--config 3" "--config 4"; do
    tag=$(echo "$cfg" | tr -d ' -')
    python bench.py --no-cpu --no-tracking --no-dropin --steps 10 $cfg > gpurun_out/gmax_${v}_$tag.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/gmax_${v}_$tag.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', '$tag', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3))"
  done
done
done
unset VRF_LIB
