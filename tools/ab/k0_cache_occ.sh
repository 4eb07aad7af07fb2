# A/B (r02): the K0 corner-cache build at 4 / 5 / 6 CTAs per SM (cache, cache5,
# cache6) against the default, config 3.
for rep in 1 2; do
for v in default cache cache5 cache6; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  python bench.py --no-cpu --no-tracking --no-dropin --steps 10 > gpurun_out/k0o_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k0o_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3))"
done
done
unset VRF_LIB
