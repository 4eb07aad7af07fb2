# A/B (r02): paired pops (VRF_K2_POP2), leader merge (VRF_K2_MERGE=1), K0 at 3 CTAs/SM.
for rep in 1 2; do
for v in default pop2 merge1 k0minb3; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  python bench.py --no-cpu --no-tracking --no-dropin --steps 10 > gpurun_out/k2v6_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k2v6_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3), 'spr', round(d['samples_per_ray'],2))"
done
done
unset VRF_LIB
