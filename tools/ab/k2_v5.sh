# A/B (r02): K2 with 32 B records (cell + midpoint stored, fp32 decode):
# 3 vs 4 CTAs/SM (VRF_K2_MINB) and leader vs factor-domain merge (VRF_K2_MERGE 1 / 3).
for rep in 1 2; do
for v in default minb4 merge1; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  python bench.py --no-cpu --no-tracking --no-dropin --steps 10 > gpurun_out/k2v5_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k2v5_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3), 'spr', round(d['samples_per_ray'],2))"
done
done
unset VRF_LIB
