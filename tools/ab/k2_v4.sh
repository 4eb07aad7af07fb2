# A/B (r02): K2 leader merge of expanded 28-vectors (default) vs factor-domain
# merge (members stage 4 factors, the leader expands them with the member's basis).
for rep in 1 2; do
for v in default fmerge; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  python bench.py --no-cpu --no-tracking --no-dropin --steps 10 > gpurun_out/k2v4_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k2v4_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3), 'spr', round(d['samples_per_ray'],2))"
done
done
unset VRF_LIB
