# A/B (r02) at config 4 (513^3 sparse, 8M rays): K2 factor merge at 4 CTAs/SM
# (default) vs 3 CTAs/SM vs the leader merge of expanded vectors.
for v in default k2minb3 merge1; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  python bench.py --config 4 --no-cpu --steps 5 > gpurun_out/c4k2_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/c4k2_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3), 'spr', round(d['samples_per_ray'],3))"
done
unset VRF_LIB
