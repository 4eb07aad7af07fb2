# A/B (r02): K2 with relabelled corner slots — merge modes and CTAs/SM.
# Variants are prebuilt by: python tools/ab/build_variants.py nomerge=VRF_K2_MERGE=0 ...
for rep in 1 2; do
for v in default nomerge colmerge minb4 nomerge4 colmerge4; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  python bench.py --no-cpu --no-tracking --steps 10 > gpurun_out/k2v3_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/k2v3_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,2), 'bwd', round(k['map_backward']/n,2))"
done
done
unset VRF_LIB
