# A/B (r02): K0 through the per-lane corner cache (cache = VRF_K0_CACHE=1)
# against the default shade_fast on every corner, at config 3 and config 4.
# (A predicated variant, cache2, was measured once: 11.2 ms at config 3.)
for rep in 1 2; do
for v in default cache; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  for cfg in "--config 3" "--config 4"; do
    tag=$(echo "$cfg" | tr -d ' -')
    python bench.py --no-cpu --no-tracking --no-dropin --steps 10 $cfg > gpurun_out/k0c_${v}_$tag.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/k0c_${v}_$tag.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', '$tag', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3), 'spr', round(d['samples_per_ray'],2), 'loss', d.get('loss_last'))"
  done
done
done
unset VRF_LIB
