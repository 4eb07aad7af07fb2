# A/B (r02): K0 with the preferred shared-memory carveout at 0 % / 10 % (max
# L1) against the driver default, at config 3, config 4 and a 32K-ray batch.
for rep in 1 2; do
for v in default carve0 carve10; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  for cfg in "--config 3" "--config 4" "--config 3 --rays 32768"; do
    tag=$(echo "$cfg" | tr -d ' -')
    python bench.py --no-cpu --no-tracking --no-dropin --steps 10 $cfg > gpurun_out/carve_${v}_$tag.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/carve_${v}_$tag.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', '$tag', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3), 'spr', round(d['samples_per_ray'],2))"
  done
done
done
unset VRF_LIB
