# A/B (r02): K2q with the per-warp vertex cache (vcache = VRF_K2_VCACHE=1)
# against the default, config 3 and 4; then the fast-path parity tests on the
# cache build.
for rep in 1 2; do
for v in default vcache; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  for cfg in "--config 3" "--config 4"; do
    tag=$(echo "$cfg" | tr -d ' -')
    python bench.py --no-cpu --no-tracking --no-dropin --steps 10 $cfg > gpurun_out/vc_${v}_$tag.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/vc_${v}_$tag.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', '$tag', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3), 'spr', round(d['samples_per_ray'],2))"
  done
done
done
export VRF_LIB=tools/ab/_lib_vcache/libvoxrf_b200.so
timeout 600 python -m pytest tests -m gpu -x -q -k "parity or configs or records or backward" 2>&1 | tail -3
unset VRF_LIB
