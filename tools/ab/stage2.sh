# A/B (r02): double-buffered merge staging, one barrier per pop round (stage2 =
# VRF_K2_STAGE2=1), config 3, 4 and 32K rays; then the parity tests on it.
for rep in 1 2; do
for v in default stage2; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  for cfg in "--config 3" "--config 4" "--config 3 --rays 32768"; do
    tag=$(echo "$cfg" | tr -d ' -')
    python bench.py --no-cpu --no-tracking --no-dropin --steps 10 $cfg > gpurun_out/stage2_${v}_$tag.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/stage2_${v}_$tag.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', '$tag', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3), 'spr', round(d['samples_per_ray'],2))"
  done
done
done
unset VRF_LIB
export VRF_LIB=tools/ab/_lib_stage2/libvoxrf_b200.so
timeout 600 python -m pytest tests -m gpu -x -q -k "parity or configs or records or backward" 2>&1 | tail -2
unset VRF_LIB
