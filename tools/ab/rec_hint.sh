# A/B (r02): sample records at L2 evict-first priority. Default since r02:
# K0 stores hinted (VRF_REC_HINT=1); nohint = 0, hintall = 3 (K2 loads too).
for rep in 1 2; do
for v in default nohint hintall; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  for cfg in "--config 3" "--config 4"; do
    tag=$(echo "$cfg" | tr -d ' -')
    python bench.py --no-cpu --no-tracking --no-dropin --steps 10 $cfg > gpurun_out/hint_${v}_$tag.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/hint_${v}_$tag.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', '$tag', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3))"
  done
done
done
unset VRF_LIB
