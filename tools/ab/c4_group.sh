# A/B (r02) at config 4: the 8-lanes-per-ray K0g / K2g (group-batched march) at
# every batch size vs the thread-per-ray K0 / K2q (default above 40K / 160K rays).
for v in default k0g k0g_k2g; do
  unset VRF_FWD_GROUP_MAX VRF_BWD_GROUP_MAX
  if [ $v != default ]; then export VRF_FWD_GROUP_MAX=1000000000; fi
  if [ $v = k0g_k2g ]; then export VRF_BWD_GROUP_MAX=1000000000; fi
  python bench.py --config 4 --no-cpu --steps 5 > gpurun_out/c4g_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/c4g_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3), 'spr', round(d['samples_per_ray'],3))"
done
for v in default k0g; do
  unset VRF_FWD_GROUP_MAX VRF_BWD_GROUP_MAX
  if [ $v != default ]; then export VRF_FWD_GROUP_MAX=1000000000; fi
  python bench.py --no-cpu --no-tracking --no-dropin --steps 5 > gpurun_out/c3g_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/c3g_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('c3 $v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3))"
done
