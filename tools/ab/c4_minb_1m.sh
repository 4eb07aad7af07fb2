# A/B (r02): K2 at 3 vs 4 CTAs/SM on config 4 at 1M rays per batch (the per-rank
# batch of an 8-GPU config-4 run): is the 3-CTA preference about the batch or
# the 513^3 grid? VRF_K2_MINB3_RAYS=0 forced 3 CTAs/SM (the knob was the batch size then; now VRF_K2_MINB3_VERTS).
for r in 1 2; do
  for v in 4 3; do
    if [ $v = 3 ]; then export VRF_K2_MINB3_VERTS=100000000000; else unset VRF_K2_MINB3_VERTS; fi
    python bench.py --config 4 --rays 1048576 --no-cpu --steps 5 > gpurun_out/c4m_$v.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/c4m_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('ctas=$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3))"
  done
done
unset VRF_K2_MINB3_VERTS
