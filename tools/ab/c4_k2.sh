# config 4 (513^3 sparse, 8M rays): queued vs direct K2
for v in queued direct queued; do
  if [ $v = direct ]; then export VRF_K2=direct; else unset VRF_K2; fi
  python bench.py --config 4 --no-cpu --no-tracking > gpurun_out/c4k2_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/c4k2_$v.json')); r=d['roofline']; print('$v', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(x,1) for k,x in r['kernel_ms'].items()}, r['launches'])"
done
