# A/B: queued K2 with same-round duplicate merging (VRF_K2_MERGE=1) vs without,
# config 3 (dense, 1M rays) and config 4 (sparse 513^3, 8M rays)
VRF_K2_MERGE=1 python -m pytest tests/test_gpu_parity.py -x -q -k "map" > gpurun_out/km_t.log 2>&1; tail -1 gpurun_out/km_t.log
for c in 3 4; do for v in 1 0; do
  VRF_K2_MERGE=$v python bench.py --config $c --no-cpu --no-tracking > gpurun_out/km_${c}_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/km_${c}_$v.json')); r=d['roofline']; print('config $c merge=$v', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(x/5,2) for k,x in r['kernel_ms'].items()})"
done; done
