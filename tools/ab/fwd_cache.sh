# A/B: K0 with the per-thread shared-memory cell cache (1: 142 regs, 2: capped
# at 4 CTAs/SM) against the plain gather (0)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_kats.py -x -q > gpurun_out/fc_t.log 2>&1; tail -2 gpurun_out/fc_t.log
for v in 0 1 2 0 1; do
  VRF_FWD_CACHE=$v python bench.py --no-cpu --no-tracking > gpurun_out/fc_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/fc_$v.json')); print('$v', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(v/5,2) for k,v in d['roofline']['kernel_ms'].items()})"
done
