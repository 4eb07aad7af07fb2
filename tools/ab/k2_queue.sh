# A/B of the K2 variants on bench config 3 (1M rays/step): queued convergent
# scatter with same-round merging (default), direct divergent scatter.
python -m pytest tests/test_gpu_parity.py -x -q -k "mapping or map" > gpurun_out/q_par.log 2>&1; tail -3 gpurun_out/q_par.log
run() { name=$1; shift; env "$@" python bench.py --no-cpu --no-tracking > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err; python -c "
import json; d=json.load(open('gpurun_out/ab_$name.json')); print('$name', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(v/5,2) for k,v in d['roofline']['kernel_ms'].items()})" ; }
run queued
run queued_minb3 VRF_REC_MINB=3
run direct VRF_K2=direct
run queued2
