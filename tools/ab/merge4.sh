# A/B (r02): K2 pairwise-first duplicate merge (VRF_K2_MERGE=4) against the
# factor-domain leader merge (default 3). Build:
#   python tools/ab/build_variants.py merge4=VRF_K2_MERGE=4
VRF_LIB=tools/ab/_lib_merge4/libvoxrf_b200.so python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast or gradient or k2q or overflow" > gpurun_out/m4_t.log 2>&1; tail -1 gpurun_out/m4_t.log
for r in 1 2; do
  for v in default merge4; do
    if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
    python bench.py --no-cpu --no-tracking --no-dropin --steps 10 > gpurun_out/m4_$v.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/m4_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3))"
  done
done
unset VRF_LIB
