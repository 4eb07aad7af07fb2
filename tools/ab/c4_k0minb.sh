# A/B (r02): K0 at 3 CTAs/SM (VRF_K0_MINB=3, no spills) vs 4 (default) on config 4
# (march-bound through occupied shell blocks). Build:
#   python tools/ab/build_variants.py k0m3=VRF_K0_MINB=3
for r in 1 2; do
  for v in default k0m3; do
    if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
    python bench.py --config 4 --no-cpu --steps 5 > gpurun_out/c4k0_$v.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/c4k0_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3))"
  done
done
unset VRF_LIB
