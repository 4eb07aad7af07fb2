# A/B (r02): Morton tile edge of the coherent ray order (VRF_RAY_TILE_LOG2;
# 4x4 pixels by default). Build:
#   python tools/ab/build_variants.py tile0=VRF_RAY_TILE_LOG2=0 tile1=VRF_RAY_TILE_LOG2=1 tile3=VRF_RAY_TILE_LOG2=3
for r in 1 2; do
  for v in default tile0 tile1 tile3; do
    if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
    python bench.py --no-cpu --no-tracking --no-dropin --steps 10 > gpurun_out/tile_$v.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/tile_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3))"
  done
done
unset VRF_LIB
