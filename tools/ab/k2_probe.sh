# Timing probe (r02), not an A/B of correct builds: K2 with its reductions
# removed (nored), with the duplicate merge disabled (nomerge), and both, to
# split K2's time between the L2 reductions and the merge. The probe builds
# compute wrong gradients; only the backward kernel time is read.
for rep in 1 2; do
for v in default nored nomerge nored_nomerge; do
  if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
  python bench.py --no-cpu --no-tracking --no-dropin --steps 10 > gpurun_out/probe_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/probe_$v.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$v', 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3), 'spr', round(d['samples_per_ray'],2))"
done
done
unset VRF_LIB
