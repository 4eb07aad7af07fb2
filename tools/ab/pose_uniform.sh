# A/B: warp-synchronous GN pose kernel (k_pose_group_u, default) vs the
# group-independent k_pose_group (VRF_POSE_UNIFORM=0)
python -m pytest tests -m gpu -x -q -k "track or slam or pose or gn" > gpurun_out/pu_t.log 2>&1; tail -1 gpurun_out/pu_t.log
for v in 1 0 1 0; do
  VRF_POSE_UNIFORM=$v python bench.py --no-cpu --rays 65536 > gpurun_out/pu_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pu_$v.json')); t=d['tracking']; print('uniform=$v', round(t['frames_per_s'],1), t['ate_rmse_m'], round(t['throughput_probe']['samples_per_s']/1e9,3))"
done
