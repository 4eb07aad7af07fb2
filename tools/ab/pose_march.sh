# A/B: group-batched march (default) vs segment-by-segment march in k_pose_group
python -m pytest tests -m gpu -x -q -k "pose or track or slam or gn" > gpurun_out/pm_t.log 2>&1; tail -2 gpurun_out/pm_t.log
for v in par serial par2; do
  if [ $v = serial ]; then export VRF_POSE_MARCH=serial; else unset VRF_POSE_MARCH; fi
  python bench.py --no-cpu > gpurun_out/pm_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pm_$v.json')); t=d['tracking']; print('$v', round(t['frames_per_s'],1), round(t['samples_per_s']/1e6,1), round(t['roofline']['frac'],3), t['ate_rmse_m'])"
done
