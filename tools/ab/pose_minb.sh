# A/B (r02): k_pose_group_u at 3 CTAs/SM (default, 168-register cap) vs 4
# (VRF_POSE_U_MINB=4: 128 registers, no spills once the ray origin is read from
# the pose instead of kept live). Build:
#   python tools/ab/build_variants.py poseu4=VRF_POSE_U_MINB=4
VRF_LIB=tools/ab/_lib_poseu4/libvoxrf_b200.so python -m pytest tests/test_gpu_pose.py tests/test_gpu_parity.py -m gpu -x -q -k "pose or gn or track" > gpurun_out/pm_t.log 2>&1; tail -1 gpurun_out/pm_t.log
for r in 1 2 3; do
  for v in default poseu4; do
    if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
    echo -n "$v: "; python -c "import sys; sys.path.insert(0,'tools'); import track_bench as t; [t.main() for _ in range(3)]"
  done
done
unset VRF_LIB
