# A/B (r02): k_pose_group_u with 2 lanes per ray (four corners per lane, 16 rays
# per warp) against the default 4. Build:
#   python tools/ab/build_variants.py lpr2m4=VRF_POSE_U_LPR=2,VRF_POSE_U_MINB=4 lpr2m3=VRF_POSE_U_LPR=2,VRF_POSE_U_MINB=3
for v in lpr2m4 lpr2m3; do
  VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so python -m pytest tests/test_gpu_pose.py -m gpu -q -x > gpurun_out/lpr2_$v.log 2>&1; echo "$v tests: $(tail -1 gpurun_out/lpr2_$v.log)"
done
for r in 1 2; do
  for v in default lpr2m4 lpr2m3; do
    if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
    echo -n "$v: "; python -c "import sys; sys.path.insert(0,'tools'); import track_bench as t; [t.main() for _ in range(2)]"
  done
done
unset VRF_LIB
