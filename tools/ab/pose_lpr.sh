# A/B (r02): k_pose_group_u with 4 lanes per ray (two corners per lane, 8 rays per
# warp) against 8 (default). Build:
#   python tools/ab/build_variants.py lpr4=VRF_POSE_U_LPR=4 lpr4m4=VRF_POSE_U_LPR=4,VRF_POSE_U_MINB=4
# (LPR 4 sums the Jacobian partials in another order, so only the oracle-tolerance
# pose tests apply; the bit-identity test against the 8-lane checker does not.)
VRF_LIB=tools/ab/_lib_lpr4/libvoxrf_b200.so python -m pytest tests/test_gpu_pose.py -m gpu -q -k "oracle" > gpurun_out/lpr_t.log 2>&1; tail -1 gpurun_out/lpr_t.log
python -m pytest tests/test_gpu_pose.py -m gpu -q > gpurun_out/lpr_t8.log 2>&1; tail -1 gpurun_out/lpr_t8.log
for r in 1 2; do
  for v in default lpr4 lpr4m4; do
    if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
    echo -n "$v: "; python -c "import sys; sys.path.insert(0,'tools'); import track_bench as t; [t.main() for _ in range(2)]"
  done
done
unset VRF_LIB
