# A/B (r02): pose kernels at 64 threads per CTA (VRF_POSE_KT=64, 6 CTAs/SM: the
# same register cap) against 128 (default): finer CTAs for the wave tail. Build:
#   python tools/ab/build_variants.py kt64=VRF_POSE_KT=64,VRF_POSE_U_MINB=6
VRF_LIB=tools/ab/_lib_kt64/libvoxrf_b200.so python -m pytest tests/test_gpu_pose.py tests/test_gpu_parity.py -m gpu -x -q -k "pose or gn or track" > gpurun_out/kt_t.log 2>&1; tail -1 gpurun_out/kt_t.log
for r in 1 2; do
  for v in default kt64; do
    if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
    echo -n "$v: "; python -c "import sys; sys.path.insert(0,'tools'); import track_bench as t; [t.main() for _ in range(3)]"
  done
done
unset VRF_LIB
