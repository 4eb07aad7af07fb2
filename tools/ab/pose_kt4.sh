# A/B (r02): the 4-lane GN pose kernel at 64 threads per CTA (16 rays, 8 CTAs/SM,
# the same 128-register cap) against 128 (default): at 16K rays the launch is one
# wave of 512 CTAs over 592 slots; finer CTAs balance the SMs. Build:
#   python tools/ab/build_variants.py kt64l4=VRF_POSE_KT=64,VRF_POSE_U_MINB=8
VRF_LIB=tools/ab/_lib_kt64l4/libvoxrf_b200.so python -m pytest tests/test_gpu_pose.py -m gpu -q -x > gpurun_out/kt4_t.log 2>&1; echo "tests: $(tail -1 gpurun_out/kt4_t.log)"
for r in 1 2 3; do
  for v in default kt64l4; do
    if [ $v = default ]; then unset VRF_LIB; else export VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so; fi
    echo -n "$v: "; python -c "import sys; sys.path.insert(0,'tools'); import track_bench as t; [t.main() for _ in range(2)]"
  done
done
unset VRF_LIB
