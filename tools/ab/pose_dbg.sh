for v in pdbg3 pdbg4; do
  VRF_LIB=tools/ab/_lib_$v/libvoxrf_b200.so timeout 300 python -m pytest tests/test_gpu_pose.py -m gpu -x -q -s -k "normal_equations_match_oracle" > gpurun_out/$v.log 2>&1
  echo "== $v"; grep dbg gpurun_out/$v.log | head -40
done
