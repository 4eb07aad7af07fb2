#!/bin/bash
# One GPU round trip: the -m gpu suite, a bench line, and an ncu capture of the
# bench's steady-state K0/K2 launches. usage: tools/gpu_round.sh TAG [pytest-args]
TAG=$1; shift
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --durations=15 "$@" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest=$?"; tail -25 gpurun_out/${TAG}_pytest.log
python bench.py --no-cpu > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench=$?"; cut -c1-400 gpurun_out/${TAG}_bench.json
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"k_map_backward_q|k_map_forward_rec" -s 6 -c 2 -o gpurun_out/${TAG}_ncu \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-tracking > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu=$?"
