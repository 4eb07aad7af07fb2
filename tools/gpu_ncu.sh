#!/bin/bash
# ncu --set full of the bench's steady-state K0 / K2 launches (config 3), plus
# the launch list of the same command. usage: tools/gpu_ncu.sh TAG [bench args]
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"k_map_backward_q|k_map_forward_rec" -s 6 -c 2 -o gpurun_out/${TAG}_ncu \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-tracking "$@" > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu "$@" \
  > gpurun_out/${TAG}_launches.log 2>&1
echo "launches=$?"
