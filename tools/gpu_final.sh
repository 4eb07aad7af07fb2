#!/bin/bash
# Round-end style check on one GPU: the -m gpu suite, smoke(), a bench line and
# the launch list of the same bench command. usage: tools/gpu_final.sh TAG
TAG=$1
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest=$?"; tail -3 gpurun_out/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke=$?"; tail -3 gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench=$?"; cut -c1-300 gpurun_out/${TAG}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu \
  > gpurun_out/${TAG}_launches.log 2>&1
echo "launches=$?"
