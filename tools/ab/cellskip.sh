# A/B: march with / without the cell-level jump inside occupied blocks
python bench.py --no-cpu > gpurun_out/cs_A.json 2> gpurun_out/cs_A.err
python tools/configs12.py --help > /dev/null 2>&1
VRF_EXTRA_NVCC_FLAGS=-DVRF_NO_CELL_SKIP python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cs_build.log 2>&1
python bench.py --no-cpu > gpurun_out/cs_B.json 2> gpurun_out/cs_B.err
python -c "import __graft_entry__ as g; g.build()" >> gpurun_out/cs_build.log 2>&1
python bench.py --no-cpu > gpurun_out/cs_A2.json 2> gpurun_out/cs_A2.err
for n in A B A2; do python -c "
import json; d=json.load(open('gpurun_out/cs_$n.json')); t=d['tracking']; print('$n', round(d['value']/1e9,3), round(t['frames_per_s'],1), round(t['samples_per_s']/1e6,1), t['ate_rmse_m'])"; done
