mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "k2q_three or larger_batches" > gpurun_out/r02x_pytest.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/r02x_pytest.log
python bench.py > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err; echo "bench=$?"
python bench.py --config 4 --no-cpu --steps 5 > gpurun_out/r02x_c4.json 2> gpurun_out/r02x_c4.err; echo "c4=$?"
VRF_K2_MINB3_VERTS=100000000000 python bench.py --config 4 --no-cpu --steps 5 > gpurun_out/r02x_c4_minb4.json 2> gpurun_out/r02x_c4_minb4.err; echo "c4b=$?"
for f in r02x_c4 r02x_c4_minb4; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); k=d['roofline']['kernel_ms']; n=d['steps']
print('$f', round(d['value']/1e9,3), 'fwd', round(k['map_forward']/n,3), 'bwd', round(k['map_backward']/n,3))"; done
