"""Per-step wall time vs per-kernel CUDA-event time of the config-3 mapping step
(diagnostics: --torch-stream, --smi = nvidia-smi -lms 200 sampler running)."""
import sys, time, os
sys.path.insert(0, '/root/repo')
import torch, numpy as np
from paper_2307_03404_b200 import Context, Rng, synth
from paper_2307_03404_b200.api import MappingConfig, CameraIntrinsics, Frame
room = synth.Room().scaled(7/4, 6/4, 1.0)
gt = synth.scene_grid(257, room, seed=2, prune_tau=1e-3)
intr = CameraIntrinsics(600, 600, 599.5, 339.5, 1200, 680, 6553.5)
path = synth.room_path(100, room, seed=4)
g = Context(0); g.load_grid(gt)
fr = []
for p in path[::10][:10]:
    im = g.render_image(intr, p); c, d = synth.quantize_frame(im.color, im.depth, intr.depth_scale); fr.append(Frame(c, d, 0, p))
ctx = Context(0)
if "--torch-stream" in sys.argv:
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ctx.init_grid(gt.geom, 0.1); ctx.load_frames(intr, fr)
smi = None
if "--smi" in sys.argv:
    import subprocess
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "200"],
                           stdout=subprocess.DEVNULL)
cfg = MappingConfig()
rng = Rng(1)
NR = int(os.environ.get("RAYS", 1 << 20))
bs = [torch.from_numpy(rng.draw_batch(10, 1200, 680, NR)).cuda() for _ in range(8)]
for i in range(3): ctx.mapping_step_device(cfg, bs[i].data_ptr(), NR)
torch.cuda.synchronize()
ctx.profile_enable(True)
t0 = time.perf_counter()
tt = []
for i in range(3, 8):
    a = time.perf_counter()
    ctx.mapping_step_device(cfg, bs[i].data_ptr(), NR)
    tt.append(time.perf_counter() - a)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
pr = ctx.profile_read()
print("wall per step ms", 1e3 * dt / 5, [round(1e3 * x, 2) for x in tt])
print({k: (round(v[0] / 5, 3) if isinstance(v, tuple) else v) for k, v in pr.items()})
ctx.profile_enable(False)
t0 = time.perf_counter()
for i in range(3, 8):
    ctx.mapping_step_device(cfg, bs[i].data_ptr(), NR)
torch.cuda.synchronize()
print("wall per step ms, profiling off", 1e3 * (time.perf_counter() - t0) / 5)
if smi:
    smi.terminate()
