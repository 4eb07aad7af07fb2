"""Config-4 step anatomy: per-step wall time (synchronised) against the
profile slots (CUDA events per phase), to find time outside the kernels."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_2307_03404_b200 import Context, Rng, synth  # noqa: E402
from paper_2307_03404_b200.api import CameraIntrinsics, Frame, MappingConfig  # noqa: E402

room = synth.Room().scaled(7 / 4, 6 / 4, 1.0)
gt = synth.scene_grid(257, room, seed=2, prune_tau=1e-3)
intr = CameraIntrinsics(600, 600, 599.5, 339.5, 1200, 680, 6553.5)
path = synth.room_path(2000, room, seed=4)
g = Context(0)
g.load_grid(gt)
fr = []
for p in path[::10][:200]:
    im = g.render_image(intr, p)
    c, d = synth.quantize_frame(im.color, im.depth, intr.depth_scale)
    fr.append(Frame(c, d, 0, p))
del g
ctx = Context(0)
ctx.load_grid(gt)
ctx.upsample(1024)
ctx.prune(1e-3)
ctx.fill_grid(0.1)
ctx.load_frames(intr, fr)
ctx.rmsprop_reset()
cfg = MappingConfig()
rng = Rng(1)
NR = 1 << 23
bs = [torch.from_numpy(rng.draw_batch(200, 1200, 680, NR)).cuda() for _ in range(8)]
for i in range(3):
    ctx.mapping_step_device(cfg, bs[i].data_ptr(), NR)
torch.cuda.synchronize()
stream = torch.cuda.current_stream()
for i in range(3, 8):  # no profiling: host wall vs device time (events on the context stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    st = ctx.mapping_step_device(cfg, bs[i].data_ptr(), NR)
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"plain step {i}: wall {1e3 * (time.perf_counter() - t0):.1f} ms, device "
          f"{e0.elapsed_time(e1):.1f} ms", flush=True)
ctx.set_stream(stream.cuda_stream)
for i in range(3, 8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    st = ctx.mapping_step_device(cfg, bs[i].data_ptr(), NR)
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"torch-stream step {i}: wall {1e3 * (time.perf_counter() - t0):.1f} ms, device "
          f"{e0.elapsed_time(e1):.1f} ms", flush=True)
for i in range(3, 8):
    ctx.profile_enable(True)
    t0 = time.perf_counter()
    st = ctx.mapping_step_device(cfg, bs[i].data_ptr(), NR)
    torch.cuda.synchronize()
    wall = 1e3 * (time.perf_counter() - t0)
    pr = ctx.profile_read()
    ctx.profile_enable(False)
    slots = {k: round(v[0], 2) for k, v in pr.items() if isinstance(v, tuple) and v[0] > 0}
    print(f"step {i}: wall {wall:.1f} ms, samples {st.samples}, slots {slots}", flush=True)
