"""The multi-GPU mapping driver on the real stack (libvoxrf_b200 + NCCL) at world
size 1: exercises the zero-copy tensor views of the context buffers, the NCCL
all-reduce / reduce-scatter / all-gather calls and the phase entry points
(vrf_map_forward / backward / apply) against a plain single-GPU mapping_step on
the same batch. (World sizes > 1 are covered on CPU by test_distributed_cpu.py;
this environment has one GPU.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2307_03404_b200 import Context, MappingConfig
from paper_2307_03404_b200.distributed import DistributedMapper, GpuEngine

from scenes import fresh_grid, room_scene

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("sparse", [False, True])
def test_nccl_world1_step_equals_single_gpu_step(oracle, sparse):
    grid, intr, frames = room_scene()
    g0 = fresh_grid(grid)
    cfg = MappingConfig()
    batch = oracle.draw_batch(3, len(frames), intr.width, intr.height, 2048)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0",
                      WORLD_SIZE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        a = Context(0, shard_multiple=1)
        a.set_stream(torch.cuda.current_stream().cuda_stream)
        a.load_grid(g0)
        a.load_frames(intr, frames)
        a.rmsprop_reset()
        mapper = DistributedMapper(GpuEngine(a, cfg))
        res = mapper.step(torch.from_numpy(batch).cuda(), cfg.lambda_d, sparse=sparse)
        # a second step: the RMSProp state carried on the block owners
        res = mapper.step(torch.from_numpy(batch[::-1].copy()).cuda(), cfg.lambda_d,
                          sparse=sparse)
        torch.cuda.synchronize()
        got = a.download_grid().data

        b = Context(0)
        b.load_grid(g0)
        b.load_frames(intr, frames)
        b.rmsprop_reset()
        b.mapping_step(cfg, batch)
        st = b.mapping_step(cfg, batch[::-1].copy())
        want = b.download_grid().data
    finally:
        dist.destroy_process_group()
    assert res.rays_color == st.rays_color and res.rays_depth == st.rays_depth
    assert res.samples == st.samples
    # two steps: the first update carries fp32 atomics-order noise into the second loss
    assert abs(res.loss_total - st.loss_total) <= 1e-6 * st.loss_total
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5 * np.abs(want).max())
