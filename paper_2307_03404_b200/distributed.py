"""Ray-sharded multi-GPU mapping: one process per GPU, the grid
replicated, each rank draws and processes its own rays (weak scaling).

Per step:
  1. forward on the local rays -> local partials (hit counts, loss sums)
  2. all-reduce of the partials (the upstream uses the GLOBAL 1/M_c, 1/M_d,
     mapping.cpp:181,188)
  3. backward with the global counts -> local fp32 gradient buffer [Vpad][28]
  4. reduce-scatter of the gradient onto equal vertex shards (NCCL over NVLink)
  5. fused RMSProp on the owned shard (skip g == 0), clears the gradient
  6. all-gather of the updated payload shards

The collectives are issued through torch.distributed on tensors that alias the
engine's device buffers (zero copy). The engine is libvoxrf_b200 on the GPU
(:class:`GpuEngine`); the CPU tests drive the same orchestration with an
oracle-backed engine over gloo.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


class _CudaArray:
    """Zero-copy view of context-owned device memory for torch (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<f4"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def shard_range(num_padded: int, world: int, rank: int):
    """Equal contiguous vertex shards [v0, v1) of the padded vertex count."""
    assert num_padded % world == 0
    per = num_padded // world
    return rank * per, (rank + 1) * per


@dataclass
class StepResult:
    loss_photometric: float
    loss_geometric: float
    loss_total: float
    rays_color: int
    rays_depth: int
    samples: int


class GpuEngine:
    """libvoxrf_b200 context as a distributed-mapping engine."""

    def __init__(self, ctx, config):
        self.ctx = ctx
        self.cfg = config
        b = ctx.device_buffers()
        self.num_vertices = int(b.num_vertices)
        self.padded = int(b.padded_vertices)
        dev = torch.device("cuda", ctx.device)
        self.grad = torch.as_tensor(_CudaArray(b.grad, self.padded * 28), device=dev)
        self.payload = torch.as_tensor(_CudaArray(b.payload, self.padded * 28), device=dev)

    def forward(self, batch):
        p = self.ctx.map_forward(self.cfg, batch.data_ptr(), batch.shape[0])
        return (p.rays_color, p.rays_depth, p.bad_ray, p.sum_photometric, p.sum_geometric,
                p.samples)

    def backward(self, m_color, m_depth):
        self.ctx.map_backward(self.cfg, m_color, m_depth)

    def apply(self, v0, v1):
        self.ctx.map_apply(self.cfg, v0, v1)


class DistributedMapper:
    def __init__(self, engine, group=None):
        self.e = engine
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.v0, self.v1 = shard_range(engine.padded, self.world, self.rank)
        self.shard = torch.empty((self.v1 - self.v0) * 28, dtype=engine.grad.dtype,
                                 device=engine.grad.device)
        self._rs = hasattr(dist, "reduce_scatter_tensor") and dist.get_backend(group) == "nccl"

    def step(self, batch, lambda_d: float) -> StepResult:
        m_c, m_d, bad, lp, lg, samples = self.e.forward(batch)
        dev = self.e.grad.device
        ints = torch.tensor([m_c, m_d, 1 if bad >= 0 else 0, samples], dtype=torch.int64,
                            device=dev)
        flts = torch.tensor([lp, lg], dtype=torch.float64, device=dev)
        dist.all_reduce(ints, group=self.group)
        dist.all_reduce(flts, group=self.group)
        M_c, M_d, n_bad, S = (int(x) for x in ints.tolist())
        if M_c == 0:
            raise RuntimeError("mapping_step: no ray hit the grid")
        if n_bad:
            raise RuntimeError("mapping_step: non-finite loss")
        self.e.backward(M_c, M_d)
        s0, s1 = self.v0 * 28, self.v1 * 28
        if self._rs:
            dist.reduce_scatter_tensor(self.shard, self.e.grad, group=self.group)
        else:  # gloo has no reduce-scatter: all-reduce and keep the owned slice
            dist.all_reduce(self.e.grad, group=self.group)
            self.shard.copy_(self.e.grad[s0:s1])
        self.e.grad.zero_()
        self.e.grad[s0:s1].copy_(self.shard)
        self.e.apply(self.v0, self.v1)
        mine = self.e.payload[s0:s1].clone()
        if hasattr(dist, "all_gather_into_tensor") and dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(self.e.payload, mine, group=self.group)
        else:
            parts = list(self.e.payload.view(self.world, -1).unbind(0))
            dist.all_gather(parts, mine, group=self.group)
            self.e.payload.copy_(torch.cat(parts))
        lp_sum, lg_sum = flts.tolist()
        l_p = lp_sum / M_c
        l_g = lg_sum / M_d if M_d > 0 else 0.0
        return StepResult(l_p, l_g, l_p + lambda_d * l_g, M_c, M_d, S)
