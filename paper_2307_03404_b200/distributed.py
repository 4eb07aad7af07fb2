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
        # the NCCL collectives run on torch's current stream: the context's kernels
        # must run on that same stream, or a reduce-scatter could read the gradient
        # before map_backward has finished writing it
        ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
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

    # ---- block-sparse exchange (8^3-vertex blocks, packed [n][512][28] fp32)
    BLOCK_FLOATS = 512 * 28

    @property
    def n_blocks(self) -> int:
        return self.ctx.blocks_count()

    def touched_flags(self):
        f = torch.empty(self.n_blocks, dtype=torch.uint8, device=self.grad.device)
        self.ctx.blocks_touched(f.data_ptr())
        return f

    def pack(self, ids, which):
        out = torch.empty(ids.numel() * self.BLOCK_FLOATS, dtype=torch.float32,
                          device=self.grad.device)
        self.ctx.blocks_pack(ids.data_ptr(), ids.numel(), which, out.data_ptr())
        return out

    def apply_blocks(self, ids, packed_grad):
        self.ctx.blocks_apply(self.cfg, ids.data_ptr(), ids.numel(), packed_grad.data_ptr())

    def unpack_payload(self, ids, packed):
        self.ctx.blocks_unpack_payload(ids.data_ptr(), ids.numel(), packed.data_ptr())

    def clear_grad(self):
        self.ctx.grad_clear()

    # ---- fused peer-memory exchange (one kernel, vrf_exchange_p2p)
    def ipc_export(self) -> bytes:
        return self.ctx.ipc_export()

    def open_peers(self, rank, handles):
        self.ctx.peers_open_ipc(rank, handles)

    def exchange_p2p(self):
        self.ctx.exchange_p2p(self.cfg)


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

    def step(self, batch, lambda_d: float, sparse: bool = False,
             exchange: str = None) -> StepResult:
        """One ray-sharded mapping step. exchange: "dense" (reduce-scatter /
        all-gather of the whole gradient / payload), "sparse" (only the 8^3-vertex
        blocks some rank touched, _exchange_sparse) or "p2p" (the fused peer-memory
        kernel, _exchange_p2p). The older flag sparse=True means "sparse"."""
        exchange = exchange or ("sparse" if sparse else "dense")
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
        if exchange == "p2p" and not self.prepare_p2p():
            exchange = "sparse"  # peer memory unavailable on some rank (p2p_error)
        if exchange == "p2p":
            self._exchange_p2p()
        elif exchange == "sparse":
            self._exchange_sparse()
        elif exchange == "dense":
            self._exchange_dense()
        else:
            raise ValueError(f"unknown exchange {exchange!r}")
        lp_sum, lg_sum = flts.tolist()
        l_p = lp_sum / M_c
        l_g = lg_sum / M_d if M_d > 0 else 0.0
        return StepResult(l_p, l_g, l_p + lambda_d * l_g, M_c, M_d, S)

    def _barrier(self):
        """Stream-ordered barrier: with NCCL a one-element all-reduce on the current
        stream (every rank's earlier kernels are complete when it returns on the
        device); other backends synchronise the device and barrier on the host."""
        if dist.get_backend(self.group) == "nccl":
            if not hasattr(self, "_tok"):
                self._tok = torch.zeros(1, dtype=torch.int32, device=self.e.grad.device)
            dist.all_reduce(self._tok, group=self.group)
        else:
            torch.cuda.synchronize(self.e.grad.device)
            dist.barrier(group=self.group)

    def prepare_p2p(self) -> bool:
        """Opens every rank's gradient / payload / touched bitmap over CUDA IPC.
        Collective: every rank must call it. Returns False on every rank if any
        rank could not open its peers (then the step falls back to the NCCL
        block-sparse exchange; the reason is kept in p2p_error)."""
        if getattr(self, "_peers_open", None) is not None:
            return self._peers_open
        err = ""
        try:
            mine = self.e.ipc_export()
        except RuntimeError as e:
            mine, err = b"", str(e)
        handles = [None] * self.world
        dist.all_gather_object(handles, mine, group=self.group)
        if not err and all(handles):
            try:
                self.e.open_peers(self.rank, handles)
            except RuntimeError as e:
                err = str(e)
        elif not err:
            err = "a peer could not export its buffers"
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=self.e.grad.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        self._peers_open = bool(ok.item())
        self.p2p_error = err or (None if self._peers_open else "a peer could not open the table")
        return self._peers_open

    def _exchange_p2p(self):
        """Fused exchange over peer memory: every rank's backward done (barrier) ->
        ONE kernel per rank: the owner of each touched block sums all ranks'
        gradients over NVLink, applies RMSProp and writes the payload block into
        every rank -> barrier -> local gradient clear. The peer table (IPC handles
        of every rank's gradient / payload / touched bitmap) is set up once."""
        if not getattr(self, "_peers_open", False):
            raise RuntimeError("p2p exchange without a peer table (prepare_p2p)")
        self._barrier()
        self.e.exchange_p2p()
        self._barrier()
        self.e.clear_grad()

    def _exchange_dense(self):
        s0, s1 = self.v0 * 28, self.v1 * 28
        if self.world == 1:  # the local gradient is the global one: apply in place
            self.e.apply(self.v0, self.v1)
            return
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

    def _exchange_sparse(self):
        """Block-sparse exchange. Blocks have a STATIC owner (id % world), so each
        block's RMSProp state lives on one rank across steps. The touched flags
        are max-all-reduced (same list on every rank); each owner's touched blocks
        are padded to the largest owner count M so the packed gradient
        [world][M][512][28] reduce-scatters into equal shards; the owner applies
        RMSProp to its M blocks and the updated payload blocks are all-gathered
        and unpacked everywhere. Untouched blocks have zero gradient on every
        rank, so the result equals the dense exchange."""
        flags = self.e.touched_flags()
        dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=self.group)
        ids = torch.nonzero(flags).flatten().to(torch.int32)
        dev = flags.device
        groups = [ids[(ids % self.world) == r] for r in range(self.world)]
        M = max(int(g.numel()) for g in groups)
        if M > 0:
            pad = torch.full((self.world, M), -1, dtype=torch.int32, device=dev)
            for r, g in enumerate(groups):
                pad[r, : g.numel()] = g
            all_ids = pad.flatten().contiguous()
            mine_ids = pad[self.rank].contiguous()
            packed = self.e.pack(all_ids, 0)
            shard = torch.empty(M * self.e.BLOCK_FLOATS, dtype=packed.dtype, device=dev)
            if self._rs:
                dist.reduce_scatter_tensor(shard, packed, group=self.group)
            else:
                dist.all_reduce(packed, group=self.group)
                shard.copy_(packed.view(self.world, -1)[self.rank])
            self.e.apply_blocks(mine_ids, shard)
            theta = self.e.pack(mine_ids, 1)
            gathered = torch.empty(self.world * theta.numel(), dtype=theta.dtype, device=dev)
            if hasattr(dist, "all_gather_into_tensor") and dist.get_backend(self.group) == "nccl":
                dist.all_gather_into_tensor(gathered, theta, group=self.group)
            else:
                parts = list(gathered.view(self.world, -1).unbind(0))
                dist.all_gather(parts, theta, group=self.group)
                gathered = torch.cat(parts)
            self.e.unpack_payload(all_ids, gathered)
        self.e.clear_grad()


# ---------------------------------------------------------------- tracking
def lm_step(jtj: np.ndarray, jtr: np.ndarray, damping: float, pose):
    """The damped Gauss-Newton step of k_gn_step on the host: solve
    (A + damping diag(A) + 1e-12 I) x = -J^T r, then apply x = [omega; tau] as
    PosePerturbation::applied_to (tracking.hpp:21-26): q <- normalize(exp(omega) q),
    t <- t + tau, exp_so3 as pose.hpp:32-41. Returns the new pose, or None if the
    system is not positive definite (the pose is then kept)."""
    from .api import Pose
    A = np.array(jtj, dtype=np.float64).reshape(6, 6).copy()
    A[np.diag_indices(6)] += damping * np.diag(A) + 1e-12
    try:
        L = np.linalg.cholesky(A)
    except np.linalg.LinAlgError:
        return None
    x = np.linalg.solve(L.T, np.linalg.solve(L, -np.asarray(jtr, dtype=np.float64)))
    w = x[:3]
    angle = float(np.sqrt((w[0] * w[0] + w[1] * w[1]) + w[2] * w[2]))
    if angle < 1e-8:
        e = np.array([1.0, 0.5 * w[0], 0.5 * w[1], 0.5 * w[2]])
        e /= np.linalg.norm(e)
    else:
        ha = 0.5 * angle
        e = np.concatenate([[np.cos(ha)], np.sin(ha) / angle * w])
    b = np.asarray(pose.q, dtype=np.float64)
    q = np.array([e[0] * b[0] - e[1] * b[1] - e[2] * b[2] - e[3] * b[3],
                  e[0] * b[1] + e[1] * b[0] + e[2] * b[3] - e[3] * b[2],
                  e[0] * b[2] + e[2] * b[0] + e[3] * b[1] - e[1] * b[3],
                  e[0] * b[3] + e[3] * b[0] + e[1] * b[2] - e[2] * b[1]])
    q /= np.linalg.norm(q)
    return Pose(tuple(q), tuple(np.asarray(pose.t, dtype=np.float64) + x[3:]))


@dataclass
class TrackResult:
    pose: object
    loss_trace: list
    rays_used: list


class DistributedTracker:
    """Ray-sharded Gauss-Newton / LM tracking (the north star's
    "tracking all-reduces only the 21+6-float normal equations"). Each rank draws
    its own valid-depth pixels (tracking.cpp:147-166 rule, rank-specific stream),
    evaluates their normal equations on its device (vrf_pose_normal_equations:
    one march per ray, per-ray 4x6 Jacobian, J^T J / J^T r sums), the 21 + 6 sums,
    the loss and the hit count are all-reduced (29 fp64 = 232 B), and every rank
    takes the identical damped step (lm_step). Worth it only when one frame's
    rays per iteration exceed what one GPU turns around in a few microseconds
    (>= 64K rays); below that, tracking runs as replicas."""

    def __init__(self, engine_ctx, intrinsics, config, group=None):
        from .api import TrackingConfig
        self.ctx = engine_ctx
        self.intr = intrinsics
        self.cfg = config
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.loss_cfg = TrackingConfig(lambda_p=config.lambda_p, lambda_d=config.lambda_d,
                                       render=config.render)
        self.device = torch.device("cuda", engine_ctx.device) \
            if dist.get_backend(group) == "nccl" else torch.device("cpu")

    def _normal_equations(self, slot, pose, pixels):
        return self.ctx.pose_normal_equations(slot, self.intr, pose, pixels, self.loss_cfg)

    def track(self, slot: int, depth: np.ndarray, init_pose, frame_seed: int = 0) -> TrackResult:
        """Tracks the frame in context slot `slot` (its depth image on the host for
        the pixel draws) from init_pose; cfg.iterations steps."""
        from .api import Rng
        n_local = self.cfg.rays_per_iteration // self.world + \
            (1 if self.rank < self.cfg.rays_per_iteration % self.world else 0)
        rng = Rng(self.cfg.seed + 0x9E3779B9 * frame_seed + 7919 * self.rank)
        pose = init_pose
        trace, used = [], []
        for _ in range(self.cfg.iterations):
            px = rng.draw_valid_pixels(depth, n_local, self.cfg.max_redraws)
            v = np.zeros(29)
            ne = None
            if len(px):
                try:
                    ne = self._normal_equations(slot, pose, px)
                except RuntimeError as e:  # this rank's rays all missed: others may not
                    if "untrackable" not in str(e):
                        raise
            if ne is not None:
                iu = np.triu_indices(6)
                v[:21] = ne.jtj[iu]
                v[21:27] = ne.jtr
                v[27] = ne.loss
                v[28] = ne.rays_used
            t = torch.from_numpy(v).to(self.device)
            dist.all_reduce(t, group=self.group)
            v = t.cpu().numpy()
            m = int(round(v[28]))
            trace.append(v[27] / m if m else 0.0)
            used.append(m)
            if m == 0:  # tracking.cpp:97 on the global sample
                raise RuntimeError("untrackable frame: all sampled rays miss the grid")
            jtj = np.zeros((6, 6))
            jtj[np.triu_indices(6)] = v[:21]
            jtj = jtj + np.triu(jtj, 1).T
            nxt = lm_step(jtj, v[21:27], self.cfg.damping, pose)
            if nxt is None:
                break
            pose = nxt
        return TrackResult(pose, trace, used)
