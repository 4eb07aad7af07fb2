"""Multi-GPU mapping orchestration (paper_2307_03404_b200/distributed.py) on CPU:
world size 2 over gloo, with an oracle-backed engine standing in for the GPU
context. One ray-sharded step (forward -> all-reduce of the partials -> backward
with the GLOBAL hit counts -> reduce-scatter -> RMSProp on the owned vertex
shard -> all-gather) must equal a single-process mapping_step over the
concatenated batch."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleEngine:
    """CPU engine with the GpuEngine interface (oracle restatement underneath)."""

    def __init__(self, grid, frames, intr, cfg, world):
        import oracle as orc
        self.o = orc.Oracle()
        self.grid, self.frames, self.intr, self.cfg = grid, frames, intr, cfg
        self.num_vertices = grid.geom.num_vertices
        self.padded = (self.num_vertices + world - 1) // world * world
        self.payload = torch.zeros(self.padded * 28, dtype=torch.float64)
        self.payload[: self.num_vertices * 28] = torch.from_numpy(grid.data.reshape(-1))
        self.grad = torch.zeros(self.padded * 28, dtype=torch.float64)
        self.v = torch.zeros(self.padded * 28, dtype=torch.float64)
        self.batch = None

    def _grid(self):
        g = self.grid.copy()
        g.data = self.payload[: self.num_vertices * 28].numpy().reshape(-1, 28).copy()
        return g

    def forward(self, batch):
        self.batch = batch.numpy()
        try:
            _, _, _, st = self.o.mapping_step(self._grid(), self.frames, self.intr, self.cfg,
                                              self.batch, apply=False)
        except RuntimeError:  # no local hit
            return 0, 0, -1, 0.0, 0.0, 0
        return (st.rays_color, st.rays_depth, st.bad_ray,
                st.loss_photometric * st.rays_color,
                st.loss_geometric * max(st.rays_depth, 1) if st.rays_depth else 0.0, st.samples)

    def backward(self, m_color, m_depth):
        grad, _ = self.o.mapping_grad_global(self._grid(), self.frames, self.intr, self.cfg,
                                             self.batch, m_color, m_depth)
        self.grad[: self.num_vertices * 28] += torch.from_numpy(grad.reshape(-1))

    def apply(self, v0, v1):
        """mapping.cpp:218-231 on the owned vertex shard."""
        s = slice(v0 * 28, min(v1, self.num_vertices) * 28)
        g, v, th = self.grad[s], self.v[s], self.payload[s]
        nz = g != 0
        slot = (torch.arange(s.start, s.stop) % 28)
        lr = torch.where(slot == 0, torch.tensor(self.cfg.lr_sigma, dtype=torch.float64),
                         torch.tensor(self.cfg.lr_sh, dtype=torch.float64))
        rho = self.cfg.rmsprop_decay
        vn = rho * v + (1.0 - rho) * g * g
        v[nz] = vn[nz]
        th[nz] = th[nz] - lr[nz] * g[nz] / torch.sqrt(v[nz] + self.cfg.rmsprop_eps)
        self.grad[v0 * 28: v1 * 28] = 0.0

    # ---- block-sparse exchange: 8^3-vertex blocks, packed [n][512][28]
    BLOCK_FLOATS = 512 * 28

    def _block_vertices(self):
        if not hasattr(self, "_bv"):
            rx, ry, rz = self.grid.geom.res
            tb = [(r + 7) // 8 for r in (rx, ry, rz)]
            nb = tb[0] * tb[1] * tb[2]
            vl = np.arange(512)
            lx, ly, lz = vl % 8, (vl // 8) % 8, vl // 64
            b = np.arange(nb)
            bx, by, bz = b % tb[0], (b // tb[0]) % tb[1], b // (tb[0] * tb[1])
            x = bx[:, None] * 8 + lx[None]
            y = by[:, None] * 8 + ly[None]
            z = bz[:, None] * 8 + lz[None]
            inside = (x < rx) & (y < ry) & (z < rz)
            self._bv = np.where(inside, x + rx * (y + ry * z), -1)
        return self._bv

    @property
    def n_blocks(self):
        return self._block_vertices().shape[0]

    def touched_flags(self):
        bv = self._block_vertices()
        g = self.grad[: self.num_vertices * 28].view(-1, 28).abs().sum(1).numpy() != 0
        gv = np.concatenate([g, [False]])  # index -1 -> False
        return torch.from_numpy(gv[bv].any(1).astype(np.uint8))

    def pack(self, ids, which):
        src = (self.grad if which == 0 else self.payload)[: self.num_vertices * 28].view(-1, 28)
        bv = self._block_vertices()
        out = torch.zeros(ids.numel(), 512, 28, dtype=src.dtype)
        for e, b in enumerate(ids.tolist()):
            if b < 0:
                continue
            v = torch.from_numpy(bv[b])
            ok = v >= 0
            out[e, ok] = src[v[ok]]
        return out.flatten()

    def apply_blocks(self, ids, packed):
        bv = self._block_vertices()
        pk = packed.view(-1, 512, 28)
        th = self.payload[: self.num_vertices * 28].view(-1, 28)
        vv = self.v[: self.num_vertices * 28].view(-1, 28)
        lr = torch.full((28,), self.cfg.lr_sh, dtype=torch.float64)
        lr[0] = self.cfg.lr_sigma
        rho = self.cfg.rmsprop_decay
        for e, b in enumerate(ids.tolist()):
            if b < 0:
                continue
            v = torch.from_numpy(bv[b])
            ok = v >= 0
            g = pk[e, ok]
            rows = v[ok]
            nz = g != 0
            vn = rho * vv[rows] + (1.0 - rho) * g * g
            vnew = torch.where(nz, vn, vv[rows])
            tnew = torch.where(nz, th[rows] - lr * g / torch.sqrt(vnew + self.cfg.rmsprop_eps),
                               th[rows])
            vv[rows] = vnew
            th[rows] = tnew

    def unpack_payload(self, ids, packed):
        bv = self._block_vertices()
        pk = packed.view(-1, 512, 28)
        th = self.payload[: self.num_vertices * 28].view(-1, 28)
        for e, b in enumerate(ids.tolist()):
            if b < 0:
                continue
            v = torch.from_numpy(bv[b])
            ok = v >= 0
            th[v[ok]] = pk[e, ok]

    def clear_grad(self):
        self.grad.zero_()


def _worker(rank, world, port, out_dir, sparse=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    sys.path.insert(0, str(ROOT / "tests"))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2307_03404_b200.api import MappingConfig
    from paper_2307_03404_b200.distributed import DistributedMapper
    from scenes import fresh_grid, room_scene

    grid, intr, frames = room_scene()
    g0 = fresh_grid(grid)
    cfg = MappingConfig()
    import oracle as orc
    full = orc.Oracle().draw_batch(31, len(frames), intr.width, intr.height, 400)
    mine = torch.from_numpy(np.array_split(full, world)[rank].copy())
    eng = OracleEngine(g0, frames, intr, cfg, world)
    res = DistributedMapper(eng).step(mine, cfg.lambda_d, sparse=sparse)
    if rank == 0:
        np.save(Path(out_dir) / "dist_payload.npy", eng.payload[: eng.num_vertices * 28].numpy())
        np.save(Path(out_dir) / "dist_stats.npy",
                np.array([res.loss_total, res.rays_color, res.rays_depth, res.samples]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("sparse", [False, True])
def test_ray_sharded_step_equals_single_process(tmp_path, oracle, sparse):
    """Dense exchange, and the block-sparse one (touched 8^3-vertex blocks with
    static owners): both equal the single-process step."""
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), sparse), nprocs=2, join=True)
    from paper_2307_03404_b200.api import MappingConfig
    from scenes import fresh_grid, room_scene

    grid, intr, frames = room_scene()
    g0 = fresh_grid(grid)
    full = oracle.draw_batch(31, len(frames), intr.width, intr.height, 400)
    data, _, _, st = oracle.mapping_step(g0, frames, intr, MappingConfig(), full)
    got = np.load(tmp_path / "dist_payload.npy").reshape(-1, 28)
    np.testing.assert_allclose(got, data, rtol=1e-9, atol=1e-9 * np.abs(data).max())
    stats = np.load(tmp_path / "dist_stats.npy")
    assert stats[1] == st.rays_color and stats[2] == st.rays_depth and stats[3] == st.samples
    assert abs(stats[0] - st.loss_total) <= 1e-12 * st.loss_total


def test_shard_ranges_cover_padded_vertices():
    from paper_2307_03404_b200.distributed import shard_range
    for world in (1, 2, 4, 8):
        padded = 4913 + (-4913) % world
        spans = [shard_range(padded, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == padded
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


class _LinearPoseCtx:
    """Stands in for a device context in the tracker: normal equations of a
    linear translation model r_p = J_p (t - t_true), J_p fixed per pixel."""
    device = 0

    def __init__(self, t_true):
        self.t_true = np.asarray(t_true)

    def pose_normal_equations(self, slot, intr, pose, pixels, cfg):
        from paper_2307_03404_b200.api import NormalEquations
        jtj = np.zeros((6, 6))
        jtr = np.zeros(6)
        loss = 0.0
        for px, py in pixels:
            g = np.random.default_rng(int(px) * 7919 + int(py))
            J = np.zeros((4, 6))
            J[:, 3:] = g.normal(size=(4, 3))
            r = J[:, 3:] @ (np.asarray(pose.t) - self.t_true)
            jtj += J.T @ J
            jtr += J.T @ r
            loss += float(r @ r)
        return NormalEquations(jtj, jtr, loss, len(pixels), 0)


def _tracker_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, str(ROOT))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2307_03404_b200.api import GNConfig, Pose
        from paper_2307_03404_b200.distributed import DistributedTracker
        t_true = (0.3, -0.2, 1.1)
        tr = DistributedTracker(_LinearPoseCtx(t_true), None,
                                GNConfig(rays_per_iteration=64, iterations=3, damping=0.0))
        depth = np.ones((12, 16))
        res = tr.track(0, depth, Pose((1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0)))
        out[rank] = (tuple(res.pose.t), tuple(res.pose.q), res.rays_used)
    finally:
        dist.destroy_process_group()


def test_distributed_tracker_gloo_world2():
    """Ray-sharded GN tracking: the all-reduced normal equations of 2 ranks x 32
    pixels solve the linear model exactly, and both ranks take the same step."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_tracker_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    (t0, q0, u0), (t1, q1, u1) = out[0], out[1]
    assert t0 == t1 and q0 == q1
    assert u0 == [64, 64, 64]
    np.testing.assert_allclose(t0, (0.3, -0.2, 1.1), atol=1e-9)
    np.testing.assert_allclose(q0, (1.0, 0.0, 0.0, 0.0), atol=1e-12)


def test_lm_step_matches_closed_form():
    """lm_step: pure translation system -> t + x exactly; small rotation -> exp map."""
    from paper_2307_03404_b200.api import Pose
    from paper_2307_03404_b200.distributed import lm_step
    A = np.diag([2.0, 2.0, 2.0, 4.0, 4.0, 4.0])
    b = -A @ np.array([0.0, 0.0, 0.1, 0.01, -0.02, 0.03])  # J^T r = -A x
    p = lm_step(A, b, 0.0, Pose((1.0, 0.0, 0.0, 0.0), (1.0, 2.0, 3.0)))
    np.testing.assert_allclose(p.t, (1.01, 1.98, 3.03), atol=1e-12)
    np.testing.assert_allclose(p.q, (np.cos(0.05), 0.0, 0.0, np.sin(0.05)), atol=1e-12)
