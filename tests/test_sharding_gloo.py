"""CPU, world_size 2 over gloo: plane sharding of the optimisation step.

1. The math: per-shard gradients (oracle restatement, global normalisers)
   summed with a gloo all-reduce equal the unsharded step's gradients, and the
   combined loss equals the full loss.
2. The orchestration (paper_2511_15022_b200.parallel.ShardedStep) all-reduces
   the gradient buffer between forward_backward and apply_update.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import holo_oracle as O
from paper_2511_15022_b200 import parallel as P
from paper_2511_15022_b200 import synthetic as S

N, C, W, H, L = 40, 3, 32, 24, 4


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def scene():
    g = S.init_gaussians(N, C, W, H, 42)
    g = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in g.items()}
    target = S.synthetic_image(42, C, H, W)
    masks = S.build_masks(S.synthetic_depth(43, H, W), L, True)
    dist_ = S.make_depth_planes(L, 3e-3, 4e-3 / 7)
    return g, target, masks, dist_


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, target, masks, d = scene()
    b, e = P.plane_shard(L, rank, world)
    r = O.step_grads(g, N, C, W, H, target, masks, d, S.WAVELENGTHS[C], planes=range(b, e), L_norm=L)
    flat = torch.from_numpy(np.concatenate([r["grads"][k] for k in O.GROUPS]))
    dist.all_reduce(flat)
    parts = torch.tensor([r["recon_sum"], r["ssim_sum"]], dtype=torch.float64)
    dist.all_reduce(parts)
    if rank == 0:
        np.save(out + "_grads.npy", flat.numpy())
        np.save(out + "_parts.npy", parts.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_plane_shard_partitions():
    for L_ in range(1, 17):
        for world in range(1, 9):
            seen = []
            for r in range(world):
                b, e = P.plane_shard(L_, r, world)
                assert 0 <= b <= e <= L_
                seen += list(range(b, e))
            assert seen == list(range(L_))
    assert P.amdahl_plane_speedup(8, 8) == pytest.approx(109 / 25)


def test_sharded_step_equals_full_step_gloo(tmp_path):
    out = str(tmp_path / "r")
    mp.spawn(_worker, args=(2, free_port(), out), nprocs=2, join=True)
    grads = np.load(out + "_grads.npy")
    parts = np.load(out + "_parts.npy")
    g, target, masks, d = scene()
    full = O.step_grads(g, N, C, W, H, target, masks, d, S.WAVELENGTHS[C])
    ref = np.concatenate([full["grads"][k] for k in O.GROUPS])
    assert np.linalg.norm(grads - ref) / np.linalg.norm(ref) < 1e-12
    loss = P.combine_loss(parts[0], parts[1], C, H, W, L)
    full_loss = P.combine_loss(full["recon_sum"], full["ssim_sum"], C, H, W, L)
    assert loss == pytest.approx(full_loss, rel=1e-12)


class FakeTrainer:
    """Stands in for holo.Trainer on CPU: gradient = (rank+1) * ones."""

    def __init__(self, rank, n):
        self.rank, self.g, self.applied = rank, torch.zeros(n), None

    def forward_backward(self):
        self.g.fill_(self.rank + 1.0)

    def grads_tensor(self):
        return self.g

    def check_grads(self):  # the summed-gradient non-finite check (device side in the real trainer)
        pass

    def apply_update(self):
        self.applied = self.g.clone()

    def loss_partials(self):
        return (10.0 * (self.rank + 1), 1.0)


def _orchestration_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tr = FakeTrainer(rank, 16)
    loss = P.ShardedStep(tr, 1, 16, 16, 2).step()
    np.save(f"{out}_{rank}.npy", np.concatenate([tr.applied.numpy(), [loss]]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_step_orchestration_gloo(tmp_path):
    out = str(tmp_path / "o")
    mp.spawn(_orchestration_worker, args=(2, free_port(), out), nprocs=2, join=True)
    a, b = np.load(out + "_0.npy"), np.load(out + "_1.npy")
    assert np.array_equal(a, b)                 # identical update on every rank
    assert np.all(a[:16] == 3.0)                # 1 + 2: the summed gradient reached Adan
    assert a[16] == pytest.approx(P.combine_loss(30.0, 2.0, 1, 16, 16, 2))


# ---- wavelength (channel) sharding ---------------------------------------------------------

def _channel_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, target, masks, d = scene()
    b, e = P.channel_shard(C, rank, world)
    gs = P.slice_channels(g, N, C, b, e)
    r = O.step_grads(gs, N, e - b, W, H, target[b:e], masks, d, S.WAVELENGTHS[C][b:e], C_norm=C)
    flat = torch.from_numpy(np.concatenate([r["grads"][k] for k in O.GROUPS]))
    for lo, hi in P.geometry_ranges(N, e - b):  # the collective of ChannelShardedStep
        dist.all_reduce(flat[lo:hi])
    parts = torch.tensor([r["recon_sum"], r["ssim_sum"]], dtype=torch.float64)
    dist.all_reduce(parts)
    np.save(f"{out}_{rank}_grads.npy", flat.numpy())
    if rank == 0:
        np.save(out + "_parts.npy", parts.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_channel_shard_partitions_and_ranges():
    for world in (1, 2, 3):
        seen = []
        for r in range(world):
            b, e = P.channel_shard(3, r, world)
            seen += list(range(b, e))
        assert seen == [0, 1, 2]
    n, c = 5, 2
    geo = sum(e - b for b, e in P.geometry_ranges(n, c))
    assert geo == 6 * n  # position 2N + scale 2N + rotation N + opacity N


def test_channel_sharded_step_equals_full_step_gloo(tmp_path):
    """Two ranks owning channels [0,2) and [2,3): all-reduced geometry gradients
    equal the full step's, each rank's amplitude/phase gradients equal the full
    step's columns, and the combined loss equals the full loss."""
    out = str(tmp_path / "c")
    mp.spawn(_channel_worker, args=(2, free_port(), out), nprocs=2, join=True)
    g, target, masks, d = scene()
    full = O.step_grads(g, N, C, W, H, target, masks, d, S.WAVELENGTHS[C])
    fg = full["grads"]
    for rank in range(2):
        b, e = P.channel_shard(C, rank, 2)
        cl = e - b
        got = np.load(f"{out}_{rank}_grads.npy")
        o = 0
        parts = {}
        for k in O.GROUPS:
            size = {"amplitude": N * cl, "phase": N * cl}.get(k, fg[k].size)
            parts[k] = got[o:o + size]
            o += size
        for k in ("pre_position", "pre_scale", "rotation", "pre_opacity"):
            assert np.linalg.norm(parts[k] - fg[k]) <= 1e-12 * np.linalg.norm(fg[k]), k
        for k in ("amplitude", "phase"):
            ref = fg[k].reshape(N, C)[:, b:e].reshape(-1)
            assert np.linalg.norm(parts[k] - ref) <= 1e-12 * max(np.linalg.norm(ref), 1e-30), k
    p = np.load(out + "_parts.npy")
    loss = P.combine_loss(p[0], p[1], C, H, W, L)
    assert loss == pytest.approx(P.combine_loss(full["recon_sum"], full["ssim_sum"], C, H, W, L), rel=1e-12)


class _FlagTrainer:
    def __init__(self, word):
        self.f = torch.tensor([word], dtype=torch.int32)

    def flags_tensor(self):
        return self.f


def _agree_worker(rank, world, port, words, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = _FlagTrainer(words[rank])
    P.agree_nonfinite(t)
    q.put((rank, int(t.f.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("words,want", [((0, 0), 0), ((1 << 5, 1 << 3 | 1 << 4), 1 << 3), ((1 << 2, 0), 1 << 2)])
def test_ranks_agree_on_the_first_nonfinite_group_gloo(words, want):
    """parallel.agree_nonfinite: every rank ends with the lowest non-finite group
    of any rank (opacity on rank 0 and amplitude on rank 1 -> both stop at
    amplitude, where the reference's Adan::step would throw first)."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_agree_worker, args=(2, free_port(), words, q), nprocs=2, join=True, start_method="spawn")
    got = dict(q.get() for _ in range(2))
    assert got == {0: want, 1: want}
