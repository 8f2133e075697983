"""Multi-GPU partitioning of the hot path.

* Plane sharding (cfg3): the forward spectrum is shared per channel, every
  plane's inverse, loss and adjoint are independent, and the backward is a sum
  over planes (propagation.cpp:231-237) that the rasterizer backward is linear
  in.  Rank r owns a contiguous block of planes; the raster forward and the
  forward row/column FFT are replicated; each rank produces the parameter
  gradient of its planes with the global normalisers (L_total, SSIM count),
  one NCCL all-reduce (sum) of the (6+2C)N gradient buffer makes them the full
  gradient, and every rank applies the identical Adan update.
* Wavelength sharding (cfg2, up to C ranks): the channels of a scene are
  independent through propagation and loss; amplitude/phase of channel c only
  see channel c, the geometry (position, scale, rotation, opacity) gets a sum
  over channels.  Rank r owns a contiguous block of channels: its trainer is
  built on that slice (wavelengths, target, amplitude/phase columns) with the
  global channel count for the loss normalisers, one NCCL all-reduce of the
  geometry gradients (6N floats) completes them, and every rank applies the
  identical geometry update plus the update of its own amplitude/phase.
* Row-slab sharding (cfg4, 4K): rank r owns H/R canvas rows and 1/R of the
  padded spectrum's column tiles.  The 2D FFTs become row FFTs on the own rows,
  an all-to-all transpose (NCCL over NVLink), column FFTs on the own tiles and
  an all-to-all back -- four transposes per step (forward and adjoint
  propagation).  The loss runs on the own rows plus 10-row SSIM halos that the
  second transpose delivers with the rows (computed redundantly, counted once),
  the rasterizer backward sums each Gaussian over the own rows only, and one
  all-reduce of the gradient buffer completes the gradient (the backward is
  linear in the gradient field).  Binning is replicated.
* Scene replicas (cfg2 at N>1, cfg5): independent problems, no collective.

The collective is torch.distributed over NCCL (gloo on CPU for the tests).
"""
from __future__ import annotations

import math
from typing import Tuple

import torch
import torch.distributed as dist


def plane_shard(L: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced block [begin, end) of the L planes for `rank`."""
    if L < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError("plane_shard: bad arguments")
    base, extra = divmod(L, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def channel_shard(C: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [begin, end) of the C channels (wavelengths) for `rank`."""
    return plane_shard(C, rank, world)


def slice_channels(groups: dict, n: int, C: int, begin: int, end: int) -> dict:
    """The six parameter groups of a scene restricted to channels [begin, end):
    amplitude and phase are N x C row-major (gaussian_set.hpp:14-19)."""
    out = dict(groups)
    for k in ("amplitude", "phase"):
        out[k] = groups[k].reshape(n, C)[:, begin:end].reshape(-1).copy()
    return out


def geometry_ranges(n: int, c: int):
    """[begin, end) ranges of the channel-independent groups in the flat layout
    [pre_position 2N | pre_scale 2N | rotation N | amplitude NC | phase NC | pre_opacity N]."""
    return [(0, 5 * n), (5 * n + 2 * n * c, 6 * n + 2 * n * c)]


def combine_loss(recon_sum: float, ssim_sum: float, C: int, H: int, W: int, L: int,
                 ssim_weight: float = 0.005) -> float:
    """training_loss from the all-reduced partial sums (loss_recon_grad loss.cpp:248-272, loss_ssim_grad :292-314, training_loss_grad :320-329)."""
    n = C * H * W
    count = L * C * (H - 10) * (W - 10)
    return recon_sum / (n * L) + ssim_weight * (1.0 - ssim_sum / count)


GROUP_NAMES = ("position", "scale", "rotation", "amplitude", "phase", "opacity")  # pipeline.cpp:244-249
_NO_GROUP = 1 << 30


def agree_nonfinite(trainer, group=None):
    """After the cross-rank gradient sum and check_grads(): keep only the lowest
    non-finite group bit of the trainer's device flag word and min-reduce it over
    the ranks, so every rank skips the same groups in apply_update -- the groups
    from the first non-finite one on, as the reference's Adan::step throw stops
    the step loop there (optimizer.cpp:52-54).  Needed when part of the gradient
    stays rank-local (channel shards) or a rank's partial alone is non-finite."""
    ft = getattr(trainer, "flags_tensor", None)
    if ft is None or not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return
    f = ft()
    low = _lowest_group_bit(f)
    dist.all_reduce(low, op=dist.ReduceOp.MIN, group=group)
    f.copy_(torch.where(low == _NO_GROUP, torch.zeros_like(low), low))


def _lowest_group_bit(f: torch.Tensor) -> torch.Tensor:
    low = f & -f
    return torch.where(low == 0, torch.full_like(low, _NO_GROUP), low)


def agree_nonfinite_local(trainers):
    """agree_nonfinite for trainers that share one process (virtual ranks)."""
    fs = [t.flags_tensor() for t in trainers]
    low = torch.stack([_lowest_group_bit(f) for f in fs]).min(dim=0).values
    word = torch.where(low == _NO_GROUP, torch.zeros_like(low), low)
    for f in fs:
        f.copy_(word)


class ErrorWatch:
    """Raises a sharded step's device errors -- the non-finite group word
    (HoloNonFinite naming the reference's group, as Adan::step's throw) and the
    peer-put timeout word -- on every step without a per-step host sync: after
    each update both words are copied into pinned host memory behind an event;
    step k raises for the last step whose copy has completed, and flush() (also
    called when the loss is read, which syncs anyway) for the current one."""

    def __init__(self, trainer, depth: int = 4):
        self.tr = trainer
        self.ok = hasattr(trainer, "flags_tensor") and torch.cuda.is_available()
        self.depth = depth
        self.k = 0
        if self.ok:
            self.host = torch.zeros((depth, 2), dtype=torch.int32).pin_memory()
            self.events = [None] * depth
            err = trainer.slab_error_tensor() if hasattr(trainer, "slab_error_tensor") else None
            self.words = [trainer.flags_tensor(), err]

    def post(self):
        if not self.ok:
            return
        slot = self.k % self.depth
        if self.events[slot] is not None:  # ring full: its copy is `depth` steps old
            self._check(slot)
        for j, w in enumerate(self.words):
            if w is not None:
                self.host[slot, j:j + 1].copy_(w, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.events[slot] = ev
        self.k += 1
        self.poll()

    def _check(self, slot):
        self.events[slot].synchronize()
        self.events[slot] = None
        flags, err = int(self.host[slot, 0]), int(self.host[slot, 1])
        if err:
            raise RuntimeError("row slab: a peer-put exchange timed out waiting for a peer")
        if flags:
            from ._lib import HoloNonFinite
            g = (flags & -flags).bit_length() - 1
            raise HoloNonFinite(f"Adan: non-finite gradient in group {GROUP_NAMES[g]}")

    def poll(self):
        if not self.ok:
            return
        for i in range(self.k - self.depth, self.k):
            slot = i % self.depth
            if i >= 0 and self.events[slot] is not None and self.events[slot].query():
                self._check(slot)

    def flush(self):
        if not self.ok:
            return
        for i in range(self.k - self.depth, self.k):
            slot = i % self.depth
            if i >= 0 and self.events[slot] is not None:
                self._check(slot)


class ShardedStep:
    """One optimisation step of a plane-sharded trainer.

    `trainer` needs forward_backward(), grads_tensor(), apply_update(),
    loss_partials() -- holo.Trainer built with plane_range=plane_shard(...).
    """

    def __init__(self, trainer, C, H, W, L_total, group=None):
        self.tr = trainer
        self.C, self.H, self.W, self.L = C, H, W, L_total
        self.group = group
        self.watch = ErrorWatch(trainer)

    def step(self, with_loss: bool = True):
        """One step; returns the loss (a host sync) or None when with_loss is False.
        Raises HoloNonFinite for a non-finite summed gradient (at the latest one
        step later when the loss is not read)."""
        self.tr.forward_backward()
        g = self.tr.grads_tensor()
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            if g.is_cuda:
                torch.cuda.current_stream().synchronize()
            dist.all_reduce(g, op=dist.ReduceOp.SUM, group=self.group)
            self.tr.check_grads()
            agree_nonfinite(self.tr, self.group)
        self.tr.apply_update()
        self.watch.post()
        if not with_loss:
            return None
        self.watch.flush()
        parts = torch.tensor(self.tr.loss_partials(), dtype=torch.float64,
                             device=g.device if g.is_cuda else "cpu")
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(parts, op=dist.ReduceOp.SUM, group=self.group)
        return combine_loss(float(parts[0]), float(parts[1]), self.C, self.H, self.W, self.L)


class ChannelShardedStep:
    """One optimisation step of a wavelength-sharded trainer: `trainer` holds
    c_local of C_total channels (holo.Trainer(..., channels_total=C_total) on
    slice_channels(...)); the geometry gradients are all-reduced, amplitude and
    phase stay local."""

    def __init__(self, trainer, n, c_local, C_total, H, W, L, group=None):
        self.tr, self.n, self.c = trainer, n, c_local
        self.C, self.H, self.W, self.L = C_total, H, W, L
        self.group = group
        self.watch = ErrorWatch(trainer)

    def step(self, with_loss: bool = True):
        """One step; returns the loss (a host sync) or None when with_loss is False."""
        self.tr.forward_backward()
        g = self.tr.grads_tensor()
        multi = dist.is_initialized() and dist.get_world_size(self.group) > 1
        if multi:
            if g.is_cuda:
                torch.cuda.current_stream().synchronize()
            for b, e in geometry_ranges(self.n, self.c):
                dist.all_reduce(g[b:e], op=dist.ReduceOp.SUM, group=self.group)
            # the summed geometry may be non-finite where this rank's partial was
            # not, and the rank-local amplitude/phase groups differ per rank
            self.tr.check_grads()
            agree_nonfinite(self.tr, self.group)
        self.tr.apply_update()
        self.watch.post()
        if not with_loss:
            return None
        self.watch.flush()
        parts = torch.tensor(self.tr.loss_partials(), dtype=torch.float64,
                             device=g.device if g.is_cuda else "cpu")
        if multi:
            dist.all_reduce(parts, op=dist.ReduceOp.SUM, group=self.group)
        return combine_loss(float(parts[0]), float(parts[1]), self.C, self.H, self.W, self.L)


def update_shard(P: int, rank: int, world: int) -> Tuple[int, int]:
    """Elements [begin, end) of the flat P-float parameter buffer whose Adan
    update `rank` owns in a sharded update: equal parts rounded to multiples of
    4 floats (the vectorised update), the last rank takes the rest."""
    per = ((P + world - 1) // world + 3) // 4 * 4
    b = min(rank * per, P)
    return b, min(b + per, P) if rank < world - 1 else P


def sharded_update(tr, group=None):
    """Reduce-scatter the gradient buffer, update this rank's shard of the
    parameters (ZeRO-1 style: the Adan moments of the other shards stay
    untouched and are never read), agree on the first non-finite group over
    the ranks, all-gather the parameters.  Same result as all-reduce +
    check_grads + replicated apply_update, with 1/world of the update work."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    g = tr.grads_tensor()
    P = g.numel()
    parts = [update_shard(P, r, world) for r in range(world)]
    b, e = parts[rank]
    # equal shards: reduce-scatter + all-gather (NCCL, or gloo on host tensors);
    # otherwise all-reduce + per-shard broadcasts (the update stays sharded)
    even = all(pe - pb == e - b for pb, pe in parts) and P % world == 0 and \
        (dist.get_backend(group) == "nccl" or not g.is_cuda)
    if even:
        out = torch.empty(e - b, dtype=g.dtype, device=g.device)
        dist.reduce_scatter_tensor(out, g, group=group)
        g[b:e].copy_(out)
    else:  # uneven shards: all-reduce (the update below is still sharded)
        dist.all_reduce(g, op=dist.ReduceOp.SUM, group=group)
    tr.check_grads_range(b, e)
    agree_nonfinite(tr, group)
    tr.apply_update_range(b, e)
    p = tr.params_tensor()
    if even:
        dist.all_gather_into_tensor(p, p[b:e].clone(), group=group)
    else:
        for r, (pb, pe) in enumerate(parts):
            dist.broadcast(p[pb:pe], src=dist.get_global_rank(group, r) if group is not None else r, group=group)


def row_slab(H: int, rank: int, world: int) -> Tuple[int, int]:
    """Rows [begin, end) of the canvas owned by `rank` (equal slabs)."""
    if world < 1 or not 0 <= rank < world or H % world:
        raise ValueError("row_slab: the canvas height must divide into equal slabs")
    hr = H // world
    return rank * hr, (rank + 1) * hr


def loss_band(H: int, rank: int, world: int, halo: int = 10) -> Tuple[int, int]:
    """Rows [begin, end) of the loss band of `rank`: its slab plus up to `halo`
    rows each side (the 11x11 SSIM windows that touch the own rows)."""
    b, e = row_slab(H, rank, world)
    return max(0, b - halo), min(H, e + halo)


class SlabShardedStep:
    """One optimisation step of a row-slab sharded trainer (cfg4): five
    stages with a transpose exchange between them (hs_trainer_slab_stage), then
    the gradient all-reduce and the replicated Adan update.

    `trainer` is a holo.Trainer on which set_row_slab(rank, world) was called.
    exchange="nccl": all_to_all_single on the peer-major send/receive buffers.
    exchange="put": the pack kernels store straight into the peers' receive
    buffers (CUDA IPC mappings of every peer's buffers, NVLink stores from the
    SMs) and signal device flags; the next stage's first kernel waits on them.
    No collective library call on the transpose data path.
    """

    def __init__(self, trainer, C, H, W, L, group=None, exchange="nccl", shard_update=True):
        self.tr = trainer
        self.C, self.H, self.W, self.L = C, H, W, L
        self.group = group
        self.shard_update = shard_update  # reduce-scatter / sharded Adan / all-gather
        self.counts = [trainer.slab_counts(e) for e in range(4)]
        self.put = exchange == "put"
        self._mapped = []
        if self.put:
            self._map_peers()
            trainer.use_graph(True)
        self.watch = ErrorWatch(trainer)

    def _map_peers(self):
        from . import holo
        rank, world = self.tr.slab
        mine = self.tr.slab_peer_buffers()
        if world == 1:
            self.tr.slab_set_peers([mine[0]], [mine[1]], [mine[2]])
            return
        handles = [None] * world
        dist.all_gather_object(handles, [holo.ipc_handle(p) for p in mine], group=self.group)
        cols = [[], [], []]
        for r, hs in enumerate(handles):
            for k in range(3):
                if r == rank:
                    cols[k].append(mine[k])
                else:
                    p = holo.ipc_open(hs[k])
                    self._mapped.append(p)
                    cols[k].append(p)
        self.tr.slab_set_peers(*cols)
        dist.barrier(group=self.group)

    def _exchange(self, e):
        if self.put:
            return  # the pack kernel already stored into the peers and signalled
        send, recv = self.tr.slab_buffers()
        sc, rc = self.counts[e]
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_to_all_single(recv[:sum(rc)], send[:sum(sc)], rc, sc, group=self.group)
        else:
            recv[:sum(rc)].copy_(send[:sum(sc)])

    def step(self, with_loss: bool = True):
        """One step; returns the loss (a host sync) or None when with_loss is False."""
        if self.put:  # the stages synchronise on device flags: one call, one CUDA graph
            self.tr.slab_forward_backward()
        else:
            for e in range(4):
                self.tr.slab_stage(e)
                self._exchange(e)
            self.tr.slab_stage(4)
        g = self.tr.grads_tensor()
        multi = dist.is_initialized() and dist.get_world_size(self.group) > 1
        if multi and self.shard_update:
            sharded_update(self.tr, self.group)
        else:
            if multi:
                dist.all_reduce(g, op=dist.ReduceOp.SUM, group=self.group)
                self.tr.check_grads()
                agree_nonfinite(self.tr, self.group)
            self.tr.apply_update()
        self.watch.post()  # non-finite groups and the peer-put timeout word, every step
        if not with_loss:
            return None
        self.watch.flush()
        parts = torch.tensor(self.tr.loss_partials(), dtype=torch.float64, device=g.device)
        if multi:
            dist.all_reduce(parts, op=dist.ReduceOp.SUM, group=self.group)
        return combine_loss(float(parts[0]), float(parts[1]), self.C, self.H, self.W, self.L)


class NativeShardedStep:
    """The sharded step run entirely inside the native library
    (hs_trainer_sharded_step) over an NCCL communicator held by the device
    context: the same decompositions as ShardedStep / ChannelShardedStep /
    SlabShardedStep (chosen by how `trainer` was built), with no torch
    collective on the step path.  torch.distributed only ships the 128-byte
    NCCL id once at construction; a C/C++ host does the same with
    hs_comm_unique_id / hs_ctx_comm_init."""

    def __init__(self, trainer, group=None):
        from . import holo
        self.tr = trainer
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        box = [holo.comm_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(box, src=0, group=group)
        holo.ctx_comm_init(box[0], world, rank)

    def step(self, with_loss: bool = True):
        return self.tr.sharded_step(with_loss)

    def close(self):
        from . import holo
        holo.ctx_comm_destroy()


class LocalSlabGroup:
    """R row-slab trainers on ONE device, stepped in lock-step with the
    all-to-all and the all-reduce done as device copies: the single-GPU
    check that the R-rank decomposition reproduces the unsharded step
    (tests and bench; a real run uses SlabShardedStep, one rank per GPU).
    put=True runs the peer-put exchange instead (the pack kernels store into
    the other trainers' receive buffers and signal their device flags), the
    same kernels a multi-GPU run uses over NVLink."""

    def __init__(self, trainers, C, H, W, L, put=False, shard_update=True):
        self.trs = list(trainers)
        self.C, self.H, self.W, self.L = C, H, W, L
        self.shard_update = shard_update
        self.counts = [[t.slab_counts(e) for e in range(4)] for t in self.trs]
        self.put = put
        self.watches = [ErrorWatch(t) for t in self.trs]
        if put:
            bufs = [t.slab_peer_buffers() for t in self.trs]
            for t in self.trs:
                t.slab_set_peers([b[0] for b in bufs], [b[1] for b in bufs], [b[2] for b in bufs])

    def _exchange(self, e):
        if self.put:
            return
        R = len(self.trs)
        for r, tr in enumerate(self.trs):
            recv = tr.slab_buffers()[1]
            off = 0
            for s, ts in enumerate(self.trs):
                sc = self.counts[s][e][0]
                so = sum(sc[:r])
                recv[off:off + sc[r]].copy_(ts.slab_buffers()[0][so:so + sc[r]])
                off += sc[r]
            assert off == sum(self.counts[r][e][1]) and len(sc) == R

    def step(self, with_loss: bool = True):
        for e in range(4):
            for t in self.trs:
                t.slab_stage(e)
            self._exchange(e)
        for t in self.trs:
            t.slab_stage(4)
        grads = [t.grads_tensor() for t in self.trs]
        total = grads[0].clone()
        for g in grads[1:]:
            total += g
        if self.shard_update:  # the sharded Adan / all-gather of sharded_update
            R, P = len(self.trs), total.numel()
            parts = [update_shard(P, r, R) for r in range(R)]
            for t, g, (b, e) in zip(self.trs, grads, parts):
                g.copy_(total)  # (every rank keeps the whole sum here, for inspection)
                t.check_grads_range(b, e)
            agree_nonfinite_local(self.trs)
            for t, (b, e) in zip(self.trs, parts):
                t.apply_update_range(b, e)
            # all-gather: assemble the shards once, hand the result to every rank
            full = total  # (the summed gradient is no longer needed)
            for t, (b, e) in zip(self.trs, parts):
                full[b:e].copy_(t.params_tensor()[b:e])
            for t in self.trs:
                t.params_tensor().copy_(full)
        else:
            for g in grads:
                g.copy_(total)
            for t in self.trs:
                t.check_grads()
                t.apply_update()
        for w in self.watches:
            w.post()
        if not with_loss:
            return None
        for w in self.watches:
            w.flush()
        parts = [t.loss_partials() for t in self.trs]
        return combine_loss(sum(p[0] for p in parts), sum(p[1] for p in parts), self.C, self.H, self.W, self.L)


def amdahl_plane_speedup(L: int, world: int) -> float:
    """Ideal speed-up of plane sharding in the byte model B = C(13+12L)A:
    13A per channel is replicated, 12A per plane is split."""
    per_rank_planes = math.ceil(L / world)
    return (13 + 12 * L) / (13 + 12 * per_rank_planes)
