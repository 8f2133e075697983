"""Row-slab peer-put exchange across PROCESSES (the multi-GPU code path): two
ranks in two processes on one B200 map each other's receive buffers and flag
arrays with CUDA IPC (hs_ipc_*), store their transposes straight into them and
synchronise on the device flags inside one captured CUDA graph per step; gloo
carries only the handle exchange and the gradient sum.  Checked against an unsharded trainer on the same scene."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

W, H, C, N, L, STEPS = 64, 48, 3, 400, 1, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene(holo, S):
    g = {k: np.asarray(v, dtype=np.float32).astype(np.float64) for k, v in S.init_gaussians(N, C, W, H, 42).items()}
    gs = holo.GaussianSet(N, C, **g)
    target = holo.RealField(C, H, W, S.synthetic_image(42, C, H, W).astype(np.float32).astype(np.float64))
    masks = S.build_masks(S.synthetic_depth(43, H, W), L, True)
    return gs, target, masks, S.make_depth_planes(L, 3e-3, 2e-3), holo.PropagationSpec(S.WAVELENGTHS[C])


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    from paper_2511_15022_b200 import holo, parallel as P, synthetic as S
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    side = torch.cuda.Stream()  # a capturable stream: the step runs as one CUDA graph
    torch.cuda.set_stream(side)
    try:
        gs, target, masks, dists, spec = _scene(holo, S)
        tr = holo.Trainer(gs, W, H, target, masks, dists, spec, 10)
        tr.set_deterministic(True)  # compared with the deterministic full trainer
        tr.set_row_slab(rank, world)
        step = P.SlabShardedStep(tr, C, H, W, L, exchange="put")  # IPC mapping of the peers, graphs on
        losses = []
        for _ in range(STEPS):
            tr.slab_forward_backward()  # stages 0..4 as one captured graph, device-flag sync
            g = tr.grads_tensor()
            gh = g.cpu()
            dist.all_reduce(gh)
            g.copy_(gh.to(g.device))
            tr.apply_update()
            parts = torch.tensor(tr.loss_partials(), dtype=torch.float64)
            dist.all_reduce(parts)
            losses.append(P.combine_loss(float(parts[0]), float(parts[1]), C, H, W, L))
        status = tr.slab_status()
        q.put((rank, losses, tr.params(), status))
        dist.barrier()
        del step
    finally:
        dist.destroy_process_group()


def test_slab_peer_put_across_processes(holo):
    import torch.multiprocessing as mp
    from paper_2511_15022_b200 import synthetic as S
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gs, target, masks, dists, spec = _scene(holo, S)
    full = holo.Trainer(gs, W, H, target, masks, dists, spec, 10)
    full.set_deterministic(True)  # the slab ranks' backward is the gather: compare like with like
    lf = [full.step() for _ in range(STEPS)]
    pf = full.params().astype(np.float64)
    for rank, losses, params, status in res:
        assert status == 0
        np.testing.assert_allclose(losses, lf, rtol=2e-6)
        p = params.astype(np.float64)
        assert np.linalg.norm(p - pf) / np.linalg.norm(pf) < 1e-6
