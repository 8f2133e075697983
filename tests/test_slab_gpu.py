"""Row-slab sharding (distributed 2D FFT with all-to-all
transposes) on the B200: R slab trainers on one device, exchanged by device
copies in the all-to-all layout (parallel.LocalSlabGroup), against the
unsharded trainer on the same scene.  The decomposition changes only the fp32
summation order of the per-Gaussian sums (rows split over ranks) and of the
loss partials, so gradients, losses and updated parameters agree far inside
the parity bars (field 1e-4, gradients 1e-3); the 2D FFTs of every rank are
the unsharded FFTs' own row and column passes.  GRAD_TOL bounds the rel-L2
gap of the summed per-rank gradients to the unsharded ones (fp32 sums split
over up to 16 row slabs).
"""
GRAD_TOL = 1e-4
import numpy as np
import pytest

from paper_2511_15022_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def scene(holo, n, c, w, h, L, seed=42):
    g = {k: np.asarray(v, dtype=np.float32).astype(np.float64) for k, v in S.init_gaussians(n, c, w, h, seed).items()}
    gs = holo.GaussianSet(n, c, **g)
    target = holo.RealField(c, h, w, S.synthetic_image(seed, c, h, w).astype(np.float32).astype(np.float64))
    masks = S.build_masks(S.synthetic_depth(seed + 1, h, w), L, True)
    dist = S.make_depth_planes(L, 3e-3, 4e-3 / 7 if L > 2 else 2e-3)
    spec = holo.PropagationSpec(S.WAVELENGTHS[c])
    return gs, target, masks, dist, spec


def run(holo, R, n, c, w, h, L, steps, put=False):
    from paper_2511_15022_b200 import parallel as P
    gs, target, masks, dist, spec = scene(holo, n, c, w, h, L)
    full = holo.Trainer(gs, w, h, target, masks, dist, spec, 20)
    full.set_deterministic(True)  # the slab ranks' backward is the gather: compare like with like
    trs = []
    for r in range(R):
        t = holo.Trainer(gs, w, h, target, masks, dist, spec, 20)
        t.set_deterministic(True)
        t.set_row_slab(r, R)
        trs.append(t)
    grp = P.LocalSlabGroup(trs, c, h, w, L, put=put)
    out = []
    for s in range(steps):
        full.forward_backward()
        gfull = full.grads_tensor().cpu().numpy().astype(np.float64)
        full.apply_update()
        lf = full.last_loss()[0]
        ls = grp.step()
        gslab = trs[0].grads_tensor().cpu().numpy().astype(np.float64)
        out.append((lf, ls, rel_l2(gslab, gfull)))
    pf = full.params()
    ps = [t.params() for t in trs]
    return out, pf, ps


@pytest.mark.parametrize("R,n,c,w,h,L", [
    (1, 400, 3, 64, 48, 1),
    (2, 400, 3, 64, 48, 1),
    (4, 400, 3, 64, 48, 2),
    (2, 3000, 1, 256, 256, 1),    # cfg1 grid, compile-time planned FFT
    (4, 800, 2, 96, 64, 3),
])
def test_slab_step_matches_unsharded(holo, R, n, c, w, h, L):
    out, pf, ps = run(holo, R, n, c, w, h, L, steps=3)
    for lf, ls, gerr in out:
        assert ls == pytest.approx(lf, rel=2e-6), (lf, ls)
        assert gerr < GRAD_TOL, gerr
    for p in ps:  # every rank applied the same update
        assert np.array_equal(p, ps[0])
    assert rel_l2(ps[0], pf) < 1e-6


@pytest.mark.parametrize("R,n,c,w,h,L", [
    (1, 400, 3, 64, 48, 1),
    (2, 400, 3, 64, 48, 2),
    (4, 800, 2, 96, 64, 3),
    (16, 3000, 1, 256, 256, 1),   # the maximum peer count, 16-row slabs, 8 column tiles each
])
def test_slab_step_peer_put_matches_unsharded(holo, R, n, c, w, h, L):
    """Peer-put exchange: the pack kernels store into the other ranks' receive
    buffers and signal their device flags (no copy or collective between the
    stages); same results as the unsharded step."""
    out, pf, ps = run(holo, R, n, c, w, h, L, steps=3, put=True)
    for lf, ls, gerr in out:
        assert ls == pytest.approx(lf, rel=2e-6), (lf, ls)
        assert gerr < GRAD_TOL, gerr
    assert rel_l2(ps[0], pf) < 1e-6


def test_slab_step_peer_put_cfg4(holo):
    out, pf, ps = run(holo, 8, 1_000_000, 3, 3840, 2160, 1, steps=2, put=True)
    for lf, ls, gerr in out:
        assert ls == pytest.approx(lf, rel=2e-6), (lf, ls)
        assert gerr < GRAD_TOL, gerr
    assert rel_l2(ps[5], pf) < 1e-6


@pytest.mark.parametrize("R,put", [(2, False), (4, False), (4, True), (8, True)])
def test_slab_step_cfg2_grid(holo, R, put):
    """1080p RGB on the compile-time planned 3840x2160 FFT (CC 4 column tiles):
    the fused slab kernels (row FFT -> peers, column pass gathering its tiles by
    TMA bulk copies from the receive buffer, rows -> peers)."""
    out, pf, ps = run(holo, R, 200_000, 3, 1920, 1080, 1, steps=2, put=put)
    for lf, ls, gerr in out:
        assert ls == pytest.approx(lf, rel=2e-6), (lf, ls)
        assert gerr < GRAD_TOL, gerr
    assert rel_l2(ps[-1], pf) < 1e-6


@pytest.mark.parametrize("R,put", [(2, False), (4, True)])
def test_slab_step_multiplane_planned_grid(holo, R, put):
    """Two planes on the compile-time planned 512x320 grid: the multi-plane
    slab column kernels (segment gather in, one spectrum for every plane,
    loss-band / slab rows straight to the peers or to the local layout)."""
    out, pf, ps = run(holo, R, 2000, 3, 256, 160, 2, steps=3, put=put)
    for lf, ls, gerr in out:
        assert ls == pytest.approx(lf, rel=2e-6), (lf, ls)
        assert gerr < GRAD_TOL, gerr
    assert rel_l2(ps[-1], pf) < 1e-6


def test_slab_step_cfg3_eight_ranks(holo):
    """cfg3 (1080p RGB, 8 depth planes) in 8 row slabs with the peer-put
    exchange fused into the multi-plane column kernels."""
    out, pf, ps = run(holo, 8, 200_000, 3, 1920, 1080, 8, steps=1, put=True)
    lf, ls, gerr = out[0]
    assert ls == pytest.approx(lf, rel=2e-6), (lf, ls)
    assert gerr < GRAD_TOL, gerr
    assert rel_l2(ps[7], pf) < 1e-6


def test_slab_step_tile_backward_matches_unsharded(holo):
    """The default per-tile backward on the row-slab bands (band tile rows
    only) against the unsharded per-tile backward: the decomposition changes
    only the atomic and partial-sum order."""
    from paper_2511_15022_b200 import parallel as P
    R, n, c, w, h, L = 4, 3000, 3, 256, 160, 2
    gs, target, masks, dist, spec = scene(holo, n, c, w, h, L)
    full = holo.Trainer(gs, w, h, target, masks, dist, spec, 20)
    trs = []
    for r in range(R):
        t = holo.Trainer(gs, w, h, target, masks, dist, spec, 20)
        t.set_row_slab(r, R)
        trs.append(t)
    grp = P.LocalSlabGroup(trs, c, h, w, L, put=True)
    for _ in range(2):
        full.forward_backward()
        gfull = full.grads_tensor().cpu().numpy().astype(np.float64)
        full.apply_update()
        lf = full.last_loss()[0]
        ls = grp.step()
        gslab = trs[0].grads_tensor().cpu().numpy().astype(np.float64)
        assert ls == pytest.approx(lf, rel=2e-6), (lf, ls)
        assert rel_l2(gslab, gfull) < GRAD_TOL


def test_slab_step_cfg4_eight_ranks(holo):
    """cfg4 (4K RGB, 1M Gaussians) split into 8 row slabs of 270 rows and 8
    column slabs of 480 two-column tiles of the 7680x4320 spectrum."""
    out, pf, ps = run(holo, 8, 1_000_000, 3, 3840, 2160, 1, steps=1)
    lf, ls, gerr = out[0]
    assert ls == pytest.approx(lf, rel=2e-6), (lf, ls)
    assert gerr < GRAD_TOL, gerr
    assert rel_l2(ps[3], pf) < 1e-6


def test_slab_layout_errors(holo):
    gs, target, masks, dist, spec = scene(holo, 100, 1, 64, 48, 1)
    t = holo.Trainer(gs, 64, 48, target, masks, dist, spec, 5)
    with pytest.raises(holo.HoloInvalidArgument):
        t.set_row_slab(0, 5)      # 48 rows do not split into 5 slabs
    with pytest.raises(holo.HoloInvalidArgument):
        t.set_row_slab(2, 2)      # rank outside the group
    with pytest.raises(holo.HoloInvalidArgument):
        t.slab_stage(0)           # not sharded yet
    t.set_row_slab(1, 2)
    with pytest.raises(holo.HoloInvalidArgument):
        t.slab_stage(7)
    # exchange 0: 24 own rows x 16 four-column tiles per peer (floats);
    # exchange 1 carries each peer's loss band: rank 0 rows [0, 34), rank 1 rows [14, 48)
    assert t.slab_counts(0) == ([2 * 4 * 16 * 24] * 2, [2 * 4 * 16 * 24] * 2)
    assert t.slab_counts(1) == ([2 * 4 * 16 * 34] * 2, [2 * 4 * 16 * 34] * 2)


def test_sharded_nonfinite_is_decided_on_the_summed_gradient(holo):
    """A NaN that only one slab rank sees: after the gradient sum every rank
    re-derives the non-finite groups (hs_trainer_check_grads), so all ranks
    refuse the same update instead of diverging."""
    from paper_2511_15022_b200 import parallel as P
    gs, target, masks, dist, spec = scene(holo, 400, 3, 64, 48, 1)
    vals = target.values.copy()
    vals[0, 40, 30] = np.nan  # inside rank 1's rows only (rows 24..47 of 48)
    bad = holo.RealField(3, 48, 64, vals)
    trs = []
    for r in range(2):
        t = holo.Trainer(gs, 64, 48, bad, masks, dist, spec, 10)
        t.set_row_slab(r, 2)
        trs.append(t)
    p0 = [t.params() for t in trs]
    grp = P.LocalSlabGroup(trs, 3, 48, 64, 1, put=True)
    with pytest.raises(holo.HoloNonFinite):
        grp.step()
        for t in trs:
            t.last_loss()  # raises on the non-finite flag
    for t, p in zip(trs, p0):
        assert np.array_equal(t.params(), p)


def test_channel_shards_agree_on_a_rank_local_nonfinite_group(holo):
    """Wavelength shards keep amplitude/phase rank-local: a NaN in rank 1's
    amplitude gradient (rank 0's is clean) must still stop BOTH ranks from the
    amplitude group on (the reference throws at "amplitude" and never reaches
    phase/opacity), while both apply the same position/scale/rotation update."""
    from paper_2511_15022_b200 import parallel as P
    n, c, w, h, L = 300, 3, 64, 48, 1
    g = {k: np.asarray(v, dtype=np.float32).astype(np.float64) for k, v in S.init_gaussians(n, c, w, h, 5).items()}
    img = S.synthetic_image(42, c, h, w)
    masks = S.build_masks(S.synthetic_depth(43, h, w), L, True)
    dist = S.make_depth_planes(L, 3e-3, 2e-3)
    wl = S.WAVELENGTHS[c]
    trs = []
    for r in range(2):
        b, e = P.channel_shard(c, r, 2)
        gs = P.slice_channels(g, n, c, b, e)
        trs.append(holo.Trainer(holo.GaussianSet(n, e - b, **gs), w, h, holo.RealField(e - b, h, w, img[b:e]),
                                masks, dist, holo.PropagationSpec(wl[b:e]), 10, channels_total=c))
    p0 = [t.params() for t in trs]
    for t in trs:
        t.forward_backward()
    grads = [t.grads_tensor() for t in trs]
    grads[1][5 * n + 7] = float("nan")  # rank 1's amplitude (rank-local group)
    geo = [P.geometry_ranges(n, 2), P.geometry_ranges(n, 1)]
    for k in range(2):  # the geometry all-reduce, as device copies
        total = grads[0][geo[0][k][0]:geo[0][k][1]] + grads[1][geo[1][k][0]:geo[1][k][1]]
        grads[0][geo[0][k][0]:geo[0][k][1]].copy_(total)
        grads[1][geo[1][k][0]:geo[1][k][1]].copy_(total)
    for t in trs:
        t.check_grads()
    assert int(trs[0].flags_tensor().item()) == 0 and int(trs[1].flags_tensor().item()) == 1 << 3
    P.agree_nonfinite_local(trs)
    watches = [P.ErrorWatch(t) for t in trs]
    for t, wt in zip(trs, watches):
        t.apply_update()
        with pytest.raises(holo.HoloNonFinite, match="group amplitude"):
            wt.post()  # raises at once when the copy has landed, else at flush()
            wt.flush()
    q = [t.params() for t in trs]
    for r, cl in ((0, 2), (1, 1)):
        geo0, opa = slice(0, 5 * n), slice(5 * n + 2 * n * cl, 6 * n + 2 * n * cl)
        assert not np.array_equal(q[r][geo0], p0[r][geo0])          # position/scale/rotation updated
        assert np.array_equal(q[r][5 * n:], p0[r][5 * n:])          # amplitude, phase, opacity untouched
    assert np.array_equal(q[0][:5 * n], q[1][:5 * n])                # the same geometry update on both ranks


def _native_scene(holo, n=400, c=3, w=64, h=48, L=2, seed=42, bad=False):
    gs, target, masks, dist, spec = scene(holo, n, c, w, h, L, seed)
    if bad:
        vals = target.values.copy()
        vals[1, 10, 10] = np.nan
        target = holo.RealField(c, h, w, vals)
    return gs, target, masks, dist, spec


@pytest.mark.parametrize("mode", ["unsharded", "slab"])
def test_native_nccl_sharded_step_one_rank(holo, mode):
    """hs_trainer_sharded_step over a 1-rank NCCL communicator held by the
    context: the all-reduces, the non-finite agreement, the loss recombination
    and (row slabs) the grouped ncclSend/ncclRecv transposes all run, and the
    step equals the plain trainer step."""
    from paper_2511_15022_b200 import parallel as P
    gs, target, masks, dist, spec = _native_scene(holo)
    ref = holo.Trainer(gs, 64, 48, target, masks, dist, spec, 10)
    t = holo.Trainer(gs, 64, 48, target, masks, dist, spec, 10)
    if mode == "slab":
        t.set_row_slab(0, 1)
    step = P.NativeShardedStep(t)
    try:
        for _ in range(3):
            lr = ref.step(sync_loss=True)
            ln = step.step(with_loss=True)
            assert ln == pytest.approx(lr, rel=2e-6), (ln, lr)
        assert rel_l2(t.params(), ref.params()) < 1e-6
    finally:
        step.close()


def test_native_nccl_sharded_step_raises_nonfinite(holo):
    from paper_2511_15022_b200 import parallel as P
    gs, target, masks, dist, spec = _native_scene(holo, bad=True)
    t = holo.Trainer(gs, 64, 48, target, masks, dist, spec, 10)
    p0 = t.params()
    step = P.NativeShardedStep(t)
    try:
        with pytest.raises(holo.HoloNonFinite, match="group position"):
            step.step(with_loss=True)
        assert np.array_equal(t.params(), p0)
    finally:
        step.close()
