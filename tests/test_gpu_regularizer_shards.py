"""The per-batch regularizers sharded over ranks ("computed once (rank 0, or sharded
by tet range)"): normal consistency by z-slabs of vertices (ts_normal_consistency_slab, each
pass over its slab plus the halo layers it reads), the eikonal by slices of its tet set.  The
slabs of all ranks must sum to the one-call result: gradients bit for bit (every vertex's
gradient is gathered by exactly one slab, in the same order), the loss to FP64 summation order.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def problem():
    import paper_2406_01579_b200 as ts
    from oracle import ts_oracle as O
    R = 24
    og = O.build_grid(R)
    of = O.noisy_field(og, noise=0.08, deform=0.4, seed=5)
    g = ts.build_grid(R)
    f = ts.FieldState.from_numpy(of.sdf, of.deformation, ts.deform_limit_for(g))
    return ts, g, f, og, of


def _nc(ts, g, f, slabs, fixed=False):
    from paper_2406_01579_b200.losses import nc_scratch_bytes, normal_consistency_loss_async
    out = ts.FixedPointGradients.zeros(g.num_vertices) if fixed else ts.GradientBuffers.zeros(g.num_vertices)
    scratch = torch.empty(nc_scratch_bytes(g), dtype=torch.uint8, device="cuda")
    total = 0.0
    for slab in slabs:
        loss = torch.zeros(1, dtype=torch.float64, device="cuda")
        normal_consistency_loss_async(g, f, out, 1000.0, loss, scratch=scratch, slab=slab)
        total += float(loss)
    return (out.to_float() if fixed else out).d_vert, total


@pytest.mark.parametrize("cuts", [(0, 25), (0, 11, 25), (0, 1, 2, 13, 24, 25), (0, 3, 6, 9, 12, 15, 18, 21, 25)])
def test_nc_slabs_sum_to_full(problem, cuts):
    ts, g, f, _, _ = problem
    full, lfull = _nc(ts, g, f, [None])
    slabs = list(zip(cuts[:-1], cuts[1:]))
    part, lpart = _nc(ts, g, f, slabs)
    assert torch.equal(part, full)
    assert lpart == pytest.approx(lfull, rel=1e-12)
    # fixed point: the same slabs, order-independent integer sums
    fx_full, _ = _nc(ts, g, f, [None], fixed=True)
    fx_part, _ = _nc(ts, g, f, slabs[::-1], fixed=True)
    assert torch.equal(fx_part, fx_full)
    assert float((fx_full - full).abs().max()) <= 1e-5 * float(full.abs().max())


def test_nc_slab_matches_oracle(problem):
    """A middle slab's gradient rows equal the oracle's full normal-consistency gradient there."""
    ts, g, f, og, of = problem
    from oracle import ts_oracle as O
    loss_ref, gb = O.normal_consistency_loss(og, of)
    d, _ = _nc(ts, g, f, [(7, 16)])
    n = 25
    rows = slice(7 * n * n, 16 * n * n)
    ref = np.concatenate([gb.d_sdf[:, None], gb.d_deform], axis=1)[rows] * 1000.0
    got = d.cpu().numpy()[rows]
    den = np.abs(ref).max()
    assert np.abs(got - ref).max() <= 1e-5 * den
    # and nothing outside the slab
    assert not d.cpu().numpy()[: 7 * n * n].any() and not d.cpu().numpy()[16 * n * n:].any()


def test_eikonal_slices_sum_to_full(problem):
    ts, g, f, _, _ = problem
    from paper_2406_01579_b200.losses import eikonal_loss_async
    tets = ts.prefilter(g, f, 20.0)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    a = ts.FixedPointGradients.zeros(g.num_vertices)
    eikonal_loss_async(g, f, tets, a, 1000.0, loss)
    lfull = float(loss)
    b = ts.FixedPointGradients.zeros(g.num_vertices)
    tot = 0.0
    W = 3
    for r in range(W):
        eikonal_loss_async(g, f, tets[r * tets.numel() // W:(r + 1) * tets.numel() // W], b, 1000.0, loss)
        tot += float(loss)
    assert torch.equal(a.fx, b.fx)
    assert tot == pytest.approx(lfull, rel=1e-12)
