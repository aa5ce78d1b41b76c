"""GPU parity of the NEXT-2 row (majority voting and sphere fitting) against the
oracle (oracle/voting.py): vote counts and membership exact (the fp64 projection takes the same
decisions), sphere centres and radii within fp32 rounding."""
import numpy as np
import pytest

from oracle import voting as Vt
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _opt(sc):
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    p = GaussianParams.from_scene(sc)
    return p, LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, len(sc.cameras), sc.width, sc.height))


def test_majority_vote_matches_oracle(torch_cuda):
    torch = torch_cuda
    sc = synth.make_scene("c2", n=30000, width=320, height=240, n_views=6)
    masks = synth.change_masks(sc)
    p, opt = _opt(sc)
    member, c, o = opt.majority_vote(p.mean_op, sc.cameras, torch.from_numpy(masks).cuda())
    c_o, o_o = Vt.vote_counts(sc.means, sc.cameras, masks)
    assert np.array_equal(c.cpu().numpy(), c_o) and np.array_equal(o.cpu().numpy(), o_o)
    mem_o = Vt.majority(c_o, o_o, len(sc.cameras))
    assert np.array_equal(member.cpu().numpy(), mem_o)
    assert mem_o.sum() > 0 and (~mem_o).sum() > 0      # the seeded masks exercise both outcomes
    opt.close()


def test_fit_spheres_matches_oracle(torch_cuda):
    torch = torch_cuda
    sc = synth.make_scene("c2", n=40000, width=320, height=240, n_views=2)
    rng = np.random.default_rng(5)
    K = 5
    seeds = sc.means[rng.choice(sc.n, K, replace=False)]
    d = ((sc.means[:, None, :] - seeds[None]) ** 2).sum(-1)
    labels = d.argmin(1).astype(np.int32)
    labels[d.min(1) > 0.3] = -1                          # unclustered points
    labels[rng.random(sc.n) < 0.01] = -1
    p, opt = _opt(sc)
    centres, radii = opt.fit_spheres(p.mean_op, torch.from_numpy(labels).cuda(), K)
    c_o, r_o = Vt.fit_spheres(sc.means, labels, K)
    assert np.allclose(centres.cpu().numpy(), c_o, rtol=1e-6, atol=1e-6)
    assert np.allclose(radii.cpu().numpy(), r_o, rtol=2e-6, atol=1e-7)
    opt.close()
