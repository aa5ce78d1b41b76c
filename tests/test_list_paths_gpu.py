"""The three ways the static cache builds the step's per-tile lists must give the same step: direct lists
(default: the step's records unsorted, pairs counted and placed per tile, each tile ordered by rank),
CLS_TL_SORT=1 (record sort + stable pair sort by tile) and CLS_NO_TL=1 (row segments merged in the
raster).  The choice is read when libcls loads, so each runs in its own process; images and losses must be
bit-identical over three steps, including a depth-tie scene (reading R13)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
out = {}
for name, sc in (("c3s", synth.make_scene("c3", n=150000, n_views=2)), ("coplanar", synth.coplanar_scene()),
                 ("c5s", synth.make_scene("c5", n=150000, n_views=5))):
    p = GaussianParams.from_scene(sc)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, len(sc.cameras), sc.width, sc.height),
                         lr=(1e-3,) * 6, static_cache=True)
    tg = torch.from_numpy(np.ascontiguousarray(sc.targets)).cuda()
    for k in range(3):
        r = opt.forward(sc.cameras, tg, images=True)
        out[f"{name}_img{k}"] = r.images.cpu().numpy()
        out[f"{name}_loss{k}"] = np.float32(r.loss.item())
        g = opt.backward(None)
        out[f"{name}_grad{k}"] = g.cpu().numpy()
        opt.adam(g)
    out[f"{name}_pairs"] = np.int64(opt.stats()["n_pairs"])
    opt.close()
np.savez(sys.argv[1], **out)
'''


def _run(tmp_path, tag, env_extra):
    path = str(tmp_path / f"{tag}.npz")
    env = dict(os.environ)
    env.pop("CLS_TL_SORT", None)
    env.pop("CLS_NO_TL", None)
    env.update(env_extra)
    subprocess.run([sys.executable, "-c", WORKER, path], cwd=ROOT, env=env, check=True, timeout=600)
    return dict(np.load(path))


def test_list_paths_agree(tmp_path):
    base = _run(tmp_path, "direct", {})
    for tag, env in (("sort", {"CLS_TL_SORT": "1"}), ("rowseg", {"CLS_NO_TL": "1"})):
        other = _run(tmp_path, tag, env)
        for k, v in base.items():
            if "_grad" in k:   # fp64 sums of the same terms, rounded once: equal up to the last bit
                np.testing.assert_allclose(other[k], v, rtol=1e-6, atol=1e-12, err_msg=f"{tag} {k}")
            elif "_pairs" in k:
                continue   # the row-segment path counts (record, tile) pairs differently
            else:
                assert np.array_equal(other[k], v), f"{tag}: {k} differs"
