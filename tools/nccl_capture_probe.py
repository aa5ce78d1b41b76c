"""Does the CUDA-graph step capture its NCCL all-reduce?  One rank (torchrun --nproc-per-node 1): the
GraphStep with a forced NCCL all_reduce of the packed loss + rows (a sum over one rank = identity)
against the GraphStep without it; same losses and parameters expected.  Multi-rank NCCL cannot run on
the one-GPU box, so this checks the capture path the bench takes at N > 1."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer, default_limits  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
sc = synth.make_scene("c3", n=150000, n_views=2)
out = []
for forced in (False, True):
    p = GaussianParams.from_scene(sc)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, 2, sc.width, sc.height, max_active=4096),
                         static_cache=True)
    tg = torch.from_numpy(np.ascontiguousarray(sc.targets)).cuda()
    gs = GraphStep(opt, sc.cameras, tg, allreduce=(lambda t: dist.all_reduce(t)) if forced else None)
    losses = [float(gs.replay().item()) for _ in range(4)]
    torch.cuda.synchronize()
    out.append((losses, p.mean_op.cpu().numpy().copy()))
    opt.close()
print("losses", out[0][0], out[1][0])
print("NCCL capture ok:", np.allclose(out[0][0], out[1][0], rtol=1e-6) and np.allclose(out[0][1], out[1][1], rtol=1e-5, atol=1e-6))
dist.destroy_process_group()
