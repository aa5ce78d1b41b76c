"""Debug helper (not part of the product): run the CUDA path and the oracle on a config and
dump the pixels that differ by more than 1e-4 and are not flagged ambiguous."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import synth  # noqa: E402
from tests import gpu_helpers as H  # noqa: E402

name = sys.argv[1]
if name == "c5s":
    sc = synth.make_scene("c5", n=150000, n_views=5)
elif name == "c4v":
    full = synth.make_scene("c4")
    sc = synth.Scene(full.name, full.means, full.log_scales, full.quats, full.opacity_logits, full.sh, full.sh_degree,
                     full.cameras[:2], full.regions, full.targets[:2])
g = H.gpu_run(sc)
fb = oracle.forward_backward(sc, with_grad=False)
out = []
for v, r in enumerate(fb["renders"]):
    d = np.abs(g["images"][v].astype(np.float64) - r["image"]).max(axis=0)
    bad = np.argwhere((d > 1e-4) & ~r["ambiguous"])
    for y, x in bad[:10]:
        out.append(dict(view=v, x=int(x), y=int(y), gpu=g["images"][v][:, y, x].tolist(),
                        orc=r["image"][:, y, x].tolist(), T=float(r["T_final"][y, x]), nc=int(r["n_contrib"][y, x])))
print(json.dumps(out))
json.dump(out, open(f"gpurun_out/bad_{name}.json", "w"))
