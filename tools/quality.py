"""Equal-sample and equal-time image error of the optional samplers (light hierarchy, environment
pyramid) against the alias tables, on the GPU at the configs' full resolution.

    python tools/quality.py [C5|C4] [spp] [ref_spp]
The reference is the mean of both samplers' renders at ref_spp (unbiased either way)."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1705_01263_b200 import scenes  # noqa: E402
from paper_1705_01263_b200.render import Renderer  # noqa: E402
from paper_1705_01263_b200.scene import pack_scene  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
spp = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ref_spp = int(sys.argv[3]) if len(sys.argv) > 3 else 512
c = scenes.CONFIGS[cfg]
sc = c.builder()
variants = {"alias": {}, "tree": {"lights": "tree"}} if cfg == "C5" else {"alias": {}, "pyramid": {"env_sampling": "pyramid"}}


def render(kw, it0, n):
    with Renderer(None, c.width, c.height, c.max_depth, packed=pack_scene(sc, **kw)) as r:
        r.render_pass(it0, it0 + 1)  # warm-up (pool allocation), discarded
        r.clear()
        torch.cuda.synchronize()
        t = time.perf_counter()
        r.render_pass(it0, it0 + n)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        return r.image(n).astype(np.float64), dt


refs = [render(kw, 100000, ref_spp)[0] for kw in variants.values()]
ref = sum(refs) / len(refs)
out = {"config": cfg, "spp": spp, "ref_spp_per_sampler": ref_spp, "resolution": [c.width, c.height]}
for name, kw in variants.items():
    img, dt = render(kw, 0, spp)
    rmse = float(np.sqrt(((img - ref) ** 2).mean()))
    out[name] = {"seconds": dt, "rmse": rmse, "rel_rmse": rmse / float(ref.mean()),
                 "efficiency": 1.0 / (rmse ** 2 * dt)}  # 1 / (variance x time): higher is better
names = list(variants)
out["efficiency_ratio"] = out[names[1]]["efficiency"] / out[names[0]]["efficiency"]
print(json.dumps(out))
