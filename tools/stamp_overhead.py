"""Device time of C2 passes with and without the stage-timing stamps (LW_INSTR_TIME)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1705_01263_b200 import scenes  # noqa: E402
from paper_1705_01263_b200.render import Renderer  # noqa: E402
from paper_1705_01263_b200.scene import pack_scene  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = scenes.CONFIGS[cfg]
packed = pack_scene(c.builder())
its = max(1, (1 << 24) // (c.width * c.height))
st = torch.cuda.Stream()
with Renderer(None, c.width, c.height, c.max_depth, packed=packed, pool_log2=24) as r:
    r.set_stream(st.cuda_stream)
    for timed in (True, False, True, False):
        r.set_instrumentation(time_kernels=timed)
        for s in range(3):
            r.render_pass(s * its, (s + 1) * its)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        K = 10
        for s in range(3, 3 + K):
            r.render_pass(s * its, (s + 1) * its)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        print(cfg, "stamps" if timed else "plain ", f"{ms:.3f} ms/pass", f"{its * c.width * c.height / ms / 1e3:.1f} Mpaths/s")
