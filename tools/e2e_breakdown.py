"""Wall-clock breakdown of one e2e step per config: context create, scene upload, configure,
pass, image readback, destroy (each phase bracketed by device syncs)."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1705_01263_b200 import _abi, scenes  # noqa: E402
from paper_1705_01263_b200.render import Renderer, RenderParams  # noqa: E402
from paper_1705_01263_b200.scene import pack_scene  # noqa: E402

lib = _abi.lib()
reps = 5
for cfg in [a for a in sys.argv[1:] if not a.startswith("--")] or ["C2"]:
    c = scenes.CONFIGS[cfg]
    packed = pack_scene(c.builder()).pinned()  # as bench.py's e2e: scene arrays in pinned memory
    its = max(1, (1 << 24) // (c.width * c.height))
    params = RenderParams(c.width, c.height, c.max_depth, 4, "wavefront", 22, 0.5, 0)
    for rep in range(reps):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        h = C.c_void_p()
        assert lib.lw_ctx_create(0, C.byref(h)) == 0
        torch.cuda.synchronize(); t.append(time.perf_counter())
        assert lib.lw_scene_upload(h, C.byref(packed.desc)) == 0
        torch.cuda.synchronize(); t.append(time.perf_counter())
        assert lib.lw_render_configure(h, C.byref(params.struct)) == 0
        torch.cuda.synchronize(); t.append(time.perf_counter())
        r = Renderer.__new__(Renderer)
        r.lib, r.ctx, r.params, r.packed, r.iterations, r.device = lib, h, params, packed, 0, 0
        r.render_pass(rep * its, (rep + 1) * its)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        dev1 = r.last_pass_timing()["total_ms"]
        if "--second-pass" in sys.argv:  # a second pass on the same context (wall, device)
            t2 = time.perf_counter()
            r.render_pass(rep * its, (rep + 1) * its)
            torch.cuda.synchronize()
            print(cfg, rep, f"second pass wall {1e3 * (time.perf_counter() - t2):.2f} device {r.last_pass_timing()['total_ms']:.2f}"
                  f" (first pass device {dev1:.2f})", flush=True)
        r.image(its)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        r.close()
        torch.cuda.synchronize(); t.append(time.perf_counter())
        d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
        names = ["create", "upload", "configure", "pass", "image", "destroy"]
        print(cfg, rep, "  ".join(f"{n} {v:.2f}" for n, v in zip(names, d)), f" total {sum(d):.2f} ms", flush=True)
