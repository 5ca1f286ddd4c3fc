"""Wall time of lw_scene_upload (pinned inputs) per config, after one warm-up upload."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1705_01263_b200 import _abi, scenes  # noqa: E402
from paper_1705_01263_b200.scene import pack_scene  # noqa: E402

lib = _abi.lib()
for cfg in sys.argv[1:] or ["C2"]:
    packed = pack_scene(scenes.CONFIGS[cfg].builder()).pinned()
    ts = []
    for i in range(6):
        h = C.c_void_p()
        lib.lw_ctx_create(0, C.byref(h))
        torch.cuda.synchronize()
        t = time.perf_counter()
        assert lib.lw_scene_upload(h, C.byref(packed.desc)) == 0
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
        lib.lw_ctx_destroy(h)
    print(cfg, "upload ms (median of 5 after warm-up):", round(sorted(ts[1:])[2], 2))
