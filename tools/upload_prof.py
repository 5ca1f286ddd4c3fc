"""One scene upload (C3 by default) for an ncu launch list of the BVH build kernels."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1705_01263_b200 import _abi, scenes  # noqa: E402
from paper_1705_01263_b200.scene import pack_scene  # noqa: E402

lib = _abi.lib()
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
packed = pack_scene(scenes.CONFIGS[cfg].builder()).pinned()
for _ in range(2):
    h = C.c_void_p()
    assert lib.lw_ctx_create(0, C.byref(h)) == 0
    assert lib.lw_scene_upload(h, C.byref(packed.desc)) == 0
    torch.cuda.synchronize()
    lib.lw_ctx_destroy(h)
