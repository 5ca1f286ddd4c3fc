import sys, time; sys.path.insert(0,'.')
import ctypes as C, torch
from paper_1705_01263_b200 import _abi, scenes
from paper_1705_01263_b200.scene import pack_scene
lib=_abi.lib()
packed=pack_scene(scenes.CONFIGS['C3'].builder()).pinned()
for rep in range(3):
    h=C.c_void_p(); lib.lw_ctx_create(0, C.byref(h))
    torch.cuda.synchronize(); t=time.perf_counter()
    assert lib.lw_scene_upload(h, C.byref(packed.desc))==0
    torch.cuda.synchronize(); print('upload ms', (time.perf_counter()-t)*1e3, flush=True)
    lib.lw_ctx_destroy(h)
