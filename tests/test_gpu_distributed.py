"""Sample-space partition on the GPU.

* two processes sharing cuda:0, each rendering its block of every pass through
  `distributed.gpu_distributed_renderer` and summing over gloo (NCCL cannot put two ranks on one
  device): the reduced framebuffer equals a single-context render bit for bit;
* the library's own NCCL path at world size 1 (communicator from lw_comm_unique_id /
  lw_ctx_comm_init, in-place lw_framebuffer_reduce) and lw_framebuffer_accumulate.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

W, H, DEPTH, SPP, PASS = 48, 32, 6, 9, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1705_01263_b200 import scenes
    from paper_1705_01263_b200.distributed import gpu_distributed_renderer, pass_schedule
    from paper_1705_01263_b200.render import Renderer
    from paper_1705_01263_b200.scene import pack_scene

    with Renderer(None, W, H, DEPTH, device=0, packed=pack_scene(scenes.cornell()), pool_log2=12) as r:
        dr = gpu_distributed_renderer(r, rank, world, backend="gloo")
        for a, b in pass_schedule(SPP, PASS):
            dr.run_pass(a, b)
        red = dr.reduced()
    if rank == 0:
        np.save(out_path, red)
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_on_one_gpu_equal_single_context(tmp_path, gpu):
    import torch.multiprocessing as mp

    from paper_1705_01263_b200 import scenes
    from paper_1705_01263_b200.render import Renderer
    from paper_1705_01263_b200.scene import pack_scene

    out = str(tmp_path / "fb.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    with Renderer(None, W, H, DEPTH, device=0, packed=pack_scene(scenes.cornell())) as r:
        r.render_pass(0, SPP)
        ref = r.framebuffer()
    assert ref.sum() > 0
    assert np.array_equal(np.load(out), ref)


def test_library_nccl_reduce_world1_and_accumulate(gpu):
    import torch

    from paper_1705_01263_b200 import scenes
    from paper_1705_01263_b200.render import Renderer
    from paper_1705_01263_b200.scene import pack_scene

    with Renderer(None, W, H, DEPTH, device=0, packed=pack_scene(scenes.cornell()), pool_log2=12) as r:
        uid = Renderer.comm_unique_id()
        assert len(uid) == 128
        r.comm_init(uid, 0, 1)
        r.render_pass(0, 3)
        fb = r.framebuffer()
        r.reduce_framebuffer()  # NCCL all-reduce over one rank: identity
        assert np.array_equal(r.framebuffer(), fb)
        glob = torch.zeros((W * H, 3), dtype=torch.int64, device="cuda")
        r.set_stream(torch.cuda.current_stream().cuda_stream)
        r.accumulate_into(glob.data_ptr())          # glob += fb, fb = 0
        r.render_pass(3, 5)
        r.accumulate_into(glob.data_ptr())
        torch.cuda.synchronize()
        assert not r.framebuffer().any()
        r.render_pass(0, 5)
        assert np.array_equal(glob.cpu().numpy(), r.framebuffer())


def test_comm_init_rejects_bad_arguments(gpu):
    from paper_1705_01263_b200 import scenes
    from paper_1705_01263_b200.render import Renderer
    from paper_1705_01263_b200.scene import pack_scene

    with Renderer(None, 8, 8, 2, device=0, packed=pack_scene(scenes.cornell()), pool_log2=10) as r:
        with pytest.raises(ValueError):
            r.comm_init(b"x" * 127, 0, 1)
        with pytest.raises(ValueError):
            r.comm_init(Renderer.comm_unique_id(), 2, 2)
        with pytest.raises(Exception):  # no communicator yet
            r.reduce_framebuffer()
