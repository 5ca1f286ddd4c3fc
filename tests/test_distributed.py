"""Sample-space partition + framebuffer sum-reduction across ranks (gloo, world_size 2, CPU).

The per-rank worker is the CPU oracle renderer (same role the GPU Renderer plays
under NCCL); the reduced framebuffer must equal the single-process render bit for
bit (GPU-count independence)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path, W, H, depth, spp, pass_its):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_1705_01263_b200 import scenes
    from paper_1705_01263_b200.distributed import DistributedRenderer, pass_schedule
    from paper_1705_01263_b200.render import RenderParams
    from paper_1705_01263_b200.scene import pack_scene

    os_ = O.OracleScene(pack_scene(scenes.cornell()))
    params = RenderParams(W, H, depth)
    local = np.zeros((W * H, 3), np.int64)

    def render_fn(a, b):
        fb, _ = os_.render(params, a, b, nthreads=2)
        local[:] += fb

    dr = DistributedRenderer(render_fn, lambda: torch.from_numpy(local.copy()), rank, world)
    for a, b in pass_schedule(spp, pass_its):
        dr.run_pass(a, b)
    red = dr.reduced()
    if rank == 0:
        np.save(out_path, red.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_reduction_equals_single_process(tmp_path, world):
    W, H, depth, spp = 32, 24, 4, 7
    out = str(tmp_path / "fb.npy")
    mp.spawn(_worker, args=(world, _free_port(), out, W, H, depth, spp, 3), nprocs=world, join=True)
    from oracle import oracle as O
    from paper_1705_01263_b200 import scenes
    from paper_1705_01263_b200.render import RenderParams
    from paper_1705_01263_b200.scene import pack_scene

    fb, _ = O.OracleScene(pack_scene(scenes.cornell())).render(RenderParams(W, H, depth), 0, spp)
    assert np.array_equal(np.load(out), fb)
