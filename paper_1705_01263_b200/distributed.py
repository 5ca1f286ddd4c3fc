"""Sample-space partitioning across GPUs and the per-pass framebuffer reduction.

SURVEY.md §8e / PAPER.md:779-817 (batch mode): every rank renders a disjoint,
contiguous block of QMC iterations of each progressive pass into its own
full-resolution int64 fixed-point framebuffer; once per pass the framebuffers
are sum-reduced with NCCL (`torch.distributed.all_reduce`, one rank per GPU).
Integer addition is associative, so the reduced image is bit-identical for any
number of ranks.
"""

from __future__ import annotations

import os

import numpy as np


def partition_iterations(it_begin: int, it_end: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of [it_begin, it_end) for `rank` of `world` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    n = it_end - it_begin
    q, r = divmod(n, world)
    a = it_begin + rank * q + min(rank, r)
    b = a + q + (1 if rank < r else 0)
    return a, b


def pass_schedule(spp: int, pass_iterations: int):
    """Progressive passes [(it_begin, it_end), ...] covering spp iterations."""
    out, k = [], 0
    while k < spp:
        out.append((k, min(spp, k + pass_iterations)))
        k = out[-1][1]
    return out


def env_rank():
    """(rank, world, local_rank) from torchrun's environment (defaults: single process)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0)))


def reduce_framebuffer(fb, group=None):
    """Sum-reduce an int64 framebuffer tensor in place across the process group."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(fb, op=dist.ReduceOp.SUM, group=group)
    return fb


class DistributedRenderer:
    """One rank of a sample-space-partitioned progressive render (one process per GPU).

    `render_fn(it_begin, it_end)` accumulates this rank's iterations into the local
    framebuffer; `fetch_fb()` returns it as a torch int64 tensor on the rank's device.
    The GPU path wires these to `render.Renderer`; the CPU tests wire them to the oracle.
    """

    def __init__(self, render_fn, fetch_fb, rank: int, world: int, group=None):
        self.render_fn, self.fetch_fb = render_fn, fetch_fb
        self.rank, self.world, self.group = rank, world, group

    def run_pass(self, it_begin: int, it_end: int):
        a, b = partition_iterations(it_begin, it_end, self.rank, self.world)
        if b > a:
            self.render_fn(a, b)
        return a, b

    def reduced(self):
        fb = self.fetch_fb()
        return reduce_framebuffer(fb, self.group)


def gpu_distributed_renderer(renderer, rank, world, group=None):
    """DistributedRenderer over a GPU `render.Renderer` (framebuffer copied D2D into a torch tensor)."""
    import torch

    dev = torch.device("cuda", renderer.device)
    buf = torch.empty((renderer.params.pixels, 3), dtype=torch.int64, device=dev)

    def fetch():
        renderer.copy_framebuffer_to(buf.data_ptr())
        return buf

    return DistributedRenderer(lambda a, b: renderer.render_pass(a, b), fetch, rank, world, group)


def fb_to_image(fb: np.ndarray, width: int, height: int, samples: int) -> np.ndarray:
    return (np.asarray(fb, dtype=np.float64) / (float(1 << 20) * samples)).reshape(height, width, 3).astype(np.float32)
