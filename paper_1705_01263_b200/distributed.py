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

LW_COMM_ID_BYTES = 128  # include/lw_b200.h (the NCCL unique id)


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

    def __init__(self, render_fn, fetch_fb, rank: int, world: int, group=None, reduce: bool = True):
        self.render_fn, self.fetch_fb = render_fn, fetch_fb
        self.rank, self.world, self.group = rank, world, group
        self.reduce = reduce  # False: fetch_fb already returns the reduced framebuffer

    def run_pass(self, it_begin: int, it_end: int):
        a, b = partition_iterations(it_begin, it_end, self.rank, self.world)
        if b > a:
            self.render_fn(a, b)
        return a, b

    def reduced(self):
        fb = self.fetch_fb()
        if not self.reduce:
            return fb
        return reduce_framebuffer(fb, self.group)


def gpu_distributed_renderer(renderer, rank, world, group=None, backend="nccl"):
    """DistributedRenderer over a GPU `render.Renderer`; `reduced()` returns the summed int64
    framebuffer (H*W, 3) as a host numpy array.

    backend="nccl": the library's own communicator (lw_ctx_comm_init; the unique id is broadcast
    over `group`), an in-place all-reduce of the device framebuffer on the context's stream
    (lw_framebuffer_reduce) -- the path for one process per GPU.
    backend="gloo": framebuffer downloaded and summed over a gloo group on the host -- for several
    processes sharing one GPU (NCCL cannot put two ranks on one device) and CPU-only tests."""
    import torch
    import torch.distributed as dist

    if backend == "nccl":
        if world > 1:
            uid = torch.zeros(LW_COMM_ID_BYTES, dtype=torch.uint8)
            if rank == 0:
                uid[:] = torch.frombuffer(bytearray(renderer.comm_unique_id()), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                uid = uid.to(torch.device("cuda", renderer.device))
            dist.broadcast(uid, src=0, group=group)
            renderer.comm_init(bytes(uid.cpu().numpy().tobytes()), rank, world)

        def fetch():
            if world > 1:
                renderer.reduce_framebuffer()
            return renderer.framebuffer()  # synchronises the context stream

        return DistributedRenderer(lambda a, b: renderer.render_pass(a, b), fetch, rank, world, group,
                                   reduce=False)
    if backend == "gloo":
        def fetch_host():
            t = torch.from_numpy(renderer.framebuffer())
            reduce_framebuffer(t, group)
            return t.numpy()

        return DistributedRenderer(lambda a, b: renderer.render_pass(a, b), fetch_host, rank, world, group,
                                   reduce=False)
    raise ValueError("backend must be 'nccl' or 'gloo'")


def fb_to_image(fb: np.ndarray, width: int, height: int, samples: int) -> np.ndarray:
    return (np.asarray(fb, dtype=np.float64) / (float(1 << 20) * samples)).reshape(height, width, 3).astype(np.float32)
