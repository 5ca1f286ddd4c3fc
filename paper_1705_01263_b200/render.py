"""Render entry points: scene in, progressive framebuffer out.

Implements the call stack the reference declares but does not ship
(`lumenwave.cli:main` -> `cmd_render`, SPEC.md:765-773 -> scheduler -> wavefront
-> integrator).  One `Renderer` owns one GPU context (liblw_b200.so `lw_ctx`);
multi-GPU rendering partitions QMC sample space (distributed.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from paper_1705_01263_b200 import _abi
from paper_1705_01263_b200._abi import LwRenderParams, LwRenderStats, check, ptr
from paper_1705_01263_b200.qmc import DimensionTable
from paper_1705_01263_b200.scene import pack_scene

ENGINES = {"wavefront": _abi.LW_ENGINE_WAVEFRONT, "megakernel": _abi.LW_ENGINE_MEGAKERNEL}
FB_SCALE = float(1 << _abi.LW_FB_FRAC_BITS)


class RenderParams:
    """Resolution, depth, QMC dimension table and engine knobs (LwRenderParams + owned arrays)."""

    def __init__(self, width, height, max_depth=8, rr_start=4, engine="wavefront", pool_log2=24,
                 regen_fraction=0.5, megakernel_tail=0):
        if engine not in ENGINES:
            raise ValueError(f"unknown engine '{engine}'")
        self.width, self.height, self.max_depth = int(width), int(height), int(max_depth)
        self.table = DimensionTable(max(self.max_depth, 1))
        self.bases = np.ascontiguousarray(self.table.bases, dtype=np.int64)
        self.perm_flat = np.ascontiguousarray(self.table.perm_flat, dtype=np.int64)
        self.perm_offset = np.ascontiguousarray(self.table.perm_offset, dtype=np.int64)
        s = LwRenderParams()
        s.width, s.height, s.max_depth, s.rr_start = self.width, self.height, self.max_depth, int(rr_start)
        s.ndims = len(self.bases)
        s.bases = ptr(self.bases, C.c_int64)
        s.perm_flat = ptr(self.perm_flat, C.c_int64)
        s.perm_len = len(self.perm_flat)
        s.perm_offset = ptr(self.perm_offset, C.c_int64)
        s.engine = ENGINES[engine]
        s.pool_log2 = int(pool_log2)
        s.regen_fraction = float(regen_fraction)
        s.megakernel_tail = int(megakernel_tail)
        self.struct = s
        self.engine = engine

    @property
    def pixels(self):
        return self.width * self.height


class Renderer:
    """Progressive renderer on one GPU."""

    def __init__(self, scene, width, height, max_depth=8, device=0, engine="wavefront", p_env=0.5, rr_start=4,
                 pool_log2=24, regen_fraction=0.5, megakernel_tail=0, packed=None):
        self.lib = _abi.lib()
        self.packed = packed if packed is not None else pack_scene(scene, p_env=p_env)
        self.params = RenderParams(width, height, max_depth, rr_start, engine, pool_log2, regen_fraction,
                                   megakernel_tail)
        self.device = int(device)
        h = C.c_void_p()
        check(self.lib.lw_ctx_create(self.device, C.byref(h)))
        self.ctx = h
        try:
            check(self.lib.lw_scene_upload(self.ctx, C.byref(self.packed.desc)))
            check(self.lib.lw_render_configure(self.ctx, C.byref(self.params.struct)))
        except Exception:
            self.close()
            raise
        self.iterations = 0

    # -- lifecycle
    def close(self):
        if getattr(self, "ctx", None):
            self.lib.lw_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- rendering
    def clear(self):
        check(self.lib.lw_framebuffer_clear(self.ctx))
        self.iterations = 0

    def render_pass(self, it_begin, it_end, pix_begin=0, pix_end=None):
        """Accumulate iterations [it_begin, it_end) (optionally a pixel range) into the framebuffer."""
        if pix_end is None:
            pix_end = self.params.pixels
        check(self.lib.lw_render_pass_pixels(self.ctx, int(it_begin), int(it_end), int(pix_begin), int(pix_end)))
        self.iterations += int(it_end) - int(it_begin)

    def synchronize(self):
        check(self.lib.lw_ctx_synchronize(self.ctx))

    def framebuffer(self) -> np.ndarray:
        """Raw int64 fixed-point framebuffer, (H*W, 3) in units of 2^-20 radiance."""
        fb = np.empty((self.params.pixels, 3), dtype=np.int64)
        check(self.lib.lw_framebuffer_download(self.ctx, ptr(fb, C.c_int64)))
        return fb

    def image(self, samples=None, out=None) -> np.ndarray:
        """Resolved (H, W, 3) float32 radiance = framebuffer / samples per pixel (GPU resolve).

        `out`: optional C-contiguous float32 (H, W, 3) array to fill (e.g. a view of pinned memory)."""
        samples = self.iterations if samples is None else samples
        shape = (self.params.height, self.params.width, 3)
        if out is None:
            out = np.empty(shape, dtype=np.float32)
        if out.shape != shape or out.dtype != np.float32 or not out.flags["C_CONTIGUOUS"]:
            raise ValueError(f"image out must be a C-contiguous float32 array of shape {shape}")
        check(self.lib.lw_framebuffer_resolve(self.ctx, 1.0 / max(samples, 1), ptr(out, C.c_float)))
        return out

    # -- checkpoint / resume (progressive state = int64 framebuffer + iteration count)
    def _fingerprint(self) -> str:
        import hashlib

        h = hashlib.sha256()
        for k in ("verts", "normals", "material", "emit_tri", "emit_rad"):
            a = self.packed.arrays.get(k)
            if isinstance(a, np.ndarray):
                h.update(np.ascontiguousarray(a).tobytes())
        p = self.params
        h.update(f"{p.width}x{p.height}d{p.max_depth}".encode())
        return h.hexdigest()

    def save_checkpoint(self, path):
        """Framebuffer + progressive state; load_checkpoint on a renderer of the same scene and
        parameters continues the render bit-identically (int64 accumulation)."""
        np.savez(path, fb=self.framebuffer(), iterations=self.iterations, fingerprint=self._fingerprint())

    def load_checkpoint(self, path):
        z = np.load(path)
        if str(z["fingerprint"]) != self._fingerprint():
            raise ValueError("checkpoint belongs to a different scene or resolution/depth")
        fb = np.ascontiguousarray(z["fb"], np.int64)
        check(self.lib.lw_framebuffer_upload(self.ctx, ptr(fb, C.c_int64)))
        self.iterations = int(z["iterations"])

    def copy_framebuffer_to(self, device_ptr: int):
        check(self.lib.lw_framebuffer_copy_device(self.ctx, C.c_void_p(device_ptr)))

    def load_framebuffer_from(self, device_ptr: int):
        check(self.lib.lw_framebuffer_load_device(self.ctx, C.c_void_p(device_ptr)))

    def set_stream(self, stream_handle: int | None):
        """Run this context's work on an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)."""
        check(self.lib.lw_ctx_set_stream(self.ctx, C.c_void_p(stream_handle or None)))

    def set_instrumentation(self, time_kernels=False, count_work=False):
        flags = (_abi.LW_INSTR_TIME if time_kernels else 0) | (_abi.LW_INSTR_COUNT if count_work else 0)
        check(self.lib.lw_ctx_set_instrumentation(self.ctx, flags))

    def kernel_profile(self) -> dict:
        p = _abi.LwKernelProfile()
        check(self.lib.lw_ctx_kernel_profile(self.ctx, C.byref(p)))
        return p.as_dict()

    def stats(self) -> dict:
        s = LwRenderStats()
        check(self.lib.lw_get_stats(self.ctx, C.byref(s)))
        return s.as_dict()

    def last_pass_timing(self) -> dict:
        tr = C.c_double()
        tot = C.c_double()
        ln = C.c_int64()
        check(self.lib.lw_ctx_last_pass_timing(self.ctx, C.byref(tr), C.byref(tot), C.byref(ln)))
        return {"trace_ms": tr.value, "total_ms": tot.value, "launches": ln.value}

    # -- parity surface
    def trace_closest(self, origins, dirs, tmaxs=None):
        o = np.ascontiguousarray(origins, np.float64)
        d = np.ascontiguousarray(dirs, np.float64)
        n = len(o)
        tm = np.full(n, np.inf) if tmaxs is None else np.ascontiguousarray(tmaxs, np.float64)
        t = np.empty(n)
        tri = np.empty(n, np.int64)
        b = np.empty((n, 2))
        check(self.lib.lw_ctx_trace_closest(self.ctx, ptr(o, C.c_double), ptr(d, C.c_double), ptr(tm, C.c_double), n,
                                            ptr(t, C.c_double), ptr(tri, C.c_int64), ptr(b, C.c_double)))
        return t, tri, b

    def trace_any(self, origins, dirs, tmaxs):
        o = np.ascontiguousarray(origins, np.float64)
        d = np.ascontiguousarray(dirs, np.float64)
        tm = np.ascontiguousarray(tmaxs, np.float64)
        occ = np.empty(len(o), np.int32)
        check(self.lib.lw_ctx_trace_any(self.ctx, ptr(o, C.c_double), ptr(d, C.c_double), ptr(tm, C.c_double), len(o),
                                        ptr(occ, C.c_int32)))
        return occ

    # -- light path expressions
    def set_lpe_layers(self, layers: dict | None):
        """Route contributions to output layers {name: expression} (lpe.py syntax); None removes them.
        Layers are cleared with clear(); both engines route them."""
        from paper_1705_01263_b200.lpe import compile_layers

        if not layers:
            check(self.lib.lw_ctx_set_lpe(self.ctx, 0, 0, None, None, 0))
            self.lpe = None
            return None
        t = compile_layers(layers)
        tr = np.ascontiguousarray(t.trans, np.int16)
        ac = np.ascontiguousarray(t.accept, np.uint8)
        check(self.lib.lw_ctx_set_lpe(self.ctx, len(t.names), len(tr), ptr(tr, C.c_int16), ptr(ac, C.c_uint8),
                                      int(t.start)))
        self.lpe = t
        return t

    def layer_framebuffers(self) -> dict:
        """{name: int64 (H*W, 3) fixed-point layer framebuffer}."""
        out = {}
        for k, n in enumerate(self.lpe.names if getattr(self, "lpe", None) else []):
            fb = np.empty((self.params.pixels, 3), dtype=np.int64)
            check(self.lib.lw_ctx_lpe_download(self.ctx, k, ptr(fb, C.c_int64)))
            out[n] = fb
        return out

    def layer_images(self, samples=None) -> dict:
        samples = self.iterations if samples is None else samples
        scale = 1.0 / (1048576.0 * max(samples, 1))
        h, w = self.params.height, self.params.width
        return {n: (fb * scale).astype(np.float32).reshape(h, w, 3) for n, fb in self.layer_framebuffers().items()}

    # -- light hierarchy (scenes packed with lights="tree")
    def light_tree(self):
        """(nodes [n,15] = lo hi tot flux[8], right [n], path [nemit], depth [nemit]) or None."""
        nn = C.c_int64()
        check(self.lib.lw_ctx_light_tree_info(self.ctx, C.byref(nn)))
        if nn.value == 0:
            return None
        ne = self.packed.nemit
        nodes = np.empty((nn.value, 15))
        right = np.empty(nn.value, np.int32)
        path = np.empty(max(ne, 1), np.uint64)
        depth = np.empty(max(ne, 1), np.int32)
        check(self.lib.lw_ctx_light_tree_download(self.ctx, ptr(nodes, C.c_double), ptr(right, C.c_int32),
                                                  ptr(path, C.c_uint64), ptr(depth, C.c_int32)))
        return nodes, right, path[:ne], depth[:ne]

    def light_sample(self, x, nrm, u):
        """sample_light: emitter, selection probability, rescaled uniform."""
        x = np.ascontiguousarray(x, np.float64)
        nrm = np.ascontiguousarray(nrm, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        n = len(u)
        e, p, uo = np.empty(n, np.int64), np.empty(n), np.empty(n)
        check(self.lib.lw_ctx_light_sample(self.ctx, ptr(x, C.c_double), ptr(nrm, C.c_double), ptr(u, C.c_double), n,
                                           ptr(e, C.c_int64), ptr(p, C.c_double), ptr(uo, C.c_double)))
        return e, p, uo

    def light_pdf(self, e, x, nrm):
        """light_pdf's selection factor of emitter e seen from (x, nrm)."""
        e = np.ascontiguousarray(e, np.int64)
        x = np.ascontiguousarray(x, np.float64)
        nrm = np.ascontiguousarray(nrm, np.float64)
        p = np.empty(len(e))
        check(self.lib.lw_ctx_light_pdf(self.ctx, ptr(e, C.c_int64), ptr(x, C.c_double), ptr(nrm, C.c_double), len(e),
                                        ptr(p, C.c_double)))
        return p

    # -- environment pyramid (scenes packed with env="pyramid")
    def env_pyramid_levels(self) -> int:
        n = C.c_int32()
        check(self.lib.lw_ctx_env_pyramid_info(self.ctx, C.byref(n)))
        return n.value

    def env_sample(self, packed_normal, uv):
        """sample_env: base texel, its probability, in-texel (u, v)."""
        pk = np.ascontiguousarray(packed_normal, np.int64)
        uv = np.ascontiguousarray(uv, np.float64)
        n = len(pk)
        t, p, o = np.empty(n, np.int64), np.empty(n), np.empty((n, 2))
        check(self.lib.lw_ctx_env_sample(self.ctx, ptr(pk, C.c_int64), ptr(uv, C.c_double), n, ptr(t, C.c_int64),
                                         ptr(p, C.c_double), ptr(o, C.c_double)))
        return t, p, o

    def env_pdf(self, packed_normal, texel):
        pk = np.ascontiguousarray(packed_normal, np.int64)
        tx = np.ascontiguousarray(texel, np.int64)
        p = np.empty(len(pk))
        check(self.lib.lw_ctx_env_pdf(self.ctx, ptr(pk, C.c_int64), ptr(tx, C.c_int64), len(pk), ptr(p, C.c_double)))
        return p

    def camera_rays(self, sample_index):
        idx = np.ascontiguousarray(sample_index, np.int64)
        o = np.empty((len(idx), 3))
        d = np.empty((len(idx), 3))
        check(self.lib.lw_ctx_camera_rays(self.ctx, ptr(idx, C.c_int64), len(idx), ptr(o, C.c_double),
                                          ptr(d, C.c_double)))
        return o, d

    def bvh(self):
        nn = C.c_int64()
        check(self.lib.lw_ctx_bvh_info(self.ctx, C.byref(nn)))
        k = nn.value
        bounds = np.empty((k, 6))
        children = np.empty((k, 2), np.int64)
        order = np.empty(max(self.packed.ntris, 1), np.int64)
        check(self.lib.lw_ctx_bvh_download(self.ctx, ptr(bounds, C.c_double), ptr(children, C.c_int64),
                                           ptr(order, C.c_int64)))
        return bounds, children, order[: self.packed.ntris]


def render(scene, width, height, spp, max_depth=8, device=0, pass_iterations=16, engine="wavefront", **kw):
    """Progressive render generator: yields (iterations_done, float32 (H, W, 3) image) after every pass."""
    with Renderer(scene, width, height, max_depth, device=device, engine=engine, **kw) as r:
        done = 0
        while done < spp:
            step = min(pass_iterations, spp - done)
            r.render_pass(done, done + step)
            done += step
            yield done, r.image(done)


def render_batch(packed, width, height, max_depth, it_begin, it_end, devices=(0,), contexts_per_device=1,
                 cap=64, **renderer_kw):
    """Batch-mode multi-device render of iterations [it_begin, it_end) (scheduler.BatchScheduler,
    PAPER.md:779-817): dynamic iteration sets, throttled merges, failure re-render.  Returns the
    master int64 framebuffer (H*W, 3) and the ledger metrics.  The image is bit-identical to a
    single-context render of the same iterations."""
    from paper_1705_01263_b200.scheduler import BatchScheduler, WorkerProfile

    slots = [d for d in devices for _ in range(contexts_per_device)]
    profiles = [WorkerProfile(k) for k in range(len(slots))]
    sch = BatchScheduler(lambda w: Renderer(None, width, height, max_depth, device=slots[w], packed=packed,
                                            **renderer_kw), profiles, cap=cap)
    fb = sch.run(it_begin, it_end)
    return fb, sch.ledger.metrics()
