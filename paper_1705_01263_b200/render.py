"""Render entry points: scene in, progressive framebuffer out.

Implements the call stack the reference declares but does not ship
(`lumenwave.cli:main` -> `cmd_render`, SPEC.md:765-773 -> scheduler -> wavefront
-> integrator).  One `Renderer` owns one GPU context (liblw_b200.so `lw_ctx`);
multi-GPU rendering partitions QMC sample space (distributed.py).
"""

from __future__ import annotations

import ctypes as C
import functools

import numpy as np

from paper_1705_01263_b200 import _abi
from paper_1705_01263_b200._abi import LwRenderParams, LwRenderStats, check, ptr
from paper_1705_01263_b200.qmc import DimensionTable
from paper_1705_01263_b200.scene import pack_scene

ENGINES = {"wavefront": _abi.LW_ENGINE_WAVEFRONT, "megakernel": _abi.LW_ENGINE_MEGAKERNEL}
ESTIMATORS = {"mis": _abi.LW_EST_MIS, "nee": _abi.LW_EST_NEE, "bsdf": _abi.LW_EST_BSDF}
FB_SCALE = float(1 << _abi.LW_FB_FRAC_BITS)


@functools.lru_cache(maxsize=None)
def _dimension_table(depth: int):
    """DimensionTable(depth) and its int64 arrays, built once per depth (qmc.py:274-305 is a pure
    function of the depth; building it costs milliseconds of Python per Renderer otherwise).  The
    arrays are shared read-only."""
    t = DimensionTable(depth)
    arrs = [np.ascontiguousarray(a, dtype=np.int64) for a in (t.bases, t.perm_flat, t.perm_offset)]
    for a in arrs:
        a.setflags(write=False)
    return (t, *arrs)


class RenderParams:
    """Resolution, depth, QMC dimension table and engine knobs (LwRenderParams + owned arrays)."""

    def __init__(self, width, height, max_depth=8, rr_start=4, engine="wavefront", pool_log2=24,
                 regen_fraction=0.5, megakernel_tail=0, estimator="mis", compact_state=False):
        if engine not in ENGINES:
            raise ValueError(f"unknown engine '{engine}'")
        if estimator not in ESTIMATORS:
            raise ValueError(f"unknown estimator '{estimator}' (mis, nee, bsdf)")
        self.width, self.height, self.max_depth = int(width), int(height), int(max_depth)
        self.table, self.bases, self.perm_flat, self.perm_offset = _dimension_table(max(self.max_depth, 1))
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
        s.estimator = ESTIMATORS[estimator]
        s.compact_state = int(bool(compact_state))
        self.compact_state = bool(compact_state)
        self.struct = s
        self.engine = engine

    @property
    def pixels(self):
        return self.width * self.height


class Renderer:
    """Progressive renderer on one GPU."""

    def __init__(self, scene, width, height, max_depth=8, device=0, engine="wavefront", p_env=0.5, rr_start=4,
                 pool_log2=24, regen_fraction=0.5, megakernel_tail=0, packed=None, estimator="mis",
                 compact_state=False):
        self.lib = _abi.lib()
        self.packed = packed if packed is not None else pack_scene(scene, p_env=p_env)
        self.params = RenderParams(width, height, max_depth, rr_start, engine, pool_log2, regen_fraction,
                                   megakernel_tail, estimator, compact_state)
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
        """Accumulate iterations [it_begin, it_end) (optionally a pixel range) into the framebuffer.
        Asynchronous: returns once the pass is queued (one CUDA-graph launch with device-side
        termination); framebuffer(), image(), stats() and synchronize() wait for it."""
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
        """Hash of everything that determines the image: every scene array (geometry, materials,
        emitters, environment), every scalar of the scene description (camera, environment
        constants and scale, p_env, BVH and sampler choices) and the render parameters that change
        samples (resolution, depth, Russian-roulette start, QMC tables).  Engine knobs (engine,
        pool size, regeneration, megakernel tail) are left out: the image does not depend on them."""
        import hashlib

        h = hashlib.sha256()
        for k in sorted(self.packed.arrays):
            a = self.packed.arrays[k]
            if isinstance(a, np.ndarray):
                h.update(k.encode() + np.ascontiguousarray(a).tobytes())
            elif isinstance(a, C.Array):  # packed lw_material records
                h.update(k.encode() + bytes(a))
        d = self.packed.desc
        for name, ctype in d._fields_:
            if issubclass(ctype, (C._Pointer, C.c_void_p)):
                continue
            v = getattr(d, name)
            h.update(f"{name}={list(v) if isinstance(v, C.Array) else v!r};".encode())
        p = self.params
        s = p.struct
        h.update(f"{s.width}x{s.height}d{s.max_depth}rr{s.rr_start}e{s.estimator}c{s.compact_state}".encode())
        for a in (p.bases, p.perm_flat, p.perm_offset):
            h.update(a.tobytes())
        return h.hexdigest()

    def save_checkpoint(self, path):
        """Framebuffer + progressive state (+ the LPE layer framebuffers and their expressions);
        load_checkpoint on a renderer of the same scene and parameters continues the render
        bit-identically (int64 accumulation)."""
        extra = {}
        if getattr(self, "lpe", None):
            extra["layer_names"] = np.array(self.lpe.names)
            extra["layer_exprs"] = np.array([self.lpe_exprs[n] for n in self.lpe.names])
            for k, fb in enumerate(self.layer_framebuffers().values()):
                extra[f"layer_fb_{k}"] = fb
        np.savez(path, fb=self.framebuffer(), iterations=self.iterations, fingerprint=self._fingerprint(), **extra)

    def load_checkpoint(self, path):
        """Restore a checkpoint.  A checkpoint with LPE layers restores them too (the expressions
        must equal the layers already set on this renderer, if any); one without layers is refused
        by a renderer that has layers (their framebuffers would start from zero while the beauty
        does not)."""
        z = np.load(path)
        if str(z["fingerprint"]) != self._fingerprint():
            raise ValueError("checkpoint belongs to a different scene, camera, material set, environment or "
                             "resolution/depth")
        saved = dict(zip([str(x) for x in z["layer_names"]], [str(x) for x in z["layer_exprs"]])) \
            if "layer_names" in z.files else {}
        have = dict(getattr(self, "lpe_exprs", None) or {}) if getattr(self, "lpe", None) else {}
        if have and have != saved:
            raise ValueError("checkpoint LPE layers differ from this renderer's layers")
        if saved and not have:
            self.set_lpe_layers(saved)
        fb = np.ascontiguousarray(z["fb"], np.int64)
        check(self.lib.lw_framebuffer_upload(self.ctx, ptr(fb, C.c_int64)))
        for k in range(len(saved)):
            lf = np.ascontiguousarray(z[f"layer_fb_{k}"], np.int64)
            check(self.lib.lw_ctx_lpe_upload(self.ctx, k, ptr(lf, C.c_int64)))
        self.iterations = int(z["iterations"])

    def accumulate_into(self, device_ptr: int, clear: bool = True):
        """dst (caller-owned device int64 (H*W, 3), 16-byte aligned) += framebuffer, and zero the
        framebuffer for the next pass (clear=True): one asynchronous kernel on the context stream."""
        check(self.lib.lw_framebuffer_accumulate(self.ctx, C.c_void_p(device_ptr), int(bool(clear))))

    # -- sample-space partition across GPUs: NCCL inside the library
    @staticmethod
    def comm_unique_id() -> bytes:
        """New NCCL unique id (create on rank 0, broadcast to the others)."""
        buf = (C.c_uint8 * _abi.LW_COMM_ID_BYTES)()
        check(_abi.lib().lw_comm_unique_id(buf))
        return bytes(buf)

    def comm_init(self, uid: bytes, rank: int, world: int):
        """Join the communicator `uid` as `rank` of `world` (one context per GPU and process)."""
        if len(uid) != _abi.LW_COMM_ID_BYTES:
            raise ValueError(f"communicator id must be {_abi.LW_COMM_ID_BYTES} bytes")
        buf = (C.c_uint8 * _abi.LW_COMM_ID_BYTES).from_buffer_copy(uid)
        check(self.lib.lw_ctx_comm_init(self.ctx, buf, int(rank), int(world)))

    def reduce_framebuffer(self):
        """Sum the pass framebuffers of all ranks in place (NCCL all-reduce on the context stream)."""
        check(self.lib.lw_framebuffer_reduce(self.ctx))

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
            self.lpe_exprs = None
            return None
        t = compile_layers(layers)
        tr = np.ascontiguousarray(t.trans, np.int16)
        ac = np.ascontiguousarray(t.accept, np.uint8)
        check(self.lib.lw_ctx_set_lpe(self.ctx, len(t.names), len(tr), ptr(tr, C.c_int16), ptr(ac, C.c_uint8),
                                      int(t.start)))
        self.lpe = t
        self.lpe_exprs = dict(layers)
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

    # -- known-answer surface of the light sampling
    def nee_light_sample(self, points, facing_normals, uv):
        """Light half of NEE at points with facing geometric normals for NEE uniforms uv [n,2]:
        dict of wi, radiance, pdf (solid angle, selection included; 0 = no light), shadow tmax,
        emitter (-1 = environment)."""
        p = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        nrm = np.ascontiguousarray(facing_normals, np.float64).reshape(-1, 3)
        uv = np.ascontiguousarray(uv, np.float64).reshape(-1, 2)
        n = len(uv)
        if len(p) == 1 and n > 1:
            p = np.ascontiguousarray(np.repeat(p, n, axis=0))
        if len(nrm) == 1 and n > 1:
            nrm = np.ascontiguousarray(np.repeat(nrm, n, axis=0))
        wi, le, pdf, tm, e = np.empty((n, 3)), np.empty((n, 3)), np.empty(n), np.empty(n), np.empty(n, np.int64)
        check(self.lib.lw_ctx_nee_light_sample(self.ctx, ptr(p, C.c_double), ptr(nrm, C.c_double),
                                               ptr(uv, C.c_double), n, ptr(wi, C.c_double), ptr(le, C.c_double),
                                               ptr(pdf, C.c_double), ptr(tm, C.c_double), ptr(e, C.c_int64)))
        return {"wi": wi, "radiance": le, "pdf": pdf, "tmax": tm, "emitter": e}

    def emission_pdf(self, origins, dirs, nprev=None):
        """What BSDF sampling meets along (o, d): radiance, the light-sampling pdf MIS weighs it
        against (nprev: packed facing normal of the vertex the ray leaves) and the emitter
        (-1 = environment, -2 = non-emissive surface)."""
        o = np.ascontiguousarray(origins, np.float64).reshape(-1, 3)
        d = np.ascontiguousarray(dirs, np.float64).reshape(-1, 3)
        n = len(d)
        if len(o) == 1 and n > 1:
            o = np.ascontiguousarray(np.repeat(o, n, axis=0))
        npv = np.zeros(n, np.int32) if nprev is None else np.ascontiguousarray(  # packed normals are 32-bit patterns
            np.broadcast_to((np.asarray(nprev, np.int64) & 0xFFFFFFFF).astype(np.uint32).view(np.int32), (n,)))
        le, pdf, e = np.empty((n, 3)), np.empty(n), np.empty(n, np.int64)
        check(self.lib.lw_ctx_emission_pdf(self.ctx, ptr(o, C.c_double), ptr(d, C.c_double), ptr(npv, C.c_int32), n,
                                           ptr(le, C.c_double), ptr(pdf, C.c_double), ptr(e, C.c_int64)))
        return {"radiance": le, "pdf": pdf, "emitter": e}

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
