#!/usr/bin/env python
"""Headline benchmark: progressive path tracing of C2 (Cornell box 1024x1024, depth 8) in paths/s.

    python bench.py [--gpus N --steps K --warmup W]            # our B200 path (N > 1: self-launches N ranks)
    python bench.py --impl reference [--steps K --warmup W]     # the CPU path on the host cores

A step is one progressive pass of `--pass-iterations` (default: ~16.8 M paths) QMC iterations per GPU
over all pixels (weak scaling: every rank renders its own disjoint iteration block of the global
pass), then the pass framebuffers are sum-reduced in place by the library's NCCL all-reduce
(lw_framebuffer_reduce, N > 1) and accumulated into the progressive image (lw_framebuffer_accumulate).
`value` is whole-job paths/s (device-timed, max over ranks); `e2e` is the same metric through the
public Python API with the scene uploaded from pinned host buffers and the resolved image read back
every step.  The reference package has no renderer: the CPU path is the oracle's C
restatement of the render (oracle/lw_oracle.c, OpenMP over all host threads), "kind": "port"; next
to it `cpu_baseline.reference_kernels` times the reference's OWN compiled kernels (halton_batch,
intersect_batch from oracle/_ref, thread pool over all host cores) on the identical index / ray
batches the GPU kernels consume.

At N = 1 the line also carries `per_config` (C1-C5 of BASELINE.json, each measured in this run) and
`roofline.kernels` (every wavefront stage kernel: CUDA-event time share, algorithmic bytes, ncu DRAM
bytes from profiles/, fraction of the measured HBM peak).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "paths/s"
CONFIGS = ("C1", "C2", "C3", "C4", "C5")


def metric_name(a):
    return f"paths/sec (samples/sec) on {a.config} {a.width}x{a.height} depth {a.depth}"


def build_scene(config):
    from paper_1705_01263_b200 import scenes

    return scenes.CONFIGS[config].builder()


def resolve(a, config):
    """Resolution, depth and iterations per step of `config` (flags override the headline's)."""
    from paper_1705_01263_b200 import scenes

    c = scenes.CONFIGS[config]
    head = config == a.config
    w = (a.width if head and a.width else 0) or c.width
    h = (a.height if head and a.height else 0) or c.height
    d = (a.depth if head and a.depth else 0) or c.max_depth
    its = (a.pass_iterations if head and a.pass_iterations else 0) or max(1, (1 << 24) // (w * h))
    return w, h, d, its


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=list(CONFIGS))
    ap.add_argument("--pass-iterations", type=int, default=0, help="QMC iterations per GPU per step (0: ~16M paths)")
    ap.add_argument("--engine", default="wavefront", choices=["wavefront", "megakernel"])
    ap.add_argument("--pool-log2", type=int, default=24)
    ap.add_argument("--regen-fraction", type=float, default=0.5)
    ap.add_argument("--megakernel-tail", type=int, default=0)
    ap.add_argument("--env-sampling", default="alias", choices=["alias", "pyramid"],
                    help="environment-image sampling: alias table (BASELINE configs) or the normal-binned pyramid")
    ap.add_argument("--lights", default="alias", choices=["alias", "tree"],
                    help="NEE emitter selection: alias table (BASELINE configs) or the light hierarchy")
    ap.add_argument("--width", type=int, default=0)
    ap.add_argument("--height", type=int, default=0)
    ap.add_argument("--depth", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="budget of the bounded CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-per-config", action="store_true", help="skip the C1-C5 table (N = 1 only)")
    ap.add_argument("--state", default="fp64", choices=["fp64", "compact"],
                    help="path state in the wavefront pool: FP64, or compact (oct-16 directions, FP32 "
                         "throughput / radiance / pdf; PAPER.md:632-635)")
    a = ap.parse_args()
    a.width, a.height, a.depth, a.pass_iterations = resolve(a, a.config)
    return a


def workload(a, config=None):
    from paper_1705_01263_b200 import scenes

    config = config or a.config
    w, h, d, its = resolve(a, config)
    return f"{config}: {scenes.CONFIGS[config].description}; {w}x{h}, depth {d}, {its} spp per GPU per step"


def config_dict(a, world):
    """The `config` object of the JSON line -- identical for both arms (same workload, same knobs)."""
    return {"workload": workload(a), "engine": a.engine, "state": a.state, "lights": a.lights,
            "env_sampling": a.env_sampling,
            "pool_slots": 1 << a.pool_log2, "regen_fraction": a.regen_fraction,
            "parallelism": f"sample-space dp{world}",
            "l2": f"wavefront state pool (~{(1 << a.pool_log2) * 250 / 1e9:.1f} GB) exceeds the 126 MB L2 "
                  "(no flush needed); Cornell-box BVHs are shared-memory resident by design"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---- clocks ---------------------------------------------------------------------------------

class ClockSampler:
    """SM clock and clock-event reasons during the timed region: NVML polled every 20 ms from a
    thread (no process start-up lag, so short timed regions still get samples); nvidia-smi as the
    fallback when NVML is unavailable."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.thread = None
        self.samples = []
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.device]) if vis and vis.split(",")[0].isdigit() else self.device
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.stop_flag = threading.Event()

            def poll():
                while not self.stop_flag.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    except Exception:  # noqa: BLE001
                        break
                    self.samples.append((sm, rs))
                    self.stop_flag.wait(0.02)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:  # noqa: BLE001  (no NVML: fall back to nvidia-smi)
            self.thread = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join()
            sm = [float(a) for a, _ in self.samples]
            reasons = sorted({n for _, r in self.samples for bit, n in self.REASONS.items() if r & bit})
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(self.smax),
                    "reasons": reasons, "samples": len(sm), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        os.unlink(self.path)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) < 9:
                continue
            for k, nm in enumerate(names):
                if r[5 + k].strip().lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(rows), "source": "nvidia-smi"}


# ---- CPU path (oracle restatement + the reference's own kernels) -----------------------------

def cpu_render_sample(a, config, budget_s, threads=0, it0=3, gpu=None):
    """Bounded sample of `config`'s workload on the host cores (oracle/lw_oracle.c, OpenMP):
    whole-frame iterations rendered one at a time until the budget is spent (a band of centre rows
    when one frame alone exceeds it).  With `gpu` (a Renderer of the same workload) the same sample
    is rendered on the GPU and compared with the CPU framebuffer (the "RMSE vs ref" half of the
    metric)."""
    import numpy as np

    from oracle import oracle as O
    from paper_1705_01263_b200.render import RenderParams
    from paper_1705_01263_b200.scene import pack_scene

    W, H, D, _ = resolve(a, config)
    packed = pack_scene(build_scene(config), lights=a.lights, env_sampling=a.env_sampling)
    osc = O.OracleScene(packed)
    params = RenderParams(W, H, D, compact_state=a.state == "compact")
    threads = threads or os.cpu_count()
    # probe: 8 centre rows, one iteration (the centre is where the geometry is)
    r0 = max(0, H // 2 - 4)
    t0 = time.perf_counter()
    osc.render(params, it0, it0 + 1, r0 * W, min(H, r0 + 8) * W, nthreads=threads)
    per_row = (time.perf_counter() - t0) / min(8, H - r0)
    if per_row * H <= 0.5 * budget_s:
        p0, p1 = 0, W * H
        desc = "full frames"
    else:
        rows = max(1, min(H, int(0.5 * budget_s / max(per_row, 1e-9))))
        r0 = max(0, H // 2 - rows // 2)
        p0, p1 = r0 * W, (r0 + rows) * W
        desc = f"{rows} centre rows"
    fb_cpu = np.zeros((W * H, 3), np.int64)
    paths = rays = 0
    its = 0
    # iterations per call: enough that one call is ~50 ms (amortises the OpenMP fork/join of tiny frames)
    per_call = max(1, int(0.05 / max(per_row * (p1 - p0) / W, 1e-9)))
    t0 = time.perf_counter()
    while True:
        fb, st = osc.render(params, it0 + its, it0 + its + per_call, p0, p1, nthreads=threads)
        fb_cpu += fb
        paths += st["paths"]
        rays += st["rays_extension"] + st["rays_shadow"]
        its += per_call
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    out = {"value": paths / dt, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"{desc} x {its} iterations (from iteration {it0}) of {config}: {paths} paths in {dt:.2f} s; "
                     f"oracle/lw_oracle.c (C restatement, OpenMP), {cpu_model()}",
           "mrays_per_s": rays / dt / 1e6}
    if gpu is not None:
        gpu.clear()
        gpu.render_pass(it0, it0 + its, p0, p1)
        fb_gpu = gpu.framebuffer()
        scale = 1.0 / (its * 1048576.0)
        diff = (fb_gpu[p0:p1].astype(np.float64) - fb_cpu[p0:p1].astype(np.float64)) * scale
        out["parity"] = {"bit_exact": bool(np.array_equal(fb_gpu, fb_cpu)), "rmse": float(np.sqrt((diff ** 2).mean())),
                         "mean_radiance": float(fb_cpu[p0:p1].astype(np.float64).mean() * scale),
                         "sample": "the cpu_baseline sample rendered on the GPU vs the CPU oracle (int64 framebuffers)"}
    return out


def _pool_map(fn, n, threads):
    """Run fn(lo, hi) over [0, n) split in `threads` contiguous slices on a thread pool (the
    reference kernels release the GIL: nogil loops, _kernels.py:220, 568)."""
    from concurrent.futures import ThreadPoolExecutor

    cuts = [n * k // threads for k in range(threads + 1)]
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda k: fn(cuts[k], cuts[k + 1]), range(threads)))


def reference_kernels_baseline(a, budget_s=6.0):
    """The reference's own compiled kernels (oracle/_ref, Cython from _kernels.py) on all host cores
    vs the GPU drop-ins on the identical batches: halton_batch over the first pass's sample indices
    and intersect_batch (corrected semantics) over the headline workload's camera rays against the
    reference-layout BVH.  Returns None when oracle/_ref is not built."""
    import numpy as np

    from oracle import oracle as O
    from paper_1705_01263_b200 import qmc
    from paper_1705_01263_b200.core import kernels
    from paper_1705_01263_b200.geometry import build_bvh
    from paper_1705_01263_b200.render import Renderer
    from paper_1705_01263_b200.scene import pack_scene

    ref = O.ref_kernels("corrected")
    if ref is None:
        return None
    threads = os.cpu_count()
    out = {"source": "oracle/_ref/corrected/_kernels*.so: the reference's _kernels.py compiled by oracle/Makefile "
                     "(Cython -> gcc -O2, D1/D2 fixes as the reference's tests specify)",
           "cpu_model": cpu_model(), "threads": threads}
    # halton_batch (_kernels.py:211-222): sample indices of the headline pass, dimension 0..3
    table = qmc.DimensionTable(a.depth)
    P = a.width * a.height
    n = 1 << 22
    idx = np.ascontiguousarray(np.arange(n, dtype=np.int64) + 3 * P)  # iteration 3 onwards, pixel order
    res_cpu = np.empty(n)
    res_gpu = np.empty(n)
    dims = 4
    t0 = time.perf_counter()
    reps = 0
    while True:
        for dim in range(dims):
            _pool_map(lambda lo, hi, dim=dim: ref.halton_batch(table.bases, table.perm_flat, table.perm_offset, dim,
                                                               idx[lo:hi], res_cpu[lo:hi]), n, threads)
        reps += 1
        if time.perf_counter() - t0 > budget_s / 3:
            break
    cpu_rate = reps * dims * n / (time.perf_counter() - t0)
    kernels.halton_batch(table.bases, table.perm_flat, table.perm_offset, 3, idx, res_gpu)  # warm
    t0 = time.perf_counter()
    for dim in range(dims):
        kernels.halton_batch(table.bases, table.perm_flat, table.perm_offset, dim, idx, res_gpu)
    gpu_rate = dims * n / (time.perf_counter() - t0)
    out["halton_batch"] = {"samples": n * dims, "cpu_samples_per_s": cpu_rate,
                           "gpu_samples_per_s_host_api": gpu_rate,
                           "bit_exact": bool(np.array_equal(res_cpu, res_gpu)),
                           "note": "GPU through the drop-in kernels.halton_batch with host numpy buffers (copies "
                                   "included); dim 3 compared"}
    # intersect_batch (_kernels.py:548-585): camera rays of the headline workload
    packed = pack_scene(build_scene(a.config))
    verts = packed.verts
    bounds, children, order = build_bvh(verts)
    inst = np.zeros(len(verts), np.int64)
    with Renderer(None, a.width, a.height, a.depth, packed=packed, pool_log2=10) as r:
        nr = 1 << 18
        o, d = r.camera_rays(np.arange(nr, dtype=np.int64) * 7 + 3 * P)
    tm = np.full(nr, np.inf)
    t_c, tri_c, b_c = np.empty(nr), np.empty(nr, np.int64), np.empty((nr, 2))
    done = 0
    t0 = time.perf_counter()
    chunk = 1 << 14
    while done < nr and time.perf_counter() - t0 < budget_s / 2:
        hi = min(nr, done + chunk)
        _pool_map(lambda lo2, hi2, base=done: ref.intersect_batch(
            bounds, children, order, verts, inst, o[base + lo2:base + hi2], d[base + lo2:base + hi2],
            tm[base + lo2:base + hi2], t_c[base + lo2:base + hi2], tri_c[base + lo2:base + hi2],
            b_c[base + lo2:base + hi2]), hi - done, threads)
        done = hi
    cpu_rate = done / (time.perf_counter() - t0)
    t_g, tri_g, b_g = np.empty(nr), np.empty(nr, np.int64), np.empty((nr, 2))
    kernels.intersect_batch(bounds, children, order, verts, inst, o, d, tm, t_g, tri_g, b_g)  # warm
    t0 = time.perf_counter()
    kernels.intersect_batch(bounds, children, order, verts, inst, o, d, tm, t_g, tri_g, b_g)
    gpu_rate = nr / (time.perf_counter() - t0)
    out["intersect_batch"] = {"rays": nr, "cpu_rays_timed": done, "cpu_mrays_per_s": cpu_rate / 1e6,
                              "gpu_mrays_per_s_host_api": gpu_rate / 1e6,
                              "bit_exact": bool(np.array_equal(t_c[:done], t_g[:done]) and
                                                np.array_equal(tri_c[:done], tri_g[:done]) and
                                                np.array_equal(b_c[:done], b_g[:done])),
                              "note": f"camera rays of {a.config} against the reference-layout median BVH "
                                      f"({len(bounds)} nodes, {len(verts)} triangles); GPU through the drop-in "
                                      "kernels.intersect_batch with host buffers (copies included)"}
    return out


def run_reference(a):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    vals = []
    for step in range(a.warmup + a.steps):
        r = cpu_render_sample(a, a.config, max(a.cpu_seconds / max(a.steps, 1), 1.0), it0=3 + step)
        if step >= a.warmup:
            vals.append(r)
    v = statistics.median([r["value"] for r in vals])
    base = vals[0]
    line = {"metric": metric_name(a), "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic procedural scene (seeded), QMC samples", "impl": "reference",
            "config": config_dict(a, a.gpus),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": base["cores"], "kind": "port",
                             "sample": base["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- our path -----------------------------------------------------------------------------

def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        return {"hbm_gbs": 6650.0, "fallback": True}


def load_kernel_traffic():
    """ncu DRAM bytes / duration per launch of every stage kernel, per config, at the bench's pool
    size (profiles/r02_kernel_traffic.json, tools/gpu_kernel_traffic.sh + tools/kernel_traffic_json.py)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "r02_kernel_traffic.json")))
    except OSError:
        return None


def load_ncu_stage():
    """ncu --set full summaries of the stage kernels (profiles/r02_ncu_stage_kernels.json, keys
    <config>_<stage>: C2 every stage, C3 / C5 trace_ext, C4 shade)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "r02_ncu_stage_kernels.json")))["kernels"]
    except (OSError, KeyError, ValueError):
        return {}


def limiter_of(n, smem_bvh_stage):
    """What bounds a stage kernel, read from its ncu summary: issue rate, dependent-load latency or
    fixed-latency arithmetic chains (profiles/README.md)."""
    if not n:
        return None
    stalls = n.get("top_stalls_per_issue") or {}
    top = max((k for k in stalls if k not in ("selected", "not_selected")), key=lambda k: stalls[k], default=None)
    issue = n.get("issue_active_pct", 0.0)
    if issue >= 65.0:
        kind = "instruction issue"
    elif top == "long_scoreboard":
        kind = "latency of dependent L1TEX/L2 loads"
    else:
        kind = "latency of FP64 dependency chains"
    text = (f"{kind}: {issue:.0f} % issue-active, {n.get('threads_per_warp_inst', 0):.1f} of 32 lanes per "
            f"instruction, {n.get('occupancy_pct', 0):.0f} % occupancy ({n.get('regs', 0):.0f} registers), top stall {top}")
    if smem_bvh_stage:
        text += "; BVH in shared memory, so the HBM bytes are the ray state only"
    return text


STAGE_KERNELS = {"generate": "k_generate", "trace_ext": "k_trace_ext_p", "shade_nee": "k_shade_nee",
                 "shade": "k_shade", "trace_shadow": "k_trace_shadow_p"}


def stage_bytes(prof, work, smem_bvh, nprev_bytes):
    """Algorithmic bytes of every wavefront stage over the passes summed in `prof`.

    State (HBM: the 2^24-slot pool, ~4.7 GB, never fits the 126 MB L2), per work item:
      generate      1 B stage tag per pool slot and wave; per path flushed 32 (radiance) + 4 (pixel)
                    + 48 (framebuffer read-modify-write); per path generated 121 (+4) (ray 48,
                    throughput/radiance 48, pdf+index 16, flags 4, pixel 4, stage 1 [, nprev 4]);
                    4 per extension-queue entry
      trace_ext     84 per extension ray (queue 4, ray 48, hit 32)
      shade_nee     120 per extension ray (queue 4, hit 32, flags 4, direction 32, throughput 32,
                    sample index 16) + 84 per shadow ray written (ray + contribution 80, queue 4)
      shade         269 (+8) per extension ray (read queue 4, ray 48, throughput 48, misc 16, flags 4,
                    hit 32 [, nprev 4]; write ray 48, throughput 48, misc 16, flags 4, stage 1 [, nprev 4])
      trace_shadow  68 per shadow ray (queue 4, ray + tmax 64) + 80 per unoccluded one (contribution
                    16, radiance read 32 + write 32)
    BVH node / triangle bytes of the trace kernels (128 per 4-wide node visit, 80 per triangle test,
    counted by the instrumented pass) are HBM/L2 bytes for global-memory BVHs and shared-memory bytes
    for the staged Cornell BVH (reported apart, not in the HBM numerator).
    Scene gathers of the shading kernels (hit triangle vertices + normals 144 B, material, light and
    environment records) are not counted: cache-resident for the Cornell box, data-dependent elsewhere.
    """
    E, S = prof["ext_rays"], prof["shadow_rays"]
    U = S * work["lit_frac"]
    paths, waves, pool = prof["paths"], prof["waves"], prof["pool_slots"]
    node_ext = (128.0 * work["ext_nodes_per_ray"] + 80.0 * work["ext_tris_per_ray"]) * E
    node_sh = (128.0 * work["sh_nodes_per_ray"] + 80.0 * work["sh_tris_per_ray"]) * S
    b = {
        "generate": waves * pool * 1.0 + paths * (32 + 4 + 48) + paths * (121 + nprev_bytes) + E * 4.0,
        "trace_ext": E * 84.0 + (0.0 if smem_bvh else node_ext),
        "shade_nee": E * 120.0 + S * 84.0,
        "shade": E * (269.0 + 2 * nprev_bytes),
        "trace_shadow": S * 68.0 + U * 80.0 + (0.0 if smem_bvh else node_sh),
    }
    smem = {"trace_ext": node_ext if smem_bvh else 0.0, "trace_shadow": node_sh if smem_bvh else 0.0}
    return b, smem


def roofline_block(a, config, prof, work, smem_bvh, nprev_bytes, peaks, traffic):
    """Per-stage-kernel roofline list and the dominant kernel's contract object."""
    peak = peaks.get("hbm_gbs", 6650.0)
    b, smem = stage_bytes(prof, work, smem_bvh, nprev_bytes)
    total_ms = prof["total_ms"]
    tcfg = ((traffic or {}).get("configs") or {}).get(config, {})
    ncu = load_ncu_stage()
    kernels = []
    for st, kname in STAGE_KERNELS.items():
        ms, n = prof["stage_ms"][st], max(prof["stage_launches"][st], 1)
        ach = b[st] / (ms / 1e3) / 1e9 if ms > 0 else 0.0
        t = tcfg.get(kname) or {}
        e = {"kernel": kname, "stage": st, "share_of_step": ms / total_ms if total_ms else None,
             "avg_launch_ms": ms / n, "launches": prof["stage_launches"][st],
             "algorithmic_bytes_per_launch": b[st] / n, "achieved_gbs": ach, "frac": ach / peak,
             "smem_bvh_bytes_per_launch": smem.get(st, 0.0) / n if smem.get(st) else 0.0,
             "ncu_dram_bytes_per_launch": t.get("dram_bytes_per_launch"),
             "ncu_duration_us_per_launch": t.get("duration_us_per_launch"),
             "ncu_dram_frac": (t["dram_bytes_per_launch"] / (t["duration_us_per_launch"] * 1e3) / peak)
             if t.get("duration_us_per_launch") else None,
             "limiter": limiter_of(ncu.get(f"{config}_{st}"), smem_bvh and st.startswith("trace"))}
        kernels.append(e)
    dom = max(kernels, key=lambda e: e["share_of_step"] or 0.0)
    return {"bound": "hbm", "achieved": dom["achieved_gbs"], "peak": peak, "unit": "GB/s", "frac": dom["frac"],
            "traffic": dom["ncu_dram_bytes_per_launch"], "kernel": dom["kernel"], "limiter": dom["limiter"],
            "avg_launch_ms": dom["avg_launch_ms"], "share_of_step": dom["share_of_step"],
            "algorithmic_bytes_per_launch": dom["algorithmic_bytes_per_launch"],
            "definition": "achieved = algorithmic bytes per launch (SoA state the stage must move, + BVH "
                          "node/triangle bytes for global-memory BVHs; bench.stage_bytes, DESIGN.md §6.3) / "
                          "CUDA-event launch time; frac vs MEASURED_PEAKS.json hbm_gbs; traffic = ncu "
                          "dram__bytes_read+write per launch at the bench pool size "
                          "(profiles/r02_kernel_traffic.json)",
            "peak_source": ("fallback 6650 GB/s (B200_PROFILING.md)" if peaks.get("fallback")
                            else "MEASURED_PEAKS.json hbm_gbs (measured copy)"),
            "kernels": kernels}


class Measure:
    """One workload on this rank's GPU: the renderer, the instrumented pass and the timed steps."""

    def __init__(self, a, config, rank, world, local, stream):
        from paper_1705_01263_b200.render import Renderer
        from paper_1705_01263_b200.scene import pack_scene

        self.a, self.config, self.rank, self.world = a, config, rank, world
        self.W, self.H, self.D, self.its = resolve(a, config)
        self.P = self.W * self.H
        self.packed = pack_scene(build_scene(config), lights=a.lights, env_sampling=a.env_sampling)
        self.r = Renderer(None, self.W, self.H, self.D, device=local, packed=self.packed, engine=a.engine,
                          pool_log2=a.pool_log2, regen_fraction=a.regen_fraction, megakernel_tail=a.megakernel_tail,
                          compact_state=a.state == "compact")
        self.r.set_stream(stream.cuda_stream)
        self.stream = stream
        self.local = local

    def comm(self):
        """Join the library's NCCL communicator (rank 0 creates the id; broadcast over torch)."""
        import torch
        import torch.distributed as dist

        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if self.rank == 0:
            uid.copy_(torch.frombuffer(bytearray(self.r.comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, src=0)
        self.r.comm_init(bytes(uid.cpu().numpy().tobytes()), self.rank, self.world)

    def step(self, s, glob):
        from paper_1705_01263_b200.distributed import partition_iterations

        lo, hi = partition_iterations(s * self.world * self.its, (s + 1) * self.world * self.its, self.rank, self.world)
        self.r.render_pass(lo, hi)
        if self.world > 1:
            self.r.reduce_framebuffer()  # NCCL all-reduce of the pass framebuffer, in place
        self.r.accumulate_into(glob.data_ptr(), clear=True)  # progressive image += pass; pass = 0

    def work(self, glob):
        """Untimed instrumented pass: traversal work per ray and the fraction of lit shadow rays."""
        self.r.set_instrumentation(count_work=True)
        self.step(10_000, glob)
        k = self.r.kernel_profile()
        self.r.set_instrumentation(time_kernels=True)
        er, sr = max(k["ext_rays"], 1), max(k["shadow_rays"], 1)
        return {"ext_nodes_per_ray": k["ext_nodes"] / er, "ext_tris_per_ray": k["ext_tris"] / er,
                "sh_nodes_per_ray": k["shadow_nodes"] / sr, "sh_tris_per_ray": k["shadow_tris"] / sr,
                "lit_frac": k["shadow_unoccluded"] / sr}

    def timed(self, steps, warmup, glob, clocks=None):
        import torch
        import torch.distributed as dist

        for s in range(warmup):
            self.step(s, glob)
        glob.zero_()
        acc = None
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if clocks:
            clocks.start()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        for s in range(warmup, warmup + steps):
            self.step(s, glob)
            kp = self.r.kernel_profile()
            if acc is None:
                acc = kp
            else:
                for k, v in kp.items():
                    if isinstance(v, dict):
                        for kk in v:
                            acc[k][kk] += v[kk]
                    elif k != "pool_slots":
                        acc[k] += v
        e1.record(self.stream)
        torch.cuda.synchronize()
        clk = clocks.stop() if clocks else None
        ms = e0.elapsed_time(e1)
        t = torch.tensor([ms, acc["ext_rays"], acc["shadow_rays"]], dtype=torch.float64, device="cuda")
        if self.world > 1:
            mx = t[:1].clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            sm = t[1:].clone()
            dist.all_reduce(sm)
            t = torch.cat([mx, sm])
        return float(t[0]), float(t[1]), float(t[2]), acc, clk

    def e2e(self, steps, tmp):
        """Same metric through the public API, scene in -> image out every step: create the context,
        upload the scene from pinned host buffers (GPU BVH builds run here), render this rank's pass,
        reduce (N > 1), read back the resolved float32 image into pinned memory."""
        import torch
        import torch.distributed as dist

        from paper_1705_01263_b200.distributed import partition_iterations
        from paper_1705_01263_b200.render import Renderer

        a = self.a
        pscene = self.packed.pinned()
        h2d = sum(v.nbytes for k, v in pscene.arrays.items() if hasattr(v, "nbytes"))
        h2d += C.sizeof(pscene.desc) + C.sizeof(self.r.params.struct) + self.r.params.bases.nbytes + \
            self.r.params.perm_flat.nbytes + self.r.params.perm_offset.nbytes
        d2h = self.P * 3 * 4
        img = torch.empty((self.H, self.W, 3), dtype=torch.float32, pin_memory=True).numpy()

        def one(s):
            with Renderer(None, self.W, self.H, self.D, device=self.local, packed=pscene, engine=a.engine,
                          pool_log2=a.pool_log2, regen_fraction=a.regen_fraction,
                          megakernel_tail=a.megakernel_tail, compact_state=a.state == "compact") as r2:
                r2.set_stream(self.stream.cuda_stream)
                lo, hi = partition_iterations(s * self.world * self.its, (s + 1) * self.world * self.its, self.rank,
                                              self.world)
                r2.render_pass(lo, hi)
                if self.world > 1:
                    r2.copy_framebuffer_to(tmp.data_ptr())
                    dist.all_reduce(tmp)
                    r2.load_framebuffer_from(tmp.data_ptr())
                r2.image(self.world * self.its, out=img)

        one(0)  # untimed warm-up (first use of the device memory pool at this scene's sizes)
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(steps):
            one(s)
        torch.cuda.synchronize()
        tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if self.world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        paths = steps * self.world * self.its * self.P
        return {"value": paths / float(tt[0]), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "note": "per step: context + scene upload from pinned host buffers (GPU SAH build + 4-wide "
                        "collapse) + pass + framebuffer all-reduce (N>1) + resolved float32 image readback into "
                        "pinned memory, host wall clock around device syncs"}

    def parity_sample(self, it0=5, rows=8):
        """GPU vs the CPU oracle on `rows` centre rows x 1 iteration of this workload (bit for bit)."""
        import numpy as np

        from oracle import oracle as O

        r0 = max(0, self.H // 2 - rows // 2)
        p0, p1 = r0 * self.W, min(self.H, r0 + rows) * self.W
        self.r.clear()
        self.r.render_pass(it0, it0 + 1, p0, p1)
        fb = self.r.framebuffer()
        self.r.clear()
        fb2, _ = O.OracleScene(self.packed).render(self.r.params, it0, it0 + 1, p0, p1)
        d = (fb[p0:p1].astype(np.float64) - fb2[p0:p1].astype(np.float64)) / 1048576.0
        return {"bit_exact": bool(np.array_equal(fb, fb2)), "rmse": float(np.sqrt((d ** 2).mean())),
                "sample": f"{p1 // self.W - r0} centre rows x 1 iteration vs oracle/lw_oracle.c"}

    def close(self):
        self.r.close()


def self_launch(a):
    """`--gpus N` without a torchrun environment: start N ranks (one per GPU) with
    torch.distributed.run on this node and relay rank 0's JSON line."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def run_ours(a):
    import torch
    import torch.distributed as dist

    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))
    if world != a.gpus:
        raise SystemExit(f"bench: WORLD_SIZE={world} but --gpus {a.gpus}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    m = Measure(a, a.config, rank, world, local, stream)
    if world > 1:
        m.comm()
    glob = torch.zeros((m.P, 3), dtype=torch.int64, device="cuda")
    tmp = torch.empty_like(glob)
    work = m.work(glob)
    clocks = ClockSampler(local)
    ms_max, rays_ext_all, rays_sh_all, prof, clk = m.timed(a.steps, a.warmup, glob, clocks)
    paths = a.steps * world * m.its * m.P
    value = paths / (ms_max / 1e3)
    e2e = None if a.no_e2e else m.e2e(a.steps, tmp)
    peaks = load_peaks()
    nprev = 4 if (a.lights == "tree" or a.env_sampling == "pyramid") else 0
    smem_bvh = m.packed.ntris <= 4096  # staged in shared memory (lw_scene_upload's placement rule)
    traffic = load_kernel_traffic()
    if a.engine == "wavefront":
        roof = roofline_block(a, a.config, prof, work, smem_bvh, nprev, peaks, traffic)
    else:  # megakernel: one launch per pass; HBM bytes are the framebuffer + BVH fetches
        roof = {"bound": "hbm", "achieved": None, "peak": peaks.get("hbm_gbs"), "unit": "GB/s", "frac": None,
                "traffic": None, "kernel": "k_megakernel (whole path per thread; no SoA state)"}
    line = {
        "metric": metric_name(a), "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms_max / a.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic procedural scene (seeded), QMC samples",
        "config": config_dict(a, world),
        "mrays_per_s": (rays_ext_all + rays_sh_all) / (ms_max / 1e3) / 1e6,
        "gsegments_per_s": rays_ext_all / (ms_max / 1e3) / 1e9,
        "gpu_launches": int(prof["kernel_launches"] + a.steps),  # + one accumulate kernel per step
        "clocks": clk,
        "roofline": roof,
        "traversal_work": work,
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cb = cpu_render_sample(a, a.config, a.cpu_seconds, gpu=m.r)
        line["parity_vs_cpu_reference"] = cb.pop("parity")
        line["cpu_baseline"] = {k: v for k, v in cb.items() if k != "mrays_per_s"}
        line["cpu_baseline"]["mrays_per_s"] = cb["mrays_per_s"]
        try:
            rk = reference_kernels_baseline(a)
        except Exception as e:  # noqa: BLE001  (reported, never fatal for the headline)
            rk = {"error": repr(e)}
        line["cpu_baseline"]["reference_kernels"] = rk if rk is not None else \
            {"unavailable": "oracle/_ref not built on this box (make -C oracle ref needs /root/reference)"}
    m.close()
    if rank == 0 and world == 1 and not a.no_per_config:
        line["per_config"] = per_config(a, stream, line)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def per_config(a, stream, head):
    """C1-C5 (BASELINE.json configs) measured in this run on this GPU: device-timed paths/s,
    Gsegments/s, Mrays/s, e2e, dominant kernel and its share, trace share, bit-exact parity sample."""
    import torch

    out = {}
    for cfg in CONFIGS:
        t0 = time.perf_counter()
        try:
            m = Measure(a, cfg, 0, 1, 0, stream)
            glob = torch.zeros((m.P, 3), dtype=torch.int64, device="cuda")
            tmp = torch.empty_like(glob)
            work = m.work(glob)
            ms, re, rs, prof, _ = m.timed(3, 2, glob)
            paths = 3 * m.its * m.P
            smem_bvh = m.packed.ntris <= 4096
            roof = roofline_block(a, cfg, prof, work, smem_bvh, 0, load_peaks(), load_kernel_traffic())
            e2e = m.e2e(2, tmp) if not a.no_e2e else None
            rec = {"workload": workload(a, cfg), "value": paths / (ms / 1e3), "unit": UNIT,
                   "gsegments_per_s": re / (ms / 1e3) / 1e9, "mrays_per_s": (re + rs) / (ms / 1e3) / 1e6,
                   "ms_per_step": ms / 3, "e2e": e2e["value"] if e2e else None,
                   "trace_share": (prof["stage_ms"]["trace_ext"] + prof["stage_ms"]["trace_shadow"]) / prof["total_ms"],
                   "dominant_kernel": roof["kernel"], "dominant_share": roof["share_of_step"],
                   "dominant_frac": roof["frac"],
                   "stage_share": {k: v / prof["total_ms"] for k, v in prof["stage_ms"].items()},
                   "parity": m.parity_sample(), "seconds": None}
            m.close()
            del glob, tmp
        except Exception as e:  # noqa: BLE001  (one config failing must not lose the headline)
            rec = {"error": repr(e)}
        rec["seconds"] = time.perf_counter() - t0
        out[cfg] = rec
    return out


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return 0
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(a)
    run_ours(a)
    return 0


if __name__ == "__main__":
    sys.exit(main())
