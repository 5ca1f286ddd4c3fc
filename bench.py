#!/usr/bin/env python
"""Headline benchmark: progressive path tracing of C2 (Cornell box 1024x1024, depth 8) in paths/s.

    python bench.py [--gpus N --steps K --warmup W]            # our B200 path (torchrun for N > 1)
    python bench.py --impl reference [--steps K --warmup W]     # the CPU path on the host cores

A step is one progressive pass of `--pass-iterations` (default 16) QMC iterations per GPU over all
1024x1024 pixels (weak scaling: every rank renders its own disjoint iteration block of the global
pass), followed by the per-pass int64 framebuffer sum-reduction (NCCL all_reduce when N > 1).
`value` is whole-job paths/s (device-timed, max over ranks); `e2e` is the same metric through the
public Python API with the scene uploaded from host buffers and the resolved image read back every
step.  The reference package has no renderer, so the CPU path is the oracle's C
restatement of the render (oracle/lw_oracle.c, OpenMP over all host threads): "kind": "port".
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "paths/s"


def metric_name(a):
    return f"paths/sec (samples/sec) on {a.config} {a.width}x{a.height} depth {a.depth}"


def build_scene(a):
    from paper_1705_01263_b200 import scenes

    return scenes.CONFIGS[a.config].builder()


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
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
    a = ap.parse_args()
    from paper_1705_01263_b200 import scenes

    c = scenes.CONFIGS[a.config]
    a.width = a.width or c.width
    a.height = a.height or c.height
    a.depth = a.depth or c.max_depth
    a.pass_iterations = a.pass_iterations or max(1, (1 << 24) // (a.width * a.height))
    return a


def workload(a):
    from paper_1705_01263_b200 import scenes

    return (f"{a.config}: {scenes.CONFIGS[a.config].description}; {a.width}x{a.height}, depth {a.depth}, "
            f"{a.pass_iterations} spp per GPU per step")


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


# ---- CPU path (oracle restatement) ----------------------------------------------------------

def cpu_render_sample(a, budget_s, threads=0, it0=3, gpu=None):
    """Bounded sample of the same workload on the host cores (oracle/lw_oracle.c, OpenMP):
    full-frame iterations (or a band of rows when one frame exceeds the budget).  With `gpu` (the
    bench's Renderer) the same sample is rendered on the GPU and compared with the CPU framebuffer
    (the "RMSE vs ref" half of the metric)."""
    from oracle import oracle as O
    from paper_1705_01263_b200.render import RenderParams
    from paper_1705_01263_b200.scene import pack_scene

    packed = pack_scene(build_scene(a), lights=a.lights, env_sampling=a.env_sampling)
    osc = O.OracleScene(packed)
    params = RenderParams(a.width, a.height, a.depth)
    threads = threads or os.cpu_count()
    rows = min(16, a.height)
    t0 = time.perf_counter()
    osc.render(params, it0, it0 + 1, 0, rows * a.width, nthreads=threads)
    per_row = (time.perf_counter() - t0) / rows
    frame = per_row * a.height
    if frame <= budget_s:
        rows, its = a.height, max(1, int(budget_s / max(frame, 1e-9)))
    else:
        rows, its = max(1, int(budget_s / max(per_row, 1e-9))), 1
    t0 = time.perf_counter()
    fb_cpu, st = osc.render(params, it0, it0 + its, 0, rows * a.width, nthreads=threads)
    dt = time.perf_counter() - t0
    out = {"value": st["paths"] / dt, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"{rows} rows x {a.width} px x {its} iterations (from iteration {it0}) of the workload: "
                     f"{st['paths']} paths in {dt:.2f} s; oracle/lw_oracle.c (C restatement, OpenMP)",
           "mrays_per_s": (st["rays_extension"] + st["rays_shadow"]) / dt / 1e6}
    if gpu is not None:
        import numpy as np

        gpu.clear()
        gpu.render_pass(it0, it0 + its, 0, rows * a.width)
        fb_gpu = gpu.framebuffer()
        scale = 1.0 / (its * 1048576.0)
        diff = (fb_gpu[: rows * a.width].astype(np.float64) - fb_cpu[: rows * a.width].astype(np.float64)) * scale
        out["parity"] = {"bit_exact": bool(np.array_equal(fb_gpu, fb_cpu)), "rmse": float(np.sqrt((diff ** 2).mean())),
                         "mean_radiance": float(fb_cpu[: rows * a.width].astype(np.float64).mean() * scale),
                         "sample": "the cpu_baseline sample rendered on the GPU vs the CPU oracle (int64 framebuffers)"}
    return out


def run_reference(a):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    vals = []
    for step in range(a.warmup + a.steps):
        r = cpu_render_sample(a, max(a.cpu_seconds / max(a.steps, 1), 1.0), it0=3 + step)
        if step >= a.warmup:
            vals.append(r)
    v = statistics.median([r["value"] for r in vals])
    base = vals[0]
    line = {"metric": metric_name(a), "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic procedural scene (seeded)", "impl": "reference",
            "config": {"workload": workload(a), "parallelism": "host threads (OpenMP)"},
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


def load_stage_profile(config):
    """ncu --set full summary of this config's k_trace_ext (profiles/r01_ncu_stage_kernels.json)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r01_ncu_stage_kernels.json")))
    except OSError:
        return None
    k = (d.get("kernels") or {}).get(f"{config}_trace_ext")
    if not k:
        return None
    return {"l1tex_throughput_pct": k.get("l1tex_throughput_pct"), "issue_active_pct": k.get("issue_active_pct"),
            "dram_throughput_gbs": round((k["dram_read_bytes"] + k["dram_write_bytes"]) / k["duration_us"] / 1e3, 1),
            "threads_per_warp_inst": k.get("threads_per_warp_inst"),
            "note": "measured limiter of this kernel: latency and SIMT efficiency (long-scoreboard stalls on node "
                    "fetches, threads_per_warp_inst of 32 lanes active; L1TEX at l1tex_throughput_pct), not HBM; "
                    "source profiles/r01_ncu_stage_kernels.json"}


def load_traffic():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "trace_ext_traffic.json")))
    except OSError:
        return None


def run_ours(a):
    import torch
    import torch.distributed as dist

    from paper_1705_01263_b200.distributed import partition_iterations
    from paper_1705_01263_b200.render import Renderer
    from paper_1705_01263_b200.scene import pack_scene

    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    packed = pack_scene(build_scene(a), lights=a.lights, env_sampling=a.env_sampling)
    W, H, P = a.width, a.height, a.width * a.height
    its = a.pass_iterations
    r = Renderer(None, W, H, a.depth, device=local, packed=packed, engine=a.engine, pool_log2=a.pool_log2,
                 regen_fraction=a.regen_fraction, megakernel_tail=a.megakernel_tail)
    r.set_stream(stream.cuda_stream)
    glob = torch.zeros((P, 3), dtype=torch.int64, device="cuda")
    tmp = torch.empty_like(glob)

    def step(s):
        # global pass s covers iterations [s*world*its, (s+1)*world*its); this rank takes its block
        lo, hi = partition_iterations(s * world * its, (s + 1) * world * its, rank, world)
        r.render_pass(lo, hi)
        r.copy_framebuffer_to(tmp.data_ptr())
        if world > 1:
            dist.all_reduce(tmp)
        glob.add_(tmp)
        r.clear()

    # untimed instrumented pass: traversal work per ray (node fetches, triangle tests)
    r.set_instrumentation(count_work=True)
    step(10_000)
    work = r.kernel_profile()
    r.set_instrumentation(time_kernels=True)
    for s in range(a.warmup):
        step(s)
    glob.zero_()
    clocks = ClockSampler(local)
    rays_ext = rays_sh = launches = 0
    prof_ms = 0.0
    prof_launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(a.warmup, a.warmup + a.steps):
        step(s)
        kp = r.kernel_profile()
        rays_ext += kp["ext_rays"]
        rays_sh += kp["shadow_rays"]
        launches += kp["kernel_launches"]
        prof_ms += kp["trace_ext_ms"]
        prof_launches += kp["trace_ext_launches"]
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms, rays_ext, rays_sh], dtype=torch.float64, device="cuda")
    if world > 1:
        mx = t[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t[1:].clone()
        dist.all_reduce(sm)
        t = torch.cat([mx, sm])
    ms_max, rays_ext_all, rays_sh_all = float(t[0]), float(t[1]), float(t[2])
    paths = a.steps * world * its * P
    value = paths / (ms_max / 1e3)

    # e2e through the public API, scene in -> image out every step: create the context, upload the
    # scene from host buffers (GPU BVH builds run here), render this rank's pass, reduce, read back
    # the resolved float32 image
    e2e = None
    if not a.no_e2e:
        pscene = packed.pinned()  # step inputs in page-locked host memory
        h2d = sum(v.nbytes for k, v in pscene.arrays.items() if hasattr(v, "nbytes"))
        h2d += C.sizeof(pscene.desc) + C.sizeof(r.params.struct) + r.params.bases.nbytes + \
            r.params.perm_flat.nbytes + r.params.perm_offset.nbytes
        d2h = P * 3 * 4
        img = torch.empty((H, W, 3), dtype=torch.float32, pin_memory=True).numpy()

        def e2e_step(s):
            with Renderer(None, W, H, a.depth, device=local, packed=pscene, engine=a.engine, pool_log2=a.pool_log2,
                          regen_fraction=a.regen_fraction, megakernel_tail=a.megakernel_tail) as r2:
                r2.set_stream(stream.cuda_stream)
                lo, hi = partition_iterations(s * world * its, (s + 1) * world * its, rank, world)
                r2.render_pass(lo, hi)
                if world > 1:
                    r2.copy_framebuffer_to(tmp.data_ptr())
                    dist.all_reduce(tmp)
                    r2.load_framebuffer_from(tmp.data_ptr())
                r2.image(world * its, out=img)

        e2e_step(0)  # untimed warm-up (first use of the device memory pool at this scene's sizes)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(a.steps):
            e2e_step(s)
        torch.cuda.synchronize()
        tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": paths / float(tt[0]), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "note": "per step: context + scene upload from pinned host buffers (GPU SAH build + 4-wide "
                       "collapse) + pass + NCCL reduce (N>1) + resolved float32 image readback into pinned "
                       "memory, host wall clock around device syncs"}

    peaks = load_peaks()
    nodes_per_ray = work["ext_nodes"] / max(work["ext_rays"], 1)
    tris_per_ray = work["ext_tris"] / max(work["ext_rays"], 1)
    # algorithmic bytes per extension ray: one 128-byte node per node visit, one 80-byte
    # triangle record per test, plus the SoA ray read (48 B), queue index (4 B) and hit write (28 B)
    bytes_per_ray = 128.0 * nodes_per_ray + 80.0 * tris_per_ray + 80.0
    if prof_launches > 0:  # wavefront: the extension-ray trace kernel, timed per launch with CUDA events
        kernel = "k_trace_ext_p (persistent closest-hit traversal, wavefront stage)"
        avg_ms = prof_ms / prof_launches
        achieved = bytes_per_ray * rays_ext / prof_ms / 1e6  # GB/s
    else:  # megakernel: the whole pass is one launch; count extension + shadow traversal bytes
        kernel = "k_megakernel (trace + shade + shadow)"
        sh_bytes = (128.0 * work["shadow_nodes"] + 80.0 * work["shadow_tris"]) / max(work["shadow_rays"], 1)
        avg_ms = ms_max / a.steps
        achieved = (bytes_per_ray * rays_ext + sh_bytes * rays_sh) / ms_max / 1e6
        prof_ms, prof_launches = ms_max, a.steps
    traffic = load_traffic()
    line = {
        "metric": metric_name(a), "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms_max / a.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic procedural scene (seeded), QMC samples",
        "config": {"workload": workload(a), "engine": a.engine, "lights": a.lights, "env_sampling": a.env_sampling, "pool_slots": 1 << a.pool_log2,
                   "regen_fraction": a.regen_fraction, "parallelism": f"sample-space dp{world}",
                   "l2": f"wavefront state pool (~{(1 << a.pool_log2) * 250 / 1e9:.1f} GB) exceeds the 126 MB L2 "
                         "(no flush needed); Cornell-box BVHs are shared-memory resident by design"},
        "mrays_per_s": (rays_ext_all + rays_sh_all) / (ms_max / 1e3) / 1e6,
        "gsegments_per_s": rays_ext_all / (ms_max / 1e3) / 1e9,
        "gpu_launches": int(launches),
        "clocks": clk,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                     "frac": achieved / peaks.get("hbm_gbs", 6650.0), "kernel": kernel,
                     "bytes_per_ray": bytes_per_ray, "nodes_per_ray": nodes_per_ray, "tris_per_ray": tris_per_ray,
                     "avg_launch_ms": avg_ms, "launches": prof_launches,
                     "trace_share_of_step": prof_ms / ms_max,
                     "traffic": ((traffic or {}).get("configs", {}).get(a.config) or {}).get("dram_bytes_per_launch"),
                     "traffic_source": "profiles/trace_ext_traffic.json (ncu dram__bytes_read+write per launch)",
                     "ncu": load_stage_profile(a.config),
                     "peak_source": ("fallback 6650 GB/s (B200_PROFILING.md)" if peaks.get("fallback")
                                     else "MEASURED_PEAKS.json hbm_gbs (measured copy)")},
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cb = cpu_render_sample(a, a.cpu_seconds, gpu=r)
        line["parity_vs_cpu_reference"] = cb.pop("parity")
        line["cpu_baseline"] = {k: v for k, v in cb.items() if k != "mrays_per_s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    r.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
