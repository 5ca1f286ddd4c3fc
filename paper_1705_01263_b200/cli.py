"""Thin `render` command (the reference declares `lumenwave = "lumenwave.cli:main"`,
pyproject.toml:12-13, with the flags of SPEC.md:800 but ships no cli module).

    python -m paper_1705_01263_b200.cli render --config C1 --out img [--res WxH] [--iterations N]
        [--depth D] [--snapshot-every N] [--engine wavefront|megakernel] [--metrics FILE] [--device K]
        [--lights alias|tree] [--env-sampling alias|pyramid]
        [--devices N [--contexts-per-device C] [--fail DEV@ITER ...]]   # batch scheduler
        [--layer NAME=EXPR ...]                                          # LPE output layers
        [--checkpoint state.npz] [--resume state.npz]                    # progressive state
    python -m paper_1705_01263_b200.cli composite --layers a.pfm b.pfm --gains 1 2 --out c.pfm

Scenes come from the procedural configs (the text-format parser is out of scope);
`--scene FILE.py` may name a Python file defining `scene()` that returns a Scene (e.g. one built
with the reference's `load_scene`).  Outputs are numbered PFM snapshots (`--out` prefix), the
bit-exact interchange format of SPEC.md DESIGN DECISIONS.  Exit codes per SPEC.md: 0 success,
2 input error, 3 config error, 4 internal error.
"""

from __future__ import annotations

import argparse
import json
import runpy
import sys
import time


def _parse_res(text):
    w, h = text.lower().split("x")
    w, h = int(w), int(h)
    if w <= 0 or h <= 0:
        raise ValueError
    return w, h


def cmd_render(args) -> int:
    from paper_1705_01263_b200 import scenes
    from paper_1705_01263_b200.imagefiles import write_pfm
    from paper_1705_01263_b200.render import Renderer

    cfg = scenes.CONFIGS.get(args.config)
    if args.scene:
        try:
            scene = runpy.run_path(args.scene)["scene"]()
        except (OSError, KeyError) as e:
            print(f"error: cannot load scene '{args.scene}': {e}", file=sys.stderr)
            return 2
    elif cfg is not None:
        scene = cfg.builder()
    else:
        print(f"error: unknown config '{args.config}'", file=sys.stderr)
        return 3
    try:
        w, h = _parse_res(args.res) if args.res else (cfg.width, cfg.height)
    except ValueError:
        print(f"error: bad --res '{args.res}' (expected WxH)", file=sys.stderr)
        return 3
    spp = args.iterations or (cfg.spp if cfg else 16)
    depth = args.depth or (cfg.max_depth if cfg else 8)
    if spp < 1:
        print("error: --iterations must be >= 1", file=sys.stderr)
        return 3
    from paper_1705_01263_b200.scene import pack_scene

    packed = pack_scene(scene, lights=args.lights, env_sampling=args.env_sampling)
    if args.devices > 1 or args.fail or args.contexts_per_device > 1:
        return _render_batch(args, packed, w, h, depth, spp)
    layers = {}
    for spec in args.layer or []:
        name, _, expr = spec.partition("=")
        if not name or not expr:
            print(f"error: bad --layer '{spec}' (expected NAME=EXPR)", file=sys.stderr)
            return 3
        layers[name] = expr
    engine = args.engine
    step = args.snapshot_every or spp
    t0 = time.perf_counter()
    with Renderer(None, w, h, depth, device=args.device, engine=engine, packed=packed) as r:
        if layers:
            from paper_1705_01263_b200.lpe import LpeError

            try:
                r.set_lpe_layers(layers)
            except LpeError as e:
                print(f"error: --layer: {e}", file=sys.stderr)
                return 2
        done0 = 0
        if args.resume:
            try:
                r.load_checkpoint(args.resume)
            except (OSError, ValueError, KeyError) as e:
                print(f"error: cannot resume from '{args.resume}': {e}", file=sys.stderr)
                return 2
            done0 = r.iterations
        done = done0
        while done < spp:
            k = min(step, spp - done)
            r.render_pass(done, done + k)
            done += k
            write_pfm(f"{args.out}_{done:06d}.pfm", r.image(done))
            if args.checkpoint:
                r.save_checkpoint(args.checkpoint)
            for name, img in (r.layer_images(done).items() if layers else []):
                write_pfm(f"{args.out}_{name}_{done:06d}.pfm", img)
        stats = r.stats()
    dt = time.perf_counter() - t0
    if args.metrics:
        stats.update({"seconds": dt, "paths_per_s": stats["paths"] / dt, "width": w, "height": h, "iterations": spp})
        with open(args.metrics, "w") as f:
            json.dump(stats, f, indent=1)
    return 0


def _render_batch(args, packed, w, h, depth, spp) -> int:
    """Batch mode: dynamic iteration sets over all device contexts, throttled
    merges, `--fail DEV@ITER` failure injection; one final snapshot."""
    import numpy as np

    from paper_1705_01263_b200.imagefiles import write_pfm
    from paper_1705_01263_b200.render import Renderer
    from paper_1705_01263_b200.scheduler import BatchScheduler, SchedulerError, WorkerProfile

    slots = [d for d in range(max(args.devices, 1)) for _ in range(max(args.contexts_per_device, 1))]
    fails = {}
    for f in args.fail or []:
        try:
            dev, it = f.split("@")
            fails[int(dev)] = int(it)
        except ValueError:
            print(f"error: bad --fail '{f}' (expected DEV@ITER)", file=sys.stderr)
            return 3
    profiles = [WorkerProfile(k, fail_after=fails.get(k)) for k in range(len(slots))]
    t0 = time.perf_counter()
    sch = BatchScheduler(lambda k: Renderer(None, w, h, depth, device=slots[k], engine=args.engine, packed=packed),
                         profiles)
    try:
        fb = sch.run(0, spp)
    except SchedulerError as e:
        print(f"error: {e}", file=sys.stderr)
        return 4
    img = (fb.astype(np.float64) * (1.0 / (1048576.0 * spp))).astype(np.float32).reshape(h, w, 3)
    write_pfm(f"{args.out}_{spp:06d}.pfm", img)
    dt = time.perf_counter() - t0
    if args.metrics:
        m = sch.ledger.metrics()
        m.update({"seconds": dt, "paths_per_s": w * h * spp / dt, "width": w, "height": h, "iterations": spp})
        with open(args.metrics, "w") as f:
            json.dump(m, f, indent=1, default=str)
    return 0


def cmd_composite(args) -> int:
    """Linear recombination of layer PFMs: out = sum gain_k * layer_k."""
    from paper_1705_01263_b200.imagefiles import read_pfm, write_pfm
    from paper_1705_01263_b200.lpe import composite

    gains = args.gains or [1.0] * len(args.layers)
    if len(gains) != len(args.layers):
        print("error: one gain per layer", file=sys.stderr)
        return 3
    try:
        imgs = {k: read_pfm(p) for k, p in enumerate(args.layers)}
    except (OSError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    if len({im.shape for im in imgs.values()}) != 1:
        print("error: layer resolutions differ", file=sys.stderr)
        return 2
    write_pfm(args.out, composite(imgs, dict(enumerate(gains))).astype("float32"))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_1705_01263_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    rp = sub.add_parser("render", help="progressive render to numbered PFM snapshots")
    rp.add_argument("--config", default="C1")
    rp.add_argument("--scene", default=None, help="Python file defining scene() -> Scene")
    rp.add_argument("--res", default=None)
    rp.add_argument("--iterations", type=int, default=0)
    rp.add_argument("--depth", type=int, default=0)
    rp.add_argument("--snapshot-every", type=int, default=0)
    rp.add_argument("--engine", default="wavefront", choices=["wavefront", "megakernel"])
    rp.add_argument("--device", type=int, default=0)
    rp.add_argument("--out", default="render")
    rp.add_argument("--metrics", default=None)
    rp.add_argument("--lights", default="alias", choices=["alias", "tree"])
    rp.add_argument("--env-sampling", default="alias", choices=["alias", "pyramid"])
    rp.add_argument("--devices", type=int, default=1, help="batch scheduler over GPUs 0..N-1")
    rp.add_argument("--contexts-per-device", type=int, default=1, help="simulated devices per GPU")
    rp.add_argument("--fail", action="append", default=None, help="inject a failure: DEV@ITER (SPEC.md:800)")
    rp.add_argument("--checkpoint", default=None, help="save the progressive state (.npz) after every snapshot")
    rp.add_argument("--resume", default=None, help="continue from a checkpoint written by --checkpoint")
    rp.add_argument("--layer", action="append", default=None,
                    help="light-path-expression output layer NAME=EXPR (lpe.py syntax), repeatable")
    cp = sub.add_parser("composite", help="sum of gain * layer PFMs")
    cp.add_argument("--layers", nargs="+", required=True)
    cp.add_argument("--gains", nargs="+", type=float, default=None)
    cp.add_argument("--out", required=True)
    args = ap.parse_args(argv)
    try:
        return cmd_composite(args) if args.cmd == "composite" else cmd_render(args)
    except (ValueError, NotImplementedError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    except Exception as e:  # surfaced as the SPEC's internal-error code
        print(f"internal error: {e}", file=sys.stderr)
        return 4


if __name__ == "__main__":
    sys.exit(main())
