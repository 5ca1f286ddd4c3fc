"""Batch-mode multi-device scheduler.

Iteration sets are assigned dynamically to devices that each accumulate into a local copy of the
full framebuffer; local progress is merged into the master framebuffer only periodically, and a
device skips a merge while a peer is merging if it holds less than half as many unmerged
iterations as any other device.  A failed device's unmerged iterations are lost
and handed out again exactly once.  Because a sample is a pure function of (pixel, iteration)
(QMC, qmc.py:185-196) and framebuffers are int64 fixed point, the final image is bit-identical for
any device count, set sizes, merge timing and failure schedule.

The cluster is simulated in-process: one host thread per device, each owning a
render context (`Renderer`, or any object with render_pass / framebuffer / clear); the ledger is a
single-writer state machine behind a lock.  Interactive stripe scheduling is out of scope
(SURVEY.md §2).
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field

import numpy as np


class SchedulerError(RuntimeError):
    pass


@dataclass
class WorkerProfile:
    """id, relative performance weight (startup estimate, then refined), alive."""

    worker: int
    weight: float = 1.0
    alive: bool = True
    speed: float = 1.0          # simulation knob: artificial slowdown factor (1 = none)
    fail_after: int | None = None  # simulation knob: fail once this many iterations were rendered

    def __post_init__(self):
        if not self.weight > 0:
            raise ValueError("worker weights must be > 0")


@dataclass
class DeviceState:
    rendered: int = 0           # iterations rendered by this device (merged or not)
    unmerged: list = field(default_factory=list)  # iteration ids in the local framebuffer
    merges: int = 0
    skips: int = 0
    sets: int = 0
    busy_s: float = 0.0
    rate: float = 0.0           # observed iterations / s (0 = unknown, use the weight)
    merging: bool = False


class IterationLedger:
    """per-device assigned sets and unmerged iterations, merged bookkeeping.

    Invariants: every iteration is assigned at most once unless its assignee failed; merged
    iterations are never double counted; assigned = merged + lost + in flight."""

    def __init__(self, it_begin: int, it_end: int, profiles: list[WorkerProfile], cap: int = 64):
        if it_end < it_begin:
            raise ValueError("empty or negative iteration range")
        if not profiles:
            raise ValueError("at least one worker required")
        self.it_begin, self.it_end, self.cap = int(it_begin), int(it_end), int(cap)
        self.next = int(it_begin)
        self.requeue: list[int] = []     # lost iterations, handed out again first
        self.profiles = {p.worker: p for p in profiles}
        self.dev = {p.worker: DeviceState() for p in profiles}
        self.merged: set[int] = set()
        self.lost = 0
        self.assigned = 0
        self.t0 = time.perf_counter()
        self.lock = threading.Lock()

    # -- queries
    def remaining(self) -> int:
        return (self.it_end - self.next) + len(self.requeue)

    def done(self) -> bool:
        return len(self.merged) == self.it_end - self.it_begin

    def alive(self) -> list[int]:
        return [w for w, p in self.profiles.items() if p.alive]

    def _rate(self, w: int) -> float:
        d = self.dev[w]
        if d.rate > 0:
            return d.rate
        tot_w = sum(self.profiles[a].weight for a in self.alive())
        known = [self.dev[a].rate for a in self.alive() if self.dev[a].rate > 0]
        scale = (sum(known) / max(1, len(known))) if known else 1.0
        return self.profiles[w].weight / tot_w * scale * len(self.alive())

    def remaining_time(self) -> float:
        """Remaining iterations / aggregate observed rate."""
        agg = sum(self._rate(w) for w in self.alive())
        return self.remaining() / agg if agg > 0 else float("inf")

    # -- operations
    def assign_iteration_set(self, w: int) -> list[int]:
        """Set size = clamp(rate * remaining_time / 2, 1, cap)."""
        with self.lock:
            if not self.profiles[w].alive:
                raise SchedulerError(f"device {w} is not alive")
            rem = self.remaining()
            if rem == 0:
                return []
            size = int(self._rate(w) * self.remaining_time() / 2.0)
            size = max(1, min(self.cap, size, rem))
            out = []
            while self.requeue and len(out) < size:
                out.append(self.requeue.pop(0))
            take = min(size - len(out), self.it_end - self.next)
            out.extend(range(self.next, self.next + take))
            self.next += take
            self.assigned += len(out)
            self.dev[w].sets += 1
            return out

    def should_merge(self, w: int) -> bool:
        """Skip while a peer is merging if this device holds less than half as many unmerged
        iterations as any other device."""
        with self.lock:
            mine = len(self.dev[w].unmerged)
            if mine == 0:
                return False
            peers = [a for a in self.alive() if a != w]
            if any(self.dev[a].merging for a in peers):
                if any(mine < 0.5 * len(self.dev[a].unmerged) for a in peers):
                    self.dev[w].skips += 1
                    return False
            return True

    def rendered(self, w: int, its: list[int], seconds: float):
        with self.lock:
            d = self.dev[w]
            d.rendered += len(its)
            d.unmerged.extend(its)
            d.busy_s += seconds
            d.rate = d.rendered / d.busy_s if d.busy_s > 0 else 0.0

    def begin_merge(self, w: int) -> list[int]:
        with self.lock:
            self.dev[w].merging = True
            return list(self.dev[w].unmerged)

    def end_merge(self, w: int, its: list[int]):
        with self.lock:
            dup = self.merged.intersection(its)
            if dup:
                raise SchedulerError(f"double merge of iterations {sorted(dup)[:8]}")
            self.merged.update(its)
            d = self.dev[w]
            done = set(its)
            d.unmerged = [i for i in d.unmerged if i not in done]
            d.merges += 1
            d.merging = False

    def fail(self, w: int, in_flight: list[int] | None = None) -> list[int]:
        """Device failure: its unmerged iterations -- and `in_flight`, iterations it was assigned
        but had not reported rendered (a device that raised mid-pass) -- are lost and re-queued
        exactly once."""
        with self.lock:
            p = self.profiles[w]
            if not p.alive:
                return []
            p.alive = False
            lost = sorted(set(self.dev[w].unmerged) | set(in_flight or []))
            self.dev[w].unmerged = []
            self.requeue.extend(lost)
            self.requeue.sort()
            self.lost += len(lost)
            if not self.alive():
                raise SchedulerError("all devices failed")
            return lost

    def metrics(self) -> dict:
        return {"assigned": self.assigned, "merged": len(self.merged), "lost": self.lost,
                "devices": {w: {"alive": self.profiles[w].alive, "rendered": d.rendered, "sets": d.sets,
                                "merges": d.merges, "skips": d.skips, "rate_its_per_s": d.rate}
                            for w, d in self.dev.items()}}


class BatchScheduler:
    """Render iterations [it_begin, it_end) of a frame on several (simulated) devices.

    `make_device(worker)` returns a render context for one device: an object with
    render_pass(it_begin, it_end), framebuffer() -> int64 (P, 3) and clear() (a `Renderer`).
    Iteration sets are rendered as maximal runs of consecutive ids (one render_pass each)."""

    def __init__(self, make_device, profiles: list[WorkerProfile], cap: int = 64):
        self.make_device = make_device
        self.profiles = profiles
        self.cap = cap
        self.master = None
        self.master_lock = threading.Lock()
        self.ledger = None
        self.errors: list[BaseException] = []
        self.abort = threading.Event()  # set when the run cannot finish (every device failed)

    @staticmethod
    def _runs(its: list[int]):
        its = sorted(its)
        start = prev = its[0]
        for i in its[1:]:
            if i != prev + 1:
                yield start, prev + 1
                start = i
            prev = i
        yield start, prev + 1

    def _merge(self, w: int, dev):
        its = self.ledger.begin_merge(w)
        fb = dev.framebuffer()
        with self.master_lock:
            if self.master is None:
                self.master = np.zeros_like(fb)
            self.master += fb
            # recorded as merged before the local clear: if clear() raises, the failure path
            # must not re-queue iterations the master already holds
            self.ledger.end_merge(w, its)
        dev.clear()

    def _worker(self, prof: WorkerProfile):
        w = prof.worker
        in_flight: list[int] = []  # assigned, not yet reported rendered
        try:
            dev = self.make_device(w)
            try:
                while not self.ledger.done() and not self.abort.is_set():
                    if not self.ledger.profiles[w].alive:
                        return
                    its = self.ledger.assign_iteration_set(w)
                    if not its:
                        if self.ledger.dev[w].unmerged:
                            self._merge(w, dev)
                            continue
                        time.sleep(0.001)  # others still merging / may fail and re-queue
                        continue
                    in_flight = its
                    t = time.perf_counter()
                    for a, b in self._runs(its):
                        dev.render_pass(a, b)
                    dt = time.perf_counter() - t
                    if prof.speed < 1.0:  # simulated slower device
                        time.sleep(dt * (1.0 / prof.speed - 1.0))
                        dt = dt / prof.speed
                    self.ledger.rendered(w, its, max(dt, 1e-9))
                    in_flight = []
                    if prof.fail_after is not None and self.ledger.dev[w].rendered >= prof.fail_after:
                        self.ledger.fail(w)  # local framebuffer (unmerged work) is lost
                        dev.clear()
                        return
                    if self.ledger.should_merge(w):
                        self._merge(w, dev)
                if self.ledger.dev[w].unmerged and not self.abort.is_set():
                    self._merge(w, dev)
            finally:
                close = getattr(dev, "close", None)
                if close:
                    close()
        except BaseException as e:  # a real device error: fail the device, re-queue its work
            self.errors.append(e)
            try:
                self.ledger.fail(w, in_flight)
            except SchedulerError as e2:  # no device left to finish the range
                self.errors.append(e2)
                self.abort.set()

    def run(self, it_begin: int, it_end: int) -> np.ndarray:
        """Master int64 framebuffer holding every iteration of the range exactly once."""
        return self._run(it_begin, it_end)

    def _run(self, it_begin: int, it_end: int) -> np.ndarray:
        self.ledger = IterationLedger(it_begin, it_end, [WorkerProfile(p.worker, p.weight, True, p.speed,
                                                                        p.fail_after) for p in self.profiles],
                                      cap=self.cap)
        self.master = None
        self.errors = []
        self.abort.clear()
        threads = [threading.Thread(target=self._worker, args=(p,), daemon=True) for p in self.profiles]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if self.abort.is_set() or (self.errors and not self.ledger.done()):
            raise self.errors[-1] if self.errors else SchedulerError("render aborted")
        if not self.ledger.done():
            raise SchedulerError("not every iteration was merged")
        m = self.ledger
        assert m.assigned == len(m.merged) + m.lost, "conservation: assigned = merged + lost"
        return self.master
