"""Batch scheduler: ledger rules, conservation, and the
determinism-under-failure property -- the merged framebuffer equals the single-device one bit for
bit for any device count, speeds and failure schedule."""

import numpy as np
import pytest

from paper_1705_01263_b200.scheduler import BatchScheduler, IterationLedger, SchedulerError, WorkerProfile

P = 64


def _contrib(i):
    return np.random.default_rng(1000 + i).integers(0, 1 << 40, (P, 3))


class FakeDevice:
    """Deterministic stand-in for a render context: iteration i adds _contrib(i)."""

    def __init__(self):
        self.fb = np.zeros((P, 3), np.int64)

    def render_pass(self, a, b):
        for i in range(a, b):
            self.fb += _contrib(i)

    def framebuffer(self):
        return self.fb.copy()

    def clear(self):
        self.fb[:] = 0


def _expected(a, b):
    return sum((_contrib(i) for i in range(a, b)), np.zeros((P, 3), np.int64))


def test_assign_set_size_formula():
    # remaining 100 s at 2 it/s -> 100 iterations (cap raised to show the formula)
    led = IterationLedger(0, 1000, [WorkerProfile(0)], cap=1000)
    led.dev[0].rate = 2.0
    led.dev[0].rendered, led.dev[0].busy_s = 2, 1.0
    led.next = 800  # 200 remaining / 2 it/s = 100 s
    assert len(led.assign_iteration_set(0)) == 100
    led2 = IterationLedger(0, 1000, [WorkerProfile(0)])
    assert len(led2.assign_iteration_set(0)) == 64  # default cap bounds the loss on failure


def test_should_merge_rule():
    # unmerged 4, peer unmerged 9 and merging -> skip (4 < 4.5)
    led = IterationLedger(0, 100, [WorkerProfile(0), WorkerProfile(1)])
    led.dev[0].unmerged = list(range(4))
    led.dev[1].unmerged = list(range(10, 19))
    led.dev[1].merging = True
    assert led.should_merge(0) is False and led.dev[0].skips == 1
    led.dev[1].merging = False
    assert led.should_merge(0) is True


def test_failure_requeues_exactly_once():
    led = IterationLedger(0, 10, [WorkerProfile(0), WorkerProfile(1)], cap=4)
    s0 = led.assign_iteration_set(0)
    led.rendered(0, s0, 1.0)
    lost = led.fail(0)
    assert lost == sorted(s0) and led.lost == len(s0)
    again = led.assign_iteration_set(1)
    assert again[: len(s0)] == sorted(s0)
    with pytest.raises(SchedulerError):
        led.fail(1)  # all devices dead -> fatal


@pytest.mark.parametrize("n,speeds,fails", [
    (1, [1.0], [None]),
    (2, [1.0, 0.5], [None, None]),
    (4, [1.0, 0.7, 0.4, 1.0], [None, 5, None, 17]),
    (8, [1.0, 0.9, 0.8, 0.7, 0.6, 0.5, 0.4, 0.3], [None, 3, None, 11, None, None, 1, None]),
])
def test_batch_render_deterministic_under_failures(n, speeds, fails):
    profiles = [WorkerProfile(k, weight=speeds[k], speed=speeds[k], fail_after=fails[k]) for k in range(n)]
    sch = BatchScheduler(lambda w: FakeDevice(), profiles, cap=8)
    out = sch.run(0, 200)
    assert np.array_equal(out, _expected(0, 200))
    m = sch.ledger.metrics()
    assert m["merged"] == 200 and m["assigned"] == m["merged"] + m["lost"]
    assert m["lost"] == 0 or any(f is not None for f in fails)


@pytest.mark.gpu
def test_batch_render_on_gpu_matches_single_context(gpu):
    from paper_1705_01263_b200 import scenes
    from paper_1705_01263_b200.render import Renderer
    from paper_1705_01263_b200.scene import pack_scene

    packed = pack_scene(scenes.cornell())
    W, H = 64, 64

    def make(w):
        return Renderer(None, W, H, 4, packed=packed, pool_log2=14)

    with make(0) as r:
        r.render_pass(0, 48)
        ref = r.framebuffer()
    profiles = [WorkerProfile(0), WorkerProfile(1, weight=0.5, speed=0.5, fail_after=6), WorkerProfile(2)]
    out = BatchScheduler(make, profiles, cap=4).run(0, 48)
    assert np.array_equal(out, ref)


@pytest.mark.gpu
def test_cli_batch_with_failure_matches_single(gpu, tmp_path):
    from paper_1705_01263_b200 import cli
    from paper_1705_01263_b200.imagefiles import read_pfm

    a, b = str(tmp_path / "single"), str(tmp_path / "batch")
    assert cli.main(["render", "--config", "C1", "--res", "32x32", "--iterations", "12", "--out", a]) == 0
    assert cli.main(["render", "--config", "C1", "--res", "32x32", "--iterations", "12", "--out", b,
                     "--contexts-per-device", "3", "--fail", "1@2", "--metrics", str(tmp_path / "m.json")]) == 0
    assert (read_pfm(a + "_000012.pfm") == read_pfm(b + "_000012.pfm")).all()


class RaisingDevice(FakeDevice):
    """Raises inside render_pass after `after` iterations (a CUDA error / OOM mid-pass); the
    iterations it half-rendered stay in its local framebuffer and must never reach the master."""

    def __init__(self, after):
        super().__init__()
        self.after = after
        self.count = 0

    def render_pass(self, a, b):
        for i in range(a, b):
            if self.count >= self.after:
                raise RuntimeError("simulated device error")
            self.fb += _contrib(i)
            self.count += 1


@pytest.mark.timeout(60)
def test_device_error_requeues_in_flight_work():
    # worker 1 raises mid-pass: its assigned-but-unreported iterations are re-queued exactly once and
    # the other workers finish the range; the image equals the single-device one bit for bit
    class Slow(FakeDevice):  # keeps the healthy devices busy long enough for device 1 to fail
        def render_pass(self, a, b):
            import time

            time.sleep(0.002)
            super().render_pass(a, b)

    devs = {0: lambda: Slow(), 1: lambda: RaisingDevice(2), 2: lambda: Slow()}
    sch = BatchScheduler(lambda w: devs[w](), [WorkerProfile(k) for k in range(3)], cap=4)
    fb = sch.run(0, 1500)
    assert np.array_equal(fb, _expected(0, 1500))
    assert any(isinstance(e, RuntimeError) for e in sch.errors)
    assert not sch.ledger.profiles[1].alive


@pytest.mark.timeout(60)
def test_every_device_erroring_raises_instead_of_hanging():
    sch = BatchScheduler(lambda w: RaisingDevice(3), [WorkerProfile(k) for k in range(2)], cap=4)
    with pytest.raises((SchedulerError, RuntimeError)):
        sch.run(0, 100)
