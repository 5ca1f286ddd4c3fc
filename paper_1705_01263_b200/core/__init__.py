"""Hot-path kernels (mirror of `lumenwave/core/__init__.py:9-27`).

`kernels` is always the sm_100a implementation; `COMPILED` is True.  The
reference's `load_interpreted()` returns its pure-Python kernel module; the
B200 build deliberately has no interpreted or CPU variant, so it raises.
"""

from paper_1705_01263_b200.core import kernels

COMPILED = bool(kernels.is_compiled())


def load_interpreted():
    raise RuntimeError(
        "paper_1705_01263_b200 has no interpreted kernel variant: every kernel runs on the GPU "
        "(the CPU restatement lives in oracle/ and is test infrastructure only)"
    )
