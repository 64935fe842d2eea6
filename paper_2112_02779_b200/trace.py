"""Optional NVTX ranges around the public entry points (SURVEY §5 "tracing").

Off by default (zero cost); ``RK_NVTX=1`` in the environment, or
``trace.enable()``, wraps each decorated call in ``torch.cuda.nvtx`` push/pop
so an ncu/nsys capture can be filtered to one API call
(``ncu --nvtx --nvtx-include "rk.register_batch/"``).
"""

from __future__ import annotations

import functools
import os

_enabled = os.environ.get("RK_NVTX", "") not in ("", "0")


def enable(on: bool = True) -> None:
    global _enabled
    _enabled = bool(on)


def enabled() -> bool:
    return _enabled


def nvtx(name: str):
    """Decorator: an NVTX range named ``rk.<name>`` around the call when enabled."""
    def wrap(fn):
        @functools.wraps(fn)
        def inner(*args, **kwargs):
            if not _enabled:
                return fn(*args, **kwargs)
            import torch
            torch.cuda.nvtx.range_push(f"rk.{name}")
            try:
                return fn(*args, **kwargs)
            finally:
                torch.cuda.nvtx.range_pop()
        return inner
    return wrap
