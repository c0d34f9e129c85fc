"""threading.hpp:9-10: set_num_threads / num_threads.  The reference's worker
threads run its CPU projector; here the compute is on the GPU and the host
threads that remain are the forward-schedule planner's (RK_PLAN_THREADS, read
at each planning) — results never depend on the count, as in the reference
(threading.hpp:12-15)."""
from __future__ import annotations

import os

from .errors import ValidationError


def set_num_threads(n: int) -> None:
    """threading.cpp:24-27 (same validation)."""
    n = int(n)
    if n < 1:
        raise ValidationError(f"thread count must be >= 1, got {n}")
    os.environ["RK_PLAN_THREADS"] = str(n)


def num_threads() -> int:
    v = os.environ.get("RK_PLAN_THREADS")
    try:
        n = int(v) if v else 0
    except ValueError:
        raise ValidationError(f"RK_PLAN_THREADS={v!r} is not an integer") from None
    return n if n > 0 else (os.cpu_count() or 1)
