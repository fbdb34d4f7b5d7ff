"""O(n^2)-pass tally by subroutine category (mirrors ``opcount.py:36-91``).

The B200 solver increments the tally at the same logical call sites as the
reference (``dual.py``, ``newton.py``, ``driver.py``), so ``RunReport.ops`` is
identical to the reference's whenever the control flow is — which makes the
op counts a cheap, exact check of control-flow parity.  Counting is host-side
bookkeeping only; device kernels never touch it.
"""

from __future__ import annotations

import os


class OpCounter:
    """Per-category pass counts with a category stack."""

    def __init__(self):
        self.by_category: dict[str, int] = {}
        self._stack: list[str] = []

    def reset(self):
        self.by_category.clear()
        self._stack.clear()

    def add(self, passes=1):
        key = self._stack[-1] if self._stack else "other"
        self.by_category[key] = self.by_category.get(key, 0) + passes

    def total(self):
        return sum(self.by_category.values())

    def snapshot(self):
        return dict(self.by_category)

    def category(self, name):
        return _Category(self._stack, name)


class _Category:
    """`with COUNTER.category(name):` — a plain context manager (the driver
    enters several per Newton step, on the host's critical path)."""

    __slots__ = ("_stack", "_name")

    def __init__(self, stack, name):
        self._stack, self._name = stack, name

    def __enter__(self):
        self._stack.append(self._name)

    def __exit__(self, *exc):
        self._stack.pop()
        return False


COUNTER = OpCounter()


def add(passes=1):
    COUNTER.add(passes)


def category(name):
    return COUNTER.category(name)


def reset():
    COUNTER.reset()


def snapshot():
    return COUNTER.snapshot()


def total():
    return COUNTER.total()


def deterministic():
    """``OTN_DETERMINISTIC=1`` (opcount.py:89-91).  The B200 kernels use fixed
    reduction trees and no floating-point atomics, so every run is
    bit-reproducible whether or not the variable is set."""
    return os.environ.get("OTN_DETERMINISTIC", "") == "1"
