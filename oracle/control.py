"""Draft-length control (paper Algorithm 1), restated.

ref:draft_control.py:17-28 (parameters, defaults l0=7, incre=2, mod=10,
limit=32), :49-69 (update rule), :72-108 (adaptive / fixed controllers).
"""

from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class AlgParams:
    l0: int = 7
    incre: int = 2
    mod: int = 10
    limit: int = 32


def alg1_update(l_draft: int, s: int, accepted, p: AlgParams) -> tuple[int, int]:
    """One Algorithm-1 step: (l, s) x accepted counts -> (l', s').

    ref:draft_control.py:49-69.  Grow by ``incre`` (clamped to ``limit``)
    when some sequence accepted its whole draft; otherwise shrink by
    ceil(l/mod) plus one more on consecutive shrinks, never below the
    largest accepted count or 1.
    """
    acc = [int(a) for a in accepted]
    if not acc:
        raise ValueError("need at least one accepted count")
    if any(a < 0 or a > l_draft for a in acc):
        raise ValueError("accepted count outside [0, l_draft]")
    if max(acc) == l_draft:
        return min(l_draft + p.incre, p.limit), 0
    shrunk = l_draft - math.ceil(l_draft / p.mod) - s
    return max([1, shrunk] + acc), 1


class AdaptiveLength:
    """ref:draft_control.py:72-88."""

    def __init__(self, params: AlgParams | None = None):
        self.params = params or AlgParams()
        self.l, self.s = self.params.l0, 0

    @property
    def length(self):
        return self.l

    @property
    def max_length(self):
        return self.params.limit

    def observe(self, accepted):
        if accepted:
            self.l, self.s = alg1_update(self.l, self.s, accepted, self.params)


class FixedLength:
    """ref:draft_control.py:91-108."""

    def __init__(self, k: int):
        self.k = k

    @property
    def length(self):
        return self.k

    @property
    def max_length(self):
        return self.k

    def observe(self, accepted):
        pass
