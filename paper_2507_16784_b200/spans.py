"""TokenSpan: half-open range of logical token indices (schema.py:36-57 contract)."""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class TokenSpan:
    start: int
    end: int

    def __post_init__(self):
        if not (0 <= self.start <= self.end):
            raise ValueError(f"bad span [{self.start}, {self.end})")

    def __len__(self) -> int:
        return self.end - self.start

    def contains(self, other: "TokenSpan") -> bool:
        return self.start <= other.start and other.end <= self.end

    def overlaps(self, other: "TokenSpan") -> bool:
        return self.start < other.end and other.start < self.end

    def shift(self, delta: int) -> "TokenSpan":
        return TokenSpan(self.start + delta, self.end + delta)
