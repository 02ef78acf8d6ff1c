"""The reference interval-algebra module's API (`memplan/intervals.py`)."""

from .ivset import Interval, IntervalSet, best_fit, intersect, subtract

__all__ = ["Interval", "IntervalSet", "best_fit", "intersect", "subtract"]
