"""The reference dynamic-reuse module's API (`memplan/reuse.py`); the
reusable spaces are computed by K8 on the device (`api.reusable_spaces`)."""

from .api import compute_reusable_space, derive_reuse_map, group_dynamic
from .plan_types import ReuseEntry, ReuseMap

__all__ = ["ReuseEntry", "ReuseMap", "compute_reusable_space", "derive_reuse_map", "group_dynamic"]
