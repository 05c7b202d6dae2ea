"""Deluxe scaling (reference scaling.py), computed by csrc/globs.cu."""

from .engine import DeviceScaling


class ScalingSet:
    """Per-glob deluxe families aligned with the GlobSet (scaling.py:36-44)."""

    def __init__(self, globs, device_scaling):
        self.globs = globs
        self.device = device_scaling

    def of(self, glob):
        return self.device.family(self.globs.index(glob))


def build_scaling(globs, ops):
    """Reference signature (scaling.py:47-57)."""
    ls = ops[0].ls
    if ls.globs is not globs:
        raise ValueError("ops were built for a different GlobSet")
    return ScalingSet(globs, DeviceScaling(ls))


__all__ = ["ScalingSet", "build_scaling"]
