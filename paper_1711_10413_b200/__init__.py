"""B200-native implicit data-sharing runtime for OpenMP generic-mode target
regions (arXiv 1711.10413).

The product is ``_build/libompds_b200.so`` (C ABI: ``include/ompds.h``):
sm_100a generic-mode kernels with the data-sharing runtime inlined
(``csrc/ompds_device.cuh``), the frame-layout descriptor builder and the
occupancy model.  This package is the host-side mirror of the reference's
interfaces over that ABI:

* :mod:`.runtime`   -- ``TeamRuntime`` (DeviceRuntime.h), executed on the GPU
* :mod:`.layout`    -- ``DepotSlot`` / ``DepotLayout`` / ``FrameGroup`` builder
* :mod:`.occupancy` -- the occupancy model + a B200 row
* :mod:`.regions`   -- generic-mode region launches (configs 1, 2, 4, 5)
"""
from . import _lib  # noqa: F401

__all__ = ["runtime", "layout", "occupancy", "regions", "build"]
