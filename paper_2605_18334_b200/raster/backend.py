"""Kernel selection (mirror of reference raster/backend.py:16-43).

The reference picks between its Cython and NumPy blend kernels.  This build
has exactly one implementation -- the sm_100a kernels in libssg_b200.so --
so the selector only validates the name for call-site compatibility: None
or "cuda" are accepted (also via the SKEWSPLAT_BACKEND environment variable),
anything else raises ValueError like the reference does for unknown names
(backend.py:32-34).  There is no CPU fallback.
"""

from __future__ import annotations

import os

from .. import _native

_NAMES = ("cuda",)


def active_backend(override: str | None = None) -> str:
    name = override or os.environ.get("SKEWSPLAT_BACKEND")
    if name is not None and name not in _NAMES:
        raise ValueError(f"unknown backend {name!r}; expected one of {_NAMES}")
    _native.lib()  # fail loudly when the extension is missing
    return "cuda"


def kernels(override: str | None = None):
    """Module exposing forward_tiles / backward_tiles (reference
    backend.py:41-43): the sm_100a plugin module, whose interface is the
    reference _core's (forward_tiles, backward_tiles, erf_probe,
    set_num_threads, get_max_threads, KERNELS)."""
    active_backend(override)
    from .. import plugin
    return plugin
