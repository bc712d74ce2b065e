"""pytest plugin: run the reference's OWN test suite with the B200 kernels
behind its kernel seam (import swap, no reference file edited).

The reference selects its hot loops with ``_accel.get_kernels()``
(_accel.py:35-43), which imports ``sssrelight._kernels_nb`` when numba is
available. This plugin registers ``paper_2203_12339_b200.kernels_b200`` under
that module name before any reference module is imported, so every caller
(wavelets, transfer, lighting, runtime) binds ``_k`` to the GPU kernels, and
``test_kernels.py``'s ``knb`` (compared bitwise with the numpy twins) IS the
GPU module. Call counts per kernel are written to $SSS_SEAM_COUNTS at exit.

SSS_SEAM_MODULE overrides the swapped-in module (the CPU test of this
mechanism swaps in a call-counting wrapper of the numpy kernels).
"""

from __future__ import annotations

import collections
import importlib
import json
import os
import sys
import types

KERNELS = ("haar2d_fwd_batch", "haar2d_inv_batch", "cdf97_fwd_batch", "cdf97_inv_batch",
           "transfer_block", "bvh_any_hit", "csc_apply", "raster_fill")

COUNTS = collections.Counter()


def _counting(mod):
    wrapped = types.ModuleType("sssrelight._kernels_nb")
    for name in dir(mod):
        if not name.startswith("__"):
            setattr(wrapped, name, getattr(mod, name))

    def wrap(name, fn):
        def call(*a, **k):
            COUNTS[name] += 1
            return fn(*a, **k)
        call.__name__ = name
        return call

    for name in KERNELS:
        setattr(wrapped, name, wrap(name, getattr(mod, name)))
    wrapped.__wrapped_module__ = mod.__name__
    return wrapped


def _install():
    target = os.environ.get("SSS_SEAM_MODULE", "paper_2203_12339_b200.kernels_b200")
    mod = _counting(importlib.import_module(target))
    import sssrelight
    from sssrelight import _accel

    if not _accel.USE_NUMBA:
        raise RuntimeError("the seam swap replaces the numba module: numba must import")
    sys.modules["sssrelight._kernels_nb"] = mod
    sssrelight._kernels_nb = mod


def _install_api():
    """SSS_API_SWAP=1: the reference's public entry points replaced by the
    B200 API seam (paper_2203_12339_b200.api): runtime.Scene and
    transfer.precompute_compressed, looked up through the module by the
    reference's tests (rt.Scene(...), tr.precompute_compressed(...))."""
    from paper_2203_12339_b200 import api
    from sssrelight import runtime, transfer

    class Scene(api.Scene):
        def __init__(self, *a, **k):
            COUNTS["api.Scene"] += 1
            super().__init__(*a, **k)

    def precompute_compressed(*a, **k):
        COUNTS["api.precompute_compressed"] += 1
        return api.precompute_compressed(*a, **k)

    runtime.Scene = Scene
    transfer.precompute_compressed = precompute_compressed


_install()
if os.environ.get("SSS_API_SWAP") == "1":
    _install_api()


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("SSS_SEAM_COUNTS")
    if path:
        with open(path, "w") as fh:
            json.dump(dict(COUNTS), fh)
