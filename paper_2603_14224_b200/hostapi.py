"""Host-array face of the drop-in API: the reference's calling convention over the GPU
implementation in :mod:`paper_2603_14224_b200.api`.

The reference (``sikv``, numpy) takes array-likes and returns numpy arrays and frozen
dataclasses holding numpy arrays.  :mod:`.api` keeps every array on the GPU (torch CUDA
tensors) so calls chain without copies.  This module wraps each public name of :mod:`.api`:

* arguments: host views are unwrapped to the device objects they stand for (numpy inputs are
  uploaded by the API functions themselves);
* results: CUDA tensors come back as numpy arrays, dataclass instances as :class:`HostView`
  proxies whose array attributes and method results are numpy as well, while the device
  object stays inside (so ``score_tokens(build_lut(q, cb), codes)`` still runs on the GPU).

``paper_2603_14224_b200/compat/sikv`` re-exports this module under the reference's package
name, so the reference's own test suites import it unmodified (tools/run_reference_suites.py).
"""

from __future__ import annotations

import dataclasses
import functools

import torch

from . import api as _api


def to_host(x):
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    if isinstance(x, HostView):
        return x
    if dataclasses.is_dataclass(x) and not isinstance(x, type) and type(x).__module__ == _api.__name__:
        if isinstance(x, (_api.QuantConfig, _api.CacheConfig, _api.OpCounters, _api.MemoryReport,
                          _api.ErrorReport)):
            return x                       # scalar-only records: already host objects
        return HostView(x)
    if isinstance(x, tuple):
        return tuple(to_host(v) for v in x)
    if isinstance(x, list):
        return [to_host(v) for v in x]
    return x


def to_device(x):
    if isinstance(x, HostView):
        return object.__getattribute__(x, "_obj")
    if isinstance(x, tuple):
        return tuple(to_device(v) for v in x)
    if isinstance(x, list):
        return [to_device(v) for v in x]
    if isinstance(x, dict):
        return {k: to_device(v) for k, v in x.items()}
    return x


def _wrap(fn):
    @functools.wraps(fn)
    def call(*args, **kwargs):
        return to_host(fn(*to_device(args), **to_device(kwargs)))
    return call


class HostView:
    """A device object seen from the host: array attributes as numpy, methods wrapped."""

    __slots__ = ("_obj",)

    def __init__(self, obj):
        object.__setattr__(self, "_obj", obj)

    def __getattr__(self, name):
        v = getattr(object.__getattribute__(self, "_obj"), name)
        if callable(v) and not isinstance(v, (type, torch.Tensor)):
            return _wrap(v)
        return to_host(v)

    def __setattr__(self, name, value):
        setattr(object.__getattribute__(self, "_obj"), name, to_device(value))

    def __len__(self):
        return len(object.__getattribute__(self, "_obj"))

    def __repr__(self):
        return f"HostView({object.__getattribute__(self, '_obj')!r})"


class _HostClass:
    """A dataclass of :mod:`.api` called from the host: construction and class methods return
    host views; ``isinstance`` checks see through to the device class."""

    def __init__(self, cls):
        self._cls = cls
        functools.update_wrapper(self, cls, updated=())

    def __call__(self, *args, **kwargs):
        return to_host(self._cls(*to_device(args), **to_device(kwargs)))

    def __getattr__(self, name):
        v = getattr(self._cls, name)
        return _wrap(v) if callable(v) and not isinstance(v, type) else v

    def __instancecheck__(self, obj):
        return isinstance(to_device(obj), self._cls)


_CLASSES = ("AttentionOutput", "Codebook", "LookupTable", "NormalizationState", "QuantizedTensor",
            "SelfIndexingCache", "SignCodeMatrix", "TokenSelection")
_PLAIN = ("CacheConfig", "QuantConfig", "OpCounters", "MemoryReport", "ErrorReport", "collect", "tally",
          "DEFAULT_POOL_WIDTH")


def _export():
    g = globals()
    import paper_2603_14224_b200 as pkg
    for name in pkg.__all__:
        obj = getattr(_api, name)
        if name in _CLASSES:
            g[name] = _HostClass(obj)
        elif name in _PLAIN or isinstance(obj, type):
            g[name] = obj
        else:
            g[name] = _wrap(obj)
    for name in _PLAIN:
        if hasattr(_api, name):
            g[name] = getattr(_api, name)
    return list(pkg.__all__)


__all__ = _export()
