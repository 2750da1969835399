"""Functions of physical points (and of grid indices) at the API boundary.

The reference calls source terms, analytic solutions and Dirichlet face data with numpy (N, 3)
arrays of physical points (reference driver.py:80-149, assembly.py:163-170, 307-384) and cross
oracles with numpy (N, d) index arrays (tensor_train/cross.py:23-42). Here those functions are
evaluated on the device: the built-ins are ``PointFn`` objects that the kernels recognise by id
(source terms inside geo_kernel, analytic solutions inside l1err_kernel) and that also run as torch
code on CUDA tensors. Called with numpy, a ``PointFn`` behaves exactly like the reference's numpy
lambda, so ``SOURCES["one"](pts)`` works as in the reference.

Any other callable a user passes is a reference-style numpy function: ``on_device`` bridges it
(points or indices copied to the host, the values back to the device). That bridge is the API
compatibility path for user code; the named sources and solutions never take it.
"""

from __future__ import annotations

import math

import numpy as np
import torch

__all__ = ["PointFn", "on_device", "index_fn_on_device"]


class PointFn:
    """A function of (N, 3) physical points with a numpy and a torch implementation.

    ``source_id`` / ``analytic_id`` (+ ``params``) name the in-kernel version (iga.cu source_fn /
    exact_fn) when there is one."""

    def __init__(self, np_fn, torch_fn, name=None, source_id=None, analytic_id=None, params=()):
        self.np_fn = np_fn
        self.torch_fn = torch_fn
        self.name = name
        self.source_id = source_id
        self.analytic_id = analytic_id
        self.params = tuple(float(p) for p in params)

    def __call__(self, pts):
        if isinstance(pts, torch.Tensor):
            return self.torch_fn(pts)
        return self.np_fn(np.asarray(pts, dtype=float))

    def __repr__(self):
        return f"PointFn({self.name!r})"


def on_device(fn):
    """torch (N, 3) CUDA points -> (N,) CUDA values for any function of points: a PointFn's torch path,
    a function marked ``_ttb_device`` as is, any other callable through the numpy bridge."""
    if isinstance(fn, PointFn):
        return fn.torch_fn
    if getattr(fn, "_ttb_device", False):
        return fn

    def bridge(pts):
        v = fn(pts.detach().cpu().numpy())
        if isinstance(v, torch.Tensor):
            return v.to(device=pts.device, dtype=torch.float64).reshape(-1)
        v = np.asarray(v, dtype=np.float64)
        if v.ndim == 0:
            v = np.full(pts.shape[0], float(v))
        return torch.as_tensor(v.reshape(-1), device=pts.device)

    return bridge


def index_fn_on_device(fn):
    """The same bridge for cross-oracle functions of int64 multi-indices."""
    if getattr(fn, "_ttb_device", False):
        return fn

    def bridge(idx):
        v = fn(idx.detach().cpu().numpy())
        if isinstance(v, torch.Tensor):
            return v.to(device=idx.device, dtype=torch.float64).reshape(-1)
        return torch.as_tensor(np.asarray(v, dtype=np.float64).reshape(-1), device=idx.device)

    return bridge


def device_marked(fn):
    """Mark a function as taking/returning CUDA tensors (internal oracles)."""
    fn._ttb_device = True
    return fn


# ---------------------------------------------------------------------------
# built-in source terms (reference driver.py:80-98 + the BASELINE exp_sines)

def _np_s3(p):
    return np.sin(np.pi * p[:, 0]) * np.sin(np.pi * p[:, 1]) * np.sin(np.pi * p[:, 2])


def _t_s3(p):
    return torch.sin(math.pi * p[:, 0]) * torch.sin(math.pi * p[:, 1]) * torch.sin(math.pi * p[:, 2])


def _np_exp_sines_source(p):
    e = np.exp(p.sum(1))
    s = np.sin(np.pi * p)
    c = np.cos(np.pi * p)
    S = s[:, 0] * s[:, 1] * s[:, 2]
    mix = c[:, 0] * s[:, 1] * s[:, 2] + s[:, 0] * c[:, 1] * s[:, 2] + s[:, 0] * s[:, 1] * c[:, 2]
    return -e * ((3.0 - 3.0 * np.pi ** 2) * S + 2.0 * np.pi * mix)


def _t_exp_sines_source(p):
    e = torch.exp(p.sum(1))
    s = torch.sin(math.pi * p)
    c = torch.cos(math.pi * p)
    S = s[:, 0] * s[:, 1] * s[:, 2]
    mix = c[:, 0] * s[:, 1] * s[:, 2] + s[:, 0] * c[:, 1] * s[:, 2] + s[:, 0] * s[:, 1] * c[:, 2]
    return -e * ((3.0 - 3.0 * math.pi ** 2) * S + 2.0 * math.pi * mix)


def builtin_sources(source_ids):
    fns = {
        "zero": (lambda p: np.zeros(p.shape[0]), lambda p: torch.zeros(p.shape[0], dtype=p.dtype, device=p.device)),
        "one": (lambda p: np.ones(p.shape[0]), lambda p: torch.ones(p.shape[0], dtype=p.dtype, device=p.device)),
        "sin_pi_xy": (lambda p: np.sin(np.pi * p[:, 0]) * np.sin(np.pi * p[:, 1]),
                      lambda p: torch.sin(math.pi * p[:, 0]) * torch.sin(math.pi * p[:, 1])),
        "sin_pi_xyz": (_np_s3, _t_s3),
        "manufactured_sines": (lambda p: 3.0 * np.pi ** 2 * _np_s3(p), lambda p: 3.0 * math.pi ** 2 * _t_s3(p)),
        "exp_sines": (_np_exp_sines_source, _t_exp_sines_source),
    }
    return {name: PointFn(*fns[name], name=name, source_id=sid) for name, sid in source_ids.items()}
