"""Host-memory entry point for the rounded TT matrix-vector product.

The reference's public call is ``tt_round(tt_matvec(A, x), eps)`` on numpy-backed TTs
(reference tensor_train/core.py:327-338 and :353-389): operator and vector cores live in
host memory and so does the result. ``tt_matvec_round_host`` is that call for host (pinned)
cores, with the PCIe transfers overlapped with the device work instead of serialized
around it:

* uploads: every operator core is sent in slices along its leading rank index on a copy
  stream; the contraction of slice a (one GEMM + one permute into the product core) starts as
  soon as slice a has landed, while slice a + 1 is in flight;
* downloads: the left factor of the last truncated SVD (the largest output core) is formed in
  row chunks, each copied to the host while the next chunk is computed; earlier output cores go
  down as soon as they are final.

The arithmetic is the device path's (same kernels, same reduction order per element), so
the result equals ``tt_round(tt_matvec(A, x), eps)`` computed on device-resident inputs.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import linalg as L
from .core import TtShapeError, _chop, _rl_orthogonalize

__all__ = ["tt_matvec_round_host"]


def _pinned(t):
    t = torch.as_tensor(t, dtype=torch.float64)
    if t.device.type != "cpu":
        raise ValueError("host cores expected")
    t = t.contiguous()
    return t if t.is_pinned() else t.pin_memory()


def tt_matvec_round_host(A_cores, x_cores, eps, max_rank=None, out=None, slices=16, chunks=8):
    """Round(A x) for host-resident cores; returns the rounded cores as pinned host tensors.

    A_cores: dense operator cores (r0, n, m, r1); x_cores: vector cores (s0, m, s1) (numpy
    arrays or CPU tensors). ``out`` may hold pinned host tensors of the expected output shapes
    (reused across calls). The function returns after the downloads completed.
    """
    if eps <= 0:
        raise ValueError("eps must be positive")
    A_cores = [_pinned(G) for G in A_cores]
    x_cores = [_pinned(G) for G in x_cores]
    if len(A_cores) != len(x_cores) or not A_cores:
        raise TtShapeError("operator and vector must have the same number of cores")
    for k, (M, G) in enumerate(zip(A_cores, x_cores)):
        if M.dim() != 4 or G.dim() != 3 or M.shape[2] != G.shape[1]:
            raise TtShapeError(f"core {k}: operator {tuple(M.shape)} does not act on vector core {tuple(G.shape)}")
    d = len(A_cores)
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream()

    # ---- uploads (vector cores first, then operator cores slice by slice) and contractions
    xd = []
    with torch.cuda.stream(copy):
        for G in x_cores:
            xd.append(G.to("cuda", non_blocking=True))
    x_ready = torch.cuda.Event()
    x_ready.record(copy)
    comp.wait_event(x_ready)
    cores = []
    for M, G in zip(A_cores, x_cores):
        Ra, n, m, Rb = M.shape
        rc, _, rd = G.shape
        # Md is allocated on (owned by) the copy stream, so the caching allocator cannot hand it memory
        # that kernels still queued on the compute stream are reading; record_stream(comp) below then
        # keeps it alive until the contractions that read it have run.
        with torch.cuda.stream(copy):
            Md = L.empty(Ra, n, m, Rb)
        Y = L.empty(Ra * rc, n, Rb * rd)
        Yv = Y.view(Ra, rc, n, Rb, rd)
        xk = xd[len(cores)]
        step = max(1, -(-Ra // slices))
        for a0 in range(0, Ra, step):
            a1 = min(Ra, a0 + step)
            with torch.cuda.stream(copy):
                Md[a0:a1].copy_(M[a0:a1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            comp.wait_event(ev)
            for a in range(a0, a1):
                T = L.tdot(Md[a], xk, ([1], [1]), emulate=True)    # (i, b, c, d)
                L.permute(T, (2, 0, 1, 3), out=Yv[a])              # (c, i, b, d)
        Md.record_stream(comp)
        cores.append(Y)
    for t in xd:
        t.record_stream(comp)

    # ---- rounding (reference order), downloads overlapped with the last core formation
    host = [] if out is None else list(out)

    def host_buf(k, shape):
        if k < len(host) and tuple(host[k].shape) == tuple(shape) and host[k].is_pinned():
            return host[k]
        buf = torch.empty(shape, dtype=torch.float64).pin_memory()
        if k < len(host):
            host[k] = buf
        else:
            host.append(buf)
        return buf

    def download(k, dev):
        h = host_buf(k, tuple(dev.shape))
        ev = torch.cuda.Event()
        ev.record(comp)
        copy.wait_event(ev)
        with torch.cuda.stream(copy):
            h.copy_(dev, non_blocking=True)
        dev.record_stream(copy)
        return h

    if d == 1:
        download(0, cores[0])
    else:
        cores, _, f0 = _rl_orthogonalize(cores, svd0=True)
        total = float(L.nrm2(cores[0]).item())
        if total == 0.0:
            cores = [L.zeros(1, G.shape[1], 1) for G in cores]
            for k, G in enumerate(cores):
                download(k, G)
        else:
            delta = eps * total / np.sqrt(d - 1)
            for k in range(d - 1):
                r0, n, r1 = cores[k].shape
                f = f0 if (k == 0 and f0 is not None) else L.SVDFactors(cores[k].reshape(r0 * n, r1))
                keep = _chop(f.s_host(), delta, max_rank)
                rows = r0 * n
                Uk = L.empty(rows, keep)
                if k < d - 2 or not f.tall:
                    f.U_rows(keep, 0, rows, Uk)
                    download(k, Uk.view(r0, n, keep))
                else:  # the largest output core: row chunks, each sent down while the next is formed
                    h = host_buf(k, (r0, n, keep)).view(rows, keep)
                    cs = max(1, -(-rows // chunks))
                    for i0 in range(0, rows, cs):
                        i1 = min(rows, i0 + cs)
                        f.U_rows(keep, i0, i1, Uk[i0:i1])
                        ev = torch.cuda.Event()
                        ev.record(comp)
                        copy.wait_event(ev)
                        with torch.cuda.stream(copy):
                            h[i0:i1].copy_(Uk[i0:i1], non_blocking=True)
                    Uk.record_stream(copy)
                cores[k] = Uk.view(r0, n, keep)
                carry = f.SVt(keep)
                nxt = cores[k + 1]
                cores[k + 1] = L.gemm(carry, nxt.reshape(nxt.shape[0], -1), emulate=True).reshape(
                    keep, nxt.shape[1], nxt.shape[2])
            download(d - 1, cores[d - 1])
    done = torch.cuda.Event()
    done.record(copy)
    comp.wait_event(done)
    done.synchronize()
    return [host[k] for k in range(len(cores))]
