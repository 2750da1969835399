"""Host-memory entry point: same result as the device-resident call, transfers overlapped."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _instance(rng, n, d, R, r):
    Rs = [1] + [R] * (d - 1) + [1]
    rs = [1] + [r] * (d - 1) + [1]
    A = [rng.standard_normal((Rs[k], n, n, Rs[k + 1])) / np.sqrt(Rs[k]) for k in range(d)]
    x = [rng.standard_normal((rs[k], n, rs[k + 1])) / np.sqrt(rs[k]) for k in range(d)]
    return A, x


@pytest.mark.parametrize("n,d,R,r,eps", [(48, 3, 4, 6, 1e-8), (40, 2, 3, 5, 1e-10), (24, 4, 3, 4, 1e-6),
                                         (64, 3, 5, 7, 1e-2)])
def test_host_matches_device(n, d, R, r, eps):
    from paper_2509_13224_b200.tensor_train import TtMatrix, TtTensor, tt_matvec, tt_matvec_round_host, tt_round
    rng = np.random.default_rng(n + d)
    A, x = _instance(rng, n, d, R, r)
    ref = tt_round(tt_matvec(TtMatrix(A), TtTensor(x)), eps)
    got = tt_matvec_round_host(A, x, eps, slices=3, chunks=5)
    assert [tuple(g.shape) for g in got] == [tuple(G.shape) for G in ref.cores]
    assert all(g.is_pinned() for g in got)
    full = TtTensor(got).full()
    want = ref.full()
    assert np.abs(full - want).max() <= 1e-13 * np.abs(want).max()
    # reuse of the output buffers
    got2 = tt_matvec_round_host(A, x, eps, out=got)
    assert all(a.data_ptr() == b.data_ptr() for a, b in zip(got, got2))
    assert np.abs(TtTensor(got2).full() - want).max() <= 1e-13 * np.abs(want).max()


def test_host_zero_and_errors():
    from paper_2509_13224_b200.tensor_train import TtShapeError, tt_matvec_round_host
    A = [np.zeros((1, 5, 5, 2)), np.zeros((2, 5, 5, 1))]
    x = [np.ones((1, 5, 3)), np.ones((3, 5, 1))]
    got = tt_matvec_round_host(A, x, 1e-8)
    assert [tuple(g.shape) for g in got] == [(1, 5, 1), (1, 5, 1)] and all(float(g.abs().max()) == 0 for g in got)
    with pytest.raises(TtShapeError):
        tt_matvec_round_host(A, [np.ones((1, 4, 3)), np.ones((3, 5, 1))], 1e-8)
    with pytest.raises(ValueError):
        tt_matvec_round_host(A, x, 0.0)


def test_host_matches_device_at_scale(monkeypatch):
    """The benchmarked host path at n=512 (every large-scale route on, pageable numpy inputs staged through
    the pinned ring in 32 MB chunks, uploads racing the contractions) against the device-resident call:
    guards the copy-stream ordering that tiny shapes cannot expose (host.py upload race)."""
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200.tensor_train import TtMatrix, TtTensor, tt_matvec, tt_matvec_round_host, tt_round
    from paper_2509_13224_b200.tensor_train import host as H
    from paper_2509_13224_b200.workloads import matvec_round_instance_np
    monkeypatch.setattr(L, "_CHOLQR2_MIN_M", 1 << 18)
    monkeypatch.setattr(L, "_GRAM_MIN_M", 1 << 18)
    A, x = matvec_round_instance_np(512, 16, 64, 3, 0)
    ref = tt_round(tt_matvec(TtMatrix(A), TtTensor(x)), 1e-8)
    got = tt_matvec_round_host(A, x, 1e-8)
    assert not any(torch.as_tensor(G).is_pinned() for G in A)
    assert [tuple(g.shape) for g in got] == [tuple(G.shape) for G in ref.cores]
    for g, G in zip(got, ref.cores):
        assert torch.equal(g, G.cpu()), "host path must give the device path's bits"
    # pinned inputs take the direct-DMA path: same bits again
    got2 = tt_matvec_round_host([torch.as_tensor(G).pin_memory() for G in A], [torch.as_tensor(G).pin_memory() for G in x],
                                1e-8)
    assert all(torch.equal(a, b) for a, b in zip(got, got2))
    assert H._STAGE_BYTES * H._STAGE_N < 512 ** 2 * 16 * 16 * 8
    # a stream of products (wait=False): the next product is issued while the previous one's downloads are
    # in flight; every result, read after its event, has the same bits
    x2 = [G * 0.5 for G in x]
    first = tt_matvec_round_host(A, x, 1e-8, wait=False)
    second = tt_matvec_round_host(A, x2, 1e-8, wait=False)
    first[1].synchronize()
    assert all(torch.equal(a, b) for a, b in zip(got, first[0]))
    second[1].synchronize()
    ref2 = tt_round(tt_matvec(TtMatrix(A), TtTensor(x2)), 1e-8)
    for g, G in zip(second[0], ref2.cores):
        assert torch.equal(g, G.cpu())


def test_host_path_benchmark_shape_class_early_carry(monkeypatch):
    """The benchmark's shape class (square first unfolding, square last core; product ranks 512 over mode size 512):
    the host path uploads the last and first operator cores before the middle one and carries the last core
    into the middle one slab by slab under the uploads, then takes the one-pass certified rounding. Same bits as
    the device-resident call."""
    from paper_2509_13224_b200 import linalg as L
    from paper_2509_13224_b200.tensor_train import TtMatrix, TtTensor, tt_matvec, tt_matvec_round_host, tt_round
    from paper_2509_13224_b200.workloads import matvec_round_instance_np
    monkeypatch.setattr(L, "_CHOLQR2_MIN_M", 1 << 18)
    monkeypatch.setattr(L, "_GRAM_MIN_M", 1 << 18)
    calls = []
    spec = L.fullrank_speculative_3core
    monkeypatch.setattr(L, "fullrank_speculative_3core", lambda *a, **k: calls.append(spec(*a, **k)) or calls[-1])
    A, x = matvec_round_instance_np(512, 8, 64, 3, 0)
    ref = tt_round(tt_matvec(TtMatrix(A), TtTensor(x)), 1e-8)
    got = tt_matvec_round_host(A, x, 1e-8)
    assert len(calls) == 2 and all(c is not None for c in calls), "one-pass certified rounding on both paths"
    assert [tuple(g.shape) for g in got] == [tuple(G.shape) for G in ref.cores]
    for g, G in zip(got, ref.cores):
        assert torch.equal(g, G.cpu()), "host path must give the device path's bits"
